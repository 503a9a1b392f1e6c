"""Rebuild profiles/r01_final.md and the numbers tables in DESIGN.md / BASELINE.md from one
`scripts/gpu_final.sh <tag>` run (its bench JSON lines, ncu launch list and full capture), and
summarise the traffic probes into profiles/traffic_<cfg>.json.

    python scripts/refresh_docs.py r01i
"""
import glob, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out = os.path.join(ROOT, "gpurun_out", tag)
os.chdir(ROOT)
for c in ("C2", "C3", "C5", "S1"):
    if os.path.exists(f"gpurun_out/traffic_{c}.csv"):
        subprocess.run([sys.executable, "scripts/traffic_probe.py", "--summarise", f"gpurun_out/traffic_{c}.csv",
                        "--config", c], capture_output=True)
fs = [f"{out}/bench.json"] + sorted(f for f in glob.glob(f"{out}/bench_*.json") if "reference" not in f)
R = {}
for f in fs:
    j = json.loads(open(f).read().strip().splitlines()[-1])
    R[j["config"]["workload"][:2]] = j
ncu = subprocess.run([sys.executable, "scripts/ncu_summary.py", f"{out}/launches.csv", f"{out}/prof.ncu-rep"],
                     capture_output=True, text=True).stdout
pyt = [l for l in open(f"{out}/pytest_gpu.log") if "passed" in l]
smoke = open(f"{out}/smoke.log").readline().strip()
L = [f"# Round 1 — round-end measurement of every config (session 3, final: gpurun call {tag})", "",
     f"`bash scripts/gpu_final.sh {tag}`: {pyt[-1].strip() if pyt else 'pytest: see log'}; {smoke}.",
     "Session-3 start (commit f990a6b, call r01f): C1 60,534 / C2 13,604 / C3 1,225 / C4 805,664 / C5 1,290 / "
     "S1 3,227 particle-steps/s.", "", "## bench.py lines (N = 1, CUDA-graph launch)", "",
     "| config | particle-steps/s | e2e | ms/step | dominant kernel | bound | roofline frac | all-GEMM useful TF/s | update HBM frac | clocks |",
     "|---|---|---|---|---|---|---|---|---|---|"]
order = ["C1", "C2", "C3", "C4", "C5", "S1"]
for c in order:
    j = R[c]; r = j["roofline"]
    L.append(f"| {c} | {j['value']:.1f} | {j['e2e']['value']:.1f} | {j['ms_per_step']:.3f} | {r['kernel']} | {r['bound']} | "
             f"{r['frac']:.3f} | {r.get('all_gemm_tflops', 0):.1f} | {r.get('svgd_update_hbm_frac', 0):.2f} | "
             f"{j['clocks']['sm_mhz']:.0f} MHz {j['clocks']['reasons']} |")
L += ["", "## Per-class phase times (ms/step, profiled eager pass, CUDA events per class)", ""]
for c in order:
    j = R[c]
    L.append(f"- {c}: " + ", ".join(f"{k} {v['ms_per_step']:.3f}" for k, v in j["phases"].items()))
L += ["", "## Non-GEMM passes against the measured HBM peak (`roofline.hbm_passes`)", ""]
for c in order:
    hp = R[c]["roofline"].get("hbm_passes", {})
    L.append(f"- {c}: " + ", ".join(f"{k} {v['gbs']:.0f} GB/s ({v['frac']:.2f})" for k, v in hp.items()))
L += ["", "## Default bench line (C2)", "", "```json", open(f"{out}/bench.json").read().strip(), "```", "",
      "## Reference arm (`bench.py --impl reference`: the fp64 oracle on the host cores)", "", "```json",
      open(f"{out}/bench_reference.json").read().strip(), "```", "", ncu]
open("profiles/r01_final.md", "w").write("\n".join(L) + "\n")

lab = {"C2": "(L2-resident)", "C3": "(ALU-bound at n_ℓ = 64)", "C4": "(L2, ALU)", "C5": "", "S1": "(ALU-bound at n_ℓ = 64)"}
rows = []
for c in order:
    j = R[c]; r = j["roofline"]; cpu = j.get("cpu_baseline", {}).get("value")
    gem = "launch-bound" if c == "C1" else ("latency / ALU" if c == "C4" else
                                           f"{100 * r['frac']:.0f} % / {100 * r.get('all_gemm_tflops', 0) / r['peak']:.0f} %")
    upd = "— (L2)" if c == "C1" else f"{100 * r.get('svgd_update_hbm_frac', 0):.0f} % {lab[c]}".strip()
    rows.append(f"| {c} | 1 | {j['value']:,.0f} | {j['param_updates_per_s']:.1e} | {j['e2e']['value']:,.0f} | {upd} | {gem} | "
                f"{('%.1f (all host cores, bounded sample)' % cpu) if cpu else '—'} |")
s = open("BASELINE.md").read()
a = s.index("| C1 | 1 |"); b = s.index("\n\nThe GEMM peak is")
s = s[:a] + "\n".join(rows) + s[b:]
import re
s = re.sub(r"\(gpurun call r01\w+, session 3;", f"(gpurun call {tag}, session 3;", s)
open("BASELINE.md", "w").write(s)

names = {"C1": "C1 4 × 1-32-32-1, B 256", "C2": "C2 16 × 2-256x4-1, B 8192", "C3": "C3 64 × 3-1024x4-1, B 8192",
         "C4": "C4 256 × 1-64x3-1, B 128", "C5": "C5 8 × 2-2048x6-1, B 1024", "S1": "S1 64 × 3-512x5-1, B 8192"}
rows = []
for c in order:
    j = R[c]; r = j["roofline"]
    dom = "launch-bound" if c == "C1" else r["kernel"].replace("gemm3xtf32 (", "").replace("_gemm)", " GEMM")
    fr = "—" if c == "C1" else f"{r['frac']:.2f} ({r['bound']})"
    tf = "—" if c in ("C1", "C4") else f"{r.get('all_gemm_tflops', 0):.1f}"
    ms = f"{j['ms_per_step']:.3f}" if j["ms_per_step"] < 10 else f"{j['ms_per_step']:.1f}"
    rows.append(f"| {names[c]} | {ms} | {j['value']:,.0f} | {j['e2e']['value']:,.0f} | {dom} | {fr} | {tf} |")
s = open("DESIGN.md").read()
a = s.index("| C1 4 × 1-32-32-1, B 256 |"); b = s.index("\n\nHBM-bound passes against")
s = s[:a] + "\n".join(rows) + s[b:]
s = re.sub(r"`profiles/r01_final.md`, gpurun call r01\w+;", f"`profiles/r01_final.md`, gpurun call {tag};", s)
st = {c: R[c]["value"] for c in order}
base = {"C2": 13604, "C3": 1225, "C4": 805664, "C5": 1290, "S1": 3227}
gains = ", ".join(f"{c} {100 * (st[c] / base[c] - 1):+.0f}%" for c in ("C2", "C3", "C4", "C5", "S1"))
s = re.sub(r"Session-3 gains \(r01f → r01\w+\): [^\n]*\n[^\n]*\.", f"Session-3 gains (r01f → {tag}): {gains}.", s)
open("DESIGN.md", "w").write(s)
print("\n".join(rows))
print(gains)
