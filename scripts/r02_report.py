"""Summarise one `scripts/gpu_final.sh <tag>` run into profiles/r02_final.md (bench lines of every config,
phases, HBM passes, the default S1 line and the reference arm verbatim, the ncu launch list and full
capture) and refresh profiles/traffic_<cfg>.json from its traffic probes.

    python scripts/r02_report.py r02b
"""
import glob, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out = os.path.join(ROOT, "gpurun_out", tag)
os.chdir(ROOT)
for c in ("C2", "C3", "C4", "C5", "S1"):
    if os.path.exists(f"gpurun_out/traffic_{c}.csv"):
        subprocess.run([sys.executable, "scripts/traffic_probe.py", "--summarise", f"gpurun_out/traffic_{c}.csv",
                        "--config", c], capture_output=True)
R = {}
for f in [f"{out}/bench.json"] + sorted(glob.glob(f"{out}/bench_C*.json")):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    R[j["config"]["workload"].split(":")[0]] = j
ncu = subprocess.run([sys.executable, "scripts/ncu_summary.py", f"{out}/launches.csv", f"{out}/prof.ncu-rep"],
                     capture_output=True, text=True).stdout
pyt = [l for l in open(f"{out}/pytest_gpu.log") if "passed" in l]
smoke = open(f"{out}/smoke.log").readline().strip()
order = [c for c in ("C1", "C2", "C3", "C4", "C5", "C5b", "S1") if c in R]
L = [f"# Round 2 — round-end measurement of every config (gpurun call {tag})", "",
     f"`bash scripts/gpu_final.sh {tag}`: {pyt[-1].strip() if pyt else 'pytest: see log'}; {smoke}.", "",
     "## bench.py lines (N = 1, CUDA-graph launch)", "",
     "| config | particle-steps/s | param-updates/s | e2e | ms/step | dominant kernel | bound | roofline frac | "
     "all-GEMM useful TF/s | a7 / a10 HBM frac | clocks |",
     "|---|---|---|---|---|---|---|---|---|---|---|"]
for c in order:
    j = R[c]; r = j["roofline"]; hp = r.get("hbm_passes", {})
    a7 = hp.get("distances", {}).get("frac", 0); a10 = hp.get("svgd_update", {}).get("frac", 0)
    L.append(f"| {c} | {j['value']:,.1f} | {j['param_updates_per_s']:.2e} | {j['e2e']['value']:,.1f} | "
             f"{j['ms_per_step']:.4f} | {r['kernel']} | {r['bound']} | {r['frac']:.3f} | "
             f"{r.get('all_gemm_tflops', 0):.1f} | {a7:.2f} / {a10:.2f} | "
             f"{j['clocks']['sm_mhz']:.0f} MHz {j['clocks']['reasons']} |")
L += ["", "## Per-class phase times (ms/step, profiled eager pass, CUDA events per class)", ""]
for c in order:
    L.append(f"- {c}: " + ", ".join(f"{k} {v['ms_per_step']:.4f}" for k, v in R[c]["phases"].items()))
L += ["", "## Non-GEMM passes against the measured HBM peak (`roofline.hbm_passes`)", ""]
for c in order:
    hp = R[c]["roofline"].get("hbm_passes", {})
    L.append(f"- {c}: " + ", ".join(f"{k} {v['gbs']:.0f} GB/s ({v['frac']:.2f})" for k, v in hp.items()))
L += ["", "## Default bench line (S1)", "", "```json", open(f"{out}/bench.json").read().strip(), "```", "",
      "## Reference arm (`bench.py --impl reference`: the fp64 oracle on the host cores, bounded sample)", "",
      "```json", open(f"{out}/bench_reference.json").read().strip(), "```", "", ncu]
open("profiles/r02_final.md", "w").write("\n".join(L) + "\n")
print("\n".join(L[:20]))

# rows for the BASELINE.md results table and DESIGN.md §12 (pasted by hand)
print("\n-- BASELINE.md rows --")
for c in order:
    j = R[c]; r = j["roofline"]; hp = r.get("hbm_passes", {})
    a7 = hp.get("distances", {}).get("frac", 0); a10 = hp.get("svgd_update", {}).get("frac", 0)
    tens = r["bound"] == "tensor" and r["frac"] > 0.01
    print(f"| {c} | 1 | {j['value']:,.0f} | {j['param_updates_per_s']:.1e} | {j['e2e']['value']:,.0f} | "
          f"{100 * a7:.0f} % / {100 * a10:.0f} % | {str(round(100 * r['frac'])) + ' %' if tens else '—'} | "
          f"{r.get('all_gemm_tflops', 0):.1f} |")
print("\n-- DESIGN.md §12 rows --")
for c in order:
    j = R[c]; r = j["roofline"]; hp = r.get("hbm_passes", {})
    a7 = hp.get("distances", {}).get("frac", 0); a10 = hp.get("svgd_update", {}).get("frac", 0)
    print(f"| {c} | {j['ms_per_step']:.4g} | {j['value']:,.0f} | {j['e2e']['value']:,.0f} | "
          f"{r['kernel'].split('(')[-1].rstrip(')')} | {r['frac']:.2f} ({r['bound']}) | {r.get('all_gemm_tflops', 0):.1f} | "
          f"{a7:.2f} / {a10:.2f} |")
