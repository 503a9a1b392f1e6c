#!/usr/bin/env python
"""bench.py — SVGD particle-steps/s of the B200-native PusH step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the whole hot path: per-particle MLP
gradient of log p on the batch, Theta/G exchange (N > 1), pairwise distances, median
bandwidth, kernel matrix and the fused SVGD update of every particle.

Default workload: BASELINE.json configs[1] = C2 (16 particles, MLP 2-256x4-1, 8192 points
of the 2-D advection field per batch) on one B200.  For N > 1 (torchrun, one rank per
GPU, NCCL) the same n particles are sharded n/N per GPU (strong scaling).

Timing: W untimed warm-up steps; K timed steps bracketed by barrier + synchronize, CUDA
events on the launching stream, max over ranks.  The per-step working set (activations
~1.1 GB for C2) exceeds the 126 MB L2, so no L2 flush is inserted.  A second, profiled
pass of K steps (CUDA events around every kernel class, push_profile_*) gives the
dominant kernel's achieved throughput for the roofline object.  e2e re-times K steps
through push_step_host (host batch -> device, step, per-particle losses -> host).
`cpu_baseline` times the float64 oracle (oracle/) on a bounded sample on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs import WORKLOADS, synth  # noqa: E402

METRIC = "SVGD particle-steps/s and param-updates/s at 1/2/4/8 B200; % HBM/tensor roofline"
UNIT = "particle-steps/s"
TF32_OVER_BF16 = 1.1 / 2.25   # nominal dense tf32 / bf16 ratio (B200_PROFILING.md)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, ws, local


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = os.path.join("/tmp", f"push_clocks_{os.getpid()}.csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        with open(self.path) as f:
            for ln in f:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------- oracle baseline
def cpu_baseline(w, budget_s: float = 20.0):
    """Time the float64 oracle as it stands on the host cores on a bounded sample of the workload:
    the gradient of k particles (k grown until ~budget/2) plus the full kernel/update phase once;
    particle-steps/s = n / (n * t_grad_per_particle + t_update)."""
    from oracle import mlp as omlp
    from oracle import svgd as osvgd
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    dims = list(w.dims)
    x, y = synth.workload_batch(w, 0)
    from oracle import init as oinit
    th = oinit.init_theta(w.n_particles, dims, 0).astype(np.float64)
    t0 = time.perf_counter()
    k = 0
    G = np.zeros_like(th)
    while k < w.n_particles:
        G[k], _ = omlp.grad_log_post(th[k], dims, x, y)
        k += 1
        if time.perf_counter() - t0 > budget_s / 2:
            break
    t_grad = (time.perf_counter() - t0) / k
    t1 = time.perf_counter()
    osvgd.svgd_step(th, G, 1e-3)
    t_upd = time.perf_counter() - t1
    per_step = w.n_particles * t_grad + t_upd
    return {"value": w.n_particles / per_step, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{k} of {w.n_particles} particle gradients (B={w.batch}, float64 numpy) + one full "
                      f"kernel/update phase; step time extrapolated as n*t_grad + t_update = {per_step:.2f} s"}


def run_reference(args, w):
    rank, ws, _ = dist_env()
    if rank != 0:
        return
    from oracle import init as oinit
    from oracle import mlp as omlp
    from oracle import svgd as osvgd
    dims = list(w.dims)
    th = oinit.init_theta(w.n_particles, dims, 0).astype(np.float64)
    # bounded sample per step: gradients of `k` particles + the full kernel/update phase
    x, y = synth.workload_batch(w, 0)
    t = time.perf_counter()
    omlp.grad_log_post(th[0], dims, x, y)
    t1 = time.perf_counter() - t
    k = max(1, min(w.n_particles, int(6.0 / max(t1, 1e-6))))
    times = []
    G = np.zeros_like(th)
    for s in range(args.warmup + args.steps):
        xs, ys = synth.workload_batch(w, s)
        t0 = time.perf_counter()
        for i in range(k):
            G[i], _ = omlp.grad_log_post(th[i], dims, xs, ys)
        tg = (time.perf_counter() - t0) / k
        t0 = time.perf_counter()
        th, _ = osvgd.svgd_step(th, G, 1e-3)
        tu = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(w.n_particles * tg + tu)
    step = float(np.mean(times))
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    v = w.n_particles / step
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name + ": " + w.note, "n_particles": w.n_particles, "d": w.d,
                       "batch": w.batch},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"per step: {k} of {w.n_particles} particle gradients timed and scaled by n, "
                                       f"plus the full kernel/update phase"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our path
def run_ours(args, w):
    import torch

    from paper_2306_06528_b200 import dist as pdist
    from paper_2306_06528_b200 import push

    rank, ws, local = dist_env()
    assert ws == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={ws}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pdist.init("nccl", dev)
    nid = pdist.bootstrap_nccl_id(rank, ws)
    dims = list(w.dims)
    if args.variant == "paper":  # NEXT-2: PusH's own update, l = 1 (h = 2), its normal prior
        cfg = push.make_config(w.n_particles, dims, max_batch=w.batch, step_size=1e-3, seed=0, bw_rule="fixed",
                               bw_h=2.0, prior="gaussian", prior_sigma=1.0, variant=push.VARIANT_PAPER)
    else:
        cfg = push.make_config(w.n_particles, dims, max_batch=w.batch, step_size=1e-3, seed=0,
                               exchange=args.exchange)
    ctx = push.Context(cfg, rank, ws, nid)
    nsteps = args.warmup + args.steps
    batches = [synth.workload_batch(w, s) for s in range(nsteps)]
    xs = [torch.from_numpy(b[0]).cuda() for b in batches]
    ys = [torch.from_numpy(b[1]).cuda() for b in batches]
    stream = torch.cuda.current_stream()

    def barrier():
        pdist.barrier(ws)
        torch.cuda.synchronize()

    def maxall(v):
        return pdist.max_over_ranks(v, ws, dev)

    def step(s):
        if args.no_graph:
            ctx.particle_grads(xs[s], ys[s])
            ctx.svgd_step()
        else:
            ctx.step_graph(xs[s], ys[s])

    for s in range(args.warmup):
        step(s)
    barrier()
    clocks = ClockSampler(local)
    time.sleep(0.3)
    l0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for s in range(args.warmup, nsteps):
        step(s)
    e1.record(stream)
    barrier()
    ms = maxall(e0.elapsed_time(e1))
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    ms_step = ms / args.steps
    value = w.n_particles * args.steps / (ms / 1e3)

    # profiled pass: per-kernel-class CUDA events (same stream)
    ctx.profile_enable(True)
    barrier()
    for s in range(args.warmup, nsteps):
        ctx.particle_grads(xs[s], ys[s])
        ctx.svgd_step()
    barrier()
    prof = ctx.profile_read()
    ctx.profile_enable(False)

    # e2e through the public C-ABI with host buffers
    xh = [torch.from_numpy(b[0]).pin_memory() for b in batches]
    yh = [torch.from_numpy(b[1]).pin_memory() for b in batches]
    barrier()
    e0.record(stream)
    for s in range(args.warmup, nsteps):
        ctx.step_host(xh[s].numpy(), yh[s].numpy())
    e1.record(stream)
    barrier()
    ms_e2e = maxall(e0.elapsed_time(e1))
    e2e = {"value": w.n_particles * args.steps / (ms_e2e / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(xs[0].numel() * 4 + ys[0].numel() * 4),
           "d2h_bytes_per_step": int(ctx.n_local * 4)}

    if rank != 0:
        ctx.close()
        pdist.finalize(ws)
        return

    peaks, peak_kind = load_peaks()
    tot = sum(r["ms"] for r in prof) or 1.0
    gemm_rows = [r for r in prof if r["name"].endswith("gemm")]
    # dominant kernel class among those with a roofline (tensor: the GEMMs; HBM: distances, update)
    roofable = [r for r in prof if r["ms"] and (r["name"].endswith("gemm") or r["name"] in ("distances", "svgd_update"))]
    dom = max(roofable or prof, key=lambda r: r["ms"])
    phases = {r["name"]: {"ms_per_step": r["ms"] / args.steps, "share": r["ms"] / tot,
                          "launches_per_step": r["launches"] / args.steps} for r in prof if r["launches"] or r["ms"]}
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{w.name}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        if dom["name"] in tj.get("classes", {}):
            traffic = tj["classes"][dom["name"]]["dram_bytes_per_launch"]
            traffic_src = f"profiles/traffic_{w.name}.json ({tj.get('how', '')})"
    per_launch = max(dom["launches"], 1)
    if dom["name"].endswith("gemm"):
        peak = peaks["bf16_tflops_sustained"] * TF32_OVER_BF16 / 3.0
        ach = dom["alg_flops"] / (dom["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "gemm3xtf32 (" + dom["name"] + ")", "achieved": ach, "peak": peak,
                "unit": "TFLOP/s", "frac": ach / peak, "traffic": traffic,
                "algorithmic_per_launch": dom["alg_flops"] / per_launch,
                "peak_note": f"{peak_kind} bf16 sustained x {TF32_OVER_BF16:.3f} (tf32/bf16 nominal) / 3 passes "
                             "(3xTF32 useful flops)"}
    else:
        # FP32 CUDA-core peak: 148 SMs x 128 FP32 lanes x 2 flops (FMA) x the max SM clock
        fp32_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        ridge = fp32_peak * 1e12 / (peaks["hbm_gbs"] * 1e9)  # flop per byte
        if dom.get("alg_flops") and dom["alg_bytes"] and dom["alg_flops"] / dom["alg_bytes"] > ridge:
            ach = dom["alg_flops"] / (dom["ms"] / 1e3) / 1e12
            roof = {"bound": "alu", "kernel": dom["name"], "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
                    "frac": ach / fp32_peak, "traffic": traffic,
                    "algorithmic_per_launch": dom["alg_flops"] / per_launch,
                    "peak_note": f"FP32 FMA issue: 148 SMs x 128 lanes x 2 x {peaks.get('sm_max_mhz', 1965.0):.0f} MHz "
                                 f"(intensity {dom['alg_flops'] / dom['alg_bytes']:.1f} flop/B > ridge {ridge:.1f})"}
        else:
            peak = peaks["hbm_gbs"]
            ach = dom["alg_bytes"] / (dom["ms"] / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": dom["name"], "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "traffic": traffic, "algorithmic_per_launch": dom["alg_bytes"] / per_launch,
                    "peak_note": f"{peak_kind} hbm_gbs"}
    if traffic_src:
        roof["traffic_note"] = "DRAM bytes per launch (read + write) from " + traffic_src
    all_gemm_ms = sum(r["ms"] for r in gemm_rows)
    all_gemm_fl = sum(r["alg_flops"] for r in gemm_rows)
    if all_gemm_ms:
        roof["all_gemm_tflops"] = all_gemm_fl / (all_gemm_ms / 1e3) / 1e12
        roof["all_gemm_share"] = all_gemm_ms / tot
    # every non-GEMM pass with algorithmic bytes, against the HBM peak (the GEMMs are tensor-bound; the
    # distances / update passes are ALU-bound at n_local >= ~11 / ~45, L2-resident for small working
    # sets: DESIGN.md §6 says which roofline binds each at each config)
    roof["hbm_passes"] = {r["name"]: {"gbs": r["alg_bytes"] / (r["ms"] / 1e3) / 1e9,
                                      "frac": r["alg_bytes"] / (r["ms"] / 1e3) / 1e9 / peaks["hbm_gbs"]}
                          for r in prof if r["ms"] and r.get("alg_bytes") and not r["name"].endswith("gemm")}
    upd = next((r for r in prof if r["name"] == "svgd_update"), None)
    if upd and upd["ms"]:
        roof["svgd_update_gbs"] = upd["alg_bytes"] / (upd["ms"] / 1e3) / 1e9
        roof["svgd_update_hbm_frac"] = roof["svgd_update_gbs"] / peaks["hbm_gbs"]

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": w.name + ": " + w.note, "n_particles": w.n_particles, "dims": dims,
                       "variant": args.variant, "exchange": args.exchange,
                       "d": w.d, "batch": w.batch, "parallelism": f"particles sharded n/{ws} per GPU",
                       "l2": "per-step working set > 126 MB L2 (no flush)",
                       "launch": "eager" if args.no_graph else "cuda-graph (batch staged D2D into the context each step)"},
            "param_updates_per_s": value * w.d, "clocks": clk, "e2e": e2e,
            "gpu_launches": int(launches), "roofline": roof, "phases": phases}
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line), flush=True)
    ctx.close()
    pdist.finalize(ws)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of the captured CUDA graph")
    ap.add_argument("--n-particles", type=int, default=0, help="override the workload's particle count (sweeps)")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "dshard"],
                    help="kernel-phase exchange for --gpus > 1 (dshard: d-sharded kernel phase, NEXT-4)")
    ap.add_argument("--variant", default="canonical", choices=["canonical", "paper"],
                    help="paper: PusH's own update (per-tensor kernel, 1/n on the repulsion, prior sum; NEXT-2)")
    args = ap.parse_args()
    w = WORKLOADS[args.config]
    if args.n_particles:
        import dataclasses
        w = dataclasses.replace(w, n_particles=args.n_particles,
                                note=f"{w.note} [n overridden to {args.n_particles}]")
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
