#!/usr/bin/env python
"""bench.py — SVGD particle-steps/s of the B200-native PusH step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the whole hot path: per-particle MLP
gradient of log p on the batch, Theta/G exchange (N > 1), pairwise distances, median
bandwidth, kernel matrix and the fused SVGD update of every particle.

Default workload: S1, the north-star scaling point (64 particles x 1,053,185 parameters, MLP
3-512x5-1, 8192 points of the Burgers field per batch), for N = 1 and
N > 1 (the metric is quoted at 1/2/4/8 GPUs on this point).  `--config C2` gives
BASELINE.json configs[1].  For N > 1 the same n particles are sharded n/N per GPU (strong
scaling), one rank per GPU over NCCL: under torchrun, or launched by bench.py itself (it
re-executes through torch.distributed.run when WORLD_SIZE is unset and --gpus N > 1).

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
DEFAULT_CONFIG = "S1"


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


def cublas_tf32_tflops(dev):
    """Measured dense TF32 tensor throughput (cuBLAS 8192^3 fp32 matmul with TF32 allowed, best of 10):
    context for the 3xTF32 roofline (the official peak stays bf16-measured x the nominal ratio)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(8192, 8192, device=dev)
        b = torch.randn(8192, 8192, device=dev)
        for _ in range(3):
            a @ b
        best = 1e9
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(10):
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * 8192 ** 3 / (best / 1e3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def allgather_busbw(w, ws, dev):
    """NCCL all-gather bus bandwidth at this config's per-rank Theta / G block (n_local x ld floats), the
    exchange's message size (SURVEY.md §8(d) NVLink row): busbw = algbw (P-1)/P, max time over ranks."""
    import torch
    import torch.distributed as dist
    ld = (w.d + 127) // 128 * 128
    cnt = (w.n_particles // ws) * ld
    src = torch.zeros(cnt, device=dev)
    dst = torch.empty(cnt * ws, device=dev)
    for _ in range(3):
        dist.all_gather_into_tensor(dst, src)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dist.all_gather_into_tensor(dst, src)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 10], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    algbw = 4.0 * cnt * ws / (ms / 1e3) / 1e9
    return {"bytes_per_rank": 4 * cnt, "ms": ms, "algbw_gbs": algbw, "busbw_gbs": algbw * (ws - 1) / ws,
            "how": "torch.distributed all_gather_into_tensor (NCCL), 10 iterations, max over ranks"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------- oracle baseline
def oracle_step_time(w, th, G, x, y, budget_s):
    """Seconds of ONE full oracle step (oracle/ as it stands, float64 numpy) estimated from a bounded
    sample: the gradients of the first k particles (k grown until ~budget/2; the per-particle cost is
    identical) scaled by n/k, plus the kernel/update phase (distances, bandwidth, K, phi) on the first
    m columns (m sized to ~budget/2; its cost is linear in the columns) scaled by d/m.
    Returns (seconds, k, m)."""
    from oracle import mlp as omlp
    from oracle import svgd as osvgd
    dims = list(w.dims)
    t0 = time.perf_counter()
    k = 0
    while k < w.n_particles:
        G[k], _ = omlp.grad_log_post(th[k], dims, x, y)
        k += 1
        if time.perf_counter() - t0 > budget_s / 2:
            break
    t_grad = (time.perf_counter() - t0) / k
    d = th.shape[1]
    m = min(d, 4096)
    while True:
        t1 = time.perf_counter()
        osvgd.svgd_step(th[:, :m], G[:, :m], 1e-3)
        t_upd = time.perf_counter() - t1
        if m == d or t_upd > budget_s / 8:
            break
        m = min(d, m * 4)
    return w.n_particles * t_grad + t_upd * d / m, k, m


def cpu_baseline(w, budget_s: float = 20.0):
    """The float64 oracle timed on the host cores on a bounded sample of the workload (oracle_step_time)."""
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    dims = list(w.dims)
    x, y = synth.workload_batch(w, 0)
    from oracle import init as oinit
    th = oinit.init_theta(w.n_particles, dims, 0).astype(np.float64)
    G = np.zeros_like(th)
    per_step, k, m = oracle_step_time(w, th, G, x, y, budget_s)
    return {"value": w.n_particles / per_step, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(),
            "nproc": os.cpu_count(), "kind": "oracle",
            "sample": f"{k} of {w.n_particles} particle gradients (B={w.batch}) scaled by n/k, plus the kernel/"
                      f"update phase on {m} of {w.d} columns scaled by d/m: one step = {per_step:.2f} s",
            "c1_single_thread": c1_single_thread()}


def c1_single_thread():
    """the oracle also timed on ONE thread on C1 (4 particles, 1-32-32-1, 10 steps)."""
    from oracle import init as oinit
    from oracle import svgd as osvgd
    w = WORKLOADS["C1"]
    dims = list(w.dims)
    th = oinit.init_theta(w.n_particles, dims, 0).astype(np.float64)
    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(limits=1)
    except Exception:
        import contextlib
        ctx = contextlib.nullcontext()
    with ctx:
        t0 = time.perf_counter()
        osvgd.svgd_run(th, dims, lambda t: synth.workload_batch(w, t), 10, 1e-3)
        dt = time.perf_counter() - t0
    return {"value": w.n_particles * 10 / dt, "unit": UNIT, "cores": 1, "sample": "C1, 10 full oracle steps"}


def run_reference(args, w):
    """Reference arm (tier rules): the oracle as it stands on the host cores, each step a bounded sample
    of the workload (oracle_step_time, ~4 s), on our arm's config / metric / unit."""
    rank, ws, _ = dist_env()
    if rank != 0:
        return
    from oracle import init as oinit
    dims = list(w.dims)
    th = oinit.init_theta(w.n_particles, dims, 0).astype(np.float64)
    G = np.zeros_like(th)
    times = []
    k = m = 0
    for s in range(args.warmup + args.steps):
        xs, ys = synth.workload_batch(w, s)
        t, k, m = oracle_step_time(w, th, G, xs, ys, 4.0)
        if s >= args.warmup:
            times.append(t)
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
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
                             "sample": f"per step: {k} of {w.n_particles} particle gradients scaled by n/k plus "
                                       f"the kernel/update phase on {m} of {w.d} columns scaled by d/m"},
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

    ag = allgather_busbw(w, ws, dev) if ws > 1 else None
    tf32_meas = cublas_tf32_tflops(dev) if rank == 0 else None

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
    traffic, traffic_src, ncu_tensor = None, None, None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{w.name}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        if dom["name"] in tj.get("classes", {}):
            traffic = tj["classes"][dom["name"]]["dram_bytes_per_launch"]
            traffic_src = f"profiles/traffic_{w.name}.json ({tj.get('how', '')})"
            ncu_tensor = tj["classes"][dom["name"]].get("tensor_pipe_pct")
    per_launch = max(dom["launches"], 1)
    if dom["name"].endswith("gemm"):
        # the profiled pass times the kernel inside a sub-second run at full clock: the BURST bf16 figure
        # applies, converted to 3xTF32 useful flops by the guide's nominal tf32/bf16 ratio
        peak = peaks["bf16_tflops"] * TF32_OVER_BF16 / 3.0
        ach = dom["alg_flops"] / (dom["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "gemm3xtf32 (" + dom["name"] + ")", "achieved": ach, "peak": peak,
                "unit": "TFLOP/s", "frac": ach / peak, "traffic": traffic,
                "algorithmic_per_launch": dom["alg_flops"] / per_launch,
                "peak_note": f"{peak_kind} bf16 burst {peaks['bf16_tflops']:.1f} TF/s x {TF32_OVER_BF16:.3f} "
                             "(tf32/bf16 nominal) / 3 products (3xTF32 useful flops); kernel timed in a "
                             "sub-second pass at full clock"}
        if tf32_meas:
            roof["cublas_tf32_tflops_measured"] = tf32_meas
            roof["frac_vs_cublas_tf32"] = ach / (tf32_meas / 3.0)
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
        if ncu_tensor is not None and dom["name"].endswith("gemm"):
            roof["ncu_tensor_pipe_pct"] = ncu_tensor  # same capture, time-weighted over the class's launches
    npath = os.path.join(ROOT, "profiles", f"ncu_{w.name}.json")
    if os.path.exists(npath):  # ncu --set full summary of this config's step (scripts/ncu_summary.py --json)
        with open(npath) as f:
            nj = json.load(f)
        if dom["name"] in nj.get("classes", {}):
            roof["ncu"] = dict(nj["classes"][dom["name"]], source=f"profiles/ncu_{w.name}.json")
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
    if ag:
        line["allgather"] = ag
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line), flush=True)
    ctx.close()
    pdist.finalize(ws)


def self_launch(args):
    """`python bench.py --gpus N` (N > 1) without a torchrun environment: re-execute this script under
    torch.distributed.run with one rank per GPU (127.0.0.1 rendezvous).  Rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def run_dry(args, w):
    """Launcher check without a GPU (tests/test_bench_launch.py): every rank joins a gloo process group,
    the max-over-ranks reduction runs, rank 0 prints one JSON line."""
    import torch.distributed as dist
    rank, ws, local = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    from paper_2306_06528_b200 import dist as pdist
    t = pdist.max_over_ranks(float(rank + 1), ws)
    r0, nl = pdist.shard_rows(w.n_particles, ws, rank)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "ranks_max": t, "workload": w.name,
                          "rows_rank0": [r0, nl]}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(WORKLOADS))
    ap.add_argument("--dry-run", action="store_true", help="launcher check on CPU (gloo), no GPU work")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of the captured CUDA graph")
    ap.add_argument("--n-particles", type=int, default=0, help="override the workload's particle count (sweeps)")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "dshard"],
                    help="kernel-phase exchange for --gpus > 1 (dshard: d-sharded kernel phase, NEXT-4)")
    ap.add_argument("--variant", default="canonical", choices=["canonical", "paper"],
                    help="paper: PusH's own update (per-tensor kernel, 1/n on the repulsion, prior sum; NEXT-2)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    w = WORKLOADS[args.config]
    if args.n_particles:
        import dataclasses
        w = dataclasses.replace(w, n_particles=args.n_particles,
                                note=f"{w.note} [n overridden to {args.n_particles}]")
    if args.dry_run:
        run_dry(args, w)
    elif args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
