"""Per-kernel-class DRAM traffic of one SVGD step, for bench.py's roofline `traffic` field.

Run under ncu (one GPU):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,\
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none \
      --csv --log-file gpurun_out/traffic_C2.csv python scripts/traffic_probe.py --config C2
then, on the dev host:
  python scripts/traffic_probe.py --summarise gpurun_out/traffic_C2.csv --config C2   -> profiles/traffic_C2.json
The probe runs one warm-up step, then one profiled eager step whose per-launch class trace (from the
library, push_profile_trace) is written next to the csv; the LAST len(trace) kernels ncu lists are
that step's kernels in the same order."""
import argparse, csv, io, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--summarise", default=None)
args = ap.parse_args()
trace_path = os.path.join(ROOT, "gpurun_out", f"traffic_trace_{args.config}.json")

if args.summarise is None:
    import torch
    from inputs import WORKLOADS, synth
    from paper_2306_06528_b200 import push
    w = WORKLOADS[args.config]
    ctx = push.Context(push.make_config(w.n_particles, list(w.dims), max_batch=w.batch, step_size=1e-3, seed=0))
    for s in range(2):
        x, y = synth.workload_batch(w, s)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        if s == 1:
            ctx.profile_enable(True)
        ctx.particle_grads(xd, yd)
        ctx.svgd_step()
    torch.cuda.synchronize()
    trace = ctx.profile_trace()
    os.makedirs(os.path.dirname(trace_path), exist_ok=True)
    json.dump(trace, open(trace_path, "w"))
    print("trace", len(trace))
else:
    trace = json.load(open(trace_path))
    lines = [l for l in open(args.summarise) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = {}
    order = []
    for r in rows:
        key = r["ID"]
        if key not in per:
            per[key] = {"kernel": r["Kernel Name"]}
            order.append(key)
        try:
            per[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        except ValueError:  # "n/a"
            pass
    kern = [per[k] for k in order][-len(trace):]
    out = {}
    for cls, k in zip(trace, kern):
        e = out.setdefault(cls, {"launches": 0, "dram_bytes": 0.0, "ncu_time_ns": 0.0, "kernels": set(),
                                 "tensor_ns": 0.0})
        e["launches"] += 1
        e["dram_bytes"] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
        tn = k.get("gpu__time_duration.sum", 0)
        e["ncu_time_ns"] += tn
        # time-weighted tensor-pipe activity (% of the elapsed peak) of the class's launches
        e["tensor_ns"] += tn * k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0) / 100
        e["kernels"].add(k["kernel"].split("(")[0][:60])
    res = {c: {"launches": e["launches"], "dram_bytes_per_launch": e["dram_bytes"] / e["launches"],
               "ncu_time_us_per_launch": e["ncu_time_ns"] / e["launches"] / 1e3,
               "tensor_pipe_pct": 100 * e["tensor_ns"] / e["ncu_time_ns"] if e["ncu_time_ns"] else 0.0,
               "kernels": sorted(e["kernels"])}
           for c, e in out.items()}
    path = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    json.dump({"config": args.config, "source": os.path.basename(args.summarise),
               "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                      "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active "
                      "--clock-control none over one eager step (scripts/traffic_probe.py)",
               "classes": res}, open(path, "w"), indent=1)
    print(json.dumps(res, indent=1))
