"""Run a few eager SVGD steps of a workload (for ncu captures of single kernels).
    python scripts/step_once.py --config S1 [--steps 2]"""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from inputs import WORKLOADS, synth
from paper_2306_06528_b200 import push

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="S1")
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
w = WORKLOADS[a.config]
ctx = push.Context(push.make_config(w.n_particles, list(w.dims), max_batch=w.batch, step_size=1e-3, seed=0))
for s in range(a.steps):
    x, y = synth.workload_batch(w, s)
    ctx.particle_grads(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    ctx.svgd_step()
torch.cuda.synchronize()
print("ok", a.config)
