"""Seeded synthetic input generators + workload catalogue (shared by oracle tests,
GPU tests and bench.py; contains none of the method's arithmetic)."""
from .configs import WORKLOADS, Workload, mlp_dims, param_count  # noqa: F401
from . import synth  # noqa: F401
