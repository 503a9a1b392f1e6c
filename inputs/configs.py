"""Workload catalogue (shapes only; no method arithmetic).

Each entry is one row of SURVEY.md §8 "Configs" / BASELINE.json `configs`.
The MLP notation "a-HxL-b" means input width a, L hidden layers of width H,
output width b, i.e. dims = [a, H, ..., H, b]: L+1 Linear layers.  Examples:

    1-32-32-1   -> dims [1, 32, 32, 1]          (3 Linear layers, d = 1,153)
    2-256x4-1   -> dims [2, 256, 256, 256, 256, 1]  (5 Linear layers, d = 198,401)

Param counts are checked in tests/test_inputs.py against SURVEY.md App. A.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Workload:
    name: str
    n_particles: int
    dims: tuple
    batch: int
    data: str            # generator name in inputs.synth
    steps: int = 1       # steps used by parity runs
    note: str = ""

    @property
    def n_layers(self) -> int:
        return len(self.dims) - 1

    @property
    def d(self) -> int:
        return param_count(self.dims)


def mlp_dims(d_in: int, hidden: int, n_hidden: int, d_out: int) -> tuple:
    return tuple([d_in] + [hidden] * n_hidden + [d_out])


def param_count(dims) -> int:
    return int(sum(dims[l] * dims[l + 1] + dims[l + 1] for l in range(len(dims) - 1)))


# BASELINE.json configs[0..4] plus the north-star scaling point S1.
WORKLOADS = {
    "C1": Workload("C1", 4, (1, 32, 32, 1), 256, "sine", steps=10,
                   note="4 particles, MLP 1-32-32-1, 1-D sine regression on 256 points"),
    "C2": Workload("C2", 16, mlp_dims(2, 256, 4, 1), 8192, "advection",
                   note="16 particles, MLP 2-256x4-1, 2-D advection field, 8192 points/batch"),
    "C3": Workload("C3", 64, mlp_dims(3, 1024, 4, 1), 8192, "burgers",
                   note="64 particles, MLP 3-1024x4-1, Burgers regression"),
    "C4": Workload("C4", 256, mlp_dims(1, 64, 3, 1), 128, "random",
                   note="256 particles, MLP 1-64x3-1, kernel-bound regime"),
    "C5": Workload("C5", 8, mlp_dims(2, 2048, 6, 1), 1024, "random",
                   note="8 particles, MLP 2-2048x6-1, GEMM-bound regime"),
    "C5b": Workload("C5b", 8, mlp_dims(2, 2048, 6, 1), 128, "random",
                    note="8 particles, MLP 2-2048x6-1 at the paper's batch of 128 (PAPER.md:355)"),
    "S1": Workload("S1", 64, mlp_dims(3, 512, 5, 1), 8192, "burgers",
                   note="64 particles x ~1M params (north-star scaling point)"),
}
