"""Workload shapes and input generators (SURVEY.md §8 configs, App. A param counts)."""
import numpy as np

from inputs import WORKLOADS, param_count, synth


def test_param_counts_match_survey_appendix():
    expect = {"C1": 1153, "C2": 198401, "C3": 3153921, "C4": 8513, "C5": 20989953, "C5b": 20989953, "S1": 1053185}
    for k, v in expect.items():
        assert WORKLOADS[k].d == v
    # the paper's scaling nets: 10 DxD layers + Dx1 (App. A)
    for D, v in ((200, 402201), (1000, 10011001), (2000, 40022001)):
        assert param_count([D] * 11 + [1]) == v


def test_generators_deterministic_float32():
    for w in WORKLOADS.values():
        x, y = synth.workload_batch(w, step=3)
        x2, y2 = synth.workload_batch(w, step=3)
        assert x.dtype == np.float32 and y.dtype == np.float32
        assert x.shape == (w.batch, w.dims[0]) and y.shape == (w.batch, w.dims[-1])
        assert np.array_equal(x, x2) and np.array_equal(y, y2)
        assert np.all(np.isfinite(x)) and np.all(np.isfinite(y))
    # random batches cycle through 10 fixed batches
    a = synth.batch("random", 16, 2, 1, 1)
    b = synth.batch("random", 16, 2, 1, 11)
    assert np.array_equal(a[0], b[0])


def test_dyadic_theta_is_exact_lattice():
    th = synth.dyadic_theta(5, 64, 0)
    assert np.all(th * 8 == np.round(th * 8)) and np.abs(th).max() <= 4.0
