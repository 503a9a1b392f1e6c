"""Helpers shared by the -m gpu parity tests (no method arithmetic here)."""
from __future__ import annotations

import numpy as np


def rel_err(gpu, ref, floor_frac=1e-3):
    """max_k |a - b| / max(|b|, floor_frac * max_k |b_i|) per row (SURVEY.md §8(c) 'GPU vs oracle')."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    ref2 = ref.reshape(ref.shape[0], -1) if ref.ndim > 1 else ref.reshape(1, -1)
    gpu2 = gpu.reshape(ref2.shape)
    floor = floor_frac * np.abs(ref2).max(axis=1, keepdims=True)
    den = np.maximum(np.abs(ref2), np.maximum(floor, 1e-30))
    return float((np.abs(gpu2 - ref2) / den).max())


def inf_rel(gpu, ref):
    """||a - b||_inf / ||b||_inf per particle row, max over rows."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    num = np.abs(gpu - ref).max(axis=-1)
    den = np.maximum(np.abs(ref).max(axis=-1), 1e-30)
    return float((num / den).max())
