"""Thin ctypes binding of include/push.h (argument marshalling only).

Every step of the SVGD particle step runs inside libpush_b200.so; this module
only converts Python/torch arguments into the C-ABI's plain pointers and
sizes.  PyTorch provides the device memory (the caller-owned workspace), the
CUDA stream and, for multi-GPU jobs, the process group that broadcasts the
NCCL unique id.  There is no fallback: if the library is missing or the
device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char, c_char_p, c_double, c_float, c_int32, c_int64, c_size_t, c_uint8,
                    c_uint64, c_void_p)

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpush_b200.so")

PUSH_OK, PUSH_E_INVALID, PUSH_E_SHAPE, PUSH_E_STATE, PUSH_E_CUDA, PUSH_E_NCCL, PUSH_E_NOMEM, PUSH_E_UNSUPPORTED = range(8)
STATUS_NAMES = ["PUSH_OK", "PUSH_E_INVALID", "PUSH_E_SHAPE", "PUSH_E_STATE", "PUSH_E_CUDA", "PUSH_E_NCCL",
                "PUSH_E_NOMEM", "PUSH_E_UNSUPPORTED"]
ACT = {"tanh": 0, "relu": 1, "identity": 2}
VAR_PER_TENSOR, VAR_PAPER_NORM, VAR_PRIOR_SUM = 1, 2, 4  # push_config.variant bits (NEXT-2)
VARIANT_PAPER = 7
XCHG = {"allgather": 0, "dshard": 1}
PRIOR = {"uniform": 0, "gaussian": 1}
BW = {"median": 0, "median_ln_n": 0, "median_ln_n1": 1, "fixed": 2}
WHAT = {"theta": 0, "grad": 1, "dist": 2, "h": 3, "loss": 4, "kernel": 5}
MAX_LAYERS = 15

# Every symbol include/push.h and include/push_debug.h declare (checked by tests/test_abi.py).
EXPORTS = ["push_version", "push_last_error", "push_get_unique_id", "push_workspace_size", "push_init",
           "push_init_local_group", "push_particle_grads", "push_set_grads", "push_svgd_step", "push_step_graph",
           "push_step_host",
           "push_gather", "push_predict", "push_ensemble_step", "push_swag_collect", "push_swag_sample",
           "push_profile_enable", "push_profile_read", "push_profile_trace", "push_launch_count",
           "push_destroy",
           "pushdbg_gemm3xtf32", "pushdbg_gemm1xtf32", "pushdbg_gemm"]


class PushConfig(Structure):
    _fields_ = [("n_particles", c_int32), ("n_layers", c_int32), ("dims", c_int32 * (MAX_LAYERS + 1)),
                ("activation", c_int32), ("prior", c_int32), ("prior_sigma", c_float), ("lik_scale", c_float),
                ("bw_rule", c_int32), ("bw_h", c_float), ("step_size", c_float), ("max_batch", c_int32),
                ("seed", c_uint64), ("swag", c_int32), ("variant", c_int32),
                ("exchange", c_int32), ("reserved", c_int32)]


class ProfileRow(Structure):
    _fields_ = [("name", c_char * 24), ("ms", c_double), ("launches", c_int64), ("alg_bytes", c_double),
                ("alg_flops", c_double)]


class PushError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


_LIB = None


def lib():
    """Load libpush_b200.so (raises if it has not been built — there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P = c_void_p
    sig = {
        "push_version": ([], c_char_p),
        "push_last_error": ([], c_char_p),
        "push_get_unique_id": ([POINTER(c_uint8)], c_int32),
        "push_workspace_size": ([POINTER(PushConfig), c_int32, POINTER(c_size_t)], c_int32),
        "push_init": ([POINTER(PushConfig), c_int32, c_int32, POINTER(c_uint8), P, c_size_t, P, POINTER(P)], c_int32),
        "push_init_local_group": ([POINTER(PushConfig), c_int32, POINTER(P), c_size_t, P, POINTER(P)], c_int32),
        "push_particle_grads": ([P, P, P, c_int32, P, P], c_int32),
        "push_set_grads": ([P, P, P], c_int32),
        "push_svgd_step": ([P, P], c_int32),
        "push_step_graph": ([P, P, P, c_int32, P, P], c_int32),
        "push_step_host": ([P, P, P, c_int32, P, P], c_int32),
        "push_gather": ([P, c_int32, P, P], c_int32),
        "push_predict": ([P, P, c_int32, P, P, P, P], c_int32),
        "push_ensemble_step": ([P, P], c_int32),
        "push_swag_collect": ([P, P], c_int32),
        "push_swag_sample": ([P, c_uint64, P, P], c_int32),
        "push_profile_enable": ([P, c_int32], c_int32),
        "push_profile_read": ([P, POINTER(ProfileRow), c_int32, POINTER(c_int32)], c_int32),
        "push_profile_trace": ([P, POINTER(c_int32), c_int32, POINTER(c_int32)], c_int32),
        "push_launch_count": ([P, POINTER(c_int64)], c_int32),
        "push_destroy": ([P], c_int32),
        "pushdbg_gemm3xtf32": ([c_int32] * 6 + [P, P, P, P], c_int32),
        "pushdbg_gemm1xtf32": ([c_int32] * 6 + [P, P, P, P], c_int32),
        "pushdbg_gemm": ([c_int32] * 8 + [P, P, P, P], c_int32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _LIB = L
    return L


def check(status: int):
    if status != PUSH_OK:
        raise PushError(status, lib().push_last_error().decode())


def make_config(n_particles: int, dims, activation="tanh", prior="uniform", prior_sigma=1.0, lik_scale=1.0,
                bw_rule="median", bw_h=1.0, step_size=1e-3, max_batch=1, seed=0, swag=False,
                variant=0, exchange="allgather") -> PushConfig:
    """variant: 0 (canonical SVGD) or an OR of VAR_PER_TENSOR / VAR_PAPER_NORM / VAR_PRIOR_SUM
    (VARIANT_PAPER = all three, include/push.h).
    exchange: "allgather" (default) or "dshard" (d-sharded kernel phase, NEXT-4)."""
    c = PushConfig()
    c.n_particles = n_particles
    c.n_layers = len(dims) - 1
    for i, v in enumerate(dims):
        c.dims[i] = int(v)
    c.activation = ACT[activation] if isinstance(activation, str) else int(activation)
    c.prior = PRIOR[prior] if isinstance(prior, str) else int(prior)
    c.prior_sigma = prior_sigma
    c.lik_scale = lik_scale
    c.bw_rule = BW[bw_rule] if isinstance(bw_rule, str) else int(bw_rule)
    c.bw_h = bw_h
    c.step_size = step_size
    c.max_batch = max_batch
    c.seed = seed
    c.swag = 1 if swag else 0
    c.variant = int(variant)
    c.exchange = XCHG[exchange] if isinstance(exchange, str) else int(exchange)
    c.reserved = 0
    return c


def workspace_size(cfg: PushConfig, world_size: int = 1) -> int:
    b = c_size_t(0)
    check(lib().push_workspace_size(ctypes.byref(cfg), world_size, ctypes.byref(b)))
    return b.value


def get_unique_id() -> bytes:
    buf = (c_uint8 * 128)()
    check(lib().push_get_unique_id(buf))
    return bytes(buf)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _ptr(t):
    return c_void_p(t.data_ptr()) if t is not None else None


def _theta_ptr(theta0, n, d):
    if theta0 is None:
        return None, None
    a = np.ascontiguousarray(theta0, dtype=np.float32)
    assert a.shape == (n, d), (a.shape, (n, d))
    return a, a.ctypes.data_as(c_void_p)


class Context:
    """One rank's SVGD state (push_ctx).  Tensors passed in must be float32 CUDA contiguous."""

    def __init__(self, cfg: PushConfig, rank: int = 0, world_size: int = 1, nccl_id: bytes | None = None,
                 theta0=None, _handle=None, _ws=None):
        import torch
        self.cfg = cfg
        self.rank, self.world_size = rank, world_size
        self.n = cfg.n_particles
        self.dims = [cfg.dims[i] for i in range(cfg.n_layers + 1)]
        self.d = int(sum(self.dims[l] * self.dims[l + 1] + self.dims[l + 1] for l in range(cfg.n_layers)))
        self.n_local = self.n // world_size
        # distance / kernel matrices per step: one per W_l and b_l under VAR_PER_TENSOR, else one
        self.n_tensors = 2 * cfg.n_layers if cfg.variant & VAR_PER_TENSOR else 1
        if _handle is not None:
            self._h, self._ws = _handle, _ws
            return
        nbytes = workspace_size(cfg, world_size)
        self._ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        keep, tp = _theta_ptr(theta0, self.n, self.d)
        idbuf = None
        if world_size > 1:
            assert nccl_id is not None and len(nccl_id) == 128
            idbuf = (c_uint8 * 128).from_buffer_copy(nccl_id)
        h = c_void_p()
        check(lib().push_init(ctypes.byref(cfg), rank, world_size, idbuf, _ptr(self._ws), nbytes, tp,
                              ctypes.byref(h)))
        self._h = h

    # -- path
    def particle_grads(self, x, y, loss=None, stream=None):
        check(lib().push_particle_grads(self._h, _ptr(x), _ptr(y), int(x.shape[0]), _ptr(loss), _stream(stream)))

    def set_grads(self, g, stream=None):
        check(lib().push_set_grads(self._h, _ptr(g), _stream(stream)))

    def svgd_step(self, stream=None):
        check(lib().push_svgd_step(self._h, _stream(stream)))

    def step_graph(self, x, y, loss=None, stream=None):
        """push_particle_grads + push_svgd_step replayed from a captured CUDA graph."""
        check(lib().push_step_graph(self._h, _ptr(x), _ptr(y), int(x.shape[0]), _ptr(loss), _stream(stream)))

    def step_host(self, x: np.ndarray, y: np.ndarray, stream=None) -> np.ndarray:
        loss = np.empty(self.n_local, dtype=np.float32)
        check(lib().push_step_host(self._h, x.ctypes.data_as(c_void_p), y.ctypes.data_as(c_void_p), int(x.shape[0]),
                                   loss.ctypes.data_as(c_void_p), _stream(stream)))
        return loss

    def gather(self, what: str, stream=None) -> np.ndarray:
        T = self.n_tensors  # dist / kernel are stacked per tensor only under VAR_PER_TENSOR
        lead = (T,) if T > 1 else ()
        shape = {"theta": (self.n, self.d), "grad": (self.n, self.d), "dist": lead + (self.n, self.n), "h": (T,),
                 "loss": (self.n,), "kernel": lead + (self.n_local, self.n)}[what]
        out = np.empty(shape, dtype=np.float32)
        check(lib().push_gather(self._h, WHAT[what], out.ctypes.data_as(c_void_p), _stream(stream)))
        return out

    def predict(self, x, stream=None):
        """Predictive pushforward (push_predict): (pred [n, B, d_out], mean [B, d_out], std [B, d_out]) tensors."""
        import torch
        B, dout = int(x.shape[0]), self.dims[-1]
        pred = torch.empty((self.n, B, dout), dtype=torch.float32, device=x.device)
        mean = torch.empty((B, dout), dtype=torch.float32, device=x.device)
        std = torch.empty((B, dout), dtype=torch.float32, device=x.device)
        check(lib().push_predict(self._h, _ptr(x), B, _ptr(pred), _ptr(mean), _ptr(std), _stream(stream)))
        return pred, mean, std

    def ensemble_step(self, stream=None):
        check(lib().push_ensemble_step(self._h, _stream(stream)))

    def swag_collect(self, stream=None):
        check(lib().push_swag_collect(self._h, _stream(stream)))

    def swag_sample(self, seed: int, stream=None):
        import torch
        out = torch.empty((self.n_local, self.d), dtype=torch.float32, device="cuda")
        check(lib().push_swag_sample(self._h, seed, _ptr(out), _stream(stream)))
        return out

    # -- instrumentation
    def profile_enable(self, on: bool = True):
        check(lib().push_profile_enable(self._h, 1 if on else 0))

    def profile_read(self):
        rows = (ProfileRow * 32)()
        n = c_int32(0)
        check(lib().push_profile_read(self._h, rows, 32, ctypes.byref(n)))
        return [dict(name=r.name.decode(), ms=r.ms, launches=r.launches, alg_bytes=r.alg_bytes,
                     alg_flops=r.alg_flops) for r in rows[:n.value]]

    def profile_trace(self):
        """Class names of every kernel launched since profile_enable(True), in launch order."""
        n = c_int32(0)
        check(lib().push_profile_trace(self._h, None, 0, ctypes.byref(n)))
        buf = (c_int32 * max(n.value, 1))()
        check(lib().push_profile_trace(self._h, buf, n.value, ctypes.byref(n)))
        names = [r["name"] for r in self.profile_read()]
        return [names[buf[i]] for i in range(n.value)]

    def launch_count(self) -> int:
        c = c_int64(0)
        check(lib().push_launch_count(self._h, ctypes.byref(c)))
        return c.value

    def close(self):
        if getattr(self, "_h", None):
            lib().push_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def local_group(cfg: PushConfig, world_size: int, theta0=None):
    """P loopback contexts on the current GPU (push_init_local_group) — for sharding tests on one device."""
    import torch
    nbytes = workspace_size(cfg, world_size)
    wss = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(world_size)]
    ptrs = (c_void_p * world_size)(*[w.data_ptr() for w in wss])
    outs = (c_void_p * world_size)()
    n = cfg.n_particles
    d = int(sum(cfg.dims[l] * cfg.dims[l + 1] + cfg.dims[l + 1] for l in range(cfg.n_layers)))
    keep, tp = _theta_ptr(theta0, n, d)
    check(lib().push_init_local_group(ctypes.byref(cfg), world_size, ptrs, nbytes, tp, outs))
    return [Context(cfg, r, world_size, _handle=c_void_p(outs[r]), _ws=wss[r]) for r in range(world_size)]


def gemm3xtf32(A, B, a_mn: bool, b_mn: bool, M: int, N: int, K: int, passes: int = 3, b_split: bool = False,
               stream=None):
    """Debug entry: C[p] = A[p] @ B[p] through the product's tcgen05 kernel (see include/push_debug.h)."""
    import torch
    batch = A.shape[0]
    C = torch.empty((batch, M, N), dtype=torch.float32, device=A.device)
    check(lib().pushdbg_gemm(passes, int(a_mn), int(b_mn), int(b_split), M, N, K, batch, _ptr(A), _ptr(B), _ptr(C),
                             _stream(stream)))
    return C
