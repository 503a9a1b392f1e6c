"""The C-ABI library loads on a CPU host and exports every symbol include/*.h declares;
host-only entry points (workspace sizing, validation) behave as documented."""
import ctypes
import os
import re

import pytest

from paper_2306_06528_b200 import push

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = set()
    for h in ("push.h", "push_debug.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(push\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(push.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return push.lib()


def test_every_declared_symbol_is_exported(L):
    declared = _declared_functions()
    assert declared == set(push.EXPORTS), declared ^ set(push.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_config_struct_layout_matches_header():
    assert ctypes.sizeof(push.PushConfig) == 128
    assert push.PushConfig.seed.offset == 104
    assert push.PushConfig.swag.offset == 112
    assert push.PushConfig.variant.offset == 116
    assert push.PushConfig.exchange.offset == 120
    assert ctypes.sizeof(push.ProfileRow) == 56


def test_version_and_error_strings(L):
    assert b"sm_100a" in L.push_version()
    assert isinstance(L.push_last_error(), bytes)


def test_workspace_size_host_only(L):
    cfg = push.make_config(16, [2, 256, 256, 256, 256, 1], max_batch=8192)
    b1 = push.workspace_size(cfg, 1)
    b2 = push.workspace_size(cfg, 2)
    assert b1 > 16 * 198401 * 4 * 3 and b2 < b1


@pytest.mark.parametrize("kw,world,status", [
    (dict(n_particles=5), 2, push.PUSH_E_INVALID),          # n % P != 0 (R18)
    (dict(bw_rule="fixed", bw_h=0.0), 1, push.PUSH_E_INVALID),  # l <= 0
    (dict(max_batch=0), 1, push.PUSH_E_SHAPE),
    (dict(prior="gaussian", prior_sigma=0.0), 1, push.PUSH_E_INVALID),
    (dict(step_size=0.0), 1, push.PUSH_E_INVALID),
    (dict(n_particles=4096), 1, push.PUSH_E_SHAPE),
])
def test_validation_errors(L, kw, world, status):
    base = dict(n_particles=4, dims=[1, 32, 32, 1], max_batch=16)
    base.update(kw)
    cfg = push.make_config(**base)
    with pytest.raises(push.PushError) as e:
        push.workspace_size(cfg, world)
    assert e.value.status == status


def test_bad_dims_rejected(L):
    cfg = push.make_config(4, [1, 0, 1], max_batch=4)
    with pytest.raises(push.PushError) as e:
        push.workspace_size(cfg, 1)
    assert e.value.status == push.PUSH_E_SHAPE


def test_variant_field_validated_on_host():
    """push_config.variant: 0..7 accepted (OR of PUSH_VAR_*), anything else PUSH_E_INVALID; per-tensor
    plans need workspace for T = 2L distance / kernel matrices (compared with a direct-form, T = 1 variant:
    the canonical plan's Gram partials are sized differently)."""
    base = push.workspace_size(push.make_config(8, [2, 64, 64, 1], max_batch=64, variant=push.VAR_PAPER_NORM))
    for v in range(8):
        ws = push.workspace_size(push.make_config(8, [2, 64, 64, 1], max_batch=64, variant=v))
        assert ws >= base if v & push.VAR_PER_TENSOR else ws > 0
    for bad in (8, -1):
        with pytest.raises(push.PushError) as e:
            push.workspace_size(push.make_config(8, [2, 64, 64, 1], max_batch=64, variant=bad))
        assert e.value.status == push.PUSH_E_INVALID


def test_exchange_field_validated_on_host():
    """push_config.exchange: ALLGATHER (0) or DSHARD (1, NEXT-4, variant 0 only); DSHARD's per-rank
    workspace (column panels n x ld/P) shrinks with the rank count."""
    mk = lambda **kw: push.make_config(64, [3, 512, 512, 1], max_batch=256, **kw)  # noqa: E731
    ag = [push.workspace_size(mk(), P) for P in (1, 2, 4, 8)]
    ds = [push.workspace_size(mk(exchange="dshard"), P) for P in (1, 2, 4, 8)]
    assert all(b > a for a, b in zip(ds[1:], ds[:-1]))  # strictly shrinking with P
    assert ds[-1] < ag[-1] * 1.5
    for bad in (dict(exchange=2), dict(exchange="dshard", variant=push.VARIANT_PAPER)):
        with pytest.raises(push.PushError) as e:
            push.workspace_size(mk(**bad), 2)
        assert e.value.status == push.PUSH_E_INVALID
    c = mk()
    c.reserved = 1
    with pytest.raises(push.PushError):
        push.workspace_size(c, 1)
