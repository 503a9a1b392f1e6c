"""World-size-2 tests of the multi-process host path on CPU (gloo), no GPU:

* the NCCL unique id that the library's communicator is built from is created through the
  C-ABI on rank 0 and reaches every rank byte-identical (paper_2306_06528_b200/dist.py);
* the device-time reduction bench.py reports is the MAX over ranks;
* the particle block shard (R18) tiles [0, n) exactly once and the C-ABI's
  workspace query accepts/rejects the same (n, P) pairs.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2306_06528_b200 import dist as pdist
    from paper_2306_06528_b200 import push
    try:
        r, w, _ = pdist.init(backend="gloo")
        nid = pdist.bootstrap_nccl_id(r, w)
        ids = [None] * w
        dist.all_gather_object(ids, nid)
        mx = pdist.max_over_ranks(1.5 + r, w)
        rows = [pdist.shard_rows(8, w, k) for k in range(w)]
        ws_ok = push.workspace_size(push.make_config(8, [2, 64, 64, 1], max_batch=64), w) > 0
        try:
            push.workspace_size(push.make_config(7, [2, 64, 64, 1], max_batch=64), w)
            ws_bad = False
        except push.PushError as e:
            ws_bad = e.status == push.PUSH_E_INVALID
        pdist.barrier(w)
        q.put((r, ids, mx, rows, ws_ok, ws_bad))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        pdist.finalize(world)


def test_world2_bootstrap_and_reductions():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 6, r
    res.sort()
    ids0 = res[0][1]
    for r, ids, mx, rows, ws_ok, ws_bad in res:
        assert ids == ids0 and len(ids[0]) == 128 and ids[0] == ids[1]
        assert mx == 2.5
        assert rows == [(0, 4), (4, 4)]
        assert ws_ok and ws_bad


@pytest.mark.parametrize("n,world", [(64, 8), (16, 2), (4, 4), (256, 8), (8, 1)])
def test_shard_rows_tile_exactly(n, world):
    from paper_2306_06528_b200 import dist as pdist
    covered = []
    for r in range(world):
        r0, nl = pdist.shard_rows(n, world, r)
        covered += list(range(r0, r0 + nl))
    assert covered == list(range(n))
    with pytest.raises(ValueError):
        pdist.shard_rows(n + 1, 2, 0)  # n is even in every case: an odd n cannot be split over 2 ranks
