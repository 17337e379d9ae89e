"""world_size-2 gloo test (CPU) of the multi-GPU selection protocol used by
etune_cu_topk_sharded and bench.py: contiguous ascending shards, per-shard top-k
records (score, global index), all-gather in rank order, merge by (score, position).
The per-shard and merge selections are the oracle's (score asc, index asc) top-k."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, q):
    import torch
    from etune_testlib import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    rng = np.random.default_rng(11)
    vals = rng.choice(rng.uniform(0.9, 3.0, 150), n)  # identical population on every rank
    bounds = np.linspace(0, n, world + 1).astype(np.int64)
    lo, hi = bounds[rank], bounds[rank + 1]
    m = min(k, hi - lo)
    loc = O.topk(vals[lo:hi], m)
    rs = np.full(k, np.inf)
    rg = np.full(k, np.iinfo(np.int64).max, np.int64)
    rs[:m] = vals[lo:hi][loc]
    rg[:m] = loc + lo
    gs = [torch.zeros(k, dtype=torch.float64) for _ in range(world)]
    gg = [torch.zeros(k, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gs, torch.from_numpy(rs))
    dist.all_gather(gg, torch.from_numpy(rg))
    cat_s = torch.cat(gs).numpy()
    cat_g = torch.cat(gg).numpy()
    sel = cat_g[O.topk(cat_s, k)]
    q.put((rank, sel.tolist(), O.topk(vals, k).tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n,k", [(20000, 1024), (1500, 1000), (10, 10)])
def test_sharded_selection_protocol_gloo(n, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    sels = {r: s for r, s, _ in res}
    want = res[0][2]
    assert sels[0] == sels[1] == want
