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


def _lib_worker(rank, world, port, q):
    """The host-side halves of the sharded Algorithm-1 round through libetune_cuda.so itself:
    (1) training on rank 0 + model broadcast -- rank 0 writes the model with the library's
    EnergyModel::to_json (etune_model_to_json), the bytes cross the process group, every rank
    parses them with the library's reader and re-serialises byte for byte; (2) the energy
    measurements split over the ranks -- each rank logs its slice with the library's JSONL writer,
    the texts are all-gathered and every rank parses the concatenation into the same full log."""
    import numpy as np
    import torch
    from paper_2411_18873_b200 import capi
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    here = os.path.dirname(os.path.abspath(__file__))
    # (1) model from rank 0
    if rank == 0:
        m = capi.model_from_json(open(os.path.join(here, "golden", "persist", "model_c2_r50_conv3x3.json")).read())
        text = capi.model_to_json(m["feature"], m["threshold"], m["left"], m["right"], m["value"], m["tree_offsets"],
                                  m["params"], m["base_score"], m["reference_energy_mj"])
        payload = torch.frombuffer(bytearray(text.encode()), dtype=torch.uint8)
        size = torch.tensor([payload.numel()], dtype=torch.int64)
    else:
        size = torch.zeros(1, dtype=torch.int64)
    dist.broadcast(size, 0)
    if rank != 0:
        payload = torch.zeros(int(size.item()), dtype=torch.uint8)
    dist.broadcast(payload, 0)
    text = bytes(payload.numpy()).decode()
    m = capi.model_from_json(text)
    again = capi.model_to_json(m["feature"], m["threshold"], m["left"], m["right"], m["value"], m["tree_offsets"],
                               m["params"], m["base_score"], m["reference_energy_mj"])
    model_ok = again == text and len(m["tree_offsets"]) == 101
    # (2) measurement log: rank r measured candidates [r*n/W, (r+1)*n/W)
    n = 96
    rng = np.random.default_rng(17)
    full = np.zeros(n, capi.LOG_RECORD_DTYPE)
    full["m"]["candidate_id"] = rng.integers(0, 2**63, n).astype(np.uint64) * 2 + 1
    full["m"]["latency_ms"] = rng.uniform(1e-3, 10, n)
    full["m"]["avg_power_w"] = rng.uniform(50, 400, n)
    full["m"]["energy_mj"] = full["m"]["avg_power_w"] * full["m"]["latency_ms"]
    full["m"]["iterations"] = rng.integers(1, 10**6, n)
    full["backend"], full["timestamp"] = b"sim", b"2026-10-17T12:34:56Z"
    lo, hi = rank * n // world, (rank + 1) * n // world
    mine = capi.measurement_log_to_jsonl(full[lo:hi])
    texts = [None] * world
    dist.all_gather_object(texts, mine)
    merged = capi.measurement_log_from_jsonl("".join(texts))
    log_ok = all((merged["m"][f] == full["m"][f]).all()
                 for f in ("candidate_id", "latency_ms", "avg_power_w", "energy_mj", "iterations"))
    q.put((rank, model_ok, log_ok, text == again))
    dist.destroy_process_group()


def test_sharded_round_host_halves_through_library_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lib_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, *_ in res) == [0, 1]
    assert all(ok_m and ok_l and same for _, ok_m, ok_l, same in res)
