"""Multi-rank paths of the library with two ranks on ONE GPU (the only configuration the build
box has): the ranks talk through torch.distributed's gloo backend, plugged into the library as
its transport (etune_cu_ctx_attach_transport), so everything except NCCL itself -- shard offsets,
per-shard selection, record packing, the W-way merge, the model broadcast, the sharded search
round -- runs in libetune_cuda.so exactly as it does over NCCL on an 8-GPU box.

Each rank's result must equal the single-rank result bit for bit."""
import os
import socket
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
OP = "conv:1,56,56,64,64,3,1,1"
MODEL = "c2_r50_conv3x3"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _forest(capi, ctx):
    import sys
    sys.path.insert(0, HERE)
    from etune_testlib import FlatForest
    g = np.load(os.path.join(HERE, "golden", "golden_reference.npz"))
    k = f"{MODEL}/model/"
    fl = FlatForest(g[k + "feature"], g[k + "threshold"], g[k + "left"], g[k + "right"], g[k + "value"],
                    g[k + "offsets"], float(g[k + "base_score"][0]), float(g[k + "learning_rate"][0]))
    return capi.Forest.from_flat(ctx, fl)


def _select_worker(rank, world, port, n, k, out_dir):
    import sys
    sys.path[:0] = [HERE, os.path.dirname(HERE)]
    import torch.distributed as dist
    from etune_testlib import parse_op
    from paper_2411_18873_b200 import capi
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = capi.Context(0)
    capi.attach_torch_transport(ctx)
    plan = capi.Plan(ctx, parse_op(OP))
    fo = _forest(capi, ctx)
    g, _, _ = capi.reproduce(plan, plan.sample_random(1024, 42), n, 7)
    lo, hi = rank * n // world, (rank + 1) * n // world  # uneven shards when world does not divide n
    shard = g[lo:hi].contiguous()
    pred = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    sc = torch.empty(k, dtype=torch.float64, device="cuda")
    fo.score_select_sharded(plan, shard, lo, k, pred, idx, sc=sc)
    ctx.synchronize()
    np.save(os.path.join(out_dir, f"idx{rank}.npy"), idx.cpu().numpy())
    np.save(os.path.join(out_dir, f"sc{rank}.npy"), sc.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _run(worker, world, *args):
    import torch.multiprocessing as mp
    mp.spawn(worker, args=(world, _free_port()) + args, nprocs=world, join=True)


@pytest.mark.parametrize("world,n,k", [(2, 1 << 18, 1024), (2, 100003, 4096), (3, 70001, 777)])
def test_sharded_score_select_matches_single(world, n, k):
    from etune_testlib import parse_op
    from paper_2411_18873_b200 import capi
    ctx = capi.Context(0)
    plan = capi.Plan(ctx, parse_op(OP))
    fo = _forest(capi, ctx)
    g, _, _ = capi.reproduce(plan, plan.sample_random(1024, 42), n, 7)
    pred = torch.empty(n, dtype=torch.float64, device="cuda")
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    fo.score_select(plan, g, k, pred, idx)
    ctx.synchronize()
    ref_idx = idx.cpu().numpy()
    ref_sc = pred.cpu().numpy()[ref_idx]
    with tempfile.TemporaryDirectory() as d:
        _run(_select_worker, world, n, k, d)
        for r in range(world):
            assert (np.load(os.path.join(d, f"idx{r}.npy")) == ref_idx).all(), f"rank {r} indices"
            assert (np.load(os.path.join(d, f"sc{r}.npy")).view(np.uint64) == ref_sc.view(np.uint64)).all()


def _search_worker(rank, world, port, out_dir):
    import sys
    sys.path[:0] = [HERE, os.path.dirname(HERE)]
    import torch.distributed as dist
    from etune_testlib import parse_op
    from paper_2411_18873_b200 import capi
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = capi.Context(0)
    capi.attach_torch_transport(ctx)
    plan = capi.Plan(ctx, parse_op("mm:1,256,256,256"))
    cfg = capi.search_config(M=256, generation_size=1024, rng_seed=11, max_rounds=4, patience=1 << 30)
    s = capi.Search(plan, cfg)
    reps = s.run()
    rows = [[r.round, r.k_before_fifths, r.k_after_fifths, r.measured, r.cumulative_measured, r.best_id,
             np.float64(r.best_latency_ms).view(np.uint64), np.float64(r.best_energy_mj).view(np.uint64),
             np.float64(r.snr_db).view(np.uint64)] for r in reps]
    np.save(os.path.join(out_dir, f"rep{rank}.npy"), np.array(rows, dtype=np.uint64))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_search_matches_single():
    """Algorithm 1 with the population sharded over 2 ranks (latency filter per shard + merge,
    energy measurements split, training on rank 0 + broadcast) reports exactly the single-rank
    rounds."""
    from etune_testlib import parse_op
    from paper_2411_18873_b200 import capi
    ctx = capi.Context(0)
    plan = capi.Plan(ctx, parse_op("mm:1,256,256,256"))
    cfg = capi.search_config(M=256, generation_size=1024, rng_seed=11, max_rounds=4, patience=1 << 30)
    reps = capi.Search(plan, cfg).run()
    ref = np.array([[r.round, r.k_before_fifths, r.k_after_fifths, r.measured, r.cumulative_measured, r.best_id,
                     np.float64(r.best_latency_ms).view(np.uint64), np.float64(r.best_energy_mj).view(np.uint64),
                     np.float64(r.snr_db).view(np.uint64)] for r in reps], dtype=np.uint64)
    with tempfile.TemporaryDirectory() as d:
        _run(_search_worker, 2, d)
        for r in range(2):
            assert (np.load(os.path.join(d, f"rep{r}.npy")) == ref).all(), f"rank {r} round reports"
