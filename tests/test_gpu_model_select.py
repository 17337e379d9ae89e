"""GPU parity of the cost-model scalars (energy_loss, snr_db) and of the
population-sharded selection (etune_cu_topk_sharded, NCCL all-gather merge)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2411_18873_b200 import capi as c
    return c


@pytest.fixture(scope="module")
def ctx(capi):
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return capi.Context(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_snr_and_loss_vs_oracle(oracle, ctx, capi, n):
    rng = np.random.default_rng(n)
    m = rng.uniform(0.5, 3.0, n)
    p = m * (1 + rng.normal(0, 0.05, n))
    assert np.float64(capi.snr_db(ctx, dev(p), dev(m))).view(np.uint64) == \
        np.float64(oracle.snr_db(p, m)).view(np.uint64)
    got = capi.energy_loss(ctx, dev(p), dev(m)).cpu().numpy()
    for i in range(0, n, max(1, n // 50)):
        assert (got[i].view(np.uint64) == oracle.energy_loss(p[i], m[i]).view(np.uint64)).all()


def test_snr_edge_cases(oracle, ctx, capi):
    m = np.array([1.0, 2.0, 3.0])
    assert capi.snr_db(ctx, dev(m), dev(m)) == 100.0  # zero error energy -> cap (energy_model.cpp:368)
    with pytest.raises(capi.EtuneError) as e:
        capi.snr_db(ctx, dev(m[:0]), dev(m[:0]))
    assert e.value.code == 11
    bad = m.copy()
    bad[2] = -1.0
    with pytest.raises(capi.EtuneError) as e:
        capi.snr_db(ctx, dev(m), dev(bad))
    assert e.value.code == 6 and e.value.index == 2


@pytest.mark.parametrize("n,k,shards", [(1 << 20, 1024, 1), (100000, 512, 4), (5000, 4096, 3), (300, 1000, 8)])
def test_topk_sharded_single_rank_shards(oracle, ctx, capi, n, k, shards):
    """Without an attached communicator every shard's call is the single-rank case;
    the merge of per-shard results (done here through the same device merge by
    calling it on the concatenated records) must equal the global selection."""
    rng = np.random.default_rng(n + k)
    vals = rng.choice(rng.uniform(0.9, 3.0, 200), n)  # heavy ties
    k = min(k, n)
    want = oracle.topk(vals, k)
    if shards == 1:
        idx, sc = capi.topk_sharded(ctx, dev(vals), 0, k)
        ctx.synchronize()
        assert (idx.cpu().numpy() == want).all()
        assert (sc.cpu().numpy() == vals[want]).all()
        return
    bounds = np.linspace(0, n, shards + 1).astype(np.int64)
    recs_s, recs_g = [], []
    for r in range(shards):
        lo, hi = bounds[r], bounds[r + 1]
        idx, sc = capi.topk_sharded(ctx, dev(vals[lo:hi]), int(lo), k)
        ctx.synchronize()
        m = min(k, hi - lo)
        assert (idx.cpu().numpy()[:m] == lo + oracle.topk(vals[lo:hi], m)).all()
        s = sc.cpu().numpy()
        g = idx.cpu().numpy()
        recs_s.append(s)
        recs_g.append(g)
    # rank-major concatenation, (score, position) selection == (score, gidx) order
    cat_s = np.concatenate(recs_s)
    cat_g = np.concatenate(recs_g)
    pos = capi.topk(ctx, dev(cat_s), k).cpu().numpy()
    assert (cat_g[pos] == want).all()


def test_topk_sharded_nccl_one_rank(oracle, ctx, capi):
    """The NCCL path with a single-rank communicator (only one GPU per call here)."""
    c2 = capi.Context(0)
    capi.attach_nccl(c2, capi.nccl_unique_id(), 1, 0)
    rng = np.random.default_rng(3)
    vals = rng.choice(rng.uniform(0.9, 3.0, 300), 70001)
    idx, sc = capi.topk_sharded(c2, dev(vals), 12345, 777)
    c2.synchronize()
    assert (idx.cpu().numpy() == 12345 + oracle.topk(vals, 777)).all()
    # the fused per-shard score + select + all-gather merge through the communicator
    from etune_testlib import FlatForest, parse_op
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_reference.npz"))
    mk = "c2_r50_conv3x3/model/"
    flat = FlatForest(g[mk + "feature"], g[mk + "threshold"], g[mk + "left"], g[mk + "right"], g[mk + "value"],
                      g[mk + "offsets"], float(g[mk + "base_score"][0]), float(g[mk + "learning_rate"][0]))
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    par, _ = oracle.sample_random(op, 256, 1)
    s, _, _, _ = oracle.reproduce(op, par, 90000, 2)
    ref = oracle.predict(flat, oracle.features(op, s))
    plan = capi.Plan(c2, op)
    fo = capi.Forest.from_flat(c2, flat)
    pred = torch.empty(len(s), dtype=torch.float64, device="cuda")
    gidx = torch.empty(1000, dtype=torch.int64, device="cuda")
    gsc = torch.empty(1000, dtype=torch.float64, device="cuda")
    fo.score_select_sharded(plan, plan.encode(dev(s)), 5000, 1000, pred, gidx, gsc)
    c2.synchronize()
    want = oracle.topk(ref, 1000)
    assert (gidx.cpu().numpy() == 5000 + want).all()
    assert (gsc.cpu().numpy().view(np.uint64) == ref[want].view(np.uint64)).all()
    buf = torch.arange(10, dtype=torch.float64, device="cuda")
    capi.broadcast(c2, buf, 0)
    c2.synchronize()
    assert (buf.cpu().numpy() == np.arange(10)).all()


@pytest.mark.parametrize("text,dev", [
    ("mm:1,512,512,512", {}), ("conv:1,56,56,64,64,3,1,1", {"noise_sigma_rel": 0.0}),
    ("mm:1,512,3072,768", {"num_sms": 148, "rng_seed": 99, "noise_sigma_rel": 0.2}),
    ("mm:1,1,1,1", {}), ("mv:1,1,1000,2048", {"sampler_hz": 30.0, "latency_floor_ms": 0.5})])
def test_sim_measure_vs_oracle(oracle, ctx, capi, text, dev):
    from etune_testlib import parse_op
    op = parse_op(text)
    s, _ = oracle.sample_random(op, min(20000, oracle.count(op)), 3)
    ref = oracle.sim_measure(op, s, dev)
    d = capi.default_device_config(**dev)
    plan = capi.Plan(ctx, op, dev=d)
    g = plan.encode(dev_t(s))
    lat, pw, en, it = plan.sim_measure(g)
    lat_only = plan.sim_measure(g, latency_only=True)
    ctx.synchronize()
    for j, t in enumerate((lat, pw, en)):
        assert (t.cpu().numpy().view(np.uint64) == ref[:, j].view(np.uint64)).all()
    assert (it.cpu().numpy() == ref[:, 3].astype(np.int64)).all()
    assert (lat_only.cpu().numpy().view(np.uint64) == ref[:, 0].view(np.uint64)).all()
    if dev.get("noise_sigma_rel", 0.05) == 0.0:  # SPEC:336 noiseless -> true power exactly
        assert np.allclose(en.cpu().numpy(), pw.cpu().numpy() * lat.cpu().numpy(), rtol=1e-15)


def dev_t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()
