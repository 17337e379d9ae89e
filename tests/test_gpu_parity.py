"""GPU parity: the CUDA path (through the C ABI) vs the oracle and the reference's
golden vectors.  Bit-exact for everything (ids, counters, features, predictions,
selected indices); predictions are compared on their IEEE bit patterns, i.e. the
stated tolerance is 0 ulp (north_star allows 1e-5 relative; we meet 0)."""
import numpy as np
import pytest

from etune_testlib import EtuneError as OracleError
from etune_testlib import FlatForest, parse_op
from golden.make_golden import MODEL_OPS, OPS

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NAMES = [n for n, _, _ in OPS]


@pytest.fixture(scope="module")
def capi():
    from paper_2411_18873_b200 import capi as c
    return c


@pytest.fixture(scope="module")
def ctx(capi):
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return capi.Context(0)


def forest_of(golden, name):
    k = f"{name}/model/"
    return FlatForest(golden[k + "feature"], golden[k + "threshold"], golden[k + "left"], golden[k + "right"],
                      golden[k + "value"], golden[k + "offsets"], float(golden[k + "base_score"][0]),
                      float(golden[k + "learning_rate"][0]))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def bits(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("name", NAMES)
def test_codec_ids_counters_features_golden(golden, ctx, capi, name):
    op = golden[f"{name}/op"]
    s = golden[f"{name}/sample_sched"]
    for sms, fkey in ((108, "features_bits"), (148, "features_bits_sms148")):
        plan = capi.Plan(ctx, op, num_sms=sms)
        assert (plan.nest() == golden[f"{name}/nest"]).all()
        assert plan.space_size() == golden[f"{name}/space"][0]
        g = plan.encode(dev(s))
        ctx.synchronize()
        assert (plan.decode(g).cpu().numpy() == s).all()
        assert (capi.as_u64(plan.ids(g)) == golden[f"{name}/sample_ids"]).all()
        f, ids = plan.features(g, with_ids=True)
        assert (bits(f) == golden[f"{name}/{fkey}"]).all()
        assert (capi.as_u64(ids) == golden[f"{name}/sample_ids"]).all()
        if sms == 108:
            assert (plan.counters(g).cpu().numpy() == golden[f"{name}/counters"]).all()


@pytest.mark.parametrize("text", ["mm:1,8,8,8", "mm:2,4,4,4", "mv:1,1,8,8", "conv:1,6,6,2,2,3,1,1",
                                  "conv:2,4,4,2,2,1,1,0", "mm:1,64,64,64", "mm:1,16,16,16",
                                  "conv:1,5,5,1,3,3,1,1", "mm:3,12,18,10"])
def test_full_space_vs_oracle(oracle, ctx, capi, text):
    op = parse_op(text)
    full = oracle.enumerate(op)
    plan = capi.Plan(ctx, op)
    assert plan.space_size() == len(full)
    g = plan.encode(dev(full))
    ctx.synchronize()
    assert (capi.as_u64(plan.ids(g)) == oracle.ids(op, full)).all()
    assert (plan.counters(g).cpu().numpy() == oracle.counters(op, full)).all()
    assert (bits(plan.features(g)) == oracle.features(op, full).view(np.uint64)).all()


@pytest.mark.parametrize("text", ["mm:1,1024,1024,1024", "conv:1,56,56,64,64,3,1,1", "mm:1,512,3072,768",
                                  "conv:1,14,14,256,256,3,1,1", "mv:1,1,1000,2048", "conv:1,28,28,128,512,1,1,0",
                                  "mm:8,384,384,64"])
def test_large_samples_vs_oracle(oracle, ctx, capi, text):
    op = parse_op(text)
    s, ids = oracle.sample_random(op, min(20000, oracle.count(op)), 42)
    plan = capi.Plan(ctx, op, num_sms=148)
    g = plan.encode(dev(s))
    f, dids = plan.features(g, with_ids=True)
    ctx.synchronize()
    assert (capi.as_u64(dids) == ids).all()
    assert (bits(f) == oracle.features(op, s, 148).view(np.uint64)).all()


@pytest.mark.parametrize("name", MODEL_OPS)
def test_score_and_predict_golden(golden, oracle, ctx, capi, name):
    op = golden[f"{name}/op"]
    fl = forest_of(golden, name)
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    s = golden[f"{name}/sample_sched"]
    g = plan.encode(dev(s))
    pred, ids = fo.score(plan, g, with_ids=True)
    ctx.synchronize()
    assert (bits(pred) == golden[f"{name}/model/pred_bits"]).all()
    assert (capi.as_u64(ids) == golden[f"{name}/sample_ids"]).all()
    p2 = fo.predict(plan.features(g))
    assert (bits(p2) == golden[f"{name}/model/pred_bits"]).all()


@pytest.mark.parametrize("name", MODEL_OPS)
def test_score_population_vs_oracle(golden, oracle, ctx, capi, name):
    """A reproduce()-bred population (duplicates, every move type) at 2^16."""
    op = golden[f"{name}/op"]
    fl = forest_of(golden, name)
    par, _ = oracle.sample_random(op, 256, 42)
    s, ids, _, _ = oracle.reproduce(op, par, 1 << 16, 7)
    ref = oracle.predict(fl, oracle.features(op, s))
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    pred, dids = fo.score(plan, plan.encode(dev(s)), with_ids=True)
    ctx.synchronize()
    assert (bits(pred) == ref.view(np.uint64)).all()
    assert (capi.as_u64(dids) == ids).all()


def test_score_other_operator_forest(golden, oracle, ctx, capi):
    """A forest trained on one operator applied to another: most tests fold away."""
    fl = forest_of(golden, "c3_bert_ffn")
    op = parse_op("conv:1,7,7,512,512,3,1,1")
    s, _ = oracle.sample_random(op, 5000, 9)
    ref = oracle.predict(fl, oracle.features(op, s))
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    pred = fo.score(plan, plan.encode(dev(s)))
    ctx.synchronize()
    assert (bits(pred) == ref.view(np.uint64)).all()


def test_trained_here_forest(oracle, ctx, capi):
    """Full depth-6 trees (up to 64 leaves: the 64-bit leaf-mask path), trained by the
    oracle on fresh data with min_leaf_weight 0."""
    op = parse_op("mm:1,256,512,384")
    s, _ = oracle.sample_random(op, 1500, 3)
    f = oracle.features(op, s)
    e = 1.0 + (f[:, 2] * 0.3 + f[:, 12] * 0.1 + f[:, 6]) % 2.7
    fl, _, _ = oracle.train(f, e, num_trees=40, max_depth=6, min_leaf_weight=0.0)
    pop, _ = oracle.sample_random(op, 30000, 4)
    ref = oracle.predict(fl, oracle.features(op, pop))
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    pred = fo.score(plan, plan.encode(dev(pop)))
    ctx.synchronize()
    assert (bits(pred) == ref.view(np.uint64)).all()


@pytest.mark.parametrize("n,k", [(1, 1), (1000, 7), (4096, 4096), (70001, 1024), (1 << 20, 262144)])
def test_topk_vs_oracle(oracle, ctx, capi, n, k):
    rng = np.random.default_rng(n)
    # heavy ties like real predictions: few distinct values
    vals = rng.choice(rng.uniform(0.9, 3.0, 300), n)
    idx = capi.topk(ctx, dev(vals), k)
    ctx.synchronize()
    assert (idx.cpu().numpy() == oracle.topk(vals, k)).all()


def test_illegal_schedule_reported_with_index(golden, ctx, capi):
    op = golden["c1_gemm1024/op"]
    s = golden["c1_gemm1024/sample_sched"].copy()
    s[37, 10] = 3  # unroll not a power of two
    s[90, 1] = 5   # tiling no longer multiplies to the extent
    plan = capi.Plan(ctx, op)
    plan.encode(dev(s))
    with pytest.raises(capi.EtuneError) as e:
        ctx.synchronize()
    assert e.value.code == 4 and e.value.index == 37
    ctx.synchronize()  # error state is cleared


def test_invalid_operator(ctx, capi):
    with pytest.raises(capi.EtuneError) as e:
        capi.Plan(ctx, parse_op("conv:1,224,224,3,64,7,2,3"))  # stride-2 R50 conv1
    assert e.value.code == 2


def test_score_host_e2e(golden, oracle, ctx, capi):
    name = "c2_r50_conv3x3"
    op = golden[f"{name}/op"]
    fl = forest_of(golden, name)
    s, ids = oracle.sample_random(op, 300000, 5)
    ref = oracle.predict(fl, oracle.features(op, s))
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    pred = np.zeros(len(s))
    hid = np.zeros(len(s), np.uint64)
    fo.score_host(plan, s, pred, hid)
    assert (pred.view(np.uint64) == ref.view(np.uint64)).all()
    assert (hid == ids).all()
    s[299999, 9] = 7  # k_tile not dividing K -> IllegalSchedule at that index
    with pytest.raises(capi.EtuneError) as e:
        fo.score_host(plan, s, pred, hid)
    assert e.value.code == 4 and e.value.index == 299999


@pytest.mark.parametrize("text,n,pinned", [("mm:1,131072,256,256", 140000, False),
                                           ("conv:1,56,56,64,64,3,1,1", 400001, False),
                                           ("conv:1,56,56,64,64,3,1,1", 400001, True)])
def test_score_host_row_widths(golden, oracle, ctx, capi, text, n, pinned):
    """score_host narrows rows on the host: u16 fields, u32 when a value needs it
    (M = 2^17 tilings), the reference layout when a field is negative; pinned and
    pageable caller buffers.  The error index of an illegal row stays exact across
    chunks."""
    fl = forest_of(golden, "c2_r50_conv3x3")
    op = parse_op(text)
    s, ids = oracle.sample_random(op, n, 9)
    if pinned:
        s = torch.from_numpy(s).pin_memory().numpy()
    ref = oracle.predict(fl, oracle.features(op, s))
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    pred = np.zeros(n)
    hid = np.zeros(n, np.uint64)
    fo.score_host(plan, s, pred, hid)
    assert (pred.view(np.uint64) == ref.view(np.uint64)).all()
    assert (hid == ids).all()
    if text.startswith("mm"):
        assert s[:, :9].max() >= 1 << 16  # the u32 path was taken
    bad = n - 2
    s[bad, 1] = -1
    with pytest.raises(capi.EtuneError) as e:
        fo.score_host(plan, s, pred, hid)
    assert e.value.code == 4 and e.value.index == bad
    # an illegal row in the first chunk (copied raw, without host narrowing, when pinned)
    s[bad, 1] = s[bad + 1, 1]
    s[5, 1] = -1
    with pytest.raises(capi.EtuneError) as e:
        fo.score_host(plan, s, pred, hid)
    assert e.value.code == 4 and e.value.index == 5


@pytest.mark.parametrize("depth,smooth", [(8, False), (6, True)])
def test_score_general_walk_path(oracle, ctx, capi, depth, smooth):
    """Forests whose compiled form is unsupported (> 64 leaves per tree) or does not fit
    shared memory (hundreds of outcome classes) take the general features + tree-walk
    kernel; results stay bit-exact."""
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    s, _ = oracle.sample_random(op, 3000, 77)
    f = oracle.features(op, s)
    if smooth:
        e = 1.0 + (f[:, 2] * 0.2 + f[:, 13] + f[:, 10] * 0.1) % 1.9
    else:
        e = 1.0 + (f[:, 1] * 0.37 + f[:, 9] * 0.11 + f[:, 13]) % 2.3
    fl, _, _ = oracle.train(f, e, num_trees=60, max_depth=depth, min_leaf_weight=0.0)
    pop, ids = oracle.sample_random(op, 40000, 5)
    ref = oracle.predict(fl, oracle.features(op, pop))
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    pred, dids = fo.score(plan, plan.encode(dev(pop)), with_ids=True)
    ctx.synchronize()
    assert (bits(pred) == ref.view(np.uint64)).all()
    assert (capi.as_u64(dids) == ids).all()


def _topk_case(kind, n):
    rng = np.random.default_rng(n)
    if kind == "all_equal":
        return np.full(n, 1.25)
    if kind == "hidden_small":  # small values where the stride-n/8192 sample never looks: overflow fallback
        v = rng.uniform(2.0, 3.0, n)
        stride = n // 8192
        mask = (np.arange(n) % stride) != 0
        idx = np.nonzero(mask)[0][:40000]
        v[idx] = rng.uniform(0.5, 0.6, len(idx))
        return v
    if kind == "hidden_large":  # sample sees only the smallest values: too few keys <= T -> fallback
        stride = n // 8192
        v = rng.uniform(5.0, 6.0, n)
        v[::stride] = rng.uniform(0.1, 0.2, len(v[::stride]))
        return v
    if kind == "two_values":
        return rng.choice([0.75, 1.5], n, p=[0.001, 0.999])
    return rng.normal(1.0, 0.1, n)


@pytest.mark.parametrize("kind", ["all_equal", "hidden_small", "hidden_large", "two_values", "normal"])
@pytest.mark.parametrize("n,k", [(1 << 20, 1024), (300000, 4096), (40000, 1)])
def test_topk_fast_path_and_fallback(oracle, ctx, capi, kind, n, k):
    vals = _topk_case(kind, n)
    idx = capi.topk(ctx, dev(vals), k)
    ctx.synchronize()
    assert (idx.cpu().numpy() == oracle.topk(vals, k)).all()
