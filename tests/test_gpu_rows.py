"""GPU parity of the row-table form (rowtab.cu), the default for large populations.

The forest is compiled on the device into one prediction per (tiling-triple key, Kuv class)
row; scoring is a gather.  Every prediction, id and selected index must equal the oracle's
(oracle/etune_oracle.cpp, pinned to the reference by tests/golden) bit for bit, and the row
form must agree with the tree walk and the host-compiled forms on the same population.
Covers: the bench's exact step (2^20 bred candidates, fused top-1024) on C2 and C3, a model
the library has never seen (fresh compile + select), device-trained forests, forests
trained on another operator, depth-8 trees, forests whose threshold lists overflow the
class kernel's shared-memory cache, and re-compiles after a plan is destroyed."""
import numpy as np
import pytest

from etune_testlib import FlatForest, parse_op

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


def bits(t):
    return t.detach().cpu().numpy().view(np.uint64)


def forest_of(golden, name):
    k = f"{name}/model/"
    return FlatForest(golden[k + "feature"], golden[k + "threshold"], golden[k + "left"], golden[k + "right"],
                      golden[k + "value"], golden[k + "offsets"], float(golden[k + "base_score"][0]),
                      float(golden[k + "learning_rate"][0]))


def score_rows(capi, ctx, plan, fl, genome, k=0, form="rows"):
    fo = capi.Forest.from_flat(ctx, fl).set_form(form)
    n = genome.shape[0]
    pred = torch.empty(n, dtype=torch.float64, device="cuda")
    ids = torch.empty(n, dtype=torch.int64, device="cuda")
    idx = torch.empty(max(k, 1), dtype=torch.int64, device="cuda")
    if k:
        fo.score_select(plan, genome, k, pred, idx, ids=ids)
    else:
        fo.score(plan, genome, out=pred, ids_out=ids)
    ctx.synchronize()
    return fo, pred, ids, idx[:k]


BENCH_OPS = [("conv:1,56,56,64,64,3,1,1", "c2_r50_conv3x3"), ("mm:1,512,3072,768", "c3_bert_ffn")]


@pytest.mark.parametrize("text,model", BENCH_OPS)
def test_bench_step_parity(golden, oracle, ctx, capi, text, model):
    """bench.py's exact step: reproduce(sample_random(op, 1024, 42), 2^20, {}, 7) bred on the
    device, row form, fused score + top-1024 -- predictions, ids and the selection vs the
    oracle (8 host threads for the oracle's 2^20 walks)."""
    op = parse_op(text)
    fl = forest_of(golden, model)
    plan = capi.Plan(ctx, op)
    parents = plan.sample_random(1024, 42)
    g, _, _ = capi.reproduce(plan, parents, 1 << 20, 7)
    sched = plan.decode(g).cpu().numpy()
    ref = oracle.score_threads(op, sched, fl, threads=8)
    ref_ids = oracle.ids(op, sched)
    fo, pred, ids, idx = score_rows(capi, ctx, plan, fl, g, k=1024)
    assert fo.score_form(plan) == "rows"
    assert (bits(pred) == ref.view(np.uint64)).all()
    assert (capi.as_u64(ids) == ref_ids).all()
    assert (idx.cpu().numpy() == oracle.topk(ref, 1024)).all()
    info = fo.rows_info(plan)
    assert info["rows"] == info["keys"] * info["kuv_classes"] and 0 < info["kuv_classes"] <= info["kuv_domain"]


@pytest.mark.parametrize("name,model", [("c1_gemm1024", "c1_gemm1024"), ("c2_r50_conv3x3", "c2_r50_conv3x3"),
                                        ("c3_bert_ffn", "c3_bert_ffn"), ("mm_1_64_64_64", "mm_1_64_64_64"),
                                        ("r50_fc", "c2_r50_conv3x3"), ("r50_conv_7x7_3x3_512", "c1_gemm1024")])
def test_rows_vs_walk_and_oracle(golden, oracle, ctx, capi, name, model):
    """Row form == tree walk == oracle on a bred 2^16 population of every golden model's op
    (and golden ops scored by another op's model)."""
    op = golden[f"{name}/op"]
    fl = forest_of(golden, model)
    plan = capi.Plan(ctx, op)
    par, _ = oracle.sample_random(op, min(256, oracle.count(op)), 42)
    s, ids, _, _ = oracle.reproduce(op, par, 1 << 16, 11)
    ref = oracle.predict(fl, oracle.features(op, s))
    g = plan.encode(dev(s))
    _, pr, dids, _ = score_rows(capi, ctx, plan, fl, g, form="rows")
    _, pw, _, _ = score_rows(capi, ctx, plan, fl, g, form="walk")
    assert (bits(pr) == ref.view(np.uint64)).all()
    assert (bits(pw) == ref.view(np.uint64)).all()
    assert (capi.as_u64(dids) == ids).all()


def test_golden_sample_predictions(golden, ctx, capi):
    """The reference's own predictions (pred_bits written by oracle/_ref) through the row form."""
    for name in ("c1_gemm1024", "c2_r50_conv3x3", "c3_bert_ffn", "mm_1_64_64_64"):
        op = golden[f"{name}/op"]
        plan = capi.Plan(ctx, op)
        g = plan.encode(dev(golden[f"{name}/sample_sched"]))
        _, pred, ids, _ = score_rows(capi, ctx, plan, forest_of(golden, name), g)
        assert (bits(pred) == golden[f"{name}/model/pred_bits"]).all(), name
        assert (capi.as_u64(ids) == golden[f"{name}/sample_ids"]).all(), name


def test_fresh_model_c3(oracle, ctx, capi):
    """A model the library has never seen (trained here by the oracle on fresh data),
    compiled on first use and selected from at once: C3, 2^18 candidates, k = 777."""
    op = parse_op("mm:1,512,3072,768")
    s, _ = oracle.sample_random(op, 2048, 1234)
    f = oracle.features(op, s)
    e = 1.0 + (f[:, 2] * 0.31 + f[:, 10] * 0.17 + f[:, 7] * 0.05 + f[:, 13]) % 2.1
    fl, _, _ = oracle.train(f, e, num_trees=100, max_depth=6)
    plan = capi.Plan(ctx, op)
    parents = plan.sample_random(512, 3)
    g, _, _ = capi.reproduce(plan, parents, 1 << 18, 19)
    sched = plan.decode(g).cpu().numpy()
    ref = oracle.score_threads(op, sched, fl, threads=8)
    fo, pred, _, idx = score_rows(capi, ctx, plan, fl, g, k=777, form="auto")
    assert fo.score_form(plan) == "rows"
    assert (bits(pred) == ref.view(np.uint64)).all()
    assert (idx.cpu().numpy() == oracle.topk(ref, 777)).all()


def test_device_trained_forest(oracle, ctx, capi):
    """Forest trained by etune_cu_train, scored through the row form without leaving the device."""
    op = parse_op("conv:1,28,28,128,128,3,1,1")
    plan = capi.Plan(ctx, op)
    g0 = plan.sample_random(3000, 5)
    s0 = plan.decode(g0).cpu().numpy()
    feats = plan.features(g0)
    f_host = feats.cpu().numpy()
    e = 1.0 + (f_host[:, 1] * 0.21 + f_host[:, 6] * 0.4 + f_host[:, 11] * 0.07) % 1.7
    tm = capi.train(ctx, feats, dev(e), num_trees=100, max_depth=6)
    fo = tm.forest().set_form("rows")
    parents = plan.sample_random(256, 8)
    g, _, _ = capi.reproduce(plan, parents, 1 << 17, 23)
    pred = fo.score(plan, g)
    ctx.synchronize()
    fe, th, le, ri, va, off, base, _, _ = tm.host()
    fl = FlatForest(fe, th, le, ri, va, off, base, 0.1)
    ref = oracle.score_threads(op, plan.decode(g).cpu().numpy(), fl, threads=8)
    assert (bits(pred) == ref.view(np.uint64)).all()
    del s0


def test_other_operator_forest(golden, oracle, ctx, capi):
    """A forest trained on BERT's FFN GEMM applied to a 7x7 conv: most tests never split its rows."""
    fl = forest_of(golden, "c3_bert_ffn")
    op = parse_op("conv:1,7,7,512,512,3,1,1")
    par, _ = oracle.sample_random(op, 512, 9)
    s, _, _, _ = oracle.reproduce(op, par, 100000, 4)
    ref = oracle.predict(fl, oracle.features(op, s))
    plan = capi.Plan(ctx, op)
    _, pred, _, idx = score_rows(capi, ctx, plan, fl, plan.encode(dev(s)), k=4096)
    assert (bits(pred) == ref.view(np.uint64)).all()
    assert (idx.cpu().numpy() == oracle.topk(ref, 4096)).all()


@pytest.mark.parametrize("depth,trees", [(8, 60), (6, 300)])
def test_deep_and_wide_forests(oracle, ctx, capi, depth, trees):
    """Depth-8 trees (walked from global memory when the node array exceeds shared memory)
    and 300 trees; f10 / f7 / f6 tested often."""
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    s, _ = oracle.sample_random(op, 4000, 77)
    f = oracle.features(op, s)
    e = 1.0 + (f[:, 10] * 0.37 + f[:, 7] * 0.11 + f[:, 6] * 0.3 + f[:, 13]) % 2.3
    fl, _, _ = oracle.train(f, e, num_trees=trees, max_depth=depth, min_leaf_weight=0.0)
    pop, ids = oracle.sample_random(op, 60000, 5)
    ref = oracle.predict(fl, oracle.features(op, pop))
    plan = capi.Plan(ctx, op)
    _, pred, dids, _ = score_rows(capi, ctx, plan, fl, plan.encode(dev(pop)))
    assert (bits(pred) == ref.view(np.uint64)).all()
    assert (capi.as_u64(dids) == ids).all()


def test_threshold_cache_overflow(oracle, ctx, capi):
    """More than 1024 thresholds on one Kuv feature: the class kernel reads the list from
    global memory instead of its shared-memory cache.  Synthetic forest: 1200 stumps on f10
    with distinct thresholds, plus stumps on f7 and f6."""
    op = parse_op("mm:1,256,256,1024")
    rng = np.random.default_rng(3)
    feats, thr = [], []
    for j in range(1400):
        fidx = 10 if j < 1200 else (7 if j < 1300 else 6)
        lo, hi = (0.0, 8.0) if fidx == 10 else (0.5, 40.0) if fidx == 7 else (0.5, 5.0)
        feats.append(fidx)
        thr.append(rng.uniform(lo, hi))
    T = len(feats)
    feature = np.empty(3 * T, np.int32)
    threshold = np.zeros(3 * T)
    left = np.full(3 * T, -1, np.int32)
    right = np.full(3 * T, -1, np.int32)
    value = np.zeros(3 * T)
    for t in range(T):
        feature[3 * t:3 * t + 3] = (feats[t], -1, -1)
        threshold[3 * t] = thr[t]
        left[3 * t], right[3 * t] = 1, 2
        value[3 * t + 1], value[3 * t + 2] = rng.normal(0, 0.01, 2)
    fl = FlatForest(feature, threshold, left, right, value, np.arange(0, 3 * T + 1, 3, dtype=np.int64), 1.5, 0.1)
    par, _ = oracle.sample_random(op, 512, 1)
    s, _, _, _ = oracle.reproduce(op, par, 1 << 16, 2)
    ref = oracle.predict(fl, oracle.features(op, s))
    plan = capi.Plan(ctx, op)
    fo, pred, _, _ = score_rows(capi, ctx, plan, fl, plan.encode(dev(s)))
    assert fo.rows_info(plan)["thr_f10"] == 1200
    assert (bits(pred) == ref.view(np.uint64)).all()


def test_plan_destroy_evicts_and_recompiles(golden, oracle, ctx, capi):
    """Destroying a plan frees the forms compiled for it; a new plan of the same op compiles
    again and still scores bit-exactly."""
    fl = forest_of(golden, "c2_r50_conv3x3")
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    par, _ = oracle.sample_random(op, 128, 2)
    s, _, _, _ = oracle.reproduce(op, par, 70000, 3)
    ref = oracle.predict(fl, oracle.features(op, s)).view(np.uint64)
    fo = capi.Forest.from_flat(ctx, fl)
    for _ in range(3):
        plan = capi.Plan(ctx, op)
        pred = fo.score(plan, plan.encode(dev(s)))
        ctx.synchronize()
        assert (bits(pred) == ref).all()
        assert fo.rows_info(plan)["rows"] > 0
        del plan


def test_auto_small_population_walks(golden, ctx, capi):
    """AUTO: a model scoring a few thousand candidates once walks (no compile); past 2^16
    cumulative candidates it switches to the row table; results identical."""
    fl = forest_of(golden, "c2_r50_conv3x3")
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    plan = capi.Plan(ctx, op)
    g = plan.sample_random(4096, 42)
    fo = capi.Forest.from_flat(ctx, fl)
    p0 = fo.score(plan, g)
    ctx.synchronize()
    assert fo.rows_info(plan)["rows"] == 0
    outs = [fo.score(plan, g) for _ in range(16)]
    ctx.synchronize()
    assert fo.rows_info(plan)["rows"] > 0
    for p in outs:
        assert (bits(p) == bits(p0)).all()


@pytest.mark.parametrize("radix", [False, True])
@pytest.mark.parametrize("kind,n,k", [("dup", 1, 1), ("dup", 70001, 4096), ("few", 100003, 1024),
                                      ("few", 513, 513), ("bred", 300000, 1), ("bred", 1 << 21, 1024),
                                      ("bred", (1 << 20) + 7, 4096), ("rand", 300001, 4096),
                                      ("rand", 600000, 1024), ("rand", 5000, 17)])
def test_rows_fused_select_edges(golden, oracle, ctx, capi, monkeypatch, kind, n, k, radix):
    """The one-kernel row selection: all candidates tied (quota split over CTAs by index), a few
    distinct rows repeated, k = n, k = 1, k = 4096, n not a multiple of the CTA size, uniformly
    sampled populations (thousands of candidates below the crossing segment, ranked by counting),
    and 2^21 candidates (beyond the grid: the bucketed fallback) -- on the exact crossing path
    (segments of <= 64 groups) and on the radix-select path (ETUNE_ROWSEL_RADIX=1, the path of
    operators with > 2^18 row groups)."""
    if radix:
        monkeypatch.setenv("ETUNE_ROWSEL_RADIX", "1")
    fl = forest_of(golden, "c2_r50_conv3x3")
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    plan = capi.Plan(ctx, op)
    if kind == "bred":
        g, _, _ = capi.reproduce(plan, plan.sample_random(1024, 42), n, 13)
    elif kind == "rand":
        g = plan.sample_random(n, 9)
    else:
        base = plan.sample_random(1 if kind == "dup" else 37, 5)
        g = base[torch.arange(n, device="cuda") % base.shape[0]].contiguous()
    sched = plan.decode(g).cpu().numpy()
    ref = oracle.score_threads(op, sched, fl, threads=8)
    _, pred, _, idx = score_rows(capi, ctx, plan, fl, g, k=k)
    assert (bits(pred) == ref.view(np.uint64)).all()
    assert (idx.cpu().numpy() == oracle.topk(ref, k)).all()
    # repeated calls: the work area and the row counters reset themselves
    _, _, _, idx2 = score_rows(capi, ctx, plan, fl, g, k=k)
    assert (idx2.cpu().numpy() == idx.cpu().numpy()).all()


@pytest.mark.parametrize("pinned", [False, True])
def test_score_select_host(golden, oracle, ctx, capi, pinned):
    """The reference-facing score + keep-the-best on HOST Schedule rows (pageable and pinned):
    predictions and the sorted top-k vs the oracle; an illegal row reports its index."""
    fl = forest_of(golden, "c2_r50_conv3x3")
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    par, _ = oracle.sample_random(op, 1024, 42)
    s, _, _, _ = oracle.reproduce(op, par, 300001, 7)
    ref = oracle.score_threads(op, s, fl, threads=8)
    plan = capi.Plan(ctx, op)
    fo = capi.Forest.from_flat(ctx, fl)
    hs = np.ascontiguousarray(s, np.int64)
    if pinned:
        hs = torch.from_numpy(hs).pin_memory().numpy()
    pred = np.zeros(len(s))
    idx = np.zeros(1024, np.int64)
    fo.score_select_host(plan, hs, 1024, idx, pred)
    assert (pred.view(np.uint64) == ref.view(np.uint64)).all()
    assert (idx == oracle.topk(ref, 1024)).all()
    bad = 200003
    hs2 = hs.copy()
    hs2[bad, 9] = 7  # k_tile 7 does not divide K = 576
    with pytest.raises(capi.EtuneError) as e:
        fo.score_select_host(plan, hs2, 1024, idx, pred)
    assert e.value.code == 4 and e.value.index == bad
