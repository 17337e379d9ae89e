"""GPU parity of the fused score + keep-the-best (etune_cu_score_select): the score
kernel buckets every prediction, the selection resolves the k-th key's bucket.  The
selected indices must equal the oracle's (prediction asc, index asc) top-k of the
oracle's predictions, bit for bit, for any population: distinct scores, heavy ties
(bucket larger than the finish CTA's shared-memory cache), every score equal, k at
the bucket edges, repeated calls (the work area resets itself)."""
import numpy as np
import pytest

from etune_testlib import FlatForest, parse_op

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

OP = "conv:1,56,56,64,64,3,1,1"
MODEL = "c2_r50_conv3x3"


@pytest.fixture(scope="module")
def capi():
    from paper_2411_18873_b200 import capi as c
    return c


@pytest.fixture(scope="module")
def ctx(capi):
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return capi.Context(0)


@pytest.fixture(scope="module")
def setup(golden, oracle, ctx, capi):
    k = f"{MODEL}/model/"
    flat = FlatForest(golden[k + "feature"], golden[k + "threshold"], golden[k + "left"], golden[k + "right"],
                      golden[k + "value"], golden[k + "offsets"], float(golden[k + "base_score"][0]),
                      float(golden[k + "learning_rate"][0]))
    op = parse_op(OP)
    plan = capi.Plan(ctx, op)
    forest = capi.Forest.from_flat(ctx, flat)
    parents, _ = oracle.sample_random(op, 1024, 42)
    return op, plan, forest, flat, parents


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_select(capi, ctx, plan, forest, sched, k):
    g = plan.encode(dev(sched))
    n = len(sched)
    pred = torch.empty(n, dtype=torch.float64, device="cuda")
    idx = torch.empty(max(k, 1), dtype=torch.int64, device="cuda")
    forest.score_select(plan, g, k, pred, idx)
    ctx.synchronize()
    return pred.cpu().numpy(), idx.cpu().numpy()[:k]


def expect(oracle, op, flat, sched, k):
    p = oracle.predict(flat, oracle.features(op, sched))
    return p, oracle.topk(p, k)


@pytest.mark.parametrize("n,k", [(1, 1), (37, 5), (4096, 4096), (100003, 1024), (1 << 18, 4096), (1 << 18, 1),
                                 (1 << 18, 1000)])
def test_score_select_bred_population(oracle, ctx, capi, setup, n, k):
    op, plan, forest, flat, parents = setup
    sched = oracle.reproduce(op, parents, n, 7 + n)[0] if n > 1024 else parents[:n]
    p_ref, want = expect(oracle, op, flat, sched, k)
    pred, got = run_select(capi, ctx, plan, forest, sched, k)
    assert (pred.view(np.uint64) == p_ref.view(np.uint64)).all()
    assert (got == want).all()


@pytest.mark.parametrize("distinct,n,k", [(1, 50000, 1024), (3, 30000, 4096), (40, 200000, 3000), (7, 9000, 8)])
def test_score_select_heavy_ties(oracle, ctx, capi, setup, distinct, n, k):
    """Few distinct schedules replicated: bucket d* holds whole tie groups (often more
    pairs than the finish CTA caches), ties resolve by lowest index."""
    op, plan, forest, flat, parents = setup
    rng = np.random.default_rng(distinct * 1000 + n)
    sched = parents[rng.integers(0, distinct, n) if distinct > 1 else np.zeros(n, np.int64)]
    p_ref, want = expect(oracle, op, flat, sched, k)
    pred, got = run_select(capi, ctx, plan, forest, sched, k)
    assert (pred.view(np.uint64) == p_ref.view(np.uint64)).all()
    assert (got == want).all()


def test_score_select_matches_unfused_and_resets(oracle, ctx, capi, setup):
    """Back-to-back calls on different populations (no host sync between them) equal
    score + cooperative top-k: the histogram and list counters reset in-kernel."""
    op, plan, forest, flat, parents = setup
    pops = [oracle.reproduce(op, parents, 60000, s)[0] for s in (1, 2, 3)]
    gs = [plan.encode(dev(s)) for s in pops]
    outs = []
    for g in gs:
        pred = torch.empty(len(g), dtype=torch.float64, device="cuda")
        idx = torch.empty(2048, dtype=torch.int64, device="cuda")
        forest.score_select(plan, g, 2048, pred, idx)
        outs.append((pred, idx))
    ctx.synchronize()
    for (pred, idx), s in zip(outs, pops):
        ref = capi.topk(ctx, pred, 2048)
        ctx.synchronize()
        assert (idx.cpu().numpy() == ref.cpu().numpy()).all()
        _, want = expect(oracle, op, flat, s, 2048)
        assert (idx.cpu().numpy() == want).all()


def test_score_select_large_k_falls_back(oracle, ctx, capi, setup):
    op, plan, forest, flat, parents = setup
    sched = oracle.reproduce(op, parents, 50000, 11)[0]
    _, want = expect(oracle, op, flat, sched, 10000)
    _, got = run_select(capi, ctx, plan, forest, sched, 10000)
    assert (got == want).all()


def test_score_select_empty_and_k0(oracle, ctx, capi, setup):
    """Edge sizes of the fused call: an empty population (k = 0), k = 0 on a non-empty one
    (predictions still written, no selection), and the k > n / negative-k errors."""
    op, plan, forest, flat, parents = setup
    g0 = plan.encode(dev(parents[:0]))
    forest.score_select(plan, g0, 0, torch.empty(0, dtype=torch.float64, device="cuda"),
                        torch.empty(1, dtype=torch.int64, device="cuda"))
    sched = parents[:777]
    p_ref, _ = expect(oracle, op, flat, sched, 1)
    pred, got = run_select(capi, ctx, plan, forest, sched, 0)
    assert len(got) == 0
    assert (pred.view(np.uint64) == p_ref.view(np.uint64)).all()
    g = plan.encode(dev(sched))
    pr = torch.empty(len(sched), dtype=torch.float64, device="cuda")
    ix = torch.empty(1024, dtype=torch.int64, device="cuda")
    for bad_k in (len(sched) + 1, -1):
        with pytest.raises(capi.EtuneError):
            forest.score_select(plan, g, bad_k, pr, ix)
    # the host-buffer entry point on an empty and a one-row population
    forest.score_host(plan, np.ascontiguousarray(sched[:0]), np.zeros(0), np.zeros(0, np.uint64))
    p1, h1 = np.zeros(1), np.zeros(1, np.uint64)
    forest.score_host(plan, np.ascontiguousarray(sched[:1]), p1, h1)
    assert p1.view(np.uint64)[0] == p_ref.view(np.uint64)[0]
    assert h1[0] == np.uint64(oracle.ids(op, sched[:1])[0])


def test_score_select_sharded_single_rank(oracle, ctx, capi, setup):
    """Shards scored + selected locally, merged (single-rank communicator semantics):
    per-shard results equal the oracle's shard top-k with global indices."""
    op, plan, forest, flat, parents = setup
    sched = oracle.reproduce(op, parents, 120000, 5)[0]
    p_ref = oracle.predict(flat, oracle.features(op, sched))
    lo, hi, k = 40000, 120000, 1024
    g = plan.encode(dev(sched[lo:hi]))
    pred = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    sc = torch.empty(k, dtype=torch.float64, device="cuda")
    forest.score_select_sharded(plan, g, lo, k, pred, idx, sc)
    ctx.synchronize()
    want = lo + oracle.topk(p_ref[lo:hi], k)
    assert (idx.cpu().numpy() == want).all()
    assert (sc.cpu().numpy().view(np.uint64) == p_ref[want].view(np.uint64)).all()


def test_profile_score_events(oracle, ctx, capi, setup):
    op, plan, forest, flat, parents = setup
    sched = oracle.reproduce(op, parents, 1 << 16, 3)[0]
    g = plan.encode(dev(sched))
    pred = torch.empty(len(sched), dtype=torch.float64, device="cuda")
    idx = torch.empty(64, dtype=torch.int64, device="cuda")
    capi.profile_score(ctx, True)
    for _ in range(3):
        forest.score_select(plan, g, 64, pred, idx)
    sort_ms, ms, sel_ms, cnt = capi.profile_score(ctx, False)
    assert cnt == 3 and ms > 0.0 and sel_ms > 0.0 and sort_ms > 0.0


@pytest.mark.parametrize("text,model", [("conv:1,56,56,64,64,3,1,1", "c2_r50_conv3x3"),
                                        ("mm:1,1024,1024,1024", "c1_gemm1024"),
                                        ("mm:1,512,3072,768", "c3_bert_ffn"),
                                        ("conv:4,14,14,64,32,3,1,1", "c2_r50_conv3x3")])
def test_keyed_path_matches_class_tables_and_oracle(golden, oracle, ctx, capi, text, model):
    """The keyed path (key sort + key-table rows) and the class-table kernel give the
    same bits as the oracle, for scores, ids and the selection."""
    k = f"{model}/model/"
    flat = FlatForest(golden[k + "feature"], golden[k + "threshold"], golden[k + "left"], golden[k + "right"],
                      golden[k + "value"], golden[k + "offsets"], float(golden[k + "base_score"][0]),
                      float(golden[k + "learning_rate"][0]))
    op = parse_op(text)
    plan = capi.Plan(ctx, op)
    n = 100000
    par, _ = oracle.sample_random(op, 512, 3)
    sched, ids_ref, _, _ = oracle.reproduce(op, par, n, 17)
    p_ref = oracle.predict(flat, oracle.features(op, sched))
    g = plan.encode(dev(sched))
    outs = []
    for keyed in (1, 2, 0):
        fo = capi.Forest.from_flat(ctx, flat).set_keyed(keyed)
        pred = torch.empty(n, dtype=torch.float64, device="cuda")
        ids = torch.empty(n, dtype=torch.int64, device="cuda")
        idx = torch.empty(1024, dtype=torch.int64, device="cuda")
        fo.score_select(plan, g, 1024, pred, idx, ids=ids)
        ctx.synchronize()
        outs.append((pred.cpu().numpy(), capi.as_u64(ids), idx.cpu().numpy()))
    for pred, ids, idx in outs:
        assert (pred.view(np.uint64) == p_ref.view(np.uint64)).all()
        assert (ids == ids_ref).all()
        assert (idx == oracle.topk(p_ref, 1024)).all()


@pytest.mark.parametrize("trees", [1, 24, 25, 26, 49, 50, 51, 77, 128])
def test_keyed_full_form_tree_counts(golden, oracle, ctx, capi, trees):
    """Full-form rows hold 25 exit slots per 16-byte quad and are read one 32-byte sector
    at a time: forests whose tree count ends inside a quad, on a quad or sector edge, or
    at the 128-tree limit (the golden forest's trees repeated) score bit-exactly."""
    k = "c2_r50_conv3x3/model/"
    off0 = np.asarray(golden[k + "offsets"], np.int64)
    reps = (trees + 99) // 100
    cols = {c: np.concatenate([golden[k + c]] * reps) for c in ("feature", "threshold", "left", "right", "value")}
    off = np.concatenate([off0[:-1] + r * off0[-1] for r in range(reps)] + [[reps * off0[-1]]])[: trees + 1]
    nn = int(off[-1])
    flat = FlatForest(*(np.ascontiguousarray(cols[c][:nn]) for c in ("feature", "threshold", "left", "right",
                                                                     "value")),
                      off, float(golden[k + "base_score"][0]), float(golden[k + "learning_rate"][0]))
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    plan = capi.Plan(ctx, op)
    parents, _ = oracle.sample_random(op, 1024, 42)
    sched = oracle.reproduce(op, parents, 1 << 16, 5 + trees)[0]  # >= 2^16: the keyed form is compiled
    p_ref = oracle.predict(flat, oracle.features(op, sched))
    fo = capi.Forest.from_flat(ctx, flat).set_keyed(1)
    assert fo.score_form(plan) == "keyed-full"
    pred, ids = fo.score(plan, plan.encode(dev(sched)), with_ids=True)
    ctx.synchronize()
    assert (pred.cpu().numpy().view(np.uint64) == p_ref.view(np.uint64)).all()
    assert (ids.cpu().numpy().view(np.uint64) == oracle.ids(op, sched).astype(np.uint64)).all()
