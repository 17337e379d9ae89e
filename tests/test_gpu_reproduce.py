"""GPU parity of etune_cu_reproduce (device reproduce, genetic.cpp:137-187) against the
reference's golden offspring and the oracle: offspring schedules, ids and lineage are
bit-exact (the device consumes the reference's single mt19937_64 stream)."""
import numpy as np
import pytest

from etune_testlib import parse_op
from golden.make_golden import OPS

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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(capi, ctx, op, parents, n, seed, rates=(0.85, 0.10, 0.05), limits=None):
    plan = capi.Plan(ctx, op, limits=limits)
    g = plan.encode(dev(parents))
    out, partner, ids = capi.reproduce(plan, g, n, seed, rates)
    sched = plan.decode(out)
    ctx.synchronize()
    return sched.cpu().numpy(), partner.cpu().numpy(), capi.as_u64(ids)


def check(oracle, capi, op, parents, n, got, seed, rates=(0.85, 0.10, 0.05), limits=None):
    s, ids, lin, ll = oracle.reproduce(op, parents, n, seed, rates, limits)
    gs, gp, gid = got
    assert (gs == s).all()
    assert (gid == ids).all()
    pid = oracle.ids(op, parents)
    base = np.arange(n) % len(parents)
    assert (lin[:, 0] == pid[base]).all()
    cro = gp >= 0
    assert (ll == np.where(cro, 2, 1)).all()
    assert (lin[cro, 1] == pid[gp[cro]]).all()


@pytest.mark.parametrize("name", NAMES)
def test_reproduce_golden(golden, ctx, capi, name):
    op = golden[f"{name}/op"]
    par = golden[f"{name}/repro_parents"]
    gs, gp, gid = run(capi, ctx, op, par, 512, 7)
    assert (gs == golden[f"{name}/repro_sched"]).all()
    assert (gid == golden[f"{name}/repro_ids"]).all()
    lin, ll = golden[f"{name}/repro_lineage"], golden[f"{name}/repro_lineage_len"]
    assert (ll == np.where(gp >= 0, 2, 1)).all()


@pytest.mark.parametrize("text,npar,n,seed", [
    ("conv:1,56,56,64,64,3,1,1", 1024, 1 << 16, 7),
    ("mm:1,1024,1024,1024", 512, 20000, 11),
    ("mm:1,512,3072,768", 2048, 50000, 3),
    ("mm:4,96,200,50", 300, 30000, 5),      # batch > 1: batch-tiling mutations draw
    ("mm:3,12,18,10", 17, 9999, 1),
    ("mv:1,1,1000,2048", 64, 4097, 99),
    ("conv:2,4,4,2,2,1,1,0", 40, 3000, 8),
])
def test_reproduce_vs_oracle(oracle, ctx, capi, text, npar, n, seed):
    op = parse_op(text)
    par, _ = oracle.sample_random(op, min(npar, oracle.count(op)), 42)
    check(oracle, capi, op, par, n, run(capi, ctx, op, par, n, seed), seed)


@pytest.mark.parametrize("rates", [(1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0), (0.3, 0.3, 0.4),
                                   (2.0, 7.0, 1.0)])
def test_reproduce_rates(oracle, ctx, capi, rates):
    op = parse_op("conv:1,28,28,128,512,1,1,0")
    par, _ = oracle.sample_random(op, 200, 4)
    check(oracle, capi, op, par, 20000, run(capi, ctx, op, par, 20000, 12, rates), 12, rates)


def test_reproduce_duplicate_parents(oracle, ctx, capi):
    """Duplicated parent ids: the crossover partner loop (genetic.cpp:172-177) must skip
    equal ids; with ALL parents identical has_other is false and no redraw happens."""
    op = parse_op("mm:1,64,64,64")
    par, _ = oracle.sample_random(op, 8, 3)
    dup = np.concatenate([np.repeat(par[:1], 30, 0), par[1:3]])  # 30 copies + 2 others
    for p in (dup, np.repeat(par[:1], 5, 0), par[:1]):
        check(oracle, capi, op, p, 5000, run(capi, ctx, op, p, 5000, 21, (0.2, 0.8, 0.0)), 21, (0.2, 0.8, 0.0))


@pytest.mark.parametrize("limits", [(128, 8, 4), (1024, 2, 1), (64, 1, 2), (1024, 32, 4)])
def test_reproduce_limits(oracle, ctx, capi, limits):
    """SpaceLimits change legal unroll/vector lists and the repair block cap."""
    op = parse_op("mm:1,256,512,384")
    lim = np.array(limits, np.int64)
    par, _ = oracle.sample_random(op, 100, 6, lim)
    check(oracle, capi, op, par, 20000, run(capi, ctx, op, par, 20000, 5, limits=lim), 5, limits=lim)


def test_reproduce_edge_sizes(oracle, ctx, capi):
    op = parse_op("mm:1,8,8,8")
    par, _ = oracle.sample_random(op, 3, 1)
    for n in (1, 2, 95, 96, 97, 313):
        check(oracle, capi, op, par, n, run(capi, ctx, op, par, n, 77), 77)


def test_reproduce_errors(ctx, capi):
    op = parse_op("mm:1,8,8,8")
    plan = capi.Plan(ctx, op)
    g = torch.zeros(0, dtype=torch.int64, device="cuda")
    with pytest.raises(capi.EtuneError) as e:
        capi.reproduce(plan, g, 10, 1)
    assert e.value.code == 2
    g = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(capi.EtuneError) as e:
        capi.reproduce(plan, g, 10, 1, (0.0, 0.0, 0.0))
    assert e.value.code == 2


@pytest.mark.parametrize("text,np_,n,seed,rates", [
    ("conv:1,56,56,64,64,3,1,1", 1024, 1 << 20, 7, (0.85, 0.10, 0.05)),
    ("mm:1,512,3072,768", 512, 200003, 9, (0.85, 0.10, 0.05)),
    ("mm:1,1024,1024,1024", 64, 100000, 3, (0.2, 0.7, 0.1)),
    ("mv:1,1,1000,2048", 3, 50000, 11, (0.0, 1.0, 0.0)),
])
def test_reproduce_counter_mode_vs_oracle(oracle, ctx, capi, text, np_, n, seed, rates):
    """The opt-in counter-based mode (etune_cu_reproduce_counter): schedules, ids and lineage
    identical to its oracle restatement (orc_reproduce_counter), including 2^20 offspring."""
    op = parse_op(text)
    parents, _ = oracle.sample_random(op, np_, 42)
    plan = capi.Plan(ctx, op)
    g = plan.encode(dev(parents))
    out, partner, ids = capi.reproduce(plan, g, n, seed, rates, counter=True)
    sched = plan.decode(out)
    ctx.synchronize()
    s, oid, lin, ll = oracle.reproduce_counter(op, parents, n, seed, rates)
    assert (sched.cpu().numpy() == s).all()
    assert (capi.as_u64(ids) == oid).all()
    gp = partner.cpu().numpy()
    assert (ll == np.where(gp >= 0, 2, 1)).all()
    pid = oracle.ids(op, parents)
    assert (lin[gp >= 0, 1] == pid[gp[gp >= 0]]).all()


def test_reproduce_counter_mode_speed(oracle, ctx, capi):
    """2^20 offspring in the counter mode well under the exact mode's single-CTA chain."""
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    plan = capi.Plan(ctx, op)
    g = plan.sample_random(1024, 42)
    capi.reproduce(plan, g, 1 << 20, 7, counter=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(5):
        capi.reproduce(plan, g, 1 << 20, 7 + r, counter=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"counter-mode reproduce 2^20: {ms:.3f} ms")
    assert ms < 10.0


# ---- the block-parallel exact path (breed_par.cu): every generation of >= 4096 offspring above
# already runs it; these pin the bench-scale case, each fallback and the speed.

@pytest.fixture
def envset():
    import os
    saved = {}

    def set_(k, v):
        saved.setdefault(k, os.environ.get(k))
        os.environ[k] = str(v)
    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def test_reproduce_exact_bench_config(oracle, ctx, capi):
    """bench.py's generation: reproduce(sample_random(conv3x3, 1024, 42), 2^20, seed 7) — the
    reference's single mt19937_64 stream, bit-exact, on the block-parallel path."""
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    par, _ = oracle.sample_random(op, 1024, 42)
    n = 1 << 20
    check(oracle, capi, op, par, n, run(capi, ctx, op, par, n, 7), 7)


@pytest.mark.parametrize("sd", ["0.05", "1.0"])
def test_reproduce_exact_window_misses(oracle, ctx, capi, envset, sd):
    """Windows far too narrow: most block starts fall outside them and the chain kernel walks
    those blocks exactly on the spot; the children are unchanged."""
    envset("ETUNE_BREED_PAR_SD", sd)
    op = parse_op("mm:1,512,3072,768")
    par, _ = oracle.sample_random(op, 333, 42)
    n = 70001
    check(oracle, capi, op, par, n, run(capi, ctx, op, par, n, 13), 13)


def test_reproduce_exact_capacity_fallback(oracle, ctx, capi, envset):
    """A stream capacity too small for the generation: the parallel path stands down on the
    device and the single-CTA chain produces the generation."""
    envset("ETUNE_BREED_PAR_WORDS", "1000")
    op = parse_op("conv:1,28,28,128,512,1,1,0")
    par, _ = oracle.sample_random(op, 200, 4)
    check(oracle, capi, op, par, 30000, run(capi, ctx, op, par, 30000, 3), 3)


def test_reproduce_exact_single_cta_agrees(oracle, ctx, capi, envset):
    """The single-CTA chain (ETUNE_BREED_PAR_MIN above n) and the parallel path give identical
    children on the same call."""
    op = parse_op("mm:4,96,200,50")
    par, _ = oracle.sample_random(op, 300, 5)
    a = run(capi, ctx, op, par, 40000, 17)
    envset("ETUNE_BREED_PAR_MIN", str(1 << 40))
    b = run(capi, ctx, op, par, 40000, 17)
    for x, y in zip(a, b):
        assert (x == y).all()


@pytest.mark.parametrize("n", [4096, 4097, 8191, 65537, 262143])
def test_reproduce_exact_sizes(oracle, ctx, capi, n):
    """Block-size boundaries (S adapts to n; ragged last blocks and sub-blocks)."""
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    par, _ = oracle.sample_random(op, 1000, 9)
    check(oracle, capi, op, par, n, run(capi, ctx, op, par, n, n), n)


def test_reproduce_exact_speed(ctx, capi):
    """2^20 offspring of the reference's own stream in well under the single-CTA chain's 252 ms."""
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    plan = capi.Plan(ctx, op)
    g = plan.sample_random(1024, 42)
    capi.reproduce(plan, g, 1 << 20, 7)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(3):
        capi.reproduce(plan, g, 1 << 20, 7 + r)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"exact reproduce 2^20 (block-parallel): {ms:.3f} ms")
    assert ms < 25.0


@pytest.mark.parametrize("text,npar,n,rates,limits", [
    ("conv:1,56,56,64,64,3,1,1", 1024, 1 << 18, (0.85, 0.10, 0.05), None),
    ("mm:1,512,3072,768", 97, 100000, (0.2, 0.7, 0.1), None),
    ("mm:1,256,512,384", 100, 100000, (0.85, 0.10, 0.05), (128, 8, 4)),   # tight block cap: re-picks
    ("mm:1,256,512,384", 100, 60000, (0.5, 0.5, 0.0), (64, 1, 2)),
    ("mm:4,96,200,50", 300, 60000, (1.0, 0.0, 0.0), None),
])
def test_reproduce_exact_fast_count_agrees(oracle, ctx, capi, envset, text, npar, n, rates, limits):
    """ETUNE_BREED_PAR_CHECK: every window walker's straight-line word count is re-derived by
    breed_body (the reference's decision code) and a disagreement fails the call; children exact."""
    envset("ETUNE_BREED_PAR_CHECK", "1")
    op = parse_op(text)
    lim = None if limits is None else np.array(limits, np.int64)
    par, _ = oracle.sample_random(op, npar, 42, lim)
    check(oracle, capi, op, par, n, run(capi, ctx, op, par, n, 23, rates, lim), 23, rates, lim)
