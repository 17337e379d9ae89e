"""GPU parity of etune_cu_sample_random (space.cpp:170-251): both branches (large-space
parallel attempts + stable dedupe; small-space enumeration + parallel Fisher-Yates)
reproduce the reference's sample bit for bit."""
import numpy as np
import pytest

from etune_testlib import parse_op

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


@pytest.mark.parametrize("text,n,seed", [
    ("mm:1,1024,1024,1024", 2048, 42),          # large space (C1)
    ("conv:1,56,56,64,64,3,1,1", 16384, 42),    # large space (C2)
    ("mm:1,512,3072,768", 65536, 7),            # large space (C3)
    ("mm:1,8,8,8", 1000, 3),                    # small space: enumerate + Fisher-Yates
    ("mm:1,8,8,8", 1900, 5),                    # the whole space
    ("mm:1,64,64,64", 20000, 11),               # small space, 39292 legal
    ("mm:4,96,200,50", 5000, 1),
    ("mv:1,1,1000,2048", 4000, 2),              # small (7980 legal)
    ("conv:2,4,4,2,2,1,1,0", 1, 9),
])
def test_sample_random_vs_oracle(oracle, ctx, capi, text, n, seed):
    op = parse_op(text)
    want, ids = oracle.sample_random(op, n, seed)
    plan = capi.Plan(ctx, op)
    g, dids = plan.sample_random(n, seed, with_ids=True)
    s = plan.decode(g)
    ctx.synchronize()
    assert (s.cpu().numpy() == want).all()
    assert (capi.as_u64(dids) == ids).all()


def test_sample_random_bert_2_20(oracle, ctx, capi):
    """C3 at 2^20: the reference takes the small-space branch (1,387,200 legal <= 2^21)."""
    op = parse_op("mm:1,512,3072,768")
    n = 1 << 20
    want, ids = oracle.sample_random(op, n, 42)
    plan = capi.Plan(ctx, op)
    g, dids = plan.sample_random(n, 42, with_ids=True)
    ctx.synchronize()
    assert (capi.as_u64(dids) == ids).all()


@pytest.mark.parametrize("limits", [(128, 8, 4), (1024, 2, 1), (256, 16, 2)])
def test_sample_random_limits(oracle, ctx, capi, limits):
    lim = np.array(limits, np.int64)
    for text, n in (("mm:1,256,512,384", 10000), ("mm:1,16,16,16", 3000)):
        op = parse_op(text)
        if oracle.count(op, lim) < n:
            continue
        want, ids = oracle.sample_random(op, n, 5, lim)
        plan = capi.Plan(ctx, op, limits=lim)
        g, dids = plan.sample_random(n, 5, with_ids=True)
        ctx.synchronize()
        assert (capi.as_u64(dids) == ids).all()


def test_sample_random_errors(ctx, capi):
    plan = capi.Plan(ctx, parse_op("mm:1,1,1,1"))
    with pytest.raises(capi.EtuneError) as e:
        plan.sample_random(2, 1)
    assert e.value.code == 3  # SpaceExhausted
    with pytest.raises(capi.EtuneError) as e:
        plan.sample_random(0, 1)
    assert e.value.code == 2
