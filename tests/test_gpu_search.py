"""GPU parity of the Algorithm-1 search loop (etune_cu_search_*) against the CPU
restatement (oracle orc_run_search): every round report (k trajectory, SNR bits,
measurement counts, best-so-far) and the final parents are identical."""
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


def f64bits(x):
    return np.float64(x).view(np.uint64)


CASES = [
    ("mm:1,64,64,64", dict(M=64, G=256, seed=42, max_rounds=6)),
    ("mm:1,1024,1024,1024", dict(M=512, G=2048, seed=42, max_rounds=10)),       # BASELINE configs[0] shape
    ("conv:1,56,56,64,64,3,1,1", dict(M=256, G=1024, seed=7, max_rounds=5, k_init_fifths=3, inverted=1)),
    ("mm:1,512,3072,768", dict(M=128, G=600, seed=3, max_rounds=4, dev={"noise_sigma_rel": 0.3, "num_sms": 148},
                               mu_db=30.0, num_trees=30, max_depth=5)),
]


@pytest.mark.parametrize("text,kw", CASES)
def test_search_vs_oracle(oracle, ctx, capi, text, kw):
    op = parse_op(text)
    kw = dict(kw)
    dev = kw.pop("dev", {})
    M, G, seed = kw.pop("M"), kw.pop("G"), kw.pop("seed")
    ri, rd, par = oracle.run_search(op, M, G, seed, dev=dev, **kw)
    plan = capi.Plan(ctx, op, dev=capi.default_device_config(**dev))
    cfg = capi.search_config(M=M, generation_size=G, rng_seed=seed,
                             **{("inverted_semantics" if k == "inverted" else k): v for k, v in kw.items()})
    s = capi.Search(plan, cfg)
    reps = s.run()
    assert len(reps) == len(ri)
    for r, a, b in zip(reps, ri, rd):
        assert (r.round, r.k_before_fifths, r.k_after_fifths, r.measured, r.cumulative_measured) == tuple(a[:5])
        assert r.best_id == np.int64(a[5]).view(np.uint64)
        if r.round > 0:
            assert f64bits(r.snr_db) == f64bits(b[0])
        assert f64bits(r.best_latency_ms) == f64bits(b[1])
        assert f64bits(r.best_energy_mj) == f64bits(b[2])
        assert f64bits(r.best_power_w) == f64bits(b[3])
    got = plan.decode(s.parents()).cpu().numpy()
    assert (got == par).all()
    sched, bid, lat, en = s.best()
    assert bid == reps[-1].best_id and en == reps[-1].best_energy_mj
    assert oracle.ids(op, sched[None, :])[0] == bid
    print(f"{text}: round wall ms = {[round(r.wall_ms, 2) for r in reps]}")
