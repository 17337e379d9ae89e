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


def test_replay_search_reproduces_sim_search(oracle, ctx, capi):
    """ReplayBackend (backend 2, measure.hpp:116-128): a JSONL measurement log of the
    SimBackend records of every schedule in the space replays the sim search round for
    round; a log lacking a candidate fails with TraceMiss."""
    op = parse_op("mm:1,64,64,64")
    plan = capi.Plan(ctx, op)
    sched = oracle.enumerate(op)
    g = plan.encode(torch.from_numpy(np.ascontiguousarray(sched)).cuda())
    lat, pw, en, it = (t.cpu().numpy() for t in plan.sim_measure(g))
    rec = np.zeros(len(sched), capi.LOG_RECORD_DTYPE)
    rec["m"]["candidate_id"] = plan.ids(g).cpu().numpy().view(np.uint64)
    rec["m"]["latency_ms"], rec["m"]["avg_power_w"], rec["m"]["energy_mj"] = lat, pw, en
    rec["m"]["iterations"] = it
    rec["backend"], rec["timestamp"] = b"sim", b"2026-10-17T00:00:00Z"
    log = capi.measurement_log_from_jsonl(capi.measurement_log_to_jsonl(rec))  # through the JSONL file format
    assert len(log) == len(sched)
    kw = dict(M=64, generation_size=256, rng_seed=42, max_rounds=6)
    sim = capi.Search(plan, capi.search_config(**kw)).run()
    rep = capi.Search(plan, capi.search_config(backend=2, **kw)).set_replay(log).run()
    assert len(rep) == len(sim)
    for a, b in zip(rep, sim):
        assert (a.round, a.k_before_fifths, a.k_after_fifths, a.measured, a.cumulative_measured, a.best_id) == \
               (b.round, b.k_before_fifths, b.k_after_fifths, b.measured, b.cumulative_measured, b.best_id)
        for f in ("snr_db", "best_latency_ms", "best_energy_mj", "best_power_w"):
            x, y = getattr(a, f), getattr(b, f)
            assert f64bits(x) == f64bits(y) or (np.isnan(x) and np.isnan(y))
    miss = capi.Search(plan, capi.search_config(backend=2, **kw)).set_replay(log[:100])
    with pytest.raises(capi.EtuneError) as e:
        miss.run()
    assert e.value.code == 15  # ETUNE_ERR_TRACE_MISS
    with pytest.raises(capi.EtuneError) as e:
        capi.Search(plan, capi.search_config(backend=2, **kw)).run()  # no log attached
    assert e.value.code == 14


@pytest.mark.parametrize("text,kw", [("mm:1,64,64,64", dict(M=64, G=256, seed=42, max_rounds=6)),
                                     ("conv:1,56,56,64,64,3,1,1", dict(M=256, G=1024, seed=7, max_rounds=5))])
def test_latency_only_search_vs_oracle(oracle, ctx, capi, text, kw):
    """run_latency_only: the same loop with steps 3-8 replaced by parent
    selection on latency; every report and the final parents equal the restatement's."""
    op = parse_op(text)
    kw = dict(kw)
    M, G, seed = kw.pop("M"), kw.pop("G"), kw.pop("seed")
    ri, rd, par = oracle.run_search(op, M, G, seed, latency_only=1, **kw)
    plan = capi.Plan(ctx, op)
    reps = capi.Search(plan, capi.search_config(M=M, generation_size=G, rng_seed=seed, latency_only=1, **kw)).run()
    assert len(reps) == len(ri)
    for r, a, b in zip(reps, ri, rd):
        assert (r.round, r.k_before_fifths, r.k_after_fifths, r.measured, r.cumulative_measured) == tuple(a[:5])
        assert r.best_id == np.int64(a[5]).view(np.uint64) and np.isnan(r.snr_db)
        assert f64bits(r.best_latency_ms) == f64bits(b[1]) and f64bits(r.best_energy_mj) == f64bits(b[2])
    s = capi.Search(plan, capi.search_config(M=M, generation_size=G, rng_seed=seed, latency_only=1, **kw))
    s.run()
    assert (plan.decode(s.parents()).cpu().numpy() == par).all()


def _space(capi, ctx, oracle, text):
    op = parse_op(text)
    plan = capi.Plan(ctx, op)
    g = plan.encode(torch.from_numpy(np.ascontiguousarray(oracle.enumerate(op))).cuda())
    lat, pw, en, _ = (t.cpu().numpy() for t in plan.sim_measure(g))
    return plan, lat, pw, en


def test_spec_acceptance_search_optimality(oracle, ctx, capi):
    """SPEC acceptance 6: on MM(1,16,16,16) the search's best measured energy is within 5 %
    of the brute-force optimum over the whole space on >= 9 of 10 seeds."""
    plan, _, _, en = _space(capi, ctx, oracle, "mm:1,16,16,16")
    best = [capi.Search(plan, capi.search_config(M=64, generation_size=256, rng_seed=s, max_rounds=30)).run()[-1]
            .best_energy_mj for s in range(10)]
    assert sum(b <= 1.05 * en.min() for b in best) >= 9


def test_spec_acceptance_measurement_budget_and_correlation(oracle, ctx, capi):
    """SPEC acceptance 8: cumulative energy measurements over 15 rounds at mu = 20 dB are
    <= 0.55x a forced k = 1.0 run; 9: Spearman(latency, power) < 0 over MM(1,64,64,64)."""
    from scipy.stats import spearmanr
    plan, lat, pw, _ = _space(capi, ctx, oracle, "mm:1,64,64,64")
    kw = dict(M=64, generation_size=256, rng_seed=3, max_rounds=15, patience=1 << 30)
    dyn = capi.Search(plan, capi.search_config(mu_db=20.0, **kw)).run()[-1].cumulative_measured
    forced = capi.Search(plan, capi.search_config(mu_db=1e9, **kw)).run()[-1].cumulative_measured
    assert forced == 64 * 16 and dyn <= 0.55 * forced
    assert spearmanr(lat, pw).correlation < 0
