"""CPU tests: the oracle restatement pinned against the reference's golden vectors
(tests/golden/golden_reference.npz, made by tests/golden/make_golden.py from the
unmodified reference) and against SPEC KATs."""
import numpy as np
import pytest

from etune_testlib import FlatForest, RefLib, have_ref, parse_op
from golden.make_golden import COUNT_KAT, MODEL_OPS, OPS

NAMES = [n for n, _, _ in OPS]


def test_log1p_kat(golden):
    # SPEC:182 [TRIVIAL] f[0] == log1p(2): the runtime glibc value
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.log1p.restype = ctypes.c_double
    libm.log1p.argtypes = [ctypes.c_double]
    assert np.array([libm.log1p(2.0)]).view(np.uint64)[0] == golden["log1p_2_bits"][0]


@pytest.mark.parametrize("name", NAMES)
def test_space_and_ids(golden, oracle, name):
    op = golden[f"{name}/op"]
    assert (oracle.nest(op) == golden[f"{name}/nest"]).all()
    assert oracle.count(op) == golden[f"{name}/space"][0]
    s = golden[f"{name}/sample_sched"]
    sr, ids = oracle.sample_random(op, len(s), 42)
    assert (sr == s).all()
    assert (ids == golden[f"{name}/sample_ids"]).all()
    assert (oracle.ids(op, s) == golden[f"{name}/sample_ids"]).all()
    if f"{name}/enum_sched" in golden:
        full = oracle.enumerate(op)
        assert (full == golden[f"{name}/enum_sched"]).all()
        ids = oracle.ids(op, full)
        assert (ids == golden[f"{name}/enum_ids"]).all()
        assert len(np.unique(ids)) == len(ids)  # SPEC: id collision-free on small spaces


@pytest.mark.parametrize("name", NAMES)
def test_features_counters_bitexact(golden, oracle, name):
    op = golden[f"{name}/op"]
    s = golden[f"{name}/sample_sched"]
    assert (oracle.counters(op, s) == golden[f"{name}/counters"]).all()
    assert (oracle.features(op, s).view(np.uint64) == golden[f"{name}/features_bits"]).all()
    assert (oracle.features(op, s, 148).view(np.uint64) == golden[f"{name}/features_bits_sms148"]).all()


@pytest.mark.parametrize("name", NAMES)
def test_reproduce_bitexact(golden, oracle, name):
    op = golden[f"{name}/op"]
    s, ids, lin, ll = oracle.reproduce(op, golden[f"{name}/repro_parents"], 512, 7)
    assert (s == golden[f"{name}/repro_sched"]).all()
    assert (ids == golden[f"{name}/repro_ids"]).all()
    assert (lin == golden[f"{name}/repro_lineage"]).all()
    assert (ll == golden[f"{name}/repro_lineage_len"]).all()


@pytest.mark.parametrize("name", MODEL_OPS)
def test_train_and_predict_bitexact(golden, oracle, name):
    op = golden[f"{name}/op"]
    k = f"{name}/model/"
    feats = oracle.features(op, golden[k + "train_sched"])
    forest, ref_e, loss = oracle.train(feats, golden[k + "train_energy"])
    for f in ("feature", "threshold", "left", "right", "value", "offsets"):
        assert (getattr(forest, f) == golden[k + f]).all(), f
    assert forest.base_score == golden[k + "base_score"][0]
    assert ref_e == golden[k + "reference_energy"][0]
    assert (loss.view(np.uint64) == golden[k + "training_loss"].view(np.uint64)).all()
    pf = oracle.features(op, golden[f"{name}/sample_sched"])
    assert (oracle.predict(forest, pf).view(np.uint64) == golden[k + "pred_bits"]).all()


@pytest.mark.parametrize("text", COUNT_KAT)
def test_count_kat(golden, oracle, text):
    assert oracle.count(parse_op(text)) == golden[f"count/{text}"][0]


def test_spec_kats(oracle):
    # SPEC:125-128 trivial MM(1,1,1,1): flops 2, glb_ld 2, glb_st 1; MM 512^3 flops
    op = parse_op("mm:1,1,1,1")
    triv = np.array([[1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1]], np.int64)
    c = oracle.counters(op, triv)[0]
    assert (c[2], c[4], c[5]) == (2, 2, 1)
    s, _ = oracle.sample_random(parse_op("mm:1,512,512,512"), 8, 3)
    assert (oracle.counters(parse_op("mm:1,512,512,512"), s)[:, 2] == 268435456).all()
    # SPEC:240-242 loss examples
    assert tuple(oracle.energy_loss(2.0, 1.0)) == (1.0, 2.0, 2.0)
    assert tuple(oracle.energy_loss(5.0, 5.0))[:2] == (0.0, 0.0)
    # SPEC:265-268 snr examples
    assert oracle.snr_db([1.0, 2.0], [1.0, 2.0]) == 100.0
    assert abs(oracle.snr_db([2.0, 4.0], [1.0, 2.0])) < 1e-12
    assert abs(oracle.snr_db([1.1, 0.9], [1.0, 1.0]) - 20.0) < 1e-9
    # SPEC:70 SpaceExhausted
    from etune_testlib import EtuneError
    with pytest.raises(EtuneError) as e:
        oracle.sample_random(parse_op("mm:1,4,4,4"), 361, 0)
    assert e.value.code == 3


def test_rng_restatement_matches_libstdcxx(oracle):
    import ctypes as C
    a = np.zeros(10000, np.uint64)
    b = np.zeros(10000, np.uint64)
    oracle.L.orc_mt64_words(5489, 10000, a)
    oracle.L.orc_std_mt64_words(5489, 10000, b)
    assert (a == b).all() and a[-1] == 9981545732273789042  # mt19937_64 check value
    for r in (1, 2, 3, 6, 7, 1000, 2**63 + 5, 2**64 - 1):
        a = np.zeros(4096, np.uint64)
        b = np.zeros(4096, np.uint64)
        x = oracle.L.orc_lemire(11, 4096, r, a)
        y = oracle.L.orc_std_uniform(11, 4096, r, b)
        assert (a == b).all() and x == y
    a = np.zeros(50000)
    b = np.zeros(50000)
    oracle.L.orc_canonical(3, 50000, a)
    oracle.L.orc_std_canonical(3, 50000, b)
    assert (a == b).all()


def test_topk_order(oracle):
    rng = np.random.default_rng(0)
    sc = rng.integers(0, 20, 5000).astype(np.float64)
    idx = oracle.topk(sc, 777)
    ref = np.lexsort((np.arange(len(sc)), sc))[:777]
    assert (idx == ref).all()


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("text", ["mm:1,1024,1024,1024", "conv:1,56,56,64,64,3,1,1",
                                  "mm:1,512,3072,768", "conv:1,14,14,256,256,3,1,1"])
def test_live_vs_reference_large(oracle, text):
    """Larger samples than the fixtures, live against the compiled reference."""
    R = RefLib()
    op = parse_op(text)
    s, ids = R.sample_random(op, 8192, 42)
    s2, ids2 = oracle.sample_random(op, 8192, 42)
    assert (s == s2).all() and (ids == ids2).all()
    assert (R.features(op, s).view(np.uint64) == oracle.features(op, s).view(np.uint64)).all()
    a = R.reproduce(op, s[:1024], 16384, 7)
    b = oracle.reproduce(op, s[:1024], 16384, 7)
    for x, y in zip(a, b):
        assert (x == y).all()


def test_sim_measure_spec_examples(oracle):
    """SPEC:318-322 examples for the sim restatement (no reference implementation)."""
    from etune_testlib import parse_op, DEFAULT_DEVICE
    op = parse_op("mm:1,1,1,1")
    s = oracle.enumerate(op)
    r = oracle.sim_measure(op, s, {"noise_sigma_rel": 0.0, "latency_floor_ms": 1.0})
    # tiny work: latency is the floor; power = constant + 1 * static + dynamic/latency
    assert r[0, 0] == 1.0
    assert abs(r[0, 1] - (60.0 + 0.55)) < 1e-3
    assert r[0, 2] == r[0, 1] * r[0, 0]  # energy identity
    # more active SMs at equal work -> more static power (SPEC:320 direction)
    op = parse_op("mm:1,64,64,64")
    full = oracle.enumerate(op)
    c = oracle.counters(op, full)
    m = oracle.sim_measure(op, full, {"noise_sigma_rel": 0.0})
    assert np.all(np.isfinite(m)) and (m[:, 0] > 0).all() and (m[:, 1] > 0).all()
    a64 = (c[:, 9] == 64)
    a1 = (c[:, 9] == 1)
    assert m[a64, 1].min() > DEFAULT_DEVICE["constant_power_w"] + 0.55 * 64 - 1e-9
    assert m[a1, 1].min() > DEFAULT_DEVICE["constant_power_w"] + 0.55 - 1e-9
    # noise: deterministic per seed, mean within 2 % at sigma 0.05
    r1 = oracle.sim_measure(op, full[:200])
    r2 = oracle.sim_measure(op, full[:200])
    r0 = oracle.sim_measure(op, full[:200], {"noise_sigma_rel": 0.0})
    assert (r1 == r2).all()
    assert np.abs(r1[:, 1] / r0[:, 1] - 1).max() < 0.02


def test_sim_noise_is_gaussian_spec(oracle):
    """the sampler's multiplicative noise is Gaussian with sigma noise_sigma_rel;
    at sigma 0.05 with >= 2 s of 50 Hz samples the average power is within 2 % of the true power
    for >= 99 of 100 seeds.  The standardised deviations of the averages over seeds and
    candidates, (avg / true - 1) / (sigma / sqrt(S)), have mean ~0 and variance ~1."""
    from etune_testlib import parse_op
    op = parse_op("mm:1,64,64,64")
    full = oracle.enumerate(op)[:40]
    r0 = oracle.sim_measure(op, full, {"noise_sigma_rel": 0.0})
    lat_s = r0[:, 0] / 1000.0
    S = np.clip(np.floor(r0[:, 3] * lat_s * 50.0), 1, 4096)
    zs, within = [], 0
    for seed in range(100):
        r = oracle.sim_measure(op, full, {"noise_sigma_rel": 0.05, "sampler_hz": 50.0, "rng_seed": seed})
        dev = r[:, 1] / r0[:, 1] - 1.0
        within += int(abs(dev[0]) < 0.02)
        zs.append(dev / (0.05 / np.sqrt(S)))
    z = np.concatenate(zs)
    assert within >= 99
    assert abs(z.mean()) < 0.05 and 0.9 < z.var() < 1.1


def test_reproduce_counter_restatement(oracle):
    """The counter-mode restatement: deterministic, prefix-stable (offspring i depends only on
    (seed, i, parents)), every child legal with a correct id and lineage, and the move mix of
    GeneticRates (mutation / crossover / copy) like the exact mode's."""
    from etune_testlib import parse_op
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    par, pid = oracle.sample_random(op, 256, 42)
    s, ids, lin, ll = oracle.reproduce_counter(op, par, 30000, 7)
    s2, _, _, _ = oracle.reproduce_counter(op, par, 30000, 7)
    assert (s == s2).all()
    s3, _, _, _ = oracle.reproduce_counter(op, par, 1000, 7)
    assert (s3 == s[:1000]).all()
    assert (oracle.ids(op, s) == ids).all()
    assert (lin[:, 0] == pid[np.arange(30000) % 256]).all()
    frac_cro = (ll == 2).mean()
    _, _, _, lle = oracle.reproduce(op, par, 30000, 7)
    assert abs(frac_cro - 0.10) < 0.01 and abs((lle == 2).mean() - 0.10) < 0.01
    s4, _, _, _ = oracle.reproduce_counter(op, par, 30000, 8)
    assert (s4 != s).any(axis=1).mean() > 0.5  # a different seed, a different generation
