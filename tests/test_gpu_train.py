"""GPU parity of etune_cu_train (device EnergyModel::train, energy_model.cpp:173-243):
every node, the base score, the reference energy and the per-round training loss are
bit-identical to the reference's golden models and to the oracle on fresh data."""
import numpy as np
import pytest

from etune_testlib import parse_op
from golden.make_golden import MODEL_OPS

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


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def same_forest(got, ref_flat, ref_energy=None, ref_loss=None):
    fe, th, le, ri, va, off, base, refe, loss = got
    assert (off == ref_flat.offsets).all()
    assert (fe == ref_flat.feature).all()
    assert (le == ref_flat.left).all()
    assert (ri == ref_flat.right).all()
    assert (bits(th) == bits(ref_flat.threshold)).all()
    assert (bits(va) == bits(ref_flat.value)).all()
    assert bits([base])[0] == bits([ref_flat.base_score])[0]
    if ref_energy is not None:
        assert bits([refe])[0] == bits([ref_energy])[0]
    if ref_loss is not None and loss is not None:
        assert (bits(loss) == bits(ref_loss)).all()


@pytest.mark.parametrize("name", MODEL_OPS)
def test_train_golden(golden, ctx, capi, name):
    """Features computed on the device from the golden training schedules, then the
    100-tree model trained on the device == the reference-trained golden model."""
    from etune_testlib import FlatForest
    op = golden[f"{name}/op"]
    k = f"{name}/model/"
    plan = capi.Plan(ctx, op)
    feats = plan.features(plan.encode(dev(golden[k + "train_sched"])))
    m = capi.train(ctx, feats, dev(golden[k + "train_energy"]))
    ref = FlatForest(golden[k + "feature"], golden[k + "threshold"], golden[k + "left"], golden[k + "right"],
                     golden[k + "value"], golden[k + "offsets"], float(golden[k + "base_score"][0]),
                     float(golden[k + "learning_rate"][0]))
    same_forest(m.host(), ref, float(golden[k + "reference_energy"][0]), golden[k + "training_loss"])


@pytest.mark.parametrize("n,trees,depth,mlw,lam", [
    (2, 5, 6, 1e-3, 1.0), (3, 10, 6, 0.0, 1.0), (97, 20, 3, 1e-3, 0.5), (1000, 30, 6, 0.0, 1.0),
    (4096, 10, 8, 1e-3, 2.0), (5000, 5, 0, 1e-3, 1.0), (700, 0, 6, 1e-3, 1.0), (20000, 4, 6, 1e-3, 1.0)])
def test_train_vs_oracle(oracle, ctx, capi, n, trees, depth, mlw, lam):
    op = parse_op("mm:1,256,512,384")
    s, _ = oracle.sample_random(op, n, n + 1)
    f = oracle.features(op, s)
    rng = np.random.default_rng(n)
    e = 1.0 + (f[:, 2] * 0.3 + f[:, 12] * 0.1 + f[:, 6]) % 2.7 + rng.uniform(0, 0.05, n)
    ref, refe, loss = oracle.train(f, e, num_trees=trees, max_depth=depth, min_leaf_weight=mlw, reg_lambda=lam)
    m = capi.train(ctx, dev(f), dev(e), num_trees=trees, max_depth=depth, min_leaf_weight=mlw, reg_lambda=lam)
    same_forest(m.host(), ref, refe, loss)


def test_train_ties_and_duplicates(oracle, ctx, capi):
    """Heavy feature ties (duplicated samples, constant columns): stable-sort order and
    the strict-greater split rule decide every threshold."""
    rng = np.random.default_rng(5)
    base = rng.integers(0, 4, (300, 16)).astype(np.float64)
    base[:, 7] = 1.0  # constant feature
    f = np.concatenate([base, base[:100], base[:50]])
    e = 1.0 + f[:, 0] * 0.5 + f[:, 3] * 0.25 + rng.integers(0, 3, len(f)) * 0.125
    ref, refe, loss = oracle.train(f, e, num_trees=25, max_depth=6, min_leaf_weight=0.0)
    m = capi.train(ctx, dev(f), dev(e), num_trees=25, max_depth=6, min_leaf_weight=0.0)
    same_forest(m.host(), ref, refe, loss)


def test_trained_forest_scores_like_oracle(oracle, ctx, capi):
    """Device-trained forest -> compiled scoring kernel == oracle predict of the oracle model."""
    op = parse_op("conv:1,56,56,64,64,3,1,1")
    s, _ = oracle.sample_random(op, 2048, 1234)
    f = oracle.features(op, s)
    e = 1.0 + (f[:, 2] * 0.2 + f[:, 13] + f[:, 10] * 0.1) % 1.9
    ref, _, _ = oracle.train(f, e)
    plan = capi.Plan(ctx, op)
    m = capi.train(ctx, plan.features(plan.encode(dev(s))), dev(e))
    fo = m.forest()
    pop, _ = oracle.sample_random(op, 50000, 8)
    pred = fo.score(plan, plan.encode(dev(pop)))
    ctx.synchronize()
    want = oracle.predict(ref, oracle.features(op, pop))
    assert (pred.cpu().numpy().view(np.uint64) == want.view(np.uint64)).all()


def test_train_errors(ctx, capi):
    f = torch.zeros((1, 16), dtype=torch.float64, device="cuda")
    with pytest.raises(capi.EtuneError) as ex:
        capi.train(ctx, f, torch.ones(1, dtype=torch.float64, device="cuda"))
    assert ex.value.code == 7  # InsufficientData
    f = torch.rand((10, 16), dtype=torch.float64, device="cuda")
    e = torch.ones(10, dtype=torch.float64, device="cuda")
    e[6] = 0.0
    capi.train(ctx, f, e, num_trees=2)
    with pytest.raises(capi.EtuneError) as ex:
        ctx.synchronize()
    assert ex.value.code == 6 and ex.value.index == 6  # NonPositiveEnergy
    with pytest.raises(capi.EtuneError) as ex:
        capi.train(ctx, f, torch.ones(10, dtype=torch.float64, device="cuda"), max_depth=11)
    assert ex.value.code == 67


def test_train_megakernel_variant():
    """The opt-in cooperative megakernel (ETUNE_TRAIN_MEGA=1, train.cu) passes the same
    parity tests; the switch is read once per process, hence the subprocess."""
    import os
    import subprocess
    import sys

    if os.environ.get("ETUNE_TRAIN_MEGA"):
        pytest.skip("already running under the variant")
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, ETUNE_TRAIN_MEGA="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_train.py"), "-k", "not megakernel"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("text", ["mm:1,512,512,512", "mv:1,1,1000,2048", "conv:1,28,28,128,128,3,1,1"])
def test_spec_acceptance_cost_model_quality(ctx, capi, text):
    """SPEC acceptance 5 (Fig. 5 analog): a device-trained model on >= 500 SimBackend
    samples ranks held-out candidates with Spearman >= 0.9."""
    from scipy.stats import spearmanr
    plan = capi.Plan(ctx, parse_op(text))
    g = plan.sample_random(1000, 11)
    _, _, en, _ = plan.sim_measure(g)
    feats = plan.features(g)
    m = capi.train(ctx, feats[:700].contiguous(), en[:700].contiguous(), with_loss=False)
    pred = m.forest().predict(feats[700:].contiguous()).cpu().numpy()
    rho = spearmanr(pred, en[700:].cpu().numpy()).correlation
    print(f"{text}: held-out Spearman {rho:.4f}")
    assert rho >= 0.9
