"""CPU check of the per-operator forest compilation (classes + leaf-mask tables,
paper_2411_18873_b200/csrc/forest.cpp) by running the device scoring core on the
host (tests/cpp) and comparing predictions bit-for-bit with the oracle."""
import numpy as np
import pytest

from etune_testlib import FlatForest, host_compiled_score, parse_op
from golden.make_golden import MODEL_OPS


def forest_of(golden, name):
    k = f"{name}/model/"
    return FlatForest(golden[k + "feature"], golden[k + "threshold"], golden[k + "left"], golden[k + "right"],
                      golden[k + "value"], golden[k + "offsets"], float(golden[k + "base_score"][0]),
                      float(golden[k + "learning_rate"][0]))


@pytest.mark.parametrize("name", MODEL_OPS)
def test_compiled_golden(golden, name):
    op = golden[f"{name}/op"]
    pred, stats = host_compiled_score(op, forest_of(golden, name), golden[f"{name}/sample_sched"])
    assert (pred.view(np.uint64) == golden[f"{name}/model/pred_bits"]).all()
    assert stats[3] <= 64


@pytest.mark.parametrize("name", MODEL_OPS)
@pytest.mark.parametrize("sms", [108, 148])
@pytest.mark.parametrize("keyed", [False, True, "byte"])
def test_compiled_bred_population(golden, oracle, name, sms, keyed):
    op = golden[f"{name}/op"]
    fl = forest_of(golden, name)
    par, _ = oracle.sample_random(op, 128, 11)
    s, _, _, _ = oracle.reproduce(op, par, 20000, 3)
    ref = oracle.predict(fl, oracle.features(op, s, sms))
    pred, _ = host_compiled_score(op, fl, s, sms, keyed=keyed)
    assert (pred.view(np.uint64) == ref.view(np.uint64)).all()


@pytest.mark.parametrize("src,dst", [("c3_bert_ffn", "conv:1,7,7,512,512,3,1,1"), ("c2_r50_conv3x3", "mm:4,96,200,50"),
                                     ("c1_gemm1024", "conv:2,14,14,64,32,3,1,1")])
@pytest.mark.parametrize("keyed", [True, "byte"])
def test_keyed_form_cross_operator(golden, oracle, src, dst, keyed):
    """The keyed forms (per tiling-triple AND of non-Kuv masks; full per (key, Kuv class)
    5-bit slots) on other operators, incl. batch > 1 (three-index keys)."""
    op = parse_op(dst)
    fl = forest_of(golden, src)
    n = min(5000, oracle.count(op))
    s, _ = oracle.sample_random(op, n, 21)
    ref = oracle.predict(fl, oracle.features(op, s))
    pred, _ = host_compiled_score(op, fl, s, keyed=keyed)
    assert (pred.view(np.uint64) == ref.view(np.uint64)).all()


@pytest.mark.parametrize("src,dst", [("c3_bert_ffn", "conv:1,7,7,512,512,3,1,1"),
                                     ("c1_gemm1024", "mv:1,1,1000,2048"),
                                     ("c2_r50_conv3x3", "mm:4,96,200,50")])
def test_compiled_cross_operator(golden, oracle, src, dst):
    op = parse_op(dst)
    fl = forest_of(golden, src)
    n = min(5000, oracle.count(op))
    s, _ = oracle.sample_random(op, n, 9)
    ref = oracle.predict(fl, oracle.features(op, s))
    pred, stats = host_compiled_score(op, fl, s)
    assert (pred.view(np.uint64) == ref.view(np.uint64)).all()
    assert stats[1] > 0  # another operator's forest: many tests fold to constants


def test_compiled_deep_forest(oracle):
    op = parse_op("mm:1,256,512,384")
    s, _ = oracle.sample_random(op, 1500, 3)
    f = oracle.features(op, s)
    e = 1.0 + (f[:, 2] * 0.3 + f[:, 12] * 0.1 + f[:, 6]) % 2.7
    fl, _, _ = oracle.train(f, e, num_trees=40, max_depth=6, min_leaf_weight=0.0)
    pop, _ = oracle.sample_random(op, 20000, 4)
    ref = oracle.predict(fl, oracle.features(op, pop))
    pred, stats = host_compiled_score(op, fl, pop)
    assert (pred.view(np.uint64) == ref.view(np.uint64)).all()
