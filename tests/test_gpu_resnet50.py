"""BASELINE configs[4] breadth: every stride-1 ResNet-50 conv layer and the fc layer (the
7 stride-2 layers are rejected by OperatorSpec::validate).  Per layer: space
size, device sample_random, features/ids, cross-operator scoring with a reference-trained
forest and device reproduce are bit-exact against the oracle."""
import numpy as np
import pytest

from etune_testlib import FlatForest, parse_op

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

R50 = [("conv:1,56,56,64,64,1,1,0", 216854), ("conv:1,56,56,64,64,3,1,1", 650562),
       ("conv:1,56,56,64,256,1,1,0", 350856), ("conv:1,56,56,256,64,1,1,0", 295710),
       ("conv:1,56,56,256,128,1,1,0", 383550), ("conv:1,28,28,128,512,1,1,0", 283842),
       ("conv:1,28,28,512,128,1,1,0", 243508), ("conv:1,28,28,128,128,3,1,1", 558636),
       ("conv:1,28,28,512,256,1,1,0", 305388), ("conv:1,14,14,256,1024,1,1,0", 162270),
       ("conv:1,14,14,1024,256,1,1,0", 141246), ("conv:1,14,14,256,256,3,1,1", 334530),
       ("conv:1,14,14,1024,512,1,1,0", 172596), ("conv:1,7,7,512,2048,1,1,0", 37026),
       ("conv:1,7,7,2048,512,1,1,0", 32634), ("conv:1,7,7,512,512,3,1,1", 79254),
       ("mv:1,1,1000,2048", 7980)]


@pytest.fixture(scope="module")
def capi():
    from paper_2411_18873_b200 import capi as c
    return c


@pytest.fixture(scope="module")
def ctx(capi):
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return capi.Context(0)


@pytest.fixture(scope="module")
def forest(golden):
    k = "c2_r50_conv3x3/model/"
    return FlatForest(golden[k + "feature"], golden[k + "threshold"], golden[k + "left"], golden[k + "right"],
                      golden[k + "value"], golden[k + "offsets"], float(golden[k + "base_score"][0]),
                      float(golden[k + "learning_rate"][0]))


@pytest.mark.parametrize("text,space", R50)
def test_resnet50_layer(oracle, ctx, capi, forest, text, space):
    op = parse_op(text)
    plan = capi.Plan(ctx, op, num_sms=148)
    assert plan.space_size() == space
    n = 4096
    want, ids = oracle.sample_random(op, n, 42)
    g, dids = plan.sample_random(n, 42, with_ids=True)
    assert (capi.as_u64(dids) == ids).all()
    f = plan.features(g)
    ref_f = oracle.features(op, want, 148)
    assert (f.cpu().numpy().view(np.uint64) == ref_f.view(np.uint64)).all()
    fo = capi.Forest.from_flat(ctx, forest)
    pred = fo.score(plan, g)
    ctx.synchronize()
    assert (pred.cpu().numpy().view(np.uint64) == oracle.predict(forest, ref_f).view(np.uint64)).all()
    kids, partner, kid_ids = capi.reproduce(plan, g[:256], 4096, 9)
    s, rid, _, _ = oracle.reproduce(op, want[:256], 4096, 9)
    assert (capi.as_u64(kid_ids) == rid).all()
    assert (plan.decode(kids).cpu().numpy() == s).all()


def test_resnet50_stride2_layers_rejected(ctx, capi):
    for text in ("conv:1,224,224,3,64,7,2,3", "conv:1,56,56,128,128,3,2,1", "conv:1,56,56,256,512,1,2,0"):
        with pytest.raises(capi.EtuneError) as e:
            capi.Plan(ctx, parse_op(text))
        assert e.value.code == 2
