"""Persistence formats against the reference's own output.

The fixtures in tests/golden/persist/ were written by the UNMODIFIED reference
(tests/golden/make_persist_golden.py).  The product's writers must reproduce them
byte for byte (nlohmann::json layout: sorted keys, shortest round-trip doubles) and
its readers must parse every double bit for bit.  Host-only functions: no GPU."""
import glob
import json
import os

import numpy as np
import pytest

from etune_testlib import have_ref

HERE = os.path.dirname(os.path.abspath(__file__))
PERSIST = os.path.join(HERE, "golden", "persist")
MODELS = sorted(glob.glob(os.path.join(PERSIST, "model_*.json")))


@pytest.fixture(scope="module")
def capi():
    from paper_2411_18873_b200 import capi as c
    return c


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("path", MODELS, ids=[os.path.basename(p) for p in MODELS])
def test_model_json_matches_reference(golden, capi, path):
    text = open(path).read()
    m = capi.model_from_json(text)
    name = os.path.basename(path)[len("model_"):-len(".json")]
    k = f"{name}/model/"
    assert (m["feature"] == golden[k + "feature"]).all()
    assert (m["left"] == golden[k + "left"]).all() and (m["right"] == golden[k + "right"]).all()
    assert (bits(m["threshold"]) == bits(golden[k + "threshold"])).all()
    assert (bits(m["value"]) == bits(golden[k + "value"])).all()
    assert (m["tree_offsets"] == golden[k + "offsets"]).all()
    assert bits(m["base_score"]) == bits(golden[k + "base_score"][0])
    assert bits(m["reference_energy_mj"]) == bits(golden[k + "reference_energy"][0])
    assert m["params"].num_trees == 100 and m["params"].max_depth == 6
    again = capi.model_to_json(m["feature"], m["threshold"], m["left"], m["right"], m["value"], m["tree_offsets"],
                               m["params"], m["base_score"], m["reference_energy_mj"])
    assert again == text  # byte-identical to EnergyModel::to_json


def test_samples_jsonl_matches_reference(capi):
    text = open(os.path.join(PERSIST, "samples.jsonl")).read()
    f, m, z = capi.samples_from_jsonl(text)
    assert f.shape[1] == 16 and len(m) == len(z) == text.count("\n")
    assert capi.samples_to_jsonl(f, m, z) == text
    f2, m2, z2 = capi.samples_from_jsonl(capi.samples_to_jsonl(f, m, z))
    assert (bits(f2) == bits(f)).all() and (bits(m2) == bits(m)).all() and (bits(z2) == bits(z)).all()


@pytest.mark.parametrize("name", ["device_a100_like.json", "device_b200_custom.json"])
def test_device_profile_matches_reference(capi, name):
    text = open(os.path.join(PERSIST, name)).read()
    d, nm = capi.device_profile_from_json(text)
    assert capi.device_profile_to_json(d, nm) == text
    if name == "device_a100_like.json":
        ref = capi.default_device_config()
        for f, _ in capi.DeviceConfig._fields_:
            if f != "reserved":
                assert getattr(d, f) == getattr(ref, f), f
        assert nm == "a100-like"
    else:
        assert d.num_sms == 148 and d.rng_seed == (1 << 64) - 1 and nm == 'b200 "sxm"\tnode\\1'


def test_persistence_errors(capi):
    good = open(MODELS[0]).read()
    cases = [
        (good.replace("etune-model-v1", "etune-model-v0"), 9),
        (good.replace("etune-features-v1", "etune-features-v2"), 9),
        (good[:-5], 12),
        (good.replace('"trees":[[', '"trees":[[],[', 1), 12),
        (good.replace('"base_score"', '"base_scor"', 1), 12),
    ]
    for text, code in cases:
        with pytest.raises(capi.EtuneError) as e:
            capi.model_from_json(text)
        assert e.value.code == code
    row = '{"features":[' + ",".join(["1.0"] * 16) + '],"measured_energy_mj":2.0,"normalized_energy":1.0}'
    assert len(capi.samples_from_jsonl(row + "\n\n" + row)[1]) == 2  # empty lines skipped
    for text, code in [(row.replace("2.0", "0.0"), 6), (row.replace('[1.0,', '['), 8), ("{bad", 12)]:
        with pytest.raises(capi.EtuneError) as e:
            capi.samples_from_jsonl(text)
        assert e.value.code == code
    dev = open(os.path.join(PERSIST, "device_a100_like.json")).read()
    for text, code in [(dev.replace("etune-profile-v1", "x"), 9), (dev.replace('"sampler_hz": 50.0', '"sampler_hz": 60.0'), 2),
                       (dev.replace('"num_sms": 108', '"num_sms": 0'), 2), ("[", 1)]:
        with pytest.raises(capi.EtuneError) as e:
            capi.device_profile_from_json(text)
        assert e.value.code == code


@pytest.mark.skipif(not have_ref(), reason="needs oracle/_ref (the compiled reference)")
def test_number_layout_vs_reference_live(capi):
    """Random doubles over the whole exponent range, written by the reference
    (nlohmann) and by the product: identical text, identical parse."""
    from etune_testlib import RefLib
    R = RefLib()
    rng = np.random.default_rng(7)
    with np.errstate(over="ignore"):
        v = rng.uniform(1, 10, 16 * 4000) * 10.0 ** rng.uniform(-310, 308, 16 * 4000)
    v = np.where(rng.random(len(v)) < 0.5, v, -v)
    v[rng.random(len(v)) < 0.05] = np.round(v[:1])
    v = v[np.isfinite(v)][: 16 * 3000]
    f = v.reshape(-1, 16)
    m = np.abs(f[:, 0]) + 1.0
    ref = R.samples_to_jsonl(f, m, f[:, 1])
    assert capi.samples_to_jsonl(f, m, f[:, 1]) == ref
    rf, rm, rz = R.samples_from_jsonl(capi.samples_to_jsonl(f, m, f[:, 1]))
    assert (bits(rf) == bits(f)).all() and (bits(rm) == bits(m)).all()


@pytest.mark.gpu
@pytest.mark.skipif(not have_ref(), reason="needs oracle/_ref (the compiled reference)")
def test_device_trained_model_round_trips_through_reference(golden, capi):
    """A forest trained on the device is written in the reference's format, loaded by
    the reference's EnergyModel::from_json, and predicts identically; the reference's
    own to_json of it is byte-identical to ours."""
    import torch
    from etune_testlib import RefLib
    ctx = capi.Context(0)
    k = "c2_r50_conv3x3/model/"
    feats = torch.from_numpy(golden["c2_r50_conv3x3/features_bits"].view(np.float64).copy()).cuda()
    en = torch.from_numpy(np.resize(golden[k + "train_energy"], feats.shape[0]).copy()).cuda()
    m = capi.train(ctx, feats, en, num_trees=30)
    fe, th, le, ri, va, off, base, ref_e, _ = m.host()
    text = capi.model_to_json(fe, th, le, ri, va, off, m.params, base, ref_e)
    R = RefLib()
    rm = R.model_from_json(text)
    assert rm.to_json() == text
    f = feats.cpu().numpy()
    dev_pred = m.forest().predict(feats).cpu().numpy()
    assert (bits(rm.predict(f)) == bits(dev_pred)).all()


def test_measurement_log_jsonl():
    """MeasurementLog (measure.hpp:63-83): round trip of n records (u64 ids
    intact), empty text -> empty log, tampered energy -> ConsistencyError naming the line,
    unparsable line -> IoError."""
    from paper_2411_18873_b200 import capi
    rng = np.random.default_rng(5)
    r = np.zeros(50, capi.LOG_RECORD_DTYPE)
    r["m"]["candidate_id"] = rng.integers(0, 2**63, 50).astype(np.uint64) * 2 + 1
    r["m"]["latency_ms"] = rng.uniform(1e-3, 10, 50)
    r["m"]["avg_power_w"] = rng.uniform(50, 400, 50)
    r["m"]["energy_mj"] = r["m"]["avg_power_w"] * r["m"]["latency_ms"]
    r["m"]["iterations"] = rng.integers(1, 10**6, 50)
    r["backend"], r["timestamp"] = b"sim", b"2026-10-17T12:34:56Z"
    text = capi.measurement_log_to_jsonl(r)
    assert text.count("\n") == 50 and text.startswith('{"avg_power_w":')
    back = capi.measurement_log_from_jsonl(text)
    for f in ("candidate_id", "latency_ms", "avg_power_w", "energy_mj", "iterations"):
        assert (back["m"][f] == r["m"][f]).all(), f
    assert (back["backend"] == r["backend"]).all() and (back["timestamp"] == r["timestamp"]).all()
    assert len(capi.measurement_log_from_jsonl("")) == 0
    lines = text.splitlines(keepends=True)
    j = json.loads(lines[7])
    j["energy_mj"] = j["energy_mj"] * (1 + 1e-6)
    lines[7] = json.dumps(j, separators=(",", ":")) + "\n"
    with pytest.raises(capi.EtuneError) as e:
        capi.measurement_log_from_jsonl("".join(lines))
    assert e.value.code == 13 and "line 8" in str(e.value)
    with pytest.raises(capi.EtuneError) as e:
        capi.measurement_log_from_jsonl(text + "{not json\n")
    assert e.value.code == 12
