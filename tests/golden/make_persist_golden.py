"""Generate tests/golden/persist/ from the UNMODIFIED reference (oracle/_ref):
the reference's own serialisations, which the product's writers must reproduce byte
for byte and its readers must parse bit for bit.

    python tests/golden/make_persist_golden.py

  model_<name>.json   EnergyModel::to_json of the golden forests (energy_model.cpp:259-284)
  samples.jsonl       save_energy_samples of golden feature rows + edge-case doubles
                      (energy_model.cpp:372-383)
  device_*.json       device_profile_to_json (device.cpp:44-62)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "persist")
sys.path.insert(0, os.path.dirname(HERE))
from etune_testlib import RefLib  # noqa: E402
from make_golden import MODEL_OPS  # noqa: E402


def model_json_from_npz(g, name):
    k = f"{name}/model/"
    off = g[k + "offsets"]
    trees = []
    for t in range(len(off) - 1):
        a, b = int(off[t]), int(off[t + 1])
        trees.append([{"f": int(g[k + "feature"][i]), "t": float(g[k + "threshold"][i]), "l": int(g[k + "left"][i]),
                       "r": int(g[k + "right"][i]), "v": float(g[k + "value"][i])} for i in range(a, b)])
    return json.dumps({"model_version": "etune-model-v1", "feature_schema": "etune-features-v1",
                       "params": {"num_trees": len(off) - 1, "max_depth": 6,
                                  "learning_rate": float(g[k + "learning_rate"][0]), "min_leaf_weight": 1e-3,
                                  "reg_lambda": 1.0},
                       "base_score": float(g[k + "base_score"][0]),
                       "reference_energy_mj": float(g[k + "reference_energy"][0]), "trees": trees})


def edge_doubles(rng, n):
    """Magnitudes across the decimal/exponential switch of nlohmann's layout and
    values whose shortest representation is long."""
    fixed = [1e-300, 5e-324, 2.2250738585072014e-308, 1e-5, 1e-4, 0.00012345, 0.001, 0.1, 0.3, 1.0, 2.0,
             123456789.0, 1e15, 9.999999999999998e14, 1e16, 1.2345678901234567e16, 1e300, 1.7976931348623157e308,
             -0.0, -1.5, -1e-7, 0.1 + 0.2, 1 / 3, 2 / 3, 100.0, 1e21, 4.35, 0.5, 65536.0]
    r = list(fixed)
    e = rng.uniform(-320, 308, n)
    r += list(rng.uniform(1, 10, n) * 10.0 ** e)
    r += list(rng.standard_normal(n))
    r += list(np.log1p(rng.integers(1, 1 << 40, n).astype(np.float64)))
    return np.array([x for x in r if np.isfinite(x)], np.float64)


def main():
    R = RefLib()
    g = np.load(os.path.join(HERE, "golden_reference.npz"))
    os.makedirs(OUT, exist_ok=True)
    for name in MODEL_OPS:
        m = R.model_from_json(model_json_from_npz(g, name))
        open(os.path.join(OUT, f"model_{name}.json"), "w").write(m.to_json())
    rng = np.random.default_rng(2411)
    vals = edge_doubles(rng, 2000)
    feats = [g[f"{n}/features_bits"].view(np.float64) for n in ("c2_r50_conv3x3", "c1_gemm1024", "mm_1_8_8_8")]
    feats.append(np.resize(vals, (len(vals) + 15) // 16 * 16).reshape(-1, 16))
    feats = np.concatenate(feats)
    meas = np.abs(np.resize(vals, len(feats))) + 1e-3
    norm = np.resize(vals[::-1], len(feats))
    open(os.path.join(OUT, "samples.jsonl"), "w").write(R.samples_to_jsonl(feats, meas, norm))
    d0 = [60.0, 0.55, 0.002, 0.125, 0.0125, 1.8e11, 3.3e11, 1e-5, 50.0, 2.0, 0.05]
    open(os.path.join(OUT, "device_a100_like.json"), "w").write(R.device_profile_to_json(108, d0, 1234, "a100-like"))
    d1 = [1e3 / 3, 1.25e-4, 3.3e-9, 0.1, 7.0, 4.5e12, 8e12, 2.5e-6, 30.0, 0.0, 0.0]
    open(os.path.join(OUT, "device_b200_custom.json"), "w").write(
        R.device_profile_to_json(148, d1, (1 << 64) - 1, 'b200 "sxm"\tnode\\1'))
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
