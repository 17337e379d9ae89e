"""The reference-side binding (integration/etune/b200_binding.hpp, shown in INTEGRATION.md)
compiled against the reference's own headers and linked with the unmodified reference library:
tests/cpp/binding_test computes every result through the reference's public API on the CPU and
through the binding on the GPU -- predictions of a 2^16 bred population, its top-1024, 20000
offspring, 4096 samples -- and exits 0 only when all are identical (and every status maps to its
etune:: exception class)."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "binding_test")


def model_json(golden, name):
    k = f"{name}/model/"
    off = golden[k + "offsets"]
    trees = []
    for t in range(len(off) - 1):
        trees.append([{"f": int(golden[k + "feature"][i]), "t": float(golden[k + "threshold"][i]),
                       "l": int(golden[k + "left"][i]), "r": int(golden[k + "right"][i]),
                       "v": float(golden[k + "value"][i])} for i in range(int(off[t]), int(off[t + 1]))])
    return json.dumps({"model_version": "etune-model-v1", "feature_schema": "etune-features-v1",
                       "params": {"num_trees": len(trees), "max_depth": 6,
                                  "learning_rate": float(golden[k + "learning_rate"][0]),
                                  "min_leaf_weight": 1e-3, "reg_lambda": 1.0},
                       "base_score": float(golden[k + "base_score"][0]), "reference_energy_mj": 1.0,
                       "trees": trees})


@pytest.mark.parametrize("op,model", [("conv:1,56,56,64,64,3,1,1", "c2_r50_conv3x3"),
                                      ("mm:1,512,3072,768", "c3_bert_ffn")])
def test_reference_binding(golden, op, model):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/binding_test is not built (needs /root/reference at build time)")
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        f.write(model_json(golden, model))
        path = f.name
    try:
        r = subprocess.run([BIN, path, op, str(1 << 16)], capture_output=True, text=True, timeout=600)
    finally:
        os.unlink(path)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "binding ok" in r.stdout
