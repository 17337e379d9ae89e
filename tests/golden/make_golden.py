"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in a container where /root/reference exists (`make -C oracle` builds
oracle/_ref/libetune_ref.so from the reference sources):

    python tests/golden/make_golden.py

Every array here is produced by the reference library itself through
oracle/ref_shim.cpp (public etune:: APIs only).  The training energies are a
fixed positive function of the reference's own counters (the SPEC:314-322
roofline/power shape, evaluated in numpy) — they are just inputs.
"""
from __future__ import annotations

import os
import platform
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from etune_testlib import RefLib, parse_op  # noqa: E402

# (name, op string, sample size)
OPS = [
    ("mm_1_8_8_8", "mm:1,8,8,8", 256),
    ("mm_2_4_4_4", "mm:2,4,4,4", 256),
    ("mv_1_1_8_8", "mv:1,1,8,8", 190),
    ("conv_1_6_6_2_2_3_1_1", "conv:1,6,6,2,2,3,1,1", 256),
    ("conv_2_4_4_2_2_1_1_0", "conv:2,4,4,2,2,1,1,0", 256),
    ("mm_1_64_64_64", "mm:1,64,64,64", 256),
    ("c1_gemm1024", "mm:1,1024,1024,1024", 256),
    ("c2_r50_conv3x3", "conv:1,56,56,64,64,3,1,1", 256),
    ("c3_bert_ffn", "mm:1,512,3072,768", 256),
    ("r50_fc", "mv:1,1,1000,2048", 256),
    ("r50_conv_7x7_3x3_512", "conv:1,7,7,512,512,3,1,1", 256),
]
MODEL_OPS = ["c1_gemm1024", "c2_r50_conv3x3", "c3_bert_ffn", "mm_1_64_64_64"]
COUNT_KAT = ["mm:1,1,1,1", "mm:1,4,4,4", "mm:1,8,8,8", "mm:1,16,16,16", "mm:1,64,64,64",
             "mm:1,512,512,512", "mm:1,1024,1024,1024", "conv:1,56,56,64,64,3,1,1",
             "mm:1,512,3072,768", "mv:1,1,1000,2048"]


def sim_energy(counters: np.ndarray, num_sms=108) -> np.ndarray:
    """SPEC:314-322 shape (a100_like coefficients, device.hpp:21-30); inputs only."""
    c = counters.astype(np.float64)
    smeff = counters[:, 8].view(np.float64)
    active = c[:, 9]
    flops, glb = c[:, 2], c[:, 4] + c[:, 5]
    shared = c[:, 6] + c[:, 7]
    t_comp = flops / (active * 1.8e11 * smeff)
    t_mem = glb / 3.3e11
    lat_ms = np.maximum(np.maximum(t_comp, t_mem) * 1e3, 1e-5)
    dyn_mj = (flops * 0.002 + glb * 0.125 + shared * 0.0125) * 1e-6
    return (60.0 + 0.55 * active) * lat_ms + dyn_mj


def main():
    R = RefLib()
    out = {}
    out["log1p_2_bits"] = np.array([R.L.ref_log1p(2.0)]).view(np.uint64)
    for name, text, n in OPS:
        op = parse_op(text)
        assert (op == R.parse(text)).all()
        space = R.count(op)
        n = min(n, space)
        s, ids = R.sample_random(op, n, 42)
        out[f"{name}/op"] = op
        out[f"{name}/space"] = np.array([space])
        out[f"{name}/nest"] = R.nest(op)
        out[f"{name}/sample_sched"] = s
        out[f"{name}/sample_ids"] = ids
        out[f"{name}/features_bits"] = R.features(op, s).view(np.uint64)
        out[f"{name}/features_bits_sms148"] = R.features(op, s, 148).view(np.uint64)
        out[f"{name}/counters"] = R.counters(op, s)
        par = s[: min(64, n)]
        rs, rid, lin, ll = R.reproduce(op, par, 512, 7)
        out[f"{name}/repro_parents"] = par
        out[f"{name}/repro_sched"] = rs
        out[f"{name}/repro_ids"] = rid
        out[f"{name}/repro_lineage"] = lin
        out[f"{name}/repro_lineage_len"] = ll
        if space <= 4096:
            full = R.enumerate(op)
            out[f"{name}/enum_sched"] = full
            out[f"{name}/enum_ids"] = R.ids(op, full)
    for name in MODEL_OPS:
        op = out[f"{name}/op"]
        s, _ = R.sample_random(op, 2048, 1234)
        feats = R.features(op, s)
        energy = sim_energy(R.counters(op, s))
        m = R.train(feats, energy)
        f = m.flat()
        pop = out[f"{name}/sample_sched"]
        pf = R.features(op, pop)
        out[f"{name}/model/feature"] = f.feature
        out[f"{name}/model/threshold"] = f.threshold
        out[f"{name}/model/left"] = f.left
        out[f"{name}/model/right"] = f.right
        out[f"{name}/model/value"] = f.value
        out[f"{name}/model/offsets"] = f.offsets
        out[f"{name}/model/base_score"] = np.array([f.base_score])
        out[f"{name}/model/learning_rate"] = np.array([f.learning_rate])
        out[f"{name}/model/reference_energy"] = np.array([m.reference_energy()])
        out[f"{name}/model/training_loss"] = m.training_loss()
        out[f"{name}/model/train_energy"] = energy
        out[f"{name}/model/train_sched"] = s
        out[f"{name}/model/pred_bits"] = m.predict(pf).view(np.uint64)
    for text in COUNT_KAT:
        out[f"count/{text}"] = np.array([R.count(parse_op(text))])
    out["meta/platform"] = np.array([platform.platform()])
    path = os.path.join(HERE, "golden_reference.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)/1e6:.2f} MB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
