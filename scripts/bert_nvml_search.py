"""BASELINE configs[2]: BERT-base FFN GEMM 512x768x3072 (mm:1,512,3072,768) energy-aware search
with the cost model updated every round from NVML-measured candidate kernels on this B200
(search backend 1: the latency filter times every generated candidate's kernel with CUDA events,
the k*M selected are measured with the NVML energy counter).

Runs the energy-aware search and the latency-only baseline (run_latency_only) from
the same seed and prints one JSON line per round plus a summary: the energy of the best kernel
each found, its latency and power, the measurements spent.

    python scripts/bert_nvml_search.py [M] [generation] [rounds] [window_ms]
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 256
G = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 5
window = float(sys.argv[4]) if len(sys.argv) > 4 else 60.0
torch.cuda.set_device(0)
ctx = capi.Context(0)
if not capi.nvml_available(ctx):
    print(json.dumps({"unavailable": "NVML energy counters not readable"}))
    sys.exit(0)
op = parse_op("mm:1,512,3072,768")
out = {}
for mode in ("energy_aware", "latency_only"):
    plan = capi.Plan(ctx, op, num_sms=148)
    cfg = capi.search_config(M=M, generation_size=G, rng_seed=42, max_rounds=rounds, patience=1 << 30, backend=1,
                             latency_reps=3, warmup_ms=20, window_ms=window, min_iterations=5,
                             latency_only=1 if mode == "latency_only" else 0)
    s = capi.Search(plan, cfg)
    t0 = time.perf_counter()
    reps = []
    r = s.initial()
    reps.append(r)
    print(json.dumps({"mode": mode, **{k: v for k, v in r.as_dict().items()}}), flush=True)
    for _ in range(rounds):
        r = s.round()
        reps.append(r)
        print(json.dumps({"mode": mode, **{k: v for k, v in r.as_dict().items()}}), flush=True)
    wall = time.perf_counter() - t0
    sched, bid, lat, en = s.best()
    out[mode] = {"best_energy_mj": en, "best_latency_ms": lat, "best_power_w": reps[-1].best_power_w,
                 "best_id": bid, "best_schedule": [int(x) for x in sched], "measurements": reps[-1].cumulative_measured,
                 "rounds": rounds, "wall_s": round(wall, 1),
                 "k_fifths": [r.k_after_fifths for r in reps], "snr_db": [r.snr_db for r in reps[1:]]}
ea, lo = out["energy_aware"], out["latency_only"]
print(json.dumps({"summary": out, "config": {"op": "mm:1,512,3072,768", "M": M, "generation": G, "rounds": rounds,
                                             "nvml_window_ms": window, "gpu": torch.cuda.get_device_name(0)},
                  "energy_saving_vs_latency_only": 1.0 - ea["best_energy_mj"] / lo["best_energy_mj"]}), flush=True)
