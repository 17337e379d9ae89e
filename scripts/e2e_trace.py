"""Diagnostic: host-side split of the e2e call (etune_cu_score_select_host on a pageable 2^20 Schedule[]):
ETUNE_E2E_TRACE=1 prints per call the total, the narrowing and the staging waits.

    ETUNE_E2E_TRACE=1 python scripts/e2e_trace.py
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import FlatForest, parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "golden_reference.npz"))
k = "c2_r50_conv3x3/model/"
fl = FlatForest(g[k + "feature"], g[k + "threshold"], g[k + "left"], g[k + "right"], g[k + "value"],
                g[k + "offsets"], float(g[k + "base_score"][0]), float(g[k + "learning_rate"][0]))
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
gen, _, _ = capi.reproduce(plan, plan.sample_random(1024, 42), 1 << 20, 7)
sched = plan.decode(gen).cpu().numpy()
if os.environ.get("E2E_PINNED") == "1":  # the caller's rows in pinned memory (raw DMA chunks)
    sched = torch.from_numpy(sched).pin_memory().numpy()
fo = capi.Forest.from_flat(ctx, fl)
idx = np.zeros(1024, np.int64)
pred = np.zeros(len(sched))
for r in range(12):
    t0 = time.perf_counter()
    fo.score_select_host(plan, sched, 1024, idx, pred)
    print(f"call {r}: {(time.perf_counter() - t0) * 1e3:.3f} ms", file=sys.stderr, flush=True)
