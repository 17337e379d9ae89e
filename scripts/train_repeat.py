"""Diagnostic: spread of repeated trainings at fixed n (wall time with a device sync)."""
import sys
import time
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
for n in [int(a) for a in sys.argv[1:]] or [13927, 15566]:
    pop, _, _ = capi.reproduce(plan, plan.sample_random(2048, 42), n, 7)
    feats = plan.features(pop)
    _, _, en, _ = plan.sim_measure(pop)
    ts = []
    for _ in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        capi.train(ctx, feats, en, with_loss=False)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(n, " ".join(f"{t:.1f}" for t in ts), flush=True)
