"""Diagnostic: device sample_random at the bench search config (ncu launch-list target)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

text = sys.argv[1] if len(sys.argv) > 1 else "conv:1,56,56,64,64,3,1,1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op(text))
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.sample_random(n, 42 + i)
    torch.cuda.synchronize()
    print(f"sample_random({text}, {n}): {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
