"""Per-kernel timing of the block-parallel exact reproduce (diagnostic)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

op_text = sys.argv[1] if len(sys.argv) > 1 else "conv:1,56,56,64,64,3,1,1"
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op(op_text))
g = plan.sample_random(1024, 42)
for n in (1 << 14, 1 << 16, 1 << 18, 1 << 20):
    capi.reproduce(plan, g, n, 7)
    torch.cuda.synchronize()
    ts = []
    for r in range(3):
        t0 = time.perf_counter()
        capi.reproduce(plan, g, n, 7 + r)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    os.environ["ETUNE_BREED_PAR_MIN"] = str(1 << 40)
    t0 = time.perf_counter()
    capi.reproduce(plan, g, n, 7)
    torch.cuda.synchronize()
    ser = (time.perf_counter() - t0) * 1e3
    del os.environ["ETUNE_BREED_PAR_MIN"]
    print(f"{op_text} n={n}: parallel {min(ts):.3f} ms, single-CTA chain {ser:.3f} ms", flush=True)
