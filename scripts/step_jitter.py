"""Diagnostic: per-step device time distribution of the bench step (score_select at 2^20),
to look for outlier steps.  Not a bench number."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = capi.Context(0)
plan = capi.Plan(ctx, bench.parse_op_text(bench.OP_TEXT))
forest = capi.Forest.from_flat(ctx, bench.load_forest())
par = plan.sample_random(1024, 42)
g0, _, _ = capi.reproduce(plan, par, 1 << 20, 7)
nb = 16
gens = [g0.clone() for _ in range(nb)]
preds = [torch.empty(1 << 20, dtype=torch.float64, device="cuda") for _ in range(nb)]
ids = [torch.empty(1 << 20, dtype=torch.int64, device="cuda") for _ in range(nb)]
top = torch.empty(1024, dtype=torch.int64, device="cuda")
for rep in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(201)]
    torch.cuda.synchronize()
    ev[0].record(st)
    for i in range(200):
        b = i % nb
        forest.score_select(plan, gens[b], 1024, preds[b], top, ids=ids[b])
        ev[i + 1].record(st)
    torch.cuda.synchronize()
    d = np.array([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(200)])
    print(f"rep {rep}: mean {d.mean():.1f} us  median {np.median(d):.1f}  p90 {np.percentile(d, 90):.1f}  "
          f"max {d.max():.1f}  total {d.sum() / 1e3:.2f} ms", flush=True)
