"""Diagnostic: feature mode (etune_cu_features: genome -> 16 f64 features + id) at 2^20 on the bench
population, events around back-to-back calls, 16 buffers cycled.

    python scripts/features_timing.py [--n 1048576]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="conv:1,56,56,64,64,3,1,1")
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op(a.op))
g, _, _ = capi.reproduce(plan, plan.sample_random(1024, 42), a.n, 7)
nb = 8
bufs = [g.clone() for _ in range(nb)]
feats = [torch.empty((a.n, 16), dtype=torch.float64, device="cuda") for _ in range(nb)]
ids = [torch.empty(a.n, dtype=torch.int64, device="cuda") for _ in range(nb)]
lib = capi.lib()


def call(i):
    b = i % nb
    capi._check(lib.etune_cu_features(ctx.h, plan.h, capi._ptr(bufs[b]), a.n, capi._ptr(feats[b]), capi._ptr(ids[b])))


for i in range(5):
    call(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for i in range(a.iters):
    call(i)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
moved = a.n * (8 + 128 + 8)
print(f"features n={a.n}: {ms * 1e3:.1f} us/call, {a.n / ms / 1e6:.2f} G cand/s, "
      f"{moved / ms / 1e6:.0f} GB/s on 144 B/cand (8 in, 128 + 8 out), SURVEY 192 B basis {a.n * 192 / ms / 1e6:.0f} GB/s")
