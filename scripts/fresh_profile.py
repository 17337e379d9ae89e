"""Diagnostic: where a fresh-model step's time goes (forest create -> device compile -> score_select -> destroy),
in-stream kernel durations from the CUDA profiler (not serialised like ncu) and the host wall per step.

    python scripts/fresh_profile.py [--n 1048576]
"""
import argparse
import collections
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import FlatForest, parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="conv:1,56,56,64,64,3,1,1")
ap.add_argument("--model", default="c2_r50_conv3x3")
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--k", type=int, default=1024)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
g = np.load(os.path.join(ROOT, "tests", "golden", "golden_reference.npz"))
k = f"{a.model}/model/"
fl = FlatForest(g[k + "feature"], g[k + "threshold"], g[k + "left"], g[k + "right"], g[k + "value"],
                g[k + "offsets"], float(g[k + "base_score"][0]), float(g[k + "learning_rate"][0]))
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op(a.op))
par = plan.sample_random(1024, 42)
gen, _, _ = capi.reproduce(plan, par, a.n, 7)
pred = torch.empty(a.n, dtype=torch.float64, device="cuda")
ids = torch.empty(a.n, dtype=torch.int64, device="cuda")
idx = torch.empty(a.k, dtype=torch.int64, device="cuda")


def fresh():
    fo = capi.Forest.from_flat(ctx, fl)
    fo.score_select(plan, gen, a.k, pred, idx, ids=ids)
    del fo


for _ in range(3):
    fresh()
torch.cuda.synchronize()
walls = []
for _ in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fresh()
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
print(f"fresh step host wall: median {statistics.median(walls) * 1e6:.0f} us over {a.reps}")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(a.reps):
        fresh()
        torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = collections.defaultdict(list)
for e in evs:
    agg[e.name[:60]].append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
print(f"{'kernel / op':62s} {'calls/step':>10s} {'us/step':>9s}")
tot = 0.0
for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    s = sum(v) / a.reps
    tot += s
    print(f"{name:62s} {len(v) / a.reps:10.1f} {s:9.1f}")
print(f"sum of device activity per step: {tot:.1f} us")
