"""Diagnostic: in-stream kernel durations of the exact block-parallel reproduce at 2^20 (CUDA profiler)."""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op(sys.argv[1] if len(sys.argv) > 1 else "conv:1,56,56,64,64,3,1,1"))
g = plan.sample_random(1024, 42)
n = 1 << 20
for s in range(3):
    capi.reproduce(plan, g, n, 7 + s)
torch.cuda.synchronize()
reps = 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for s in range(reps):
        capi.reproduce(plan, g, n, 7 + s)
        torch.cuda.synchronize()
agg = collections.defaultdict(list)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        agg[e.name[:70]].append(e.device_time if hasattr(e, "device_time") else e.cuda_time)
for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{name:72s} {len(v) / reps:6.1f} {sum(v) / reps / 1e3:9.3f} ms")
