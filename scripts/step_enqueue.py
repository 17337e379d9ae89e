"""Diagnostic: host enqueue cost of one score_select call vs the device time per step
(is the back-to-back step loop host-bound?).  Also replays the same steps from a CUDA graph.

    python scripts/step_enqueue.py [--n 1048576]
"""
import argparse
import os
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
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--bufs", type=int, default=16)
ap.add_argument("--no-ids", action="store_true", help="score without candidate ids")
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
nb = a.bufs
bufs = [gen.clone() for _ in range(nb)]
preds = [torch.empty(a.n, dtype=torch.float64, device="cuda") for _ in range(nb)]
idss = [None if a.no_ids else torch.empty(a.n, dtype=torch.int64, device="cuda") for _ in range(nb)]
idx = torch.empty(a.k, dtype=torch.int64, device="cuda")
fo = capi.Forest.from_flat(ctx, fl)
fo.compile(plan)
for i in range(5):
    fo.score_select(plan, bufs[i % nb], a.k, preds[i % nb], idx, ids=idss[i % nb])
torch.cuda.synchronize()
ref = idx.clone()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)
    return e


for rep in range(3):
    torch.cuda.synchronize()
    e0 = ev()
    t0 = time.perf_counter()
    for i in range(a.iters):
        fo.score_select(plan, bufs[i % nb], a.k, preds[i % nb], idx, ids=idss[i % nb])
    t1 = time.perf_counter()
    e1 = ev()
    torch.cuda.synchronize()
    print(f"eager: host enqueue {(t1 - t0) / a.iters * 1e6:.1f} us/call, device {e0.elapsed_time(e1) / a.iters * 1e3:.1f} us/step",
          flush=True)
# a busy-wait kernel in front so the host runs ahead: device time with a full queue
for rep in range(2):
    torch.cuda.synchronize()
    torch.cuda._sleep(50_000_000)
    e0 = ev()
    for i in range(a.iters):
        fo.score_select(plan, bufs[i % nb], a.k, preds[i % nb], idx, ids=idss[i % nb])
    e1 = ev()
    torch.cuda.synchronize()
    print(f"queued: device {e0.elapsed_time(e1) / a.iters * 1e3:.1f} us/step", flush=True)
assert torch.equal(idx, ref)
