"""Quick timing of the scoring forms at the bench config (diagnostic, not the bench):
device compile of the row table, frozen-model score_select step per form, and a fresh-model
step (forest create from host arrays + compile + score_select + destroy).

    python scripts/rows_timing.py [--op conv:1,56,56,64,64,3,1,1] [--model c2_r50_conv3x3]
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
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--forms", default="rows,keyed,class,walk")
ap.add_argument("--no-fresh", action="store_true")
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
bufs = [gen.clone() for _ in range(8)]
pred = torch.empty(a.n, dtype=torch.float64, device="cuda")
ids = torch.empty(a.n, dtype=torch.int64, device="cuda")
idx = torch.empty(a.k, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)
    return e


for form in a.forms.split(","):
    fo = capi.Forest.from_flat(ctx, fl).set_form(form)
    e0 = ev()
    t0 = time.perf_counter()
    fo.compile(plan)
    e1 = ev()
    torch.cuda.synchronize()
    host_ms = (time.perf_counter() - t0) * 1e3
    comp = e0.elapsed_time(e1)
    iters = a.iters if form != "walk" else 5
    for i in range(3):
        fo.score_select(plan, bufs[i % 8], a.k, pred, idx, ids=ids)
    torch.cuda.synchronize()
    e0 = ev()
    for i in range(iters):
        fo.score_select(plan, bufs[i % 8], a.k, pred, idx, ids=ids)
    e1 = ev()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / iters
    capi.profile_score(ctx, True)
    for i in range(iters):
        fo.score_select(plan, bufs[i % 8], a.k, pred, idx, ids=ids)
    _, sc_ms, sel_ms, calls = capi.profile_score(ctx, False)
    calls = max(calls, 1)
    extra = fo.rows_info(plan) if form == "rows" else {}
    print(f"{form:6s} compile: {comp:8.3f} ms device-event / {host_ms:8.3f} ms host wall | step {step*1e3:8.1f} us "
          f"(score kernel {sc_ms/calls*1e3:7.1f} us, select {sel_ms/calls*1e3:6.1f} us) "
          f"-> {a.n/step/1e6:.2f} G cand/s {extra}", flush=True)
    del fo

# fresh model: forest from host arrays + device compile + score_select, every step a new model
torch.cuda.synchronize()
for rep in range(0 if a.no_fresh else 2):
    walls = []
    e0 = ev()
    for i in range(10):
        t0 = time.perf_counter()
        fo = capi.Forest.from_flat(ctx, fl)
        fo.score_select(plan, bufs[i % 8], a.k, pred, idx, ids=ids)
        del fo
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
    e1 = ev()
    torch.cuda.synchronize()
    print(f"fresh-model step (create + compile + score_select + destroy): {e0.elapsed_time(e1)/10:.3f} ms avg "
          f"(host wall median {np.median(walls):.3f} ms)", flush=True)
