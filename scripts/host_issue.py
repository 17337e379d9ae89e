"""Diagnostic: host issue time vs device time of the bench step loop, with and without
bench.ClockSampler running (step = score_select at 2^20)."""
import os
import sys
import time

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


def loop(clk):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    if clk:
        clk.sample()
    t0 = time.perf_counter()
    for i in range(200):
        b = i % nb
        forest.score_select(plan, gens[b], 1024, preds[b], top, ids=ids[b])
    t1 = time.perf_counter()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 200 * 1e3, (t1 - t0) / 200 * 1e6


for _ in range(5):
    loop(None)
for mode in ("plain", "clock", "plain", "clock", "plain", "clock"):
    if mode == "clock":
        with bench.ClockSampler(0) as clk:
            d, h = loop(clk)
    else:
        d, h = loop(None)
    print(f"{mode:6s} device {d:.1f} us/step  host issue {h:.1f} us/step", flush=True)
