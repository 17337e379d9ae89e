"""Diagnostic: does NVML polling from a background thread slow the bench step loop?
(step = score_select at 2^20; device time of 200 steps)"""
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import bench  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402
import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
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


def loop():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for i in range(200):
        b = i % nb
        forest.score_select(plan, gens[b], 1024, preds[b], top, ids=ids[b])
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 200 * 1e3


def poll(fn, period, stop, calls):
    while not stop.wait(period):
        t = time.perf_counter()
        fn()
        calls.append(time.perf_counter() - t)


for _ in range(3):
    loop()
variants = {"none": None,
            "clock 5ms": lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
            "reasons 5ms": lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
            "busy-python 5ms": lambda: sum(range(20000))}
for name, fn in variants.items():
    res = []
    for rep in range(3):
        stop = threading.Event()
        calls = []
        th = None
        if fn:
            th = threading.Thread(target=poll, args=(fn, 0.005, stop, calls), daemon=True)
            th.start()
        res.append(loop())
        stop.set()
        if th:
            th.join()
    print(f"{name:16s} step us {['%.1f' % r for r in res]}  call ms {1e3 * np.mean(calls) if calls else 0:.3f}",
          flush=True)
