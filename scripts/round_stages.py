"""Diagnostic: device time of each stage of one Algorithm-1 round at the bench's search
config (conv R50 3x3, generation 16384, M 4096), each stage synchronised.  Not a bench number."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
G, M = 16384, 4096


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{label:44s} {best * 1e3:8.3f} ms", flush=True)
    return out


par = plan.sample_random(M // 2, 42)
pop, _, _ = t("reproduce G from M/2 parents", lambda: capi.reproduce(plan, par, G, 7))
lat = t("sim latency G", lambda: plan.sim_measure(pop, latency_only=True))
idx = t("topk M of G", lambda: capi.topk(ctx, lat, M))
mgen = pop[idx]
_, _, en0, _ = plan.sim_measure(mgen)
for n in (8192, 16384, 24576):
    g = pop[:n] if n <= G else torch.cat([pop, pop[: n - G]])
    feats = plan.features(g)
    _, _, en, _ = plan.sim_measure(g)
    m = t(f"train 100 trees on {n}", lambda: capi.train(ctx, feats, en, with_loss=False), reps=2)
    fo = t("forest from device", lambda: m.forest())
    t("score M (first use: compile)", lambda: capi.Forest.score(m.forest(), plan, mgen), reps=1)
    t("score M (compiled)", lambda: fo.score(plan, mgen))
t("sim energy kM", lambda: plan.sim_measure(mgen))
t("features kM", lambda: plan.features(mgen))
