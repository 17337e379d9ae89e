"""Wall-clock per stage of one search round (C1 shape) on the GPU, synchronised per
call.  Diagnostic only (not a bench number)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import Oracle, parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402


def t(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{label:48s} {best * 1e3:9.3f} ms", flush=True)
    return out


O = Oracle()
ctx = capi.Context(0)
for text, G, M, nsamp in (("mm:1,1024,1024,1024", 2048, 512, 2048), ("conv:1,56,56,64,64,3,1,1", 16384, 4096, 16384)):
    print(f"== {text} G={G} M={M} samples={nsamp}")
    op = parse_op(text)
    plan = capi.Plan(ctx, op)
    pop = t("sample_random G", lambda: plan.sample_random(G, 42))
    lat = t("sim latency G", lambda: plan.sim_measure(pop, latency_only=True))
    idx = t("topk M of G", lambda: capi.topk(ctx, lat, M))
    par = pop[idx]
    t("reproduce G from M parents", lambda: capi.reproduce(plan, par, G, 7))
    s, _ = O.sample_random(op, nsamp, 1234)
    g = plan.encode(torch.from_numpy(s).cuda())
    feats = plan.features(g)
    _, _, en, _ = plan.sim_measure(g)
    m = t(f"train 100 trees on {nsamp}", lambda: capi.train(ctx, feats, en, with_loss=False), reps=2)
    fo = t("forest from device (host copy + predict blob)", lambda: m.forest())
    t("score M (incl. first-use compile)", lambda: capi.Forest.score(m.forest(), plan, par), reps=2)
    t("score M (compiled)", lambda: fo.score(plan, par))
    t("snr", lambda: capi.snr_db(ctx, en[:M], en[:M] * 1.01))
    # training sub-stages: vary trees to separate per-tree cost from setup
    for nt in (1, 10):
        t(f"train {nt} trees", lambda nt=nt: capi.train(ctx, feats, en, num_trees=nt, with_loss=False), reps=2)
