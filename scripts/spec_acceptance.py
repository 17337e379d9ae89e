"""SPEC acceptance criteria 6, 8 and 9 (SPEC.md "ACCEPTANCE CRITERIA") on the device search
and SimBackend: search optimality vs the brute-force optimum of MM(1,16,16,16), the
measurement-budget speedup against a forced k = 1.0 run, and the latency/power
inverse correlation over the MM(1,64,64,64) space.  (7 is scripts/paired_latency_only.py.)"""
import os
import sys

import numpy as np
import torch
from scipy.stats import spearmanr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import Oracle, parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

O = Oracle()
ctx = capi.Context(0)


def space(text):
    op = parse_op(text)
    plan = capi.Plan(ctx, op)
    g = plan.encode(torch.from_numpy(np.ascontiguousarray(O.enumerate(op))).cuda())
    lat, pw, en, _ = (t.cpu().numpy() for t in plan.sim_measure(g))
    return plan, lat, pw, en


# 6. search optimality at desk scale
plan, lat, pw, en = space("mm:1,16,16,16")
opt = en.min()
ok = 0
for seed in range(10):
    r = capi.Search(plan, capi.search_config(M=64, generation_size=256, rng_seed=seed, max_rounds=30)).run()[-1]
    within = r.best_energy_mj <= 1.05 * opt
    ok += within
    print(f"6. seed {seed}: best {r.best_energy_mj:.6g} mJ vs optimum {opt:.6g} mJ ({100 * (r.best_energy_mj / opt - 1):+.2f}%)"
          f" after {r.round} rounds", flush=True)
print(f"6. MM(1,16,16,16), {len(en)} schedules: within 5% of the brute-force optimum on {ok}/10 seeds (need >= 9)")

# 8. measurement-budget speedup over 15 rounds (mu = 20 dB) vs forced k = 1.0
plan, *_ = space("mm:1,64,64,64")
ratios = []
for seed in range(5):
    kw = dict(M=64, generation_size=256, rng_seed=seed, max_rounds=15, patience=1 << 30)
    dyn = capi.Search(plan, capi.search_config(mu_db=20.0, **kw)).run()[-1].cumulative_measured
    forced = capi.Search(plan, capi.search_config(mu_db=1e9, **kw)).run()[-1].cumulative_measured  # snr < mu: k stays 1
    ratios.append(dyn / forced)
    print(f"8. seed {seed}: cumulative measurements {dyn} vs forced k=1.0 {forced}: {dyn / forced:.3f}x", flush=True)
print(f"8. MM(1,64,64,64): ratio max {max(ratios):.3f} (need <= 0.55)")

# 9. inverse correlation premise
_, lat, pw, en = space("mm:1,64,64,64")
rho = spearmanr(lat, pw).correlation
print(f"9. MM(1,64,64,64), {len(lat)} schedules: Spearman(latency, power) = {rho:.4f} (need < 0)")
