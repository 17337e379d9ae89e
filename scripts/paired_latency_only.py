"""SPEC acceptance 7 (energy-aware vs latency-only, Table 2 direction): paired device
searches per seed on the sim backend; prints best energy / latency of both flows."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

text = sys.argv[1] if len(sys.argv) > 1 else "mm:1,512,512,512"
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op(text))
wins = lower5 = 0
for seed in range(seeds):
    kw = dict(M=64, generation_size=256, rng_seed=seed, max_rounds=30)
    ea = capi.Search(plan, capi.search_config(**kw)).run()[-1]
    lo = capi.Search(plan, capi.search_config(latency_only=1, **kw)).run()[-1]
    wins += ea.best_energy_mj <= lo.best_energy_mj
    lower5 += ea.best_energy_mj <= 0.95 * lo.best_energy_mj
    print(f"seed {seed:2d}: energy-aware E={ea.best_energy_mj:.6g} mJ L={ea.best_latency_ms:.6g} ms | "
          f"latency-only E={lo.best_energy_mj:.6g} mJ L={lo.best_latency_ms:.6g} ms | "
          f"dE={100 * (ea.best_energy_mj / lo.best_energy_mj - 1):+.1f}% dL={100 * (ea.best_latency_ms / lo.best_latency_ms - 1):+.1f}%",
          flush=True)
print(f"{text}: energy-aware <= latency-only on {wins}/{seeds} seeds, >= 5% lower on {lower5}/{seeds}")
