"""Diagnostic: per-stage times of Algorithm-1 rounds at the bench's search config
(ETUNE_SEARCH_TRACE=1 synchronises after every stage).  Not a bench number."""
import os
import sys

os.environ.setdefault("ETUNE_SEARCH_TRACE", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
cfg = capi.search_config(M=4096, generation_size=16384, rng_seed=42, max_rounds=rounds, patience=1 << 30)
s = capi.Search(plan, cfg)
print("initial", round(s.initial().wall_ms, 3), flush=True)
for _ in range(rounds):
    r = s.round()
    print(f"round wall {r.wall_ms:.3f} ms", flush=True)
