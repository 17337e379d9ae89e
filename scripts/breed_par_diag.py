"""Diagnostic: block-parallel exact reproduce at 2^20 under different window widths."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
g = plan.sample_random(1024, 42)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
for sd in sys.argv[2:] or ["5.0"]:
    os.environ["ETUNE_BREED_PAR_SD"] = sd
    capi.reproduce(plan, g, n, 7)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    capi.reproduce(plan, g, n, 8)
    e1.record()
    torch.cuda.synchronize()
    print(f"n={n} sd={sd}: {e0.elapsed_time(e1):.3f} ms", flush=True)
