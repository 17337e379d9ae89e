"""SimBackend measurement of the C2 search's M candidates (diagnostic target for ncu)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
g = plan.sample_random(n, 42)
plan.sim_measure(g)
torch.cuda.synchronize()
t0 = time.perf_counter()
plan.sim_measure(g)
torch.cuda.synchronize()
print(f"sim_measure {n}: {(time.perf_counter() - t0) * 1e3:.3f} ms")
