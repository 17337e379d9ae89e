"""One device reproduce at the C2 search shape (diagnostic target for ncu)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
par = plan.sample_random(P, 42)
capi.reproduce(plan, par, G, 7)
torch.cuda.synchronize()
t0 = time.perf_counter()
out, partner, ids = capi.reproduce(plan, par, G, 8)
torch.cuda.synchronize()
print(f"reproduce {G} from {P}: {(time.perf_counter() - t0) * 1e3:.2f} ms")
