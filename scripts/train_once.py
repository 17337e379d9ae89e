"""One device training (diagnostic target for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import Oracle, parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
trees = int(sys.argv[2]) if len(sys.argv) > 2 else 2
O = Oracle()
ctx = capi.Context(0)
op = parse_op("conv:1,56,56,64,64,3,1,1")
plan = capi.Plan(ctx, op)
s, _ = O.sample_random(op, n, 1234)
g = plan.encode(torch.from_numpy(s).cuda())
feats = plan.features(g)
_, _, en, _ = plan.sim_measure(g)
torch.cuda.synchronize()
m = capi.train(ctx, feats, en, num_trees=trees, with_loss=False)
torch.cuda.synchronize()
print("ok")
