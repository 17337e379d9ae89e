"""Diagnostic: per-barrier timeline of the training megakernel (ETUNE_TRAIN_TRACE=1),
on the bench's search config at n samples.  Not a bench number."""
import os
import sys

os.environ["ETUNE_TRAIN_TRACE"] = "1"
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
pop, _, _ = capi.reproduce(plan, plan.sample_random(2048, 42), n, 7)
feats = plan.features(pop)
_, _, en, _ = plan.sim_measure(pop)
for _ in range(2):
    capi.train(ctx, feats, en, with_loss=False)
    torch.cuda.synchronize()
