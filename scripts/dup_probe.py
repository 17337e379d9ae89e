import os, sys
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
import torch
from etune_testlib import parse_op
from paper_2411_18873_b200 import capi
ctx = capi.Context(0)
plan = capi.Plan(ctx, parse_op("conv:1,56,56,64,64,3,1,1"))
gen, _, _ = capi.reproduce(plan, plan.sample_random(1024, 42), 1 << 20, 7)
g = gen.view(torch.int64)
n = g.numel(); per = 7; T = 1024
grid = (n + per * T - 1) // (per * T)
pad = torch.full((grid * per * T,), -1, dtype=torch.int64, device=g.device); pad[:n] = g
v = pad.view(grid, per, T)  # [cta][j][t]
# distinct genomes among a thread's 7 candidates
s, _ = torch.sort(v, dim=1)
distinct = 1 + (s[:, 1:, :] != s[:, :-1, :]).sum(dim=1)
print("mean distinct genomes per thread of 7:", distinct.float().mean().item())
print("distinct genomes overall:", torch.unique(g).numel(), "of", n)
# within a warp at fixed j: distinct among 32 lanes
w = v.view(grid, per, T // 32, 32)
s2, _ = torch.sort(w, dim=3)
d2 = 1 + (s2[..., 1:] != s2[..., :-1]).sum(dim=3)
print("mean distinct genomes per warp-load of 32:", d2.float().mean().item())
