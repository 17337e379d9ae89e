"""BASELINE configs[4]: energy-aware search over the whole ResNet-50 operator set (the 16
stride-1 conv layers + fc; the 7 stride-2 layers are rejected by OperatorSpec::validate,
SURVEY H8).  Layers are sharded over ranks (torchrun: rank r searches layers r, r+W, ...);
each search runs Algorithm 1 on its GPU with the SimBackend.  Prints one JSON line per
layer and a summary (rank 0)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from etune_testlib import parse_op  # noqa: E402
from paper_2411_18873_b200 import capi  # noqa: E402
from test_gpu_resnet50 import R50  # noqa: E402

rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
gen = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
M = int(sys.argv[2]) if len(sys.argv) > 2 else 512
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 10
ctx = capi.Context(local)
total_ms = 0.0
for li, (text, _) in enumerate(R50):
    if li % world != rank:
        continue
    plan = capi.Plan(ctx, parse_op(text), num_sms=148)
    cfg = capi.search_config(M=M, generation_size=gen, rng_seed=42 + li, max_rounds=rounds)
    s = capi.Search(plan, cfg)
    t0 = time.perf_counter()
    reps = s.run()
    ms = (time.perf_counter() - t0) * 1e3
    total_ms += ms
    print(json.dumps({"layer": text, "rank": rank, "rounds": len(reps) - 1, "search_ms": round(ms, 1),
                      "best_energy_mj": reps[-1].best_energy_mj, "best_latency_ms": reps[-1].best_latency_ms,
                      "measured": reps[-1].cumulative_measured}), flush=True)
print(json.dumps({"rank": rank, "layers": len(range(rank, len(R50), world)), "total_search_ms": round(total_ms, 1)}))
