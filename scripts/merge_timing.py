"""Time the sharded keep-the-best's W-way merge (merge_records_kernel) for W ranks x k records on ONE
GPU: a fake in-process transport presents W ranks whose all-gather replicates this rank's k records
W times (timing only: the merge is the same code path as over NCCL).  Run it under
`ncu --metrics gpu__time_duration.sum -k regex:merge` for the kernel time.

    python scripts/merge_timing.py [W] [k]
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2411_18873_b200 import capi  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
torch.cuda.set_device(0)
ctx = capi.Context(0)


def allgather(user, d_send, d_recv, nbytes, stream):
    torch.cuda.synchronize()
    src = capi._dev_bytes(d_send, nbytes)
    dst = capi._dev_bytes(d_recv, nbytes * W)
    for w in range(W):
        dst[w * nbytes:(w + 1) * nbytes].copy_(src)
    torch.cuda.synchronize()
    return 0


def broadcast(user, d_buf, nbytes, root, stream):
    return 0


t = capi.Transport(None, W, 0, capi._ALLGATHER_FN(allgather), capi._BROADCAST_FN(broadcast))
capi._check(capi.lib().etune_cu_ctx_attach_transport(ctx.h, C.byref(t)))
n = 1 << 20
score = torch.rand(n, dtype=torch.float64, device="cuda")
for _ in range(5):
    idx, sc = capi.topk_sharded(ctx, score, 0, k)
ctx.synchronize()
ok = bool((sc[1:] >= sc[:-1]).all().item())
print(f"W={W} k={k}: merged top-{k} sorted={ok}")
