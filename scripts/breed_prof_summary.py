"""Summarise ETUNE_BREED_PAR_PROF device timing lines (diagnostic)."""
import sys

import numpy as np

lines = [l.split() for l in open(sys.argv[1]) if l.startswith("ITEM") or l.startswith("GEN")]
idx = [i for i, l in enumerate(lines) if l[0] == "GEN"]
sec = lines[idx[-1]:]
g0, g1 = int(sec[0][1]), int(sec[0][2])
it = np.array([[int(x) for x in l[1:]] for l in sec[1:] if l[0] == "ITEM"])
item, b, Wn, sm, ts, tr, te, ev, sl, nl = it.T[:10]
ck = it.T[10:] if it.shape[1] > 10 else None
dur = (te - tr) / 1e6
print(f"items {len(it)}  gen {(g1 - g0) / 1e6:.3f} ms  last end {(te.max() - g0) / 1e6:.3f} ms  "
      f"last start {(ts.max() - g0) / 1e6:.3f} ms")
print(f"item ms mean {dur.mean():.3f} max {dur.max():.3f}; wait mean {((tr - ts) / 1e6).mean():.3f}")
print(f"evals {ev.sum():.3g}  slow frac {sl.sum() / ev.sum():.4f}  final live mean {nl.mean():.1f}")
T = np.linspace(ts.min(), te.max(), 16)
print("concurrency", [int(((ts <= t) & (te > t)).sum()) for t in T])
for lo, hi in [(0, 100), (100, 1000), (1000, 2048), (2048, 2049)]:
    m = (Wn >= lo) & (Wn < hi)
    if m.any():
        print(f"Wn [{lo},{hi}) n={m.sum()} dur {dur[m].mean():.3f} ms evals {ev[m].mean():.0f}")
if ck is not None:
    for lo, hi in [(0, 100), (2048, 2049)]:
        m = (Wn >= lo) & (Wn < hi)
        print(f"thread-0 cycles/step Wn[{lo},{hi}): step_base {ck[0][m].mean():.0f} A {ck[1][m].mean():.0f} "
              f"barrier {ck[2][m].mean():.0f} B {ck[3][m].mean():.0f}")
