# e2e (etune_cu_score_select_host, pageable 2^20 rows): host split per call for chunk sizes and host thread counts
O=gpurun_out/e2e_sweep.log
: > $O
nproc >> $O
python - >> $O 2>&1 <<'PY'
import numpy as np, time
a = np.ones(100 * 2**20 // 8); b = np.empty_like(a)
for _ in range(3): np.copyto(b, a)
t0 = time.perf_counter(); np.copyto(b, a); dt = time.perf_counter() - t0
print(f"numpy single-thread copy 100 MB: {200 / dt / 1e3:.1f} GB/s (read + write)")
PY
for cl in 16 17 18; do for th in 8 16; do
  echo "== chunk 2^$cl threads $th" >> $O
  ETUNE_E2E_TRACE=1 ETUNE_E2E_CHUNK_LOG2=$cl ETUNE_HOST_THREADS=$th python scripts/e2e_trace.py 2>&1 | grep -v Warn | tail -6 >> $O
done; done
