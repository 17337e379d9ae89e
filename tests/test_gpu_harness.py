"""The NVML measurement harness (etune_cu_candidate_run / etune_cu_nvml_measure): the
candidate kernels compute the operator correctly for every schedule shape they accept
(checked against torch fp32), and the measurement records obey the energy identity."""
import numpy as np
import pytest

from etune_testlib import parse_op

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2411_18873_b200 import capi as c
    return c


@pytest.fixture(scope="module")
def ctx(capi):
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return capi.Context(0)


def _operands(op, nest):
    g = torch.Generator(device="cuda").manual_seed(0)
    if op[0] == 2:
        b, h, w, cin, cout, ks, st, pad = (int(op[i]) for i in (1, 5, 6, 7, 8, 9, 10, 11))
        x = torch.rand((b, cin, h, w), generator=g, device="cuda") - 0.5
        wt = torch.rand((cout, cin, ks, ks), generator=g, device="cuda") - 0.5
        ref = torch.nn.functional.conv2d(x, wt, stride=st, padding=pad).reshape(b, cout, -1)
        return x, wt.reshape(cout, -1).contiguous(), ref
    B, M, N, K = (int(v) for v in nest)
    a = torch.rand((B, M, K), generator=g, device="cuda") - 0.5
    bm = torch.rand((B, K, N), generator=g, device="cuda") - 0.5
    return a, bm, torch.bmm(a, bm)


@pytest.mark.parametrize("text", ["mm:1,64,96,80", "mm:3,32,48,40", "mv:1,1,256,128", "conv:1,14,14,16,32,3,1,1",
                                  "conv:2,8,8,8,16,1,1,0", "conv:1,12,12,4,8,3,3,0"])
def test_candidate_kernels_compute_the_operator(oracle, ctx, capi, text):
    op = parse_op(text)
    plan = capi.Plan(ctx, op)
    nest = plan.nest()
    a, b, ref = _operands(op, nest)
    sched, _ = oracle.sample_random(op, min(60, oracle.count(op)), 5)
    ran = 0
    for s in sched:
        c = torch.full(ref.shape, float("nan"), device="cuda")
        try:
            capi.candidate_run(plan, s, a, b, c)
        except capi.EtuneError as e:
            assert e.code == 67  # infeasible for the kernel (per-thread tile / smem / registers)
            continue
        torch.cuda.synchronize()
        ran += 1
        assert torch.allclose(c, ref, rtol=1e-4, atol=1e-4), s
    assert ran > 0


def test_nvml_measure_records(oracle, ctx, capi):
    if not capi.nvml_available(ctx):
        pytest.skip("NVML energy counters not readable here")
    op = parse_op("mm:1,512,512,512")
    sched, ids = oracle.sample_random(op, 6, 3)
    recs = capi.nvml_measure(capi.Plan(ctx, op), sched, warmup_ms=20, window_ms=120, min_iterations=5)
    assert [r["candidate_id"] for r in recs] == list(ids)
    for r in recs:
        if not r["feasible"]:
            assert r["latency_ms"] == float("inf")
            continue
        assert r["latency_ms"] > 0 and r["iterations"] >= 5
        assert 20.0 < r["avg_power_w"] < 2000.0
        assert abs(r["energy_mj"] - r["avg_power_w"] * r["latency_ms"]) <= 1e-9 * r["energy_mj"]
    bad = sched.copy()
    bad[2, 10] = 3
    with pytest.raises(capi.EtuneError) as e:
        capi.nvml_measure(capi.Plan(ctx, op), bad)
    assert e.value.code == 4 and e.value.index == 2


def test_search_on_the_gpu_backend(oracle, ctx, capi):
    """Algorithm 1 with measurements on this B200 (BASELINE configs[2] shape: BERT FFN
    GEMM, the cost model updated every round from NVML-measured candidate kernels)."""
    if not capi.nvml_available(ctx):
        pytest.skip("NVML energy counters not readable here")
    op = parse_op("mm:1,512,3072,768")
    plan = capi.Plan(ctx, op)
    cfg = capi.search_config(M=32, generation_size=128, rng_seed=5, max_rounds=2, backend=1, latency_reps=2,
                             warmup_ms=10, window_ms=40, min_iterations=3, num_trees=30)
    s = capi.Search(plan, cfg)
    reps = s.run()
    assert len(reps) == 3
    assert reps[0].measured == 32 and reps[0].cumulative_measured == 32
    best = [r.best_energy_mj for r in reps]
    assert all(b2 <= b1 for b1, b2 in zip(best, best[1:]))
    assert 0 < best[-1] < 1e30 and reps[-1].best_power_w > 20
    sched, bid, lat, en = s.best()
    assert oracle.ids(op, sched[None, :])[0] == bid and lat > 0
