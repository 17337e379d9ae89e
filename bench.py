"""Benchmark: candidate schedules scored per second and search-round latency (BASELINE.json metric).

Step = one pass of the hot path over one batch: fused score (features -> 100-tree
energy model -> prediction + candidate id) of the rank's population shard, then
"keep the best": top-k by (score, index); for N>1 the per-shard top-k records are
all-gathered over NCCL and merged identically on every rank.

    python bench.py [--gpus N --steps K --warmup W]            # our B200 path
    python bench.py --impl reference [--gpus N ...]            # reference CPU path
    torchrun --nproc-per-node N bench.py --gpus N ...          # N>1

Workload (config.workload): the ResNet-50 3x3 conv layer of BASELINE configs[1]
(conv:1,56,56,64,64,3,1,1), population 2^20 per GPU (north_star / configs[3] top
size), bred exactly like SURVEY §8(d): reproduce(sample_random(op,1024,42), 2^20,
GeneticRates{}, seed 7); model = the reference-trained 100-tree forest on
sample_random(op,2048,1234) (tests/golden fixture).  L2: 16 distinct population
buffers (384 MB incl. outputs) are cycled so no step reads another's data from the
126 MB L2.

Also reported: e2e (the same scoring through the reference-facing C-ABI call on HOST
Schedule[] buffers, H2D/D2H inside the timed region), search_round_latency (Algorithm 1
rounds of BASELINE configs[1]: generation 16384, M 4096, on the device), roofline of the
score kernel and the reference CPU path (cpu_baseline).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

OP_TEXT = "conv:1,56,56,64,64,3,1,1"
MODEL_KEY = "c2_r50_conv3x3"
METRIC = "candidate schedules scored/sec"
UNIT = "candidates/s"
# algorithmic bytes per candidate, score mode: 48 B schedule in (12 x int32 SoA) + 8 B f64
# prediction + 8 B u64 id out.  This design's population is an 8-byte genome, so the kernel itself moves
# DESIGN_BYTES (8 in + 16 out); both fractions are reported.
ALGO_BYTES = 64
DESIGN_BYTES = 24


def workload(k: int) -> str:
    """config.workload, identical for both arms."""
    return f"score (features -> 100-tree GBDT -> prediction) + top-{k} of {OP_TEXT} candidates"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--pop", type=int, default=1 << 20, help="candidates per GPU per step")
    p.add_argument("--k", type=int, default=1024, help="top-k kept per step")
    p.add_argument("--bufs", type=int, default=16)
    p.add_argument("--cpu-seconds", type=float, default=10.0, help="target CPU-baseline sample duration")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-search", action="store_true", help="skip the search-round latency measurement")
    p.add_argument("--search-rounds", type=int, default=5)
    return p.parse_args()


def load_forest():
    from etune_testlib import FlatForest
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_reference.npz"))
    k = f"{MODEL_KEY}/model/"
    return FlatForest(g[k + "feature"], g[k + "threshold"], g[k + "left"], g[k + "right"], g[k + "value"],
                      g[k + "offsets"], float(g[k + "base_score"][0]), float(g[k + "learning_rate"][0]))


def make_population(n: int, seed: int = 7):
    """SURVEY §8(d) population: reproduce(sample_random(op,1024,42), n, {}, seed)."""
    from etune_testlib import Oracle, parse_op
    O = Oracle()
    op = parse_op(OP_TEXT)
    par, _ = O.sample_random(op, 1024, 42)
    s, _, _, _ = O.reproduce(op, par, n, seed)
    return op, s


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def forest_json(f) -> str:
    """etune-model-v1 JSON (energy_model.cpp:259-284) so the reference loads the same model."""
    trees = []
    for t in range(f.num_trees):
        a, b = int(f.offsets[t]), int(f.offsets[t + 1])
        trees.append([{"f": int(f.feature[i]), "t": float(f.threshold[i]), "l": int(f.left[i]),
                       "r": int(f.right[i]), "v": float(f.value[i])} for i in range(a, b)])
    return json.dumps({"model_version": "etune-model-v1", "feature_schema": "etune-features-v1",
                       "params": {"num_trees": f.num_trees, "max_depth": 6, "learning_rate": f.learning_rate,
                                  "min_leaf_weight": 1e-3, "reg_lambda": 1.0},
                       "base_score": f.base_score, "reference_energy_mj": 1.0, "trees": trees})


def cpu_score_runner():
    """Returns (kind, fn(op, sched) -> preds, threads).  Prefers the unmodified reference
    (oracle/_ref) over the restatement (oracle/lib)."""
    from etune_testlib import Oracle, RefLib, have_ref
    forest = load_forest()
    threads = cpu_threads()
    if have_ref():
        R = RefLib()
        model = R.model_from_json(forest_json(forest))
        return "reference", (lambda op, s: model.score_threads(op, s, threads)), threads
    O = Oracle()
    return "port", (lambda op, s: O.score_threads(op, s, forest, threads)), threads


def time_cpu(op, sched, target_s: float):
    """Bounded CPU sample: whole passes over (a prefix of) the population until
    ~target_s of work has been timed."""
    kind, fn, threads = cpu_score_runner()
    m = min(len(sched), 20000)
    t0 = time.perf_counter()
    fn(op, sched[:m])
    rate = m / max(time.perf_counter() - t0, 1e-9)
    total = int(max(m, rate * target_s))
    done, dt = 0, 0.0
    while done < total:
        chunk = sched[: min(len(sched), total - done)]
        t0 = time.perf_counter()
        fn(op, chunk)
        dt += time.perf_counter() - t0
        done += len(chunk)
    return {"value": done / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{done} candidates (passes over the bench population, {OP_TEXT}); the reference's "
                      f"extract_features + EnergyModel::predict per candidate over {threads} std::threads; "
                      f"{dt:.1f} s"}


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML during the timed region
    (a background thread every 5 ms, plus explicit samples at its start and end)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm, self.max_sm, self.reasons = [], 0.0, set()
        self.stop = threading.Event()
        self.nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nv = None

    def sample(self):
        if not self.nv:
            return
        try:
            self.sm.append(float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for nm, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(nm)
        except Exception:
            pass

    def _loop(self):
        while not self.stop.wait(0.005):
            self.sample()

    def __enter__(self):
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm or None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    op, sched = make_population(args.pop)
    kind, fn, threads = cpu_score_runner()
    # bounded sample per step so the whole run ends in a few minutes
    m = min(len(sched), 20000)
    t0 = time.perf_counter()
    fn(op, sched[:m])
    rate = m / max(time.perf_counter() - t0, 1e-9)
    per_step = int(min(len(sched), max(10000, rate * 8.0 / max(args.steps + args.warmup, 1))))
    for w in range(args.warmup):
        fn(op, sched[:per_step])
    times = []
    for s in range(args.steps):
        lo = (s * per_step) % max(1, len(sched) - per_step)
        t0 = time.perf_counter()
        preds = fn(op, sched[lo:lo + per_step])
        order = np.lexsort((np.arange(len(preds)), preds))[: args.k]  # keep the best (score, index)
        times.append(time.perf_counter() - t0)
        del order
    value = per_step * len(times) / sum(times)
    sample = (f"{per_step} candidates/step of the bench population ({OP_TEXT}): the reference's "
              f"extract_features + EnergyModel::predict over {threads} threads + top-{args.k}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(args.k), "op": OP_TEXT, "population_per_step": per_step, "k": args.k,
                   "implementation": "the reference's CPU path (oracle/_ref: unmodified sources) over all host threads, "
                                     "bounded sample per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def search_round_latency(ctx, capi, rounds: int):
    """Algorithm-1 round latency on the device: BASELINE configs[1] search
    (conv R50 3x3, generation 16384, M = 4096, SimBackend), median wall ms of `rounds`
    rounds after the initial round (each round: reproduce, latency filter, score,
    select, measure, SNR, retrain on all samples, parents)."""
    op = parse_op_text(OP_TEXT)
    plan = capi.Plan(ctx, op)
    cfg = capi.search_config(M=4096, generation_size=16384, rng_seed=42, max_rounds=rounds, patience=1 << 30)
    s = capi.Search(plan, cfg)
    init = s.initial()
    ms = [s.round().wall_ms for _ in range(rounds)]
    return {"value": statistics.median(ms), "unit": "ms", "rounds": rounds, "per_round_ms": [round(x, 3) for x in ms],
            "initial_round_ms": round(init.wall_ms, 3),
            "config": "conv:1,56,56,64,64,3,1,1 generation 16384, M 4096, k from 1.0, mu 20 dB, SimBackend, "
                      "100-tree retrain on all accumulated samples every round"}


def parse_op_text(text):
    from etune_testlib import parse_op
    return parse_op(text)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream(local)
    torch.cuda.set_stream(stream)  # the ctx, events and collectives all run on this stream
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2411_18873_b200 import capi

    forest_flat = load_forest()
    op = parse_op_text(OP_TEXT)
    ctx = capi.Context(local)
    if world > 1:  # the library's own NCCL communicator (per-shard top-k all-gather)
        uid = [capi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        capi.attach_nccl(ctx, uid[0], world, rank)
    plan = capi.Plan(ctx, op)
    forest = capi.Forest.from_flat(ctx, forest_flat)
    # the SURVEY §8(d) population, bred on the device (bit-exact with the reference's
    # sample_random + reproduce): reproduce(sample_random(op, 1024, 42), n, {}, 7 + rank)
    parents = plan.sample_random(1024, 42)
    g0, _, _ = capi.reproduce(plan, parents, args.pop, 7 + rank)
    sched = plan.decode(g0).cpu().numpy()  # host Schedule[] for the e2e call and the CPU baseline
    ctx.synchronize()
    n = len(sched)
    nb = args.bufs
    genomes = [g0.clone() for _ in range(nb)]
    preds = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nb)]
    ids = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(nb)]
    K = min(args.k, n)
    top = torch.empty(K, dtype=torch.int64, device="cuda")
    top_sc = torch.empty(K, dtype=torch.float64, device="cuda")

    def step(i):
        b = i % nb
        if world > 1:  # fused score + local top-k -> ncclAllGather of (score, global idx) -> identical merge
            forest.score_select_sharded(plan, genomes[b], rank * n, K, preds[b], top, sc=top_sc, ids=ids[b])
        else:  # fused score + top-k (etune_cu_score_select)
            forest.score_select(plan, genomes[b], K, preds[b], top, ids=ids[b])

    # NVML is initialised before the warm-up: its first queries perturb a running GPU
    # (measured: one ~25 % slower timed loop when nvmlInit ran inside it)
    clk = ClockSampler(local)
    clk.sample()
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = capi.lib().etune_cu_launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clk.sm.clear()
    with clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        clk.sample()
        for i in range(args.steps):
            step(args.warmup + i)
        ev1.record(stream)
        clk.sample()
        torch.cuda.synchronize()
    launches = capi.lib().etune_cu_launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    # kernel split: a separate pass with CUDA events around the score kernel and the
    # selection kernels of each call (events serialise the PDL overlap, so the timed
    # loop above runs without them)
    capi.profile_score(ctx, True)
    for i in range(args.steps):
        step(args.warmup + args.steps + i)
    _, score_ms, select_ms, score_calls = capi.profile_score(ctx, False)
    kernel_ms = score_ms / max(score_calls, 1)
    select_ms = select_ms / max(score_calls, 1)
    if world > 1:
        t = torch.tensor([ms, kernel_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kernel_ms = t.tolist()
        dist.barrier()
    value = world * n / (ms / 1e3)

    # ---- e2e through the reference-facing C-ABI call with host buffers
    e2e = None
    if not args.no_e2e:
        h_sched = torch.from_numpy(sched).pin_memory()
        h_pred = torch.empty(n, dtype=torch.float64).pin_memory()
        h_ids = torch.empty(n, dtype=torch.int64).pin_memory()
        hs, hp, hi = h_sched.numpy(), h_pred.numpy(), h_ids.numpy()
        for _ in range(2):
            forest.score_host(plan, hs, hp, hi)
        if world > 1:
            dist.barrier()
        reps = max(3, args.steps // 4)
        t0 = time.perf_counter()
        for _ in range(reps):
            forest.score_host(plan, hs, hp, hi)
        dt = (time.perf_counter() - t0) / reps
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = t.item()
        # score_host narrows each row to the smallest field width holding it (u16 here); with a
        # pinned caller buffer every 4th 2^17-row chunk is copied raw (96 B/row) instead
        fb = 2 if (sched.min() >= 0 and sched.max() < 1 << 16) else 4 if sched.max() < 1 << 32 else 8
        chunk, raw_every = 1 << int(os.environ.get("ETUNE_E2E_CHUNK_LOG2", "17")), \
            int(os.environ.get("ETUNE_E2E_RAW_EVERY", "4"))
        h2d = 0
        for i, lo in enumerate(range(0, n, chunk)):
            m = min(chunk, n - lo)
            raw = raw_every > 0 and i % raw_every == 0 and n > chunk
            h2d += m * 12 * (8 if raw else fb)
        e2e = {"value": world * n / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(n * 16), "ms_per_step": dt * 1e3,
               "api": "etune_cu_score_host (host Schedule[] 96 B/row -> host-pool narrowing into pinned "
                      "staging (every 4th chunk copied raw from the pinned caller buffer) -> H2D -> "
                      "encode+validate -> score -> D2H, chunked 3-stream pipeline)"}

    round_latency = None
    if rank == 0 and world == 1 and not args.no_search:
        round_latency = search_round_latency(ctx, capi, args.search_rounds)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    achieved = n * ALGO_BYTES / (kernel_ms / 1e3) / 1e9
    traffic = None
    sm_bound = None
    try:  # DRAM bytes per launch + the binding SM unit from the committed ncu --set full capture
        t = json.load(open(os.path.join(ROOT, "profiles", "score_kernel_traffic.json")))
        traffic = int(t["dram_bytes_read_per_launch"]) + int(t["dram_bytes_write_per_launch"])
        if "binding_unit" in t:
            sm_bound = {"unit": t["binding_unit"], "pct_of_peak": t["l1tex_pct_of_peak"],
                        "issue_active_pct": t["issue_active_pct"], "source": t["source"]}
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(K), "op": OP_TEXT, "population_per_gpu": n,
                   "implementation": "etune_cu_score_select: keyed score kernel (per candidate one 64-byte row of "
                                     "5-bit exit slots per (tiling triple, Kuv class) from an L2-resident key table, "
                                     "two 256-bit loads; leaf words from shared memory; + ids, + selection histogram) "
                                     "-> bucket filter -> rank selection, PDL-chained",
                   "k": K, "model": "reference-trained 100-tree depth-6 GBDT (tests/golden c2 fixture)",
                   "parallelism": f"dp{world} (population sharded; NCCL all-gather of per-shard top-k records "
                                  f"inside the C ABI)",
                   "l2": f"{nb} distinct population buffers cycled ({nb * n * 24 / 2**20:.0f} MB > 126 MB L2)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": "score_keyed_kernel", "kernel_ms": kernel_ms,
                     "algorithmic_bytes_per_candidate": ALGO_BYTES,
                     "algorithmic_bytes_source": "SURVEY.md §8(d) score mode: 48 B schedule (12 x int32) in + 8 B "
                                                 "prediction + 8 B id out",
                     "design_bytes_per_candidate": DESIGN_BYTES,
                     "design_frac": n * DESIGN_BYTES / (kernel_ms / 1e3) / 1e9 / hbm,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else
                                    "fallback 6650 GB/s (B200_PROFILING.md)",
                     "note": "SM-bound (issue + shared-memory pipe); per-candidate key-table row reads are "
                             "L2-resident, not HBM; see profiles/",
                     "select_ms": select_ms, "sm_bound": sm_bound},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if round_latency:
        line["search_round_latency"] = round_latency
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = time_cpu(op, sched, args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
