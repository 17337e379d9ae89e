"""Benchmark: candidate schedules scored/sec and search-round latency (BASELINE.json metric).

Step = one pass of the hot path over one batch: score the rank's population shard with the
energy cost model (features -> 100-tree GBDT -> prediction + candidate id) and keep the best,
top-k by (prediction, index); for N>1 the per-shard top-k records are all-gathered over NCCL
and merged identically on every rank.

    python bench.py [--gpus N --steps K --warmup W]            # our B200 path
    python bench.py --impl reference [--gpus N ...]            # the reference's CPU path
    torchrun --nproc-per-node N bench.py --gpus N ...          # N>1

Workload (config.workload): the ResNet-50 3x3 conv layer of BASELINE configs[1]
(conv:1,56,56,64,64,3,1,1), population 2^20 per GPU (north_star / configs[3] top size), bred
exactly like SURVEY §8(d): reproduce(sample_random(op,1024,42), 2^20, GeneticRates{}, seed 7 +
rank); model = the reference-trained 100-tree forest on sample_random(op,2048,1234)
(tests/golden fixture).  L2: 16 distinct population buffers (384 MB incl. outputs) are cycled
so no step reads another's data from the 126 MB L2.

The JSON line also carries:
  fresh_model   the same step with a model the library has never seen: forest created from the
                host arrays, compiled on the device (row table), scored + selected, destroyed
  sweep         configs[3]: populations 2^14 .. 2^20, frozen and fresh-model steps
  e2e           the reference-facing call on HOST Schedule rows (pageable, like the reference's
                std::vector<Candidate>), H2D/D2H inside the timed region: etune_cu_score_select_host
                (predictions + top-k back); the pinned-buffer figure beside it
  search_round_latency   Algorithm 1 rounds of BASELINE configs[1] on the device, with the
                reference's own single-threaded train + reproduce + predict of one such round
                timed on the host beside it (cpu_round)
  roofline      the step kernel (score_select_rows_kernel) against the measured HBM peak
  cpu_baseline  the reference's CPU path (oracle/_ref, unmodified sources) on all host threads:
                extract_features + predict + the k best by (prediction, index) via partial_sort
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

# the harness's own CPU threads (torch / numpy OpenMP pools) must not spin-wait on the host cores
# the library's host pool narrows rows on during the e2e leg
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

OP_TEXT = "conv:1,56,56,64,64,3,1,1"
MODEL_KEY = "c2_r50_conv3x3"
METRIC = "candidate schedules scored/sec"
UNIT = "candidates/s"
# algorithmic bytes per candidate, score mode: 48 B schedule in (12 x int32 SoA) + 8 B f64
# prediction + 8 B u64 id out.  This design's population is an 8-byte genome, so the kernel itself must move
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
    p.add_argument("--no-sweep", action="store_true")
    p.add_argument("--no-search", action="store_true", help="skip the search-round latency measurement")
    p.add_argument("--search-rounds", type=int, default=5)
    p.add_argument("--no-reproduce", action="store_true", help="skip the reproduce (2^20 offspring) timing")
    p.add_argument("--no-graph", action="store_true", help="time the eager launch loop only (no CUDA graph replay)")
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


def cpu_select_runner(k: int):
    """Returns (kind, fn(op, sched) -> (preds, top-k idx), threads): the reference's scoring + keep-the-best
    on every host thread.  Prefers the unmodified reference (oracle/_ref) over the restatement (oracle/lib)."""
    from etune_testlib import Oracle, RefLib, have_ref
    forest = load_forest()
    threads = cpu_threads()
    if have_ref():
        R = RefLib()
        model = R.model_from_json(forest_json(forest))
        return "reference", (lambda op, s: model.score_select_threads(op, s, threads, min(k, len(s)))), threads
    O = Oracle()

    def port(op, s):
        p = O.score_threads(op, s, forest, threads)
        kk = min(k, len(p))
        part = np.argpartition(p, kk - 1)[:kk] if kk < len(p) else np.arange(len(p))
        return p, part[np.lexsort((part, p[part]))]
    return "port", port, threads


def time_cpu(op, sched, target_s: float, k: int):
    """Bounded CPU sample: whole passes over (a prefix of) the population until ~target_s of work."""
    kind, fn, threads = cpu_select_runner(k)
    m = min(len(sched), 20000)
    t0 = time.perf_counter()
    fn(op, sched[:m])
    rate = m / max(time.perf_counter() - t0, 1e-9)
    per = int(min(len(sched), max(m, rate * target_s / 4)))
    done, dt = 0, 0.0
    while dt < target_s:
        t0 = time.perf_counter()
        fn(op, sched[:per])
        dt += time.perf_counter() - t0
        done += per
    return {"value": done / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{done} candidates in passes of {per} over the bench population ({OP_TEXT}): the reference's "
                      f"extract_features + EnergyModel::predict per candidate and the {k} best by (prediction, index) "
                      f"(per-thread std::partial_sort + merge) over {threads} std::threads; {dt:.1f} s"}


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML during the timed region
    (a background thread every 1 ms, plus explicit samples at its start and end)."""

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
        while not self.stop.wait(0.001):
            self.sample()

    def __enter__(self):
        self.stop.clear()
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
    kind, fn, threads = cpu_select_runner(args.k)
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
        fn(op, sched[lo:lo + per_step])
        times.append(time.perf_counter() - t0)
    value = per_step * len(times) / sum(times)
    sample = (f"{per_step} candidates/step of the bench population ({OP_TEXT}): the reference's "
              f"extract_features + EnergyModel::predict and the {args.k} best by (prediction, index) "
              f"(std::partial_sort per thread + merge) over {threads} threads")
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


def cpu_round_baseline(rounds_info):
    """The reference's own work of one search round (train and reproduce timed
    single-threaded), at the sample count of the median GPU round: EnergyModel::train on that
    many SimBackend samples (energies from the oracle's SPEC:317 formula), reproduce(2048 parents
    -> 16384), extract_features + predict of the 4096 kept + keep-the-best.  oracle/_ref only."""
    from etune_testlib import Oracle, RefLib, have_ref, parse_op
    if not have_ref():
        return None
    R, O = RefLib(), Oracle()
    op = parse_op(OP_TEXT)
    n_train = int(rounds_info.get("median_samples") or 8192)
    s, _ = O.sample_random(op, n_train, 1234)
    f = O.features(op, s)
    en = O.sim_measure(op, s)[:, 2]
    t0 = time.perf_counter()
    model = R.train(f, en, num_trees=100, max_depth=6)
    t_train = time.perf_counter() - t0
    par = s[:2048]
    t0 = time.perf_counter()
    kids = R.reproduce(op, par, 16384, 43)[0]
    t_repro = time.perf_counter() - t0
    t0 = time.perf_counter()
    model.score_select_threads(op, kids[:4096], 1, 2048)
    t_pred = time.perf_counter() - t0
    total = t_train + t_repro + t_pred
    return {"value": total * 1e3, "unit": "ms", "cores": 1, "kind": "reference",
            "train_ms": t_train * 1e3, "reproduce_ms": t_repro * 1e3, "predict_select_ms": t_pred * 1e3,
            "sample": f"EnergyModel::train on {n_train} SimBackend samples (the median GPU round's sample count), "
                      f"reproduce(2048 parents -> 16384), extract_features + predict + top-2048 of 4096; "
                      f"one thread (the reference is single-threaded); latency filter and measurement excluded"}


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
    reps = [s.round() for _ in range(rounds)]
    ms = [r.wall_ms for r in reps]
    samples = sorted(int(r.cumulative_measured) for r in reps)
    return {"value": statistics.median(ms), "unit": "ms", "rounds": rounds, "per_round_ms": [round(x, 3) for x in ms],
            "initial_round_ms": round(init.wall_ms, 3), "median_samples": samples[len(samples) // 2],
            "config": "conv:1,56,56,64,64,3,1,1 generation 16384, M 4096, k from 1.0, mu 20 dB, SimBackend, "
                      "100-tree retrain on all accumulated samples every round"}


def reproduce_timing(ctx, capi, plan, parents, n: int, with_cpu: bool):
    """reproduce (genetic.cpp:137-187) of an n-offspring generation from the bench's 1024 parents:
    the exact mode (the reference's one mt19937_64 stream, block-parallel), the same call on the
    single-CTA chain, the opt-in counter mode; device time with CUDA events on the ctx stream,
    median of 3 after one warm-up.  Beside it the reference's own reproduce (oracle/_ref,
    single-threaded, as the reference runs) on a 2^17 sample of the same generation."""
    import torch

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        out = []
        for r in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return statistics.median(out)

    res = {"offspring": n, "parents": int(parents.shape[0]), "unit": "ms"}
    res["exact_ms"] = timed(lambda: capi.reproduce(plan, parents, n, 7))
    res["counter_ms"] = timed(lambda: capi.reproduce(plan, parents, n, 7, counter=True))
    os.environ["ETUNE_BREED_PAR_MIN"] = str(1 << 62)
    try:
        res["single_cta_exact_ms"] = timed(lambda: capi.reproduce(plan, parents, n, 7), reps=1)
    finally:
        del os.environ["ETUNE_BREED_PAR_MIN"]
    res["exact_offspring_per_s"] = n / (res["exact_ms"] / 1e3)
    if with_cpu:
        try:
            from etune_testlib import RefLib, have_ref
            if have_ref():
                import numpy as np
                par = plan.decode(parents).cpu().numpy().astype(np.int64)
                m = 1 << 17
                t0 = time.perf_counter()
                RefLib().reproduce(parse_op_text(OP_TEXT), par, m, 7)
                dt = time.perf_counter() - t0
                res["cpu_reference"] = {"offspring_per_s": m / dt, "cores": 1, "kind": "reference",
                                        "projected_ms": n / (m / dt) * 1e3,
                                        "sample": f"etune::reproduce(1024 parents -> {m}) of oracle/_ref, one thread"}
        except Exception as e:  # reported, never required
            res["cpu_reference"] = {"unavailable": str(e)[:200]}
    res["what"] = ("exact: block-parallel resolution of the reference's single RNG stream (breed_par.cu), "
                   "bit-exact; single_cta_exact: the same children on round 1's one-CTA chain; counter: the opt-in "
                   "per-offspring counter-based stream (not the reference's)")
    return res


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

    def step(fo, i, m=n):
        b = i % nb
        g = genomes[b] if m == n else genomes[b][:m]
        kk = min(K, m)
        if world > 1:  # fused score + local top-k -> ncclAllGather of (score, global idx) -> identical merge
            fo.score_select_sharded(plan, g, rank * m, kk, preds[b], top, sc=top_sc, ids=ids[b])
        else:  # fused score + top-k (etune_cu_score_select)
            fo.score_select(plan, g, kk, preds[b], top, ids=ids[b])

    # compile the row table of the bench model (timed: device events around the asynchronous compile)
    e_c0, e_c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_c0.record(stream)
    forest.compile(plan)
    e_c1.record(stream)
    torch.cuda.synchronize()
    compile_ms = e_c0.elapsed_time(e_c1)

    # NVML is initialised before the warm-up: its first queries perturb a running GPU
    clk = ClockSampler(local)
    clk.sample()
    for i in range(args.warmup):
        step(forest, i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # The K timed steps are captured once into a CUDA graph (the library launches on the ctx stream,
    # which is the capture stream) and replayed: back-to-back launches of a 148-CTA cooperative kernel
    # cost ~2 us less per launch from a graph than from the stream (scripts/micro/step_floor.cu).  The
    # eager launch loop is timed as well (eager_ms_per_step).  N > 1 (NCCL inside the step) stays eager.
    use_graph = world == 1 and not args.no_graph
    graph = None
    launches0 = capi.lib().etune_cu_launch_count()
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(args.steps):
                step(forest, args.warmup + i)
        launches = capi.lib().etune_cu_launch_count() - launches0  # our kernels in the graph (one per step)
        graph.replay()  # untimed: the graph's first launch uploads it
        torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def timed_loop():
        clk.sm.clear()
        with clk:
            torch.cuda.synchronize()
            ev0.record(stream)
            clk.sample()
            if graph is not None:
                graph.replay()
            else:
                for i in range(args.steps):
                    step(forest, args.warmup + i)
            ev1.record(stream)
            clk.sample()
            torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / args.steps

    if world > 1:
        dist.barrier()
    ms = timed_loop()
    clocks = clk.summary()
    if graph is None:
        launches = capi.lib().etune_cu_launch_count() - launches0
        eager_ms = ms
    else:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            step(forest, args.warmup + i)
        e1.record(stream)
        torch.cuda.synchronize()
        eager_ms = e0.elapsed_time(e1) / args.steps
    # kernel duration: CUDA events around the step kernel of each call (a separate pass: the events
    # separate the launches the timed loop runs back to back)
    capi.profile_score(ctx, True)
    for i in range(args.steps):
        step(forest, args.warmup + args.steps + i)
    _, score_ms, select_ms, score_calls = capi.profile_score(ctx, False)
    event_kernel_ms = score_ms / max(score_calls, 1)
    select_ms = select_ms / max(score_calls, 1)
    # the roofline's per-launch duration: the graph-replayed step is this one kernel back to back
    kernel_ms = ms if graph is not None else event_kernel_ms
    if world > 1:
        t = torch.tensor([ms, kernel_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kernel_ms = t.tolist()
        dist.barrier()
    value = world * n / (ms / 1e3)

    # ---- score only (SURVEY §8(d) "scored" = features -> prediction, no keep-the-best): etune_cu_score on the
    # row table, the same population and outputs, from a CUDA graph like the step
    score_only = None
    if world == 1:
        def sstep(i):
            b = i % nb
            forest.score(plan, genomes[b], out=preds[b], ids_out=ids[b])

        for i in range(3):
            sstep(i)
        torch.cuda.synchronize()
        sg2 = None
        if use_graph:
            sg2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(sg2, stream=stream):
                for i in range(args.steps):
                    sstep(i)
            sg2.replay()
            torch.cuda.synchronize()
        se0, se1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        se0.record(stream)
        if sg2 is not None:
            sg2.replay()
        else:
            for i in range(args.steps):
                sstep(i)
        se1.record(stream)
        torch.cuda.synchronize()
        sms = se0.elapsed_time(se1) / args.steps
        del sg2
        score_only = {"value": n / (sms / 1e3), "unit": UNIT, "ms_per_step": sms,
                      "what": "etune_cu_score (row table: genome -> prediction + candidate_id, no selection) over the "
                              "bench population, the K steps from a CUDA graph",
                      "roofline": {"bound": "hbm", "achieved": n * ALGO_BYTES / (sms / 1e3) / 1e9, "unit": "GB/s",
                                   "algorithmic_bytes_per_candidate": ALGO_BYTES,
                                   "design_bytes_per_candidate": 24,
                                   "design_achieved": n * 24 / (sms / 1e3) / 1e9,
                                   "note": "SURVEY's 64 B count the 48-byte schedule the row-table path never reads "
                                           "(it reads the 8-byte genome), so frac can reach 1; design_frac is the "
                                           "HBM utilisation on the 24 B it moves (8 B in, 16 B out)"}}

    # ---- feature mode: etune_cu_features, genome -> 16 f64 features + id; HBM-bound
    feature_mode = None
    if world == 1:
        fb = min(nb, 4)
        fbufs = [torch.empty((n, 16), dtype=torch.float64, device="cuda") for _ in range(fb)]

        def fstep(i):
            b = i % fb
            capi._check(capi.lib().etune_cu_features(ctx.h, plan.h, capi._ptr(genomes[i % nb]), n,
                                                     capi._ptr(fbufs[b]), capi._ptr(ids[i % nb])))

        for i in range(3):
            fstep(i)
        torch.cuda.synchronize()
        fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fe0.record(stream)
        for i in range(args.steps):
            fstep(i)
        fe1.record(stream)
        torch.cuda.synchronize()
        fms = fe0.elapsed_time(fe1) / args.steps
        del fbufs
        feature_mode = {
            "value": n / (fms / 1e3), "unit": UNIT, "ms_per_step": fms,
            "what": "etune_cu_features over the bench population: the 16 f64 features of features_from_counters "
                    "(features.cpp:15-51, bit-exact) + candidate_id per candidate, eager launches, "
                    f"{min(nb, 4)} output buffers cycled ({min(nb, 4) * n * 128 / 2**20:.0f} MB)",
            "roofline": {"bound": "hbm", "achieved": n * 192 / (fms / 1e3) / 1e9, "peak": None, "unit": "GB/s",
                         "algorithmic_bytes_per_candidate": 192,
                         "algorithmic_bytes_source": "SURVEY.md §8(d) feature mode: 48 B schedule in + 8 B "
                                                     "prediction + 8 B id + 128 B features",
                         "design_bytes_per_candidate": 144,
                         "design_achieved": n * 144 / (fms / 1e3) / 1e9,
                         "note": "design bytes: 8 B genome in, 128 B features + 8 B id out"},
        }

    # ---- fresh model: every step a model the library has not seen (created from the host arrays,
    # compiled on the device, scored + selected, destroyed); host wall clock around synchronised steps
    def fresh_steps(m, reps):
        walls = []
        for i in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fo = capi.Forest.from_flat(ctx, forest_flat)
            step(fo, i, m)
            del fo
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        return statistics.median(walls[1:] if len(walls) > 2 else walls)

    fresh_s = fresh_steps(n, 12)
    if world > 1:
        t = torch.tensor([fresh_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        fresh_s = t.item()
    fresh = {"value": world * n / fresh_s, "unit": UNIT, "ms_per_step": fresh_s * 1e3, "compile_ms": compile_ms,
             "what": "per step: etune_cu_forest_create from the host arrays (H2D of the nodes), the device compile "
                     "(Kuv classes, row predictions, rows in prediction order), score_select, destroy; host wall "
                     "clock around a synchronised step, median of 11"}

    # ---- configs[3] sweep 2^14 .. 2^20 (frozen and fresh model)
    sweep = []
    if not args.no_sweep and world == 1:
        for lg in range(14, 21):
            m = 1 << lg
            if m > n:
                break
            reps = 50
            for i in range(3):
                step(forest, i, m)
            torch.cuda.synchronize()
            sg = None
            if use_graph:
                sg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(sg, stream=stream):
                    for i in range(reps):
                        step(forest, i, m)
                sg.replay()
                torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            if sg is not None:
                sg.replay()
            else:
                for i in range(reps):
                    step(forest, i, m)
            a1.record(stream)
            torch.cuda.synchronize()
            fm = a0.elapsed_time(a1) / reps
            del sg
            fs = fresh_steps(m, 6)
            sweep.append({"population": m, "frozen_ms": fm, "frozen_value": m / (fm / 1e3),
                          "fresh_ms": fs * 1e3, "fresh_value": m / fs})

    # ---- e2e through the reference-facing C-ABI call with HOST buffers
    e2e = None
    if not args.no_e2e:
        h_pred = np.zeros(n)
        h_idx = np.zeros(K, np.int64)
        pageable = np.ascontiguousarray(sched)
        pinned = torch.from_numpy(sched).pin_memory().numpy()

        def e2e_time(hs, reps):
            for _ in range(2):
                forest.score_select_host(plan, hs, K, h_idx, h_pred)
            if world > 1:
                dist.barrier()
            calls = []  # each call is synchronous (host results back): median of the per-call walls
            for _ in range(reps):
                t0 = time.perf_counter()
                forest.score_select_host(plan, hs, K, h_idx, h_pred)
                calls.append(time.perf_counter() - t0)
            dt = statistics.median(calls)
            if world > 1:
                t = torch.tensor([dt], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = t.item()
            return dt

        def h2d_bytes(pinned_rows):
            # the host pool narrows each chunk (2^17 rows) to the smallest field width holding it (u16 here);
            # with a pinned caller buffer every 4th chunk is copied raw (96 B/row) instead
            fb = 2 if (sched.min() >= 0 and sched.max() < 1 << 16) else 4 if sched.max() < 1 << 32 else 8
            chunk, raw_every = 1 << int(os.environ.get("ETUNE_E2E_CHUNK_LOG2", "17")), \
                int(os.environ.get("ETUNE_E2E_RAW_EVERY", "4"))
            tot, lo, i = 0, 0, 0
            while lo < n:  # the library's chunk schedule: full chunks, the final one a quarter chunk
                rem, q = n - lo, chunk // 4
                mm = rem if rem <= q else rem - q if rem <= chunk + q else chunk
                raw = pinned_rows and raw_every > 0 and i % raw_every == 0 and mm == chunk
                tot += mm * 12 * (8 if raw else fb)
                lo, i = lo + mm, i + 1
            return tot

        reps = max(5, args.steps // 4)
        dt_pg = e2e_time(pageable, reps)
        dt_pin = e2e_time(pinned, reps)
        e2e = {"value": world * n / dt_pg, "unit": UNIT, "h2d_bytes_per_step": int(h2d_bytes(False)),
               "d2h_bytes_per_step": int(n * 8 + K * 8), "ms_per_step": dt_pg * 1e3, "input": "pageable",
               "timing": f"host wall of each synchronous call (results back in host memory), median of {reps}",
               "pinned": {"value": world * n / dt_pin, "ms_per_step": dt_pin * 1e3,
                          "h2d_bytes_per_step": int(h2d_bytes(True))},
               "api": f"etune_cu_score_select_host (host Schedule[] 96 B/row -> host-pool narrowing into pinned "
                      f"staging -> H2D -> encode+validate -> score -> predictions D2H; top-{K} by (prediction, "
                      f"index) on the device -> indices D2H; chunked 3-stream pipeline)"}

    round_latency = None
    cpu_round = None
    if not args.no_search:
        # N>1: the population-sharded search (per-shard latency filter + merge, measurements split
        # over the ranks, training on rank 0 + model broadcast, all over the ctx's NCCL communicator)
        round_latency = search_round_latency(ctx, capi, args.search_rounds)
        if world > 1:
            t = torch.tensor([round_latency["value"]], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            round_latency["value"] = t.item()
            round_latency["sharded_over_ranks"] = world
    repro = None
    if rank == 0 and not args.no_reproduce:
        repro = reproduce_timing(ctx, capi, plan, parents, 1 << 20, with_cpu=(world == 1 and not args.no_cpu_baseline))
    if rank == 0 and world == 1 and not args.no_search:
        if not args.no_cpu_baseline:
            try:
                cpu_round = cpu_round_baseline(round_latency)
            except Exception as e:  # the baseline is reported, never required
                cpu_round = {"unavailable": str(e)[:200]}

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
    try:  # DRAM bytes per launch from the committed ncu --set full capture
        t = json.load(open(os.path.join(ROOT, "profiles", "score_kernel_traffic.json")))
        traffic = int(t["dram_bytes_read_per_launch"]) + int(t["dram_bytes_write_per_launch"])
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(K), "op": OP_TEXT, "population_per_gpu": n,
                   "implementation": "etune_cu_score_select on the device-compiled row table: ONE cooperative "
                                     "kernel per step (genome -> (tiling-triple key, Kuv class) row -> prediction "
                                     "+ id, per-row candidate counts; k-th prediction from the rows in prediction "
                                     "order; ties by index; k sorted)",
                   "k": K, "model": "reference-trained 100-tree depth-6 GBDT (tests/golden c2 fixture), frozen "
                                    "(compiled once; fresh_model times a new model every step)",
                   "parallelism": f"dp{world} (population sharded; NCCL all-gather of per-shard top-k records "
                                  f"inside the C ABI)",
                   "l2": f"{nb} distinct population buffers cycled ({nb * n * 24 / 2**20:.0f} MB > 126 MB L2)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": "score_select_rows_kernel", "kernel_ms": kernel_ms,
                     "algorithmic_bytes_per_candidate": ALGO_BYTES,
                     "algorithmic_bytes_source": "SURVEY.md §8(d) score mode: 48 B schedule (12 x int32) in + 8 B "
                                                 "prediction + 8 B id out",
                     "design_bytes_per_candidate": DESIGN_BYTES,
                     "design_frac": n * DESIGN_BYTES / (kernel_ms / 1e3) / 1e9 / hbm,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else
                                    "fallback 6650 GB/s (B200_PROFILING.md)",
                     "note": "the step is this one kernel (score + select fused); design_frac is the HBM utilisation "
                             "on the bytes it must move (8 B genome in, 8 B prediction + 8 B id out); row-table "
                             "gathers and per-row counters are L2 traffic; see profiles/",
                     "select_ms": select_ms, "event_kernel_ms": event_kernel_ms,
                     "kernel_ms_source": "CUDA-graph replay of the K timed steps (one kernel per step, back to "
                                         "back) / K" if graph is not None else "CUDA events around each launch"},
        "compile_ms": compile_ms,
        "fresh_model": fresh,
        "gpu_launches": int(launches),
        "launch": "CUDA graph of the K steps (captured on the ctx stream, replayed once)" if graph is not None
                  else "eager stream launches",
        "eager_ms_per_step": eager_ms,
        "clocks": clocks,
    }
    if score_only:
        score_only["roofline"]["peak"] = hbm
        score_only["roofline"]["frac"] = score_only["roofline"]["achieved"] / hbm
        score_only["roofline"]["design_frac"] = score_only["roofline"]["design_achieved"] / hbm
        line["score_only"] = score_only
    if feature_mode:
        fr = feature_mode["roofline"]
        fr["peak"] = hbm
        fr["frac"] = fr["achieved"] / hbm
        fr["design_frac"] = fr["design_achieved"] / hbm
        line["feature_mode"] = feature_mode
    if sweep:
        line["sweep"] = sweep
    if e2e:
        line["e2e"] = e2e
    if repro:
        line["reproduce"] = repro
    if round_latency:
        line["search_round_latency"] = round_latency
        if cpu_round:
            line["search_round_latency"]["cpu_round"] = cpu_round
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = time_cpu(op, sched, args.cpu_seconds, K)
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
