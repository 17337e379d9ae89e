"""ctypes binding of libetune_cuda.so (include/etune_cuda.h) for Python callers.

PyTorch is used only as the device-memory / stream plumbing: tensors are passed to
the C ABI as raw device pointers on the current torch stream.  There is no CPU
fallback: if the shared library or an sm_100 device is missing, every call raises.

uint64 payloads (genomes, ids) live in int64 tensors (same bits); use
``as_u64(t)`` to view them as numpy uint64 on the host.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "lib", "libetune_cuda.so")
HEADER = os.path.join(ROOT, "include", "etune_cuda.h")

STATUS_NAMES = {
    0: "OK", 1: "ParseError", 2: "ValidationError", 3: "SpaceExhausted", 4: "IllegalSchedule",
    5: "TooLarge", 6: "NonPositiveEnergy", 7: "InsufficientData", 8: "SchemaMismatch",
    9: "VersionMismatch", 10: "LengthMismatch", 11: "EmptyInput", 12: "IoError",
    13: "ConsistencyError", 14: "BackendUnavailable", 15: "TraceMiss", 64: "InvalidArgument",
    65: "CudaError", 66: "NoDevice", 67: "Unsupported",
}


class EtuneError(RuntimeError):
    """Mirrors etune::Error (errors.hpp:9-12); .code is the etune_status."""

    def __init__(self, code: int, msg: str, index: int = -1):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.index = index


class OpSpec(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("kind", "batch", "m", "n", "k", "height", "width", "in_channels",
                                         "out_channels", "kernel_size", "stride", "padding")]


class SpaceLimits(C.Structure):
    _fields_ = [("max_block_threads", C.c_int64), ("max_unroll", C.c_int64), ("max_vectorize", C.c_int64)]


class DeviceConfig(C.Structure):
    _fields_ = [("num_sms", C.c_int32), ("reserved", C.c_int32)] + [
        (n, C.c_double) for n in (
            "constant_power_w", "static_power_per_sm_w", "dynamic_energy_per_flop_nj",
            "dynamic_energy_per_glb_access_nj", "dynamic_energy_per_shared_access_nj",
            "base_throughput_flops_per_s_per_sm", "mem_bandwidth_elems_per_s", "latency_floor_ms",
            "sampler_hz", "warmup_s", "noise_sigma_rel")] + [("rng_seed", C.c_uint64)]


class GeneticRates(C.Structure):
    _fields_ = [("mutation", C.c_double), ("crossover", C.c_double), ("copy", C.c_double)]


class BoostParams(C.Structure):
    _fields_ = [("num_trees", C.c_int32), ("max_depth", C.c_int32), ("learning_rate", C.c_double),
                ("min_leaf_weight", C.c_double), ("reg_lambda", C.c_double)]


class NvmlParams(C.Structure):
    _fields_ = [("warmup_ms", C.c_double), ("window_ms", C.c_double), ("min_iterations", C.c_int64),
                ("max_iterations", C.c_int64)]


class Measurement(C.Structure):
    _fields_ = [("candidate_id", C.c_uint64), ("latency_ms", C.c_double), ("avg_power_w", C.c_double),
                ("energy_mj", C.c_double), ("iterations", C.c_int64), ("feasible", C.c_int32),
                ("reserved", C.c_int32)]


class SearchConfig(C.Structure):
    _fields_ = [("M", C.c_int64), ("generation_size", C.c_int64), ("k_init_fifths", C.c_int32),
                ("max_rounds", C.c_int32), ("patience", C.c_int32), ("inverted_semantics", C.c_int32),
                ("mu_db", C.c_double), ("improve_rel", C.c_double), ("rng_seed", C.c_uint64),
                ("rates", GeneticRates), ("boost", BoostParams), ("backend", C.c_int32),
                ("latency_reps", C.c_int32), ("nvml", NvmlParams), ("latency_only", C.c_int32),
                ("counter_rng", C.c_int32)]


class RoundReport(C.Structure):
    _fields_ = [("round", C.c_int64), ("k_before_fifths", C.c_int32), ("k_after_fifths", C.c_int32),
                ("snr_db", C.c_double), ("measured", C.c_int64), ("cumulative_measured", C.c_int64),
                ("best_id", C.c_uint64), ("best_latency_ms", C.c_double), ("best_energy_mj", C.c_double),
                ("best_power_w", C.c_double), ("wall_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ModelHost(C.Structure):
    _fields_ = [("num_trees", C.c_int64), ("num_nodes", C.c_int64), ("feature", C.POINTER(C.c_int32)),
                ("threshold", C.POINTER(C.c_double)), ("left", C.POINTER(C.c_int32)),
                ("right", C.POINTER(C.c_int32)), ("value", C.POINTER(C.c_double)),
                ("tree_offsets", C.POINTER(C.c_int64)), ("params", BoostParams), ("base_score", C.c_double),
                ("reference_energy_mj", C.c_double)]


class SamplesHost(C.Structure):
    _fields_ = [("n", C.c_int64), ("features", C.POINTER(C.c_double)),
                ("measured_energy_mj", C.POINTER(C.c_double)), ("normalized_energy", C.POINTER(C.c_double))]


_VP = C.c_void_p
_I64 = C.c_int64
_PTR = C.c_void_p

_ALLGATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
_BROADCAST_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)


class Transport(C.Structure):
    """etune_transport (include/etune_cuda.h): caller-provided collectives."""
    _fields_ = [("user", C.c_void_p), ("nranks", C.c_int32), ("rank", C.c_int32), ("allgather", _ALLGATHER_FN),
                ("broadcast", _BROADCAST_FN)]

_SIGS = {
    "etune_default_device_config": (None, [C.POINTER(DeviceConfig)]),
    "etune_default_space_limits": (None, [C.POINTER(SpaceLimits)]),
    "etune_cu_last_error": (C.c_char_p, []),
    "etune_cu_abi_version": (C.c_int, []),
    "etune_cu_launch_count": (C.c_uint64, []),
    "etune_cu_ctx_create": (C.c_int, [C.c_int, _VP, C.POINTER(_VP)]),
    "etune_cu_ctx_destroy": (C.c_int, [_VP]),
    "etune_cu_ctx_set_stream": (C.c_int, [_VP, _VP]),
    "etune_cu_ctx_stream": (_VP, [_VP]),
    "etune_cu_synchronize": (C.c_int, [_VP, C.POINTER(_I64)]),
    "etune_cu_plan_create": (C.c_int, [_VP, C.POINTER(OpSpec), C.POINTER(DeviceConfig),
                                       C.POINTER(SpaceLimits), C.POINTER(_VP)]),
    "etune_cu_plan_destroy": (C.c_int, [_VP]),
    "etune_cu_plan_nest": (C.c_int, [_VP, _PTR]),
    "etune_cu_plan_space_size": (C.c_int, [_VP, C.POINTER(_I64)]),
    "etune_cu_encode": (C.c_int, [_VP, _VP, _PTR, _I64, _PTR]),
    "etune_cu_decode": (C.c_int, [_VP, _VP, _PTR, _I64, _PTR]),
    "etune_cu_candidate_ids": (C.c_int, [_VP, _VP, _PTR, _I64, _PTR]),
    "etune_cu_counters": (C.c_int, [_VP, _VP, _PTR, _I64, _PTR]),
    "etune_cu_features": (C.c_int, [_VP, _VP, _PTR, _I64, _PTR, _PTR]),
    "etune_cu_forest_create": (C.c_int, [_VP, _PTR, _PTR, _PTR, _PTR, _PTR, _PTR, _I64, C.c_double,
                                         C.c_double, C.POINTER(_VP)]),
    "etune_cu_forest_destroy": (C.c_int, [_VP]),
    "etune_cu_predict": (C.c_int, [_VP, _VP, _PTR, _I64, _PTR]),
    "etune_cu_score": (C.c_int, [_VP, _VP, _VP, _PTR, _I64, _PTR, _PTR]),
    "etune_cu_score_select": (C.c_int, [_VP, _VP, _VP, _PTR, _I64, _I64, _PTR, _PTR, _PTR]),
    "etune_cu_score_select_sharded": (C.c_int, [_VP, _VP, _VP, _PTR, _I64, _I64, _I64, _PTR, _PTR, _PTR, _PTR]),
    "etune_model_to_json": (C.c_int, [_PTR, _PTR, _PTR, _PTR, _PTR, _PTR, _I64, C.POINTER(BoostParams), C.c_double,
                                      C.c_double, C.c_char_p, _I64, C.POINTER(_I64)]),
    "etune_model_from_json": (C.c_int, [C.c_char_p, _I64, C.POINTER(ModelHost)]),
    "etune_model_host_free": (None, [C.POINTER(ModelHost)]),
    "etune_samples_to_jsonl": (C.c_int, [_PTR, _PTR, _PTR, _I64, C.c_char_p, _I64, C.POINTER(_I64)]),
    "etune_samples_from_jsonl": (C.c_int, [C.c_char_p, _I64, C.POINTER(SamplesHost)]),
    "etune_measurement_log_to_jsonl": (C.c_int, [_PTR, _I64, C.c_char_p, _I64, C.POINTER(_I64)]),
    "etune_measurement_log_from_jsonl": (C.c_int, [C.c_char_p, _I64, C.POINTER(_VP), C.POINTER(_I64)]),
    "etune_measurement_log_free": (None, [_VP]),
    "etune_cu_search_set_replay": (C.c_int, [_VP, _PTR, _I64]),
    "etune_samples_host_free": (None, [C.POINTER(SamplesHost)]),
    "etune_device_profile_to_json": (C.c_int, [C.POINTER(DeviceConfig), C.c_char_p, C.c_char_p, _I64,
                                               C.POINTER(_I64)]),
    "etune_device_profile_from_json": (C.c_int, [C.c_char_p, _I64, C.POINTER(DeviceConfig), C.c_char_p, _I64]),
    "etune_cu_profile_score": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.POINTER(_I64)]),
    "etune_cu_forest_set_keyed": (C.c_int, [_VP, C.c_int]),
    "etune_cu_forest_set_form": (C.c_int, [_VP, C.c_int]),
    "etune_cu_forest_compile": (C.c_int, [_VP, _VP, _VP]),
    "etune_cu_forest_rows_info": (C.c_int, [_VP, _VP, _VP, _PTR]),
    "etune_cu_forest_score_form": (C.c_int, [_VP, _VP, C.POINTER(C.c_int)]),
    "etune_cu_score_host": (C.c_int, [_VP, _VP, _VP, _PTR, _I64, _PTR, _PTR, C.POINTER(_I64)]),
    "etune_cu_score_select_host": (C.c_int, [_VP, _VP, _VP, _PTR, _I64, _I64, _PTR, _PTR, C.POINTER(_I64)]),
    "etune_cu_topk": (C.c_int, [_VP, _PTR, _I64, _I64, _PTR]),
    "etune_cu_train": (C.c_int, [_VP, _PTR, _PTR, _I64, C.POINTER(BoostParams), _PTR, _PTR, _PTR, _PTR, _PTR, _PTR,
                                 _PTR, _PTR]),
    "etune_cu_forest_from_device": (C.c_int, [_VP, _PTR, _PTR, _PTR, _PTR, _PTR, _PTR, _I64, _PTR, C.c_double,
                                              C.POINTER(_VP)]),
    "etune_cu_sample_random": (C.c_int, [_VP, _VP, _I64, C.c_uint64, _PTR, _PTR]),
    "etune_cu_sim_measure": (C.c_int, [_VP, _VP, _PTR, _I64, _PTR, _PTR, _PTR, _PTR]),
    "etune_default_nvml_params": (None, [C.POINTER(NvmlParams)]),
    "etune_cu_nvml_available": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "etune_cu_candidate_run": (C.c_int, [_VP, _VP, _PTR, _PTR, _PTR, _PTR]),
    "etune_cu_nvml_measure": (C.c_int, [_VP, _VP, _PTR, _I64, C.POINTER(NvmlParams), _PTR, C.POINTER(_I64)]),
    "etune_cu_energy_loss": (C.c_int, [_VP, _PTR, _PTR, _I64, _PTR]),
    "etune_cu_snr_db": (C.c_int, [_VP, _PTR, _PTR, _I64, C.POINTER(C.c_double), C.POINTER(_I64)]),
    "etune_cu_nccl_unique_id": (C.c_int, [_PTR]),
    "etune_cu_ctx_attach_nccl": (C.c_int, [_VP, _PTR, C.c_int, C.c_int]),
    "etune_cu_topk_sharded": (C.c_int, [_VP, _PTR, _I64, _I64, _I64, _PTR, _PTR]),
    "etune_cu_broadcast": (C.c_int, [_VP, _PTR, _I64, C.c_int]),
    "etune_cu_ctx_attach_transport": (C.c_int, [_VP, C.POINTER(Transport)]),
    "etune_cu_device_alloc": (C.c_int, [_VP, C.POINTER(_VP), _I64]),
    "etune_cu_device_free": (C.c_int, [_VP, _VP]),
    "etune_cu_memcpy_h2d": (C.c_int, [_VP, _PTR, _PTR, _I64]),
    "etune_cu_memcpy_d2h": (C.c_int, [_VP, _PTR, _PTR, _I64]),
    "etune_default_search_config": (None, [C.POINTER(SearchConfig)]),
    "etune_cu_search_create": (C.c_int, [_VP, _VP, C.POINTER(SearchConfig), C.POINTER(_VP)]),
    "etune_cu_search_destroy": (C.c_int, [_VP]),
    "etune_cu_search_initial": (C.c_int, [_VP, C.POINTER(RoundReport)]),
    "etune_cu_search_round": (C.c_int, [_VP, C.POINTER(RoundReport)]),
    "etune_cu_search_run": (C.c_int, [_VP, _PTR, _I64, C.POINTER(_I64)]),
    "etune_cu_search_best": (C.c_int, [_VP, _PTR, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "etune_cu_search_parents": (C.c_int, [_VP, _PTR, _I64, C.POINTER(_I64)]),
    "etune_cu_reproduce": (C.c_int, [_VP, _VP, _PTR, _I64, _I64, C.POINTER(GeneticRates), C.c_uint64, _PTR, _PTR,
                                     _PTR]),
    "etune_cu_reproduce_counter": (C.c_int, [_VP, _VP, _PTR, _I64, _I64, C.POINTER(GeneticRates), C.c_uint64, _PTR,
                                             _PTR, _PTR]),
}

_lib = None


def header_functions() -> list[str]:
    """Every function the public header declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:etune_status|void\*?|const char\*|int|uint64_t)\s+(etune_\w+)\s*\(", txt, re.M)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EtuneError(65, f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        # libetune_cuda.so and torch both need libnccl.so.2; whichever loads first provides
        # it process-wide.  Load torch's (newer) copy first so a later `import torch` still
        # finds every symbol it expects.
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int, index: int = -1):
    if st != 0:
        raise EtuneError(st, lib().etune_cu_last_error().decode(), index)


def op_spec(op) -> OpSpec:
    w = [int(x) for x in np.asarray(op, dtype=np.int64).reshape(12)]
    return OpSpec(*w)


def default_device_config(num_sms: Optional[int] = None, **fields) -> DeviceConfig:
    """DeviceConfig::a100_like() (device.hpp:17-45) with optional field overrides."""
    d = DeviceConfig()
    lib().etune_default_device_config(C.byref(d))
    if num_sms is not None:
        d.num_sms = int(num_sms)
    for k, v in fields.items():
        setattr(d, k, type(getattr(d, k))(v))
    return d


def _ptr(t) -> int:
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def as_u64(t) -> np.ndarray:
    a = t.detach().cpu().numpy() if hasattr(t, "detach") else np.asarray(t)
    return a.view(np.uint64)


class Context:
    """etune_cu_ctx bound to a device and (by default) torch's current stream."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self._torch_stream = stream
        h = C.c_void_p()
        _check(lib().etune_cu_ctx_create(device, C.c_void_p(stream.cuda_stream), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().etune_cu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        bad = C.c_int64(-1)
        st = lib().etune_cu_synchronize(self.h, C.byref(bad))
        _check(st, bad.value)


class Plan:
    def __init__(self, ctx: Context, op, num_sms: int = 108, limits=None, dev: Optional[DeviceConfig] = None):
        self.ctx = ctx
        self.op = np.asarray(op, dtype=np.int64).reshape(12).copy()
        d = dev if dev is not None else default_device_config(num_sms)
        lim = None
        if limits is not None:
            lim = SpaceLimits(*[int(x) for x in limits])
        h = C.c_void_p()
        _check(lib().etune_cu_plan_create(ctx.h, C.byref(op_spec(self.op)), C.byref(d),
                                          C.byref(lim) if lim is not None else None, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().etune_cu_plan_destroy(self.h)
        except Exception:
            pass

    def nest(self):
        out = np.zeros(4, np.int64)
        _check(lib().etune_cu_plan_nest(self.h, out.ctypes.data))
        return out

    def space_size(self) -> int:
        v = C.c_int64()
        _check(lib().etune_cu_plan_space_size(self.h, C.byref(v)))
        return v.value

    # --- codec / features (device tensors in, device tensors out)
    def encode(self, sched):
        import torch
        n = sched.shape[0]
        g = torch.empty(n, dtype=torch.int64, device=sched.device)
        _check(lib().etune_cu_encode(self.ctx.h, self.h, _ptr(sched), n, _ptr(g)))
        return g

    def decode(self, genome):
        import torch
        n = genome.shape[0]
        s = torch.empty((n, 12), dtype=torch.int64, device=genome.device)
        _check(lib().etune_cu_decode(self.ctx.h, self.h, _ptr(genome), n, _ptr(s)))
        return s

    def ids(self, genome):
        import torch
        out = torch.empty_like(genome)
        _check(lib().etune_cu_candidate_ids(self.ctx.h, self.h, _ptr(genome), genome.shape[0], _ptr(out)))
        return out

    def counters(self, genome):
        import torch
        out = torch.empty((genome.shape[0], 10), dtype=torch.int64, device=genome.device)
        _check(lib().etune_cu_counters(self.ctx.h, self.h, _ptr(genome), genome.shape[0], _ptr(out)))
        return out

    def sample_random(self, n: int, seed: int, with_ids: bool = False):
        """sample_random (space.cpp:170-251) on the device -> genomes (+ ids)."""
        import torch
        g = torch.empty(n, dtype=torch.int64, device=torch.device("cuda", self.ctx.device))
        ids = torch.empty_like(g) if with_ids else None
        _check(lib().etune_cu_sample_random(self.ctx.h, self.h, int(n), C.c_uint64(seed), _ptr(g), _ptr(ids)))
        return (g, ids) if with_ids else g

    def sim_measure(self, genome, latency_only: bool = False):
        """SimBackend on device genomes -> (latency_ms, power_w, energy_mj, iterations)."""
        import torch
        n = genome.shape[0]
        lat = torch.empty(n, dtype=torch.float64, device=genome.device)
        if latency_only:
            _check(lib().etune_cu_sim_measure(self.ctx.h, self.h, _ptr(genome), n, _ptr(lat), None, None, None))
            return lat
        pw = torch.empty_like(lat)
        en = torch.empty_like(lat)
        it = torch.empty(n, dtype=torch.int64, device=genome.device)
        _check(lib().etune_cu_sim_measure(self.ctx.h, self.h, _ptr(genome), n, _ptr(lat), _ptr(pw), _ptr(en),
                                          _ptr(it)))
        return lat, pw, en, it

    def features(self, genome, with_ids: bool = False):
        import torch
        n = genome.shape[0]
        f = torch.empty((n, 16), dtype=torch.float64, device=genome.device)
        ids = torch.empty_like(genome) if with_ids else None
        _check(lib().etune_cu_features(self.ctx.h, self.h, _ptr(genome), n, _ptr(f), _ptr(ids)))
        return (f, ids) if with_ids else f


def reproduce(plan: "Plan", parents, n: int, seed: int, rates=(0.85, 0.10, 0.05), counter: bool = False):
    """reproduce (genetic.cpp:137-187) on device genomes -> (offspring genomes, partner idx, ids).
    Offspring i's base parent is i % len(parents); partner[i] = -1 unless a crossover.
    counter=True: the opt-in counter-based RNG mode (etune_cu_reproduce_counter), not the reference's stream."""
    import torch
    dev = parents.device
    out = torch.empty(n, dtype=torch.int64, device=dev)
    partner = torch.empty(n, dtype=torch.int32, device=dev)
    ids = torch.empty(n, dtype=torch.int64, device=dev)
    r = GeneticRates(*[float(x) for x in rates])
    fn = lib().etune_cu_reproduce_counter if counter else lib().etune_cu_reproduce
    _check(fn(plan.ctx.h, plan.h, _ptr(parents), parents.shape[0], n, C.byref(r), C.c_uint64(seed), _ptr(out),
              _ptr(partner), _ptr(ids)))
    return out, partner, ids


class TrainedModel:
    """Device-resident output of etune_cu_train (EnergyModel::train, energy_model.cpp:173-243)."""

    def __init__(self, ctx, nodes, offsets, scalars, loss, num_trees, learning_rate, params):
        self.ctx, self.nodes, self.offsets, self.scalars, self.loss = ctx, nodes, offsets, scalars, loss
        self.num_trees, self.learning_rate, self.params = num_trees, learning_rate, params

    def host(self):
        """(feature, threshold, left, right, value, offsets, base_score, reference_energy, loss) on the host."""
        self.ctx.synchronize()
        off = self.offsets.cpu().numpy()
        nn = int(off[-1])
        fe, th, le, ri, va = (t[:nn].cpu().numpy() for t in self.nodes)
        sc = self.scalars.cpu().numpy()
        loss = self.loss.cpu().numpy() if self.loss is not None else None
        return fe, th, le, ri, va, off, float(sc[0]), float(sc[1]), loss

    def forest(self) -> "Forest":
        fe, th, le, ri, va = self.nodes
        h = C.c_void_p()
        _check(lib().etune_cu_forest_from_device(self.ctx.h, _ptr(fe), _ptr(th), _ptr(le), _ptr(ri), _ptr(va),
                                                 _ptr(self.offsets), self.num_trees, _ptr(self.scalars),
                                                 float(self.learning_rate), C.byref(h)))
        return Forest._wrap(self.ctx, h)


def train(ctx: "Context", feats, energy, num_trees: int = 100, max_depth: int = 6, learning_rate: float = 0.1,
          min_leaf_weight: float = 1e-3, reg_lambda: float = 1.0, with_loss: bool = True) -> TrainedModel:
    import torch
    dev = feats.device
    n = feats.shape[0]
    cap = max(1, num_trees * ((1 << (max_depth + 1)) - 1))
    nodes = (torch.empty(cap, dtype=torch.int32, device=dev), torch.empty(cap, dtype=torch.float64, device=dev),
             torch.empty(cap, dtype=torch.int32, device=dev), torch.empty(cap, dtype=torch.int32, device=dev),
             torch.empty(cap, dtype=torch.float64, device=dev))
    off = torch.zeros(num_trees + 1, dtype=torch.int64, device=dev)
    sc = torch.zeros(2, dtype=torch.float64, device=dev)
    loss = torch.zeros(num_trees + 1, dtype=torch.float64, device=dev) if with_loss else None
    p = BoostParams(int(num_trees), int(max_depth), float(learning_rate), float(min_leaf_weight), float(reg_lambda))
    _check(lib().etune_cu_train(ctx.h, _ptr(feats), _ptr(energy), n, C.byref(p), *[_ptr(t) for t in nodes], _ptr(off),
                                _ptr(sc), _ptr(loss)))
    return TrainedModel(ctx, nodes, off, sc, loss, num_trees, learning_rate, p)


class Forest:
    def __init__(self, ctx: Context, feature, threshold, left, right, value, offsets, base_score: float,
                 learning_rate: float):
        self.ctx = ctx
        self._keep = [np.ascontiguousarray(feature, np.int32), np.ascontiguousarray(threshold, np.float64),
                      np.ascontiguousarray(left, np.int32), np.ascontiguousarray(right, np.int32),
                      np.ascontiguousarray(value, np.float64), np.ascontiguousarray(offsets, np.int64)]
        fe, th, le, ri, va, off = self._keep
        h = C.c_void_p()
        _check(lib().etune_cu_forest_create(ctx.h, fe.ctypes.data, th.ctypes.data, le.ctypes.data, ri.ctypes.data,
                                            va.ctypes.data, off.ctypes.data, len(off) - 1, float(base_score),
                                            float(learning_rate), C.byref(h)))
        self.h = h

    @staticmethod
    def _wrap(ctx: Context, h) -> "Forest":
        f = Forest.__new__(Forest)
        f.ctx, f.h, f._keep = ctx, h, []
        return f

    @staticmethod
    def from_flat(ctx: Context, f) -> "Forest":
        return Forest(ctx, f.feature, f.threshold, f.left, f.right, f.value, f.offsets, f.base_score,
                      f.learning_rate)

    def __del__(self):
        try:
            lib().etune_cu_forest_destroy(self.h)
        except Exception:
            pass

    def predict(self, feats):
        import torch
        n = feats.shape[0]
        out = torch.empty(n, dtype=torch.float64, device=feats.device)
        _check(lib().etune_cu_predict(self.ctx.h, self.h, _ptr(feats), n, _ptr(out)))
        return out

    def score(self, plan: Plan, genome, with_ids: bool = False, out=None, ids_out=None):
        import torch
        n = genome.shape[0]
        pred = out if out is not None else torch.empty(n, dtype=torch.float64, device=genome.device)
        ids = ids_out if ids_out is not None else (torch.empty_like(genome) if with_ids else None)
        _check(lib().etune_cu_score(self.ctx.h, plan.h, self.h, _ptr(genome), n, _ptr(pred), _ptr(ids)))
        return (pred, ids) if (with_ids or ids_out is not None) else pred

    def set_keyed(self, mode):
        """Scoring form for large populations: True/1 keyed (full form when it fits, default),
        2 keyed byte form only, False/0 class-table kernel only."""
        _check(lib().etune_cu_forest_set_keyed(self.h, int(mode)))
        return self

    FORMS = {"auto": 0, "rows": 1, "walk": 2, "class": 3, "keyed": 4, "keyed-byte": 5}

    def set_form(self, form: str):
        """Scoring form (ETUNE_FORM_*): 'auto' (default: device-compiled row table for large
        populations, tree walk for small ones), 'rows', 'walk', 'class', 'keyed', 'keyed-byte'."""
        _check(lib().etune_cu_forest_set_form(self.h, self.FORMS[form]))
        return self

    def compile(self, plan: Plan):
        """Compile for `plan` now (row table: enqueued on the ctx stream, asynchronous)."""
        _check(lib().etune_cu_forest_compile(self.ctx.h, self.h, plan.h))
        return self

    def rows_info(self, plan: Plan) -> dict:
        """Row-table diagnostics (synchronises): keys, Kuv classes, rows, bytes, thresholds on f10/f7/f6,
        legal (k, u, v) triples."""
        out = np.zeros(8, np.int64)
        _check(lib().etune_cu_forest_rows_info(self.ctx.h, self.h, plan.h, out.ctypes.data))
        keys = ("keys", "kuv_classes", "rows", "bytes", "thr_f10", "thr_f7", "thr_f6", "kuv_domain")
        return dict(zip(keys, (int(x) for x in out)))

    def score_form(self, plan: Plan) -> str:
        """Form that scores large populations of `plan`: 'class', 'keyed-byte', 'keyed-full', 'walk' or 'rows'."""
        v = C.c_int(-1)
        _check(lib().etune_cu_forest_score_form(self.h, plan.h, C.byref(v)))
        return ("class", "keyed-byte", "keyed-full", "walk", "rows")[v.value]

    def score_select(self, plan: Plan, genome, k: int, pred, idx, ids=None):
        """Fused score + keep-the-best (etune_cu_score_select) into preallocated tensors."""
        _check(lib().etune_cu_score_select(self.ctx.h, plan.h, self.h, _ptr(genome), genome.shape[0], int(k),
                                           _ptr(pred), _ptr(ids), _ptr(idx)))
        return pred, idx

    def score_select_sharded(self, plan: Plan, genome, global_offset: int, k: int, pred, idx, sc=None, ids=None):
        """Fused score + per-shard keep-the-best + all-gather merge (etune_cu_score_select_sharded)."""
        _check(lib().etune_cu_score_select_sharded(self.ctx.h, plan.h, self.h, _ptr(genome), genome.shape[0],
                                                   int(global_offset), int(k), _ptr(pred), _ptr(ids), _ptr(idx),
                                                   _ptr(sc)))
        return idx, sc

    def score_host(self, plan: Plan, sched: np.ndarray, pred: np.ndarray, ids: Optional[np.ndarray] = None):
        """Reference-facing call on HOST buffers (pinned numpy views recommended)."""
        n = sched.shape[0]
        bad = C.c_int64(-1)
        st = lib().etune_cu_score_host(self.ctx.h, plan.h, self.h, _ptr(sched), n, _ptr(pred), _ptr(ids),
                                       C.byref(bad))
        _check(st, bad.value)

    def score_select_host(self, plan: Plan, sched: np.ndarray, k: int, idx: np.ndarray,
                          pred: Optional[np.ndarray] = None):
        """Score HOST schedules and keep the k best (etune_cu_score_select_host); idx int64[k] out."""
        n = sched.shape[0]
        bad = C.c_int64(-1)
        st = lib().etune_cu_score_select_host(self.ctx.h, plan.h, self.h, _ptr(sched), n, int(k), _ptr(pred),
                                              _ptr(idx), C.byref(bad))
        _check(st, bad.value)
        return idx


def nvml_available(ctx: Context) -> bool:
    v = C.c_int()
    _check(lib().etune_cu_nvml_available(ctx.h, C.byref(v)))
    return bool(v.value)


def candidate_run(plan: "Plan", sched_row: np.ndarray, a, b, c):
    """One run of a schedule's candidate kernel on caller device buffers (fp32)."""
    s = np.ascontiguousarray(sched_row, np.int64).reshape(12)
    _check(lib().etune_cu_candidate_run(plan.ctx.h, plan.h, s.ctypes.data, _ptr(a), _ptr(b), _ptr(c)))


def nvml_measure(plan: "Plan", sched: np.ndarray, warmup_ms=50.0, window_ms=200.0, min_iterations=10,
                 max_iterations=1000000):
    """Measure host schedules with the NVML harness -> structured numpy records."""
    s = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
    n = len(s)
    out = (Measurement * max(n, 1))()
    p = NvmlParams(float(warmup_ms), float(window_ms), int(min_iterations), int(max_iterations))
    bad = C.c_int64(-1)
    st = lib().etune_cu_nvml_measure(plan.ctx.h, plan.h, s.ctypes.data, n, C.byref(p), C.cast(out, C.c_void_p),
                                     C.byref(bad))
    _check(st, bad.value)
    return [{k: getattr(out[i], k) for k, _ in Measurement._fields_} for i in range(n)]


def energy_loss(ctx: Context, pred, meas):
    """energy_loss (Eq. 1) per sample -> (n, 3) {value, gradient, hessian}."""
    import torch
    out = torch.empty((pred.shape[0], 3), dtype=torch.float64, device=pred.device)
    _check(lib().etune_cu_energy_loss(ctx.h, _ptr(pred), _ptr(meas), pred.shape[0], _ptr(out)))
    return out


def snr_db(ctx: Context, pred, meas) -> float:
    out = C.c_double()
    bad = C.c_int64(-1)
    st = lib().etune_cu_snr_db(ctx.h, _ptr(pred), _ptr(meas), pred.shape[0], C.byref(out), C.byref(bad))
    _check(st, bad.value)
    return out.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().etune_cu_nccl_unique_id(buf))
    return buf.raw


def attach_nccl(ctx: Context, unique_id: bytes, nranks: int, rank: int):
    buf = C.create_string_buffer(bytes(unique_id), 128)
    _check(lib().etune_cu_ctx_attach_nccl(ctx.h, buf, int(nranks), int(rank)))


class _CudaBuf:
    """A raw device range as a torch tensor (__cuda_array_interface__), no copy."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _dev_bytes(ptr: int, nbytes: int):
    import torch
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device="cuda")


def attach_torch_transport(ctx: Context, group=None):
    """Route the library's collectives (per-shard top-k all-gather, model broadcast) through
    torch.distributed (any backend -- gloo lets several ranks share one GPU) instead of NCCL.
    The callbacks synchronise the device, stage through host memory and synchronise again."""
    import traceback

    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)

    def allgather(user, d_send, d_recv, nbytes, stream):
        try:
            torch.cuda.synchronize()
            src = _dev_bytes(d_send, nbytes).cpu() if nbytes else torch.empty(0, dtype=torch.uint8)
            outs = [torch.empty(int(nbytes), dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, src, group=group)
            if nbytes:
                _dev_bytes(d_recv, nbytes * world).copy_(torch.cat(outs).cuda())
            torch.cuda.synchronize()
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    def broadcast(user, d_buf, nbytes, root, stream):
        try:
            torch.cuda.synchronize()
            buf = _dev_bytes(d_buf, nbytes)
            host = buf.cpu()
            dist.broadcast(host, src=int(root), group=group)
            buf.copy_(host.cuda())
            torch.cuda.synchronize()
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    t = Transport(None, world, rank, _ALLGATHER_FN(allgather), _BROADCAST_FN(broadcast))
    ctx._transport = t  # the callbacks must outlive the ctx's use of them
    _check(lib().etune_cu_ctx_attach_transport(ctx.h, C.byref(t)))
    return ctx


def topk_sharded(ctx: Context, score, global_offset: int, k: int, idx=None, sc=None):
    """Population-sharded keep-the-best: identical (global idx, score) on every rank."""
    import torch
    idx = idx if idx is not None else torch.empty(k, dtype=torch.int64, device=score.device)
    sc = sc if sc is not None else torch.empty(k, dtype=torch.float64, device=score.device)
    _check(lib().etune_cu_topk_sharded(ctx.h, _ptr(score), score.shape[0], int(global_offset), int(k), _ptr(idx),
                                       _ptr(sc)))
    return idx, sc


def broadcast(ctx: Context, t, root: int = 0):
    _check(lib().etune_cu_broadcast(ctx.h, _ptr(t), t.numel() * t.element_size(), int(root)))
    return t


def search_config(**kw) -> SearchConfig:
    """etune_default_search_config with overrides; rates/boost fields by name."""
    cfg = SearchConfig()
    lib().etune_default_search_config(C.byref(cfg))
    for k, v in kw.items():
        if k in ("warmup_ms", "window_ms", "min_iterations", "max_iterations"):
            setattr(cfg.nvml, k, type(getattr(cfg.nvml, k))(v))
        elif hasattr(cfg.rates, k):
            setattr(cfg.rates, k, float(v))
        elif hasattr(cfg.boost, k):
            setattr(cfg.boost, k, type(getattr(cfg.boost, k))(v))
        else:
            setattr(cfg, k, type(getattr(cfg, k))(v))
    return cfg


class Search:
    """Algorithm 1 on the device (etune_cu_search_*), SimBackend measurements."""

    def __init__(self, plan: "Plan", cfg: SearchConfig):
        self.plan, self.cfg = plan, cfg
        h = C.c_void_p()
        _check(lib().etune_cu_search_create(plan.ctx.h, plan.h, C.byref(cfg), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().etune_cu_search_destroy(self.h)
        except Exception:
            pass

    def set_replay(self, records):
        """ReplayBackend log (backend 2): MEASUREMENT_DTYPE records (or LOG_RECORD_DTYPE)."""
        r = np.asarray(records)
        if r.dtype == LOG_RECORD_DTYPE:
            r = r["m"]
        r = np.ascontiguousarray(r, MEASUREMENT_DTYPE)
        _check(lib().etune_cu_search_set_replay(self.h, r.ctypes.data, len(r)))
        return self

    def initial(self) -> RoundReport:
        r = RoundReport()
        _check(lib().etune_cu_search_initial(self.h, C.byref(r)))
        return r

    def round(self) -> RoundReport:
        r = RoundReport()
        _check(lib().etune_cu_search_round(self.h, C.byref(r)))
        return r

    def run(self):
        cap = int(self.cfg.max_rounds) + 2
        arr = (RoundReport * cap)()
        n = C.c_int64()
        _check(lib().etune_cu_search_run(self.h, C.cast(arr, C.c_void_p), cap, C.byref(n)))
        return [arr[i] for i in range(min(n.value, cap))]

    def best(self):
        s = np.zeros(12, np.int64)
        i, lat, en = C.c_uint64(), C.c_double(), C.c_double()
        _check(lib().etune_cu_search_best(self.h, s.ctypes.data, C.byref(i), C.byref(lat), C.byref(en)))
        return s, i.value, lat.value, en.value

    def parents(self):
        import torch
        n = C.c_int64()
        _check(lib().etune_cu_search_parents(self.h, None, 0, C.byref(n)))
        out = torch.empty(n.value, dtype=torch.int64, device=torch.device("cuda", self.plan.ctx.device))
        _check(lib().etune_cu_search_parents(self.h, _ptr(out), n.value, C.byref(n)))
        return out


def profile_score(ctx: Context, on: bool):
    """(key-sort ms, score-kernel ms, selection ms, calls) recorded inside score_select since
    the last call; then timing on/off."""
    srt = C.c_double()
    ms = C.c_double()
    sel = C.c_double()
    cnt = _I64()
    _check(lib().etune_cu_profile_score(ctx.h, int(bool(on)), C.byref(srt), C.byref(ms), C.byref(sel), C.byref(cnt)))
    return srt.value, ms.value, sel.value, cnt.value


def topk(ctx: Context, score, k: int, out=None):
    import torch
    out = out if out is not None else torch.empty(k, dtype=torch.int64, device=score.device)
    _check(lib().etune_cu_topk(ctx.h, _ptr(score), score.shape[0], k, _ptr(out)))
    return out


# ------------------------------------------------------------------ persistence
def _emit(call) -> str:
    """Two-phase writer call: length query, then the text."""
    n = _I64()
    _check(call(None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(call(buf, n.value + 1, C.byref(n)))
    return buf.raw[:n.value].decode()


def model_to_json(feature, threshold, left, right, value, tree_offsets, params: BoostParams, base_score: float,
                  reference_energy_mj: float) -> str:
    """EnergyModel::to_json (energy_model.cpp:259-284) of host arrays."""
    a = [np.ascontiguousarray(feature, np.int32), np.ascontiguousarray(threshold, np.float64),
         np.ascontiguousarray(left, np.int32), np.ascontiguousarray(right, np.int32),
         np.ascontiguousarray(value, np.float64), np.ascontiguousarray(tree_offsets, np.int64)]
    nt = len(a[5]) - 1
    return _emit(lambda out, cap, n: lib().etune_model_to_json(*[x.ctypes.data for x in a], nt, C.byref(params),
                                                               float(base_score), float(reference_energy_mj),
                                                               out, cap, n))


def model_from_json(text: str) -> dict:
    """EnergyModel::from_json (energy_model.cpp:286-336) -> flat host arrays + scalars."""
    b = text.encode()
    m = ModelHost()
    _check(lib().etune_model_from_json(b, len(b), C.byref(m)))
    try:
        nn, nt = m.num_nodes, m.num_trees

        def arr(ptr, k, dt):
            return np.ctypeslib.as_array(ptr, shape=(k,)).astype(dt, copy=True) if k else np.zeros(0, dt)
        out = {"feature": arr(m.feature, nn, np.int32), "threshold": arr(m.threshold, nn, np.float64),
               "left": arr(m.left, nn, np.int32), "right": arr(m.right, nn, np.int32),
               "value": arr(m.value, nn, np.float64), "tree_offsets": arr(m.tree_offsets, nt + 1, np.int64),
               "params": BoostParams(m.params.num_trees, m.params.max_depth, m.params.learning_rate,
                                     m.params.min_leaf_weight, m.params.reg_lambda),
               "base_score": m.base_score, "reference_energy_mj": m.reference_energy_mj}
    finally:
        lib().etune_model_host_free(C.byref(m))
    return out


def samples_to_jsonl(features, measured, normalized) -> str:
    """save_energy_samples (energy_model.cpp:372-383) as text."""
    f = np.ascontiguousarray(features, np.float64).reshape(-1, 16)
    m = np.ascontiguousarray(measured, np.float64)
    z = np.ascontiguousarray(normalized, np.float64)
    return _emit(lambda out, cap, n: lib().etune_samples_to_jsonl(f.ctypes.data, m.ctypes.data, z.ctypes.data,
                                                                  len(m), out, cap, n))


def samples_from_jsonl(text: str):
    """load_energy_samples (energy_model.cpp:385-420) -> (features n x 16, measured, normalized)."""
    b = text.encode()
    s = SamplesHost()
    _check(lib().etune_samples_from_jsonl(b, len(b), C.byref(s)))
    try:
        n = s.n
        if n == 0:
            return np.zeros((0, 16)), np.zeros(0), np.zeros(0)
        return (np.ctypeslib.as_array(s.features, shape=(n * 16,)).reshape(n, 16).copy(),
                np.ctypeslib.as_array(s.measured_energy_mj, shape=(n,)).copy(),
                np.ctypeslib.as_array(s.normalized_energy, shape=(n,)).copy())
    finally:
        lib().etune_samples_host_free(C.byref(s))


# etune_measurement (MeasurementRecord) and etune_log_record (one MeasurementLog line)
MEASUREMENT_DTYPE = np.dtype([("candidate_id", "<u8"), ("latency_ms", "<f8"), ("avg_power_w", "<f8"),
                              ("energy_mj", "<f8"), ("iterations", "<i8"), ("feasible", "<i4"), ("reserved", "<i4")])
LOG_RECORD_DTYPE = np.dtype([("m", MEASUREMENT_DTYPE), ("backend", "S16"), ("timestamp", "S32")])


def measurement_log_to_jsonl(records) -> str:
    """log_append text of LOG_RECORD_DTYPE records (measure.hpp:76-77)."""
    r = np.ascontiguousarray(records, LOG_RECORD_DTYPE)
    return _emit(lambda out, cap, n: lib().etune_measurement_log_to_jsonl(r.ctypes.data, len(r), out, cap, n))


def measurement_log_from_jsonl(text: str):
    """log_load (measure.hpp:79-83): LOG_RECORD_DTYPE records; ConsistencyError (13) names the line."""
    b = text.encode()
    p, n = C.c_void_p(), C.c_int64()
    _check(lib().etune_measurement_log_from_jsonl(b, len(b), C.byref(p), C.byref(n)))
    try:
        if n.value == 0:
            return np.zeros(0, LOG_RECORD_DTYPE)
        buf = (C.c_char * (n.value * LOG_RECORD_DTYPE.itemsize)).from_address(p.value)
        return np.frombuffer(bytes(buf), LOG_RECORD_DTYPE).copy()
    finally:
        lib().etune_measurement_log_free(p)


def device_profile_to_json(dev: DeviceConfig, name: str = "a100-like") -> str:
    """device_profile_to_json (device.cpp:44-62)."""
    nm = name.encode()
    return _emit(lambda out, cap, n: lib().etune_device_profile_to_json(C.byref(dev), nm, out, cap, n))


def device_profile_from_json(text: str):
    """device_profile_from_json (device.cpp:64-101) -> (DeviceConfig, name)."""
    b = text.encode()
    d = DeviceConfig()
    name = C.create_string_buffer(4096)
    _check(lib().etune_device_profile_from_json(b, len(b), C.byref(d), name, 4096))
    return d, name.value.decode()
