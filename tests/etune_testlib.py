"""ctypes wrappers for the TEST-ONLY CPU libraries.

* ``Oracle``  -> oracle/lib/liboracle.so  (the CPU restatement, oracle/etune_oracle.cpp)
* ``RefLib``  -> oracle/_ref/libetune_ref.so (the unmodified reference + oracle/ref_shim.cpp)

Both share the array encodings documented in oracle/etune_oracle.h.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu-baseline / reference legs use this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "lib", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libetune_ref.so")

I64P = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
U64P = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
I8P = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
U8P = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")

# ------------------------------------------------------------------ encodings
MM, MV, CONV = 0, 1, 2


def parse_op(text: str) -> np.ndarray:
    """'mm:1,512,512,512' -> int64[12] exactly as etune::parse_operator builds it
    (opspec.cpp:169-202; unset fields keep OperatorSpec defaults, opspec.hpp:30-47)."""
    head, dims = text.split(":")
    d = [int(x) for x in dims.split(",")]
    op = np.array([0, 1, 1, 1, 1, 0, 0, 0, 0, 0, 1, 0], dtype=np.int64)
    if head == "mm":
        op[0] = MM
        op[1:5] = d
    elif head == "mv":
        op[0] = MV
        op[1], op[2], op[3], op[4] = d[0], 1, d[2], d[3]
    elif head == "conv":
        op[0] = CONV
        op[1] = d[0]
        op[5:12] = d[1:8]
    else:
        raise ValueError(head)
    return op


def default_limits() -> np.ndarray:
    return np.array([1024, 8, 4], dtype=np.int64)


# DeviceConfig::a100_like() numeric fields (device.hpp:17-45), etune_device_config order
DEVICE_FIELDS = ("num_sms", "constant_power_w", "static_power_per_sm_w", "dynamic_energy_per_flop_nj",
                 "dynamic_energy_per_glb_access_nj", "dynamic_energy_per_shared_access_nj",
                 "base_throughput_flops_per_s_per_sm", "mem_bandwidth_elems_per_s", "latency_floor_ms",
                 "sampler_hz", "warmup_s", "noise_sigma_rel")
DEFAULT_DEVICE = dict(num_sms=108, constant_power_w=60.0, static_power_per_sm_w=0.55,
                      dynamic_energy_per_flop_nj=0.002, dynamic_energy_per_glb_access_nj=0.125,
                      dynamic_energy_per_shared_access_nj=0.0125, base_throughput_flops_per_s_per_sm=1.8e11,
                      mem_bandwidth_elems_per_s=3.3e11, latency_floor_ms=1e-5, sampler_hz=50.0, warmup_s=2.0,
                      noise_sigma_rel=0.05, rng_seed=1234)


class EtuneError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"status {code}: {msg}")
        self.code = code


@dataclass
class FlatForest:
    feature: np.ndarray   # int32[nodes]
    threshold: np.ndarray  # float64[nodes]
    left: np.ndarray      # int32
    right: np.ndarray     # int32
    value: np.ndarray     # float64
    offsets: np.ndarray   # int64[num_trees+1]
    base_score: float
    learning_rate: float

    @property
    def num_trees(self) -> int:
        return len(self.offsets) - 1

    def savez(self, path, **extra):
        np.savez_compressed(path, feature=self.feature, threshold=self.threshold, left=self.left,
                            right=self.right, value=self.value, offsets=self.offsets,
                            base_score=self.base_score, learning_rate=self.learning_rate, **extra)

    @staticmethod
    def from_npz(z) -> "FlatForest":
        return FlatForest(z["feature"], z["threshold"], z["left"], z["right"], z["value"], z["offsets"],
                          float(z["base_score"]), float(z["learning_rate"]))


class _Lib:
    def _check(self, st: int):
        if st != 0:
            raise EtuneError(st, self._err().decode())


class Oracle(_Lib):
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        self._err = L.orc_last_error
        L.orc_op_nest.argtypes = [I64P, I64P]
        L.orc_validate_schedule.argtypes = [I64P, I64P]
        L.orc_candidate_ids.argtypes = [I64P, I64P, C.c_int64, U64P]
        L.orc_count_schedules.argtypes = [I64P, I64P, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_enumerate.argtypes = [I64P, I64P, C.c_int64, I64P, C.POINTER(C.c_int64)]
        L.orc_counters.argtypes = [I64P, I64P, C.c_int64, C.c_int, I64P]
        L.orc_features.argtypes = [I64P, I64P, C.c_int64, C.c_int, F64P]
        L.orc_sim_measure.argtypes = [I64P, I64P, C.c_int64, F64P, C.c_uint64, F64P]
        L.orc_run_search.argtypes = [I64P, I64P, F64P, C.c_uint64, I64P, F64P, C.c_uint64, C.c_int64, I64P, F64P,
                                     C.POINTER(C.c_int64), I64P, C.POINTER(C.c_int64)]
        for nm in ("orc_mt64_words", "orc_std_mt64_words"):
            getattr(L, nm).argtypes = [C.c_uint64, C.c_int64, U64P]
        for nm in ("orc_lemire", "orc_std_uniform"):
            getattr(L, nm).argtypes = [C.c_uint64, C.c_int64, C.c_uint64, U64P]
            getattr(L, nm).restype = C.c_uint64
        for nm in ("orc_canonical", "orc_std_canonical"):
            getattr(L, nm).argtypes = [C.c_uint64, C.c_int64, F64P]
        L.orc_sample_random.argtypes = [I64P, C.c_int64, C.c_uint64, I64P, I64P, U64P]
        L.orc_reproduce.argtypes = [I64P, I64P, C.c_int64, C.c_int64, F64P, C.c_uint64, I64P,
                                    I64P, U64P, U64P, I8P]
        L.orc_reproduce_counter.argtypes = L.orc_reproduce.argtypes
        L.orc_predict.argtypes = [I32P, F64P, I32P, I32P, F64P, I64P, C.c_int64, C.c_double,
                                  C.c_double, F64P, C.c_int64, F64P]
        L.orc_train.argtypes = [F64P, F64P, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_double, I32P, F64P, I32P, I32P, F64P, I64P,
                                C.POINTER(C.c_double), C.POINTER(C.c_double), F64P]
        L.orc_energy_loss.argtypes = [C.c_double, C.c_double, F64P]
        L.orc_snr_db.argtypes = [F64P, F64P, C.c_int64, C.POINTER(C.c_double)]
        L.orc_topk.argtypes = [F64P, C.c_int64, C.c_int64, I64P]
        L.orc_score_threads.argtypes = [I64P, I64P, C.c_int64, C.c_int, I32P, F64P, I32P, I32P,
                                        F64P, I64P, C.c_int64, C.c_double, C.c_double, C.c_int,
                                        F64P]

    # --- space / features
    def nest(self, op):
        out = np.zeros(4, np.int64)
        self._check(self.L.orc_op_nest(op, out))
        return out

    def validate(self, op, sched) -> int:
        return self.L.orc_validate_schedule(op, np.ascontiguousarray(sched, np.int64))

    def ids(self, op, sched):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros(len(sched), np.uint64)
        self._check(self.L.orc_candidate_ids(op, sched, len(sched), out))
        return out

    def count(self, op, limits=None, cap=0):
        out = C.c_int64()
        self._check(self.L.orc_count_schedules(op, default_limits() if limits is None else limits, cap,
                                               C.byref(out)))
        return out.value

    def enumerate(self, op, limits=None, cap=None):
        cap = self.count(op, limits) if cap is None else cap
        out = np.zeros((max(cap, 1), 12), np.int64)
        n = C.c_int64()
        self._check(self.L.orc_enumerate(op, default_limits() if limits is None else limits, cap, out,
                                         C.byref(n)))
        return out[: n.value]

    def counters(self, op, sched, num_sms=108):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros((len(sched), 10), np.int64)
        self._check(self.L.orc_counters(op, sched, len(sched), num_sms, out))
        return out

    def features(self, op, sched, num_sms=108):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros((len(sched), 16), np.float64)
        self._check(self.L.orc_features(op, sched, len(sched), num_sms, out))
        return out

    def sim_measure(self, op, sched, dev=None):
        """SimBackend restatement: n x {latency_ms, avg_power_w, energy_mj, iterations}.
        dev: dict of DeviceConfig numeric fields (defaults: a100_like, device.hpp:17-45)."""
        d = dict(DEFAULT_DEVICE)
        d.update(dev or {})
        dev12 = np.array([d[k] for k in DEVICE_FIELDS], np.float64)
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros((len(sched), 4), np.float64)
        self._check(self.L.orc_sim_measure(op, sched, len(sched), dev12, int(d["rng_seed"]), out))
        return out

    def run_search(self, op, M, G, seed, max_rounds=10, patience=5, k_init_fifths=5, inverted=0, num_trees=100,
                   max_depth=6, mu_db=20.0, improve_rel=0.001, rates=(0.85, 0.10, 0.05), lr=0.1,
                   min_leaf_weight=1e-3, reg_lambda=1.0, dev=None, limits=None, latency_only=0):
        """Algorithm 1 restatement -> (reports_int n x 6, reports_f64 n x 4, parent schedules)."""
        d = dict(DEFAULT_DEVICE)
        d.update(dev or {})
        dev12 = np.array([d[k] for k in DEVICE_FIELDS], np.float64)
        cfg_i = np.array([M, G, k_init_fifths, max_rounds, patience, inverted, num_trees, max_depth, latency_only],
                         np.int64)
        cfg_d = np.array([mu_db, improve_rel, *rates, lr, min_leaf_weight, reg_lambda], np.float64)
        cap = max_rounds + 1
        ri = np.zeros((cap, 6), np.int64)
        rd = np.zeros((cap, 4), np.float64)
        par = np.zeros(((M + 1) // 2 if max_rounds > 0 else M, 12), np.int64)
        par = np.zeros((M, 12), np.int64)
        nr, npar = C.c_int64(), C.c_int64()
        self._check(self.L.orc_run_search(op, default_limits() if limits is None else limits, dev12,
                                          int(d["rng_seed"]), cfg_i, cfg_d, seed, cap, ri, rd, C.byref(nr), par,
                                          C.byref(npar)))
        return ri[:nr.value], rd[:nr.value], par[:npar.value]

    # --- search primitives
    def sample_random(self, op, n, seed, limits=None):
        s = np.zeros((n, 12), np.int64)
        ids = np.zeros(n, np.uint64)
        self._check(self.L.orc_sample_random(op, n, seed, default_limits() if limits is None else limits,
                                             s, ids))
        return s, ids

    def reproduce(self, op, parents, n, seed, rates=(0.85, 0.10, 0.05), limits=None):
        parents = np.ascontiguousarray(parents, np.int64).reshape(-1, 12)
        s = np.zeros((n, 12), np.int64)
        ids = np.zeros(n, np.uint64)
        lin = np.zeros((n, 2), np.uint64)
        ll = np.zeros(n, np.int8)
        self._check(self.L.orc_reproduce(op, parents, len(parents), n, np.array(rates, np.float64), seed,
                                         default_limits() if limits is None else limits, s, ids, lin, ll))
        return s, ids, lin, ll

    def reproduce_counter(self, op, parents, n, seed, rates=(0.85, 0.10, 0.05), limits=None):
        """The opt-in counter-based reproduce mode (per-offspring splitmix64 streams)."""
        parents = np.ascontiguousarray(parents, np.int64).reshape(-1, 12)
        s = np.zeros((n, 12), np.int64)
        ids = np.zeros(n, np.uint64)
        lin = np.zeros((n, 2), np.uint64)
        ll = np.zeros(n, np.int8)
        self._check(self.L.orc_reproduce_counter(op, parents, len(parents), n, np.array(rates, np.float64), seed,
                                                 default_limits() if limits is None else limits, s, ids, lin, ll))
        return s, ids, lin, ll

    # --- cost model
    def predict(self, forest: FlatForest, feats):
        feats = np.ascontiguousarray(feats, np.float64).reshape(-1, 16)
        out = np.zeros(len(feats), np.float64)
        f = forest
        self._check(self.L.orc_predict(f.feature, f.threshold, f.left, f.right, f.value, f.offsets,
                                       f.num_trees, f.base_score, f.learning_rate, feats, len(feats), out))
        return out

    def train(self, feats, energy, num_trees=100, max_depth=6, lr=0.1, min_leaf_weight=1e-3,
              reg_lambda=1.0):
        feats = np.ascontiguousarray(feats, np.float64).reshape(-1, 16)
        energy = np.ascontiguousarray(energy, np.float64)
        cap = num_trees * ((1 << (max_depth + 1)) - 1)
        fe = np.zeros(cap, np.int32)
        th = np.zeros(cap, np.float64)
        le = np.zeros(cap, np.int32)
        ri = np.zeros(cap, np.int32)
        va = np.zeros(cap, np.float64)
        off = np.zeros(num_trees + 1, np.int64)
        base, ref = C.c_double(), C.c_double()
        loss = np.zeros(num_trees + 1, np.float64)
        self._check(self.L.orc_train(feats, energy, len(feats), num_trees, max_depth, lr, min_leaf_weight,
                                     reg_lambda, fe, th, le, ri, va, off, C.byref(base), C.byref(ref), loss))
        m = int(off[-1])
        return FlatForest(fe[:m].copy(), th[:m].copy(), le[:m].copy(), ri[:m].copy(), va[:m].copy(), off,
                          base.value, lr), ref.value, loss

    def energy_loss(self, p, m):
        out = np.zeros(3, np.float64)
        self._check(self.L.orc_energy_loss(p, m, out))
        return out

    def snr_db(self, p, m):
        out = C.c_double()
        p = np.ascontiguousarray(p, np.float64)
        m = np.ascontiguousarray(m, np.float64)
        self._check(self.L.orc_snr_db(p, m, len(p), C.byref(out)))
        return out.value

    def topk(self, score, k):
        score = np.ascontiguousarray(score, np.float64)
        out = np.zeros(k, np.int64)
        self._check(self.L.orc_topk(score, len(score), k, out))
        return out

    def score_threads(self, op, sched, forest: FlatForest, threads=1, num_sms=108):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros(len(sched), np.float64)
        f = forest
        self._check(self.L.orc_score_threads(op, sched, len(sched), num_sms, f.feature, f.threshold,
                                             f.left, f.right, f.value, f.offsets, f.num_trees,
                                             f.base_score, f.learning_rate, threads, out))
        return out


class RefLib(_Lib):
    """The unmodified reference (oracle/_ref).  Available wherever oracle/_ref was built."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        self._err = L.ref_last_error
        L.ref_op_nest.argtypes = [I64P, I64P]
        L.ref_parse_operator.argtypes = [C.c_char_p, I64P]
        L.ref_count_schedules.argtypes = [I64P, I64P, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_enumerate.argtypes = [I64P, I64P, C.c_int64, I64P, C.POINTER(C.c_int64)]
        L.ref_candidate_ids.argtypes = [I64P, I64P, C.c_int64, U64P]
        L.ref_is_legal.argtypes = [I64P, I64P, C.c_int64, U8P]
        L.ref_counters.argtypes = [I64P, I64P, C.c_int64, C.c_int, I64P]
        L.ref_interpret_counters.argtypes = [I64P, I64P, C.c_int, I64P]
        L.ref_features.argtypes = [I64P, I64P, C.c_int64, C.c_int, F64P]
        L.ref_log1p.argtypes = [C.c_double]
        L.ref_log1p.restype = C.c_double
        L.ref_sample_random.argtypes = [I64P, C.c_int64, C.c_uint64, I64P, I64P, U64P]
        L.ref_reproduce.argtypes = [I64P, I64P, C.c_int64, C.c_int64, F64P, C.c_uint64, I64P, I64P,
                                    U64P, U64P, I8P]
        L.ref_train.argtypes = [F64P, F64P, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_double, C.POINTER(C.c_void_p)]
        L.ref_model_from_json.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_to_json.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_model_to_json.restype = C.c_int64
        L.ref_model_info.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_model_nodes.argtypes = [C.c_void_p, I32P, F64P, I32P, I32P, F64P, I64P]
        L.ref_training_loss.argtypes = [C.c_void_p, F64P, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_predict.argtypes = [C.c_void_p, F64P, C.c_int64, F64P]
        L.ref_device_profile_to_json.argtypes = [C.c_int, F64P, C.c_uint64, C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_device_profile_to_json.restype = C.c_int64
        L.ref_device_profile_from_json.argtypes = [C.c_char_p, C.POINTER(C.c_int), F64P, C.POINTER(C.c_uint64),
                                                   C.c_char_p, C.c_int64]
        L.ref_samples_save.argtypes = [F64P, F64P, F64P, C.c_int64, C.c_char_p]
        L.ref_samples_load.argtypes = [C.c_char_p, F64P, F64P, F64P, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_snr_db.argtypes = [F64P, F64P, C.c_int64, C.POINTER(C.c_double)]
        L.ref_energy_loss.argtypes = [C.c_double, C.c_double, F64P]
        L.ref_spearman.argtypes = [F64P, F64P, C.c_int64, C.POINTER(C.c_double)]
        L.ref_score_threads.argtypes = [I64P, I64P, C.c_int64, C.c_int, C.c_void_p, C.c_int, F64P]
        L.ref_score_select_threads.argtypes = [I64P, I64P, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_int64,
                                               F64P, I64P]

    def parse(self, text):
        out = np.zeros(12, np.int64)
        self._check(self.L.ref_parse_operator(text.encode(), out))
        return out

    def nest(self, op):
        out = np.zeros(4, np.int64)
        self._check(self.L.ref_op_nest(op, out))
        return out

    def count(self, op, limits=None, cap=0):
        out = C.c_int64()
        self._check(self.L.ref_count_schedules(op, default_limits() if limits is None else limits, cap,
                                               C.byref(out)))
        return out.value

    def enumerate(self, op, limits=None, cap=None):
        cap = self.count(op, limits) if cap is None else cap
        out = np.zeros((max(cap, 1), 12), np.int64)
        n = C.c_int64()
        self._check(self.L.ref_enumerate(op, default_limits() if limits is None else limits, cap, out,
                                         C.byref(n)))
        return out[: n.value]

    def ids(self, op, sched):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros(len(sched), np.uint64)
        self._check(self.L.ref_candidate_ids(op, sched, len(sched), out))
        return out

    def legal(self, op, sched):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros(len(sched), np.uint8)
        self._check(self.L.ref_is_legal(op, sched, len(sched), out))
        return out.astype(bool)

    def counters(self, op, sched, num_sms=108):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros((len(sched), 10), np.int64)
        self._check(self.L.ref_counters(op, sched, len(sched), num_sms, out))
        return out

    def interpret(self, op, sched, num_sms=108):
        out = np.zeros(10, np.int64)
        self._check(self.L.ref_interpret_counters(op, np.ascontiguousarray(sched, np.int64), num_sms, out))
        return out

    def features(self, op, sched, num_sms=108):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros((len(sched), 16), np.float64)
        self._check(self.L.ref_features(op, sched, len(sched), num_sms, out))
        return out

    def sample_random(self, op, n, seed, limits=None):
        s = np.zeros((n, 12), np.int64)
        ids = np.zeros(n, np.uint64)
        self._check(self.L.ref_sample_random(op, n, seed, default_limits() if limits is None else limits,
                                             s, ids))
        return s, ids

    def reproduce(self, op, parents, n, seed, rates=(0.85, 0.10, 0.05), limits=None):
        parents = np.ascontiguousarray(parents, np.int64).reshape(-1, 12)
        s = np.zeros((n, 12), np.int64)
        ids = np.zeros(n, np.uint64)
        lin = np.zeros((n, 2), np.uint64)
        ll = np.zeros(n, np.int8)
        self._check(self.L.ref_reproduce(op, parents, len(parents), n, np.array(rates, np.float64), seed,
                                         default_limits() if limits is None else limits, s, ids, lin, ll))
        return s, ids, lin, ll

    def train(self, feats, energy, num_trees=100, max_depth=6, lr=0.1, min_leaf_weight=1e-3,
              reg_lambda=1.0) -> "RefModel":
        feats = np.ascontiguousarray(feats, np.float64).reshape(-1, 16)
        energy = np.ascontiguousarray(energy, np.float64)
        h = C.c_void_p()
        self._check(self.L.ref_train(feats, energy, len(feats), num_trees, max_depth, lr, min_leaf_weight,
                                     reg_lambda, C.byref(h)))
        return RefModel(self, h)

    # ---- persistence formats (device.cpp:44-101, energy_model.cpp:372-420)
    DEV_FIELDS = ("constant_power_w", "static_power_per_sm_w", "dynamic_energy_per_flop_nj",
                  "dynamic_energy_per_glb_access_nj", "dynamic_energy_per_shared_access_nj",
                  "base_throughput_flops_per_s_per_sm", "mem_bandwidth_elems_per_s", "latency_floor_ms",
                  "sampler_hz", "warmup_s", "noise_sigma_rel")

    def device_profile_to_json(self, num_sms: int, fields, seed: int, name: str) -> str:
        f = np.ascontiguousarray(fields, np.float64)
        need = self.L.ref_device_profile_to_json(num_sms, f, seed, name.encode(), None, 0)
        buf = C.create_string_buffer(int(need))
        self.L.ref_device_profile_to_json(num_sms, f, seed, name.encode(), buf, need)
        return buf.value.decode()

    def device_profile_from_json(self, text: str):
        n = C.c_int()
        f = np.zeros(11, np.float64)
        seed = C.c_uint64()
        name = C.create_string_buffer(4096)
        self._check(self.L.ref_device_profile_from_json(text.encode(), C.byref(n), f, C.byref(seed), name, 4096))
        return n.value, f, seed.value, name.value.decode()

    def samples_to_jsonl(self, feats, meas, norm) -> str:
        import tempfile
        feats = np.ascontiguousarray(feats, np.float64).reshape(-1, 16)
        meas = np.ascontiguousarray(meas, np.float64)
        norm = np.ascontiguousarray(norm, np.float64)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "s.jsonl")
            self._check(self.L.ref_samples_save(feats, meas, norm, len(meas), path.encode()))
            return open(path).read()

    def samples_from_jsonl(self, text: str):
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "s.jsonl")
            open(path, "w").write(text)
            cap = text.count("\n") + 1
            f = np.zeros((cap, 16), np.float64)
            m = np.zeros(cap, np.float64)
            z = np.zeros(cap, np.float64)
            n = C.c_int64()
            self._check(self.L.ref_samples_load(path.encode(), f, m, z, cap, C.byref(n)))
            k = n.value
            return f[:k], m[:k], z[:k]

    def model_from_json(self, text: str) -> "RefModel":
        h = C.c_void_p()
        self._check(self.L.ref_model_from_json(text.encode(), C.byref(h)))
        return RefModel(self, h)

    def snr_db(self, p, m):
        out = C.c_double()
        p = np.ascontiguousarray(p, np.float64)
        m = np.ascontiguousarray(m, np.float64)
        self._check(self.L.ref_snr_db(p, m, len(p), C.byref(out)))
        return out.value

    def energy_loss(self, p, m):
        out = np.zeros(3, np.float64)
        self._check(self.L.ref_energy_loss(p, m, out))
        return out


class RefModel:
    def __init__(self, lib: RefLib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.L.ref_model_free(self.h)
        except Exception:
            pass

    def to_json(self) -> str:
        need = self.lib.L.ref_model_to_json(self.h, None, 0)
        buf = C.create_string_buffer(int(need))
        self.lib.L.ref_model_to_json(self.h, buf, need)
        return buf.value.decode()

    def flat(self) -> FlatForest:
        b, lr, re = C.c_double(), C.c_double(), C.c_double()
        nt, nn = C.c_int64(), C.c_int64()
        self.lib.L.ref_model_info(self.h, C.byref(b), C.byref(lr), C.byref(re), C.byref(nt), C.byref(nn))
        n = nn.value
        fe = np.zeros(max(n, 1), np.int32)
        th = np.zeros(max(n, 1), np.float64)
        le = np.zeros(max(n, 1), np.int32)
        ri = np.zeros(max(n, 1), np.int32)
        va = np.zeros(max(n, 1), np.float64)
        off = np.zeros(nt.value + 1, np.int64)
        self.lib.L.ref_model_nodes(self.h, fe, th, le, ri, va, off)
        return FlatForest(fe[:n], th[:n], le[:n], ri[:n], va[:n], off, b.value, lr.value)

    def reference_energy(self) -> float:
        b, lr, re = C.c_double(), C.c_double(), C.c_double()
        nt, nn = C.c_int64(), C.c_int64()
        self.lib.L.ref_model_info(self.h, C.byref(b), C.byref(lr), C.byref(re), C.byref(nt), C.byref(nn))
        return re.value

    def training_loss(self):
        out = np.zeros(4096, np.float64)
        n = C.c_int64()
        self.lib.L.ref_training_loss(self.h, out, 4096, C.byref(n))
        return out[: n.value]

    def predict(self, feats):
        feats = np.ascontiguousarray(feats, np.float64).reshape(-1, 16)
        out = np.zeros(len(feats), np.float64)
        self.lib._check(self.lib.L.ref_predict(self.h, feats, len(feats), out))
        return out

    def score_threads(self, op, sched, threads, num_sms=108):
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros(len(sched), np.float64)
        self.lib._check(self.lib.L.ref_score_threads(op, sched, len(sched), num_sms, self.h, threads, out))
        return out

    def score_select_threads(self, op, sched, threads, k, num_sms=108):
        """extract_features + predict + k best by (prediction, index), all on `threads` threads
        (ref_shim.cpp ref_score_select_threads) -> (predictions, sorted indices)."""
        sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
        out = np.zeros(len(sched), np.float64)
        idx = np.zeros(max(k, 1), np.int64)
        self.lib._check(self.lib.L.ref_score_select_threads(op, sched, len(sched), num_sms, self.h, threads, int(k),
                                                            out, idx))
        return out, idx[:k]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


SCC_SO = os.path.join(ROOT, "tests", "cpp", "libscorecheck.so")


def host_compiled_score(op, forest: "FlatForest", sched, num_sms=108, keyed=False):
    """Forest compiler + scoring core run on the CPU (tests/cpp/score_core_check.cpp);
    keyed=True scores through the keyed form (full (key, Kuv class) table when it fits),
    keyed="byte" through the per-key byte table only."""
    L = C.CDLL(SCC_SO)
    L.scc_last_error.restype = C.c_char_p
    fn = L.scc_score_keyed8 if keyed == "byte" else L.scc_score_keyed if keyed else L.scc_score
    fn.argtypes = [I64P, C.c_int, I32P, F64P, I32P, I32P, F64P, I64P, C.c_int64, C.c_double, C.c_double,
                   I64P, C.c_int64, F64P, I64P]
    sched = np.ascontiguousarray(sched, np.int64).reshape(-1, 12)
    out = np.zeros(len(sched))
    stats = np.zeros(8, np.int64)
    f = forest
    st = fn(np.ascontiguousarray(op, np.int64), num_sms, f.feature, f.threshold, f.left, f.right, f.value,
            f.offsets, f.num_trees, f.base_score, f.learning_rate, sched, len(sched), out, stats)
    if st:
        raise EtuneError(st, L.scc_last_error().decode())
    return out, stats
