"""CPU oracle for the PUFFINN (arXiv 1906.12211) batched LSH-forest k-NN query path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares no code with
``paper_1906_12211_b200`` (the product) and never imports it; the product never imports this.

The arithmetic lives in ``oracle.c`` (plain scalar C, ``-O2 -ffp-contract=off``); this module
only compiles it and marshals numpy arrays through ctypes.  Each C function cites the
PAPER.md passage it restates; DESIGN.md lists the readings ("R-n") it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

HP, FHTCP, CP = 0, 1, 2
INDEPENDENT, POOL, TENSOR = 0, 1, 2


def build_lib(force: bool = False) -> str:
    """Compile oracle.c into oracle/liboracle.so (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
                               "-shared", "-std=c11", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build_lib())
        L = _lib
        P = C.c_void_p
        L.or_mix64.restype = C.c_uint64; L.or_mix64.argtypes = [C.c_uint64]
        L.or_draw.restype = C.c_uint64; L.or_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.or_stream_key.restype = C.c_uint64; L.or_stream_key.argtypes = [C.c_uint64, C.c_uint64]
        L.or_gauss_d.restype = C.c_double; L.or_gauss_d.argtypes = [C.c_uint64, C.c_uint64]
        L.or_normalize.restype = C.c_int64; L.or_normalize.argtypes = [P, C.c_int64, C.c_int, P]
        L.or_dot.restype = C.c_float; L.or_dot.argtypes = [P, P, C.c_int]
        L.or_sim.restype = C.c_float; L.or_sim.argtypes = [P, P, C.c_int]
        L.or_hp_bit.restype = C.c_int; L.or_hp_bit.argtypes = [P, P, C.c_int]
        L.or_fht.restype = None; L.or_fht.argtypes = [P, C.c_int]
        L.or_fhtcp_code.restype = C.c_uint32; L.or_fhtcp_code.argtypes = [P, C.c_int, C.c_int, P]
        L.or_cp_code.restype = C.c_uint32; L.or_cp_code.argtypes = [P, P, C.c_int, C.c_int]
        L.or_cp_table.restype = None
        L.or_cp_table.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, P, P]
        L.or_build.restype = P
        L.or_build.argtypes = [P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_int, C.c_uint64, C.c_int, C.c_int, P]
        L.or_free.restype = None; L.or_free.argtypes = [P]
        L.or_info.restype = None; L.or_info.argtypes = [P, P]
        L.or_get_rep.restype = None; L.or_get_rep.argtypes = [P, C.c_int, P, P]
        L.or_get_data.restype = None; L.or_get_data.argtypes = [P, P]
        L.or_get_sketches.restype = None; L.or_get_sketches.argtypes = [P, P]
        L.or_get_slots.restype = None; L.or_get_slots.argtypes = [P, P]
        L.or_get_sel.restype = None; L.or_get_sel.argtypes = [P, P]
        L.or_get_cp.restype = None; L.or_get_cp.argtypes = [P, P]
        L.or_hash.restype = C.c_int64; L.or_hash.argtypes = [P, P, C.c_int64, P, P]
        L.or_prefix_table.restype = None; L.or_prefix_table.argtypes = [P, C.c_int, P]
        L.or_grid_bucket.restype = C.c_int; L.or_grid_bucket.argtypes = [C.c_float]
        L.or_P.restype = C.c_double; L.or_P.argtypes = [P, C.c_int, C.c_float]
        L.or_fixed16.restype = C.c_int16; L.or_fixed16.argtypes = [C.c_float]
        L.or_quantize.restype = None; L.or_quantize.argtypes = [P, C.c_int64, C.c_int, P]
        L.or_sim16.restype = C.c_float; L.or_sim16.argtypes = [P, P, C.c_int]
        L.or_set_storage.restype = None; L.or_set_storage.argtypes = [P, C.c_int]
        L.or_get_data16.restype = None; L.or_get_data16.argtypes = [P, P]
        L.or_should_stop.restype = C.c_int
        L.or_should_stop.argtypes = [P, C.c_int, C.c_int, C.c_float, C.c_double, C.c_int]
        L.or_tau.restype = C.c_int; L.or_tau.argtypes = [C.c_float, C.c_float]
        L.or_tau_prob.restype = C.c_int; L.or_tau_prob.argtypes = [C.c_float, C.c_double]
        L.or_sim_seq.restype = C.c_float; L.or_sim_seq.argtypes = [P, P, C.c_int]
        L.or_search.restype = None
        L.or_search.argtypes = [P, P, C.c_int64, C.c_int, C.c_float, P, C.c_int, P, P, P, P, C.c_int]
        L.or_widen.restype = None
        L.or_widen.argtypes = [P, C.c_int64, C.c_uint32, C.c_int, C.c_int, C.c_int, P, P]
        L.or_lower_bound_pub.restype = C.c_int64
        L.or_lower_bound_pub.argtypes = [P, C.c_int64, C.c_uint64]
        L.or_bruteforce.restype = None
        L.or_bruteforce.argtypes = [P, C.c_int64, C.c_int, P, C.c_int64, C.c_int, P, P]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- primitives
def mix64(z: int) -> int:
    return int(lib().or_mix64(z))


def draw(key: int, c: int) -> int:
    return int(lib().or_draw(key, c))


def stream_key(seed: int, tag: int) -> int:
    return int(lib().or_stream_key(seed, tag))


def gauss_d(key: int, i: int) -> float:
    return float(lib().or_gauss_d(key, i))


def normalize(x) -> np.ndarray:
    x = _f32(x)
    out = np.empty_like(x)
    e = lib().or_normalize(_p(x), x.shape[0], x.shape[1], _p(out))
    if e >= 0:
        raise ZeroDivisionError(f"zero vector at row {e}")
    return out


def dot(a, b) -> float:
    a, b = _f32(a), _f32(b)
    return float(lib().or_dot(_p(a), _p(b), a.shape[0]))


def sim(a, b) -> float:
    """canonical similarity (32-lane tree order, R-2)"""
    a, b = _f32(a), _f32(b)
    return float(lib().or_sim(_p(a), _p(b), a.shape[0]))


def fixed16(x) -> np.ndarray:
    """R-25: 16-bit fixed point of normalised coordinates (clamp(rint(x 2^15)))"""
    x = _f32(np.atleast_1d(x))
    out = np.empty(x.shape, dtype=np.int16)
    lib().or_quantize(_p(x), 1, x.size, _p(out))
    return out


def sim16(a16, b16) -> float:
    """R-25: the exact fixed-point inner product, scaled by 2^-30"""
    a16 = np.ascontiguousarray(a16, dtype=np.int16)
    b16 = np.ascontiguousarray(b16, dtype=np.int16)
    return float(lib().or_sim16(_p(a16), _p(b16), a16.shape[0]))


def hp_bit(a, x) -> int:
    a, x = _f32(a), _f32(x)
    return int(lib().or_hp_bit(_p(a), _p(x), a.shape[0]))


def fht(y) -> np.ndarray:
    y = _f32(y).copy()
    lib().or_fht(_p(y), y.shape[0])
    return y


def fhtcp_code(x, dp: int, signs) -> int:
    x, s = _f32(x), _f32(signs)
    return int(lib().or_fhtcp_code(_p(x), x.shape[0], dp, _p(s)))


def cp_code(A, x) -> int:
    """exact cross-polytope value of x under hyperplanes A [d][d]"""
    A, x = _f32(A), _f32(x)
    d = x.shape[0]
    ell = 1 + int(np.ceil(np.log2(d))) if d > 1 else 1
    return int(lib().or_cp_code(_p(A), _p(x), d, ell))


def cp_table(family: int, d: int, seed: int, draws: int = 1000):
    """Monte-Carlo collision table T[b][a] (b = 0..ell, a = 0..40 on the alpha grid)."""
    T = np.zeros(34 * 41, dtype=np.float64)
    ell = C.c_int(0)
    lib().or_cp_table(family, d, seed, draws, _p(T), C.byref(ell))
    return T[: (ell.value + 1) * 41].reshape(ell.value + 1, 41)


def grid_bucket(ip: float) -> int:
    return int(lib().or_grid_bucket(ip))


def tau(ipk: float, eps: float = 0.0) -> int:
    return int(lib().or_tau(ipk, eps))


def tau_prob(ipk: float, delta: float) -> int:
    """R-26: smallest t with P[Binomial(64, acos(ipk)/pi) <= t] >= 1 - delta"""
    return int(lib().or_tau_prob(ipk, delta))


def sim_seq(a, b) -> float:
    """O-11 plain-order similarity (sequential fmaf chain)"""
    a, b = _f32(a), _f32(b)
    return float(lib().or_sim_seq(_p(a), _p(b), a.shape[0]))


def lower_bound(codes, v: int) -> int:
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    return int(lib().or_lower_bound_pub(_p(c), c.shape[0], v))


def widen(codes, qcode: int, K: int, i: int, B: int, elo: int, ehi: int):
    """one widening step of a repetition's emitted range to prefix length i -> (elo, ehi)"""
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    lo, hi = C.c_int64(elo), C.c_int64(ehi)
    lib().or_widen(_p(c), c.shape[0], qcode, K, i, B, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def bruteforce(x, q, k: int):
    """exact top-k by double similarity (x, q already normalised)"""
    x, q = _f32(x), _f32(q)
    nq = q.shape[0]
    ids = np.empty((nq, k), dtype=np.int64)
    sims = np.empty((nq, k), dtype=np.float64)
    lib().or_bruteforce(_p(x), x.shape[0], x.shape[1], _p(q), nq, k, _p(ids), _p(sims))
    return ids, sims


# ---------------------------------------------------------------- index
class _SOpts(C.Structure):
    _fields_ = [("rep_chunk", C.c_int32), ("stop_rule", C.c_int32), ("per_round", C.c_int32),
                ("segment", C.c_int32), ("use_filter", C.c_int32), ("eps", C.c_float),
                ("uniform_chunks", C.c_int32), ("sim_order", C.c_int32), ("tau_rule", C.c_int32),
                ("rerank", C.c_int32)]


class OracleIndex:
    """Oracle LSH forest.  family: HP | FHTCP; strategy: INDEPENDENT | POOL | TENSOR; explicit L, K, M."""

    def __init__(self, data, family: int, L: int, seed: int = 1, K: int = 24, M: int = 32,
                 strategy: int = INDEPENDENT, pool_bits: int = 3072, lazy: bool = False,
                 cp_draws: int = 1000, storage: str = "f32"):
        data = _f32(data)
        self.n, self.d = data.shape
        if strategy == TENSOR:
            s = int(round(L ** 0.5))
            ell = 1 if family == HP else 1 + int(np.ceil(np.log2(max(2, 1 << int(np.ceil(np.log2(self.d)))))))
            if s * s != L or (s & (s - 1)) or (K % ell) or ((K // ell) % 2):
                raise ValueError("tensor: L must be an even power of two and K an even number of whole functions")
        err = C.c_int64(-1)
        self._h = lib().or_build(_p(data), self.n, self.d, family, strategy, L, K, M, pool_bits,
                                 seed, int(lazy), cp_draws, C.byref(err))
        if not self._h:
            raise ZeroDivisionError(f"zero vector at row {err.value}")
        info = np.zeros(9, dtype=np.int64)
        lib().or_info(self._h, _p(info))
        (_, _, self.dp, self.ell, self.c, self.L, self.K, self.M, self.m) = [int(v) for v in info]
        self.family, self.strategy = family, strategy
        self.storage = storage
        if storage == "i16":
            lib().or_set_storage(self._h, 1)
        elif storage != "f32":
            raise ValueError("storage must be 'f32' or 'i16'")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().or_free(h)
            self._h = None

    def rep(self, j: int):
        codes = np.empty(self.n, dtype=np.uint32)
        ids = np.empty(self.n, dtype=np.uint32)
        lib().or_get_rep(self._h, j, _p(codes), _p(ids))
        return codes, ids

    def prefix_table(self, j: int) -> np.ndarray:
        pt = np.empty(8193, dtype=np.uint32)
        lib().or_prefix_table(self._h, j, _p(pt))
        return pt

    def data(self) -> np.ndarray:
        x = np.empty((self.n, self.d), dtype=np.float32)
        lib().or_get_data(self._h, _p(x))
        return x

    def data16(self) -> np.ndarray:
        x = np.empty((self.n, self.d), dtype=np.int16)
        lib().or_get_data16(self._h, _p(x))
        return x

    def sketches(self) -> np.ndarray:
        s = np.empty((self.n, self.M), dtype=np.uint64)
        lib().or_get_sketches(self._h, _p(s))
        return s

    def slots(self) -> np.ndarray:
        s = np.empty(self.L, dtype=np.int32)
        lib().or_get_slots(self._h, _p(s))
        return s

    def pool_sel(self) -> np.ndarray:
        s = np.zeros((self.L, self.c), dtype=np.int32)
        lib().or_get_sel(self._h, _p(s))
        return s

    def cp(self) -> np.ndarray:
        T = np.empty((self.ell + 1) * 41, dtype=np.float64)
        lib().or_get_cp(self._h, _p(T))
        return T.reshape(self.ell + 1, 41)

    def hash(self, raw):
        raw = _f32(raw)
        nq = raw.shape[0]
        codes = np.empty((nq, self.L), dtype=np.uint32)
        sk = np.empty((nq, max(self.M, 1)), dtype=np.uint64)
        e = lib().or_hash(self._h, _p(raw), nq, _p(codes), _p(sk))
        if e >= 0:
            raise ZeroDivisionError(f"zero vector at row {e}")
        return codes, sk[:, : self.M]

    def P(self, i: int, ip: float) -> float:
        return float(lib().or_P(self._h, i, ip))

    def should_stop(self, i: int, j: int, ip: float, delta: float, rule: int = 0) -> bool:
        return bool(lib().or_should_stop(self._h, i, j, ip, delta, rule))

    def search(self, queries, k: int, recall: float, rep_chunk: int = 1, stop_rule: int = 0,
               per_round: bool = False, segment: int = 12, use_filter: bool = True, eps: float = 0.0,
               threads: int = 1, trace_cap: int = 0, uniform_chunks: bool = False, sim_order: int = 0,
               tau_rule: int = 0, rerank: bool = True):
        """returns ids[nq,k] int64, sims[nq,k] f32, trace[nq,8] int32
        (i_stop, j_stop, emitted, filtered, dups, evaluated, flags, 0)
        and, if trace_cap > 0, the evaluated ids in evaluation order [nq, trace_cap] (uint32)."""
        q = _f32(queries)
        nq = q.shape[0]
        ids = np.empty((nq, k), dtype=np.int64)
        sims = np.empty((nq, k), dtype=np.float32)
        trace = np.zeros((nq, 8), dtype=np.int32)
        tids = np.zeros((nq, max(trace_cap, 1)), dtype=np.uint32)
        o = _SOpts(rep_chunk, stop_rule, int(per_round), segment, int(use_filter), eps, int(uniform_chunks),
                   int(sim_order), int(tau_rule), int(rerank))
        lib().or_search(self._h, _p(q), nq, k, recall, C.byref(o), threads, _p(ids), _p(sims), _p(trace),
                        _p(tids) if trace_cap > 0 else None, trace_cap)
        if trace_cap > 0:
            return ids, sims, trace, tids
        return ids, sims, trace
