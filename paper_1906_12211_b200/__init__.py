"""paper_1906_12211_b200 — B200-native batched LSH-forest k-NN (PUFFINN, arXiv 1906.12211).

Thin Python binding over the C-ABI library ``libpfg.so`` (include/pfg.h).  This module only
marshals arguments: every step of the build and of the search runs in the library's CUDA
kernels.  PyTorch is used for device memory and streams; numpy arrays are passed as host
pointers (the library then copies through its own device buffers).  There is no CPU fallback:
if the library is missing, importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from ._build import LIB as _LIB_PATH

SIMHASH, CROSSPOLYTOPE_FHT = 0, 1
DEFAULT_REP_CHUNK = 16  # R of pfg_search_opts (R-17); measured best on config 2
INDEPENDENT, POOL, TENSOR = 0, 1, 2
CROSSPOLYTOPE = 2
FAMILIES = {"simhash": SIMHASH, "hp": SIMHASH, "fht_cp": CROSSPOLYTOPE_FHT, "crosspolytope_fht": CROSSPOLYTOPE_FHT,
            "cp": CROSSPOLYTOPE, "crosspolytope": CROSSPOLYTOPE}
STRATEGIES = {"independent": INDEPENDENT, "pool": POOL, "tensor": TENSOR}

EXPORT_TABLE, EXPORT_PREFIX, EXPORT_SKETCH, EXPORT_DATA, EXPORT_CP, EXPORT_SLOTS, EXPORT_POOLSEL = 1, 2, 3, 4, 5, 6, 7
EXPORT_DATA16 = 8

STATUS = {0: "PFG_OK", 1: "PFG_E_ARG", 2: "PFG_E_ZERO_VECTOR", 3: "PFG_E_BUDGET", 4: "PFG_E_CUDA",
          5: "PFG_E_OOM", 7: "PFG_E_STATE"}

# symbols include/pfg.h declares (checked by tests/test_abi.py)
EXPORTED = ["pfg_build", "pfg_search", "pfg_merge_topk", "pfg_index_info", "pfg_derive_reps", "pfg_export",
            "pfg_hash_queries", "pfg_stop_tables", "pfg_last_timing", "pfg_last_phases", "pfg_free", "pfg_last_error",
            "pfg_abi_version", "pfg_save", "pfg_load", "pfg_kernel_timing", "pfg_round_stats",
            "pfg_hash_queries_reps"]


class PfgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class BuildOpts(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("strategy", C.c_int32), ("pool_bits", C.c_int32),
                ("prefix_bits", C.c_int32), ("reps_override", C.c_int32), ("sketch_words", C.c_int32),
                ("cp_draws", C.c_int32), ("max_reps", C.c_int32), ("storage", C.c_int32),
                ("id_offset", C.c_int64)]


class SearchOpts(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("rep_chunk", C.c_int32), ("segment", C.c_int32),
                ("stop_rule", C.c_int32), ("stop_granularity", C.c_int32), ("use_filter", C.c_int32),
                ("filter_eps", C.c_float), ("trace_cap", C.c_int32), ("timing", C.c_int32),
                ("trace_ids", C.c_void_p), ("engine", C.c_int32), ("uniform_chunks", C.c_int32),
                ("rounds", C.c_int32), ("wide", C.c_int32), ("tau_rule", C.c_int32), ("rerank", C.c_int32),
                ("loop_min", C.c_int32), ("loop_max", C.c_int32), ("wide_arrays", C.c_int32),
                ("wide_tiles_min", C.c_int32), ("ext_codes", C.c_void_p), ("ext_reps", C.c_int32),
                ("ext_sketches", C.c_void_p), ("pipelines", C.c_int32)]


class IndexInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("d_pad", C.c_int32), ("family", C.c_int32),
                ("strategy", C.c_int32), ("prefix_bits", C.c_int32), ("reps", C.c_int32), ("ell", C.c_int32),
                ("funcs_per_rep", C.c_int32), ("sketch_words", C.c_int32), ("pool_funcs", C.c_int32),
                ("fht_dim", C.c_int32), ("device", C.c_int32), ("reserved0", C.c_int32),
                ("index_bytes", C.c_uint64), ("scratch_bytes", C.c_uint64), ("seed", C.c_uint64),
                ("id_offset", C.c_int64)]


STATS_DTYPE = np.dtype([("i_stop", np.int32), ("j_stop", np.int32), ("emitted", np.uint32),
                        ("filtered", np.uint32), ("dups", np.uint32), ("evaluated", np.uint32),
                        ("flags", np.uint32), ("probes", np.uint32)])

_lib = None


def lib() -> C.CDLL:
    """The loaded libpfg.so.  Raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(_LIB_PATH)
        P, S = C.c_void_p, C.c_int
        L.pfg_build.restype = S
        L.pfg_build.argtypes = [P, C.c_int64, C.c_int32, C.c_uint64, C.c_int32, C.c_uint64, P, P, P]
        L.pfg_search.restype = S
        L.pfg_search.argtypes = [P, P, C.c_int64, C.c_int32, C.c_float, P, P, P, P, P]
        L.pfg_merge_topk.restype = S
        L.pfg_merge_topk.argtypes = [P, P, C.c_int32, C.c_int64, C.c_int32, P, P, P]
        L.pfg_index_info.restype = S
        L.pfg_index_info.argtypes = [P, P]
        L.pfg_derive_reps.restype = S
        L.pfg_derive_reps.argtypes = [C.c_int64, C.c_int32, C.c_int32, C.c_uint64, P, P, P, P]
        L.pfg_export.restype = S
        L.pfg_export.argtypes = [P, C.c_int32, C.c_int32, P, C.c_uint64]
        L.pfg_hash_queries.restype = S
        L.pfg_hash_queries.argtypes = [P, P, C.c_int64, P, P, P]
        L.pfg_hash_queries_reps.restype = S
        L.pfg_hash_queries_reps.argtypes = [P, P, C.c_int64, C.c_int32, P, P, P]
        L.pfg_stop_tables.restype = S
        L.pfg_stop_tables.argtypes = [P, C.c_float, P, P, P]
        L.pfg_last_timing.restype = S
        L.pfg_last_timing.argtypes = [P, P, P]
        L.pfg_last_phases.restype = S
        L.pfg_last_phases.argtypes = [P, P, C.c_int32]
        L.pfg_free.restype = None
        L.pfg_free.argtypes = [P]
        L.pfg_last_error.restype = C.c_char_p
        L.pfg_last_error.argtypes = []
        L.pfg_abi_version.restype = C.c_int32
        L.pfg_abi_version.argtypes = []
        L.pfg_kernel_timing.restype = S
        L.pfg_kernel_timing.argtypes = [P, C.c_int32, C.c_int32, P, P]
        L.pfg_round_stats.restype = S
        L.pfg_round_stats.argtypes = [P, P, C.c_int32]
        L.pfg_save.restype = S
        L.pfg_save.argtypes = [P, C.c_char_p, P]
        L.pfg_load.restype = S
        L.pfg_load.argtypes = [C.c_char_p, P, P]
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise PfgError(status, lib().pfg_last_error().decode())


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x):
    """(pointer, keepalive, is_cuda) of a torch tensor or numpy array (contiguous)."""
    if x is None:
        return None, None, False
    if _is_torch(x):
        assert x.is_contiguous(), "tensors must be contiguous"
        return C.c_void_p(x.data_ptr()), x, x.is_cuda
    a = np.ascontiguousarray(x)
    return C.c_void_p(a.ctypes.data), a, False


def _stream(x, stream):
    if stream is not None:
        return C.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
    if x is not None and _is_torch(x) and x.is_cuda:
        import torch
        return C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    return C.c_void_p(0)


def _f32(x):
    if _is_torch(x):
        import torch
        return x.to(torch.float32).contiguous()
    return np.ascontiguousarray(x, dtype=np.float32)


def derive_reps(n: int, d: int, family, budget: int, **opts):
    """(L, minimum budget, index bytes) the cost model derives (host only, no GPU)."""
    bo = _build_opts(**opts)
    L, mb, ib = C.c_int32(0), C.c_uint64(0), C.c_uint64(0)
    st = lib().pfg_derive_reps(n, d, _family(family), budget, C.byref(bo), C.byref(L), C.byref(mb), C.byref(ib))
    if st != 0:
        raise PfgError(st, lib().pfg_last_error().decode())
    return L.value, mb.value, ib.value


def _family(f) -> int:
    return FAMILIES[f] if isinstance(f, str) else int(f)


STORAGES = {"f32": 0, "i16": 1}


def _build_opts(strategy=INDEPENDENT, pool_bits=0, prefix_bits=0, reps=0, sketch_words=0, cp_draws=0,
                max_reps=0, id_offset=0, storage="f32") -> BuildOpts:
    o = BuildOpts()
    o.struct_size = C.sizeof(BuildOpts)
    o.storage = STORAGES[storage] if isinstance(storage, str) else int(storage)
    o.strategy = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
    o.pool_bits, o.prefix_bits, o.reps_override = pool_bits, prefix_bits, reps
    o.sketch_words, o.cp_draws, o.max_reps, o.id_offset = sketch_words, cp_draws, max_reps, id_offset
    return o


class Index:
    """An LSH-forest index on one GPU.  `data` [n, d] (torch CUDA/CPU tensor or numpy array).
    memory_budget: bytes (includes data and hash functions); `reps` overrides L."""

    def __init__(self, data, memory_budget: int = 0, family="simhash", seed: int = 1, stream=None, **opts):
        data = _f32(data)
        n, d = data.shape
        self._bo = _build_opts(**opts)
        h = C.c_void_p()
        p, keep, _ = _ptr(data)
        _check(lib().pfg_build(p, n, d, memory_budget, _family(family), seed, C.byref(self._bo),
                               _stream(data, stream), C.byref(h)))
        self._h = h
        self.info = self._info()

    def save(self, path: str, stream=None):
        """write the index to `path` (pfg_save)"""
        _check(lib().pfg_save(self._h, os.fsencode(path), _stream(None, stream)))

    @classmethod
    def load(cls, path: str, stream=None) -> "Index":
        """an index read from a pfg_save file onto the current CUDA device (pfg_load)"""
        self = cls.__new__(cls)
        self._bo = None
        h = C.c_void_p()
        _check(lib().pfg_load(os.fsencode(path), _stream(None, stream), C.byref(h)))
        self._h = h
        self.info = self._info()
        return self

    def _info(self) -> dict:
        inf = IndexInfo()
        _check(lib().pfg_index_info(self._h, C.byref(inf)))
        return {f: getattr(inf, f) for f, _ in IndexInfo._fields_ if not f.startswith("reserved")}

    def __getattr__(self, k):
        info = self.__dict__.get("info")
        if info is not None and k in info:
            return info[k]
        raise AttributeError(k)

    def close(self):
        h = self.__dict__.get("_h")
        if h:
            lib().pfg_free(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _sopts(rep_chunk=DEFAULT_REP_CHUNK, segment=12, stop_rule=0, per_round=False, use_filter=True, eps=0.0,
               trace_cap=0, trace_ptr=None, timing=False, engine=0, uniform_chunks=False, rounds=0,
               wide=0, tau_rule=0, rerank=True, loop_min=0, loop_max=0, wide_arrays=0,
               wide_tiles_min=False, ext_codes=None, ext_sketches=None, pipelines=0) -> SearchOpts:
        o = SearchOpts()
        o.struct_size = C.sizeof(SearchOpts)
        o.rep_chunk, o.segment, o.stop_rule = rep_chunk, segment, stop_rule
        o.stop_granularity = int(per_round)
        o.use_filter = 1 if use_filter else -1
        o.filter_eps = eps
        o.trace_cap = trace_cap
        o.trace_ids = trace_ptr
        o.timing = int(timing)
        o.engine = int(engine)
        o.uniform_chunks = int(uniform_chunks)
        o.rounds = int(rounds)
        o.wide = int(wide)
        o.tau_rule = int(tau_rule)
        o.rerank = 0 if rerank else -1
        o.loop_min, o.loop_max, o.wide_arrays = int(loop_min), int(loop_max), int(wide_arrays)
        o.wide_tiles_min = int(wide_tiles_min)
        o.pipelines = int(pipelines)
        if ext_codes is not None:   # device tensors [nq, reps] uint32 (int32 view) / [nq, M] uint64 (int64 view)
            assert _is_torch(ext_codes) and ext_codes.is_cuda and ext_codes.is_contiguous()
            o.ext_codes, o.ext_reps = ext_codes.data_ptr(), int(ext_codes.shape[1])
        if ext_sketches is not None:
            assert _is_torch(ext_sketches) and ext_sketches.is_cuda and ext_sketches.is_contiguous()
            o.ext_sketches = ext_sketches.data_ptr()
        return o

    def last_timing(self):
        """(prep ms, query-kernel ms, whole-call ms, kernels launched) of the last timed search"""
        ms = (C.c_float * 3)()
        n = C.c_int32(0)
        _check(lib().pfg_last_timing(self._h, ms, C.byref(n)))
        return float(ms[0]), float(ms[1]), float(ms[2]), int(n.value)

    PHASES = ("expand", "scan", "dedupe", "sims", "merge", "fused", "other", "loop")

    def last_phases(self) -> dict:
        """per-phase ms of the query kernels of the last timed search (see pfg_last_phases)"""
        ms = (C.c_float * 8)()
        _check(lib().pfg_last_phases(self._h, ms, 8))
        return {name: float(ms[i]) for i, name in enumerate(self.PHASES)}

    def kernel_timing(self, reset: bool = False):
        """(summed ms, launches) of the bulk k_sims launches of searches with timing=3 (pfg_kernel_timing)"""
        ms, n = C.c_double(0), C.c_int64(0)
        _check(lib().pfg_kernel_timing(self._h, 0, int(reset), C.byref(ms), C.byref(n)))
        return float(ms.value), int(n.value)

    ROUND_STATS = ("sims_rows", "blind_rounds", "loop_rounds", "fused_beside_loop", "fused_after_loop",
                   "wide_arrays", "sims_rows_blind")

    def round_stats(self) -> dict:
        """round-engine counters of the last search (pfg_round_stats)"""
        out = (C.c_uint64 * 7)()
        _check(lib().pfg_round_stats(self._h, out, 7))
        return {name: int(out[i]) for i, name in enumerate(self.ROUND_STATS)}

    def search(self, queries, k: int, recall: float, stats: bool = False, trace_cap: int = 0, out=None,
               stream=None, **sopts):
        """-> ids [nq,k] int64, sims [nq,k] f32 (+ stats structured array, + trace [nq,trace_cap]).
        Outputs live where the queries live (CUDA tensor in -> CUDA tensors out; numpy in -> numpy out),
        unless `out=(ids, sims)` is given."""
        queries = _f32(queries)
        nq = queries.shape[0]
        cuda = _is_torch(queries) and queries.is_cuda
        if out is not None:
            ids, sims = out
        elif cuda:
            import torch
            ids = torch.empty((nq, k), dtype=torch.int64, device=queries.device)
            sims = torch.empty((nq, k), dtype=torch.float32, device=queries.device)
        else:
            ids = np.empty((nq, k), dtype=np.int64)
            sims = np.empty((nq, k), dtype=np.float32)
        st_arr = np.zeros(nq, dtype=STATS_DTYPE) if stats else None
        tr = np.zeros((nq, trace_cap), dtype=np.uint32) if trace_cap > 0 else None
        o = self._sopts(trace_cap=trace_cap, trace_ptr=(tr.ctypes.data if tr is not None else None), **sopts)
        qp, qk, _ = _ptr(queries)
        ip, ik, _ = _ptr(ids)
        sp, sk_, _ = _ptr(sims)
        stp = C.c_void_p(st_arr.ctypes.data) if st_arr is not None else None
        _check(lib().pfg_search(self._h, qp, nq, k, recall, C.byref(o), ip, sp, stp, _stream(queries, stream)))
        res = [ids, sims]
        if stats:
            res.append(st_arr)
        if tr is not None:
            res.append(tr)
        return tuple(res)

    def hash_queries(self, queries):
        """-> codes [nq, L] uint32 (K-bit repetition codes), sketches [nq, M] uint64 (host arrays)"""
        q = np.ascontiguousarray(queries if not _is_torch(queries) else queries.cpu().numpy(), dtype=np.float32)
        nq = q.shape[0]
        codes = np.empty((nq, self.info["reps"]), dtype=np.uint32)
        sk = np.empty((nq, max(1, self.info["sketch_words"])), dtype=np.uint64)
        _check(lib().pfg_hash_queries(self._h, C.c_void_p(q.ctypes.data), nq, C.c_void_p(codes.ctypes.data),
                                      C.c_void_p(sk.ctypes.data), C.c_void_p(0)))
        return codes, sk[:, : self.info["sketch_words"]]

    def hash_queries_reps(self, queries, nreps: int, stream=None):
        """-> codes [nq, nreps] (int32 view of the uint32 codes), sketches [nq, M] (int64 view of the
        uint64 words): CUDA tensors for CUDA queries (pfg_hash_queries_reps)"""
        import torch
        queries = _f32(queries)
        assert _is_torch(queries) and queries.is_cuda
        nq = queries.shape[0]
        codes = torch.empty((nq, nreps), dtype=torch.int32, device=queries.device)
        sk = torch.empty((nq, max(1, self.info["sketch_words"])), dtype=torch.int64, device=queries.device)
        _check(lib().pfg_hash_queries_reps(self._h, C.c_void_p(queries.data_ptr()), nq, nreps,
                                           C.c_void_p(codes.data_ptr()), C.c_void_p(sk.data_ptr()),
                                           _stream(queries, stream)))
        return codes, sk[:, : self.info["sketch_words"]].contiguous()

    def _export(self, what, arg, shape, dtype):
        a = np.empty(shape, dtype=dtype)
        _check(lib().pfg_export(self._h, what, arg, C.c_void_p(a.ctypes.data), a.nbytes))
        return a

    def export_table(self, j: int) -> np.ndarray:
        """[n, 2] uint64: (code << 32 | id, inline sketch word of repetition j's slot)"""
        return self._export(EXPORT_TABLE, j, (self.info["n"], 2), np.uint64)

    def export_prefix(self, j: int) -> np.ndarray:
        return self._export(EXPORT_PREFIX, j, (8193,), np.uint32)

    def export_sketches(self) -> np.ndarray:
        return self._export(EXPORT_SKETCH, 0, (self.info["n"], self.info["sketch_words"]), np.uint64)

    def export_data(self) -> np.ndarray:
        return self._export(EXPORT_DATA, 0, (self.info["n"], self.info["d"]), np.float32)

    def export_data16(self) -> np.ndarray:
        """int16 [n, d] fixed-point rows of a storage="i16" index (R-25)"""
        return self._export(EXPORT_DATA16, 0, (self.info["n"], self.info["d"]), np.int16)

    def export_cp(self) -> np.ndarray:
        return self._export(EXPORT_CP, 0, (self.info["ell"] + 1, 41), np.float64)

    def export_slots(self) -> np.ndarray:
        return self._export(EXPORT_SLOTS, 0, (self.info["reps"],), np.int32)

    def export_pool_sel(self) -> np.ndarray:
        return self._export(EXPORT_POOLSEL, 0, (self.info["reps"], self.info["funcs_per_rep"]), np.int32)

    def stop_tables(self, recall: float, **sopts):
        """-> thr [K, L] f32 (stop iff k-th sim >= thr[i-1, j-1]), tau breakpoints [65] f32"""
        thr = np.empty((self.info["prefix_bits"], self.info["reps"]), dtype=np.float32)
        tau = np.empty(65, dtype=np.float32)
        o = self._sopts(**sopts)
        _check(lib().pfg_stop_tables(self._h, recall, C.byref(o), C.c_void_p(thr.ctypes.data),
                                     C.c_void_p(tau.ctypes.data)))
        return thr, tau


def merge_topk(ids, sims, stream=None):
    """ids [w, nq, k] int64, sims [w, nq, k] f32 CUDA tensors -> merged (ids [nq,k], sims [nq,k])"""
    import torch
    w, nq, k = ids.shape
    oi = torch.empty((nq, k), dtype=torch.int64, device=ids.device)
    os_ = torch.empty((nq, k), dtype=torch.float32, device=ids.device)
    _check(lib().pfg_merge_topk(C.c_void_p(ids.data_ptr()), C.c_void_p(sims.data_ptr()), w, nq, k,
                                C.c_void_p(oi.data_ptr()), C.c_void_p(os_.data_ptr()), _stream(ids, stream)))
    return oi, os_
