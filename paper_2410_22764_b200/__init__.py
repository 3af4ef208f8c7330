"""B200-native DFA minimization engine (arxiv 2410.22764), Python host mirror.

The engine is ``libdfm.so`` (hand-written sm_100a CUDA behind the C-ABI in
``include/dfm.h``).  This module binds that C-ABI with ctypes and mirrors the
reference ``dfamin`` C++ interface for the minimize path — same names,
argument meaning and error behaviour:

==========================  ============================================
reference (proj/include)    here
==========================  ============================================
``Dfa`` core.hpp:24         :class:`Dfa` (numpy SoA rows, delta[a][q])
``Partition`` core.hpp:52   :class:`Partition`
``RunStats``/``MinResult``  :class:`RunStats` / :class:`MinResult`
``Limits`` core.hpp:81      :class:`Limits`
``sort_pr`` min_sort:72     :func:`sort_pr`
``naive_pr`` min_partref    :func:`naive_pr` / :func:`naive_pr_cas`
``expand_alphabet``         :func:`expand_alphabet` (raises CapacityError)
``trans_pr`` min_transpr    :func:`trans_pr`
``trans_minimize``          :func:`trans_minimize`
``run_algorithm`` bench:83  :func:`run_algorithm`
==========================  ============================================

There is no CPU fallback: if ``libdfm.so`` is missing or no sm_100 GPU is
visible, creating an :class:`Engine` raises :class:`EngineUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

__all__ = [
    "Dfa", "Partition", "RunStats", "MinResult", "Limits", "RunStatus", "RacePolicy", "Algo",
    "SortOptions", "SortTrace", "PrOptions", "PrTrace", "TransInspect", "AlgoRunConfig",
    "ExpandedDfa", "CapacityError", "EngineError", "EngineUnavailable", "Engine", "DeviceDfa",
    "sort_pr", "naive_pr", "naive_pr_cas", "expand_alphabet", "trans_pr", "trans_minimize",
    "run_algorithm", "power_levels", "expand_required_bytes", "trans_required_bytes",
    "canonicalize", "partitions_equal", "random_dfa", "default_engine", "lib_path",
]

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    return os.environ.get("DFM_LIB", os.path.join(_HERE, "libdfm.so"))


# ------------------------------------------------------------------ types
class RunStatus(enum.IntEnum):  # core.hpp:58
    ok = 0
    timeout = 1
    capacity_exceeded = 2

    def __str__(self) -> str:
        return {0: "ok", 1: "timeout", 2: "capacity-exceeded"}[int(self)]


class RacePolicy(enum.IntEnum):  # substrate.hpp:24
    arbitrary_winner = 0
    deterministic_min = 1
    deterministic_max = 2


class Algo(enum.IntEnum):  # bench.hpp:23
    trans = 0
    naive = 1
    naive_cas = 2
    sort = 3
    transpr = 4
    oracle = 5


class EngineError(RuntimeError):
    """Infrastructure fault inside libdfm (CUDA error, bad argument, OOM)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libdfm error {code}: {msg}")
        self.code = code


class EngineUnavailable(EngineError):
    """libdfm.so missing or no sm_100 device: the engine never falls back to the CPU."""


class CapacityError(RuntimeError):  # core.hpp:93-101
    def __init__(self, what: str, required_bytes: int):
        super().__init__(what)
        self._required = int(required_bytes)

    def required_bytes(self) -> int:
        return self._required


@dataclass
class Dfa:  # core.hpp:24-33
    num_states: int
    alphabet_size: int
    delta: np.ndarray  # (alphabet_size, num_states) uint32, row a = successors on letter a
    accepting: np.ndarray  # (num_states,) uint8
    initial: int = 0

    def __post_init__(self):
        self.delta = np.ascontiguousarray(
            np.asarray(self.delta, dtype=np.uint32).reshape(self.alphabet_size, self.num_states))
        self.accepting = np.ascontiguousarray(np.asarray(self.accepting, dtype=np.uint8))

    @classmethod
    def from_rows(cls, rows: Sequence[Sequence[int]], accepting: Sequence[int],
                  initial: int = 0) -> "Dfa":
        acc = np.asarray(accepting, dtype=np.uint8)
        delta = np.asarray(rows, dtype=np.uint32).reshape(len(rows), acc.size)
        return cls(int(acc.size), len(rows), delta, acc, initial)

    def is_accepting(self, q: int) -> bool:
        return bool(self.accepting[q])


@dataclass
class Partition:  # core.hpp:52-56
    block: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint32))
    num_blocks: int = 0


@dataclass
class RunStats:  # core.hpp:71-77
    iterations: int = 0
    closure_steps: int = 0
    elapsed_ms: float = 0.0
    peak_memory_estimate: int = 0
    status: RunStatus = RunStatus.ok
    executed_passes: int = 0  # passes whose kernels ran (<= iterations; not in the reference)


@dataclass
class MinResult:  # core.hpp:87-90
    partition: Partition
    stats: RunStats


@dataclass
class Limits:  # core.hpp:81-84
    max_memory_bytes: int = 16 << 30
    timeout_ms: int = 300_000


@dataclass
class SortTrace:  # min_sort.hpp:21-24
    partitions: list = field(default_factory=list)
    block_counts: list = field(default_factory=list)


@dataclass
class SortOptions:  # min_sort.hpp:26-29
    timeout_ms: int = 300_000
    trace: Optional[SortTrace] = None


@dataclass
class PrTrace:  # min_partref.hpp:21-24
    leader_arrays: list = field(default_factory=list)
    partitions: list = field(default_factory=list)


@dataclass
class PrOptions:  # min_partref.hpp:26-30
    policy: RacePolicy = RacePolicy.arbitrary_winner
    timeout_ms: int = 300_000
    trace: Optional[PrTrace] = None


@dataclass
class TransInspect:  # min_trans.hpp:41-44
    apart: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint8))
    apart_popcounts: list = field(default_factory=list)


@dataclass
class AlgoRunConfig:  # bench.hpp:78-81
    policy: RacePolicy = RacePolicy.arbitrary_winner
    limits: Limits = field(default_factory=Limits)


@dataclass
class ExpandedDfa:  # min_transpr.hpp:31-53
    num_states: int
    base_alphabet: int
    levels: int
    delta: np.ndarray  # (levels*base_alphabet, n)
    accepting: np.ndarray
    initial: int = 0

    def row(self, letter: int, level: int) -> np.ndarray:
        return self.delta[level * self.base_alphabet + letter]

    def as_dfa(self) -> Dfa:
        return Dfa(self.num_states, self.delta.shape[0], self.delta.copy(), self.accepting.copy(),
                   self.initial)


# ------------------------------------------------------------------ ctypes layer
class _CDfa(C.Structure):
    _fields_ = [("num_states", C.c_uint32), ("alphabet_size", C.c_uint32),
                ("delta", C.POINTER(C.c_void_p)), ("accepting", C.c_void_p),
                ("initial", C.c_uint32)]


class _CStats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("closure_steps", C.c_uint64),
                ("elapsed_ms", C.c_double), ("peak_memory_estimate", C.c_uint64),
                ("status", C.c_int32), ("executed_passes", C.c_uint64)]


class _CLimits(C.Structure):
    _fields_ = [("max_memory_bytes", C.c_uint64), ("timeout_ms", C.c_int64)]


_PASS_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32), C.c_uint32,
                       C.c_uint32)


class _CTrace(C.Structure):
    _fields_ = [("on_pass", _PASS_FN), ("user", C.c_void_p)]


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise EngineUnavailable(5, f"{path} not built (run __graft_entry__.build() or `make`)")
    lib = C.CDLL(path)
    vp, u32, u64, i32, i64 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32, C.c_int64
    sig = {
        "dfm_version": (C.c_char_p, []),
        "dfm_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "dfm_ctx_destroy": (None, [vp]),
        "dfm_last_error": (C.c_char_p, [vp]),
        "dfm_ctx_set_stream": (C.c_int, [vp, vp]),
        "dfm_ctx_set_profiling": (C.c_int, [vp, C.c_int]),
        "dfm_ctx_set_sortpr_engine": (C.c_int, [vp, C.c_int]),
        "dfm_ctx_set_trans_engine": (C.c_int, [vp, C.c_int]),
        "dfm_profile_get": (C.c_int, [vp, C.c_char_p, C.POINTER(u64), C.POINTER(C.c_double),
                                      C.POINTER(u64)]),
        "dfm_kernel_launches": (u64, []),
        "dfm_profile_names": (C.c_char_p, [vp]),
        "dfm_profile_reset": (C.c_int, [vp]),
        "dfm_ctx_device_bytes": (u64, [vp]),
        "dfm_sort_pr": (C.c_int, [vp, vp, i64, vp, vp, C.POINTER(u32), C.POINTER(_CStats)]),
        "dfm_naive_pr": (C.c_int, [vp, vp, i32, i64, vp, vp, C.POINTER(u32), C.POINTER(_CStats)]),
        "dfm_naive_pr_cas": (C.c_int, [vp, vp, i64, vp, vp, C.POINTER(u32), C.POINTER(_CStats)]),
        "dfm_power_levels": (u32, [u32]),
        "dfm_expand_required_bytes": (u64, [u32, u32]),
        "dfm_expand_alphabet": (C.c_int, [vp, vp, u64, vp, C.POINTER(u32), C.POINTER(u64)]),
        "dfm_trans_pr": (C.c_int, [vp, vp, i32, C.POINTER(_CLimits), vp, C.POINTER(u32),
                                   C.POINTER(_CStats)]),
        "dfm_trans_required_bytes": (u64, [u64]),
        "dfm_trans_minimize": (C.c_int, [vp, vp, C.POINTER(_CLimits), vp, vp, u32, vp,
                                         C.POINTER(u32), C.POINTER(_CStats)]),
        "dfm_run_algorithm": (C.c_int, [vp, i32, vp, i32, C.POINTER(_CLimits), vp,
                                        C.POINTER(u32), C.POINTER(_CStats)]),
        "dfm_ddfa_upload": (C.c_int, [vp, vp, C.POINTER(vp)]),
        "dfm_ddfa_random": (C.c_int, [vp, u32, u32, u64, C.c_double, C.POINTER(vp)]),
        "dfm_ddfa_download": (C.c_int, [vp, vp, vp, vp]),
        "dfm_ddfa_shape": (C.c_int, [vp, C.POINTER(u32), C.POINTER(u32)]),
        "dfm_ddfa_free": (None, [vp]),
        "dfm_run_algorithm_dev": (C.c_int, [vp, i32, vp, i32, C.POINTER(_CLimits), vp,
                                            C.POINTER(u32), C.POINTER(_CStats)]),
        "dfm_gen_random_dfa": (C.c_int, [u32, u32, u64, C.c_double, vp, vp]),
        "dfm_quotient": (C.c_int, [vp, vp, vp, u32, vp, vp, C.POINTER(u32)]),
        "dfm_ddfa_quotient": (C.c_int, [vp, vp, vp, u32, C.POINTER(vp)]),
        "dfm_remove_unreachable": (C.c_int, [vp, vp, C.POINTER(u32), vp, vp, C.POINTER(u32)]),
        "dfm_ddfa_remove_unreachable": (C.c_int, [vp, vp, C.POINTER(vp)]),
        "dfm_ddfa_initial": (C.c_int, [vp, C.POINTER(u32)]),
        "dfm_write_dfa_bin": (C.c_int, [C.c_char_p, vp]),
        "dfm_ddfa_load_bin": (C.c_int, [vp, C.c_char_p, C.POINTER(vp)]),
        "dfm_ddfa_save_bin": (C.c_int, [vp, vp, C.c_char_p]),
        "dfm_lts_parse": (C.c_int, [C.c_char_p, u64, C.POINTER(vp), C.POINTER(u64), C.c_char_p,
                                    u32]),
        "dfm_lts_info": (C.c_int, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32),
                                   C.POINTER(u64)]),
        "dfm_lts_label": (C.c_int, [vp, u32, C.POINTER(C.c_void_p), C.POINTER(u64)]),
        "dfm_lts_transitions": (C.c_int, [vp, vp, vp, vp]),
        "dfm_lts_free": (None, [vp]),
        "dfm_lts_build": (C.c_int, [u32, u32, u32, vp, vp, u64, vp, vp, vp, C.POINTER(vp)]),
        "dfm_determinize": (C.c_int, [vp, u64, C.POINTER(vp), C.POINTER(u64)]),
        "dfm_pdfa_shape": (C.c_int, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
        "dfm_pdfa_rows": (C.c_int, [vp, vp]),
        "dfm_complete": (C.c_int, [vp, C.POINTER(u32), vp, vp]),
        "dfm_pdfa_free": (None, [vp]),
        "dfm_pdfa_build": (C.c_int, [u32, u32, u32, vp, C.POINTER(vp)]),
        "dfm_nccl_get_unique_id": (C.c_int, [vp]),
        "dfm_ctx_create_sharded": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, C.POINTER(vp)]),
        "dfm_ctx_create_sharded_local": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p,
                                                   C.POINTER(vp)]),
        "dfm_ctx_shard_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                         C.POINTER(C.c_char_p)]),
        "dfm_shard_bounds": (None, [u64, C.c_int, C.c_int, C.POINTER(u64), C.POINTER(u64)]),
        "dfm_sort_pr_sharded": (C.c_int, [vp, u64, vp, C.c_int, vp, C.POINTER(u32), i64,
                                          C.POINTER(_CStats)]),
        "dfm_sort_pr_sharded_dev": (C.c_int, [vp, u64, u32, u32, vp, vp, vp, C.POINTER(u32), i64,
                                              C.POINTER(_CStats)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# pure host helpers that need no GPU
def power_levels(n: int) -> int:  # min_transpr.hpp:21-23
    return int(n).bit_length()


def expand_required_bytes(n: int, k: int) -> int:  # min_transpr.hpp:25-27
    return power_levels(n) * k * n * 4


def trans_required_bytes(n: int) -> int:  # min_trans.hpp:24-27 (exact, unbounded int)
    return (n ** 4 + 7) // 8


def canonicalize(raw) -> Partition:
    """Host helper: first-occurrence relabel (core.hpp:123-136)."""
    raw = np.asarray(raw, dtype=np.uint32)
    if raw.size == 0:
        return Partition(np.empty(0, np.uint32), 0)
    _, first_idx, inverse = np.unique(raw, return_index=True, return_inverse=True)
    order = np.argsort(first_idx, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    return Partition(rank[inverse].astype(np.uint32), int(order.size))


def partitions_equal(p: Partition, q: Partition) -> bool:  # core.hpp:144-149
    if len(p.block) != len(q.block):
        raise ValueError("partitions cover different state counts")
    return bool(np.array_equal(canonicalize(p.block).block, canonicalize(q.block).block))


def random_dfa(n: int, k: int, seed: int, accept_prob: float = 0.5) -> Dfa:
    """generators.hpp:130-145, bit-exact, multi-threaded host generation (libdfm)."""
    if n < 1 or k < 1:
        raise ValueError("random_dfa needs n >= 1 and k >= 1")
    lib = _load()
    delta = np.empty((k, n), np.uint32)
    acc = np.empty(n, np.uint8)
    rc = lib.dfm_gen_random_dfa(n, k, seed & (2 ** 64 - 1), accept_prob, delta.ctypes.data,
                                acc.ctypes.data)
    if rc != 0:
        raise EngineError(rc, "dfm_gen_random_dfa failed")
    return Dfa(n, k, delta, acc, 0)


# ------------------------------------------------------------------ engine
class Engine:
    """One libdfm context (device, stream, scratch arena)."""

    def __init__(self, device: int = 0):
        lib = _load()
        self.lib = lib
        h = C.c_void_p()
        rc = lib.dfm_ctx_create(device, C.byref(h))
        if rc != 0:
            msg = (lib.dfm_last_error(None) or b"").decode()
            raise EngineUnavailable(rc, msg)
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self.lib.dfm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing
    def _check(self, rc: int) -> None:
        if rc != 0:
            msg = (self.lib.dfm_last_error(self.handle) or b"").decode()
            raise EngineError(rc, msg)

    @staticmethod
    def _cdfa(d: Dfa):
        rows = (C.c_void_p * max(d.alphabet_size, 1))()
        for a in range(d.alphabet_size):
            rows[a] = d.delta[a].ctypes.data
        cd = _CDfa(d.num_states, d.alphabet_size, C.cast(rows, C.POINTER(C.c_void_p)),
                   d.accepting.ctypes.data, d.initial)
        return cd, rows

    @staticmethod
    def _stats(st: _CStats) -> RunStats:
        return RunStats(int(st.iterations), int(st.closure_steps), float(st.elapsed_ms),
                        int(st.peak_memory_estimate), RunStatus(st.status),
                        int(st.executed_passes))

    def _result(self, block, nb, st) -> MinResult:
        stats = self._stats(st)
        if stats.status != RunStatus.ok:
            return MinResult(Partition(), stats)
        return MinResult(Partition(block, int(nb.value)), stats)

    @staticmethod
    def _make_trace(cb: Callable):
        fn = _PASS_FN(lambda user, it, blk, n, count: cb(
            int(it), np.ctypeslib.as_array(blk, shape=(n,)).copy(), int(count)))
        return _CTrace(fn, None), fn

    # -- reference API
    def sort_pr(self, d: Dfa, opt=None, out: Optional[np.ndarray] = None) -> MinResult:
        """`out`: optional caller-owned uint32[n] result buffer (pass pinned memory for a
        full-bandwidth device-to-host copy)."""
        if opt is None:
            opt = SortOptions()
        elif isinstance(opt, int):
            opt = SortOptions(timeout_ms=opt)
        cd, keep = self._cdfa(d)
        block = out if out is not None else np.empty(d.num_states, np.uint32)
        assert block.dtype == np.uint32 and block.size == d.num_states and block.flags.c_contiguous
        nb = C.c_uint32(0)
        st = _CStats()
        tr = None
        if opt.trace is not None:
            t = opt.trace

            def on_pass(it, raw, count):
                t.partitions.append(canonicalize(raw))
                t.block_counts.append(count)
            tr, fn = self._make_trace(on_pass)
        self._check(self.lib.dfm_sort_pr(self.handle, C.byref(cd), opt.timeout_ms,
                                         C.byref(tr) if tr is not None else None,
                                         block.ctypes.data, C.byref(nb), C.byref(st)))
        return self._result(block, nb, st)

    def naive_pr(self, d: Dfa, opt=None, timeout_ms: int = 300_000) -> MinResult:
        if opt is None:
            opt = PrOptions()
        elif not isinstance(opt, PrOptions):
            opt = PrOptions(policy=RacePolicy(opt), timeout_ms=timeout_ms)
        return self._leader(d, opt, fused=False)

    def naive_pr_cas(self, d: Dfa, timeout_ms: int = 300_000,
                     trace: Optional[PrTrace] = None) -> MinResult:
        return self._leader(d, PrOptions(timeout_ms=timeout_ms, trace=trace), fused=True)

    def _leader(self, d: Dfa, opt: PrOptions, fused: bool) -> MinResult:
        cd, keep = self._cdfa(d)
        block = np.empty(d.num_states, np.uint32)
        nb = C.c_uint32(0)
        st = _CStats()
        tr = None
        if opt.trace is not None:
            t = opt.trace

            def on_pass(it, raw, count):
                t.leader_arrays.append(raw)
                t.partitions.append(canonicalize(raw))
            tr, fn = self._make_trace(on_pass)
        trp = C.byref(tr) if tr is not None else None
        if fused:
            rc = self.lib.dfm_naive_pr_cas(self.handle, C.byref(cd), opt.timeout_ms, trp,
                                           block.ctypes.data, C.byref(nb), C.byref(st))
        else:
            rc = self.lib.dfm_naive_pr(self.handle, C.byref(cd), int(opt.policy), opt.timeout_ms,
                                       trp, block.ctypes.data, C.byref(nb), C.byref(st))
        self._check(rc)
        return self._result(block, nb, st)

    def expand_alphabet(self, d: Dfa, limits: Optional[Limits] = None) -> ExpandedDfa:
        limits = limits or Limits()
        cd, keep = self._cdfa(d)
        levels = power_levels(d.num_states)
        req = expand_required_bytes(d.num_states, d.alphabet_size)
        rows = np.empty((levels * d.alphabet_size, d.num_states), np.uint32) \
            if req <= limits.max_memory_bytes else None
        lv = C.c_uint32(0)
        rq = C.c_uint64(0)
        rc = self.lib.dfm_expand_alphabet(self.handle, C.byref(cd), limits.max_memory_bytes,
                                          rows.ctypes.data if rows is not None else None,
                                          C.byref(lv), C.byref(rq))
        if rc == 3:
            raise CapacityError(
                f"alphabet expansion needs {rq.value} bytes, limit is {limits.max_memory_bytes}",
                rq.value)
        self._check(rc)
        return ExpandedDfa(d.num_states, d.alphabet_size, int(lv.value), rows,
                           d.accepting.copy(), d.initial)

    def trans_pr(self, d: Dfa, opt=None, limits: Optional[Limits] = None,
                 timeout_ms: int = 300_000) -> MinResult:
        if opt is None:
            opt = PrOptions()
        elif not isinstance(opt, PrOptions):  # trans_pr(d, policy, timeout, limits), :114
            opt = PrOptions(policy=RacePolicy(opt), timeout_ms=timeout_ms)
            limits = Limits((limits or Limits()).max_memory_bytes, timeout_ms)
        limits = limits or Limits()
        lim = _CLimits(limits.max_memory_bytes, opt.timeout_ms)
        cd, keep = self._cdfa(d)
        block = np.empty(d.num_states, np.uint32)
        nb = C.c_uint32(0)
        st = _CStats()
        self._check(self.lib.dfm_trans_pr(self.handle, C.byref(cd), int(opt.policy), C.byref(lim),
                                          block.ctypes.data, C.byref(nb), C.byref(st)))
        return self._result(block, nb, st)

    def trans_minimize(self, d: Dfa, limits: Optional[Limits] = None,
                       inspect: Optional[TransInspect] = None) -> MinResult:
        limits = limits or Limits()
        lim = _CLimits(limits.max_memory_bytes, limits.timeout_ms)
        cd, keep = self._cdfa(d)
        n = d.num_states
        block = np.empty(n, np.uint32)
        nb = C.c_uint32(0)
        st = _CStats()
        apart = np.empty(n * n, np.uint8) if inspect is not None else None
        pops = np.zeros(4096, np.uint64) if inspect is not None else None
        self._check(self.lib.dfm_trans_minimize(
            self.handle, C.byref(cd), C.byref(lim),
            apart.ctypes.data if apart is not None else None,
            pops.ctypes.data if pops is not None else None, 4096, block.ctypes.data,
            C.byref(nb), C.byref(st)))
        r = self._result(block, nb, st)
        if inspect is not None and r.stats.status == RunStatus.ok:
            inspect.apart = apart
            inspect.apart_popcounts = [int(x) for x in pops[: r.stats.iterations]]
        return r

    def run_algorithm(self, algo: Algo, d: Dfa, cfg: Optional[AlgoRunConfig] = None) -> MinResult:
        cfg = cfg or AlgoRunConfig()
        lim = _CLimits(cfg.limits.max_memory_bytes, cfg.limits.timeout_ms)
        cd, keep = self._cdfa(d)
        block = np.empty(d.num_states, np.uint32)
        nb = C.c_uint32(0)
        st = _CStats()
        self._check(self.lib.dfm_run_algorithm(self.handle, int(algo), C.byref(cd),
                                               int(cfg.policy), C.byref(lim), block.ctypes.data,
                                               C.byref(nb), C.byref(st)))
        return self._result(block, nb, st)

    # -- post-/pre-processing (core.hpp:152-187, 256-290)
    def quotient(self, d: Dfa, p: Partition) -> Dfa:
        """core.hpp:256-290 on the GPU.  Raises ValueError with the reference's
        std::invalid_argument message for a non-canonical or inconsistent partition."""
        block = np.ascontiguousarray(p.block, dtype=np.uint32)
        if block.size != d.num_states:
            raise ValueError("partition covers a different state count")
        nb = int(p.num_blocks)
        cd, keep = self._cdfa(d)
        delta = np.empty((d.alphabet_size, nb), np.uint32)
        acc = np.empty(nb, np.uint8)
        init = C.c_uint32(0)
        rc = self.lib.dfm_quotient(self.handle, C.byref(cd), block.ctypes.data, nb,
                                   delta.ctypes.data, acc.ctypes.data, C.byref(init))
        if rc == 1:  # DFM_ERR_INVALID: the reference throws std::invalid_argument
            raise ValueError((self.lib.dfm_last_error(self.handle) or b"").decode())
        self._check(rc)
        return Dfa(nb, d.alphabet_size, delta, acc, int(init.value))

    def remove_unreachable(self, d: Dfa) -> Dfa:
        """core.hpp:152-187 on the GPU (breadth-first search + dense renumbering)."""
        cd, keep = self._cdfa(d)
        delta = np.empty(max(d.alphabet_size * d.num_states, 1), np.uint32)
        acc = np.empty(d.num_states, np.uint8)
        kept, init = C.c_uint32(0), C.c_uint32(0)
        self._check(self.lib.dfm_remove_unreachable(self.handle, C.byref(cd), C.byref(kept),
                                                    delta.ctypes.data, acc.ctypes.data,
                                                    C.byref(init)))
        n = int(kept.value)
        rows = delta[: d.alphabet_size * n].reshape(d.alphabet_size, n).copy()
        return Dfa(n, d.alphabet_size, rows, acc[:n].copy(), int(init.value))

    # -- bulk input path (binary DFA files, csrc/io.cu)
    def load_bin(self, path: str) -> "DeviceDfa":
        h = C.c_void_p()
        self._check(self.lib.dfm_ddfa_load_bin(self.handle, os.fsencode(path), C.byref(h)))
        n, k = C.c_uint32(0), C.c_uint32(0)
        self._check(self.lib.dfm_ddfa_shape(h, C.byref(n), C.byref(k)))
        return DeviceDfa(self, h, int(n.value), int(k.value))

    # -- device-resident path (bench "value", sharded driver)
    def upload(self, d: Dfa) -> "DeviceDfa":
        cd, keep = self._cdfa(d)
        h = C.c_void_p()
        self._check(self.lib.dfm_ddfa_upload(self.handle, C.byref(cd), C.byref(h)))
        return DeviceDfa(self, h, d.num_states, d.alphabet_size)

    def random_dfa_device(self, n: int, k: int, seed: int, accept_prob: float = 0.5) -> "DeviceDfa":
        h = C.c_void_p()
        self._check(self.lib.dfm_ddfa_random(self.handle, n, k, seed & (2 ** 64 - 1), accept_prob,
                                             C.byref(h)))
        return DeviceDfa(self, h, n, k)

    def run_device(self, algo: Algo, dd: "DeviceDfa", cfg: Optional[AlgoRunConfig] = None,
                   block_out_ptr: Optional[int] = None):
        cfg = cfg or AlgoRunConfig()
        lim = _CLimits(cfg.limits.max_memory_bytes, cfg.limits.timeout_ms)
        nb = C.c_uint32(0)
        st = _CStats()
        self._check(self.lib.dfm_run_algorithm_dev(self.handle, int(algo), dd.handle,
                                                   int(cfg.policy), C.byref(lim),
                                                   block_out_ptr, C.byref(nb), C.byref(st)))
        return int(nb.value), self._stats(st)

    # -- profiling
    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """Run on a caller stream (e.g. torch.cuda.current_stream().cuda_stream).  torch's
        default stream has handle 0, which is passed as cudaStreamLegacy (0x1); None
        restores the engine's own stream."""
        if stream_ptr is None:
            ptr = None
        else:
            ptr = int(stream_ptr) or 1  # 0 = legacy default stream -> cudaStreamLegacy
        self._check(self.lib.dfm_ctx_set_stream(self.handle, ptr))

    def set_sortpr_engine(self, engine: str) -> None:
        """'hash' (default) or 'radix' (the paper's sort); same results."""
        self._check(self.lib.dfm_ctx_set_sortpr_engine(
            self.handle, {"hash": 0, "radix": 1}[engine]))

    def set_trans_engine(self, engine: str) -> None:
        """Cho–Huynh squaring: 'auto' (default), 'bit' (CUDA cores) or 'tensor' (tcgen05)."""
        self._check(self.lib.dfm_ctx_set_trans_engine(
            self.handle, {"auto": 0, "bit": 1, "tensor": 2}[engine]))

    def set_profiling(self, on: bool) -> None:
        self._check(self.lib.dfm_ctx_set_profiling(self.handle, int(bool(on))))

    def profile(self) -> dict:
        """{family: (timed scopes, total ms, total algorithmic bytes)}"""
        names = (self.lib.dfm_profile_names(self.handle) or b"").decode()
        out = {}
        for name in filter(None, names.split(",")):
            launches = C.c_uint64(0)
            ms = C.c_double(0)
            nbytes = C.c_uint64(0)
            if self.lib.dfm_profile_get(self.handle, name.encode(), C.byref(launches),
                                        C.byref(ms), C.byref(nbytes)) == 0:
                out[name] = (int(launches.value), float(ms.value), int(nbytes.value))
        return out

    def kernel_launches(self) -> int:
        return int(self.lib.dfm_kernel_launches())

    def profile_reset(self) -> None:
        self._check(self.lib.dfm_profile_reset(self.handle))

    def device_bytes(self) -> int:
        return int(self.lib.dfm_ctx_device_bytes(self.handle))


class DeviceDfa:
    """A DFA resident in HBM (SoA rows, [k][n] u32 + n u8)."""

    def __init__(self, eng: Engine, handle: C.c_void_p, n: int, k: int):
        self.engine, self.handle, self.num_states, self.alphabet_size = eng, handle, n, k

    def download(self) -> Dfa:
        delta = np.empty((self.alphabet_size, self.num_states), np.uint32)
        acc = np.empty(self.num_states, np.uint8)
        self.engine._check(self.engine.lib.dfm_ddfa_download(self.engine.handle, self.handle,
                                                             delta.ctypes.data, acc.ctypes.data))
        init = C.c_uint32(0)
        self.engine._check(self.engine.lib.dfm_ddfa_initial(self.handle, C.byref(init)))
        return Dfa(self.num_states, self.alphabet_size, delta, acc, int(init.value))

    def quotient(self, block_dev_ptr: int, num_blocks: int) -> "DeviceDfa":
        """Device quotient by canonical device labels (run_device(..., block_out_ptr))."""
        h = C.c_void_p()
        e = self.engine
        rc = e.lib.dfm_ddfa_quotient(e.handle, self.handle, block_dev_ptr, num_blocks, C.byref(h))
        if rc == 1:
            raise ValueError((e.lib.dfm_last_error(e.handle) or b"").decode())
        e._check(rc)
        return DeviceDfa(e, h, num_blocks, self.alphabet_size)

    def save_bin(self, path: str) -> None:
        e = self.engine
        e._check(e.lib.dfm_ddfa_save_bin(e.handle, self.handle, os.fsencode(path)))

    def remove_unreachable(self) -> "DeviceDfa":
        h = C.c_void_p()
        e = self.engine
        e._check(e.lib.dfm_ddfa_remove_unreachable(e.handle, self.handle, C.byref(h)))
        n = C.c_uint32(0)
        k = C.c_uint32(0)
        e._check(e.lib.dfm_ddfa_shape(h, C.byref(n), C.byref(k)))
        return DeviceDfa(e, h, int(n.value), int(k.value))

    def free(self) -> None:
        if self.handle:
            self.engine.lib.dfm_ddfa_free(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass


_default: Optional[Engine] = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(int(os.environ.get("DFM_DEVICE", "0")))
    return _default


# module-level mirrors of the reference free functions
def sort_pr(d: Dfa, opt=None) -> MinResult:
    return default_engine().sort_pr(d, opt)


def naive_pr(d: Dfa, opt=None, timeout_ms: int = 300_000) -> MinResult:
    return default_engine().naive_pr(d, opt, timeout_ms)


def naive_pr_cas(d: Dfa, timeout_ms: int = 300_000, trace: Optional[PrTrace] = None) -> MinResult:
    return default_engine().naive_pr_cas(d, timeout_ms, trace)


def expand_alphabet(d: Dfa, limits: Optional[Limits] = None) -> ExpandedDfa:
    return default_engine().expand_alphabet(d, limits)


def trans_pr(d: Dfa, opt=None, limits: Optional[Limits] = None, timeout_ms: int = 300_000):
    return default_engine().trans_pr(d, opt, limits, timeout_ms)


def trans_minimize(d: Dfa, limits: Optional[Limits] = None,
                   inspect: Optional[TransInspect] = None) -> MinResult:
    return default_engine().trans_minimize(d, limits, inspect)


def run_algorithm(algo: Algo, d: Dfa, cfg: Optional[AlgoRunConfig] = None) -> MinResult:
    return default_engine().run_algorithm(algo, d, cfg)


def quotient(d: Dfa, p: Partition) -> Dfa:  # core.hpp:256
    return default_engine().quotient(d, p)


def remove_unreachable(d: Dfa) -> Dfa:  # core.hpp:152
    return default_engine().remove_unreachable(d)


_BIN_MAGIC = b"DFMBIN01"


def write_dfa_bin(path: str, d: Dfa) -> None:
    """Binary DFA file (include/dfm.h, dfm_write_dfa_bin) — host only, no GPU needed."""
    lib = _load()
    cd, keep = Engine._cdfa(d)
    rc = lib.dfm_write_dfa_bin(os.fsencode(path), C.byref(cd))
    if rc != 0:
        raise EngineError(rc, f"cannot write {path}")


def read_dfa_bin(path: str) -> Dfa:
    """Host reader of the binary format (memory-mapped, zero-copy rows)."""
    raw = np.memmap(path, dtype=np.uint8, mode="r")
    if bytes(raw[:8]) != _BIN_MAGIC:
        raise ValueError(f"{path}: not a DFMBIN01 file")
    n, k, initial, _ = np.frombuffer(raw[8:24].tobytes(), dtype="<u4")
    n, k = int(n), int(k)
    acc = np.array(raw[24:24 + n])
    off = 24 + ((n + 3) & ~3)
    delta = np.frombuffer(raw[off:off + 4 * n * k].tobytes(), dtype="<u4").reshape(k, n).copy()
    return Dfa(n, k, delta, acc, int(initial))


# ---------------------------------------------------------------- LTS ingestion (host)
# ingest.hpp:130-284 behind libdfm's dfm_lts_* / dfm_determinize / dfm_complete (no GPU
# needed): the same automaton, numbering and errors as the reference.
class ParseError(ValueError):  # ingest.hpp:20-28
    def __init__(self, line: int, what: str):
        super().__init__(what)
        self._line = int(line)

    def line(self) -> int:
        return self._line


class SubsetBudgetExceeded(RuntimeError):  # ingest.hpp:31-39
    def __init__(self, budget: int):
        super().__init__(f"subset construction exceeded {budget} states")
        self._budget = int(budget)

    def budget(self) -> int:
        return self._budget


K_MISSING = 0xFFFFFFFF  # PartialDfa::kMissing


@dataclass
class Lts:  # core.hpp:36-47 (transitions as three aligned arrays)
    num_states: int
    initial: int
    labels: list
    src: np.ndarray
    label: np.ndarray
    dst: np.ndarray

    @property
    def transitions(self):
        return list(zip(self.src.tolist(), self.label.tolist(), self.dst.tolist()))


@dataclass
class PartialDfa:  # ingest.hpp:177-184
    num_states: int
    alphabet_size: int
    delta: np.ndarray  # (alphabet_size, num_states) uint32, K_MISSING where absent
    initial: int = 0
    kMissing = K_MISSING


def _lts_handle(lts: Lts):
    lib = _load()
    h = C.c_void_p()
    enc = [x.encode() for x in lts.labels]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    lens = (C.c_uint64 * max(len(enc), 1))(*[len(x) for x in enc])
    src = np.ascontiguousarray(lts.src, dtype=np.uint32)
    lab = np.ascontiguousarray(lts.label, dtype=np.uint32)
    dst = np.ascontiguousarray(lts.dst, dtype=np.uint32)
    rc = lib.dfm_lts_build(lts.num_states, lts.initial, len(enc), C.cast(arr, C.c_void_p),
                           C.cast(lens, C.c_void_p), src.size, src.ctypes.data, lab.ctypes.data,
                           dst.ctypes.data, C.byref(h))
    if rc != 0:
        raise ValueError("malformed LTS")
    return h


def parse_lts(text) -> Lts:
    """ingest.hpp:130-175; raises ParseError(line) like the reference."""
    lib = _load()
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    line = C.c_uint64(0)
    err = C.create_string_buffer(512)
    rc = lib.dfm_lts_parse(data, len(data), C.byref(h), C.byref(line), err, 512)
    if rc == 6:
        msg = err.value.decode()
        raise ParseError(int(line.value), msg)
    if rc != 0:
        raise EngineError(rc, "dfm_lts_parse failed")
    try:
        n, init, nl, m = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        lib.dfm_lts_info(h, C.byref(n), C.byref(init), C.byref(nl), C.byref(m))
        labels = []
        for i in range(nl.value):
            p, ln = C.c_void_p(), C.c_uint64()
            lib.dfm_lts_label(h, i, C.byref(p), C.byref(ln))
            labels.append(C.string_at(p, ln.value).decode())
        src = np.empty(m.value, np.uint32)
        lab = np.empty(m.value, np.uint32)
        dst = np.empty(m.value, np.uint32)
        lib.dfm_lts_transitions(h, src.ctypes.data, lab.ctypes.data, dst.ctypes.data)
        return Lts(int(n.value), int(init.value), labels, src, lab, dst)
    finally:
        lib.dfm_lts_free(h)


def determinize(lts: Lts, max_subset_states: int = 1 << 22) -> PartialDfa:
    """ingest.hpp:187-245 (subset construction, BFS numbering); raises
    SubsetBudgetExceeded like the reference."""
    lib = _load()
    h = _lts_handle(lts)
    try:
        p = C.c_void_p()
        budget = C.c_uint64(0)
        rc = lib.dfm_determinize(h, max_subset_states, C.byref(p), C.byref(budget))
        if rc == 7:
            raise SubsetBudgetExceeded(int(budget.value))
        if rc != 0:
            raise EngineError(rc, "dfm_determinize failed")
        try:
            n, k, init = C.c_uint32(), C.c_uint32(), C.c_uint32()
            lib.dfm_pdfa_shape(p, C.byref(n), C.byref(k), C.byref(init))
            delta = np.empty((k.value, n.value), np.uint32)
            lib.dfm_pdfa_rows(p, delta.ctypes.data)
            return PartialDfa(int(n.value), int(k.value), delta, int(init.value))
        finally:
            lib.dfm_pdfa_free(p)
    finally:
        lib.dfm_lts_free(h)


def complete(p: PartialDfa) -> Dfa:
    """ingest.hpp:253-284: one rejecting sink appended iff a transition is missing."""
    lib = _load()
    h = C.c_void_p()
    delta = np.ascontiguousarray(p.delta, dtype=np.uint32)
    if lib.dfm_pdfa_build(p.num_states, p.alphabet_size, p.initial, delta.ctypes.data,
                          C.byref(h)) != 0:
        raise ValueError("malformed partial DFA")
    try:
        n = C.c_uint32()
        lib.dfm_complete(h, C.byref(n), None, None)
        out = np.empty((p.alphabet_size, n.value), np.uint32)
        acc = np.empty(n.value, np.uint8)
        lib.dfm_complete(h, C.byref(n), out.ctypes.data, acc.ctypes.data)
        return Dfa(int(n.value), p.alphabet_size, out, acc, p.initial)
    finally:
        lib.dfm_pdfa_free(h)
