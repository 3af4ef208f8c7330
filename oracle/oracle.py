"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the CPU oracle.

Two libraries sit behind this module:

* ``liboracle.so`` — the plain-C restatement (``dfm_oracle.c``) of the
  reference algorithms; every function there cites the reference file:line.
* ``_ref/libdfamin_ref.so`` — the unmodified reference headers compiled from
  ``/root/reference/proj/include`` behind a thin C-ABI (``ref_shim.cpp``).
  Present where it was built (this container, and the GPU box via the gpurun
  snapshot); ``ref_available()`` says whether it loaded.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg import this module.  The product package never does.

All functions take/return numpy arrays: ``delta`` is (k, n) uint32 (row a is
the reference's ``delta[a]``), ``acc`` is (n,) uint8.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
U32P = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
U8P = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
U64P = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")

POLICY = {"arbitrary": 0, "min": 1, "max": 2}
STATUS = {0: "ok", 1: "timeout", 2: "capacity-exceeded"}


class _OrcDfa(C.Structure):
    _fields_ = [("n", C.c_uint32), ("k", C.c_uint32), ("delta", C.c_void_p),
                ("acc", C.c_void_p), ("initial", C.c_uint32)]


class _OrcStats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("closure_steps", C.c_uint64),
                ("peak_memory_estimate", C.c_uint64), ("status", C.c_int32)]


class _RefStats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("closure_steps", C.c_uint64),
                ("elapsed_ms", C.c_double), ("peak_memory_estimate", C.c_uint64),
                ("status", C.c_int32), ("call_ms", C.c_double)]


PASS_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint32), C.c_uint32,
                      C.c_uint32)


@dataclass
class Result:
    block: np.ndarray  # canonical labels (empty unless status == "ok")
    num_blocks: int
    iterations: int
    closure_steps: int
    peak_memory_estimate: int
    status: str
    elapsed_ms: float = 0.0  # the reference's RunStats.elapsed_ms (excludes its canonicalize)
    call_ms: float = 0.0     # wall time of the whole reference call (oracle/_ref only)


def _build_if_missing() -> None:
    if not os.path.exists(os.path.join(HERE, "liboracle.so")):
        import subprocess
        subprocess.check_call(["make", "-s", "-C", HERE, os.path.join(HERE, "liboracle.so")])


_build_if_missing()
_lib = C.CDLL(os.path.join(HERE, "liboracle.so"))
_ref = None
_ref_path = os.path.join(HERE, "_ref", "libdfamin_ref.so")
if os.path.exists(_ref_path):
    try:
        _ref = C.CDLL(_ref_path)
    except OSError:  # pragma: no cover - wrong-arch prebuilt
        _ref = None


def ref_available() -> bool:
    return _ref is not None


def _dfa(delta: np.ndarray, acc: np.ndarray):
    delta = np.ascontiguousarray(delta, dtype=np.uint32)
    acc = np.ascontiguousarray(acc, dtype=np.uint8)
    k = delta.shape[0]
    n = acc.shape[0]
    d = _OrcDfa(n, k, delta.ctypes.data if delta.size else None, acc.ctypes.data, 0)
    return d, delta, acc


# ---------------------------------------------------------------- generators
def random_dfa(n: int, k: int, seed: int, p: float = 0.5):
    delta = np.empty((k, n), np.uint32)
    acc = np.empty(n, np.uint8)
    _lib.orc_random_dfa(C.c_uint32(n), C.c_uint32(k), C.c_uint64(seed), C.c_double(p),
                        delta.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p))
    return delta, acc


def fib_len(idx: int) -> int:
    _lib.orc_fib_len.restype = C.c_uint32
    return int(_lib.orc_fib_len(C.c_uint32(idx)))


def fib_dfa(idx: int):
    n = fib_len(idx)
    delta = np.empty((1, n), np.uint32)
    acc = np.empty(n, np.uint8)
    if _lib.orc_fib_dfa(C.c_uint32(idx), delta.ctypes.data_as(C.c_void_p),
                        acc.ctypes.data_as(C.c_void_p)) != 0:
        raise ValueError("fib_dfa needs 2 <= idx <= 45")
    return delta, acc


def bit_splitter(bits: int):
    if bits < 1 or bits > 26:
        raise ValueError("bit_splitter needs 1 <= bits <= 26")
    n = 1 << bits
    delta = np.zeros((bits - 1, n), np.uint32)
    acc = np.empty(n, np.uint8)
    _lib.orc_bit_splitter(C.c_uint32(bits), delta.ctypes.data_as(C.c_void_p),
                          acc.ctypes.data_as(C.c_void_p))
    return delta, acc


def chain_dfa(length: int):
    delta = np.empty((1, length), np.uint32)
    acc = np.empty(length, np.uint8)
    if _lib.orc_chain_dfa(C.c_uint32(length), delta.ctypes.data_as(C.c_void_p),
                          acc.ctypes.data_as(C.c_void_p)) != 0:
        raise ValueError("chain_dfa needs len >= 2")
    return delta, acc


def comb_dfa(L: int, t: int):
    n = L * (t + 1) + 1
    delta = np.empty((2, n), np.uint32)
    acc = np.empty(n, np.uint8)
    _lib.orc_comb_dfa(C.c_uint32(L), C.c_uint32(t), delta.ctypes.data_as(C.c_void_p),
                      acc.ctypes.data_as(C.c_void_p))
    return delta, acc


def vlts_dfa(m: int, n: int, k: int, base_seed: int = 7, inflate_seed: int = 9,
             p: float = 0.4, window: int = 16):
    delta = np.empty((k, n), np.uint32)
    acc = np.empty(n, np.uint8)
    if _lib.orc_vlts_dfa(C.c_uint32(m), C.c_uint32(n), C.c_uint32(k), C.c_uint64(base_seed),
                         C.c_uint64(inflate_seed), C.c_double(p), C.c_uint32(window),
                         delta.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p)) != 0:
        raise ValueError("vlts_dfa needs n % m == 0")
    return delta, acc


# ---------------------------------------------------------------- core
def canonicalize(raw) -> tuple[np.ndarray, int]:
    raw = np.ascontiguousarray(raw, dtype=np.uint32)
    out = np.empty_like(raw)
    _lib.orc_canonicalize.restype = C.c_uint32
    c = _lib.orc_canonicalize(raw.ctypes.data_as(C.c_void_p), C.c_uint32(raw.size),
                              out.ctypes.data_as(C.c_void_p))
    return out, int(c)


def moore(delta, acc) -> Result:
    d, delta, acc = _dfa(delta, acc)
    out = np.empty(acc.size, np.uint32)
    rounds = C.c_uint64(0)
    _lib.orc_moore.restype = C.c_uint32
    c = _lib.orc_moore(C.byref(d), out.ctypes.data_as(C.c_void_p), C.byref(rounds))
    return Result(out, int(c), int(rounds.value), 0, 0, "ok")


def _result(block, nb, st) -> Result:
    status = STATUS[st.status]
    return Result(block if status == "ok" else np.empty(0, np.uint32), int(nb.value),
                  int(st.iterations), int(st.closure_steps), int(st.peak_memory_estimate),
                  status, float(getattr(st, "elapsed_ms", 0.0)), float(getattr(st, "call_ms", 0.0)))


def sort_pr(delta, acc, trace: list | None = None) -> Result:
    d, delta, acc = _dfa(delta, acc)
    block = np.empty(acc.size, np.uint32)
    nb = C.c_uint32(0)
    st = _OrcStats()
    cb = None
    if trace is not None:
        def _cb(user, it, blk, n, count):
            raw = np.ctypeslib.as_array(blk, shape=(n,)).copy()
            trace.append((count, canonicalize(raw)[0]))
        cb = PASS_CB(_cb)
    _lib.orc_sort_pr(C.byref(d), block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st),
                     cb, None)
    return _result(block, nb, st)


def naive_pr(delta, acc, policy: str = "min", fused_cas: bool = False,
             trace: list | None = None) -> Result:
    d, delta, acc = _dfa(delta, acc)
    block = np.empty(acc.size, np.uint32)
    nb = C.c_uint32(0)
    st = _OrcStats()
    cb = None
    if trace is not None:
        def _cb(user, it, blk, n, count):
            raw = np.ctypeslib.as_array(blk, shape=(n,)).copy()
            trace.append((count, raw))
        cb = PASS_CB(_cb)
    _lib.orc_naive_pr(C.byref(d), C.c_int(POLICY[policy]), C.c_int(int(fused_cas)),
                      block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st), cb, None)
    return _result(block, nb, st)


def power_levels(n: int) -> int:
    return int(n).bit_length()


def expand_alphabet(delta, acc, max_memory_bytes: int = 16 << 30):
    """Returns (rows (levels*k, n), levels) or raises MemoryError(required)."""
    d, delta, acc = _dfa(delta, acc)
    k, n = delta.shape[0], acc.size
    levels = power_levels(n)
    req = levels * k * n * 4
    if req > max_memory_bytes:
        err = MemoryError(f"alphabet expansion needs {req} bytes")
        err.required_bytes = req
        raise err
    rows = np.empty((levels * k, n), np.uint32)
    lv = C.c_uint32(0)
    rq = C.c_uint64(0)
    _lib.orc_expand_alphabet(C.byref(d), C.c_uint64(max_memory_bytes),
                             rows.ctypes.data_as(C.c_void_p), C.byref(lv), C.byref(rq))
    return rows, int(lv.value)


def trans_pr(delta, acc, policy: str = "min", max_memory_bytes: int = 16 << 30) -> Result:
    d, delta, acc = _dfa(delta, acc)
    block = np.empty(acc.size, np.uint32)
    nb = C.c_uint32(0)
    st = _OrcStats()
    _lib.orc_trans_pr(C.byref(d), C.c_int(POLICY[policy]), C.c_uint64(max_memory_bytes),
                      block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st))
    return _result(block, nb, st)


def trans_minimize(delta, acc, max_memory_bytes: int = 16 << 30, inspect: dict | None = None):
    d, delta, acc = _dfa(delta, acc)
    n = acc.size
    block = np.empty(n, np.uint32)
    nb = C.c_uint32(0)
    st = _OrcStats()
    apart = np.zeros(n * n, np.uint8) if inspect is not None else None
    pops = np.zeros(4096, np.uint64) if inspect is not None else None
    _lib.orc_trans_minimize(C.byref(d), C.c_uint64(max_memory_bytes),
                            block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st),
                            apart.ctypes.data_as(C.c_void_p) if apart is not None else None,
                            pops.ctypes.data_as(C.c_void_p) if pops is not None else None,
                            C.c_uint32(4096))
    r = _result(block, nb, st)
    if inspect is not None and r.status == "ok":
        inspect["apart"] = apart.reshape(n, n)
        inspect["apart_popcounts"] = pops[: r.iterations].copy()
    return r


# ---------------------------------------------------------------- the reference itself
# ---------------------------------------------------------------- post-processing
class QuotientError(ValueError):
    """The reference's std::invalid_argument from quotient (core.hpp:256-290)."""


def quotient(delta, acc, block, num_blocks: int, initial: int = 0):
    """core.hpp:256-290 restated (orc_quotient): (delta_q, acc_q, initial_q) or
    QuotientError with the reference's message."""
    delta = np.ascontiguousarray(delta, dtype=np.uint32)
    acc = np.ascontiguousarray(acc, dtype=np.uint8)
    block = np.ascontiguousarray(block, dtype=np.uint32)
    k, n = delta.shape[0], acc.size
    if block.size != n:
        raise QuotientError("partition covers a different state count")
    d = _OrcDfa(n, k, delta.ctypes.data if delta.size else None, acc.ctypes.data, initial)
    dq = np.zeros((k, max(num_blocks, 0)), np.uint32)
    aq = np.zeros(max(num_blocks, 0), np.uint8)
    iq, bb, bl = C.c_uint32(0), C.c_uint32(0), C.c_uint32(0)
    rc = _lib.orc_quotient(C.byref(d), block.ctypes.data_as(C.c_void_p), C.c_uint32(num_blocks),
                           dq.ctypes.data_as(C.c_void_p), aq.ctypes.data_as(C.c_void_p),
                           C.byref(iq), C.byref(bb), C.byref(bl))
    if rc == 1:
        raise QuotientError("partition is not in canonical form")
    if rc == 2:
        raise QuotientError(f"inconsistent partition: block {bb.value} mixes accepting and "
                            "rejecting states")
    if rc == 3:
        raise QuotientError(f"inconsistent partition: block {bb.value} splits on letter {bl.value}")
    return dq, aq, int(iq.value)


def remove_unreachable(delta, acc, initial: int = 0):
    """core.hpp:152-187 restated (orc_remove_unreachable): (delta', acc', initial')."""
    delta = np.ascontiguousarray(delta, dtype=np.uint32)
    acc = np.ascontiguousarray(acc, dtype=np.uint8)
    k, n = delta.shape[0], acc.size
    d = _OrcDfa(n, k, delta.ctypes.data if delta.size else None, acc.ctypes.data, initial)
    flat = np.zeros(max(k * n, 1), np.uint32)
    ao = np.zeros(max(n, 1), np.uint8)
    io = C.c_uint32(0)
    _lib.orc_remove_unreachable.restype = C.c_uint32
    kept = int(_lib.orc_remove_unreachable(C.byref(d), flat.ctypes.data_as(C.c_void_p),
                                           ao.ctypes.data_as(C.c_void_p), C.byref(io)))
    return flat[: k * kept].reshape(k, kept).copy(), ao[:kept].copy(), int(io.value)


class Reference:
    """The unmodified reference (oracle/_ref) behind ref_shim.cpp."""

    def __init__(self):
        if _ref is None:
            raise RuntimeError("oracle/_ref/libdfamin_ref.so is not built")
        self.lib = _ref
        self.lib.ref_moore.restype = C.c_uint32
        self.lib.ref_canonicalize.restype = C.c_uint32
        self.lib.ref_worker_count.restype = C.c_uint

    def set_threads(self, n: int) -> None:
        self.lib.ref_set_threads(C.c_uint(n))

    def worker_count(self) -> int:
        return int(self.lib.ref_worker_count())

    @staticmethod
    def _args(delta, acc):
        delta = np.ascontiguousarray(delta, dtype=np.uint32)
        acc = np.ascontiguousarray(acc, dtype=np.uint8)
        return delta, acc, C.c_uint32(acc.size), C.c_uint32(delta.shape[0])

    def _res(self, block, nb, st):
        return _result(block, nb, st)

    def sort_pr(self, delta, acc, timeout_ms: int = 300_000, trace_counts: list | None = None):
        delta, acc, n, k = self._args(delta, acc)
        block = np.empty(acc.size, np.uint32)
        nb = C.c_uint32(0)
        st = _RefStats()
        tc = np.zeros(1 << 16, np.uint32) if trace_counts is not None else None
        self.lib.ref_sort_pr(n, k, delta.ctypes.data_as(C.c_void_p),
                             acc.ctypes.data_as(C.c_void_p), C.c_int64(timeout_ms),
                             block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st),
                             tc.ctypes.data_as(C.c_void_p) if tc is not None else None,
                             C.c_uint32(1 << 16))
        r = self._res(block, nb, st)
        if trace_counts is not None:
            trace_counts.extend(int(x) for x in tc[: r.iterations])
        return r

    def naive_pr(self, delta, acc, policy: str = "min", fused_cas: bool = False,
                 timeout_ms: int = 300_000):
        delta, acc, n, k = self._args(delta, acc)
        block = np.empty(acc.size, np.uint32)
        nb = C.c_uint32(0)
        st = _RefStats()
        self.lib.ref_naive_pr(n, k, delta.ctypes.data_as(C.c_void_p),
                              acc.ctypes.data_as(C.c_void_p), C.c_int(POLICY[policy]),
                              C.c_int(int(fused_cas)), C.c_int64(timeout_ms),
                              block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st))
        return self._res(block, nb, st)

    def trans_pr(self, delta, acc, policy: str = "min", timeout_ms: int = 300_000,
                 max_memory_bytes: int = 16 << 30):
        delta, acc, n, k = self._args(delta, acc)
        block = np.empty(acc.size, np.uint32)
        nb = C.c_uint32(0)
        st = _RefStats()
        self.lib.ref_trans_pr(n, k, delta.ctypes.data_as(C.c_void_p),
                              acc.ctypes.data_as(C.c_void_p), C.c_int(POLICY[policy]),
                              C.c_int64(timeout_ms), C.c_uint64(max_memory_bytes),
                              block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st))
        return self._res(block, nb, st)

    def expand_alphabet(self, delta, acc, max_memory_bytes: int = 16 << 30):
        delta, acc, n, k = self._args(delta, acc)
        levels = power_levels(acc.size)
        rows = np.empty((max(levels * delta.shape[0], 1), acc.size), np.uint32)
        lv = C.c_uint32(0)
        rq = C.c_uint64(0)
        rc = self.lib.ref_expand_alphabet(n, k, delta.ctypes.data_as(C.c_void_p),
                                          acc.ctypes.data_as(C.c_void_p),
                                          C.c_uint64(max_memory_bytes),
                                          rows.ctypes.data_as(C.c_void_p), C.byref(lv),
                                          C.byref(rq))
        if rc == -2:
            err = MemoryError("capacity")
            err.required_bytes = int(rq.value)
            raise err
        return rows[: levels * delta.shape[0]], int(lv.value)

    def trans_minimize(self, delta, acc, timeout_ms: int = 300_000,
                       max_memory_bytes: int = 16 << 30, inspect: dict | None = None):
        delta, acc, n, k = self._args(delta, acc)
        nn = acc.size
        block = np.empty(nn, np.uint32)
        nb = C.c_uint32(0)
        st = _RefStats()
        apart = np.zeros(max(nn * nn, 1), np.uint8) if inspect is not None else None
        pops = np.zeros(4096, np.uint64) if inspect is not None else None
        self.lib.ref_trans_minimize(n, k, delta.ctypes.data_as(C.c_void_p),
                                    acc.ctypes.data_as(C.c_void_p), C.c_int64(timeout_ms),
                                    C.c_uint64(max_memory_bytes),
                                    block.ctypes.data_as(C.c_void_p), C.byref(nb), C.byref(st),
                                    apart.ctypes.data_as(C.c_void_p) if apart is not None
                                    else None,
                                    pops.ctypes.data_as(C.c_void_p) if pops is not None else None,
                                    C.c_uint32(4096))
        r = self._res(block, nb, st)
        if inspect is not None and r.status == "ok":
            inspect["apart"] = apart[: nn * nn].reshape(nn, nn)
            inspect["apart_popcounts"] = pops[: r.iterations].copy()
        return r

    def sort_session(self, n: int, k: int, seed: int, p: float = 0.5) -> "RefSortSession":
        """sortPR one pass per call on the reference-generated random_dfa (ref_shim.cpp)."""
        return RefSortSession(self.lib, n, k, seed, p)

    def moore(self, delta, acc):
        delta, acc, n, k = self._args(delta, acc)
        block = np.empty(acc.size, np.uint32)
        rounds = C.c_uint64(0)
        c = self.lib.ref_moore(n, k, delta.ctypes.data_as(C.c_void_p),
                               acc.ctypes.data_as(C.c_void_p), block.ctypes.data_as(C.c_void_p),
                               C.byref(rounds))
        return Result(block, int(c), int(rounds.value), 0, 0, "ok")

    def random_dfa(self, n, k, seed, p=0.5):
        delta = np.empty((k, n), np.uint32)
        acc = np.empty(n, np.uint8)
        self.lib.ref_random_dfa(C.c_uint32(n), C.c_uint32(k), C.c_uint64(seed), C.c_double(p),
                                delta.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p))
        return delta, acc

    def fib_dfa(self, idx):
        n = fib_len(idx)
        delta = np.empty((1, n), np.uint32)
        acc = np.empty(n, np.uint8)
        self.lib.ref_fib_dfa(C.c_uint32(idx), delta.ctypes.data_as(C.c_void_p),
                             acc.ctypes.data_as(C.c_void_p))
        return delta, acc

    def bit_splitter(self, bits):
        n = 1 << bits
        delta = np.zeros((bits - 1, n), np.uint32)
        acc = np.empty(n, np.uint8)
        self.lib.ref_bit_splitter(C.c_uint32(bits), delta.ctypes.data_as(C.c_void_p),
                                  acc.ctypes.data_as(C.c_void_p))
        return delta, acc

    def chain_dfa(self, length):
        delta = np.empty((1, length), np.uint32)
        acc = np.empty(length, np.uint8)
        self.lib.ref_chain_dfa(C.c_uint32(length), delta.ctypes.data_as(C.c_void_p),
                               acc.ctypes.data_as(C.c_void_p))
        return delta, acc


def _ref_quotient(self, delta, acc, block, num_blocks: int, initial: int = 0):
    delta, acc, n, k = self._args(delta, acc)
    block = np.ascontiguousarray(block, dtype=np.uint32)
    dq = np.zeros((delta.shape[0], max(num_blocks, 0)), np.uint32)
    aq = np.zeros(max(num_blocks, 0), np.uint8)
    iq = C.c_uint32(0)
    err = C.create_string_buffer(256)
    rc = self.lib.ref_quotient(n, k, delta.ctypes.data_as(C.c_void_p), acc.ctypes.data_as(C.c_void_p),
                               C.c_uint32(initial), block.ctypes.data_as(C.c_void_p),
                               C.c_uint32(num_blocks), dq.ctypes.data_as(C.c_void_p),
                               aq.ctypes.data_as(C.c_void_p), C.byref(iq), err, C.c_uint32(256))
    if rc != 0:
        raise QuotientError(err.value.decode())
    return dq, aq, int(iq.value)


def _ref_remove_unreachable(self, delta, acc, initial: int = 0):
    delta, acc, n, k = self._args(delta, acc)
    flat = np.zeros(max(delta.size, 1), np.uint32)
    ao = np.zeros(max(acc.size, 1), np.uint8)
    io = C.c_uint32(0)
    self.lib.ref_remove_unreachable.restype = C.c_uint32
    kept = int(self.lib.ref_remove_unreachable(n, k, delta.ctypes.data_as(C.c_void_p),
                                               acc.ctypes.data_as(C.c_void_p), C.c_uint32(initial),
                                               flat.ctypes.data_as(C.c_void_p),
                                               ao.ctypes.data_as(C.c_void_p), C.byref(io)))
    kk = delta.shape[0]
    return flat[: kk * kept].reshape(kk, kept).copy(), ao[:kept].copy(), int(io.value)


Reference.quotient = _ref_quotient
Reference.remove_unreachable = _ref_remove_unreachable


class RefSortSession:
    """The reference sort_pr loop (min_sort.hpp:80-123) one pass per call, over
    its own functions (ref_shim.cpp ref_sort_session_*): bench.py's bounded
    per-step sample of the workload.  ``pass_()`` -> (elapsed ms, fresh count,
    fixpoint reached); ``full()`` runs the reference's whole sort_pr."""

    def __init__(self, lib, n, k, seed, p):
        self.lib = lib
        lib.ref_sort_session_random.restype = C.c_void_p
        lib.ref_sort_session_random.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_double]
        lib.ref_sort_session_pass.argtypes = [C.c_void_p, C.POINTER(C.c_double),
                                              C.POINTER(C.c_uint32)]
        lib.ref_sort_session_full.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.c_void_p]
        lib.ref_sort_session_free.argtypes = [C.c_void_p]
        self.h = lib.ref_sort_session_random(n, k, seed, p)
        self.n, self.k = n, k

    def pass_(self):
        ms = C.c_double(0)
        fresh = C.c_uint32(0)
        done = self.lib.ref_sort_session_pass(self.h, C.byref(ms), C.byref(fresh))
        return float(ms.value), int(fresh.value), bool(done)

    def reset(self) -> None:
        self.lib.ref_sort_session_reset.argtypes = [C.c_void_p]
        self.lib.ref_sort_session_reset(self.h)

    def full(self) -> Result:
        nb = C.c_uint32(0)
        st = _RefStats()
        self.lib.ref_sort_session_full(self.h, C.byref(nb), C.byref(st))
        return _result(np.empty(0, np.uint32), nb, st)

    def close(self):
        if self.h:
            self.lib.ref_sort_session_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def ref_ingest(text, max_subsets: int = 1 << 22) -> dict:
    """The reference's parse_lts -> determinize -> complete on `text` (oracle/_ref):
    {"status": "ok"|"parse"|"budget", "line", "what", "lts": (n, init, labels, src,
    label, dst), "pdfa": delta (k, n), "dfa": (delta, acc)}."""
    lib = _ref
    lib.ref_ingest.restype = C.c_void_p
    lib.ref_ingest.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64]
    lib.ref_ingest_label.restype = C.c_char_p
    for f in ("ref_ingest_status", "ref_ingest_lts", "ref_ingest_lts_arrays", "ref_ingest_label",
              "ref_ingest_pdfa", "ref_ingest_dfa", "ref_ingest_free"):
        getattr(lib, f).argtypes = None
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p(lib.ref_ingest(data, len(data), max_subsets))
    try:
        line = C.c_uint64(0)
        msg = C.create_string_buffer(512)
        st = lib.ref_ingest_status(h, C.byref(line), msg, C.c_uint32(512))
        out = {"status": ["ok", "parse", "budget"][st], "line": int(line.value),
               "what": msg.value.decode()}
        if st != 0:
            return out
        n, init, nl, m = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint64()
        lib.ref_ingest_lts(h, C.byref(n), C.byref(init), C.byref(nl), C.byref(m))
        src = np.empty(m.value, np.uint32)
        lab = np.empty(m.value, np.uint32)
        dst = np.empty(m.value, np.uint32)
        lib.ref_ingest_lts_arrays(h, src.ctypes.data_as(C.c_void_p), lab.ctypes.data_as(C.c_void_p),
                                  dst.ctypes.data_as(C.c_void_p))
        labels = [lib.ref_ingest_label(h, C.c_uint32(i)).decode() for i in range(nl.value)]
        out["lts"] = (int(n.value), int(init.value), labels, src, lab, dst)
        pn, pk = C.c_uint32(), C.c_uint32()
        lib.ref_ingest_pdfa(h, C.byref(pn), C.byref(pk), None)
        pd = np.empty((pk.value, pn.value), np.uint32)
        lib.ref_ingest_pdfa(h, C.byref(pn), C.byref(pk), pd.ctypes.data_as(C.c_void_p))
        out["pdfa"] = pd
        dn = C.c_uint32()
        lib.ref_ingest_dfa(h, C.byref(dn), None, None)
        dd = np.empty((pk.value, dn.value), np.uint32)
        da = np.empty(dn.value, np.uint8)
        lib.ref_ingest_dfa(h, C.byref(dn), dd.ctypes.data_as(C.c_void_p),
                           da.ctypes.data_as(C.c_void_p))
        out["dfa"] = (dd, da)
        return out
    finally:
        lib.ref_ingest_free(h)
