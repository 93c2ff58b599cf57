"""ORACLE — test infrastructure only (imported by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs; never by the product).

Python face of the C restatement in ``oracle/lru_oracle.c`` of the reference's
LRU pool (``offsim.cache.SparsePool``, /root/reference/pkg/src/offsim/cache.py:29-134)
and ``replay`` (cache.py:166-196), plus an independent pure-Python linear-scan
LRU (same role as the reference's ``ListLRU`` test oracle,
pkg/tests/test_cache.py:8-43) for small cases.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "liblru_oracle.so")
_lib = None

_ERRORS = {
    -1: "capacity must be >= 1",
    -2: "capacity may only grow",
    -3: "duplicate generated entry id",
    -4: "out of memory",
    -5: "sparse_ratio must be in (0, 1]",
    -6: "entry ids must be >= 0",
}


def build() -> str:
    """Compile the C restatement (gcc) into oracle/build/."""
    src = os.path.join(_HERE, "lru_oracle.c")
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        i64, p = ctypes.c_int64, ctypes.c_void_p
        P64 = ctypes.POINTER(ctypes.c_int64)
        L.lru_new.restype = p
        L.lru_new.argtypes = [i64]
        L.lru_free.argtypes = [p]
        L.lru_grow.argtypes = [p, i64]
        L.lru_grow.restype = ctypes.c_int
        L.lru_size.argtypes = [p]
        L.lru_size.restype = i64
        L.lru_capacity.argtypes = [p]
        L.lru_capacity.restype = i64
        L.lru_stats.argtypes = [p, P64]
        L.lru_contains.argtypes = [p, i64]
        L.lru_contains.restype = ctypes.c_int
        L.lru_warmup_window.argtypes = [p, P64, i64]
        L.lru_warmup_window.restype = i64
        L.lru_access.argtypes = [p, P64, i64, P64, P64, P64, P64, P64, P64]
        L.lru_access.restype = ctypes.c_int
        L.lru_append.argtypes = [p, P64, i64]
        L.lru_append.restype = i64
        L.lru_order.argtypes = [p, P64]
        L.lru_order.restype = i64
        L.lru_pool_capacity.argtypes = [ctypes.c_double, i64]
        L.lru_pool_capacity.restype = i64
        L.lru_replay.argtypes = [i64, i64, i64, ctypes.c_double, P64, P64, P64,
                                 i64, P64, P64, ctypes.c_int, ctypes.c_int, P64]
        L.lru_replay.restype = ctypes.c_int
        _lib = L
    return _lib


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _check(rc: int) -> int:
    if rc < 0:
        raise ValueError(_ERRORS.get(rc, f"oracle error {rc}"))
    return rc


@dataclass
class OracleAccess:
    hit_ids: list
    miss_ids: list
    evicted_ids: list
    h2d_blocks: int


class OraclePool:
    """Same surface as offsim.cache.SparsePool (cache.py:29-134), C-backed."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        self._L = lib()
        self._p = self._L.lru_new(int(capacity))

    def __del__(self):
        if getattr(self, "_p", None):
            self._L.lru_free(self._p)
            self._p = None

    @property
    def capacity(self) -> int:
        return int(self._L.lru_capacity(self._p))

    def __len__(self):
        return int(self._L.lru_size(self._p))

    def __contains__(self, x):
        return bool(self._L.lru_contains(self._p, int(x)))

    def _stats(self):
        out = np.zeros(3, np.int64)
        self._L.lru_stats(self._p, _p64(out))
        return out

    hits = property(lambda self: int(self._stats()[0]))
    misses = property(lambda self: int(self._stats()[1]))
    evictions = property(lambda self: int(self._stats()[2]))

    def grow_capacity(self, c: int):
        _check(self._L.lru_grow(self._p, int(c)))

    def warmup(self, windows) -> int:
        total = 0
        for w in windows:
            a = np.ascontiguousarray(np.asarray(w, dtype=np.int64))
            total += _check(int(self._L.lru_warmup_window(self._p, _p64(a), len(a))))
        return total

    def access_step(self, requested) -> OracleAccess:
        r = np.ascontiguousarray(np.asarray(list(requested), dtype=np.int64))
        n = len(r)
        h, m, e = (np.zeros(max(n, 1), np.int64) for _ in range(3))
        nh, nm, ne = (np.zeros(1, np.int64) for _ in range(3))
        _check(self._L.lru_access(self._p, _p64(r), n, _p64(h), _p64(nh), _p64(m),
                                  _p64(nm), _p64(e), _p64(ne)))
        return OracleAccess(h[:nh[0]].tolist(), m[:nm[0]].tolist(), e[:ne[0]].tolist(),
                            int(nm[0]))

    def append_generated(self, new_ids) -> int:
        a = np.ascontiguousarray(np.asarray(list(new_ids), dtype=np.int64))
        return _check(int(self._L.lru_append(self._p, _p64(a), len(a))))

    def lru_order(self) -> list:
        out = np.zeros(max(len(self), 1), np.int64)
        k = self._L.lru_order(self._p, _p64(out))
        return out[:k].tolist()

    def resident_ids(self) -> list:
        return sorted(self.lru_order())


def pool_capacity(ratio: float, history: int) -> int:
    return int(lib().lru_pool_capacity(float(ratio), int(history)))


def replay_misses(steps, accepted, context_len, ratio, windows=None,
                  use_warmup=True, preload_full_history=False) -> np.ndarray:
    """cache.py:166-196 in C.  ``steps[t][l]`` are id arrays; returns misses[L, T]."""
    T = len(steps)
    L = len(steps[0]) if T else (len(windows) if windows else 0)
    flat, off = [], [0]
    for t in range(T):
        for l in range(L):
            a = np.asarray(steps[t][l], dtype=np.int64)
            flat.append(a)
            off.append(off[-1] + len(a))
    ids = np.ascontiguousarray(np.concatenate(flat) if flat else np.zeros(1, np.int64))
    sel_off = np.asarray(off, dtype=np.int64)
    acc = np.asarray(accepted, dtype=np.int64)
    W = len(windows[0]) if windows else 0
    wflat, woff = [], [0]
    if W:
        for l in range(L):
            for w in range(W):
                a = np.asarray(windows[l][w], dtype=np.int64)
                wflat.append(a)
                woff.append(woff[-1] + len(a))
    wids = np.ascontiguousarray(np.concatenate(wflat) if wflat else np.zeros(1, np.int64))
    win_off = np.asarray(woff, dtype=np.int64)
    out = np.zeros((max(L, 1), max(T, 1)), np.int64)
    _check(lib().lru_replay(L, T, int(context_len), float(ratio), _p64(ids), _p64(sel_off),
                            _p64(acc), W, _p64(wids), _p64(win_off), int(bool(use_warmup)),
                            int(bool(preload_full_history)), _p64(out)))
    return out[:L, :T]


class LinearLRU:
    """Independent brute-force LRU (list, MRU at the tail) for small cases; the
    same semantics the reference's tests pin (pkg/tests/test_cache.py:8-43,
    test_acceptance.py:57-89), extended with warm-up (cache.py:73-88)."""

    def __init__(self, capacity):
        self.capacity = capacity
        self.order = []

    def warmup(self, windows):
        ins = 0
        for w in windows:
            for x in w:
                x = int(x)
                if x in self.order:
                    self.order.remove(x)
                else:
                    ins += 1
                self.order.append(x)
                while len(self.order) > self.capacity:
                    self.order.pop(0)
        return ins

    def access(self, requested):
        requested = [int(x) for x in requested]
        hits = [x for x in requested if x in self.order]
        misses = [x for x in requested if x not in self.order]
        evicted = []
        if len(requested) > self.capacity:
            keep = requested[-self.capacity:]
            evicted = [x for x in self.order if x not in keep]
            self.order = [x for x in self.order if x in keep]
            for x in keep:
                if x in self.order:
                    self.order.remove(x)
                self.order.append(x)
        else:
            for x in hits:
                self.order.remove(x)
                self.order.append(x)
            for x in misses:
                if len(self.order) >= self.capacity:
                    evicted.append(self.order.pop(0))
                self.order.append(x)
        return hits, misses, sorted(evicted)

    def append(self, new_ids):
        for x in new_ids:
            if len(self.order) >= self.capacity:
                self.order.pop(0)
            self.order.append(int(x))
