"""GPU latent-cache manager: the drop-in for ``offsim.cache``
(/root/reference/pkg/src/offsim/cache.py).

* ``PoolSet`` — P independent LRU pools resident on the GPU (one per (request,
  layer)), driven by the K3 kernels in csrc/pool.cu.  Batched,
  asynchronous, device tensors in and out: the decode hot path uses this.
* ``SparsePool`` — the reference's single-pool class (cache.py:29-134) with the
  same methods, results and ValueErrors, backed by a one-pool ``PoolSet``.
* ``replay`` — cache.py:166-196 with every layer's pool stepped in one launch.
* ``MissProfile``, ``pool_capacity`` and the miss-profile CSV helpers
  (cache.py:137-163, :199-229).
"""

from __future__ import annotations

import csv
import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .trace import AccessTrace


def pool_capacity(sparse_ratio: float, history_len: int) -> int:
    """max(1, floor(rho * history))  (cache.py:137-138)."""
    return max(1, math.floor(sparse_ratio * history_len))


@dataclass
class AccessResult:
    hit_ids: list
    miss_ids: list
    evicted_ids: list
    h2d_blocks: int
    d2h_blocks: int = 0


@dataclass
class AccessBatch:
    """Device-side results of one batched access (rows = pools of the call)."""
    counts: torch.Tensor            # [num, 4] int32: nhit, nmiss, nevicted, ntransient
    sel_row: torch.Tensor | None    # [num, K] slot-store row of each requested id
    miss_ids: torch.Tensor | None   # [num, K] misses in requested order
    miss_row: torch.Tensor | None   # [num, K] destination row of each miss
    hit_ids: torch.Tensor | None = None
    evicted_ids: torch.Tensor | None = None
    hit_row: torch.Tensor | None = None  # [num, K] row of each hit (resident before the step)


def _i32(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.int32).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.int32), device=device)


class PoolSet:
    """P LRU pools over entry ids [0, max_ids) with at most ``cap_max`` slots each.

    With ``row_bytes`` = 1152 (576 x f16) the set also owns the GPU slot store of
    attention-ready rows, dequantised once on admission (cap_max rows per
    pool + ``staging_rows`` transient rows for oversize requests, cache.py:103-111).
    All methods enqueue on the current CUDA stream; ``check()`` synchronises and
    raises the reference's exceptions for errors detected on the device.
    """

    def __init__(self, num_pools: int, max_ids: int, cap_max: int, capacity=None,
                 row_bytes: int = 0, staging_rows: int = 0, device=None):
        _lib.require_cuda()
        self.device = torch.device(device if device is not None else "cuda")
        self.num_pools, self.max_ids, self.cap_max = int(num_pools), int(max_ids), int(cap_max)
        self.row_bytes, self.staging_rows = int(row_bytes), int(staging_rows)
        self._L = _lib.load()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._L.ess_pool_create(ctypes.byref(h), self.num_pools, self.max_ids,
                                               self.cap_max, self.row_bytes, self.staging_rows),
                       "ess_pool_create")
        self._h = h
        self.rows_per_pool = self.cap_max + self.staging_rows
        if capacity is not None:
            self.reset(capacity)

    # -- lifecycle --------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            torch.cuda.synchronize(self.device)
            self._L.ess_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def _range(self, begin, num):
        num = self.num_pools - begin if num is None else num
        if begin < 0 or num < 0 or begin + num > self.num_pools:
            raise ValueError("pool range out of bounds")
        return begin, num

    def _caps(self, capacity, num):
        if isinstance(capacity, (int, np.integer)):
            capacity = [int(capacity)] * num
        return _i32(capacity, self.device)

    def reset(self, capacity, begin: int = 0, num: int | None = None):
        begin, num = self._range(begin, num)
        c = self._caps(capacity, num)
        _lib.check(self._L.ess_pool_reset(self._h, begin, num, c.data_ptr(), _lib.stream_handle()))
        self._keep = c

    def grow(self, capacity, begin: int = 0, num: int | None = None):
        begin, num = self._range(begin, num)
        c = self._caps(capacity, num)
        _lib.check(self._L.ess_pool_grow(self._h, begin, num, c.data_ptr(), _lib.stream_handle()))
        self._keep = c

    # -- K3 -----------------------------------------------------------------------------
    def warmup(self, ids: torch.Tensor, n: torch.Tensor, begin: int = 0,
               inserted: torch.Tensor | None = None) -> torch.Tensor:
        """One window per pool (rows of ``ids``, ``n[i]`` valid, duplicate-free)."""
        num = ids.shape[0]
        self._range(begin, num)
        if inserted is None:
            inserted = torch.zeros(num, dtype=torch.int64, device=self.device)
        _lib.check(self._L.ess_pool_warmup(self._h, begin, num, ids.data_ptr(), n.data_ptr(),
                                           ids.stride(0), inserted.data_ptr(), _lib.stream_handle()))
        return inserted

    def access(self, req: torch.Tensor, n: torch.Tensor, begin: int = 0, lists: bool = False,
               sort_evicted: bool = True, out: AccessBatch | None = None) -> AccessBatch:
        """One selection set per pool.  Hot path: counts, sel_row, hit rows, miss
        ids/rows.  ``lists=True`` also returns hit ids and evicted ids (API/tests)."""
        num, K = req.shape
        self._range(begin, num)
        if out is None:
            z = lambda: torch.empty((num, K), dtype=torch.int32, device=self.device)  # noqa: E731
            out = AccessBatch(counts=torch.empty((num, 4), dtype=torch.int32, device=self.device),
                              sel_row=z(), miss_ids=z(), miss_row=z(), hit_row=z(),
                              hit_ids=z() if lists else None, evicted_ids=z() if lists else None)
        flags = _lib.ESS_ACCESS_SORT_EVICTED if sort_evicted else 0
        stride = next(t.stride(0) for t in (out.sel_row, out.miss_ids, out.miss_row, out.hit_row,
                                            out.hit_ids, out.evicted_ids, req) if t is not None)
        _lib.check(self._L.ess_pool_access(
            self._h, begin, num, req.data_ptr(), n.data_ptr(), req.stride(0),
            _lib.ptr(out.hit_ids), _lib.ptr(out.miss_ids), _lib.ptr(out.evicted_ids),
            _lib.ptr(out.sel_row), _lib.ptr(out.hit_row), _lib.ptr(out.miss_row),
            out.counts.data_ptr(), stride, flags, _lib.stream_handle()))
        return out

    def access_mtp(self, req: torch.Tensor, n: torch.Tensor, begin: int = 0, lists: bool = False,
                   sort_evicted: bool = True, out: AccessBatch | None = None,
                   sel_row: torch.Tensor | None = None, tok_split=None,
                   ready: torch.Tensor | None = None) -> AccessBatch:
        """MTP: ``qtok`` selection sets per pool, req [num, qtok, K] / n [num, qtok] (the
        layout of ``indexer.topk_mtp``), taken as qtok consecutive access_steps per pool in
        one launch — recency is updated by every selected set.  ``sel_row``
        [num, qtok, K] gets each set's slot rows; the hit/miss/evicted lists of a pool's
        sets are appended in set order in its [num, qtok*K] rows; counts are the sums.
        ``tok_split`` = (hit_row, fresh_row [num, qtok, K], counts [num, qtok, 2]): per set,
        the rows resident before the step and those fetched this step (attention pass 1
        beside the gather, pass 2 after it).  ``ready`` (int32 [num]): each pool's flag is
        set once its lists are stored (for a concurrently running ``gather_stream``)."""
        num, qtok, K = req.shape
        self._range(begin, num)
        if not 1 <= qtok <= _lib.MAX_QTOK:
            raise ValueError(f"qtok must be in [1, {_lib.MAX_QTOK}]")
        if not req.is_contiguous() or n.shape != (num, qtok) or not n.is_contiguous():
            raise ValueError("req must be contiguous [num, qtok, K] and n [num, qtok]")
        if out is None:
            z = lambda: torch.empty((num, qtok * K), dtype=torch.int32, device=self.device)  # noqa: E731
            out = AccessBatch(counts=torch.empty((num, 4), dtype=torch.int32, device=self.device),
                              sel_row=None, miss_ids=z(), miss_row=z(), hit_row=z(),
                              hit_ids=z() if lists else None, evicted_ids=z() if lists else None)
        if sel_row is None:
            sel_row = torch.empty((num, qtok, K), dtype=torch.int32, device=self.device)
        if sel_row.shape != (num, qtok, K) or not sel_row.is_contiguous():
            raise ValueError("sel_row must be contiguous [num, qtok, K]")
        lists_ = [t for t in (out.miss_ids, out.miss_row, out.hit_row, out.hit_ids, out.evicted_ids)
                  if t is not None]
        stride = lists_[0].stride(0) if lists_ else qtok * K
        if any(t.stride(0) != stride or t.stride(1) != 1 for t in lists_) or stride < qtok * K:
            raise ValueError("list outputs must share a row stride >= qtok * K")
        if tok_split is not None:
            th, tf, tc = tok_split
            if (th.shape != (num, qtok, K) or tf.shape != (num, qtok, K) or tc.shape != (num, qtok, 2)
                    or not (th.is_contiguous() and tf.is_contiguous() and tc.is_contiguous())):
                raise ValueError("tok_split must be contiguous [num, qtok, K] x2 and [num, qtok, 2]")
        flags = _lib.ESS_ACCESS_SORT_EVICTED if sort_evicted else 0
        _lib.check(self._L.ess_pool_access_mtp(
            self._h, begin, num, qtok, req.data_ptr(), n.data_ptr(), K,
            _lib.ptr(out.hit_ids), _lib.ptr(out.miss_ids), _lib.ptr(out.evicted_ids),
            sel_row.data_ptr(), _lib.ptr(out.hit_row), _lib.ptr(out.miss_row),
            out.counts.data_ptr(), stride,
            *((_lib.ptr(t) for t in tok_split) if tok_split is not None else (None, None, None)),
            _lib.ptr(ready), flags, _lib.stream_handle()), "ess_pool_access_mtp")
        out.sel_row = sel_row
        return out

    def split(self, req: torch.Tensor, n: torch.Tensor, out: AccessBatch, begin: int = 0) -> AccessBatch:
        """Early-gather K3a: read-only hit/miss split; misses point at staging rows
        (needs staging_rows >= 2048; see ess_pool_split)."""
        num = req.shape[0]
        self._range(begin, num)
        _lib.check(self._L.ess_pool_split(
            self._h, begin, num, req.data_ptr(), n.data_ptr(), req.stride(0), out.hit_row.data_ptr(),
            out.miss_ids.data_ptr(), out.miss_row.data_ptr(), out.counts.data_ptr(),
            out.miss_ids.stride(0), _lib.stream_handle()), "ess_pool_split")
        return out

    def settle(self, slots: torch.Tensor, counts: torch.Tensor, begin: int = 0) -> None:
        """Fetched miss rows: staging -> their final slots (ess_pool_settle)."""
        num = slots.shape[0]
        self._range(begin, num)
        _lib.check(self._L.ess_pool_settle(self._h, begin, num, slots.data_ptr(), counts.data_ptr(),
                                           slots.stride(0), _lib.stream_handle()), "ess_pool_settle")

    def append(self, ids: torch.Tensor, m: torch.Tensor, begin: int = 0,
               slots: torch.Tensor | None = None) -> torch.Tensor:
        num = ids.shape[0]
        self._range(begin, num)
        if slots is None:
            slots = torch.empty_like(ids)
        _lib.check(self._L.ess_pool_append(self._h, begin, num, ids.data_ptr(), m.data_ptr(),
                                           ids.stride(0), slots.data_ptr(), _lib.stream_handle()))
        return slots

    def lru_order(self, begin: int = 0, num: int | None = None):
        begin, num = self._range(begin, num)
        out = torch.empty((num, self.cap_max), dtype=torch.int32, device=self.device)
        cnt = torch.empty(num, dtype=torch.int32, device=self.device)
        _lib.check(self._L.ess_pool_lru_order(self._h, begin, num, out.data_ptr(), cnt.data_ptr(),
                                              _lib.stream_handle()))
        return out, cnt

    def counters(self, begin: int = 0, num: int | None = None) -> torch.Tensor:
        """[num, 8] int64: capacity, size, hits, misses, evictions, clock, watermark, 0."""
        begin, num = self._range(begin, num)
        out = torch.empty((num, 8), dtype=torch.int64, device=self.device)
        _lib.check(self._L.ess_pool_counters(self._h, begin, num, out.data_ptr(),
                                             _lib.stream_handle()))
        return out

    def lookup(self, pool: int, ids: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(ids)
        _lib.check(self._L.ess_pool_lookup(self._h, pool, ids.data_ptr(), ids.numel(),
                                           out.data_ptr(), _lib.stream_handle()))
        return out

    def copy_from(self, src: "PoolSet", begin: int = 0, src_begin: int = 0, num: int | None = None):
        num = src.num_pools - src_begin if num is None else num
        _lib.check(self._L.ess_pool_copy_state(self._h, begin, src._h, src_begin, num,
                                               _lib.stream_handle()))

    def rows_ptr(self) -> int:
        p = ctypes.c_void_p()
        _lib.check(self._L.ess_pool_info(self._h, None, None, None, None, None, ctypes.byref(p)))
        return p.value or 0

    def rows_view(self) -> torch.Tensor:
        """The slot store as an aliasing view: [P, rows_per_pool, 656] uint8 raw latent rows
        (FP8 slot format), or [P, rows_per_pool, 576] float16 dequantised NoPE (512) ++
        RoPE (64) rows (f16 slot format)."""
        if not self.row_bytes:
            raise ValueError("pool set has no slot store")
        n = self.num_pools * self.rows_per_pool * self.row_bytes
        raw = _wrap_device(self.rows_ptr(), n, self.device, self)
        if self.row_bytes == _lib.SLOT_ROW_BYTES_FP8:
            return raw.view(self.num_pools, self.rows_per_pool, self.row_bytes)
        return raw.view(torch.float16).view(self.num_pools, self.rows_per_pool, self.row_bytes // 2)

    def status(self) -> int:
        st = ctypes.c_int32(0)
        _lib.check(self._L.ess_pool_status(self._h, ctypes.byref(st)))
        return st.value

    def check(self, what: str = "pool") -> None:
        """Synchronise and raise the first error latched by the device."""
        _lib.check(self.status(), what)


class _DevBuf:
    """Minimal __cuda_array_interface__ exporter so torch can alias library memory."""

    def __init__(self, ptr, nbytes, owner):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}
        self._owner = owner


def _wrap_device(ptr: int, nbytes: int, device, owner) -> torch.Tensor:
    with torch.cuda.device(device):
        return torch.as_tensor(_DevBuf(ptr, nbytes, owner), device=device)


# =====================================================================================
# Reference-compatible single pool (cache.py:29-134)
# =====================================================================================

def _runs_without_repeats(ids, limit):
    """Split a touch sequence into maximal duplicate-free chunks of <= limit ids;
    running them in order is exactly the sequential touch order."""
    run, seen = [], set()
    for x in ids:
        if x in seen or len(run) == limit:
            yield run
            run, seen = [], set()
        run.append(x)
        seen.add(x)
    if run:
        yield run


class SparsePool:
    """LRU-ordered set of resident entry ids with a hard slot capacity, on the GPU.

    Same surface as offsim.cache.SparsePool: ``warmup``, ``access_step``,
    ``append_generated``, ``grow_capacity``, ``lru_order``, ``resident_ids``,
    ``len``/``in`` and the ``hits``/``misses``/``evictions`` counters.
    """

    _ID_SPAN = 1 << 16

    def __init__(self, capacity: int, max_ids: int | None = None, cap_max: int | None = None,
                 device=None):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        self._dev = torch.device(device if device is not None else "cuda")
        self._set = PoolSet(1, max_ids or self._ID_SPAN,
                            cap_max or max(2 * capacity, capacity + 1024), capacity,
                            device=self._dev)
        self._cap = int(capacity)

    # -- helpers ------------------------------------------------------------------------
    def _ensure(self, max_id: int = -1, cap: int = 0):
        """Migrate to a larger pool set when an id or the capacity outgrows it."""
        s = self._set
        if max_id < s.max_ids and cap <= s.cap_max:
            return
        new_ids = s.max_ids
        while new_ids <= max_id:
            new_ids *= 2
        new_cap = s.cap_max
        while new_cap < cap:
            new_cap *= 2
        bigger = PoolSet(1, new_ids, new_cap, device=self._dev)
        bigger.copy_from(s)
        s.close()
        self._set = bigger

    def _ids(self, seq) -> list:
        out = [int(x) for x in seq]
        if any(x < 0 for x in out):
            raise ValueError("entry ids must be >= 0")
        return out

    def _counter(self, i: int) -> int:
        return int(self._set.counters()[0, i].item())

    # -- reference surface --------------------------------------------------------------
    @property
    def capacity(self) -> int:
        return self._cap

    @property
    def hits(self) -> int:
        return self._counter(2)

    @property
    def misses(self) -> int:
        return self._counter(3)

    @property
    def evictions(self) -> int:
        return self._counter(4)

    def __len__(self) -> int:
        return self._counter(1)

    def __contains__(self, entry_id) -> bool:
        x = int(entry_id)
        if x < 0 or x >= self._set.max_ids:
            return False
        ids = torch.tensor([x], dtype=torch.int32, device=self._dev)
        return bool(self._set.lookup(0, ids)[0].item() >= 0)

    def lru_order(self) -> list:
        out, cnt = self._set.lru_order()
        return out[0, :int(cnt[0].item())].tolist()

    def resident_ids(self) -> list:
        out, cnt = self._set.lru_order()
        return torch.sort(out[0, :int(cnt[0].item())]).values.tolist()

    def grow_capacity(self, capacity: int) -> None:
        if capacity < self._cap:
            raise ValueError("capacity may only grow")
        self._ensure(cap=capacity)
        self._set.grow(int(capacity))
        self._set.check("grow_capacity")
        self._cap = int(capacity)

    def warmup(self, prefill_windows) -> int:
        inserted = torch.zeros(1, dtype=torch.int64, device=self._dev)
        for window in prefill_windows:
            ids = self._ids(window)
            if not ids:
                continue
            self._ensure(max_id=max(ids))
            for run in _runs_without_repeats(ids, _lib.MAX_REQUEST):
                t = torch.tensor([run], dtype=torch.int32, device=self._dev)
                n = torch.tensor([len(run)], dtype=torch.int32, device=self._dev)
                self._set.warmup(t, n, inserted=inserted)
        self._set.check("warmup")
        return int(inserted.item())

    def access_step(self, requested) -> AccessResult:
        req = self._ids(requested)
        if len(set(req)) != len(req):
            raise ValueError("requested ids must be unique")
        if len(req) > _lib.MAX_REQUEST:
            raise ValueError(f"at most {_lib.MAX_REQUEST} ids per access (top-k bound)")
        if req:
            self._ensure(max_id=max(req))
        K = max(1, len(req))
        t = torch.full((1, K), -1, dtype=torch.int32, device=self._dev)
        if req:
            t[0, :len(req)] = torch.tensor(req, dtype=torch.int32, device=self._dev)
        n = torch.tensor([len(req)], dtype=torch.int32, device=self._dev)
        r = self._set.access(t, n, lists=True)
        self._set.check("access_step")
        c = r.counts[0].tolist()
        return AccessResult(hit_ids=r.hit_ids[0, :c[0]].tolist(),
                            miss_ids=r.miss_ids[0, :c[1]].tolist(),
                            evicted_ids=r.evicted_ids[0, :c[2]].tolist(),
                            h2d_blocks=c[1])

    def append_generated(self, new_ids) -> int:
        ids = self._ids(new_ids)
        if not ids:
            return 0
        self._ensure(max_id=max(ids))
        t = torch.tensor([ids], dtype=torch.int32, device=self._dev)
        m = torch.tensor([len(ids)], dtype=torch.int32, device=self._dev)
        self._set.append(t, m)
        try:
            self._set.check("append_generated")
        except ValueError as e:
            raise ValueError(f"duplicate generated entry id in {ids}") from e
        return len(ids)


# =====================================================================================
# Replay (cache.py:141-196)
# =====================================================================================

@dataclass
class MissProfile:
    """Per-layer, per-step miss counts from a single-request replay."""
    misses: np.ndarray  # (num_layers, num_steps) int64
    sparse_ratio: float

    @property
    def num_layers(self) -> int:
        return self.misses.shape[0]

    @property
    def num_steps(self) -> int:
        return self.misses.shape[1]

    def layer_means(self) -> np.ndarray:
        return self.misses.mean(axis=1)

    def mean_misses(self) -> float:
        return float(self.misses.mean())

    def total_misses(self) -> int:
        return int(self.misses.sum())


def _pad_windows(windows_per_pool, device):
    """List (per pool) of id arrays -> ([P, W] int32 padded, [P] int32 counts)."""
    width = max(1, max(len(w) for w in windows_per_pool))
    a = np.full((len(windows_per_pool), width), -1, np.int32)
    n = np.zeros(len(windows_per_pool), np.int32)
    for i, w in enumerate(windows_per_pool):
        a[i, :len(w)] = w
        n[i] = len(w)
    return torch.as_tensor(a, device=device), torch.as_tensor(n, device=device)


def replay(trace: AccessTrace, sparse_ratio: float, use_warmup: bool = True,
           preload_full_history: bool = False, device=None) -> MissProfile:
    """cache.py:166-196: one pool per layer, all layers stepped per launch."""
    if not (0.0 < sparse_ratio <= 1.0):
        raise ValueError(f"sparse_ratio must be in (0, 1], got {sparse_ratio}")
    dev = torch.device(device if device is not None else "cuda")
    L, T, ctx = trace.num_layers, trace.num_steps, trace.context_len
    total = ctx + sum(s.tokens_accepted for s in trace.steps)
    cap0 = pool_capacity(sparse_ratio, ctx)
    pools = PoolSet(L, max(total, 1), pool_capacity(sparse_ratio, total), cap0, device=dev)
    MAXR = _lib.MAX_REQUEST
    if preload_full_history:
        full = np.arange(ctx, dtype=np.int32)
        for c0 in range(0, ctx, MAXR):
            ids, n = _pad_windows([full[c0:c0 + MAXR]] * L, dev)
            pools.warmup(ids, n)
    elif use_warmup and trace.prefill_windows is not None:
        nwin = max(len(w) for w in trace.prefill_windows)
        for w in range(nwin):
            per = [trace.prefill_windows[l][w] if w < len(trace.prefill_windows[l])
                   else np.zeros(0, np.int32) for l in range(L)]
            width = max(len(x) for x in per)
            for c0 in range(0, max(width, 1), MAXR):
                ids, n = _pad_windows([np.asarray(x[c0:c0 + MAXR], np.int32) for x in per], dev)
                pools.warmup(ids, n)
    # the whole trace goes to the device once; per step: access, grow, append
    K = max(1, max((len(a) for s in trace.steps for a in s.layers), default=1))
    if K > MAXR:
        raise ValueError(f"selection sets longer than {MAXR} are not supported")
    req = np.full((max(T, 1), L, K), -1, np.int32)
    cnt = np.zeros((max(T, 1), L), np.int32)
    for t, s in enumerate(trace.steps):
        for l, a in enumerate(s.layers):
            req[t, l, :len(a)] = a
            cnt[t, l] = len(a)
    d_req, d_cnt = torch.as_tensor(req, device=dev), torch.as_tensor(cnt, device=dev)
    misses = torch.zeros((L, max(T, 1)), dtype=torch.int64, device=dev)
    out = None
    history = ctx
    for t, s in enumerate(trace.steps):
        out = pools.access(d_req[t], d_cnt[t], out=out)
        misses[:, t] = out.counts[:, 1]
        acc = s.tokens_accepted
        new = torch.arange(history, history + acc, dtype=torch.int32, device=dev).expand(L, acc)
        history += acc
        pools.grow(pool_capacity(sparse_ratio, history))
        if acc:
            pools.append(new.contiguous(), torch.full((L,), acc, dtype=torch.int32, device=dev))
    pools.check("replay")
    prof = misses[:, :T].cpu().numpy()
    pools.close()
    return MissProfile(misses=prof, sparse_ratio=sparse_ratio)


def write_miss_profile_csv(profile: MissProfile, path) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["layer", "step", "misses"])
        for l in range(profile.num_layers):
            for t in range(profile.num_steps):
                w.writerow([l, t, int(profile.misses[l, t])])


def write_miss_summary_csv(profile: MissProfile, path) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["layer", "mean_misses", "min", "max"])
        for l in range(profile.num_layers):
            row = profile.misses[l]
            w.writerow([l, f"{row.mean():.6f}", int(row.min()), int(row.max())])


def read_miss_profile_csv(path) -> MissProfile:
    with open(path, newline="") as f:
        recs = [(int(r["layer"]), int(r["step"]), int(r["misses"])) for r in csv.DictReader(f)]
    if not recs:
        raise ValueError(f"empty miss profile: {path}")
    m = np.zeros((max(r[0] for r in recs) + 1, max(r[1] for r in recs) + 1), np.int64)
    for l, t, v in recs:
        m[l, t] = v
    return MissProfile(misses=m, sparse_ratio=float("nan"))
