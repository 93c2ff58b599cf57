"""Lightning indexer (K1) and top-k selection (K2) — the two operators the
reference reduces to the cost entries ``indexer_logits`` / ``indexer_topk``
(/root/reference/pkg/src/offsim/costmodel.py:18-27, used at pipeline.py:215-216).

K2's output is the canonical selection set of ``AccessTrace`` (trace.py:31-46):
ascending unique ids, |set| = min(k, len) (scenario.py:110-112).
"""

from __future__ import annotations

import torch

from . import _lib

HEADS = 64
DIM = 128
TOPK = 2048


def indexer_logits(q_fp8: torch.Tensor, w: torch.Tensor, k_cache: torch.Tensor,
                   k_scale: torch.Tensor, lens: torch.Tensor,
                   out: torch.Tensor | None = None, max_ctas: int = 0, pdl: bool = False) -> torch.Tensor:
    """logits[b, s] = k_scale[b, s] * sum_h w[b, h] * relu(q[b, h] . k[b, s]) for s < lens[b].

    q_fp8 [B, 64, 128] and k_cache [B, Lmax, 128] hold e4m3 bytes (uint8 or
    float8_e4m3fn), w [B, 64] f32, k_scale [B, Lmax] f32, lens [B] int32.
    Lmax must be a multiple of 128 and k_cache 16-byte aligned (TMA).
    Entries at s >= lens[b] are left untouched.  ``max_ctas`` > 0 caps the
    persistent grid (SMs left free for a concurrent gather); 0 = every SM.  ``pdl``:
    programmatic dependent launch (ESS_LAUNCH_PDL) behind the previous kernel of the
    stream, whose results K1 does not read.
    """
    _lib.require_cuda(k_cache)
    if k_cache.dim() != 3:
        raise ValueError("expected k [B,Lmax,128]")
    B, Lmax, D = k_cache.shape
    if D != DIM or Lmax % 128:
        raise ValueError("expected k [B,Lmax,128] with Lmax a multiple of 128")
    dev = k_cache.device
    fp8 = (torch.uint8, torch.float8_e4m3fn)
    _lib.check_tensor(k_cache, "k_cache", fp8, device=dev)
    _lib.check_tensor(q_fp8, "q_fp8", fp8, (B, HEADS, DIM), device=dev)
    _lib.check_tensor(w, "w", torch.float32, (B, HEADS), device=dev)
    _lib.check_tensor(k_scale, "k_scale", torch.float32, (B, Lmax), device=dev)
    _lib.check_tensor(lens, "lens", torch.int32, (B,), device=dev)
    if out is None:
        out = torch.empty((B, Lmax), dtype=torch.float32, device=dev)
    _lib.check_tensor(out, "out", torch.float32, (B, Lmax), device=dev)
    _lib.check(_lib.load().ess_indexer_logits_ex(
        q_fp8.data_ptr(), w.data_ptr(), k_cache.data_ptr(), k_scale.data_ptr(), lens.data_ptr(),
        B, Lmax, out.data_ptr(), max_ctas | (_lib.ESS_LAUNCH_PDL if pdl else 0), _lib.stream_handle()),
        "ess_indexer_logits")
    return out


def indexer_logits_mtp(q_fp8: torch.Tensor, w: torch.Tensor, k_cache: torch.Tensor,
                       k_scale: torch.Tensor, lens: torch.Tensor,
                       out: torch.Tensor | None = None, max_ctas: int = 0) -> torch.Tensor:
    """MTP indexer: ``qtok`` = mtp + 1 query tokens per request (pipeline.py:213-215).

    logits[b, j, s] = k_scale[b, s] * sum_h w[b, j, h] * relu(q[b, j, h] . k[b, s]), s < lens[b]
    with q_fp8 [B, qtok, 64, 128] e4m3, w [B, qtok, 64] f32, out [B, qtok, Lmax] f32.
    Every token of a request scores the same cached keys (the selection universe is the
    cache history, trace.py:151-154); the keys are read once per request."""
    _lib.require_cuda(k_cache)
    if k_cache.dim() != 3 or q_fp8.dim() != 4:
        raise ValueError("expected k [B,Lmax,128] and q [B,qtok,64,128]")
    B, Lmax, D = k_cache.shape
    qtok = q_fp8.shape[1]
    if D != DIM or Lmax % 128:
        raise ValueError("expected k [B,Lmax,128] with Lmax a multiple of 128")
    if not 1 <= qtok <= _lib.MAX_QTOK:
        raise ValueError(f"qtok must be in [1, {_lib.MAX_QTOK}]")
    dev = k_cache.device
    fp8 = (torch.uint8, torch.float8_e4m3fn)
    _lib.check_tensor(k_cache, "k_cache", fp8, device=dev)
    _lib.check_tensor(q_fp8, "q_fp8", fp8, (B, qtok, HEADS, DIM), device=dev)
    _lib.check_tensor(w, "w", torch.float32, (B, qtok, HEADS), device=dev)
    _lib.check_tensor(k_scale, "k_scale", torch.float32, (B, Lmax), device=dev)
    _lib.check_tensor(lens, "lens", torch.int32, (B,), device=dev)
    if out is None:
        out = torch.empty((B, qtok, Lmax), dtype=torch.float32, device=dev)
    _lib.check_tensor(out, "out", torch.float32, (B, qtok, Lmax), device=dev)
    _lib.check(_lib.load().ess_indexer_logits_mtp(
        q_fp8.data_ptr(), w.data_ptr(), k_cache.data_ptr(), k_scale.data_ptr(), lens.data_ptr(),
        B, qtok, Lmax, out.data_ptr(), max_ctas, _lib.stream_handle()), "ess_indexer_logits_mtp")
    return out


def topk_mtp(logits: torch.Tensor, lens: torch.Tensor, k: int = TOPK,
             out: torch.Tensor | None = None, count: torch.Tensor | None = None):
    """Top-k of every query token's row: logits [B, qtok, ld] (indexer_logits_mtp),
    row (b, j) over lens[b] tokens.  Returns (idx [B, qtok, k], count [B, qtok])."""
    _lib.require_cuda(logits)
    if logits.dim() != 3 or logits.dtype != torch.float32 or not logits.is_contiguous():
        raise ValueError("logits must be a contiguous CUDA float32 [B, qtok, ld] tensor")
    B, qtok, ld = logits.shape
    if not 1 <= qtok <= _lib.MAX_QTOK:
        raise ValueError(f"qtok must be in [1, {_lib.MAX_QTOK}]")
    _lib.check_tensor(lens, "lens", torch.int32, (B,), device=logits.device)
    if not 1 <= k <= 65535:
        raise ValueError("k must be in [1, 65535]")
    if out is None:
        out = torch.empty((B, qtok, k), dtype=torch.int32, device=logits.device)
    if count is None:
        count = torch.empty((B, qtok), dtype=torch.int32, device=logits.device)
    _lib.check_tensor(out, "out", torch.int32, (B, qtok, k), device=logits.device)
    _lib.check_tensor(count, "count", torch.int32, (B, qtok), device=logits.device)
    _lib.check(_lib.load().ess_topk_mtp(logits.data_ptr(), ld, lens.data_ptr(), B, qtok, k,
                                        out.data_ptr(), k, count.data_ptr(), _lib.stream_handle()),
               "ess_topk_mtp")
    return out, count


def topk(logits: torch.Tensor, lens: torch.Tensor, k: int = TOPK,
         out: torch.Tensor | None = None, count: torch.Tensor | None = None):
    """Top-k of each row logits[b, :lens[b]] by (score desc, index asc), ascending ids.

    Returns (idx [B, k] int32, count [B] int32) with count = min(k, lens)."""
    _lib.require_cuda(logits)
    B, ld = _check_topk_args(logits, lens, k)
    if out is None:
        out = torch.empty((B, k), dtype=torch.int32, device=logits.device)
    if count is None:
        count = torch.empty(B, dtype=torch.int32, device=logits.device)
    _check_topk_out(out, count, B, k, logits.device)
    _lib.check(_lib.load().ess_topk(logits.data_ptr(), logits.stride(0), lens.data_ptr(), B, k,
                                    out.data_ptr(), out.stride(0), count.data_ptr(),
                                    _lib.stream_handle()), "ess_topk")
    return out, count


def topk_split(logits: torch.Tensor, lens: torch.Tensor, k: int, out: torch.Tensor, count: torch.Tensor,
               pool, acc, begin: int = 0, pdl: bool = False):
    """K2 fused with the early-gather hit/miss split of pools [begin, begin + B)
    (ess_topk_split_ex): selection ids into ``out``/``count``; hit rows, miss ids, staging
    rows and counts into ``acc`` (an AccessBatch of row slices).  ``pdl``: launched
    programmatically behind the indexer on the same stream (waits for it on the device)."""
    _lib.require_cuda(logits)
    B, ld = _check_topk_args(logits, lens, k)
    _check_topk_out(out, count, B, k, logits.device)
    for name in ("hit_row", "miss_ids", "miss_row"):
        t = getattr(acc, name)
        _lib.check_tensor(t, f"acc.{name}", torch.int32, (B, None), contiguous=False, device=logits.device)
        if t.stride(1) != 1 or t.stride(0) != acc.miss_ids.stride(0) or t.shape[1] < k:
            raise ValueError(f"acc.{name} rows must be unit-stride, share one row stride and hold k ids")
    _lib.check_tensor(acc.counts, "acc.counts", torch.int32, (B, 4), device=logits.device)
    _lib.check(_lib.load().ess_topk_split_ex(
        logits.data_ptr(), logits.stride(0), lens.data_ptr(), B, k, out.data_ptr(), out.stride(0),
        count.data_ptr(), pool.handle, begin, acc.hit_row.data_ptr(), acc.miss_ids.data_ptr(),
        acc.miss_row.data_ptr(), acc.counts.data_ptr(), acc.miss_ids.stride(0),
        _lib.ESS_LAUNCH_PDL if pdl else 0, _lib.stream_handle()), "ess_topk_split")
    return out, count


def _check_topk_args(logits, lens, k):
    if logits.dim() != 2 or logits.dtype != torch.float32 or logits.stride(1) != 1 or not logits.is_cuda:
        raise ValueError("logits must be a CUDA float32 [B, ld] tensor with unit column stride")
    B, ld = logits.shape
    _lib.check_tensor(lens, "lens", torch.int32, (B,), device=logits.device)
    if not 1 <= k <= 65535:
        raise ValueError("k must be in [1, 65535]")
    return B, ld


def _check_topk_out(out, count, B, k, device):
    _lib.check_tensor(out, "out", torch.int32, (B, None), contiguous=False, device=device)
    if out.stride(1) != 1 or out.shape[1] < k:
        raise ValueError("out must be int32 [B, >= k] with unit column stride")
    _lib.check_tensor(count, "count", torch.int32, (B,), device=device)


def indexer_logits_stream(q_fp8, w, k_cache, k_scale, lens, out, done, group: int, max_ctas: int):
    """K1 of the streamed step (ess_indexer_logits_stream): requests in groups of ``group``
    with the whole grid, per-request completion counters ``done`` (int32 [B], zero at
    launch) for the concurrent streamed top-k.  Shapes as ``indexer_logits``."""
    _lib.require_cuda(k_cache)
    B, Lmax, _ = k_cache.shape
    _lib.check_tensor(q_fp8, "q_fp8", (torch.uint8, torch.float8_e4m3fn), (B, HEADS, DIM), device=k_cache.device)
    _lib.check_tensor(w, "w", torch.float32, (B, HEADS), device=k_cache.device)
    _lib.check_tensor(k_scale, "k_scale", torch.float32, (B, Lmax), device=k_cache.device)
    _lib.check_tensor(lens, "lens", torch.int32, (B,), device=k_cache.device)
    _lib.check_tensor(out, "out", torch.float32, (B, Lmax), device=k_cache.device)
    _lib.check_tensor(done, "done", torch.int32, (B,), device=k_cache.device)
    _lib.check(_lib.load().ess_indexer_logits_stream(
        q_fp8.data_ptr(), w.data_ptr(), k_cache.data_ptr(), k_scale.data_ptr(), lens.data_ptr(), B, Lmax,
        out.data_ptr(), max_ctas, group, done.data_ptr(), _lib.stream_handle()), "ess_indexer_logits_stream")
    return out


def topk_split_stream(logits, lens, k: int, out, count, pool, acc, done, ready, ctas: int, begin: int = 0):
    """K2 + K3a of the streamed step (ess_topk_split_stream): ``ctas`` persistent CTAs take
    the requests in order, each once ``done`` says its logits are complete; ``ready``
    (int32 [B], zero at launch) is set per request when its split is stored."""
    _lib.require_cuda(logits)
    B, ld = _check_topk_args(logits, lens, k)
    _check_topk_out(out, count, B, k, logits.device)
    for name in ("hit_row", "miss_ids", "miss_row"):
        t = getattr(acc, name)
        if t.stride(1) != 1 or t.stride(0) != acc.miss_ids.stride(0) or t.shape[1] < k:
            raise ValueError(f"acc.{name} rows must be unit-stride, share one row stride and hold k ids")
    _lib.check_tensor(done, "done", torch.int32, (B,), device=logits.device)
    _lib.check_tensor(ready, "ready", torch.int32, (B,), device=logits.device)
    _lib.check(_lib.load().ess_topk_split_stream(
        logits.data_ptr(), logits.stride(0), lens.data_ptr(), B, k, out.data_ptr(), out.stride(0),
        count.data_ptr(), pool.handle, begin, acc.hit_row.data_ptr(), acc.miss_ids.data_ptr(),
        acc.miss_row.data_ptr(), acc.counts.data_ptr(), acc.miss_ids.stride(0), done.data_ptr(),
        ready.data_ptr(), ctas, _lib.stream_handle()), "ess_topk_split_stream")
    return out, count
