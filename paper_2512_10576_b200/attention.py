"""Sparse MLA decode (K5) over the GPU slot store — the operators the reference
reduces to ``op_time("sparse_mla" | "merge_attn", ...)`` (costmodel.py:18-27,
pipeline.py:217-219) and the DA split (Attn0 on resident rows while the misses
are fetched, Attn1 on the fetched rows, merge; PAPER.md:350-352,
pipeline.py:125-141).
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .cache import PoolSet

HEADS = 128
QK_DIM = 576
V_DIM = 512
# DeepSeek-V3.2 MLA: softmax scale over the 192-d (128 NoPE + 64 RoPE) qk head dim
DEFAULT_SM_SCALE = 1.0 / math.sqrt(192.0)


class SplitWorkspace:
    """Carry-over state between the two attention passes: unnormalised O (f32) and
    the running (max, sum) per head."""

    def __init__(self, batch: int, device, splits: int = 1):
        self.splits = splits
        self.o = torch.empty((batch * splits, HEADS, V_DIM), dtype=torch.float32, device=device)
        self.ml = torch.empty((batch * splits, HEADS, 2), dtype=torch.float32, device=device)


def sparse_mla(pool: PoolSet, q: torch.Tensor, sel_row: torch.Tensor, count: torch.Tensor,
               sm_scale: float = DEFAULT_SM_SCALE, pool_begin: int = 0,
               out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
               workspace: SplitWorkspace | None = None, mode: str = "full", split: int = 1,
               qtok: int = 1):
    """out[b, h] = softmax_j(q[b, h] . K_j * sm_scale) V_j over rows sel_row[b, :count[b]]
    of pool (pool_begin + b)'s slot store.

    q [B, 128, 576] bf16; ``count`` may be a strided view (e.g. AccessBatch.counts[:, 0]).
    mode "full" returns (out [B, 128, 512] bf16, lse [B, 128] f32, natural log);
    "partial" stores the unnormalised state into ``workspace`` (Attn0); "resume"
    continues from it over further rows and returns the merged result (Attn1 + merge).
    ``split`` > 1 (full mode) cuts each request's rows into that many shares on
    2 * split CTAs and merges them (``workspace`` with ``splits >= split``): small batches.
    ``qtok`` > 1 (MTP): q rows are (request, query token) pairs, B = requests * qtok; row r
    attends over sel_row[r, :count[r]] in pool pool_begin + r // qtok.
    """
    _lib.require_cuda(q)
    B = q.shape[0]
    if q.shape != (B, HEADS, QK_DIM) or q.dtype != torch.bfloat16:
        raise ValueError("q must be [B, 128, 576] bfloat16")
    flags = {"full": 0, "partial": _lib.ESS_MLA_PARTIAL, "resume": _lib.ESS_MLA_RESUME}[mode]
    if flags and workspace is None:
        raise ValueError(f"mode {mode!r} needs a SplitWorkspace")
    if not 1 <= qtok <= _lib.MAX_QTOK or B % qtok:
        raise ValueError(f"qtok must be in [1, {_lib.MAX_QTOK}] and divide the {B} query rows")
    flags |= (qtok - 1) << _lib.ESS_MLA_QTOK_SHIFT
    if not 1 <= split <= _lib.ESS_MLA_MAX_SPLIT:
        raise ValueError(f"split must be in [1, {_lib.ESS_MLA_MAX_SPLIT}]")
    if split > 1:
        if mode != "full" or workspace is None or workspace.splits < split or workspace.o.shape[0] < B * split:
            raise ValueError("split > 1 needs mode 'full' and a SplitWorkspace(batch, splits >= split)")
        flags |= (split - 1) << _lib.ESS_MLA_SPLIT_SHIFT
    if mode != "partial":
        if out is None:
            out = torch.empty((B, HEADS, V_DIM), dtype=torch.bfloat16, device=q.device)
        if lse is None:
            lse = torch.empty((B, HEADS), dtype=torch.float32, device=q.device)
    ws_o = _lib.ptr(workspace.o) if workspace is not None else None
    ws_ml = _lib.ptr(workspace.ml) if workspace is not None else None
    _lib.check(_lib.load().ess_sparse_mla(
        pool.handle, pool_begin, q.data_ptr(), sel_row.data_ptr(), sel_row.stride(0),
        count.data_ptr(), count.stride(0), B, float(sm_scale), _lib.ptr(out), _lib.ptr(lse),
        ws_o, ws_ml, flags, _lib.stream_handle()), "ess_sparse_mla")
    return out, lse


def sparse_mla_da(pool: PoolSet, q: torch.Tensor, acc, landed: torch.Tensor,
                  sm_scale: float = DEFAULT_SM_SCALE, pool_begin: int = 0,
                  out: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                  split: int = 1, workspace: SplitWorkspace | None = None):
    """The DA schedule as one launch: attention over the resident
    rows ``acc.hit_row[b, :counts[b, 0]]``, then — once ``landed[b]`` reaches
    ``counts[b, 1]`` — over the fetched rows ``acc.miss_row[b, :counts[b, 1]]`` that a
    concurrent ``gather(..., landed=landed)`` is writing.  Same (out, lse) as
    ``sparse_mla`` over the union; no workspace round trip, no second prologue.
    The gather must run concurrently on the SMs this launch leaves free.  ``landed``
    starts zeroed; the kernel leaves it zero again for the next step.  ``split`` > 1
    spreads each request's rows over 2 * split CTAs (small batches) and merges them
    through ``workspace`` (SplitWorkspace(batch, splits >= split))."""
    _lib.require_cuda(q)
    B = q.shape[0]
    if q.shape != (B, HEADS, QK_DIM) or q.dtype != torch.bfloat16:
        raise ValueError("q must be [B, 128, 576] bfloat16")
    if acc.hit_row.stride(0) != acc.miss_row.stride(0):
        raise ValueError("hit_row and miss_row must share a row stride")
    if landed.dtype != torch.int32 or landed.numel() < B:
        raise ValueError("landed must be int32 with one counter per request")
    if split > 1 and (workspace is None or workspace.splits < split or workspace.o.shape[0] < B * split):
        raise ValueError("split > 1 needs a SplitWorkspace(batch, splits >= split)")
    if out is None:
        out = torch.empty((B, HEADS, V_DIM), dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty((B, HEADS), dtype=torch.float32, device=q.device)
    ws_o = _lib.ptr(workspace.o) if workspace is not None else None
    ws_ml = _lib.ptr(workspace.ml) if workspace is not None else None
    _lib.check(_lib.load().ess_sparse_mla_da_split(
        pool.handle, pool_begin, q.data_ptr(), acc.hit_row.data_ptr(), acc.miss_row.data_ptr(),
        acc.hit_row.stride(0), acc.counts.data_ptr(), acc.counts.stride(0), landed.data_ptr(), B,
        float(sm_scale), out.data_ptr(), lse.data_ptr(), ws_o, ws_ml, int(split),
        _lib.stream_handle()), "ess_sparse_mla_da")
    return out, lse
