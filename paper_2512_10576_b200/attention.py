"""Sparse MLA decode (K5) over the GPU slot store — the operator the reference
reduces to ``op_time("sparse_mla", ...)`` (costmodel.py:18-27, pipeline.py:217-218).
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


def sparse_mla(pool: PoolSet, q: torch.Tensor, sel_row: torch.Tensor, count: torch.Tensor,
               sm_scale: float = DEFAULT_SM_SCALE, pool_begin: int = 0,
               out: torch.Tensor | None = None, lse: torch.Tensor | None = None):
    """out[b, h] = softmax_j(q[b, h] . K_j * sm_scale) V_j over rows sel_row[b, :count[b]]
    of pool (pool_begin + b)'s slot store.

    q [B, 128, 576] bf16; returns (out [B, 128, 512] bf16, lse [B, 128] f32, natural log).
    """
    _lib.require_cuda(q)
    B = q.shape[0]
    if q.shape != (B, HEADS, QK_DIM) or q.dtype != torch.bfloat16:
        raise ValueError("q must be [B, 128, 576] bfloat16")
    if out is None:
        out = torch.empty((B, HEADS, V_DIM), dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty((B, HEADS), dtype=torch.float32, device=q.device)
    _lib.check(_lib.load().ess_sparse_mla(
        pool.handle, pool_begin, q.data_ptr(), sel_row.data_ptr(), sel_row.stride(0),
        count.data_ptr(), B, float(sm_scale), out.data_ptr(), lse.data_ptr(),
        _lib.stream_handle()), "ess_sparse_mla")
    return out, lse
