"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(), bench.py
cpu_baseline / --impl reference).  Never imported by the product path.

numpy restatement of the three DSA operators that the reference reduces to cost
scalars (``op_time("indexer_logits"|"indexer_topk"|"sparse_mla", ...)``,
/root/reference/pkg/src/offsim/costmodel.py:18-27, consumed at
pkg/src/offsim/pipeline.py:207-224).  The reference holds NO code for their
values, so these restatements follow the DeepSeek-V3.2-Exp DSA definition and
are pinned only to the reference's sizes: top-k 2048 (scenario.py:24), the
K <= len clamp (scenario.py:110-112), the 656-byte latent block
(scenario.py:25, costmodel.py:31) and the 132-byte indexer entry implied by
scenario.py:30-33.  PARITY UNPINNED for indexer scores and attention values
(see DESIGN.md §3); top-k is pinned to the tie rule recorded in DESIGN.md
(score descending, index ascending; the reference's generator uses
``argpartition`` + ``sort`` with no tie rule, trace.py:107-112, :139-146).

Byte layouts (shared with the CUDA kernels, see include/ess_b200.h):
  latent row (656 B): [0,512) e4m3 NoPE | [512,528) 4 x fp32 group scales
                      (one per 128 NoPE elements) | [528,656) 64 x bf16 RoPE
  indexer key: 128 x e4m3 + one fp32 scale per token (separate arrays)
"""

from __future__ import annotations

import numpy as np

LATENT_ROW_BYTES = 656
NOPE_DIM = 512
ROPE_DIM = 64
NOPE_GROUP = 128
INDEXER_HEADS = 64
INDEXER_DIM = 128


def _e4m3_table() -> np.ndarray:
    """Value of every e4m3fn byte (bias 7, no inf, 0x7F/0xFF = NaN)."""
    t = np.zeros(256, np.float32)
    for b in range(256):
        s = -1.0 if b & 0x80 else 1.0
        e = (b >> 3) & 0xF
        m = b & 0x7
        if e == 0xF and m == 0x7:
            t[b] = np.nan
        elif e == 0:
            t[b] = s * (m / 8.0) * 2.0 ** -6
        else:
            t[b] = s * (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return t


E4M3 = _e4m3_table()


def e4m3_decode(u8: np.ndarray) -> np.ndarray:
    return E4M3[np.asarray(u8, dtype=np.uint8)]


def bf16_decode(u16: np.ndarray) -> np.ndarray:
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# --------------------------------------------------------------------------------------
# K1 lightning indexer
# --------------------------------------------------------------------------------------

def indexer_logits(q_u8, w, k_u8, kscale, length: int) -> np.ndarray:
    """logits[s] = kscale[s] * sum_h w[h] * relu(q[h] . k[s]), s < length, fp32.

    q_u8 [64,128] e4m3 bytes, w [64] f32, k_u8 [>=length,128] e4m3 bytes,
    kscale [>=length] f32.  Accumulates in float64 and rounds once, so it is the
    exact value whenever the operands are small integers/powers of two (the
    exact-arithmetic regime the tests use for bit-exact checks).
    """
    q = e4m3_decode(q_u8).astype(np.float64)
    k = e4m3_decode(k_u8[:length]).astype(np.float64)
    dots = k @ q.T                                   # [len, 64]
    s = np.maximum(dots, 0.0) @ np.asarray(w, np.float64)
    return (s * np.asarray(kscale[:length], np.float64)).astype(np.float32)


# --------------------------------------------------------------------------------------
# K2 top-k
# --------------------------------------------------------------------------------------

def topk_indices(logits, length: int, k: int) -> np.ndarray:
    """Top-k of logits[:length] by (score desc, index asc), returned ascending.

    -0.0 and +0.0 compare equal (IEEE), which is what the kernel's key
    canonicalisation implements.  len <= k returns arange(len)
    (scenario.py:110-112 clamp).
    """
    x = np.asarray(logits[:length], np.float32) + np.float32(0.0)
    if length <= k:
        return np.arange(length, dtype=np.int32)
    order = np.lexsort((np.arange(length), -x.astype(np.float64)))
    return np.sort(order[:k]).astype(np.int32)


# --------------------------------------------------------------------------------------
# K5 sparse MLA decode
# --------------------------------------------------------------------------------------

def unpack_latent_rows(rows_u8: np.ndarray):
    """[n, 656] bytes -> (k_nope [n,512] f32 dequantised, k_rope [n,64] f32)."""
    rows_u8 = np.ascontiguousarray(rows_u8, dtype=np.uint8)
    n = rows_u8.shape[0]
    nope = e4m3_decode(rows_u8[:, :NOPE_DIM])
    scales = rows_u8[:, NOPE_DIM:NOPE_DIM + 16].copy().view(np.float32).reshape(n, 4)
    k_nope = nope * np.repeat(scales, NOPE_GROUP, axis=1)
    rope = rows_u8[:, NOPE_DIM + 16:].copy().view(np.uint16).reshape(n, ROPE_DIM)
    return k_nope.astype(np.float32), bf16_decode(rope)


def slot_rows(rows_u8: np.ndarray) -> np.ndarray:
    """[n, 656] latent rows -> [n, 576] f16 slot rows, the GPU slot-store format
    (include/ess_b200.h): NoPE = f16(f32(e4m3) * f32 scale), RoPE = f16(bf16)."""
    rows_u8 = np.ascontiguousarray(rows_u8, dtype=np.uint8)
    n = rows_u8.shape[0]
    nope = e4m3_decode(rows_u8[:, :NOPE_DIM]).astype(np.float32)
    scales = rows_u8[:, NOPE_DIM:NOPE_DIM + 16].copy().view(np.float32).reshape(n, 4)
    k_nope = (nope * np.repeat(scales, NOPE_GROUP, axis=1)).astype(np.float16)
    rope = bf16_decode(rows_u8[:, NOPE_DIM + 16:].copy().view(np.uint16).reshape(n, ROPE_DIM))
    return np.concatenate([k_nope, rope.astype(np.float16)], axis=1)


def sparse_mla(q: np.ndarray, rows_u8: np.ndarray, sm_scale: float):
    """One request: q [H, 576] f32 (bf16 values), rows_u8 [n, 656] selected rows.

    Returns (out [H, 512] f32, lse [H] f32, natural log).  fp64 internally.
    """
    k_nope, k_rope = unpack_latent_rows(rows_u8)
    K = np.concatenate([k_nope, k_rope], axis=1).astype(np.float64)   # [n, 576]
    s = (np.asarray(q, np.float64) @ K.T) * sm_scale                # [H, n]
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    denom = p.sum(axis=1, keepdims=True)
    out = (p / denom) @ k_nope.astype(np.float64)
    lse = (np.log(denom) + m)[:, 0]
    return out.astype(np.float32), lse.astype(np.float32)


def sparse_mla_on_slot_rows(q: np.ndarray, slot_f16: np.ndarray, sm_scale: float):
    """fp64 attention over rows ALREADY in the kernel's operand precision: slot_f16
    [n, 576] f16 (= slot_rows(), the exact K / V values K5's tensor cores multiply;
    V = the first 512 columns).  The K5 tests compare against this, so the tolerance
    only has to cover K5's own roundings (P to f16, the bf16 output), not the f16
    dequantisation of the rows."""
    K = np.asarray(slot_f16, np.float64)
    s = (np.asarray(q, np.float64) @ K.T) * sm_scale
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    denom = p.sum(axis=1, keepdims=True)
    out = (p / denom) @ K[:, :NOPE_DIM]
    lse = (np.log(denom) + m)[:, 0]
    return out.astype(np.float32), lse.astype(np.float32)
