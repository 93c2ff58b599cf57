"""Third-party comparators for the DSA operators (test / bench infrastructure only —
never on the product path).

The reference (offsim) has no code for the indexer, top-k or sparse-attention values
(SURVEY §8c), so these public implementations that ship in this image pin the
restated oracle (oracle/dsa.py) and serve as the speed bar for K2 / K5:

  * FlashMLA sparse decode (vLLM's vendored build, ``vllm._flashmla_C``): DeepSeek's own
    V3.2 DSA decode kernel, reading the same 656-B FP8 latent rows (512 e4m3 NoPE, 4 f32
    group scales, 64 bf16 RoPE) through a top-k index list — what K5 computes.
  * DeepGEMM's torch reference of the lightning indexer, ``fp8_mqa_logits_torch``
    (vLLM, v1/attention/ops/rocm_aiter_mla_sparse.py) — what K1 computes.
  * flashinfer ``top_k`` with the small-index tie break — what K2 computes.
"""

from __future__ import annotations

import torch


def flashmla_available() -> bool:
    try:
        import vllm._flashmla_C  # noqa: F401
        return torch.cuda.is_available() and torch.cuda.get_device_capability()[0] == 10
    except Exception:
        return False


def flashmla_sparse_decode(q: torch.Tensor, kv_rows: torch.Tensor, indices: torch.Tensor,
                           sm_scale: float, lengths: torch.Tensor | None = None,
                           block: int = 64, meta=None):
    """q [B, 128, 576] bf16; kv_rows [N, 656] uint8 latent rows (N % block == 0);
    indices [B, k] int32 row numbers into kv_rows.  Returns (out [B, 128, 512] bf16,
    lse [B, 128] f32 natural log, meta) — meta is FlashMLA's scheduler state, reusable
    for calls of the same shapes."""
    from vllm.third_party.flashmla.flash_mla_interface import flash_mla_with_kvcache, get_mla_metadata
    B = q.shape[0]
    N = kv_rows.shape[0]
    assert N % block == 0 and kv_rows.shape[1] == 656
    k_cache = kv_rows.view(torch.float8_e4m3fn).view(N // block, block, 1, 656)
    if meta is None:
        meta, _ = get_mla_metadata()
    out, lse = flash_mla_with_kvcache(q.view(B, 1, 128, 576), k_cache, None, None, 512, meta,
                                      softmax_scale=sm_scale, is_fp8_kvcache=True,
                                      indices=indices.view(B, 1, -1), topk_length=lengths)
    return out.view(B, 128, 512), lse.view(B, 128), meta


def fp8_mqa_logits_reference(q_u8: torch.Tensor, k_u8: torch.Tensor, kscale: torch.Tensor,
                             w: torch.Tensor, length: int) -> torch.Tensor:
    """DeepGEMM's torch reference of the indexer for one request (CPU or GPU):
    q [64, 128] e4m3 bytes, k [L, 128] e4m3 bytes, kscale [L] f32, w [64] f32."""
    from vllm.v1.attention.ops.rocm_aiter_mla_sparse import fp8_mqa_logits_torch
    q = q_u8.view(torch.float8_e4m3fn)[None]
    k = k_u8[:length].view(torch.float8_e4m3fn)
    ks = torch.zeros(1, dtype=torch.int32, device=q.device)
    ke = torch.full((1,), length, dtype=torch.int32, device=q.device)
    return fp8_mqa_logits_torch(q, (k, kscale[:length].float()), w.float()[None], ks, ke)[0]


def flashinfer_topk_sets(logits: torch.Tensor, lens, k: int):
    """flashinfer top_k (small-index tie break) per row, as ascending id arrays."""
    import flashinfer
    from flashinfer.topk import TopKTieBreak
    out = []
    for b, n in enumerate(lens):
        n = int(n)
        if n <= k:
            out.append(torch.arange(n, dtype=torch.int64))
            continue
        _, idx = flashinfer.top_k(logits[b:b + 1, :n].contiguous(), k, tie_break=TopKTieBreak.SMALL)
        out.append(torch.sort(idx[0].long().cpu()).values)
    return out
