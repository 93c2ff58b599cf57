"""Third-party golden vectors pinning oracle/dsa.py (the reference has no
code for the DSA operator values, so public implementations that ship in this image
pin the restatement instead).

    python tests/golden/make_dsa_golden.py indexer      (here, CPU: imports vLLM)
    python tests/golden/make_dsa_golden.py flashmla     (on the B200: FlashMLA kernel)

indexer  -> tests/golden/dsa_indexer_deepgemm.npz: DeepGEMM's torch reference of the
            lightning indexer as vendored by vLLM (``fp8_mqa_logits_torch``,
            vllm/v1/attention/ops/rocm_aiter_mla_sparse.py; vLLM 0.22 in this image) on
            an exact-arithmetic case (small-integer e4m3, power-of-two weights / scales)
            and a random case.  Its scores go through bf16 (einsum of bf16 operands), so
            the random case pins the formula to bf16 precision; the exact case bit for bit.
flashmla -> tests/golden/dsa_attention_flashmla.npz: FlashMLA's sm100 FP8 sparse decode
            (``vllm._flashmla_C`` sparse_decode_fwd, DeepSeek's V3.2 DSA kernel) over
            656-B latent rows with power-of-two group scales, 128 heads, top-512 of 1024.
"""
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def e4m3(x):
    return x.clamp(-448, 448).to(torch.float8_e4m3fn).view(torch.uint8)


def make_indexer(out_dir):
    import thirdparty as tp
    g = torch.Generator().manual_seed(5)
    cases = {}
    L = 700
    # exact regime: q.k <= 128 in magnitude (exact in bf16), power-of-two w and scales
    q = e4m3(torch.randint(-1, 2, (64, 128), generator=g).float())
    k = e4m3(torch.randint(-1, 2, (L, 128), generator=g).float())
    w = torch.exp2(torch.randint(-6, 0, (64,), generator=g).float()) * (torch.randint(0, 2, (64,), generator=g) * 2 - 1)
    ks = torch.exp2(torch.randint(-4, 2, (L,), generator=g).float())
    cases["exact"] = (q, k, w, ks)
    q = e4m3(torch.randn((64, 128), generator=g) * 2)
    k = e4m3(torch.randn((L, 128), generator=g) * 2)
    w = torch.randn(64, generator=g) / 8
    ks = torch.rand(L, generator=g) + 0.5
    cases["random"] = (q, k, w, ks)
    arrays = {}
    for name, (q, k, w, ks) in cases.items():
        ref = tp.fp8_mqa_logits_reference(q, k, ks, w, L)
        arrays.update({f"{name}_q": q.numpy(), f"{name}_k": k.numpy(), f"{name}_w": w.numpy(),
                       f"{name}_kscale": ks.numpy(), f"{name}_logits": ref.numpy()})
    path = os.path.join(out_dir, "dsa_indexer_deepgemm.npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path)


def make_flashmla(out_dir):
    import thirdparty as tp
    from paper_2512_10576_b200.decode import random_latent_rows
    g = torch.Generator(device="cuda").manual_seed(9)
    N, K, B = 1024, 512, 1
    rows = random_latent_rows(N, "cuda", g)
    q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    idx = torch.stack([torch.randperm(N, device="cuda", generator=g)[:K] for _ in range(B)]).int()
    sm = 1.0 / 192 ** 0.5
    out, lse, _ = tp.flashmla_sparse_decode(q, rows, idx, sm)
    torch.cuda.synchronize()
    path = os.path.join(out_dir, "dsa_attention_flashmla.npz")
    np.savez_compressed(path, rows=rows.cpu().numpy(), q=q.view(torch.uint16).cpu().numpy(),
                        idx=idx.cpu().numpy(), sm_scale=np.float64(sm),
                        out=out.view(torch.uint16).cpu().numpy(), lse=lse.cpu().numpy())
    print("wrote", path)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "indexer"
    out_dir = sys.argv[2] if len(sys.argv) > 2 else HERE
    {"indexer": make_indexer, "flashmla": make_flashmla}[what](out_dir)
