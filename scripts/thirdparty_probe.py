"""GPU probe: FlashMLA / flashinfer comparators against the oracle and our kernels,
and FlashMLA's sparse decode time at C2 (B=64, top-2048) beside K5.

    python scripts/thirdparty_probe.py  ->  gpurun_out/thirdparty_probe.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

from oracle import dsa  # noqa: E402
import thirdparty as tp  # noqa: E402
from paper_2512_10576_b200.decode import random_latent_rows  # noqa: E402

res = {}
torch.manual_seed(0)
dev = "cuda"
g = torch.Generator(device=dev).manual_seed(3)
sm = 1.0 / 192 ** 0.5

# ---- FlashMLA numerics vs the fp64 oracle -----------------------------------------
B, N, K = 4, 8192, 2048
rows = random_latent_rows(N, dev, g)
q = (torch.randn((B, 128, 576), device=dev, generator=g) * 0.5).to(torch.bfloat16)
idx = torch.stack([torch.randperm(N, device=dev, generator=g)[:K] for _ in range(B)]).int()
def scales_variant(rows, kind):
    r = rows.clone()
    n = r.shape[0]
    if kind == "pow2":
        sc = 2.0 ** torch.randint(-7, -3, (n, 4), device=dev, generator=g).float()
        r[:, 512:528] = sc.view(torch.uint8)
    elif kind == "one":
        r[:, 512:528] = torch.ones((n, 4), device=dev).view(torch.uint8)
    elif kind == "norope":
        r[:, 528:] = 0
    return r


for kind in ("random", "pow2", "one", "norope"):
    try:
        rv = scales_variant(rows, kind)
        out, lse, _ = tp.flashmla_sparse_decode(q, rv, idx, sm)
        torch.cuda.synchronize()
        errs = []
        for b in range(2):
            ro, rl = dsa.sparse_mla(q[b].float().cpu().numpy(), rv.cpu().numpy()[idx[b].cpu().numpy()], sm)
            o = out[b].float().cpu().numpy()
            errs.append({"rel_l2": float(np.linalg.norm(o - ro) / np.linalg.norm(ro)),
                         "rel_l2_h0_63": float(np.linalg.norm(o[:64] - ro[:64]) / np.linalg.norm(ro[:64])),
                         "rel_l2_h64_127": float(np.linalg.norm(o[64:] - ro[64:]) / np.linalg.norm(ro[64:])),
                         "lse_max_abs": float(np.abs(lse[b].cpu().numpy() - rl).max()),
                         "lse_ref_mean": float(rl.mean()), "lse_got_mean": float(lse[b].cpu().numpy().mean())})
        res[f"flashmla_vs_oracle_{kind}"] = errs
    except Exception as e:  # record, keep probing
        res[f"flashmla_error_{kind}"] = repr(e)

# ---- FlashMLA time at C2 shape ---------------------------------------------------
try:
    B = 64
    N = 64 * 8192
    rows = torch.randint(0, 120, (N, 656), dtype=torch.uint8, device=dev)
    rows[:, 512:528] = torch.full((N, 4), 0.03, device=dev).view(torch.uint8)
    rows[:, 528:] = 0
    q = (torch.randn((B, 128, 576), device=dev, generator=g) * 0.5).to(torch.bfloat16)
    idx = torch.stack([b * 8192 + torch.randperm(8192, device=dev, generator=g)[:K] for b in range(B)]).int()
    out, lse, meta = tp.flashmla_sparse_decode(q, rows, idx, sm)
    for _ in range(5):
        tp.flashmla_sparse_decode(q, rows, idx, sm, meta=meta)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        tp.flashmla_sparse_decode(q, rows, idx, sm, meta=meta)
    e1.record()
    torch.cuda.synchronize()
    res["flashmla_c2_us"] = e0.elapsed_time(e1) / 20 * 1e3
except Exception as e:
    res["flashmla_time_error"] = repr(e)

# ---- flashinfer top_k vs oracle ----------------------------------------------------
try:
    lens = [32768, 40000, 131072, 5000]
    L = torch.randn((len(lens), max(lens)), device=dev, generator=g)
    L[1] = torch.relu(torch.round(L[1] * 3))  # ties
    sets = tp.flashinfer_topk_sets(L, lens, 2048)
    ok = []
    for b, n in enumerate(lens):
        want = dsa.topk_indices(L[b].cpu().numpy(), n, 2048)
        ok.append(bool(np.array_equal(sets[b].numpy(), want)))
    res["flashinfer_topk_equal_oracle"] = ok
except Exception as e:
    res["flashinfer_error"] = repr(e)

# ---- DeepGEMM torch indexer reference vs oracle (exact regime) -------------------
try:
    Lq = 3000
    qi = torch.randint(-1, 2, (64, 128), device=dev).float().to(torch.float8_e4m3fn).view(torch.uint8)
    ki = torch.randint(-1, 2, (Lq, 128), device=dev).float().to(torch.float8_e4m3fn).view(torch.uint8)
    w = (2.0 ** torch.randint(-6, 0, (64,), device=dev).float())
    ks = 2.0 ** torch.randint(-4, 2, (Lq,), device=dev).float()
    ref = tp.fp8_mqa_logits_reference(qi, ki, ks, w, Lq).cpu().numpy()
    want = dsa.indexer_logits(qi.cpu().numpy(), w.cpu().numpy(), ki.cpu().numpy(), ks.cpu().numpy(), Lq)
    res["deepgemm_ref_equal_oracle_exact"] = bool(np.array_equal(ref, want))
except Exception as e:
    res["deepgemm_error"] = repr(e)

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "thirdparty_probe.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
