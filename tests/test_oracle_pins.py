"""oracle/dsa.py pinned to third-party implementations of the DSA operators (the
reference has no code for their values).  Fixtures from
tests/golden/make_dsa_golden.py:

  * indexer: DeepGEMM's torch reference ``fp8_mqa_logits_torch`` (vLLM 0.22) —
    bit-exact in the exact-arithmetic regime; its random case computes q.k in bf16, so
    there the oracle agrees to bf16 rounding of the per-head scores.
  * attention: FlashMLA's sm100 FP8 sparse decode (DeepSeek's V3.2 DSA kernel) on
    656-B latent rows with power-of-two group scales — the oracle's fp64 result agrees
    to the kernel's bf16 operand / output rounding (rel-L2 <= 5e-3, lse <= 1e-3).
"""
import os

import numpy as np
import pytest

from oracle import dsa

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_indexer_oracle_matches_deepgemm_reference():
    z = np.load(os.path.join(GOLD, "dsa_indexer_deepgemm.npz"))
    for case in ("exact", "random"):
        q, k, w, ks, ref = (z[f"{case}_{n}"] for n in ("q", "k", "w", "kscale", "logits"))
        got = dsa.indexer_logits(q, w, k, ks, k.shape[0])
        if case == "exact":
            np.testing.assert_array_equal(got, ref)
        else:
            # per-head scores rounded to bf16 in the reference (8-bit mantissa)
            tol = 2 ** -7 * np.abs(w).sum() * np.abs(ks).max() * np.abs(
                dsa.e4m3_decode(k).astype(np.float64) @ dsa.e4m3_decode(q).T).max()
            assert np.abs(got - ref).max() <= tol
            assert np.corrcoef(got, ref)[0, 1] > 0.9999


def test_topk_of_deepgemm_logits_is_the_oracle_tie_rule():
    """The reference's selection on the DeepGEMM logits (exact case: many ties) through
    the oracle top-k: the set is the k largest and ties go to the smaller index."""
    z = np.load(os.path.join(GOLD, "dsa_indexer_deepgemm.npz"))
    ref = z["exact_logits"]
    sel = dsa.topk_indices(ref, ref.shape[0], 256)
    thr = np.sort(ref)[::-1][255]
    assert (ref[sel] >= thr).all() and len(sel) == 256
    tied = np.flatnonzero(ref == thr)
    assert set(tied[:np.sum(ref[sel] == thr)]) == set(sel[ref[sel] == thr])


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLD, "dsa_attention_flashmla.npz")),
                    reason="FlashMLA fixture not generated yet")
def test_attention_oracle_matches_flashmla():
    z = np.load(os.path.join(GOLD, "dsa_attention_flashmla.npz"))
    rows, idx = z["rows"], z["idx"]
    q = dsa.bf16_decode(z["q"])
    out = dsa.bf16_decode(z["out"])
    for b in range(q.shape[0]):
        ref_o, ref_l = dsa.sparse_mla(q[b], rows[idx[b]], float(z["sm_scale"]))
        rel = np.linalg.norm(out[b] - ref_o) / np.linalg.norm(ref_o)
        assert rel <= 5e-3, rel
        assert np.abs(z["lse"][b] - ref_l).max() <= 1e-3
