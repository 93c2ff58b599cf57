"""Parity of the product step at the exact shapes and schedules bench.py times
(BASELINE.json configs[1] / [3] / [4] and the all-HBM ceiling), against the CPU oracle
chain (tests/_chain.py): every request's top-k bit-exact on the GPU logits, every
request's hit / miss counts and final LRU order bit-exact against the C restatement of
offsim's SparsePool (cache.py:90-134), attention within rel-L2 1e-2 on a sample of
requests (each micro-batch represented), indexer logits on a sample.

The layers come from bench.product_layer, so the schedule checked here is the one the
bench line reports: C2 = B 64, 32K, rho 0.25, DBA 16 | 48 with the early gather and the
fused DA attention (128 CTAs waiting on the gather's arrival counters); C4 = B 64, 128K,
rho 0.10, three micro-batches 12 | 26 | 26 with 4-CTA cluster top-k rows + fused split;
C5 = the mixed 8K-128K batch."""
import pytest
import torch

from tests._chain import OracleChain

pytestmark = pytest.mark.gpu

STEPS = 3


def _run(cfg_name, attn_sample, logit_sample, steps=STEPS, overlap="dba"):
    import bench
    from paper_2512_10576_b200.decode import random_latent_rows
    cfg = bench.CONFIGS[cfg_name]
    layer, lens, wins = bench.product_layer(cfg, "cuda", steps + 2, drift=0.97, record=True)
    try:
        chain = OracleChain(layer, lens, wins, attn_sample=attn_sample, logit_sample=logit_sample)
        eager = layer.capture(overlap, layer.gather_ctas)   # one eager step, then the graph
        chain.mirror(counts=eager)
        B = layer.B
        for _ in range(steps):
            q_idx, q = layer.next_queries()
            layer.step(q_idx, q, random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656))
            chain.mirror(q=q, q_idx=q_idx)
        chain.check_final()
        assert chain.misses > 0 and chain.hits > 0
        return layer.micro_batches(layer.micro)
    finally:
        layer.close()
        torch.cuda.synchronize()


def test_c2_benchmarked_step_matches_oracle_chain():
    ranges = _run("c2", attn_sample=(0, 15, 16, 40, 63), logit_sample=(0, 63))
    assert ranges == [(0, 16), (16, 64)]  # the DBA 16 | 48 split of the bench line


def test_c2_streamed_step_matches_oracle_chain():
    """The streamed schedule (bench.py --overlap stream) at the C2 shape: K1 / K2 / K4 as
    concurrent grids handing the 64 requests on through counters."""
    _run("c2", attn_sample=(0, 7, 8, 40, 63), logit_sample=(0,), overlap="stream")


def test_c2_dbs_step_matches_oracle_chain():
    """DBA with the second micro-batch handed on per request (bench.py --overlap dbs)."""
    _run("c2", attn_sample=(0, 15, 16, 17, 63), logit_sample=(0,), overlap="dbs")


def test_c4_dbs_step_matches_oracle_chain():
    _run("c4", attn_sample=(0, 12, 37, 38, 63), logit_sample=(), steps=2, overlap="dbs")


def test_c4_benchmarked_step_matches_oracle_chain():
    ranges = _run("c4", attn_sample=(0, 11, 12, 37, 38, 63), logit_sample=(5,), steps=2)
    assert ranges == [(0, 12), (12, 38), (38, 64)]


def test_c5_benchmarked_step_matches_oracle_chain():
    _run("c5", attn_sample=(0, 23, 24, 63), logit_sample=(), steps=2)


@pytest.mark.parametrize("sched", ["none", "da"])
def test_all_hbm_ceiling_step_matches_oracle_chain(sched):
    """The ceiling the bench divides by (rho = 1, whole history resident; bench.py takes
    the fastest schedule — DA at C2 — so both the sequential and the DA step are
    checked): every selection hits, nothing is gathered, and the results are the same
    as the offloaded step's oracle chain."""
    import bench
    from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows
    cfg = bench.CONFIGS["c2"]
    B, L = cfg["batch"], cfg["context_len"]
    layer = DSADecodeLayer(B, L, 1.0, bench.TOPK, max_new_tokens=16, device="cuda", seed=99, drift=0.97)
    try:
        layer.preload_full_history()
        chain = OracleChain(layer, [L] * B, None, attn_sample=(0, 31, 63))
        for o in chain.orc:  # the oracle pools hold the whole history too
            for c0 in range(0, L, 2048):
                o.warmup([list(range(c0, min(L, c0 + 2048)))])
        eager = layer.capture(sched, 32)
        chain.mirror(counts=eager)
        for _ in range(2):
            q_idx, q = layer.next_queries()
            layer.step(q_idx, q, random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656))
            chain.mirror(q=q)
        assert chain.misses == 0
        chain.check_final()
    finally:
        layer.close()
