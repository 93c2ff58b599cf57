"""MTP decode (mtp + 1 query tokens per request and step; pipeline.py:213-215,
trace.py:127, cache.py:191-195) against the CPU oracle chain: the MTP indexer equals
the single-token indexer per token (bit-exact) and the fp64 oracle (1e-3), top-k per
token row equals the oracle's on the GPU logits (bit-exact), the pool takes the qtok
sets as consecutive access_steps — hit/miss counts, appended miss lists
and final LRU order bit-exact against the C restatement of offsim's SparsePool — and
attention for every (request, token) row matches fp64 over the host store's rows."""
import numpy as np
import pytest
import torch

from oracle import dsa
from oracle import lru as olru

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("qtok", [2, 3, 4])
def test_indexer_mtp_equals_per_token_indexer(qtok):
    from paper_2512_10576_b200.decode import _e4m3
    from paper_2512_10576_b200.indexer import indexer_logits, indexer_logits_mtp
    g = torch.Generator(device="cuda").manual_seed(qtok)
    B, L = 5, 4096 + 256
    lens = torch.tensor([4096, 1, 300, 4096 + 200, 129], dtype=torch.int32, device="cuda")
    k = _e4m3(torch.randn((B, L, 128), device="cuda", generator=g) * 8)
    ks = torch.rand((B, L), device="cuda", generator=g) + 0.5
    q = _e4m3(torch.randn((B, qtok, 64, 128), device="cuda", generator=g) * 4)
    w = torch.randn((B, qtok, 64), device="cuda", generator=g) / 8
    out = torch.full((B, qtok, L), 7.0, device="cuda")
    indexer_logits_mtp(q, w, k, ks, lens, out=out)
    for j in range(qtok):
        one = torch.full((B, L), 7.0, device="cuda")
        indexer_logits(q[:, j].contiguous(), w[:, j].contiguous(), k, ks, lens, out=one)
        assert torch.equal(out[:, j], one), j   # same MMA sums, same fold order
    for b in (0, 2, 3):
        n = int(lens[b])
        for j in range(qtok):
            ref = dsa.indexer_logits(q[b, j].cpu().numpy(), w[b, j].cpu().numpy(), k[b].cpu().numpy(),
                                     ks[b].cpu().numpy(), n)
            got = out[b, j, :n].cpu().numpy()
            assert np.abs(got - ref).max() <= 1e-3 * np.abs(ref).max() + 1e-5
            assert (out[b, j, n:] == 7.0).all()   # past len untouched


def test_topk_mtp_rows_use_their_request_length():
    from paper_2512_10576_b200.indexer import topk_mtp
    g = torch.Generator(device="cuda").manual_seed(5)
    B, Q, L, K = 4, 3, 40960, 2048
    lens = torch.tensor([40960, 1000, 2049, 30000], dtype=torch.int32, device="cuda")
    logits = torch.randn((B, Q, L), device="cuda", generator=g)
    logits[1, 2, :500] = 0.0   # ties
    idx, cnt = topk_mtp(logits, lens, K)
    lg = logits.cpu().numpy()
    for b in range(B):
        for j in range(Q):
            want = dsa.topk_indices(lg[b, j], int(lens[b]), K)
            assert int(cnt[b, j]) == len(want)
            np.testing.assert_array_equal(idx[b, j, :len(want)].cpu().numpy(), want)


def test_access_mtp_is_sequential_access_steps():
    from paper_2512_10576_b200.cache import PoolSet
    rng = np.random.default_rng(3)
    P, Q, K, ids, cap = 6, 3, 2048, 30000, 7000
    ps = PoolSet(P, ids, cap, [cap] * P)
    orc = [olru.OraclePool(cap) for _ in range(P)]
    for step in range(4):
        sets = [[np.sort(rng.choice(ids if step else 9000, size=K - 37 * j, replace=False)) for j in range(Q)]
                for _ in range(P)]
        req = torch.zeros((P, Q, K), dtype=torch.int32)
        n = torch.zeros((P, Q), dtype=torch.int32)
        for p in range(P):
            for j in range(Q):
                req[p, j, :len(sets[p][j])] = torch.from_numpy(sets[p][j].astype(np.int32))
                n[p, j] = len(sets[p][j])
        th = torch.full((P, Q, K), -7, dtype=torch.int32, device="cuda")
        tf = torch.full((P, Q, K), -7, dtype=torch.int32, device="cuda")
        tc = torch.empty((P, Q, 2), dtype=torch.int32, device="cuda")
        acc = ps.access_mtp(req.cuda(), n.cuda(), lists=True, tok_split=(th, tf, tc))
        torch.cuda.synchronize()
        th, tf, tc = th.cpu().numpy(), tf.cpu().numpy(), tc.cpu().numpy()
        counts = acc.counts.cpu().numpy()
        miss = acc.miss_ids.cpu().numpy()
        hit = acc.hit_ids.cpu().numpy()
        ev = acc.evicted_ids.cpu().numpy()
        sel = acc.sel_row.cpu().numpy()
        for p in range(P):
            hs, ms, es = [], [], []
            fetched = set()
            for j in range(Q):
                r = orc[p].access_step(sets[p][j].tolist())
                # attention split of set j: ids resident before the step vs fetched by
                # this or an earlier set (in requested order); rows checked below
                fetched |= set(r.miss_ids)
                fr = [x in fetched for x in sets[p][j].tolist()]
                assert tc[p, j].tolist() == [len(fr) - sum(fr), sum(fr)], (step, p, j)
                rows = ps.lookup(p, torch.from_numpy(sets[p][j].astype(np.int32)).cuda()).cpu().numpy()
                np.testing.assert_array_equal(th[p, j, :len(fr) - sum(fr)], rows[~np.array(fr)])
                np.testing.assert_array_equal(tf[p, j, :sum(fr)], rows[np.array(fr)])
                hs += list(r.hit_ids)
                ms += list(r.miss_ids)
                es += list(r.evicted_ids)
            assert counts[p, :3].tolist() == [len(hs), len(ms), len(es)], (step, p)
            assert miss[p, :len(ms)].tolist() == ms
            assert hit[p, :len(hs)].tolist() == hs
            assert ev[p, :len(es)].tolist() == es
            # every set's slot rows are those of its ids after the whole step
            for j in range(Q):
                slots = ps.lookup(p, torch.from_numpy(sets[p][j].astype(np.int32)).cuda()).cpu().numpy()
                np.testing.assert_array_equal(sel[p, j, :len(sets[p][j])], slots)
    ps.check()
    out, cnt = ps.lru_order()
    for p in range(P):
        assert out[p, :int(cnt[p])].tolist() == orc[p].lru_order()
    ps.close()


def _mtp_chain(layer, orc, hist, accepted, q=None, q_idx=None, counts=None, attn=True):
    """Mirror one MTP step: per request, the qtok sets through the oracle pool in token
    order, then grow + admit the accepted ids."""
    from paper_2512_10576_b200.cache import pool_capacity
    torch.cuda.synchronize()
    B, Q, K = layer.B, layer.qtok, layer.K
    logits = layer.logits.cpu().numpy()
    idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
    counts = (layer.step_counts() if counts is None else counts).cpu().numpy()
    miss = layer.acc.miss_ids.cpu().numpy()
    host = layer.store.host.numpy() if attn else None
    for b in range(B):
        hs = ms = 0
        mlist = []
        for j in range(Q):
            want = dsa.topk_indices(logits[b, j], hist[b], K)
            assert cnt[b, j] == len(want)
            np.testing.assert_array_equal(idx[b, j, :cnt[b, j]], want, err_msg=f"top-k req {b} tok {j}")
            r = orc[b].access_step(want.tolist())
            hs += len(r.hit_ids)
            ms += len(r.miss_ids)
            mlist += list(r.miss_ids)
            if attn and q is not None:
                ref_o, ref_l = dsa.sparse_mla(q[b, j].float().cpu().numpy(), host[b, want], layer.sm_scale)
                o = layer.out[b, j].float().cpu().numpy()
                assert np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o) <= 1e-2, (b, j)
                assert np.abs(layer.lse[b, j].cpu().numpy() - ref_l).max() <= 1e-2
            if q_idx is not None and b == 0:
                ref = dsa.indexer_logits(q_idx[b, j].cpu().numpy(), layer.w[b, j].cpu().numpy(),
                                         layer.k_cache[b].cpu().numpy(), layer.k_scale[b].cpu().numpy(), hist[b])
                assert np.abs(logits[b, j, :hist[b]] - ref).max() <= 1e-3 * np.abs(ref).max() + 1e-5
        assert counts[b, 0] == hs and counts[b, 1] == ms, (b, counts[b].tolist(), hs, ms)
        assert miss[b, :ms].tolist() == mlist
    for b in range(B):
        m = int(accepted[b])
        new = list(range(hist[b], hist[b] + m))
        hist[b] += m
        orc[b].grow_capacity(pool_capacity(layer.rho, hist[b]))
        orc[b].append_generated(new)


@pytest.mark.parametrize("mtp,overlap", [(2, "dba"), (2, "none"), (2, "da"), (1, "dba"), (3, "dba"),
                                         (2, "dba+streamed-gather")])
def test_mtp_layer_matches_oracle_chain(mtp, overlap):
    from paper_2512_10576_b200.cache import pool_capacity
    from paper_2512_10576_b200.mtp import MTPDecodeLayer, draw_accepted
    B, K, ctx, rho = 4, 2048, 32768, 0.25
    layer = MTPDecodeLayer(B, ctx, rho, K, mtp=mtp, max_new_tokens=6, seed=7, drift=0.97)
    if overlap.endswith("+streamed-gather"):  # gathers taking requests as K3 publishes them
        overlap, layer.stream_gather = "dba", True
    wins = layer.prefill_warmup(windows=6, record=True)
    orc = [olru.OraclePool(pool_capacity(rho, ctx)) for _ in range(B)]
    for w in wins:
        for b in range(B):
            orc[b].warmup([w[b].tolist()])
    hist = [ctx] * B
    rng = np.random.default_rng(mtp)
    for step in range(3):
        q_idx, q = layer.next_queries()
        layer.attend(q_idx, q, overlap=overlap)
        acc = draw_accepted(rng, B, 1.7, layer.qtok)
        _mtp_chain(layer, orc, hist, acc, q=q, q_idx=q_idx if step == 0 else None)
        layer.append_tokens(acc)
    layer.pool.check()
    out, cnt = layer.pool.lru_order()
    for b in range(B):
        assert out[b, :int(cnt[b])].tolist() == orc[b].lru_order()
    assert layer.lens.tolist() == hist
    layer.close()


def test_mtp_graph_step_matches_oracle_chain():
    """The captured MTP step (2 micro-batches, gathers on a side stream, per-request
    accepted counts admitted on device) at B = 16, 32K, MTP = 2."""
    from paper_2512_10576_b200.cache import pool_capacity
    from paper_2512_10576_b200.decode import random_latent_rows
    from paper_2512_10576_b200.mtp import MTPDecodeLayer, draw_accepted
    B, K, ctx, rho = 16, 2048, 32768, 0.25
    layer = MTPDecodeLayer(B, ctx, rho, K, mtp=2, max_new_tokens=8, seed=9, drift=0.97)
    wins = layer.prefill_warmup(windows=4, record=True)
    orc = [olru.OraclePool(pool_capacity(rho, ctx)) for _ in range(B)]
    for w in wins:
        for b in range(B):
            orc[b].warmup([w[b].tolist()])
    hist = [ctx] * B
    rng = np.random.default_rng(1)
    acc0 = draw_accepted(rng, B, 1.7, 3)
    eager = layer.capture(overlap="dba", accepted=acc0)
    _mtp_chain(layer, orc, hist, acc0, counts=eager, attn=False)
    for _ in range(3):
        q_idx, q = layer.next_queries()
        rows = random_latent_rows(B * 3, "cuda", layer.gen).view(B, 3, 656)
        acc = draw_accepted(rng, B, 1.7, 3)
        layer.step(q_idx, q, rows, torch.from_numpy(acc).cuda(), max_accepted=int(acc.max()))
        _mtp_chain(layer, orc, hist, acc, q=q)
    layer.pool.check()
    out, cnt = layer.pool.lru_order()
    for b in range(B):
        assert out[b, :int(cnt[b])].tolist() == orc[b].lru_order()
    assert layer.lens.tolist() == hist
    layer.close()


def test_mtp_step_rejects_accepted_counts_beyond_the_verified_tokens():
    """A request cannot accept more tokens than the step verified (qtok): host counts are
    refused before the launch, device counts latch ESS_ERR_ARG in the admission kernel
    (it would otherwise read the next request's rows)."""
    from paper_2512_10576_b200.decode import random_latent_rows
    from paper_2512_10576_b200.mtp import MTPDecodeLayer
    layer = MTPDecodeLayer(2, 16384, 0.5, 2048, mtp=2, max_new_tokens=6, seed=3, drift=0.97)
    layer.prefill_warmup(windows=2)
    layer.capture("dba", accepted=[1, 2])
    layer.pool.check("capture")
    q_idx, q = layer.next_queries()
    rows = random_latent_rows(6, "cuda", layer.gen).view(2, 3, 656)
    with pytest.raises(ValueError):
        layer.step(q_idx, q, rows, torch.tensor([4, 1], dtype=torch.int32))
    layer.step(q_idx, q, rows, torch.tensor([4, 1], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        layer.pool.check("device accepted > qtok")
    layer.close()
