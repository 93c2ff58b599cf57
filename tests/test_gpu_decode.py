"""End-to-end parity of one offloaded DSA decode layer (K1 -> K5 + append) against
the CPU oracle chain: oracle top-k on the GPU's logits, the C LRU oracle driven
with the same selections, and fp64 attention over the HOST store's rows of the
selected ids (so the gather is checked too)."""
import numpy as np
import pytest
import torch

from oracle import dsa
from oracle import lru as olru

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ctx,rho,fuse,overlap", [(8192, 0.25, True, "dba"), (4096, 0.25, True, "dba"),
                                                  (8192, 0.25, False, "dba"), (8192, 0.25, True, "da"),
                                                  (8192, 0.25, True, "none"), (8192, 0.25, True, "stream"),
                                                  (32768, 0.25, True, "stream"), (131072, 0.1, True, "stream"),
                                                  (8192, 0.25, True, "dbs"), (131072, 0.1, True, "dbs")])
def test_decode_layer_matches_oracle_chain(ctx, rho, fuse, overlap):
    """fuse: the DA schedule as one K5 launch waiting on the gather's arrival counters
    (sparse_mla_da) vs. two K5 passes merged through the workspace."""
    from paper_2512_10576_b200.cache import pool_capacity
    from paper_2512_10576_b200.decode import DSADecodeLayer
    B, K = 3, 2048
    layer = DSADecodeLayer(B, ctx, rho, K, max_new_tokens=8, seed=1, drift=0.97)
    layer.fuse_da = fuse
    windows = layer.prefill_warmup(windows=8, record=True)
    orc = [olru.OraclePool(pool_capacity(rho, ctx)) for _ in range(B)]
    for w in windows:
        for b in range(B):
            orc[b].warmup([w[b].tolist()])
    hist = ctx
    for step in range(4):
        q_idx, q = layer.next_queries()
        out, lse = layer.attend(q_idx, q, overlap=overlap)
        torch.cuda.synchronize()
        logits = layer.logits.cpu().numpy()
        idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
        counts = layer.step_counts().cpu().numpy()
        host = layer.store.host.numpy()
        o_all, l_all = out.float().cpu().numpy(), lse.cpu().numpy()
        qf = q.float().cpu().numpy()
        for b in range(B):
            n = hist
            want = dsa.topk_indices(logits[b], n, K)
            np.testing.assert_array_equal(idx[b, :cnt[b]], want)
            r = orc[b].access_step(want.tolist())
            assert counts[b, 0] == len(r.hit_ids) and counts[b, 1] == len(r.miss_ids)
            ref_o, ref_l = dsa.sparse_mla(qf[b], host[b, want], layer.sm_scale)
            rel = np.linalg.norm(o_all[b] - ref_o) / np.linalg.norm(ref_o)
            assert rel <= 1e-2, (step, b, rel)
            assert np.abs(l_all[b] - ref_l).max() <= 1e-2
        layer.append_token()
        hist += 1
        for o in orc:
            o.grow_capacity(pool_capacity(rho, hist))
            o.append_generated([hist - 1])
    layer.pool.check()
    out, cnt = layer.pool.lru_order()
    for b in range(B):
        assert out[b, :int(cnt[b])].tolist() == orc[b].lru_order()
    layer.close()


@pytest.mark.parametrize("overlap,micro,B", [("dba", 2, 4), ("dba", 3, 4), ("da", 1, 4), ("dba", 2, 40),
                                             ("stream", 1, 4), ("stream", 1, 40), ("dbs", 2, 4), ("dbs", 3, 40),
                                             ("dba+pdl", 2, 40), ("da+pdl", 1, 4)])
def test_graph_step_with_overlap_matches_oracle_chain(overlap, micro, B):
    """The product step — two micro-batches, gathers on a side stream, whole step
    captured as a CUDA graph, history/capacity computed on device — stays bit-exact
    on selections and cache accounting and within tolerance on attention (B = 4: K5
    KV-split shares; B = 40: one share per request)."""
    from paper_2512_10576_b200.cache import pool_capacity
    from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows
    K, ctx, rho = 2048, 8192, 0.25
    layer = DSADecodeLayer(B, ctx, rho, K, max_new_tokens=12, seed=3, drift=0.97)
    windows = layer.prefill_warmup(windows=6, record=True)
    orc = [olru.OraclePool(pool_capacity(rho, ctx)) for _ in range(B)]
    for w in windows:
        for b in range(B):
            orc[b].warmup([w[b].tolist()])
    hist = ctx

    def mirror(check_attention, q=None, counts=None):
        nonlocal hist
        torch.cuda.synchronize()
        logits = layer.logits.cpu().numpy()
        idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
        counts = (layer.step_counts() if counts is None else counts).cpu().numpy()
        host = layer.store.host.numpy()
        for b in range(B):
            want = dsa.topk_indices(logits[b], hist, K)
            np.testing.assert_array_equal(idx[b, :cnt[b]], want)
            r = orc[b].access_step(want.tolist())
            assert counts[b, 0] == len(r.hit_ids) and counts[b, 1] == len(r.miss_ids)
            if check_attention:
                ref_o, ref_l = dsa.sparse_mla(q[b].float().cpu().numpy(), host[b, want], layer.sm_scale)
                o = layer.out[b].float().cpu().numpy()
                assert np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o) <= 1e-2
        hist += 1
        for o in orc:
            o.grow_capacity(pool_capacity(rho, hist))
            o.append_generated([hist - 1])

    layer.micro = micro
    if overlap.endswith("+pdl"):  # the first micro-batch's K1 -> K2 + K3a (-> next K1) as PDL launches
        layer.pdl, overlap = True, overlap[:-4]
    eager = layer.capture(overlap=overlap)    # runs one eager step first
    mirror(False, counts=eager)
    for _ in range(3):
        q_idx, q = layer.next_queries()
        rows = random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656)
        layer.step(q_idx, q, rows)
        mirror(True, q)
    layer.pool.check()
    out, cnt = layer.pool.lru_order()
    for b in range(B):
        assert out[b, :int(cnt[b])].tolist() == orc[b].lru_order()
    assert int(layer.lens[0]) == hist
    layer.close()


def test_multilayer_model_graph_matches_oracle_per_layer():
    """C3's DSADecodeModel: layers run back to back inside one CUDA graph; every layer
    keeps its own pools and host store and stays bit-exact on selections and cache
    accounting, within tolerance on attention."""
    _model_chain(plan_theta=False)


def test_layer_plan_mixed_schedules_match_oracle_per_layer():
    """§8f.2 layer-wise plan (pipeline.py:190-195): layers with different query drift
    (so different miss means) run two uniform DA steps, the plan from the pools' live
    miss means puts DBA on the high-miss layers and DA elsewhere, and the graph
    re-captured with that mixed plan stays bit-exact per layer on selections, cache
    accounting and LRU order, within tolerance on attention."""
    _model_chain(plan_theta=True)


def _model_chain(plan_theta):
    from paper_2512_10576_b200.cache import pool_capacity
    from paper_2512_10576_b200.decode import DSADecodeModel, random_latent_rows
    from paper_2512_10576_b200.plan import MissMeter
    NL, B, K, ctx, rho = 3, 2, 2048, 8192, 0.25
    drift = [0.99, 0.85, 0.95] if plan_theta else 0.97
    model = DSADecodeModel(NL, B, ctx, rho, K, max_new_tokens=12, seed=11, drift=drift)
    model.set_schedule(2, None)
    orcs = []
    for layer in model.layers:
        wins = layer.prefill_warmup(windows=4, record=True)
        orc = [olru.OraclePool(pool_capacity(rho, ctx)) for _ in range(B)]
        for w in wins:
            for b in range(B):
                orc[b].warmup([w[b].tolist()])
        orcs.append(orc)
    hist = ctx

    def mirror(check_attention, qs=None):
        nonlocal hist
        torch.cuda.synchronize()
        for li, layer in enumerate(model.layers):
            logits = layer.logits.cpu().numpy()
            idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
            counts = layer.step_counts().cpu().numpy()
            host = layer.store.host.numpy()
            for b in range(B):
                want = dsa.topk_indices(logits[b], hist, K)
                np.testing.assert_array_equal(idx[b, :cnt[b]], want)
                r = orcs[li][b].access_step(want.tolist())
                assert counts[b, 1] == len(r.miss_ids), (li, b)
                if check_attention:
                    q = qs[li][1]
                    ref_o, _ = dsa.sparse_mla(q[b].float().cpu().numpy(), host[b, want], layer.sm_scale)
                    o = layer.out[b].float().cpu().numpy()
                    assert np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o) <= 1e-2
        hist += 1
        for orc in orcs:
            for o in orc:
                o.grow_capacity(pool_capacity(rho, hist))
                o.append_generated([hist - 1])

    model.capture("da" if plan_theta else "dba")
    mirror(False)
    meter = MissMeter(model)
    rows = random_latent_rows(B, "cuda").view(B, 1, 656)
    for _ in range(2):
        qs = model.next_queries()
        model.step(qs, rows)
        mirror(True, qs)
    if plan_theta:
        means = meter.means()
        assert len(set(means.tolist())) == NL, means
        theta = float(np.sort(means)[1])   # the two higher-miss layers get DBA
        plan = model.plan_layers(theta, meter)
        assert plan.counts() == {"dba": 2, "da": 1}, (means, plan)
        assert plan.strategies[int(np.argmin(means))] == "da"
        model.capture(plan=plan)
        assert model.launches_per_step() == sum(
            l.launches_per_step(o) for l, o in zip(model.layers, plan.strategies))
        mirror(False)
        for _ in range(2):
            qs = model.next_queries()
            model.step(qs, rows)
            mirror(True, qs)
    model.check()
    for li, layer in enumerate(model.layers):
        out, cnt = layer.pool.lru_order()
        for b in range(B):
            assert out[b, :int(cnt[b])].tolist() == orcs[li][b].lru_order()
    model.close()


@pytest.mark.parametrize("overlap", ["dba", "none"])
def test_mixed_length_batch_matches_oracle(overlap):
    """C5-style batch: per-request context lengths (and so per-request pool capacities);
    graph-captured product steps stay bit-exact on selections and cache accounting."""
    from paper_2512_10576_b200.cache import pool_capacity
    from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows
    lens = [9000, 4100, 16384, 2500]   # one request below the 4 x 2048 pool floor
    B, K, rho = len(lens), 2048, 0.25
    layer = DSADecodeLayer(B, lens, rho, K, max_new_tokens=8, seed=21, drift=0.97)
    wins = layer.prefill_warmup(windows=4, record=True)
    orc = [olru.OraclePool(pool_capacity(rho, n)) for n in lens]
    for w in wins:
        for b in range(B):
            orc[b].warmup([w[b].tolist()])
    hist = list(lens)

    def mirror(check_attention, q=None):
        torch.cuda.synchronize()
        logits = layer.logits.cpu().numpy()
        idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
        counts = layer.step_counts().cpu().numpy()
        host = layer.store.host.numpy()
        for b in range(B):
            want = dsa.topk_indices(logits[b], hist[b], K)
            np.testing.assert_array_equal(idx[b, :cnt[b]], want)
            r = orc[b].access_step(want.tolist())
            assert counts[b, 0] == len(r.hit_ids) and counts[b, 1] == len(r.miss_ids), b
            if check_attention:
                ref_o, _ = dsa.sparse_mla(q[b].float().cpu().numpy(), host[b, want], layer.sm_scale)
                o = layer.out[b].float().cpu().numpy()
                assert np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o) <= 1e-2
        for b in range(B):
            hist[b] += 1
            orc[b].grow_capacity(pool_capacity(rho, hist[b]))
            orc[b].append_generated([hist[b] - 1])

    layer.capture(overlap=overlap)
    mirror(False)
    for _ in range(3):
        q_idx, q = layer.next_queries()
        layer.step(q_idx, q, random_latent_rows(B, "cuda", layer.gen).view(B, 1, 656))
        mirror(True, q)
    layer.pool.check()
    out, cnt = layer.pool.lru_order()
    for b in range(B):
        assert out[b, :int(cnt[b])].tolist() == orc[b].lru_order()
    assert layer.lens.tolist() == hist
    layer.close()


def test_preload_full_history_mixed_lengths():
    """The all-HBM ceiling's state for a mixed-length batch (C5): every pool holds its own
    request's whole history at rho = 1, so a step hits every selected row."""
    from paper_2512_10576_b200.decode import DSADecodeLayer
    layer = DSADecodeLayer(3, [5000, 9000, 12000], 1.0, 2048, max_new_tokens=4, seed=5, drift=0.97)
    layer.preload_full_history()
    q_idx, q = layer.next_queries()
    layer.attend(q_idx, q, overlap="none")
    torch.cuda.synchronize()
    counts = layer.step_counts().cpu().numpy()
    assert (counts[:, 1] == 0).all() and (counts[:, 0] == 2048).all(), counts
    layer.pool.check()
    layer.close()


@pytest.mark.parametrize("serial", [False, True])
def test_step_host_matches_device_step(serial):
    """The public host-buffer step (queries from pinned memory, output back to pinned
    memory) equals the device-input step on the same inputs: selections and cache
    accounting bit for bit, attention to 1e-3.  serial: capture_host's link-serial
    pipeline (per-slot graphs, external upload / gathered events)."""
    from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows
    B, ctx, rho, K = 8, 8192, 0.25, 2048
    layers = [DSADecodeLayer(B, ctx, rho, K, max_new_tokens=12, seed=5, drift=0.97) for _ in range(2)]
    for lay in layers:
        lay.prefill_warmup(windows=6)
        lay.capture("dba")
    dev, host = layers
    if serial:
        host.capture_host("dba")
    outs = []
    for t in range(4):
        q_idx, q = dev.next_queries()
        host.next_queries()  # keep the two layers' query streams in step
        rows = random_latent_rows(B, "cuda", dev.gen).view(B, 1, 656)
        host.gen.set_state(dev.gen.get_state())
        h_out = torch.empty(dev.out.shape, dtype=dev.out.dtype).pin_memory()
        out, _ = dev.step(q_idx, q, rows)
        host.step_host(q_idx.cpu().pin_memory(), q.cpu().pin_memory(), rows.clone(), h_out)
        host.host_sync()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host.idx.cpu().numpy(), dev.idx.cpu().numpy())
        np.testing.assert_array_equal(host.step_counts().cpu().numpy(), dev.step_counts().cpu().numpy())
        o_dev, o_host = out.float().cpu(), h_out.float()
        assert float((o_host - o_dev).norm() / o_dev.norm()) <= 1e-3, t
        outs.append(float(o_host.norm()))
    for lay in layers:
        lay.pool.check()
    a, ca = dev.pool.lru_order()
    b, cb = host.pool.lru_order()
    assert torch.equal(ca, cb) and all(a[i, :int(ca[i])].tolist() == b[i, :int(cb[i])].tolist() for i in range(B))
    for lay in layers:
        lay.close()
