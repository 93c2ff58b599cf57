"""K1 / K2 / K4 / K5 parity on the GPU against the CPU oracle (oracle/dsa.py).

Tolerances (stated per north star):
  * top-k: bit-exact given the same logits (tie rule score desc, index asc)
  * indexer: bit-exact in the exact-arithmetic regime (small-integer e4m3 q/k,
    power-of-two w and scales: every product and partial sum is exact in fp32);
    otherwise |err| <= 1e-3 * max|logit| + 1e-5
  * gather / write-back: bit-exact (slot row = f16(f32(e4m3) * scale) ++ f16(bf16))
  * sparse MLA: rel-L2 <= 1e-2 and max-abs <= 2e-2 * max|ref| against the fp64
    reference on the same dequantised rows; lse abs <= 1e-2
"""
import numpy as np
import pytest
import torch

from oracle import dsa

pytestmark = pytest.mark.gpu


def e4m3(x):
    return x.clamp(-448, 448).to(torch.float8_e4m3fn).view(torch.uint8)


# ---------------------------------------------------------------------------- K2
@pytest.mark.parametrize("lens", [[32768, 4096, 2049, 2048, 100, 0, 131072, 5001],
                                  [32768] * 16, [49000, 20000, 2049, 1, 0, 3000],
                                  [2500] * 80,
                                  [40960 + 4099 * i for i in range(10)],  # 2-CTA clusters
                                  [200000, 170000, 3000, 2049]])  # 8-CTA clusters
def test_topk_matches_oracle(lens):
    from paper_2512_10576_b200.indexer import topk
    g = torch.Generator(device="cuda").manual_seed(7)
    B, ld = len(lens), max(lens) + 3  # odd stride exercises the scalar path
    logits = torch.randn((B, ld), device="cuda", generator=g)
    logits[1::2] = torch.relu(torch.round(logits[1::2] * 3))  # heavy exact ties (ReLU zeros)
    logits[0, 5] = -0.0
    L = torch.tensor(lens, dtype=torch.int32, device="cuda")
    idx, cnt = topk(logits, L, 2048)
    idx, cnt, host = idx.cpu().numpy(), cnt.cpu().numpy(), logits.cpu().numpy()
    for b, n in enumerate(lens):
        want = dsa.topk_indices(host[b], n, 2048)
        assert cnt[b] == len(want)
        np.testing.assert_array_equal(idx[b, :cnt[b]], want)


@pytest.mark.parametrize("n", [32768, 40000, 131072])
def test_topk_sorted_rows(n):
    """Candidates bunched at the end of the row (ascending scores) overflow the one-pass
    list's per-warp segments; descending rows bunch them at the start."""
    from paper_2512_10576_b200.indexer import topk
    up = torch.arange(n, device="cuda", dtype=torch.float32) / n
    logits = torch.stack([up, up.flip(0), torch.round(up * 50)])
    L = torch.full((3,), n, dtype=torch.int32, device="cuda")
    idx, cnt = topk(logits, L, 2048)
    idx, cnt, host = idx.cpu().numpy(), cnt.cpu().numpy(), logits.cpu().numpy()
    for b in range(3):
        want = dsa.topk_indices(host[b], n, 2048)
        assert cnt[b] == len(want)
        np.testing.assert_array_equal(idx[b, :cnt[b]], want)


@pytest.mark.parametrize("n", [40000, 40960, 65536, 131072, 200000])
def test_topk_all_equal_row(n):
    """Mass ties: every key equal, so the first k ids win (index asc).  Rows past 32K
    equal keys once overflowed a signed packed (greater, equal) count and wrote ids
    before the row; the output rows sit between sentinel guard rows that must survive."""
    from paper_2512_10576_b200.indexer import topk
    K, G = 2048, 4
    logits = torch.zeros((3, n), device="cuda")
    logits[2, n // 2:] = 1.0  # half the row tied above the rest
    L = torch.tensor([n, n - 1, n], dtype=torch.int32, device="cuda")
    buf = torch.full((G + 3 + G, K), -12345, dtype=torch.int32, device="cuda")
    idx = buf[G:G + 3]
    cnt = torch.empty(3, dtype=torch.int32, device="cuda")
    topk(logits, L, K, out=idx, count=cnt)
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    assert (got[:G] == -12345).all() and (got[G + 3:] == -12345).all(), "writes outside the output rows"
    assert (got[G] == np.arange(K)).all() and (got[G + 1] == np.arange(K)).all()
    assert (got[G + 2] == np.arange(n // 2, n // 2 + K)).all()
    assert cnt.cpu().tolist() == [K, K, K]


# ---------------------------------------------------------------------------- K1
def _indexer_inputs(B, Lmax, exact, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if exact:
        q = torch.randint(-4, 5, (B, 64, 128), device="cuda", generator=g).float()
        k = torch.randint(-4, 5, (B, Lmax, 128), device="cuda", generator=g).float()
        w = 2.0 ** torch.randint(-6, 0, (B, 64), device="cuda", generator=g).float()
        w = w * (torch.randint(0, 2, (B, 64), device="cuda", generator=g) * 2 - 1)
        ks = 2.0 ** torch.randint(-4, 2, (B, Lmax), device="cuda", generator=g).float()
    else:
        q = torch.randn((B, 64, 128), device="cuda", generator=g) * 2
        k = torch.randn((B, Lmax, 128), device="cuda", generator=g) * 2
        w = torch.randn((B, 64), device="cuda", generator=g) / 8
        ks = torch.rand((B, Lmax), device="cuda", generator=g) + 0.5
    return e4m3(q), w.contiguous(), e4m3(k), ks.contiguous()


@pytest.mark.parametrize("exact", [True, False])
def test_indexer_matches_oracle(exact):
    from paper_2512_10576_b200.indexer import indexer_logits
    lens = [4096, 130, 1, 0, 4000, 2048]
    B, Lmax = len(lens), 4096
    q, w, k, ks = _indexer_inputs(B, Lmax, exact)
    L = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = torch.full((B, Lmax), 12345.0, device="cuda")
    indexer_logits(q, w, k, ks, L, out=out)
    got = out.cpu().numpy()
    qn, wn, kn, ksn = (t.cpu().numpy() for t in (q, w, k, ks))
    for b, n in enumerate(lens):
        want = dsa.indexer_logits(qn[b], wn[b], kn[b], ksn[b], n)
        if exact:
            np.testing.assert_array_equal(got[b, :n], want)
        else:
            tol = 1e-3 * max(1e-6, float(np.abs(want).max(initial=0))) + 1e-5
            assert np.abs(got[b, :n] - want).max(initial=0) <= tol
        assert (got[b, n:] == 12345.0).all()  # nothing written past len


def test_indexer_then_topk_exact_regime_end_to_end():
    from paper_2512_10576_b200.indexer import indexer_logits, topk
    B, Lmax = 4, 32768
    q, w, k, ks = _indexer_inputs(B, Lmax, True, seed=3)
    L = torch.tensor([32768, 32000, 20000, 2500], dtype=torch.int32, device="cuda")
    logits = indexer_logits(q, w, k, ks, L)
    idx, cnt = topk(logits, L, 2048)
    qn, wn, kn, ksn = (t.cpu().numpy() for t in (q, w, k, ks))
    for b in range(B):
        n = int(L[b])
        want = dsa.topk_indices(dsa.indexer_logits(qn[b], wn[b], kn[b], ksn[b], n), n, 2048)
        np.testing.assert_array_equal(idx[b].cpu().numpy()[:cnt[b]], want)


# ---------------------------------------------------------------------------- K4
def _fill_slots(pools, rows_u8_per_pool, count):
    """Test setup: write 656-B latent rows into the slot store in its format (the
    dequantised f16 form, or the raw FP8 row when the store keeps 656-B rows)."""
    rv = pools.rows_view()
    for b, rows in enumerate(rows_u8_per_pool):
        if pools.row_bytes == 656:
            rv[b, :count].copy_(rows[:count])
        else:
            rv[b, :count].copy_(torch.as_tensor(dsa.slot_rows(rows.cpu().numpy()), device="cuda"))


def _slot_ref(q, rows_u8, sm):
    """fp64 attention over the exact f16 operands K5 multiplies (dsa.slot_rows)."""
    return dsa.sparse_mla_on_slot_rows(q, dsa.slot_rows(rows_u8), sm)


def _bf16(x):
    return torch.as_tensor(x).to(torch.bfloat16).float().numpy()


# K5 tolerances against _slot_ref (same operands): the output is bf16 (relative
# rounding <= 2^-9 per element, ~1.6e-3 rel-L2), P is rounded to f16 (2^-11).  So:
# rel-L2 to the exact result <= 3e-3, and to the exact result ROUNDED to bf16 <= 1.2e-3
# (away from rounding ties only K5's own f16-P / f32-sum error remains); lse to 1e-3.
K5_REL = 3e-3
K5_REL_BF16 = 1.2e-3
K5_LSE = 1e-3


def _check_k5(o, lse, ref_o, ref_l, what):
    rel = np.linalg.norm(o - ref_o) / max(np.linalg.norm(ref_o), 1e-12)
    relb = np.linalg.norm(o - _bf16(ref_o)) / max(np.linalg.norm(ref_o), 1e-12)
    assert rel <= K5_REL, (what, "rel-L2", rel)
    assert relb <= K5_REL_BF16, (what, "rel-L2 vs bf16(ref)", relb)
    assert np.abs(lse - ref_l).max() <= K5_LSE + 1e-6 * np.abs(ref_l).max(), (what, "lse")


@pytest.mark.parametrize("fmt", [656, 1152], ids=["fp8slots", "f16slots"])
@pytest.mark.parametrize("bulk,vmm", [(False, False), (True, False), (False, True)],
                         ids=["ld16", "bulk", "ld16-vmmstore"])
def test_gather_and_write_back_are_exact(bulk, vmm, fmt):
    """K4 reads 656-B rows over the host link and admits them dequantised; the slot
    row must equal the oracle's f16(f32(e4m3) * scale) ++ f16(bf16) bit for bit.
    vmm: the host store as one host-located VMM allocation (ESS_HOST_VMM)."""
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    from paper_2512_10576_b200.transfer import HostLatentStore, gather, write_generated
    P, ids, cap = 3, 5000, 1200
    store = HostLatentStore(P, ids, vmm=vmm)
    assert store.vmm == vmm
    for p in range(P):
        store.host[p].copy_(random_latent_rows(ids, "cuda"))
    pools = PoolSet(P, ids, cap, cap, row_bytes=fmt, staging_rows=0)
    rng = np.random.default_rng(0)
    sets = np.stack([rng.choice(4000, size=1000, replace=False) for _ in range(P)]).astype(np.int32)
    acc = pools.access(torch.as_tensor(sets, device="cuda"),
                       torch.full((P,), 1000, dtype=torch.int32, device="cuda"))
    gather(pools, store, acc, bulk=bulk)
    rows = pools.rows_view().cpu().numpy()
    sel = acc.sel_row.cpu().numpy()
    host = store.host.numpy()
    for p in range(P):
        want = host[p, sets[p]] if fmt == 656 else dsa.slot_rows(host[p, sets[p]]).view(np.uint16)
        np.testing.assert_array_equal(rows[p, sel[p]].view(want.dtype), want)
    # write-back of generated rows (append) lands in host store and (dequantised) slot
    new = torch.full((P, 1), 4500, dtype=torch.int32, device="cuda")
    one = torch.ones(P, dtype=torch.int32, device="cuda")
    slots = pools.append(new, one)
    src = random_latent_rows(P, "cuda").view(P, 1, 656)
    write_generated(pools, store, new, one, slots, src)
    torch.cuda.synchronize()
    rows = pools.rows_view().cpu().numpy()
    s = slots.cpu().numpy()[:, 0]
    srcn = src.cpu().numpy()
    for p in range(P):
        np.testing.assert_array_equal(store.host.numpy()[p, 4500], srcn[p, 0])
        want = srcn[p, 0] if fmt == 656 else dsa.slot_rows(srcn[p, :1])[0].view(np.uint16)
        np.testing.assert_array_equal(rows[p, s[p]].view(want.dtype), want)
    pools.check()
    store.close()


# ---------------------------------------------------------------------------- K5
FMT = pytest.mark.parametrize("fmt", [656, 1152], ids=["fp8slots", "f16slots"])


@FMT
@pytest.mark.parametrize("split", [1, 2, 3, 4])
@pytest.mark.parametrize("counts", [[2048, 1000, 17, 1], [2048] * 3])
def test_sparse_mla_matches_oracle(counts, split, fmt):
    """split > 1: each request's rows on 2 * split CTAs, partial states merged by the
    combine kernel (small-batch path) — same tolerance as one pass."""
    from paper_2512_10576_b200.attention import SplitWorkspace, sparse_mla, DEFAULT_SM_SCALE
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    B, cap = len(counts), 4096
    pools = PoolSet(B, 8192, cap, cap, row_bytes=fmt)
    g = torch.Generator(device="cuda").manual_seed(11)
    lat = [random_latent_rows(cap, "cuda", g) for _ in range(B)]
    _fill_slots(pools, lat, cap)
    sel = torch.stack([torch.randperm(cap, device="cuda", generator=g)[:2048] for _ in range(B)]).int()
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    ws = SplitWorkspace(B, "cuda", splits=split) if split > 1 else None
    out, lse = sparse_mla(pools, q, sel, cnt, workspace=ws, split=split)
    out, lse = out.float().cpu().numpy(), lse.cpu().numpy()
    qf = q.float().cpu().numpy()
    for b, n in enumerate(counts):
        rows = lat[b].cpu().numpy()[sel[b, :n].cpu().numpy()]
        ref_o, ref_l = _slot_ref(qf[b], rows, DEFAULT_SM_SCALE)
        _check_k5(out[b], lse[b], ref_o, ref_l, (b, n, split))
        # and against the unrounded dequantised rows (the end-to-end tolerance)
        ref_o, ref_l = dsa.sparse_mla(qf[b], rows, DEFAULT_SM_SCALE)
        rel = np.linalg.norm(out[b] - ref_o) / max(np.linalg.norm(ref_o), 1e-12)
        assert rel <= 1e-2, (b, n, rel)


@FMT
@pytest.mark.parametrize("n", [2048, 2047, 33, 1])
def test_sparse_mla_counts_every_row_once(n, fmt):
    """Exact row accounting: q = 0 makes every score 0, so the softmax is uniform and
    out = (sum of the selected V rows) / n exactly.  Each slot row is one-hot in a
    slot-dependent NoPE dim (value 1.0), so out[:, d] = (#selected rows hashed to d) / n
    — a dropped, duplicated or wrong row changes some dim by 1/n: compared bit for bit
    (for n = 2048 every count / n is exact in bf16)."""
    from paper_2512_10576_b200.attention import sparse_mla
    from paper_2512_10576_b200.cache import PoolSet
    B, cap = 2, 4096
    pools = PoolSet(B, 8192, cap, cap, row_bytes=fmt)
    dims = (np.arange(cap) * 37 + 11) % 512
    rows = np.zeros((cap, 656), np.uint8)
    rows[np.arange(cap), dims] = 0x38                               # e4m3 1.0
    rows[:, 512:528] = np.ones((cap, 4), np.float32).view(np.uint8)  # scales 1.0
    lat = [torch.as_tensor(rows, device="cuda")] * B
    _fill_slots(pools, lat, cap)
    g = torch.Generator(device="cuda").manual_seed(23)
    sel = torch.stack([torch.randperm(cap, device="cuda", generator=g)[:2048] for _ in range(B)]).int()
    cnt = torch.full((B,), n, dtype=torch.int32, device="cuda")
    q = torch.zeros((B, 128, 576), dtype=torch.bfloat16, device="cuda")
    out, lse = sparse_mla(pools, q, sel, cnt)
    out, lse = out.float().cpu().numpy(), lse.cpu().numpy()
    for b in range(B):
        want = np.broadcast_to(np.bincount(dims[sel[b, :n].cpu().numpy()], minlength=512) / n, (128, 512))
        if n == 2048:  # count / 2^11 is exact in bf16: bit for bit
            np.testing.assert_array_equal(out[b], _bf16(want))
        else:  # one bf16 ulp of double rounding allowed; one row more or less is >= 1/count
            np.testing.assert_allclose(out[b], want, rtol=8e-3, atol=0)
        np.testing.assert_allclose(lse[b], np.log(n), rtol=1e-6)
    pools.close()


@FMT
def test_sparse_mla_dominant_row(fmt):
    """One selected row outscores the rest by > 40 nats for every head, so the output is
    that row's V (to bf16 rounding); a dropped or shifted row (the ring's first, last or
    middle slot) would replace it with a blend of the others."""
    from paper_2512_10576_b200.attention import sparse_mla
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    B, cap = 3, 4096
    pools = PoolSet(B, 8192, cap, cap, row_bytes=fmt)
    g = torch.Generator(device="cuda").manual_seed(29)
    lat = [random_latent_rows(cap, "cuda", g) for _ in range(B)]
    _fill_slots(pools, lat, cap)
    sel = torch.stack([torch.randperm(cap, device="cuda", generator=g)[:2048] for _ in range(B)]).int()
    cnt = torch.full((B,), 2048, dtype=torch.int32, device="cuda")
    pick = [0, 1023, 2047]  # position of the dominant row in the selection
    q = torch.empty((B, 128, 576), dtype=torch.bfloat16, device="cuda")
    for b in range(B):
        k = torch.as_tensor(dsa.slot_rows(lat[b][sel[b, pick[b]]].cpu().numpy()[None])[0].astype(np.float32))
        q[b] = (k / k.norm() * 600.0).to(torch.bfloat16).expand(128, -1)
    out, lse = sparse_mla(pools, q, sel, cnt)
    for b in range(B):
        rows = lat[b].cpu().numpy()[sel[b].cpu().numpy()]
        ref_o, ref_l = _slot_ref(q[b].float().cpu().numpy(), rows, 1.0 / 192 ** 0.5)
        v = dsa.slot_rows(rows[pick[b]][None])[0, :512].astype(np.float32)
        assert np.abs(ref_o - v).max() <= 1e-3 * np.abs(v).max()  # the setup is one-hot
        _check_k5(out[b].float().cpu().numpy(), lse[b].cpu().numpy(), ref_o, ref_l, b)
    pools.close()


def _lib_slot_bytes():
    from paper_2512_10576_b200 import _lib
    return _lib.SLOT_ROW_BYTES


@FMT
def test_sparse_mla_rescale_path(fmt):
    """Scores that grow tile by tile force the lazy O rescale (> 2^8 jumps)."""
    from paper_2512_10576_b200.attention import sparse_mla
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    B, n = 2, 2048
    pools = PoolSet(B, 4096, n, n, row_bytes=fmt)
    g = torch.Generator(device="cuda").manual_seed(2)
    lat = []
    for b in range(B):
        rows = random_latent_rows(n, "cuda", g)
        # scale rows so later tiles have larger norms -> larger scores
        sc = rows[:, 512:528].clone().view(torch.float32) * torch.linspace(0.2, 3.0, n, device="cuda")[:, None]
        rows[:, 512:528] = sc.view(torch.uint8)
        lat.append(rows)
    _fill_slots(pools, lat, n)
    sel = torch.arange(n, dtype=torch.int32, device="cuda").repeat(B, 1).contiguous()
    cnt = torch.full((B,), n, dtype=torch.int32, device="cuda")
    q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 2).to(torch.bfloat16)
    out, lse = sparse_mla(pools, q, sel, cnt, sm_scale=0.2)
    for b in range(B):
        ref_o, ref_l = dsa.sparse_mla(q[b].float().cpu().numpy(), lat[b].cpu().numpy(), 0.2)
        o = out[b].float().cpu().numpy()
        assert np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o) <= 1e-2
        # scores reach ~70 here; f16 K rows carry 2^-11 relative rounding, so the
        # log-sum-exp tolerance is relative at this scale
        got_l = lse[b].cpu().numpy()
        assert (np.abs(got_l - ref_l) <= 1e-2 + 1e-3 * np.abs(ref_l)).all()


@FMT
@pytest.mark.parametrize("split", [(1900, 148), (0, 300), (2048, 0), (5, 1)])
def test_split_attention_partial_then_resume(split, fmt):
    """DA split: Attn0 over one row set -> workspace, Attn1 resumes
    over the other set = attention over the union (merge_attn semantics)."""
    from paper_2512_10576_b200.attention import SplitWorkspace, sparse_mla, DEFAULT_SM_SCALE
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    n1, n2 = split
    B, cap = 3, 4096
    pools = PoolSet(B, 8192, cap, cap, row_bytes=fmt)
    g = torch.Generator(device="cuda").manual_seed(17)
    lat = [random_latent_rows(cap, "cuda", g) for _ in range(B)]
    _fill_slots(pools, lat, cap)
    perm = torch.stack([torch.randperm(cap, device="cuda", generator=g)[:n1 + n2] for _ in range(B)]).int()
    rows1 = torch.zeros((B, 2048), dtype=torch.int32, device="cuda")
    rows2 = torch.zeros((B, 2048), dtype=torch.int32, device="cuda")
    rows1[:, :n1] = perm[:, :n1]
    rows2[:, :n2] = perm[:, n1:]
    counts = torch.tensor([[n1, n2, 0, 0]] * B, dtype=torch.int32, device="cuda")
    q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    ws = SplitWorkspace(B, "cuda")
    sparse_mla(pools, q, rows1, counts[:, 0], workspace=ws, mode="partial")
    out, lse = sparse_mla(pools, q, rows2, counts[:, 1], workspace=ws, mode="resume")
    out, lse = out.float().cpu().numpy(), lse.cpu().numpy()
    for b in range(B):
        rows = lat[b].cpu().numpy()[perm[b].cpu().numpy()]
        ref_o, ref_l = dsa.sparse_mla(q[b].float().cpu().numpy(), rows, DEFAULT_SM_SCALE)
        rel = np.linalg.norm(out[b] - ref_o) / max(np.linalg.norm(ref_o), 1e-12)
        assert rel <= 1e-2, (split, b, rel)
        assert np.abs(lse[b] - ref_l).max() <= 1e-2


@FMT
def test_early_gather_split_access_settle_matches_plain_access(fmt):
    """Early-gather form of K3 + K4: the read-only split (misses -> staging rows), the
    gather into staging, the LRU update reporting final slots and the settle copy end in
    the same pool state and slot contents as one plain access + gather."""
    from paper_2512_10576_b200.cache import AccessBatch, PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    from paper_2512_10576_b200.transfer import HostLatentStore, gather
    P, ids, cap, K = 3, 9000, 2500, 2048
    store = HostLatentStore(P, ids)
    for p in range(P):
        store.host[p].copy_(random_latent_rows(ids, "cuda"))
    a = PoolSet(P, ids, cap, cap, row_bytes=fmt, staging_rows=K)
    b = PoolSet(P, ids, cap, cap, row_bytes=fmt, staging_rows=K)
    rng = np.random.default_rng(3)
    z = lambda: torch.zeros((P, K), dtype=torch.int32, device="cuda")  # noqa: E731
    for step in range(4):
        sets = [np.sort(rng.choice(6000 + 500 * step, size=K, replace=False)) for _ in range(P)]
        req = torch.as_tensor(np.stack(sets).astype(np.int32), device="cuda")
        n = torch.full((P,), K, dtype=torch.int32, device="cuda")
        ra = a.access(req, n, lists=True)
        gather(a, store, ra)
        sb = AccessBatch(counts=torch.zeros((P, 4), dtype=torch.int32, device="cuda"), sel_row=z(),
                         miss_ids=z(), miss_row=z(), hit_row=z())
        b.split(req, n, out=sb)
        settle, cb = z(), torch.zeros((P, 4), dtype=torch.int32, device="cuda")
        gather(b, store, sb)
        b.access(req, n, out=AccessBatch(counts=cb, sel_row=None, miss_ids=None, miss_row=settle,
                                         hit_row=None))
        b.settle(settle, sb.counts)
        torch.cuda.synchronize()
        a.check()
        b.check()
        ca, cs = ra.counts.cpu().numpy(), sb.counts.cpu().numpy()
        np.testing.assert_array_equal(ca[:, :2], cs[:, :2])
        np.testing.assert_array_equal(cb.cpu().numpy()[:, :2], cs[:, :2])
        for p in range(P):
            m = int(ca[p, 1])
            np.testing.assert_array_equal(ra.miss_ids[p, :m].cpu().numpy(), sb.miss_ids[p, :m].cpu().numpy())
            # staging rows for the misses, the plain access's slots for its misses
            assert sb.miss_row[p, :m].tolist() == list(range(b.cap_max, b.cap_max + m))
            np.testing.assert_array_equal(settle[p, :m].cpu().numpy(), ra.miss_row[p, :m].cpu().numpy())
        oa, na = a.lru_order()
        ob, nb = b.lru_order()
        np.testing.assert_array_equal(na.cpu().numpy(), nb.cpu().numpy())
        for p in range(P):
            assert oa[p, :int(na[p])].tolist() == ob[p, :int(nb[p])].tolist()
    ra_rows, rb_rows = a.rows_view().cpu().numpy(), b.rows_view().cpu().numpy()
    for p in range(P):
        order = oa[p, :int(na[p])].cpu().numpy()
        sa = a.lookup(p, torch.as_tensor(order, device="cuda")).cpu().numpy()
        sbl = b.lookup(p, torch.as_tensor(order, device="cuda")).cpu().numpy()
        np.testing.assert_array_equal(sa, sbl)
        np.testing.assert_array_equal(ra_rows[p, sa], rb_rows[p, sbl])
    a.close()
    b.close()
    store.close()


@pytest.mark.parametrize("lens", [[32768, 4096, 2049, 2048, 1000], [131072, 40000]])
def test_topk_split_fused_matches_topk_then_split(lens):
    """K2 with the fused hit/miss split (one launch for rows <= 40K, two otherwise) gives
    the same selection and the same hit rows / miss ids / staging rows / counts as top-k
    followed by ess_pool_split."""
    from paper_2512_10576_b200.cache import AccessBatch, PoolSet
    from paper_2512_10576_b200.indexer import topk, topk_split
    B, K = len(lens), 2048
    ld = ((max(lens) + 127) // 128) * 128
    g = torch.Generator(device="cuda").manual_seed(5)
    logits = torch.randn((B, ld), device="cuda", generator=g)
    ln = torch.tensor(lens, dtype=torch.int32, device="cuda")
    cap = 4096
    pool = PoolSet(B, ld, cap, cap, row_bytes=1152, staging_rows=K)
    rng = np.random.default_rng(1)
    for b, n in enumerate(lens):  # make a random part of the history resident
        w = rng.choice(n, size=min(n, 2000), replace=False).astype(np.int32)
        ids = torch.as_tensor(w, device="cuda").view(1, -1)
        pool.warmup(ids, torch.tensor([ids.shape[1]], dtype=torch.int32, device="cuda"), begin=b)
    z = lambda: torch.full((B, K), -7, dtype=torch.int32, device="cuda")  # noqa: E731
    mk = lambda: AccessBatch(counts=torch.zeros((B, 4), dtype=torch.int32, device="cuda"),  # noqa: E731
                             sel_row=None, miss_ids=z(), miss_row=z(), hit_row=z())
    i1, c1 = topk(logits, ln, K)
    r1 = mk()
    pool.split(i1, c1, out=r1)
    i2, c2 = torch.empty_like(i1), torch.empty_like(c1)
    r2 = mk()
    topk_split(logits, ln, K, i2, c2, pool, r2)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    for b in range(B):
        n = int(c1[b])
        assert torch.equal(i1[b, :n], i2[b, :n])
        h, m = int(r1.counts[b, 0]), int(r1.counts[b, 1])
        assert h + m == n and h > 0
        assert torch.equal(r1.counts[b], r2.counts[b])
        assert torch.equal(r1.hit_row[b, :h], r2.hit_row[b, :h])
        assert torch.equal(r1.miss_ids[b, :m], r2.miss_ids[b, :m])
        assert torch.equal(r1.miss_row[b, :m], r2.miss_row[b, :m])
    pool.close()


# ------------------------------------------------------------ f16 range guard (K4 / K5)
@FMT
def test_sparse_mla_flags_q_outside_f16_range(fmt):
    """K5 multiplies f16 operands: a bf16 q element of magnitude >= 65520 has no f16
    value, so the launch latches ESS_ERR_RANGE (ValueError at pool.check) instead of
    returning silently wrong output; in-range q leaves the status clean."""
    from paper_2512_10576_b200.attention import sparse_mla
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    B, cap = 2, 2048
    pools = PoolSet(B, 4096, cap, cap, row_bytes=fmt)
    g = torch.Generator(device="cuda").manual_seed(3)
    _fill_slots(pools, [random_latent_rows(cap, "cuda", g) for _ in range(B)], cap)
    sel = torch.arange(cap, dtype=torch.int32, device="cuda").repeat(B, 1)
    cnt = torch.full((B,), cap, dtype=torch.int32, device="cuda")
    q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    q[1, 7, 3] = 60000.0   # large but representable in f16: no error
    sparse_mla(pools, q, sel, cnt)
    pools.check("in range")
    for bad in (70000.0, float("inf"), -1e6, 5e5):
        q2 = q.clone()
        q2[1, 100, 511 if bad > 0 else 560] = bad
        sparse_mla(pools, q2, sel, cnt)
        with pytest.raises(ValueError, match="f16 range"):
            pools.check("q out of range")
    pools.close()


def test_gather_flags_slot_rows_outside_f16_range():
    """The f16 slot format dequantises each fetched row once: a latent row whose RoPE
    (bf16) or scaled NoPE value does not fit f16 latches ESS_ERR_RANGE in the gather."""
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    from paper_2512_10576_b200.transfer import HostLatentStore, gather
    P, ids, cap = 2, 3000, 1024
    store = HostLatentStore(P, ids)
    for p in range(P):
        store.host[p].copy_(random_latent_rows(ids, "cuda"))
    h = store.host.numpy()
    rope = h[1, 10, 528:].view(np.uint16)
    rope[5] = 0x47C3   # bf16 99840: beyond f16
    sc = h[0, 20, 512:528].view(np.float32)
    sc[2] = 1024.0     # e4m3 values up to 448 x 1024: beyond f16 for |nope| > 64
    for which, row_id in ((1, 10), (0, 20)):
        pools = PoolSet(P, ids, cap, cap, row_bytes=1152)
        sets = np.tile(np.arange(100, 200, dtype=np.int32), (P, 1))   # clean rows ...
        sets[which, 0] = row_id                                       # ... and one bad one
        acc = pools.access(torch.as_tensor(sets, device="cuda"),
                           torch.full((P,), 100, dtype=torch.int32, device="cuda"))
        gather(pools, store, acc)
        with pytest.raises(ValueError, match="f16 range"):
            pools.check("slot row out of range")
        pools.close()
    pools = PoolSet(P, ids, cap, cap, row_bytes=1152)   # rows 100.. are clean
    sets = np.tile(np.arange(100, 400, dtype=np.int32), (P, 1))
    acc = pools.access(torch.as_tensor(sets, device="cuda"), torch.full((P,), 300, dtype=torch.int32, device="cuda"))
    gather(pools, store, acc)
    pools.check("in range")
    pools.close()
    store.close()


@FMT
def test_sparse_mla_small_q_below_f16_normal_range(fmt):
    """q of magnitude ~1e-6 (below f16's normal range, 6.1e-5: kept as f16 subnormals,
    the smallest ~6e-8 flush to zero) still matches fp64 on the unrounded q within the
    end-to-end tolerance: the scores are ~0 and the softmax near uniform."""
    from paper_2512_10576_b200.attention import sparse_mla, DEFAULT_SM_SCALE
    from paper_2512_10576_b200.cache import PoolSet
    from paper_2512_10576_b200.decode import random_latent_rows
    B, cap = 2, 2048
    pools = PoolSet(B, 4096, cap, cap, row_bytes=fmt)
    g = torch.Generator(device="cuda").manual_seed(5)
    lat = [random_latent_rows(cap, "cuda", g) for _ in range(B)]
    _fill_slots(pools, lat, cap)
    sel = torch.arange(cap, dtype=torch.int32, device="cuda").repeat(B, 1)
    cnt = torch.full((B,), cap, dtype=torch.int32, device="cuda")
    q = (torch.randn((B, 128, 576), device="cuda", generator=g) * 1e-6).to(torch.bfloat16)
    out, lse = sparse_mla(pools, q, sel, cnt)
    pools.check("small q")
    qf = q.float().cpu().numpy()
    for b in range(B):
        ref_o, ref_l = dsa.sparse_mla(qf[b], lat[b].cpu().numpy(), DEFAULT_SM_SCALE)
        o = out[b].float().cpu().numpy()
        assert np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o) <= 1e-2
        assert np.abs(lse[b].cpu().numpy() - ref_l).max() <= 1e-2
    pools.close()
