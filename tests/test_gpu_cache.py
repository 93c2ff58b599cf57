"""K3 parity on the GPU: the device cache manager must reproduce the reference
LRU bit-exactly — hit/miss lists in requested order, evicted ids, h2d blocks,
LRU order, inserted counts and counters.  Truth = golden vectors produced by the
real offsim (tests/golden/) and the C oracle (oracle/lru_oracle.c) at scale."""
import numpy as np
import pytest
import torch

from oracle import lru as olru
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ess():
    from paper_2512_10576_b200 import cache
    return cache


def test_sparse_pool_matches_reference_workloads(ess):
    from tests.test_oracle_golden import run_workload
    ws = G.lru_workloads()
    for w in ws[:200]:
        pool = run_workload(ess.SparsePool, w)
        assert [pool.hits, pool.misses, pool.evictions] == w["stats"]


def test_sparse_pool_hand_examples(ess):
    pool = ess.SparsePool(4)
    r1 = pool.access_step([1, 2, 3, 4])
    assert r1.miss_ids == [1, 2, 3, 4] and r1.h2d_blocks == 4
    r2 = pool.access_step([3, 4, 5])
    assert (r2.hit_ids, r2.miss_ids, r2.evicted_ids) == ([3, 4], [5], [1])
    assert pool.resident_ids() == [2, 3, 4, 5] and pool.lru_order() == [2, 3, 4, 5]
    assert 3 in pool and 1 not in pool and len(pool) == 4
    p = ess.SparsePool(2)
    r = p.access_step([10, 11, 12, 13])
    assert r.h2d_blocks == 4 and p.resident_ids() == [12, 13]
    p = ess.SparsePool(4)
    assert p.warmup([[1, 2, 3], [2, 4, 5]]) == 5
    assert p.lru_order() == [3, 2, 4, 5] and p.misses == 0


def test_sparse_pool_errors(ess):
    with pytest.raises(ValueError):
        ess.SparsePool(0)
    p = ess.SparsePool(3)
    p.access_step([0, 1])
    assert p.append_generated([100, 101]) == 2
    assert p.resident_ids() == [1, 100, 101]
    with pytest.raises(ValueError, match="duplicate"):
        p.append_generated([101])
    with pytest.raises(ValueError, match="duplicate"):
        p.append_generated([50])
    p.grow_capacity(5)
    with pytest.raises(ValueError, match="only grow"):
        p.grow_capacity(4)
    # growth past the allocated slot range migrates the pool transparently
    q = ess.SparsePool(2, cap_max=4)
    q.access_step([1, 2])
    q.grow_capacity(9)
    q.access_step(list(range(3, 10)))
    assert q.lru_order() == [1, 2, 3, 4, 5, 6, 7, 8, 9]


def test_sparse_pool_random_vs_linear_oracle(ess):
    rng = np.random.default_rng(5)
    for _ in range(60):
        cap = int(rng.integers(1, 40))
        pool, lin = ess.SparsePool(cap), olru.LinearLRU(cap)
        nxt = 5000
        for _ in range(int(rng.integers(1, 10))):
            req = [int(x) for x in rng.choice(300, size=int(rng.integers(1, 60)), replace=False)]
            r = pool.access_step(req)
            h, m, e = lin.access(req)
            assert (r.hit_ids, r.miss_ids, r.evicted_ids) == (h, m, e)
            if rng.random() < 0.3:
                new = list(range(nxt, nxt + int(rng.integers(1, 4))))
                nxt += 10
                pool.append_generated(new)
                lin.append(new)
            assert pool.lru_order() == lin.order


@pytest.mark.parametrize("name", ["small", "c1", "mtp", "c2"])
def test_replay_matches_reference(ess, name):
    exp = G.replay_expect()[name]
    t = G.replay_trace(name)
    for res in exp["results"]:
        prof = ess.replay(t, res["ratio"], use_warmup=res["use_warmup"],
                          preload_full_history=res["preload"])
        np.testing.assert_array_equal(prof.misses, np.asarray(res["misses"]),
                                      err_msg=f"{name} {res}")


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_step_lists_match_reference(ess, name):
    """Per-step hit/miss/evicted lists of layer 0 at the BASELINE sizes (c1: oversize
    path every step; c2: 32K ctx, cap 8192) against offsim's own lists."""
    want = G.step_lists(name)
    t = G.replay_trace(name)
    ratio, L = 0.25, t.num_layers
    total = t.context_len + sum(s.tokens_accepted for s in t.steps)
    pools = ess.PoolSet(L, total, ess.pool_capacity(ratio, total),
                        ess.pool_capacity(ratio, t.context_len))
    for w in range(len(t.prefill_windows[0])):
        ids, n = ess._pad_windows([t.prefill_windows[l][w] for l in range(L)], "cuda")
        pools.warmup(ids, n)
    hist = t.context_len
    for step_i, s in enumerate(t.steps):
        req, n = t.padded_step(step_i)
        r = pools.access(torch.as_tensor(req, device="cuda"), torch.as_tensor(n, device="cuda"),
                         lists=True)
        c = r.counts[0].tolist()
        assert r.hit_ids[0, :c[0]].tolist() == want["hits"][step_i]
        assert r.miss_ids[0, :c[1]].tolist() == want["misses"][step_i]
        assert r.evicted_ids[0, :c[2]].tolist() == want["evicted"][step_i]
        hist += s.tokens_accepted
        pools.grow(ess.pool_capacity(ratio, hist))
        new = torch.arange(hist - s.tokens_accepted, hist, dtype=torch.int32, device="cuda")
        pools.append(new.expand(L, -1).contiguous(),
                     torch.full((L,), s.tokens_accepted, dtype=torch.int32, device="cuda"))
    out, cnt = pools.lru_order(0, 1)
    assert out[0, :int(cnt[0])].tolist() == want["lru_final"]
    ctr = pools.counters(0, 1)[0].tolist()
    assert ctr[2:5] == want["stats"]
    pools.check()


def _random_sets(rng, P, K, universe, prev=None, keep=0.9):
    out = np.zeros((P, K), np.int32)
    for p in range(P):
        if prev is None:
            s = rng.choice(universe, size=K, replace=False)
        else:
            kept = prev[p][rng.random(K) < keep]
            pool = np.setdiff1d(np.arange(universe), kept, assume_unique=False)
            s = np.concatenate([kept, rng.choice(pool, size=K - len(kept), replace=False)])
        rng.shuffle(s)  # arbitrary request order: lists must follow it
        out[p] = s
    return out


@pytest.mark.parametrize("P,cap,K,universe", [(64, 8192, 2048, 32768), (8, 1024, 2048, 4096),
                                              (16, 13107, 2048, 131072), (4, 3000, 1500, 9000)])
def test_batched_pools_vs_c_oracle_at_scale(ess, P, cap, K, universe):
    rng = np.random.default_rng(P + cap)
    pools = ess.PoolSet(P, universe + 64, cap + 64, cap)
    orc = [olru.OraclePool(cap) for _ in range(P)]
    prev = None
    gen = universe
    for step in range(6):
        sets = _random_sets(rng, P, K, universe, prev)
        prev = sets
        n = np.full(P, K, np.int32)
        r = pools.access(torch.as_tensor(sets, device="cuda"), torch.as_tensor(n, device="cuda"),
                         lists=True)
        counts = r.counts.cpu().numpy()
        hits, misses, ev = r.hit_ids.cpu().numpy(), r.miss_ids.cpu().numpy(), r.evicted_ids.cpu().numpy()
        for p in range(P):
            o = orc[p].access_step(sets[p].tolist())
            assert hits[p, :counts[p, 0]].tolist() == o.hit_ids
            assert misses[p, :counts[p, 1]].tolist() == o.miss_ids
            assert ev[p, :counts[p, 2]].tolist() == o.evicted_ids
        # grow + append one generated id per pool
        for o in orc:
            o.grow_capacity(cap + step + 1)
            o.append_generated([gen])
        pools.grow(cap + step + 1)
        pools.append(torch.full((P, 1), gen, dtype=torch.int32, device="cuda"),
                     torch.ones(P, dtype=torch.int32, device="cuda"))
        gen += 1
    out, cnt = pools.lru_order()
    out, cnt = out.cpu().numpy(), cnt.cpu().numpy()
    for p in range(P):
        assert out[p, :cnt[p]].tolist() == orc[p].lru_order()
    ctr = pools.counters().cpu().numpy()
    for p in range(P):
        assert ctr[p, 2:5].tolist() == [orc[p].hits, orc[p].misses, orc[p].evictions]
    pools.check()


def test_sel_row_and_miss_rows_consistent(ess):
    """sel_row is where every requested id lives after the step; miss_row lists the
    misses' rows in requested order; transient (oversize) ids land in staging."""
    P, cap, K = 4, 1000, 2048
    pools = ess.PoolSet(P, 8192, cap, cap, row_bytes=1152, staging_rows=K)
    rng = np.random.default_rng(1)
    sets = _random_sets(rng, P, K, 8192)
    n = np.full(P, K, np.int32)
    r = pools.access(torch.as_tensor(sets, device="cuda"), torch.as_tensor(n, device="cuda"))
    sel = r.sel_row.cpu().numpy()
    keep0 = K - cap
    assert (sel[:, :keep0] == cap + np.arange(keep0)).all()   # staging rows = cap_max + i
    for p in range(P):
        slots = pools.lookup(p, torch.as_tensor(sets[p], device="cuda")).cpu().numpy()
        assert (slots[:keep0] == -1).all()
        np.testing.assert_array_equal(slots[keep0:], sel[p, keep0:])
        assert len(set(sel[p, keep0:].tolist())) == cap
    pools.check()


def test_device_errors_latch(ess):
    pools = ess.PoolSet(2, 100, 10, 5)
    bad = torch.tensor([[1, 200], [3, 4]], dtype=torch.int32, device="cuda")
    pools.access(bad, torch.tensor([2, 2], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        pools.check()
    pools.grow(3)
    with pytest.raises(ValueError, match="only grow"):
        pools.check()
