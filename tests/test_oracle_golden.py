"""Pin the CPU oracle to the reference: every golden vector produced by the real
offsim (tests/golden/make_golden.py) must be reproduced exactly."""
import numpy as np
import pytest

from oracle import lru as olru
from tests import _golden as G


def run_workload(pool_cls, w):
    pool = pool_cls(w["capacity"])
    for op in w["ops"]:
        if op["op"] == "warmup":
            assert pool.warmup(op["windows"]) == op["inserted"]
        elif op["op"] == "access":
            r = pool.access_step(op["req"])
            assert r.hit_ids == op["hit"]
            assert r.miss_ids == op["miss"]
            assert r.evicted_ids == op["evicted"]
            assert r.h2d_blocks == op["h2d"]
        else:
            pool.grow_capacity(op["grow_to"])
            assert pool.append_generated(op["new"]) == op["d2h"]
        assert pool.lru_order() == op["lru"]
    return pool


def test_c_oracle_matches_reference_lru_workloads():
    ws = G.lru_workloads()
    assert len(ws) == 400
    for w in ws:
        pool = run_workload(olru.OraclePool, w)
        assert [pool.hits, pool.misses, pool.evictions] == w["stats"]


def test_linear_oracle_matches_reference_lru_workloads():
    for w in G.lru_workloads()[:150]:
        lin = olru.LinearLRU(w["capacity"])
        for op in w["ops"]:
            if op["op"] == "warmup":
                assert lin.warmup(op["windows"]) == op["inserted"]
            elif op["op"] == "access":
                h, m, e = lin.access(op["req"])
                assert (h, m, e) == (op["hit"], op["miss"], op["evicted"])
            else:
                lin.capacity = op["grow_to"]
                lin.append(op["new"])
            assert lin.order == op["lru"]


@pytest.mark.parametrize("name", ["small", "c1", "mtp", "c2"])
def test_c_oracle_replay_matches_reference(name):
    exp = G.replay_expect()[name]
    t = G.replay_trace(name)
    for res in exp["results"]:
        got = olru.replay_misses([s.layers for s in t.steps], [s.tokens_accepted for s in t.steps],
                                 t.context_len, res["ratio"], t.prefill_windows,
                                 use_warmup=res["use_warmup"], preload_full_history=res["preload"])
        np.testing.assert_array_equal(got, np.asarray(res["misses"]))


def test_oracle_pool_capacity_constants():
    for r, h, c in G.constants()["pool_capacity"]:
        assert olru.pool_capacity(r, h) == c


def test_oracle_errors_match_reference():
    with pytest.raises(ValueError):
        olru.OraclePool(0)
    p = olru.OraclePool(3)
    p.grow_capacity(5)
    with pytest.raises(ValueError, match="only grow"):
        p.grow_capacity(4)
    p.access_step([0, 1])
    p.append_generated([100, 101])
    with pytest.raises(ValueError, match="duplicate"):
        p.append_generated([101])
    with pytest.raises(ValueError, match="duplicate"):
        p.append_generated([50])
