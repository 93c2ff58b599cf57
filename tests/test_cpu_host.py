"""CPU-only tests: the C ABI library loads and exports every header symbol, host-side
validation mirrors the reference's errors, trace tooling and transfer constants
match the reference's golden vectors, and the data-parallel sharding/aggregation
works across 2 gloo ranks."""
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_10576_b200 import _lib
from paper_2512_10576_b200 import trace as tr
from tests import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ess_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ess_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = _lib.load()  # no CUDA call happens here
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"
    assert L.ess_version().decode().startswith("ess_b200")
    assert "only grow" in _lib.status_text(_lib.ESS_ERR_SHRINK)


def test_header_constants_match_python_mirror():
    src = open(os.path.join(ROOT, "include", "ess_b200.h")).read()
    defs = dict(re.findall(r"#define (ESS_[A-Z0-9_]+) \(?(-?[0-9]+)", src))
    assert int(defs["ESS_LATENT_ROW_BYTES"]) == _lib.LATENT_ROW_BYTES == 656
    assert int(defs["ESS_SLOT_ROW_BYTES"]) == _lib.SLOT_ROW_BYTES_F16 == 1152
    assert int(defs["ESS_SLOT_ROW_BYTES_FP8"]) == _lib.SLOT_ROW_BYTES_FP8 == 656
    assert _lib.SLOT_ROW_BYTES in (656, 1152)
    assert int(defs["ESS_TOPK_MAX_K"]) == 65535
    assert int(defs["ESS_HOST_ROW_PITCH"]) == _lib.HOST_ROW_PITCH
    assert _lib.HOST_ROW_PITCH % 64 == 0 and _lib.HOST_ROW_PITCH >= _lib.LATENT_ROW_BYTES
    assert int(defs["ESS_MLA_PARTIAL"]) == _lib.ESS_MLA_PARTIAL
    assert int(defs["ESS_MLA_RESUME"]) == _lib.ESS_MLA_RESUME
    assert int(defs["ESS_GATHER_EXCLUSIVE_SM"]) == _lib.ESS_GATHER_EXCLUSIVE_SM
    assert int(defs["ESS_GATHER_BULK"]) == _lib.ESS_GATHER_BULK
    assert re.search(r"#define ESS_LAUNCH_PDL \(1 << 30\)", src) and _lib.ESS_LAUNCH_PDL == 1 << 30


def test_launch_flags_are_validated_without_gpu():
    """ess_topk_split_ex rejects unknown launch flags before touching the device."""
    L = _lib.load()
    rc = L.ess_topk_split_ex(None, 128, None, 1, 1, None, 1, None, None, 0, None, None, None, None, 1,
                             1 << 3, None)
    assert rc == _lib.ESS_ERR_ARG


def test_status_mapping():
    with pytest.raises(ValueError, match="duplicate"):
        _lib.check(_lib.ESS_ERR_DUPLICATE)
    with pytest.raises(MemoryError):
        _lib.check(_lib.ESS_ERR_NOMEM)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ESS_ERR_CUDA)
    _lib.check(_lib.ESS_OK)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_validation_without_gpu():
    from paper_2512_10576_b200 import cache
    with pytest.raises(ValueError):
        cache.SparsePool(0)
    with pytest.raises(ValueError):
        cache.replay(G.replay_trace("small"), 0.0)
    with pytest.raises(ValueError):
        cache.replay(G.replay_trace("small"), 1.5)
    for r, h, c in G.constants()["pool_capacity"]:
        assert cache.pool_capacity(r, h) == c


def test_runs_without_repeats_is_sequential_split():
    from paper_2512_10576_b200.cache import _runs_without_repeats
    runs = list(_runs_without_repeats([1, 2, 1, 3, 3, 4], 2048))
    assert runs == [[1, 2], [1, 3], [3, 4]]
    assert [len(r) for r in _runs_without_repeats(list(range(5000)), 2048)] == [2048, 2048, 904]


def test_transfer_constants_match_reference():
    from paper_2512_10576_b200.transfer import TransferModel, transfer_time
    models = {"batched": TransferModel(mode="batched"), "per_call": TransferModel(mode="per_call")}
    for mode, blocks, d, want in G.constants()["transfer"]:
        assert transfer_time(models[mode], blocks, d) == pytest.approx(want, rel=1e-12)
    assert transfer_time(models["batched"], 2048, "h2d") == pytest.approx(36.3, abs=0.1)
    with pytest.raises(ValueError):
        transfer_time(models["batched"], -1, "h2d")
    with pytest.raises(ValueError):
        TransferModel(mode="bogus")


# ---------------------------------------------------------------- trace tooling
def small(**kw):
    base = dict(num_layers=2, context_len=1024, topk=128, num_steps=20,
                target_similarity=0.9, seed=7)
    base.update(kw)
    return tr.TraceGenParams(**base)


@pytest.mark.parametrize("name", ["small", "c1", "mtp", "c2"])
def test_generator_reproduces_reference_traces(name):
    """Our generator's selection sets are identical to offsim's (same numpy)."""
    exp = G.replay_expect()[name]
    ref = G.replay_trace(name)
    got = tr.generate_trace(tr.TraceGenParams(**exp["params"]))
    assert tr.encode_trace(got) == tr.encode_trace(ref)
    sims = [s.mean for s in tr.similarity_summary(got)]
    np.testing.assert_allclose(sims, exp["similarity"], rtol=0, atol=1e-12)


def test_generator_properties():
    t = tr.generate_trace(small())
    t.check()
    assert all(len(a) == 128 for s in t.steps for a in s.layers)
    assert all(len(w) == tr.PREFILL_WINDOW_COUNT for w in t.prefill_windows)
    for s in tr.similarity_summary(tr.generate_trace(small(num_steps=60))):
        assert s.mean == pytest.approx(0.9, abs=0.03)
    top = max(int(s.layers[0].max()) for s in tr.generate_trace(small(num_steps=40, target_similarity=0.2)).steps)
    assert top >= 1024
    assert tr.TraceGenParams(target_similarity=1.5).violations()
    with pytest.raises(ValueError):
        tr.generate_trace(tr.TraceGenParams(target_similarity=-0.1))


def test_trace_io_errors(tmp_path):
    t = tr.generate_trace(small(num_steps=3))
    p = tmp_path / "t.bin"
    tr.write_trace(t, p)
    data = p.read_bytes()
    back = tr.read_trace(p)
    assert tr.encode_trace(back) == data
    p.write_bytes(b"NOTATRCE" + b"\0" * 32)
    with pytest.raises(tr.TraceFormatError, match="magic") as e:
        tr.read_trace(p)
    assert e.value.offset == 0
    p.write_bytes(data[: len(data) // 2])
    with pytest.raises(tr.TraceFormatError, match="truncated") as e:
        tr.read_trace(p)
    assert 0 < e.value.offset <= len(data) // 2
    p.write_bytes(data + b"\0\1")
    with pytest.raises(tr.TraceFormatError, match="trailing"):
        tr.read_trace(p)
    t.steps[1].layers[0] = np.array([5, 4], dtype=np.uint32)
    with pytest.raises(ValueError, match="strictly increasing"):
        t.check()
    t2 = tr.generate_trace(small(num_steps=2))
    t2.steps[0].layers[0] = np.array([t2.context_len + 100], dtype=np.uint32)
    tr.write_trace(t2, p)
    with pytest.raises(tr.TraceFormatError, match="out of range"):
        tr.read_trace(p)


# ---------------------------------------------------------------- data parallel (gloo)
def test_shard_requests_partition():
    from paper_2512_10576_b200.dp import shard_requests
    for world in (1, 2, 4, 8):
        parts = [shard_requests(128, world, r) for r in range(world)]
        assert sorted(sum(parts, [])) == list(range(128))
    lens = np.random.default_rng(0).integers(8192, 131072, size=40)
    parts = [shard_requests(40, 8, r, lens) for r in range(8)]
    assert sorted(sum(parts, [])) == list(range(40))
    loads = [int(lens[p].sum()) for p in parts]
    assert max(loads) - min(loads) <= int(lens.max())


def _worker(rank, world, port, q):
    from paper_2512_10576_b200.dp import aggregate, shard_requests
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    mine = shard_requests(64, world, rank)
    tok, sec = aggregate(len(mine), 0.5 + rank)
    q.put((rank, mine, tok, sec))
    dist.destroy_process_group()


def test_dp_aggregate_two_gloo_ranks():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert sorted(res[0][1] + res[1][1]) == list(range(64))
    assert all(r[2] == 64 and r[3] == 1.5 for r in res)


def test_micro_batch_partitions():
    """DBA request ranges: contiguous, covering the batch, first-share / explicit sizes."""
    import types
    from paper_2512_10576_b200.decode import DSADecodeLayer
    mb = DSADecodeLayer.micro_batches
    o = types.SimpleNamespace(B=64, first_frac=None, mb_sizes=None)
    assert mb(o, 1) == [(0, 64)]
    assert mb(o, 2) == [(0, 32), (32, 64)]
    o.first_frac = 0.25
    assert mb(o, 2) == [(0, 16), (16, 64)]
    assert mb(o, 3) == [(0, 16), (16, 40), (40, 64)]
    o.mb_sizes = [8, 16, 40]
    assert mb(o, 3) == [(0, 8), (8, 24), (24, 64)]
    o.mb_sizes = [8, 8]
    with pytest.raises(ValueError):
        mb(o, 2)
    o = types.SimpleNamespace(B=3, first_frac=0.9, mb_sizes=None)
    r = mb(o, 3)
    assert r[0][0] == 0 and r[-1][1] == 3 and all(a < b for a, b in r)


def test_bench_request_lengths():
    """C5's mixed batch: seeded log-uniform lengths within the configured range."""
    import bench
    lens = bench.request_lengths(bench.CONFIGS["c5"], 64, seed=0)
    assert len(lens) == 64 and min(lens) >= 8192 and max(lens) <= 131072
    assert lens == bench.request_lengths(bench.CONFIGS["c5"], 64, seed=0)
    assert lens != bench.request_lengths(bench.CONFIGS["c5"], 64, seed=1)
    assert bench.request_lengths(bench.CONFIGS["c2"], 4) == [32768] * 4
