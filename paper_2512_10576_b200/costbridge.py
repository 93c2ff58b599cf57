"""Measured-cost bridge into the reference simulator.

The reference reduces every GPU operator of the decode step to a cost-table lookup
``op_time(table, op, batch, context)`` (/root/reference/pkg/src/offsim/costmodel.py:
93-101) over a CSV ``op,batch,context,time_us`` whose points form a full
batch x context grid per op (costmodel.py:44-68, :104-125), and prices the host link
with ``TransferModel(bw_h2d_gbs=...)`` (costmodel.py:140-170).  Its shipped profiles
are synthetic fits (profiles.py:1-7).  This module measures the operators this repo
implements on the B200 and writes them in exactly that format, so
``offsim simulate/sweep --profile <csv>`` predicts decode on B200 from real kernel
times ("metadata collected from real machine executions"):

==================  =================================================================
``indexer_logits``  K1 over ``batch`` requests x ``context`` tokens (one launch)
``indexer_topk``    K2 top-2048 over the same rows
``sparse_mla``      K5 over min(2048, context) selected rows per request
``merge_attn``      K5 resume pass with no new rows: the LSE merge of a split attention
==================  =================================================================

Ops outside the hot path (``pre_attn``, ``dense_mlp``, ``moe_dispatch``,
``moe_combine``) are not measured; ``merge_cost_tables`` fills them from a base
profile CSV (e.g. one saved from ``offsim.profiles.calibrated_profile``).

Only the GPU timing needs CUDA; the CSV helpers are plain Python.
"""

from __future__ import annotations

import csv
import json
import os

OP_NAMES = ("indexer_logits", "indexer_topk", "pre_attn", "sparse_mla", "dense_mlp",
            "moe_dispatch", "moe_combine", "merge_attn")   # costmodel.py:18-27, same order
MEASURED_OPS = ("indexer_logits", "indexer_topk", "sparse_mla", "merge_attn")
DEFAULT_BATCHES = (1, 4, 16, 64, 128)
DEFAULT_CONTEXTS = (4096, 16384, 32768, 65536, 131072)
TOPK = 2048


# -------------------------------------------------------------------------------------
# CSV side (the reference's format; no CUDA)
# -------------------------------------------------------------------------------------
def check_grid(entries: dict) -> None:
    """The reference CostTable invariants (costmodel.py:44-68): known op names,
    positive times, no duplicate (batch, context), a full grid per op."""
    for op, pts in entries.items():
        if op not in OP_NAMES:
            raise ValueError(f"unknown op name: {op}")
        if not pts:
            raise ValueError(f"op {op} has no points")
        seen = set()
        for b, c, t in pts:
            if not t > 0:
                raise ValueError(f"op {op}: non-positive time at batch={b} context={c}")
            if (b, c) in seen:
                raise ValueError(f"op {op}: duplicate point batch={b} context={c}")
            seen.add((b, c))
        bs, cs = {b for b, _ in seen}, {c for _, c in seen}
        if len(seen) != len(bs) * len(cs):
            raise ValueError(f"op {op}: points do not form a full batch x context grid")


def write_cost_table(entries: dict, path) -> None:
    """save_cost_table's format (costmodel.py:118-125): header op,batch,context,time_us,
    ops in OP_NAMES order, points batch-major."""
    check_grid(entries)
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["op", "batch", "context", "time_us"])
        for op in OP_NAMES:
            for b, c, t in sorted(entries.get(op, [])):
                w.writerow([op, f"{b:g}", f"{c:g}", f"{t:.9g}"])


def read_cost_table(path) -> dict:
    """load_cost_table's parse (costmodel.py:104-115) into {op: [(batch, ctx, us)]}."""
    entries: dict = {}
    with open(path, newline="") as f:
        r = csv.DictReader(f)
        if set(r.fieldnames or []) != {"op", "batch", "context", "time_us"}:
            raise ValueError(f"{path}: expected header op,batch,context,time_us")
        for lineno, rec in enumerate(r, start=2):
            if rec["op"] not in OP_NAMES:
                raise ValueError(f"{path}:{lineno}: unknown op name {rec['op']!r}")
            entries.setdefault(rec["op"], []).append(
                (float(rec["batch"]), float(rec["context"]), float(rec["time_us"])))
    check_grid(entries)
    return entries


def merge_cost_tables(measured: dict, base: dict) -> dict:
    """Measured ops replace the base profile's; every other op keeps the base grid."""
    out = {op: list(pts) for op, pts in base.items()}
    out.update({op: list(pts) for op, pts in measured.items()})
    check_grid(out)
    return out


def transfer_model_dict(h2d_gbs: float, d2h_gbs: float | None = None) -> dict:
    """TransferModel fields (costmodel.py:140-170) for the measured batched gather:
    ``mode="batched"`` is the FlashTrans-style address-list copy this repo's K4 is."""
    return {"mode": "batched", "bw_h2d_gbs": float(h2d_gbs),
            "bw_d2h_gbs": float(d2h_gbs if d2h_gbs is not None else h2d_gbs),
            "block_bytes": 656}


# -------------------------------------------------------------------------------------
# GPU side: time each op on the B200 kernels
# -------------------------------------------------------------------------------------
def _time_us(fn, iters: int = 5, warmup: int = 2) -> float:
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        torch.cuda._sleep(200_000)  # the host runs ahead: launch latency stays hidden
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def measure_ops(batches=DEFAULT_BATCHES, contexts=DEFAULT_CONTEXTS, device=None, seed: int = 0,
                iters: int = 5) -> dict:
    """{op: [(batch, context, us)]} for MEASURED_OPS on the current GPU.  Inputs are
    synthetic of the DSA shapes (decode.random_latent_rows, N(0,1) e4m3 keys); K5 and
    the merge read min(2048, context) distinct rows of a slot pool per request."""
    import torch

    from .attention import SplitWorkspace, sparse_mla
    from .cache import PoolSet
    from .decode import _e4m3
    from .indexer import indexer_logits, topk

    dev = torch.device(device if device is not None else "cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    out: dict = {op: [] for op in MEASURED_OPS}
    bmax, cmax = max(batches), max(contexts)
    cap = max(TOPK, 4096)
    pools = PoolSet(bmax, cap, cap, cap, row_bytes=1152, staging_rows=0, device=dev)
    rv = pools.rows_view()
    rv.copy_((torch.randn(rv.shape, device=dev, generator=g) * 0.5).half())
    q = (torch.randn((bmax, 128, 576), device=dev, generator=g) * 0.5).to(torch.bfloat16)
    sel = torch.stack([torch.randperm(cap, device=dev, generator=g)[:TOPK] for _ in range(bmax)]).int()
    ws = SplitWorkspace(bmax, dev)
    zero = torch.zeros(bmax, dtype=torch.int32, device=dev)
    k_all = _e4m3(torch.randn((bmax, cmax, 128), device=dev, generator=g) * 8)
    ks_all = torch.rand((bmax, cmax), device=dev, generator=g) + 0.5
    w = torch.randn((bmax, 64), device=dev, generator=g) / 8
    qi = _e4m3(torch.randn((bmax, 64, 128), device=dev, generator=g) * 4)
    logits = torch.empty((bmax, cmax), device=dev)
    idx = torch.empty((bmax, TOPK), dtype=torch.int32, device=dev)
    cnt = torch.empty(bmax, dtype=torch.int32, device=dev)
    for B in batches:
        for C in contexts:
            # caches allocated for the longest context, len = C (the decode layout)
            lens = torch.full((B,), C, dtype=torch.int32, device=dev)
            k, ks, lg = k_all[:B], ks_all[:B], logits[:B]
            t1 = _time_us(lambda: indexer_logits(qi[:B], w[:B], k, ks, lens, out=lg), iters)
            t2 = _time_us(lambda: topk(lg, lens, TOPK, out=idx[:B], count=cnt[:B]), iters)
            n = torch.full((B,), min(TOPK, C), dtype=torch.int32, device=dev)
            t5 = _time_us(lambda: sparse_mla(pools, q[:B], sel[:B], n), iters)
            sparse_mla(pools, q[:B], sel[:B], n, workspace=ws, mode="partial")
            tm = _time_us(lambda: sparse_mla(pools, q[:B], sel[:B], zero[:B], workspace=ws,
                                             mode="resume"), iters)
            for op, t in zip(MEASURED_OPS, (t1, t2, t5, tm)):
                out[op].append((float(B), float(C), float(t)))
    pools.close()
    return out


def export(path_csv: str, gather_gbs: float | None = None, **kw) -> dict:
    """Measure, write the CSV (and a .transfer.json next to it when the gather rate is
    given), return the entries."""
    entries = measure_ops(**kw)
    write_cost_table(entries, path_csv)
    if gather_gbs is not None:
        with open(os.path.splitext(path_csv)[0] + ".transfer.json", "w") as f:
            json.dump(transfer_model_dict(gather_gbs), f, indent=1)
    return entries
