"""Regenerate the golden fixtures from the REAL reference (offsim), imported from
/root/reference/pkg/src in the build container.  The GPU box has no
/root/reference, so tests only ever read the committed outputs of this script.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (all under tests/golden/):
  lru_workloads.json.gz  random op sequences on offsim.cache.SparsePool with every
                         result (hit/miss/evicted lists, h2d blocks, inserted counts,
                         lru_order after each op, final stats) — cache.py:29-134
  replay_<name>.esstrace trace files written by offsim.trace.write_trace
  replay_expect.json     offsim.cache.replay miss profiles for each trace and
                         (ratio, warm-up, preload) combination — cache.py:166-196
  steps_<name>.npz       per-step access results (hits, misses, evicted) for one
                         layer of a trace at scale, plus the final lru_order
  constants.json         transfer_time / pool_capacity known answers
                         (costmodel.py:173-186, cache.py:137-138)
"""

from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from offsim import cache, trace as tr  # noqa: E402
from offsim.costmodel import TransferModel, transfer_time  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def lru_workloads(n_work=400, seed=20260):
    rng = np.random.default_rng(seed)
    out = []
    for w in range(n_work):
        cap = int(rng.integers(1, 65))
        universe = int(rng.choice([40, 128, 400]))
        pool = cache.SparsePool(cap)
        ops = []
        if rng.random() < 0.4:
            wins = [sorted(int(x) for x in rng.choice(universe, size=int(rng.integers(1, min(80, universe))),
                                                       replace=False))
                    for _ in range(int(rng.integers(1, 5)))]
            ins = pool.warmup(wins)
            ops.append({"op": "warmup", "windows": wins, "inserted": ins,
                        "lru": pool.lru_order()})
        next_gen = 1000
        for _ in range(int(rng.integers(1, 14))):
            size = int(rng.integers(1, min(80, universe)))
            req = [int(x) for x in rng.choice(universe, size=size, replace=False)]
            if rng.random() < 0.5:
                req.sort()
            r = pool.access_step(req)
            ops.append({"op": "access", "req": req, "hit": r.hit_ids, "miss": r.miss_ids,
                        "evicted": r.evicted_ids, "h2d": r.h2d_blocks,
                        "lru": pool.lru_order()})
            if rng.random() < 0.35:
                new = list(range(next_gen, next_gen + int(rng.integers(1, 4))))
                next_gen = new[-1] + 1
                grow = int(rng.integers(0, 4))
                pool.grow_capacity(pool.capacity + grow)
                d2h = pool.append_generated(new)
                ops.append({"op": "append", "grow_to": pool.capacity, "new": new,
                            "d2h": d2h, "lru": pool.lru_order()})
        out.append({"capacity": cap, "ops": ops,
                    "stats": [pool.hits, pool.misses, pool.evictions]})
    return out


REPLAY_TRACES = {
    # name: (TraceGenParams kwargs)
    "small": dict(num_layers=2, context_len=1024, topk=128, num_steps=20,
                  target_similarity=0.9, seed=0),
    "c1": dict(num_layers=2, context_len=4096, topk=2048, num_steps=6,
               target_similarity=0.9, mean_accept=1.0, seed=3),
    "mtp": dict(num_layers=3, context_len=2048, topk=256, num_steps=24,
                target_similarity=0.8, mean_accept=2.2, seed=11),
    "c2": dict(num_layers=1, context_len=32768, topk=2048, num_steps=4,
               target_similarity=0.9, mean_accept=1.0, seed=0),
}
REPLAY_COMBOS = [(0.1, True, False), (0.2, True, False), (0.25, True, False),
                 (0.25, False, False), (0.4, True, False), (0.6, False, False),
                 (1.0, True, False), (1.0, False, True)]


def per_step_results(trace, ratio, layer=0):
    """Drive offsim pools exactly like cache.replay (cache.py:176-195) and record
    one layer's per-step lists."""
    pools = [cache.SparsePool(cache.pool_capacity(ratio, trace.context_len))
             for _ in range(trace.num_layers)]
    for l, p in enumerate(pools):
        p.warmup(trace.prefill_windows[l])
    hits, misses, evicted, hist = [], [], [], trace.context_len
    for step in trace.steps:
        for l, p in enumerate(pools):
            r = p.access_step(step.layers[l])
            if l == layer:
                hits.append(np.asarray(r.hit_ids, np.int32))
                misses.append(np.asarray(r.miss_ids, np.int32))
                evicted.append(np.asarray(r.evicted_ids, np.int32))
        new = range(hist, hist + step.tokens_accepted)
        hist += step.tokens_accepted
        for p in pools:
            p.grow_capacity(cache.pool_capacity(ratio, hist))
            p.append_generated(new)
    pack = {}
    for name, seq in (("hits", hits), ("misses", misses), ("evicted", evicted)):
        pack[name + "_off"] = np.cumsum([0] + [len(a) for a in seq]).astype(np.int64)
        pack[name] = np.concatenate(seq) if seq else np.zeros(0, np.int32)
    pack["lru_final"] = np.asarray(pools[layer].lru_order(), np.int32)
    pack["stats"] = np.asarray([pools[layer].hits, pools[layer].misses,
                                pools[layer].evictions], np.int64)
    return pack


def main():
    with gzip.open(os.path.join(HERE, "lru_workloads.json.gz"), "wt") as f:
        json.dump(lru_workloads(), f, separators=(",", ":"))

    expect = {}
    for name, kw in REPLAY_TRACES.items():
        t = tr.generate_trace(tr.TraceGenParams(**kw))
        tr.write_trace(t, os.path.join(HERE, f"replay_{name}.esstrace"))
        res = []
        for ratio, warm, pre in REPLAY_COMBOS:
            prof = cache.replay(t, ratio, use_warmup=warm, preload_full_history=pre)
            res.append({"ratio": ratio, "use_warmup": warm, "preload": pre,
                        "misses": prof.misses.tolist()})
        expect[name] = {"params": kw, "results": res,
                        "similarity": [s.mean for s in tr.similarity_summary(t)]}
        if name in ("c1", "c2"):
            np.savez_compressed(os.path.join(HERE, f"steps_{name}.npz"),
                                **per_step_results(t, 0.25))
    with open(os.path.join(HERE, "replay_expect.json"), "w") as f:
        json.dump(expect, f)

    batched, per_call = TransferModel(mode="batched"), TransferModel(mode="per_call")
    const = {
        "transfer": [[m.mode, b, d, transfer_time(m, b, d)]
                     for m in (batched, per_call) for b in (0, 1, 150, 2048, 9600)
                     for d in ("h2d", "d2h")],
        "pool_capacity": [[r, h, cache.pool_capacity(r, h)]
                          for r in (0.001, 0.1, 0.2, 0.25, 0.5, 1.0)
                          for h in (1, 100, 4096, 32768, 131072, 131073)],
    }
    with open(os.path.join(HERE, "constants.json"), "w") as f:
        json.dump(const, f)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
