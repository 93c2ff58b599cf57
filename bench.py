"""Offloaded DSA decode step benchmark (BASELINE.json metric: decode tokens/s/GPU with
the latent cache offloaded, plus H2D gather GB/s).

    python bench.py [--gpus N --steps K --warmup W] [--config c2|c4] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, weak scaling)

One step = one DSA layer decode for every request on the GPU: K1 lightning indexer
-> K2 top-2048 -> K3 LRU cache manager -> K4 zero-copy miss gather -> K5 sparse MLA,
then each request appends its generated token (grow, admit, D2H write-back).
Synthetic inputs of DeepSeek-V3.2-Exp shapes, random weights; every per-step input
is generated before the timed region.  The working set (indexer keys + slot pool,
>600 MB/GPU at C2) is larger than the 126 MB L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]: one V3.2-Exp DSA layer, batch 64, ctx 32K, 25% slot pool
    # micro / first: the DBA split (micro-batches, share of the first one), tuned per
    # workload on B200: a small first micro-batch starts the host-link
    # gather early; more micro-batches pay when the gather dominates (C4)
    "c2": dict(name="c2", batch=64, context_len=32768, sparse_ratio=0.25, micro=2, first=0.25,
               workload="C2: one DSA layer decode, batch 64/GPU, ctx 32K, 25% GPU slot pool"),
    # configs[3]: ctx 128K, batch 64/GPU, 10% slot pool
    # configs[2]: the full 61-layer attention path, global batch 128 over 8 GPUs = 16/GPU
    "c3": dict(name="c3", batch=16, context_len=32768, sparse_ratio=0.25, micro=1, first=None, layers=61,
               workload="C3: 61-layer decode step (attention path), batch 16/GPU "
                        "(global 128 over 8 GPUs), ctx 32K, 25% GPU slot pool"),
    # configs[4]: mixed-length batch, context log-uniform over [8K, 128K] (seeded per rank);
    # the pool-size / hit-rate sweep is scripts/sweep_c5.py
    "c5": dict(name="c5", batch=64, context_len=(8192, 131072), sparse_ratio=0.25, micro=2, first=0.375,
               workload="C5: one DSA layer decode, batch 64/GPU of mixed 8K-128K contexts "
                        "(log-uniform), 25% GPU slot pool"),
    "c4": dict(name="c4", batch=64, context_len=131072, sparse_ratio=0.10, micro=3, first=0.1875,
               workload="C4: one DSA layer decode, batch 64/GPU, ctx 128K, 10% GPU slot pool"),
}
TOPK = 2048
LINK_ROW_BYTES = 64 * ((656 + 63) // 64)  # a 64-B aligned 656-B row in 64-B read completions
# K4 alone in the breakdown: 64 CTAs.  Random row reads across a multi-GB host store are
# limited per SM (address translation), not per request in flight: at C4's 5.5-GiB store
# 20 / 32 CTAs reach 30 / 36 GB/s, >= 48 CTAs the 41-42 GB/s that 20 reach at C2's 1.4 GiB
# (profiles/r02_gather_store_size.txt)
BREAKDOWN_GATHER_CTAS = 64
METRIC = "decode tokens/s/GPU at 32K/128K ctx, latent cache offloaded; H2D gather GB/s"


def request_lengths(cfg, n, seed=0):
    """Per-request context lengths: the config's single length, or (C5) a seeded
    log-uniform draw over [lo, hi] — the mixed 8K-128K batch of BASELINE configs[4]."""
    L = cfg["context_len"]
    if isinstance(L, int):
        return [L] * n
    import numpy as np
    lo, hi = L
    rng = np.random.default_rng(seed)
    return [int(x) for x in np.exp(rng.uniform(np.log(lo), np.log(hi), size=n)).round()]


def workload_config(cfg, args):
    """The workload both arms run, identical in our line and the reference arm's (the
    implementation's schedule and the host go in sibling keys): BASELINE's config name,
    shapes, pool ratio, query drift, and the L2 statement of the timing rules."""
    L = cfg["context_len"]
    return {"workload": cfg["workload"], "layers": 1, "batch_per_gpu": cfg["batch"],
            "context_len": L if isinstance(L, int) else "mixed {}-{} log-uniform".format(*L),
            "sparse_ratio": cfg["sparse_ratio"],
            "topk": TOPK, "query_drift": args.drift,
            "l2": "inputs larger than L2 (indexer keys + slot pool > 600 MB/GPU)"}


def init_ranks(local: int, world: int):
    """One process per GPU (NCCL for the barrier and the max-over-ranks timing).  With
    more ranks than GPUs (a harness check on a 1-GPU box) ranks share devices round-robin
    and the reductions go over gloo on the host.  Returns (device, aggregate device)."""
    import torch
    import torch.distributed as dist
    ndev = max(1, torch.cuda.device_count())
    dev = torch.device("cuda", local % ndev)
    torch.cuda.set_device(dev)
    if world <= 1:
        return dev, dev
    if world <= ndev:
        dist.init_process_group("nccl", device_id=dev)
        return dev, dev
    dist.init_process_group("gloo")
    return dev, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML every 2 ms
    during the timed region (the recipe's nvidia-smi clocks line, at a rate that
    also covers millisecond-scale regions)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown"}

    def __init__(self, device):
        self.device, self.rows, self.stop = device, [], threading.Event()

    def _handle(self, nv):
        import torch
        try:
            p = torch.cuda.get_device_properties(self.device)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.device.index or 0)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)

            def loop():
                while not self.stop.is_set():
                    self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                      nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    time.sleep(0.002)
            self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                              nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: say so in the JSON
            self.err = repr(e)
        return self

    def __exit__(self, *a):
        self.stop.set()
        if hasattr(self, "t"):
            self.t.join(timeout=1)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "error": getattr(self, "err", None)}
        reasons = sorted({name for _, r in self.rows for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows)}


# -------------------------------------------------------------------------------------
# CPU leg: the oracle port on host cores (cpu_baseline and --impl reference)
# -------------------------------------------------------------------------------------
CPU_WARM_WINDOWS = 8  # prefill windows per request in the CPU leg (the GPU layer uses 32)
CPU_WARM_STEPS = 2    # untimed decode steps before the timed one (the GPU bench warms up too)


def _cpu_request(task):
    """One request's decode step on one host core (oracle port), the GPU step's work in
    order: numpy indexer -> top-k -> C LRU access step -> miss gather (the fetched 656-B
    rows copied from the host store into the slot store) -> numpy sparse MLA over the
    slot rows -> admission of the generated token (grow, append, row write-back).  The
    pool is warmed first with prefill windows from the same drifting query process
    (q_t = a q_{t-1} + sqrt(1-a^2) eps, the GPU layer's), untimed.  Returns (timed
    seconds, hits, misses)."""
    L, rho, seed, drift = task
    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import dsa
    from oracle import lru as olru

    import torch

    def e4(a):  # e4m3 bytes, saturating (the GPU layer's _e4m3)
        return torch.from_numpy(np.asarray(a, np.float32)).clamp(-448, 448).to(torch.float8_e4m3fn) \
            .view(torch.uint8).numpy()

    rng = np.random.default_rng(seed)
    Lx = L + CPU_WARM_STEPS + 1                          # history grows by one token per step
    k = e4(rng.standard_normal((Lx, 128)) * 8)          # the GPU layer's key / query scales
    w = rng.standard_normal(64).astype(np.float32) / 8
    ks = (rng.random(Lx).astype(np.float32) * 0.5 + 0.75)
    host = rng.integers(0, 120, size=(Lx + 1, 656), dtype=np.uint8)  # latent rows (+ the new ones)
    host[:, 512:528] = np.full((Lx + 1, 4), 0.03, np.float32).view(np.uint8)
    host[:, 528:] = 0
    slots = np.zeros_like(host)                                       # the slot store
    a, sd = drift, float(np.sqrt(max(0.0, 1.0 - drift * drift)))
    zi = rng.standard_normal((64, 128))
    qa = rng.standard_normal((128, 576)).astype(np.float32)
    pool = olru.OraclePool(olru.pool_capacity(rho, L))
    with threadpool_limits(1):  # one core per request; requests run in parallel processes
        for _ in range(CPU_WARM_WINDOWS):   # prefill -> decode handoff, untimed
            zi = a * zi + sd * rng.standard_normal(zi.shape)
            pool.warmup([dsa.topk_indices(dsa.indexer_logits(e4(zi * 4), w, k, ks, L), L, TOPK).tolist()])
        res = pool.lru_order()
        slots[res] = host[res]

        def step(h):  # one decode step over a history of h tokens; the new token is id h
            nonlocal zi
            zi = a * zi + sd * rng.standard_normal(zi.shape)
            q = e4(zi * 4)
            t0 = time.perf_counter()
            logits = dsa.indexer_logits(q, w, k, ks, h)
            idx = dsa.topk_indices(logits, h, TOPK)
            r = pool.access_step(idx.tolist())
            miss = np.asarray(r.miss_ids, dtype=np.int64)
            slots[miss] = host[miss]                                  # K4: the miss gather
            dsa.sparse_mla(qa, slots[idx], 1.0 / 192 ** 0.5)          # K5 over the slot rows
            pool.grow_capacity(olru.pool_capacity(rho, h + 1))       # admission (cache.py:191-195)
            pool.append_generated([h])
            slots[h] = host[h]
            return time.perf_counter() - t0, len(r.hit_ids), len(r.miss_ids)

        for s_ in range(CPU_WARM_STEPS):  # untimed, like the GPU bench's warm-up steps
            step(L + s_)
        return step(L + CPU_WARM_STEPS)


def _cpu_pool(workers):
    import multiprocessing as mp
    if not hasattr(_cpu_pool, "p"):
        # spawn: the parent holds a CUDA context, which must not be forked
        _cpu_pool.p = mp.get_context("spawn").Pool(workers)
        _cpu_pool.p.map(_cpu_request, [(4096, 0.25, i, 0.97) for i in range(workers)])  # imports, oracle lib
    return _cpu_pool.p


def _cpu_pool_close():
    p = getattr(_cpu_pool, "p", None)
    if p is not None:
        p.close()
        p.join()
        del _cpu_pool.p


def cpu_reference_rate(cfg, budget_s: float = 12.0, seed: int = 0, drift: float = 0.97):
    """The CPU oracle on every host core: rounds of one request per core (one decode step
    each, the config's shapes and query drift, after an untimed warm-up), timed per
    request inside the worker.  Rate = cores / mean timed seconds per request-step (each
    core runs one request at a time).  Returns (tokens/s, sample, cores, hit rate)."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    lens = request_lengths(cfg, max(cfg["batch"], cores), seed=seed + 17)
    pool = _cpu_pool(cores)
    n_req, wall, rnd, times, hits, misses = 0, 0.0, 0, [], 0, 0
    while n_req < 1 or (wall < budget_s and n_req < 4 * max(cfg["batch"], cores)):
        tasks = [(lens[(n_req + i) % len(lens)], cfg["sparse_ratio"], seed + 1000 * rnd + i, drift)
                 for i in range(cores)]
        t0 = time.perf_counter()
        for t, h, m in pool.map(_cpu_request, tasks, chunksize=1):
            times.append(t)
            hits += h
            misses += m
        wall += time.perf_counter() - t0
        n_req += cores
        rnd += 1
    mean_t = sum(times) / len(times)
    hit_rate = hits / max(1, hits + misses)
    sample = (f"{n_req} request-steps of the {cfg['workload']} workload at query drift {drift}, {cores} at a "
              f"time (one per core, spawn processes, single-threaded BLAS), each after an untimed "
              f"{CPU_WARM_WINDOWS}-window prefill warm-up and {CPU_WARM_STEPS} decode steps: numpy indexer + "
              f"top-k + C LRU step + miss gather "
              f"into the slot store + numpy sparse MLA + admission (oracle port); mean {mean_t * 1e3:.1f} ms "
              f"per request-step, hit rate {hit_rate:.3f}, {wall:.2f} s wall")
    return cores / mean_t, sample, cores, hit_rate


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    vals = []
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, budget_s=1.0, drift=args.drift)
    t0 = time.perf_counter()
    sample = threads = hit_rate = None
    for i in range(args.steps):
        v, sample, threads, hit_rate = cpu_reference_rate(cfg, budget_s=3.0, seed=i, drift=args.drift)
        vals.append(v)
    el = time.perf_counter() - t0
    _cpu_pool_close()
    value = statistics.mean(vals)
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": workload_config(cfg, args),
            "schedule": {"overlap": "none (one request per core, sequential K1..K5 + admission)",
                         "prefill_windows": CPU_WARM_WINDOWS, "untimed_decode_steps": CPU_WARM_STEPS},
            "hit_rate": hit_rate,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------------------------
# GPU leg
# -------------------------------------------------------------------------------------
def host_link_peak_gbs(device, nbytes=1 << 28):
    """Bulk pinned H2D cudaMemcpy bandwidth (the K4 roofline denominator)."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=device)
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(5):
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def run_steps(layer, inputs, new_rows, overlap, counts=None):
    """The product decode step: layer.attend (K1..K5, micro-batched overlap) + append."""
    for t, (q_idx, q) in enumerate(inputs):
        layer.attend(q_idx, q, gather_ctas=layer.gather_ctas, overlap=overlap)
        layer.append_token(new_rows=new_rows[t])
        if counts is not None:
            counts.append(layer.step_counts().clone())


def kernel_breakdown(layer, inputs, new_rows):
    """Sequential steps with CUDA events around every kernel of the path (one stream,
    no overlap): per-kernel device time for the roofline and the gather GB/s.  Each
    timed kernel is preceded by a GPU sleep so host launch latency never leaks into
    the events (the GPU is always behind the host)."""
    import torch
    from paper_2512_10576_b200.attention import sparse_mla
    from paper_2512_10576_b200.indexer import indexer_logits, topk
    from paper_2512_10576_b200.transfer import gather
    from paper_2512_10576_b200.cache import AccessBatch
    names = ["indexer", "topk", "cache", "gather", "sparse_mla", "append"]
    ms = {n: 0.0 for n in names}
    counts = []
    acc = layer.acc  # preallocated step buffers (no allocation inside a timed region)
    # link wake-up before each timed gather: 32 rows per pool that no step selects (ids
    # at the end of the store, past every history) into the pool's staging rows — so the
    # timed gather reads its own, cold miss list rather than re-reading warm rows
    wake = None
    if layer.pool.staging_rows >= 32:
        B, d = layer.B, layer.device
        ids = torch.arange(layer.Lmax - 32, layer.Lmax, dtype=torch.int32, device=d).repeat(B, 1)
        rows = torch.arange(layer.pool.cap_max, layer.pool.cap_max + 32, dtype=torch.int32, device=d).repeat(B, 1)
        cnt = torch.zeros((B, 4), dtype=torch.int32, device=d)
        cnt[:, 1] = 32
        wake = AccessBatch(cnt, None, ids.contiguous(), rows.contiguous())

    def timed(name, fn, warm=None):
        torch.cuda._sleep(2_000_000)
        if warm is not None:  # an idempotent untimed launch first (host link out of idle)
            warm()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        timed.ev.append((name, e0, e1))
        return r
    timed.ev = []
    for t, (q_idx, q) in enumerate(inputs):
        timed("indexer", lambda: indexer_logits(q_idx, layer.w, layer.k_cache, layer.k_scale,
                                                layer.lens, out=layer.logits))
        timed("topk", lambda: topk(layer.logits, layer.lens, layer.K, out=layer.idx, count=layer.cnt))
        acc = timed("cache", lambda: layer.pool.access(layer.idx, layer.cnt, out=acc))
        g = lambda: gather(layer.pool, layer.store, acc, max_ctas=BREAKDOWN_GATHER_CTAS)  # noqa: E731
        w = (lambda: gather(layer.pool, layer.store, wake, max_ctas=BREAKDOWN_GATHER_CTAS)) if wake else None
        timed("gather", g, warm=w)
        timed("sparse_mla", lambda: sparse_mla(layer.pool, q, acc.sel_row, layer.cnt, layer.sm_scale,
                                               out=layer.out, lse=layer.lse))
        timed("append", lambda: layer._append_device(new_rows[t]))  # the graph's device-side append
        counts.append(acc.counts.clone())
    torch.cuda.synchronize()
    for name, e0, e1 in timed.ev:
        ms[name] += e0.elapsed_time(e1) / len(inputs)
    return ms, torch.stack(counts), q


def product_layer(cfg, dev, steps, drift=0.97, rank=0, micro=None, first=None, gather_ctas=32,
                  record=False, world=1):
    """The benchmarked product layer of a single-layer config, set up exactly as the timed
    run uses it (the parity tests at the benchmarked shapes build it through here): this
    rank's share of the global request set (dp.shard_requests: round-robin, LPT by length
    for mixed batches), pools at floor(rho * history), the DBA micro-batch split and the
    32-window prefill warm-up.  Returns (layer, lens, windows or None)."""
    from paper_2512_10576_b200.decode import DSADecodeLayer
    from paper_2512_10576_b200.dp import shard_requests
    rho = cfg["sparse_ratio"]
    glob = request_lengths(cfg, cfg["batch"] * world, seed=0)
    mixed = not isinstance(cfg["context_len"], int)
    mine = shard_requests(len(glob), world, rank, glob if mixed else None)
    lens = [glob[i] for i in mine]
    B = len(lens)
    L = lens if not isinstance(cfg["context_len"], int) else cfg["context_len"]
    layer = DSADecodeLayer(B, L, rho, TOPK, max_new_tokens=steps + 16, device=dev,
                           seed=1234 + rank, drift=drift, slot_format=cfg.get("slot_format"))
    layer.gather_ctas = gather_ctas
    layer.micro = cfg["micro"] if micro is None else micro
    layer.first_frac = (cfg["first"] if layer.micro == cfg["micro"] else None) if first is None else first
    windows = layer.prefill_warmup(windows=32, record=record)
    return layer, lens, (windows if record else None)


def host_info(bound_node):
    """CPU model, NUMA layout and the GPU's node (BASELINE.md §3 asks for them beside
    the CPU baseline; SURVEY §8e's one-NUMA-local-host-pool-per-GPU placement)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        nodes = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")])
    except OSError:
        nodes = None
    return {"cpu_model": model, "cpus": os.cpu_count(), "numa_nodes": nodes, "gpu_numa_node": bound_node}


def selection_similarity(layer, inputs, new_rows, steps=4):
    """Eq. (1) step-to-step overlap r (offsim trace.py:164-177, |K_{t-1} & K_t| / |K_t|) of
    the product layer's live K2 selections over a few extra (untimed) steps, averaged over
    requests and step pairs."""
    import numpy as np
    prev, rs = None, []
    for t in range(steps):
        layer.step(inputs[t][0], inputs[t][1], new_rows[t])
        idx, cnt = layer.idx.cpu().numpy(), layer.cnt.cpu().numpy()
        cur = [idx[b, :cnt[b]] for b in range(layer.B)]
        if prev is not None:
            rs += [len(np.intersect1d(p, c, assume_unique=True)) / len(c) for p, c in zip(prev, cur) if len(c)]
        prev = cur
    return float(np.mean(rs))


def flashmla_bar(layer, q, sel_row, counts, k5_ms):
    """The speed bar for K5: FlashMLA's sm100 FP8 sparse decode (DeepSeek's V3.2 DSA kernel,
    vLLM's build) over the same number of requests / selected rows / slot indices, its 656-B
    rows in one HBM cache of the pool's size.  Returns (us, K5 speed-up) or None."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    try:
        import thirdparty as tp
        if not tp.flashmla_available():
            return None
        B, rows = layer.B, layer.pool.rows_per_pool
        cache = torch.randint(0, 120, (B * rows, 656), dtype=torch.uint8, device=layer.device)
        cache[:, 512:528] = torch.full((B * rows, 4), 2.0 ** -5, device=layer.device).view(torch.uint8)
        n = counts.clone()
        kp = (int(n.max()) + 63) // 64 * 64
        idx = (sel_row[:, :kp].clamp(0, rows - 1) + torch.arange(B, device=layer.device).view(B, 1) * rows)
        idx = idx.int().contiguous()
        _, _, meta = tp.flashmla_sparse_decode(q, cache, idx, layer.sm_scale, lengths=n)
        for _ in range(3):
            tp.flashmla_sparse_decode(q, cache, idx, layer.sm_scale, lengths=n, meta=meta)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        e0.record()
        for _ in range(10):
            tp.flashmla_sparse_decode(q, cache, idx, layer.sm_scale, lengths=n, meta=meta)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        del cache
        return {"flashmla_us": us, "k5_us": k5_ms * 1e3, "k5_speedup_vs_flashmla": us / (k5_ms * 1e3)}
    except Exception as e:  # comparator unavailable: say so, never fail the bench
        return {"error": repr(e)[:200]}


def measure(args, cfg, dev, rank, world, agg_dev, drift, full, peaks, peak_kind, link_peak=None):
    """One single-layer workload: the product step (graph replays, device clock) and, when
    ``full``, the per-kernel breakdown (K1 roofline, cold-list gather GB/s, K5 vs FlashMLA),
    the Eq. (1) similarity and the e2e host-buffer run.  Returns (record, layer-free)."""
    import torch
    import torch.distributed as dist
    from paper_2512_10576_b200.decode import random_latent_rows
    from paper_2512_10576_b200.dp import aggregate

    W, K, NB = args.warmup, args.steps, args.breakdown_steps
    total = W + K + NB + 4
    # token budget per request: the graph warm-ups, timed steps, breakdown, similarity
    # probe and the e2e pipeline (its capture and K steps) each append one token per step
    layer, lens, _ = product_layer(cfg, dev, 2 * total + 2 * K + 32, drift=drift, rank=rank, micro=args.micro,
                                   first=args.first, gather_ctas=args.gather_ctas, world=world)
    B = layer.B
    inputs = [layer.next_queries() for _ in range(total)]
    new_rows = [random_latent_rows(B, dev, layer.gen).view(B, 1, 656) for _ in range(total)]
    torch.cuda.synchronize()
    # warm-up (untimed): capture the whole step as one CUDA graph (its first, eager
    # execution is a real step), then W-1 graph replays
    layer.capture(args.overlap, args.gather_ctas)
    for t in range(1, W):
        layer.step(inputs[t][0], inputs[t][1], new_rows[t])
    torch.cuda.synchronize()
    hits0, misses0 = layer.access_totals()
    if world > 1:
        dist.barrier()
    # timed region: K product steps (graph replays incl. input copies), device clock
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        start.record()
        for t in range(W, W + K):
            layer.step(inputs[t][0], inputs[t][1], new_rows[t])
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = start.elapsed_time(end) / K
    layer.pool.check("bench")
    tokens_total, t_max = aggregate(B * K, step_ms * K / 1e3, device=agg_dev)
    hits, misses = (x - y for x, y in zip(layer.access_totals(), (hits0, misses0)))
    rec = {"value": tokens_total / t_max, "unit": "tokens/s", "ms_per_step": t_max * 1e3 / K,
           "batch_per_gpu": B, "query_drift": drift, "hit_rate": hits / max(1, hits + misses),
           "slot_row_bytes": layer.pool.row_bytes,
           "slot_store_gb": layer.pool.num_pools * layer.pool.rows_per_pool * layer.pool.row_bytes / 1e9,
           "misses_per_request_step": misses / (B * K), "clocks": clocks.summary(),
           "gpu_launches": layer.launches_per_step(args.overlap) * K,
           "micro_batches": layer.micro_batches(layer.micro) if args.overlap in ("dba", "dbs") else [(0, B)],
           "context_len": cfg["context_len"] if isinstance(cfg["context_len"], int)
           else "mixed {}-{} log-uniform, mean {:.0f}".format(*cfg["context_len"], sum(lens) / B)}
    # Eq. (1) selection similarity r over 4 more (untimed) steps
    rec["similarity_r"] = selection_similarity(layer, inputs[W + K:W + K + 4], new_rows[W + K:W + K + 4])
    if args.quick or not full:
        layer.close()
        return rec
    # per-kernel breakdown (sequential, separate steps) for the roofline
    ktimes, bcounts, bq = kernel_breakdown(layer, inputs[W + K + 4:W + K + 4 + NB],
                                           new_rows[W + K + 4:W + K + 4 + NB])
    lens_mean = sum(lens) / B + W + K + 4 + (NB - 1) / 2
    idx_bytes = B * lens_mean * (132 + 4) + B * (64 * 128 + 64 * 4)
    achieved = idx_bytes / (ktimes["indexer"] * 1e-3) / 1e9
    gather_bytes = bcounts[:, :, 1].sum().item() * 656 / NB
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{cfg['name']}.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get("indexer_dram_bytes_per_launch")
    gather_gbs = gather_bytes / (ktimes["gather"] * 1e-3) / 1e9 if ktimes["gather"] else None
    rec["kernels_ms"] = ktimes
    rec["roofline"] = {"bound": "hbm", "kernel": "indexer (K1)", "achieved": achieved,
                       "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                       "traffic": traffic, "peak_kind": peak_kind,
                       "algorithmic_bytes_per_launch": idx_bytes}
    k5_flop = 2 * 128 * (576 + 512) * bcounts[:, :, :2].sum().item() / NB
    rec["k5"] = {"tflops": k5_flop / (ktimes["sparse_mla"] * 1e-3) / 1e12,
                 "frac_of_bf16_peak": k5_flop / (ktimes["sparse_mla"] * 1e-3) / 1e12 / peaks["bf16_tflops"],
                 "bar": flashmla_bar(layer, bq, layer.acc.sel_row, layer.cnt, ktimes["sparse_mla"])}
    # useful bytes = 656 per miss; on the link each 64-B-aligned row (704-B host pitch)
    # moves as 11 64-B read completions = 704 B.  Timed on the step's own (cold) miss list.
    rec["gather"] = {"bytes_per_step": gather_bytes, "gbs": gather_gbs,
                     "host_link_peak_gbs": link_peak,
                     "host_link_peak_kind": "pinned cudaMemcpy H2D, 256 MB, best of 5, this box "
                                            "(45-55 GB/s on most boxes; on a slow-DMA box the SM "
                                            "gather can exceed it)",
                     "frac_of_link_peak": gather_gbs / link_peak if gather_gbs and link_peak else None,
                     "link_bytes_per_row": LINK_ROW_BYTES,
                     "link_gbs": gather_gbs * LINK_ROW_BYTES / 656 if gather_gbs else None,
                     "link_frac_of_link_peak": (gather_gbs * LINK_ROW_BYTES / 656 / link_peak
                                                if gather_gbs and link_peak else None),
                     "miss_list": "cold: the breakdown step's own misses, after a gather of other rows",
                     "ctas": BREAKDOWN_GATHER_CTAS,
                     "paper_flashtrans_gbs": 37.0}
    # e2e: through the public API with host buffers: every step copies its queries H2D
    # from pinned memory and its attention output D2H (layer.step_host: copy stream,
    # double-buffered staging, so transfers of step t overlap compute of t-1 / t+1)
    if args.e2e:
        # link-serial pipeline (per-slot graphs: the query upload and the miss gather
        # take turns on the host link) for the DA / DBA schedules
        serial = args.overlap in ("da", "dba") and os.environ.get("ESS_E2E_SERIAL", "1") == "1"
        if serial:
            layer.capture_host(args.overlap, args.gather_ctas)
        h_in = [(qi.cpu().pin_memory(), q.cpu().pin_memory()) for qi, q in inputs[W:W + K]]
        h_out = [torch.empty(layer.out.shape, dtype=layer.out.dtype).pin_memory() for _ in range(K)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(K):
            layer.step_host(h_in[t][0], h_in[t][1], new_rows[W + t], h_out[t])
        layer._ds.synchronize()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / K
        e2e_tok, e2e_t = aggregate(B * K, e2e_ms * K / 1e3, device=agg_dev)
        h2d = h_in[0][0].numel() + h_in[0][1].numel() * 2
        rec["e2e"] = {"value": e2e_tok / e2e_t, "unit": "tokens/s",
                      "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": h_out[0].numel() * 2,
                      "pipeline": "link-serial" if serial else "overlapped"}
        # the H2D link carries the queries (DMA) and the misses (SM reads, 704 B each):
        # its achieved rate vs the measured pinned-DMA peak, and the e2e bound it sets
        if link_peak:
            link_bytes = h2d + rec["misses_per_request_step"] * B * LINK_ROW_BYTES
            rec["e2e"]["h2d_link_gbs"] = link_bytes / (e2e_ms * 1e-3) / 1e9
            rec["e2e"]["h2d_link_frac_of_peak"] = rec["e2e"]["h2d_link_gbs"] / link_peak
            rec["e2e"]["link_bound_tokens_per_s"] = B / (link_bytes / (link_peak * 1e9))
    layer.close()
    return rec


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev, agg_dev = init_ranks(local, world)
    # launch loop and pinned staging on the GPU's NUMA node (ESS_BIND_NUMA=0: off);
    # the CPU baseline below gets the full affinity back
    from paper_2512_10576_b200.transfer import bind_to_gpu_node
    prev_aff, bound_node = bind_to_gpu_node(dev) if os.environ.get("ESS_BIND_NUMA", "1") == "1" else (None, None)
    peaks, peak_kind = measured_peaks()
    link_peak = host_link_peak_gbs(dev)
    main = measure(args, cfg, dev, rank, world, agg_dev, args.drift, True, peaks, peak_kind, link_peak)
    if args.quick:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": main["value"], "unit": "tokens/s", "n_gpus": world,
                              "ms_per_step": main["ms_per_step"], "quick": True,
                              "micro_batches": args.micro, "first": args.first,
                              "hit_rate": main["hit_rate"], "similarity_r": main["similarity_r"]}), flush=True)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    ceiling = run_ceiling(args, cfg, dev) if (args.ceiling and world == 1) else None
    subs = {}
    if args.sub and world == 1:
        # the metric's other half (128K, BASELINE configs[3]) and a lower-locality row
        c4 = dict(CONFIGS["c4"])
        a4 = argparse.Namespace(**{**vars(args), "micro": c4["micro"], "first": c4["first"], "e2e": False})
        subs["c4"] = measure(a4, c4, dev, rank, world, agg_dev, args.drift, True, peaks, peak_kind, link_peak)
        if args.ceiling:
            subs["c4"]["all_hbm_ceiling"] = run_ceiling(a4, c4, dev)
            subs["c4"]["all_hbm_ceiling"]["frac_of_ceiling"] = (
                subs["c4"]["value"] / subs["c4"]["all_hbm_ceiling"]["value"])
        # the same workload with the 656-B FP8 slot format (K5 = the CTA-pair kernel that
        # dequantises on chip): a 25% pool then costs 25% of the latent bytes
        f8 = {**cfg, "slot_format": "fp8"}
        a8 = argparse.Namespace(**{**vars(args), "e2e": False})
        subs[f"{cfg['name']}_fp8_slots"] = measure(a8, f8, dev, rank, world, agg_dev, args.drift, True, peaks,
                                                   peak_kind, link_peak)
        if cfg["name"] == "c2" and args.mtp:
            # MTP = 2, accept 1.7 (the paper's Table 2 32K setting) on the same shapes,
            # beside its all-HBM ceiling (rho = 1, nothing to gather)
            m = measure_mtp(args, cfg, dev, mtp=2, mean_accept=1.7)
            m["all_hbm_ceiling"] = mtp_ceiling(args, cfg, dev, m)
            subs["c2_mtp2"] = m
        lo = argparse.Namespace(**{**vars(args), "e2e": False})
        subs[f"{cfg['name']}_drift_0.9"] = measure(lo, cfg, dev, rank, world, agg_dev, 0.9, False, peaks,
                                                   peak_kind, link_peak)
        if ceiling:
            r = subs[f"{cfg['name']}_drift_0.9"]
            r["frac_of_ceiling"] = r["value"] / ceiling["value"]
    if prev_aff is not None:
        os.sched_setaffinity(0, prev_aff)
    line = None
    if rank == 0:
        cpu_v, cpu_sample, cpu_threads, _ = cpu_reference_rate(cfg, budget_s=12.0, drift=args.drift)
        _cpu_pool_close()
        line = {
            "metric": METRIC, "value": main["value"], "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "e4m3/f16/f32",
            "data": "synthetic (random-weight DeepSeek-V3.2-Exp DSA shapes, drifting queries)",
            "config": workload_config(cfg, args),
            "schedule": {"overlap": args.overlap, "micro_batches": main["micro_batches"],
                         "context_len": main["context_len"],
                         "slot_row_bytes": main["slot_row_bytes"], "slot_store_gb": main["slot_store_gb"],
                         "parallelism": f"dp{world} (requests sharded by dp.shard_requests, no collective)"},
            "host": host_info(bound_node),
            "e2e": main.get("e2e"),
            "roofline": main["roofline"],
            "cpu_baseline": {"value": cpu_v, "unit": "tokens/s", "cores": cpu_threads, "kind": "port",
                             "sample": cpu_sample},
            # this library's kernels per step (graph kernel nodes; DSADecodeLayer.launches_per_step)
            "gpu_launches": main["gpu_launches"],
            "cuda_graph": True,
            "clocks": main["clocks"],
            "kernels_ms": main["kernels_ms"],
            "k5": main["k5"],
            "gather": main["gather"],
            "hit_rate": main["hit_rate"],
            "misses_per_request_step": main["misses_per_request_step"],
            "similarity_r": main["similarity_r"],
        }
        if ceiling:
            line["all_hbm_ceiling"] = ceiling
            line["all_hbm_ceiling"]["frac_of_ceiling"] = main["value"] / ceiling["value"]
        if subs:
            line["sub"] = subs
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_model(args, cfg):
    """Multi-layer configs (C3): the whole num_layers-layer step as one CUDA graph,
    device-timed like run_ours; per-layer breakdown, e2e and the CPU leg are the
    single-layer configs' (C2 is the same layer shape at 4x the batch)."""
    import torch
    import torch.distributed as dist
    from paper_2512_10576_b200.decode import DSADecodeModel, random_latent_rows
    from paper_2512_10576_b200.dp import aggregate

    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev, agg_dev = init_ranks(local, world)
    B, L, rho, NL = cfg["batch"], cfg["context_len"], cfg["sparse_ratio"], cfg["layers"]
    W, K = args.warmup, args.steps
    t_setup = time.perf_counter()
    drift = args.drift
    if args.layer_drift:  # per-layer query drift, linearly spaced (layers differ in misses)
        lo, hi = (float(x) for x in args.layer_drift.split(","))
        drift = [lo + (hi - lo) * i / max(1, NL - 1) for i in range(NL)]
    # uniform-schedule steps before the timed ones: they feed the plan's miss means (and
    # with --pre-steps put uniform runs at the same decode position as planned ones)
    plan_w = max(W if args.plan_theta is not None else 0, args.pre_steps)
    model = DSADecodeModel(NL, B, L, rho, TOPK, max_new_tokens=W + K + plan_w + 8, device=dev,
                           seed=1234 + 100003 * rank, drift=drift)
    model.set_schedule(args.micro, args.first)
    model.prefill_warmup(windows=32)
    rows = random_latent_rows(B, dev).view(B, 1, 656)
    model.capture(args.overlap, args.gather_ctas)
    queries = [model.next_queries() for _ in range(W + K + plan_w)]
    plan = layer_means = None
    if plan_w:
        # the layer-wise plan (pipeline.py:190-195) from the pools' live miss means over
        # W uniform-schedule steps, then the step re-captured with each layer's strategy
        from paper_2512_10576_b200.plan import MissMeter
        meter = MissMeter(model)
        for t in range(plan_w):
            model.step(queries[W + K + t], rows)
        torch.cuda.synchronize()
        layer_means = meter.means().tolist()
        if args.plan_theta is not None:
            plan = model.plan_layers(args.plan_theta, meter)
            model.capture(plan=plan, gather_ctas=args.gather_ctas)
    for t in range(1, W):
        model.step(queries[t], rows)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    h0, m0 = model.access_totals()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        start.record()
        for t in range(W, W + K):
            model.step(queries[t], rows)
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = start.elapsed_time(end) / K
    model.check("bench")
    h, m = (x - y for x, y in zip(model.access_totals(), (h0, m0)))
    tokens_total, t_max = aggregate(B * K, step_ms * K / 1e3, device=agg_dev)
    launches = model.launches_per_step() * K
    model.close()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": tokens_total / t_max, "unit": "tokens/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": t_max * 1e3 / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "e4m3/f16/f32",
            "data": "synthetic (random-weight DeepSeek-V3.2-Exp DSA shapes, drifting queries)",
            "config": {"workload": cfg["workload"], "layers": NL, "batch_per_gpu": B,
                       "context_len": L, "sparse_ratio": rho, "topk": TOPK,
                       "query_drift": args.drift, "overlap": args.overlap,
                       "micro_batches": args.micro, "first_micro_batch_share": args.first,
                       "parallelism": f"dp{world} (requests sharded, no collective)",
                       "l2": "inputs larger than L2"},
            "us_per_layer": step_ms * 1e3 / NL, "hit_rate": h / max(1, h + m),
            "misses_per_request_layer_step": m / (B * K * NL),
            "gpu_launches": launches,
            "cuda_graph": True, "clocks": clocks.summary(), "setup_s": setup_s,
            "e2e": None, "note": "secondary config: per-kernel roofline, e2e and CPU leg on c2/c4",
            "layer_drift": args.layer_drift,
            "pre_steps": plan_w, "layer_miss_means": layer_means,
            "plan": None if plan is None else {
                "theta": plan.threshold, "counts": plan.counts(), "strategies": plan.strategies}}),
            flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def mtp_ceiling(args, cfg, dev, m):
    """The MTP step's all-HBM ceiling: every schedule at rho = 1, the fastest (strict)."""
    runs = {s: measure_mtp(args, cfg, dev, mtp=m["mtp"], mean_accept=1.7, rho=1.0, overlap=s)
            for s in ("none", "da", "dba")}
    best = min(runs, key=lambda s: runs[s]["ms_per_step"])
    mc = runs[best]
    return {"value": mc["value"], "ms_per_step": mc["ms_per_step"], "hit_rate": mc["hit_rate"],
            "schedule": best, "schedules_us": {s: round(r["ms_per_step"] * 1e3, 1) for s, r in runs.items()},
            "frac_of_ceiling": m["value"] / mc["value"]}


def measure_mtp(args, cfg, dev, mtp=2, mean_accept=1.7, rho=None, overlap="dba", seed=4321):
    """The MTP decode step (MTPDecodeLayer: mtp + 1 query tokens per request; the paper's
    Table 2 setting MTP = 2, accept 1.7 at 32K): graph replays with
    per-request accepted counts drawn as Poisson(mean - 1) + 1 capped at mtp + 1
    (trace.py:127), device clock.  ``value`` counts accepted tokens (the reference's
    OTPS x batch, costmodel.py:232-234); ``verified`` counts all query tokens."""
    import numpy as np
    import torch
    from paper_2512_10576_b200.decode import random_latent_rows
    from paper_2512_10576_b200.attention import sparse_mla
    from paper_2512_10576_b200.indexer import indexer_logits_mtp, topk_mtp
    from paper_2512_10576_b200.mtp import MTPDecodeLayer, draw_accepted
    B, ctx = cfg["batch"], cfg["context_len"]
    rho = cfg["sparse_ratio"] if rho is None else rho
    W, K = args.warmup, args.steps
    Q = mtp + 1
    layer = MTPDecodeLayer(B, ctx, rho, TOPK, mtp=mtp, max_new_tokens=W + K + 8, device=dev, seed=seed,
                           drift=args.drift)
    layer.micro, layer.first_frac = cfg["micro"], cfg["first"]
    if rho >= 1.0:
        layer.preload_full_history()
    else:
        layer.prefill_warmup(windows=32)
    rng = np.random.default_rng(seed)
    total = W + K
    acc_h = [draw_accepted(rng, B, mean_accept, Q) for _ in range(total)]
    # each step starts where the previous one's accepted tokens end (query = f(position))
    inputs = [layer.next_queries(None if t == 0 else acc_h[t - 1]) for t in range(total)]
    rows = [random_latent_rows(B * Q, dev, layer.gen).view(B, Q, 656) for _ in range(total)]
    acc_d = [torch.from_numpy(a).to(dev) for a in acc_h]
    layer.capture(overlap, args.gather_ctas, accepted=acc_h[0])
    for t in range(1, W):
        layer.step(inputs[t][0], inputs[t][1], rows[t], acc_d[t], max_accepted=int(acc_h[t].max()))
    torch.cuda.synchronize()
    hits0, misses0 = layer.access_totals()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        e0.record()
        for t in range(W, total):
            layer.step(inputs[t][0], inputs[t][1], rows[t], acc_d[t], max_accepted=int(acc_h[t].max()))
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    layer.pool.check("bench mtp")
    hits, misses = (x - y for x, y in zip(layer.access_totals(), (hits0, misses0)))
    accepted = float(sum(int(a.sum()) for a in acc_h[W:total]))
    rec = {"value": accepted / (ms * 1e-3 * K), "unit": "accepted tokens/s", "ms_per_step": ms,
           "verified_tokens_per_s": B * Q / (ms * 1e-3), "mtp": mtp, "mean_accept_drawn": accepted / (B * K),
           "batch_per_gpu": B, "context_len": ctx, "sparse_ratio": rho,
           "hit_rate": hits / max(1, hits + misses), "misses_per_request_step": misses / (B * K),
           "gpu_launches": layer.launches_per_step(overlap) * K, "schedule": overlap,
           "clocks": clocks.summary()}
    # the idempotent kernels alone on the last step's buffers (K1: the MTP indexer reads
    # each request's keys once; K2: B * qtok rows; K5: B * qtok query rows)
    L = int(layer.lens.float().mean())

    def alone(fn, n=5):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in ev:
            torch.cuda._sleep(1_000_000)
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in ev)
    k1_ms = alone(lambda: indexer_logits_mtp(inputs[0][0], layer.w, layer.k_cache, layer.k_scale, layer.lens,
                                             out=layer.logits))
    rec["kernels_ms"] = {
        "indexer": k1_ms,
        "topk": alone(lambda: topk_mtp(layer.logits, layer.lens, TOPK, out=layer.idx, count=layer.cnt)),
        "sparse_mla": alone(lambda: sparse_mla(layer.pool, layer.q_in.view(B * Q, 128, 576),
                                               layer.sel_row.view(B * Q, TOPK), layer.cnt.view(B * Q),
                                               layer.sm_scale, out=layer.out.view(B * Q, 128, 512),
                                               lse=layer.lse.view(B * Q, 128), qtok=Q))}
    k1_bytes = B * L * (132 + 4 * Q) + B * Q * (64 * 128 + 64 * 4)
    rec["indexer"] = {"ms": k1_ms, "algorithmic_bytes": k1_bytes, "gbs": k1_bytes / (k1_ms * 1e-3) / 1e9,
                      "tflops": 2 * 64 * 128 * Q * B * L / (k1_ms * 1e-3) / 1e12}
    layer.close()
    return rec


def run_ceiling(args, cfg, dev):
    """Same kernels with the whole latent cache in HBM (rho = 1, full history preloaded):
    every selection hits and the gather moves nothing (SURVEY §8d ceiling).  Every
    schedule is timed and the fastest is the ceiling (the strict one); all timings are
    reported in ``schedules_us``."""
    import torch
    from paper_2512_10576_b200.decode import DSADecodeLayer, random_latent_rows
    B = cfg["batch"]
    lens = request_lengths(cfg, B, seed=int(os.environ.get("RANK", "0")))
    L = lens if not isinstance(cfg["context_len"], int) else cfg["context_len"]
    total = args.warmup + args.steps
    # up to five schedules, each a capture step + (warmup - 1) + steps appended tokens
    layer = DSADecodeLayer(B, L, 1.0, TOPK, max_new_tokens=6 * total + 16, device=dev, seed=99,
                           drift=args.drift)
    layer.gather_ctas = args.gather_ctas
    layer.preload_full_history()
    inputs = [layer.next_queries() for _ in range(total)]
    new_rows = [random_latent_rows(B, dev, layer.gen).view(B, 1, 656) for _ in range(total)]
    # all-HBM: nothing to gather, but the overlapped schedules still overlap attention
    # with the top-k / cache manager of other requests, so every schedule is a candidate
    # and the ceiling is the fastest (strict): sequential, DA, DBA (the config's split)
    # and, when their preconditions hold, the streamed ones (dbs, stream)
    schedules = ["none", "da", "dba"] + (["dbs", "stream"] if layer.stream_ok() else [])
    best, measured = None, {}
    layer.micro = cfg["micro"]
    layer.first_frac = cfg["first"]
    for sched in schedules:
        layer.capture(sched, args.gather_ctas)
        for t in range(1, args.warmup):
            layer.step(inputs[t][0], inputs[t][1], new_rows[t])
        torch.cuda.synchronize()
        hits0, misses0 = layer.access_totals()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(args.warmup, total):
            layer.step(inputs[t][0], inputs[t][1], new_rows[t])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        c = [x - y for x, y in zip(layer.access_totals(), (hits0, misses0))]
        measured[sched] = round(ms * 1e3, 1)
        if best is None or ms < best["ms_per_step"]:
            best = {"value": B / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms,
                    "hit_rate": c[0] / max(1, c[0] + c[1]), "schedule": sched}
    best["schedules_us"] = measured
    layer.pool.check("ceiling")
    layer.close()
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--drift", type=float, default=0.97)
    ap.add_argument("--gather-ctas", type=int, default=32)
    ap.add_argument("--overlap", default="dba", choices=["dba", "dbs", "da", "none", "stream"])
    ap.add_argument("--micro", type=int, default=None, help="DBA micro-batches per step (default: per config)")
    ap.add_argument("--first", type=float, default=None,
                    help="DBA: fraction of the batch in the first micro-batch (default: per config)")
    ap.add_argument("--rho", type=float, default=None, help="override the config's GPU slot-pool ratio")
    ap.add_argument("--quick", action="store_true",
                    help="schedule sweeps: skip the CPU baseline, e2e and per-kernel breakdown")
    ap.add_argument("--breakdown-steps", type=int, default=5)
    ap.add_argument("--no-ceiling", dest="ceiling", action="store_false")
    ap.add_argument("--no-sub", dest="sub", action="store_false",
                    help="skip the sub-records (C4 at 128K + its ceiling, drift 0.9); N=1 only")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-mtp", dest="mtp", action="store_false", help="skip the MTP = 2 sub-record")
    ap.add_argument("--mtp-only", action="store_true", help="print only the MTP sub-record (C2 shapes)")
    ap.add_argument("--plan-theta", type=float, default=None,
                    help="multi-layer configs: layer-wise DA/DBA plan at this miss threshold")
    ap.add_argument("--pre-steps", type=int, default=0,
                    help="multi-layer configs: untimed uniform-schedule steps before the timed ones")
    ap.add_argument("--layer-drift", default=None,
                    help="multi-layer configs: 'lo,hi' per-layer query drift, linearly spaced")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    cfg = dict(CONFIGS[args.config])
    if args.rho is not None:
        cfg["sparse_ratio"] = args.rho
    if args.micro is None:
        args.micro = cfg["micro"]
    if args.first is None:
        args.first = cfg["first"] if args.micro == cfg["micro"] else None
    if args.mtp_only:
        import torch
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        m = measure_mtp(args, cfg, dev, mtp=2, mean_accept=1.7)
        m["all_hbm_ceiling"] = mtp_ceiling(args, cfg, dev, m)
        print(json.dumps(m), flush=True)
    elif args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.get("layers", 1) > 1:
        run_model(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
