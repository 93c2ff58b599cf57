"""One offloaded DSA decode layer on one GPU: K1 -> K2 -> K3 -> K4 -> K5.

This is the paper's per-layer decode step that the
reference only composes from cost scalars (``layer_cost_inputs``,
/root/reference/pkg/src/offsim/pipeline.py:207-224):

    indexer_logits -> indexer_topk -> cache manager -> H2D miss gather -> sparse_mla

The indexer key cache stays in HBM; the latent cache lives in a pinned host
store with a GPU slot pool of ``floor(rho * history)`` rows per request in front
of it (cache.py:137-138).  After the layer, each request appends its generated
token: the pool admits it at top recency (cache.py:122-134), its latent row is
written to the slot and back to host (D2H) and its indexer key
joins the HBM cache.

``synthetic_layer`` builds random-weight inputs of DeepSeek-V3.2-Exp shapes:
indexer q/k e4m3 (64 heads x 128), latent rows 512 e4m3 + 4 f32 scales + 64 bf16,
attention q bf16 (128 heads x 576).  Queries drift between steps,
q_t = a q_{t-1} + sqrt(1-a^2) eps, which sets the step-to-step selection overlap
(Eq. (1), trace.py:164-177); the achieved overlap is measured, not assumed.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .attention import DEFAULT_SM_SCALE, SplitWorkspace, sparse_mla, sparse_mla_da
from .cache import AccessBatch, PoolSet, pool_capacity
from .indexer import indexer_logits, indexer_logits_stream, topk, topk_split, topk_split_stream
from .transfer import HostLatentStore, gather, gather_stream, write_generated

ROW = 656


def _e4m3(x: torch.Tensor) -> torch.Tensor:
    return x.clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8)


def random_latent_rows(n: int, device, gen=None) -> torch.Tensor:
    """[n, 656] latent rows in DeepSeek-V3.2's FP8 KV-cache format: e4m3 NoPE (values
    ~N(0,1)*32 quantised), one power-of-two scale per 128-element group (2^-6..2^-4,
    the UE8M0-style scales FlashMLA's FP8 sparse decode expects — it matches the oracle
    only for those, profiles/r02_thirdparty_probe.json), bf16 RoPE ~N(0,1)."""
    nope = _e4m3(torch.randn((n, 512), device=device, generator=gen) * 32.0)
    scales = torch.exp2(torch.randint(-6, -3, (n, 4), device=device, generator=gen).float())
    rope = torch.randn((n, 64), device=device, generator=gen).to(torch.bfloat16)
    return torch.cat([nope, scales.view(torch.uint8), rope.view(torch.uint8)], dim=1)


@dataclass
class StepStats:
    nhit: int = 0
    nmiss: int = 0
    steps: int = 0
    overlap: list = field(default_factory=list)


class DSADecodeLayer:
    """Device-resident state + buffers for one layer over ``batch`` requests."""

    def __init__(self, batch: int, context_len, sparse_ratio: float, topk_k: int = 2048,
                 max_new_tokens: int = 64, device=None, seed: int = 0, drift: float = 0.95,
                 sm_scale: float = DEFAULT_SM_SCALE, hugepages: bool = True, slot_format: str | None = None):
        """``context_len``: one length for every request, or a sequence of ``batch``
        per-request lengths (mixed batches, C5); each request's pool holds
        floor(rho * its own history) rows (cache.py:137-138).  ``slot_format``: the GPU
        slot store's row format, "f16" (1152 B, dequantised on admission) or "fp8" (the
        656-B latent row, dequantised by K5 on chip); default ESS_SLOT_FORMAT / f16."""
        _lib.require_cuda()
        self.device = torch.device(device if device is not None else "cuda")
        if isinstance(context_len, (list, tuple, np.ndarray)):
            self.ctx_lens = [int(x) for x in context_len]
            if len(self.ctx_lens) != batch or min(self.ctx_lens) < 1:
                raise ValueError("need one positive context length per request")
        else:
            self.ctx_lens = [int(context_len)] * batch
        context_len = max(self.ctx_lens)
        self.B, self.ctx, self.rho, self.K = batch, context_len, sparse_ratio, topk_k
        self.drift, self.sm_scale = drift, sm_scale
        self.fuse_da = True  # DA as one K5 launch waiting on the gather (when it fits)
        self.micro = 2       # DBA micro-batches per step (overlap="dba")
        self.max_split = 4   # fused K5: KV splits per request at small batch
        self.min_gather_sms = 20
        self.early_gather_sms = int(os.environ.get("ESS_EARLY_GATHER_SMS", "20"))
        self.late_k1_ctas = int(os.environ.get("ESS_LATE_K1_CTAS", "0"))
        # DBA gathers on SMs shared with the indexer / attention CTAs (no exclusive-SM
        # shared-memory reservation) and their CTA counts (0 = the exclusive defaults)
        self.gather_shared = os.environ.get("ESS_GATHER_SHARED", "1") == "1"
        self.shared_early_gather_ctas = int(os.environ.get("ESS_SHARED_EARLY_GATHER_CTAS", "48"))
        self.shared_late_gather_ctas = int(os.environ.get("ESS_SHARED_LATE_GATHER_CTAS", "0"))
        # DA / DBA: the first micro-batch's K1 -> K2 + K3a (-> K4) as programmatic
        # dependent launches on one stream
        self.pdl = os.environ.get("ESS_PDL", "0") == "1"
        self.pdl_gather = int(os.environ.get("ESS_PDL_K1", "0"))  # 1: the next K1 without PDL
        # streamed schedule (overlap="stream"): request group of the indexer, persistent
        # top-k and gather grid sizes
        self.stream_group = int(os.environ.get("ESS_STREAM_GROUP", "8"))
        self.stream_first = int(os.environ.get("ESS_STREAM_FIRST", "0"))  # first group (0: = group)
        self.stream_topk_ctas = int(os.environ.get("ESS_STREAM_TOPK_CTAS", "16"))
        self.stream_gather_ctas = int(os.environ.get("ESS_STREAM_GATHER_CTAS", "20"))
        self.Lmax = ((context_len + max_new_tokens + 127) // 128) * 128
        self.gen = torch.Generator(device=self.device).manual_seed(seed)
        d, g, B = self.device, self.gen, batch
        self.lens = torch.tensor(self.ctx_lens, dtype=torch.int32, device=d)
        self.history = context_len  # the longest request's history (= ctx + steps)
        # indexer key cache (HBM): e4m3 keys + f32 per-token scale
        self.k_cache = _e4m3(torch.randn((B, self.Lmax, 128), device=d, generator=g) * 8.0)
        self.k_scale = torch.rand((B, self.Lmax), device=d, generator=g) * 0.5 + 0.75
        # host latent store (pinned, mapped) + GPU slot pool
        self.store = HostLatentStore(B, self.Lmax, hugepages=hugepages, device=self.device)
        for b in range(B):  # fill through the GPU: random rows copied into pinned memory
            self.store.host[b].copy_(random_latent_rows(self.Lmax, d, g), non_blocking=False)
        caps = [pool_capacity(sparse_ratio, n) for n in self.ctx_lens]
        self.cap0 = min(caps)
        self.cap_max = pool_capacity(sparse_ratio, self.Lmax)
        # early gather (DA/DBA): misses land in per-pool staging rows while the cache
        # manager still selects victims; needs every pool to hold a whole selection
        self.early_gather = self.cap0 >= topk_k and os.environ.get("ESS_EARLY_GATHER", "1") == "1"
        staging = topk_k if (self.cap0 < topk_k or self.early_gather) else 0
        if slot_format is not None and slot_format not in _lib.SLOT_FORMATS:
            raise ValueError(f"slot_format must be one of {sorted(_lib.SLOT_FORMATS)}")
        row_bytes = _lib.SLOT_FORMATS[slot_format] if slot_format else _lib.SLOT_ROW_BYTES
        self.pool = PoolSet(B, self.Lmax, self.cap_max, caps, row_bytes=row_bytes,
                            staging_rows=staging, device=d)
        # drifting queries
        self._zi = torch.randn((B, 64, 128), device=d, generator=g)
        self._za = torch.randn((B, 128, 576), device=d, generator=g)
        self.w = (torch.randn((B, 64), device=d, generator=g) / 8.0).contiguous()
        # step buffers
        self.logits = torch.empty((B, self.Lmax), dtype=torch.float32, device=d)
        self.idx = torch.empty((B, topk_k), dtype=torch.int32, device=d)
        self.cnt = torch.empty(B, dtype=torch.int32, device=d)
        self.acc = None
        self.out = torch.empty((B, 128, 512), dtype=torch.bfloat16, device=d)
        self.lse = torch.empty((B, 128), dtype=torch.float32, device=d)
        self.stats = StepStats()

    # -- synthetic model inputs ----------------------------------------------------------
    def next_queries(self):
        a = self.drift
        s = math.sqrt(max(0.0, 1.0 - a * a))
        self._zi = a * self._zi + s * torch.randn(self._zi.shape, device=self.device, generator=self.gen)
        self._za = a * self._za + s * torch.randn(self._za.shape, device=self.device, generator=self.gen)
        q_idx = _e4m3(self._zi * 4.0)
        q = (self._za * 0.5).to(torch.bfloat16)
        return q_idx, q

    def prefill_warmup(self, windows: int = 32, record: bool = False):
        """LRU warm-up from the last ``windows`` prefill selections (PAPER.md:285,
        cache.py:73-88), then fill the resident slots from the host store — the
        prefill->decode handoff, outside decode timing."""
        rec = []
        for _ in range(windows):
            q_idx, _q = self.next_queries()
            indexer_logits(q_idx, self.w, self.k_cache, self.k_scale, self.lens, out=self.logits)
            topk(self.logits, self.lens, self.K, out=self.idx, count=self.cnt)
            self.pool.warmup(self.idx, self.cnt)
            if record:
                rec.append([self.idx[b, :int(self.cnt[b])].cpu().numpy() for b in range(self.B)])
        self._fill_resident()
        return rec

    def _fill_resident(self) -> None:
        """The prefill->decode handoff's data movement: every resident id's slot row is
        filled from the host store (after the warm-up decided the residents)."""
        order, n = self.pool.lru_order()
        order = order[:, :self.cap_max].contiguous()
        slots = torch.stack([self.pool.lookup(b, order[b].clamp_min(0)) for b in range(self.B)])
        counts = torch.zeros((self.B, 4), dtype=torch.int32, device=self.device)
        counts[:, 1] = n
        from .cache import AccessBatch
        gather(self.pool, self.store, AccessBatch(counts=counts, sel_row=None, miss_ids=order,
                                                  miss_row=slots.contiguous()), max_ctas=148)
        self.pool.check("prefill_warmup")

    def preload_full_history(self) -> None:
        """The all-HBM ceiling's state: every request's whole history made
        resident in its pool (needs sparse_ratio = 1) and its slot rows filled from the
        host store, so every selection hits and no step gathers anything."""
        if any(pool_capacity(self.rho, n) < n for n in self.ctx_lens):  # each pool its own history
            raise ValueError("preload_full_history needs a pool that holds the whole history (rho = 1)")
        B, d = self.B, self.device
        full = torch.arange(self.ctx, dtype=torch.int32, device=d)
        for c0 in range(0, self.ctx, _lib.MAX_REQUEST):
            ids = full[c0:c0 + _lib.MAX_REQUEST].expand(B, -1).contiguous()
            nb = torch.tensor([min(_lib.MAX_REQUEST, max(0, n - c0)) for n in self.ctx_lens],
                              dtype=torch.int32, device=d)
            self.pool.warmup(ids, nb)
            slots = torch.stack([self.pool.lookup(b, ids[b]) for b in range(B)])
            cnt = torch.zeros((B, 4), dtype=torch.int32, device=d)
            cnt[:, 1] = nb
            gather(self.pool, self.store, AccessBatch(cnt, None, ids, slots.contiguous()), max_ctas=148)
        self.pool.check("preload_full_history")

    # -- the decode step -------------------------------------------------------------------
    def _select(self, q_idx, a, b, max_ctas: int = 0):
        """K1 -> K2 -> K3 for requests [a, b) on the current stream, writing into the
        step's shared access buffers (row slices)."""
        indexer_logits(q_idx[a:b], self.w[a:b], self.k_cache[a:b], self.k_scale[a:b],
                       self.lens[a:b], out=self.logits[a:b], max_ctas=max_ctas)
        topk(self.logits[a:b], self.lens[a:b], self.K, out=self.idx[a:b], count=self.cnt[a:b])
        return self.pool.access(self.idx[a:b], self.cnt[a:b], begin=a, out=self._acc_view(a, b))

    def _acc_view(self, a, b):
        acc = self.acc
        return AccessBatch(counts=acc.counts[a:b], sel_row=acc.sel_row[a:b],
                           miss_ids=acc.miss_ids[a:b], miss_row=acc.miss_row[a:b],
                           hit_row=acc.hit_row[a:b])

    def micro_batches(self, n: int):
        """[a, b) request ranges of the DBA split: contiguous; the first holds
        ``first_frac`` of the batch when set (a small first micro-batch starts the
        host-link gather early), the rest split evenly."""
        sizes = getattr(self, "mb_sizes", None) or (
            [int(x) for x in os.environ["ESS_MB_SIZES"].split(",")] if os.environ.get("ESS_MB_SIZES") else None)
        if sizes and n > 1:  # explicit micro-batch sizes (must cover the batch)
            if sum(sizes) != self.B or min(sizes) < 1:
                raise ValueError(f"micro-batch sizes {sizes} do not partition {self.B} requests")
            edges = [0]
            for z in sizes:
                edges.append(edges[-1] + z)
            return [(edges[i], edges[i + 1]) for i in range(len(sizes))]
        n = max(1, min(n, self.B))
        ff = getattr(self, "first_frac", None)
        if n == 1 or not ff:
            edges = [self.B * i // n for i in range(n + 1)]
        else:
            f = min(self.B - (n - 1), max(1, round(self.B * ff)))
            edges = [0] + [f + (self.B - f) * i // (n - 1) for i in range(n)]
        return [(edges[i], edges[i + 1]) for i in range(n)]

    def attend(self, q_idx, q, gather_ctas: int = 32, overlap: str = "dba", new_rows=None,
               micro: int = 2):
        """K1..K5 for every request of the layer.

        overlap="da" is the paper's DA schedule (the reference
        models it as span DAGs, pipeline.py:125-141): right after the cache manager,
        the host-link miss gather (K4) runs on a high-priority side stream while
        attention over the rows that were already resident (Attn0) runs on the main
        stream; the fetched rows are attended once they land (Attn1) — the merge is
        the resumed online softmax.  overlap="none" runs K4 then one K5 pass.

        overlap="dba" adds the paper's batch split (DBA; pipeline.py
        :144-167): the requests are cut into ``micro`` contiguous micro-batches whose
        K1 -> K2 -> K3 run back to back; micro-batch i's gather starts as soon as its
        cache manager is done and overlaps micro-batch i+1's indexer, which runs on the
        SMs the gather leaves free.  Attention is still one launch over all requests
        (Attn0 for every request right away, Attn1 per request as its rows land).

        ``new_rows`` (DA/DBA) also admits this step's generated rows, on a third
        stream right after the last cache manager: admission touches no row the step
        reads (its LRU victim is never one of the rows K3 just stamped, and the new
        token id is outside the selection), so it hides under the gather instead of
        trailing the step.  The LRU state afterwards is the same as access-then-append.
        """
        B = self.B
        if self.acc is None:
            z = lambda: torch.empty((B, self.K), dtype=torch.int32, device=self.device)  # noqa: E731
            self.acc = AccessBatch(counts=torch.empty((B, 4), dtype=torch.int32, device=self.device),
                                   sel_row=z(), miss_ids=z(), miss_row=z(), hit_row=z())
            self._settle = z()
            self._counts_b = torch.empty((B, 4), dtype=torch.int32, device=self.device)
        acc = self.acc
        if overlap == "stream":
            return self._attend_stream(q_idx, q, new_rows, gather_ctas)
        if overlap == "none":
            self._select(q_idx, 0, B)
            gather(self.pool, self.store, acc, max_ctas=gather_ctas)
            sparse_mla(self.pool, q, acc.sel_row, self.cnt, self.sm_scale, out=self.out, lse=self.lse)
            return self.out, self.lse
        if overlap not in ("da", "dba", "dbs"):
            raise ValueError(f"unknown overlap schedule {overlap!r}")
        # dbs: DBA whose later micro-batches are handed on per request (streamed K1 ->
        # K2+K3a -> K4 as in overlap="stream"), so their first misses reach the link
        # while the micro-batch's indexer still runs
        dbs = overlap == "dbs"
        if dbs and not self.stream_ok():
            raise ValueError("the dbs schedule needs early gather, rows <= 40K tokens per CTA and the fused DA")
        main = torch.cuda.current_stream(self.device)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device, priority=-1)
            self._ws = SplitWorkspace(B, self.device)
            self._landed = torch.zeros(B, dtype=torch.int32, device=self.device)
        side = self._side
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        # one fused K5 launch when its 2B CTAs and the gather fit the GPU at once (its
        # CTAs wait for the gather's arrival counters); two passes + merge otherwise
        fused = self.fuse_da and 2 * B <= sms - 8
        # small batches: spread each request's rows over 2 * split CTAs (KV split +
        # combine) while leaving the gather its SMs; attention takes one SM per CTA
        split = 1
        if fused:
            split = max(1, min(self.max_split, (sms - 8 - self.min_gather_sms) // (2 * B)))
        gsms = max(8, sms - 2 * B * split)
        if split > 1 and getattr(self, "_ws_split", None) is None:
            self._ws_split = SplitWorkspace(B, self.device, splits=split)
        ranges = self.micro_batches(micro if overlap in ("dba", "dbs") else 1)
        if dbs:
            if getattr(self, "_sync", None) is None:
                self._sync = torch.zeros(3 * B, dtype=torch.int32, device=self.device)  # done | ready | claim
            self._sync.zero_()
            done_c, ready_c, claim_c = self._sync[:B], self._sync[B:2 * B], self._sync[2 * B:]
            cln = 1  # CTAs per streamed top-k row (rows > 40K tokens take a cluster)
            while cln < 8 and -(-self.Lmax // cln) > 40 * 1024:
                cln *= 2
            nk2 = min(B, self.stream_topk_ctas)
        if getattr(self, "_sel", None) is None:
            self._sel = torch.cuda.Stream(self.device)
            self._lru = torch.cuda.Stream(self.device)
        sel, lru = self._sel, self._lru
        ready = None
        # step_host's link-serial graphs (capture_host): the first gather waits for the
        # external "queries uploaded" event, the last one records "gathered"
        ext = getattr(self, "_ext", None)
        if ext is not None and dbs:
            raise ValueError("capture_host supports the da / dba schedules")
        ext_wait = ext is not None
        pdl_next = False  # launch the next indexer programmatically (behind a main-stream gather)
        prev = 0  # requests of the previous micro-batch (its K2/K3 run beside this K1)
        for i, (a, b) in enumerate(ranges):
            # K1 of micro-batch i on the main stream; its top-k and cache manager on the
            # selection stream, so they overlap the NEXT micro-batch's indexer, which
            # leaves SMs free for them (one per request) and for the running gather
            # gathers of earlier micro-batches run beside the next indexer, not beside
            # attention, and may take more SMs (early_gather_sms) than the last one
            g_i = gsms if i == len(ranges) - 1 else max(gsms, self.early_gather_sms)
            g_prev = 0 if i == 0 else (gsms if i - 1 == len(ranges) - 1 else max(gsms, self.early_gather_sms))
            if self.gather_shared:
                # the gather's CTAs sit beside the indexer's / attention's on the same SMs
                late = i == len(ranges) - 1
                want = self.shared_late_gather_ctas if late else self.shared_early_gather_ctas
                g_i = want or g_i
                g_prev = 0
            ctas = 0 if i == 0 else sms - g_prev - prev
            if i > 0 and self.late_k1_ctas:  # cap: less HBM pressure beside the gather
                ctas = min(ctas, self.late_k1_ctas)
            if dbs and i > 0:
                self._attend_dbs_mb(q_idx, a, b, sms - g_prev - max(prev, nk2 * cln), nk2, cln, g_i,
                                    done_c, ready_c, claim_c, fused)
                ready, fetched = self._dbs_selected, self._dbs_fetched
                self._lru_mb(a, b, ready, fetched)
                lru_ready = self._lru_ready
                prev = nk2 * cln
                continue
            indexer_logits(q_idx[a:b], self.w[a:b], self.k_cache[a:b], self.k_scale[a:b],
                           self.lens[a:b], out=self.logits[a:b], max_ctas=ctas, pdl=pdl_next)
            pdl_next = False
            if self.pdl and self.early_gather and i == 0:
                # the first micro-batch's K1 -> K2 + K3a -> K4 chain back to back on the main
                # stream with programmatic dependent launches: each kernel becomes resident
                # on the SMs its producer's tail frees and waits on the device, so the first
                # misses reach the host link without two launch latencies.  With one
                # micro-batch (DA) the gather stays on the side stream (attention, next on
                # the main stream, overlaps it).
                topk_split(self.logits[a:b], self.lens[a:b], self.K, self.idx[a:b], self.cnt[a:b],
                           self.pool, self._acc_view(a, b), begin=a, pdl=True)
                ready = torch.cuda.Event()
                ready.record(main)
                # the next indexer reads nothing the split writes: it launches beside it.
                # The gather stays on the side stream — an event recorded after a gather on
                # the main stream would hold the next micro-batch's top-k until the gather ends.
                pdl_next = self.pdl_gather == 0
                side.wait_event(ready)
                if ext_wait:
                    ext[0].wait(side)
                    ext_wait = False
                with torch.cuda.stream(side):
                    gather(self.pool, self.store, self._acc_view(a, b), begin=a, max_ctas=g_i,
                           exclusive=not self.gather_shared, landed=self._landed[a:b] if fused else None)
                    fetched = torch.cuda.Event()
                    fetched.record(side)
                self._lru_mb(a, b, ready, fetched)
                lru_ready = self._lru_ready
                prev = b - a
                continue
            scored = torch.cuda.Event()
            scored.record(main)
            sel.wait_event(scored)
            with torch.cuda.stream(sel):
                if self.early_gather:
                    # K2 + K3a (the hit/miss split; misses -> staging rows) in one launch:
                    # the gather starts right after the top-k
                    topk_split(self.logits[a:b], self.lens[a:b], self.K, self.idx[a:b], self.cnt[a:b],
                               self.pool, self._acc_view(a, b), begin=a)
                else:
                    topk(self.logits[a:b], self.lens[a:b], self.K, out=self.idx[a:b], count=self.cnt[a:b])
                    self.pool.access(self.idx[a:b], self.cnt[a:b], begin=a, out=self._acc_view(a, b))
                ready = torch.cuda.Event()
                ready.record(sel)
            side.wait_event(ready)
            if ext_wait:
                ext[0].wait(side)
                ext_wait = False
            with torch.cuda.stream(side):
                gather(self.pool, self.store, self._acc_view(a, b), begin=a, max_ctas=g_i,
                       exclusive=not self.gather_shared, landed=self._landed[a:b] if fused else None)
                fetched = torch.cuda.Event()
                fetched.record(side)
            if self.early_gather:
                self._lru_mb(a, b, ready, fetched)
                lru_ready = self._lru_ready
            else:
                lru_ready = ready
            prev = b - a
        if self.early_gather:
            settled = torch.cuda.Event()
            settled.record(lru)
        main.wait_event(ready)  # attention reads every micro-batch's selections
        if ext is not None:
            ext[1].record(side)  # every gather of the step issued on the side stream
            ext[0].wait(main)    # attention reads the uploaded queries
        if new_rows is not None:
            if getattr(self, "_adm", None) is None:
                self._adm = torch.cuda.Stream(self.device)
            self._adm.wait_event(lru_ready)  # the final LRU state of every micro-batch
            with torch.cuda.stream(self._adm):
                self._append_device(new_rows)
            admitted = torch.cuda.Event()
            admitted.record(self._adm)
        done = torch.cuda.Event()
        done.record(side)
        if fused:
            sparse_mla_da(self.pool, q, acc, self._landed, self.sm_scale, out=self.out, lse=self.lse,
                          split=split, workspace=self._ws_split if split > 1 else None)
            main.wait_event(done)
            if self.early_gather:
                main.wait_event(settled)
            if new_rows is not None:
                main.wait_event(admitted)
            return self.out, self.lse
        sparse_mla(self.pool, q, acc.hit_row, acc.counts[:, 0], self.sm_scale,
                   workspace=self._ws, mode="partial")
        main.wait_event(done)
        sparse_mla(self.pool, q, acc.miss_row, acc.counts[:, 1], self.sm_scale, out=self.out,
                   lse=self.lse, workspace=self._ws, mode="resume")
        if self.early_gather:
            main.wait_event(settled)
        if new_rows is not None:
            main.wait_event(admitted)
        return self.out, self.lse

    def _lru_mb(self, a, b, ready, fetched) -> None:
        """K3b (the LRU update proper, reporting each miss's final slot) and the settle
        (staging -> final slots, after the gather) of requests [a, b) on their own stream,
        so neither delays the next micro-batch's selection or gather."""
        lru = self._lru
        lru.wait_event(ready)
        with torch.cuda.stream(lru):
            self.pool.access(self.idx[a:b], self.cnt[a:b], begin=a, out=AccessBatch(
                counts=self._counts_b[a:b], sel_row=None, miss_ids=None,
                miss_row=self._settle[a:b], hit_row=None))
            self._lru_ready = torch.cuda.Event()
            self._lru_ready.record(lru)
            lru.wait_event(fetched)
            self.pool.settle(self._settle[a:b], self.acc.counts[a:b], begin=a)

    def _attend_dbs_mb(self, q_idx, a, b, k1_ctas, nk2, cln, g, done, ready, claim, fused) -> None:
        """One later micro-batch of the dbs schedule: its indexer (main stream) counts each
        request's stored logits rows, a persistent top-k + split grid (selection stream,
        after the previous micro-batch's top-k) starts each row once complete and
        publishes it, and a persistent gather (side stream, after the previous gather)
        fetches each published miss list.  Progress: the indexer waits on nothing, so
        its CTAs always finish and free SMs for any not yet resident; the waiting grids
        take nk2 * cln + g SMs."""
        main, sel, side = torch.cuda.current_stream(self.device), self._sel, self._side
        acc = self._acc_view(a, b)
        # the top-k grid runs BESIDE this indexer: it waits only for what precedes it on
        # the main stream (the zeroed counters, the previous indexer), not for it
        before = torch.cuda.Event()
        before.record(main)
        indexer_logits_stream(q_idx[a:b], self.w[a:b], self.k_cache[a:b], self.k_scale[a:b], self.lens[a:b],
                              self.logits[a:b], done[a:b], self.stream_group | (self.stream_first << 16),
                              max(8, k1_ctas))
        sel.wait_event(before)
        side.wait_event(before)  # the zeroed counters (the previous gather may be elsewhere)
        with torch.cuda.stream(sel):
            topk_split_stream(self.logits[a:b], self.lens[a:b], self.K, self.idx[a:b], self.cnt[a:b],
                              self.pool, acc, done[a:b], ready[a:b], nk2, begin=a)
            self._dbs_selected = torch.cuda.Event()
            self._dbs_selected.record(sel)
        with torch.cuda.stream(side):
            gather_stream(self.pool, self.store, acc, ready[a:b], claim[a:b],
                          self._landed[a:b] if fused else None, begin=a, max_ctas=g)
            self._dbs_fetched = torch.cuda.Event()
            self._dbs_fetched.record(side)

    def stream_ok(self) -> bool:
        """The streamed schedule's preconditions: early gather (every pool holds a whole
        selection, staging rows), rows of at most 8 top-k CTAs, and the fused DA launch."""
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        return (self.early_gather and self.Lmax <= 8 * 40 * 1024 and self.fuse_da and 2 * self.B <= sms - 8)

    def _attend_stream(self, q_idx, q, new_rows, gather_ctas):
        """The streamed step: K1, K2+K3a and K4 run CONCURRENTLY as three persistent grids
        handing each request on through per-request counters instead of micro-batch
        boundaries (PAPER.md:363-367's overlap taken to request granularity): the indexer
        finishes the requests group by group (``stream_group`` requests with the whole
        grid) and counts each request's stored logits rows; the top-k grid starts a row
        as soon as its logits are complete and publishes its hit/miss split; the gather
        grid fetches a request's misses as soon as that split is published.  The host
        link thus starts ~one top-k after the first group instead of after a micro-
        batch's indexer + top-k.  K3b, the settle, the admission and the fused DA
        attention follow as in the DBA schedule.  The three grids are sized to be
        co-resident (each CTA takes an SM): K1 gets the SMs the top-k and the gather
        grids leave."""
        if not self.stream_ok():
            raise ValueError("the streamed schedule needs early gather, rows <= 40K tokens and the fused DA")
        B, K, d, acc = self.B, self.K, self.device, self.acc
        main = torch.cuda.current_stream(d)
        if getattr(self, "_sync", None) is None:
            self._sync = torch.zeros(3 * B, dtype=torch.int32, device=d)  # done | ready | claim
        for name, prio in (("_side", -1), ("_sel", 0), ("_lru", 0), ("_adm", 0)):
            if getattr(self, name, None) is None:
                setattr(self, name, torch.cuda.Stream(d, priority=prio))
        if getattr(self, "_landed", None) is None:
            self._landed = torch.zeros(B, dtype=torch.int32, device=d)
            self._ws = SplitWorkspace(B, d)
        side, sel, lru = self._side, self._sel, self._lru
        done, ready, claim = self._sync[:B], self._sync[B:2 * B], self._sync[2 * B:]
        sms = torch.cuda.get_device_properties(d).multi_processor_count
        nk2 = self.stream_topk_ctas
        nk2 = min(B, nk2) if nk2 > 0 else -min(B, -nk2)
        g = self.stream_gather_ctas
        split = max(1, min(self.max_split, (sms - 8 - g) // (2 * B)))
        if split > 1 and getattr(self, "_ws_split", None) is None:
            self._ws_split = SplitWorkspace(B, d, splits=split)
        self._sync.zero_()
        start = torch.cuda.Event()
        start.record(main)
        cln = 1  # CTAs per top-k row: the smallest cluster whose slice fits (rows > 40K tokens)
        while cln < 8 and -(-self.Lmax // cln) > 40 * 1024:
            cln *= 2
        k2_sms = nk2 * cln if nk2 > 0 else -nk2 * max(2, cln)   # < 0: at least CTA pairs
        indexer_logits_stream(q_idx, self.w, self.k_cache, self.k_scale, self.lens, self.logits, done,
                              self.stream_group | (self.stream_first << 16), sms - k2_sms - g)
        sel.wait_event(start)
        with torch.cuda.stream(sel):
            topk_split_stream(self.logits, self.lens, K, self.idx, self.cnt, self.pool, acc, done, ready, nk2)
            selected = torch.cuda.Event()
            selected.record(sel)
        side.wait_event(start)
        with torch.cuda.stream(side):
            gather_stream(self.pool, self.store, acc, ready, claim, self._landed, max_ctas=g)
            fetched = torch.cuda.Event()
            fetched.record(side)
        lru.wait_event(selected)
        with torch.cuda.stream(lru):  # K3b (LRU update, final slots), then the settle
            self.pool.access(self.idx, self.cnt, out=AccessBatch(
                counts=self._counts_b, sel_row=None, miss_ids=None, miss_row=self._settle, hit_row=None))
            lru_ready = torch.cuda.Event()
            lru_ready.record(lru)
            lru.wait_event(fetched)
            self.pool.settle(self._settle, acc.counts)
            settled = torch.cuda.Event()
            settled.record(lru)
        if new_rows is not None:
            self._adm.wait_event(lru_ready)
            with torch.cuda.stream(self._adm):
                self._append_device(new_rows)
                admitted = torch.cuda.Event()
                admitted.record(self._adm)
        main.wait_event(selected)
        sparse_mla_da(self.pool, q, acc, self._landed, self.sm_scale, out=self.out, lse=self.lse,
                      split=split, workspace=self._ws_split if split > 1 else None)
        main.wait_event(fetched)
        main.wait_event(settled)
        if new_rows is not None:
            main.wait_event(admitted)
        return self.out, self.lse

    # -- whole-step CUDA graph ------------------------------------------------------------
    def _append_device(self, new_rows: torch.Tensor) -> None:
        """append_token with every per-step scalar derived on the device: the new id is
        each request's history length and the capacity floor(rho * (history + 1))
        (cache.py:137-138, :191-195) — float64, bit-identical to math.floor."""
        _lib.check(_lib.load().ess_pool_admit(
            self.pool.handle, 0, self.B, self.lens.data_ptr(), None, float(self.rho),
            new_rows.data_ptr(), new_rows.stride(0) // ROW, self.store.pool_ptr(0),
            self.store.rows_per_pool, None, _lib.stream_handle()), "ess_pool_admit")

    def _device_step(self, overlap: str, gather_ctas: int) -> None:
        # admission overlaps attention only while every pool holds more than K rows:
        # a smaller pool keeps part of the selection in rows the admission may evict
        # (capacity only grows with history, so this holds for every later replay)
        hist_min = min(self.ctx_lens) + self.history - self.ctx
        early = overlap in ("da", "dba", "dbs", "stream") and math.floor(self.rho * hist_min) > self.K
        self.attend(self.q_idx_in, self.q_in, gather_ctas=gather_ctas, overlap=overlap,
                    new_rows=self.rows_in if early else None, micro=self.micro)
        if not early:
            self._append_device(self.rows_in)

    def launches_per_step(self, overlap: str) -> int:
        """Kernels of this library one captured step launches (the graph's kernel nodes):
        per micro-batch K1, K2, K3 (or K3a + K3b with the early gather), K4 (+ settle);
        then K5 (+ the KV-split combine) and the admission."""
        if overlap == "none":
            return 6  # K1, K2, K3, K4, K5, admission
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        if overlap == "stream":  # K1, K2+K3a, K4, K3b, settle, K5 (+ combine), admission
            split = max(1, min(self.max_split, (sms - 8 - self.stream_gather_ctas) // (2 * self.B)))
            return 7 + (split > 1)
        micro = self.micro if overlap in ("dba", "dbs") else 1
        # early gather: K2 + K3a fused, + K3b, settle
        per_mb = 5 if self.early_gather else 4
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        fused = self.fuse_da and 2 * self.B <= sms - 8
        split = max(1, min(self.max_split, (sms - 8 - self.min_gather_sms) // (2 * self.B))) if fused else 1
        k5 = (1 + (split > 1)) if fused else 2
        return per_mb * micro + k5 + 1

    def access_totals(self) -> tuple[int, int]:
        """(hits, misses) summed over the layer's pools since creation (the pools'
        own counters, cache.py:41-43): the difference across a run gives its hit rate."""
        c = self.pool.counters()
        return int(c[:, 2].sum()), int(c[:, 3].sum())

    def _alloc_static(self) -> None:
        """The graph's static input buffers, filled with the next queries."""
        B, d = self.B, self.device
        self.q_idx_in = torch.empty((B, 64, 128), dtype=torch.uint8, device=d)
        self.q_in = torch.empty((B, 128, 576), dtype=torch.bfloat16, device=d)
        self.rows_in = torch.zeros((B, 1, ROW), dtype=torch.uint8, device=d)
        self._ids = torch.empty((B, 1), dtype=torch.int32, device=d)
        self._one = torch.ones(B, dtype=torch.int32, device=d)
        self._caps = torch.empty(B, dtype=torch.int32, device=d)
        q_idx, q = self.next_queries()
        self.q_idx_in.copy_(q_idx)
        self.q_in.copy_(q)

    def capture(self, overlap: str = "dba", gather_ctas: int = 32) -> None:
        """Record one full decode step (K1..K5 for every micro-batch, the side-stream
        gathers, grow/append/write-back) as a CUDA graph; ``step`` replays it.  The
        first (eager) step also runs here — it advances the state like any step."""
        d = self.device
        self._alloc_static()
        s = torch.cuda.Stream(d)
        s.wait_stream(torch.cuda.current_stream(d))
        with torch.cuda.stream(s):
            self._device_step(overlap, gather_ctas)  # eager: sets up attrs / maps
        torch.cuda.current_stream(d).wait_stream(s)
        torch.cuda.synchronize(d)
        eager_counts = self.step_counts().clone()
        self.history += 1
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._device_step(overlap, gather_ctas)
        return eager_counts  # access counts of the eager step (graph buffers are unwritten)

    def step(self, q_idx: torch.Tensor, q: torch.Tensor, new_rows: torch.Tensor):
        """One decode step through the captured graph: inputs land in the graph's
        static buffers (two device copies), then a single graph launch."""
        self._check_room()
        _lib.copy_many([(self.q_idx_in, q_idx), (self.q_in, q), (self.rows_in, new_rows)])
        self.graph.replay()
        self.history += 1
        return self.out, self.lse

    def _check_room(self) -> None:
        """A replayed step admits one generated id per request at its history length;
        past Lmax the admission kernel latches ESS_ERR_ARG and stops advancing, so the
        host refuses the step before it is launched (the device status is the backstop,
        read by ``pool.check``)."""
        if self.history + 1 > self.Lmax:
            raise ValueError(f"decode step {self.history - self.ctx + 1} exceeds max_new_tokens: "
                             f"history {self.history} + 1 > Lmax {self.Lmax}")

    def capture_host(self, overlap: str = "dba", gather_ctas: int = 32) -> None:
        """Graphs for ``step_host``'s link-serial pipeline (after ``capture``): one per
        host-staging slot, reading that slot's queries in place and writing its own
        output buffer.  The queries' H2D copy (copy engine) and the miss gather (SM
        reads) share the host link, and run together they both slow down (the copy
        engines' traffic throttles SM-initiated host reads), so the
        pipeline keeps them apart: step t+1's query upload starts when step t's last
        gather has issued (an external event recorded inside graph t) and graph t+1's
        first gather and its attention wait for that upload (an external event wait
        node), while its indexer / top-k run under the upload."""
        if overlap not in ("da", "dba"):
            raise ValueError("capture_host supports the da / dba schedules")
        if getattr(self, "graph", None) is None:
            self.capture(overlap, gather_ctas)
        base = (self.q_idx_in, self.q_in, self.out)
        self._hslots = []
        for _ in range(2):
            slot = {"qi": torch.empty_like(base[0]), "q": torch.empty_like(base[1]),
                    "out": torch.empty_like(base[2]), "uploaded": torch.cuda.Event(external=True),
                    "gathered": torch.cuda.Event(external=True)}
            for e in ("qi_ready", "in_free", "done", "out_free"):
                slot[e] = torch.cuda.Event()
            for e in ("uploaded", "gathered"):  # create the CUDA events before capture
                slot[e].record()
            slot["qi"].copy_(base[0])
            slot["q"].copy_(base[1])
            self.q_idx_in, self.q_in, self.out = slot["qi"], slot["q"], slot["out"]
            self._ext = (slot["uploaded"], slot["gathered"])
            try:
                slot["graph"] = torch.cuda.CUDAGraph()
                with torch.cuda.graph(slot["graph"]):
                    self._device_step(overlap, gather_ctas)
            finally:
                self._ext = None
                self.q_idx_in, self.q_in, self.out = base
            self._hslots.append(slot)
        torch.cuda.synchronize(self.device)

    def step_host(self, h_q_idx: torch.Tensor, h_q: torch.Tensor, new_rows: torch.Tensor,
                  h_out: torch.Tensor) -> None:
        """One step with the queries in pinned host memory and the attention output
        returned to pinned host memory.  H2D and D2H run on copy streams into
        double-buffered device staging, so step t's transfers overlap steps t-1 / t+1
        while every step still moves its own inputs and result over the host link;
        after ``capture_host`` the query upload is kept off the link while the gathers
        run (link-serial pipeline).  Asynchronous: synchronise before reading ``h_out``."""
        d = self.device
        self._check_room()
        if getattr(self, "_hslots", None):
            return self._step_host_serial(h_q_idx, h_q, new_rows, h_out)
        if getattr(self, "_cs", None) is None:
            self._cs = torch.cuda.Stream(d)    # H2D copies
            self._ds = torch.cuda.Stream(d)    # D2H copies (other PCIe direction)
            self._stage = [(torch.empty_like(self.q_idx_in), torch.empty_like(self.q_in),
                            torch.empty_like(self.out)) for _ in range(2)]
            self._ev = [{k: torch.cuda.Event() for k in ("in_ready", "in_free", "out_ready", "out_free")}
                        for _ in range(2)]
            self._slot = 0
        main, cs, ds = torch.cuda.current_stream(d), self._cs, self._ds
        s = self._slot
        self._slot ^= 1
        st_qi, st_q, st_out = self._stage[s]
        ev = self._ev[s]
        cs.wait_event(ev["in_free"])           # staging slot s no longer read by main
        with torch.cuda.stream(cs):
            st_qi.copy_(h_q_idx, non_blocking=True)
            st_q.copy_(h_q, non_blocking=True)
            ev["in_ready"].record(cs)
        main.wait_event(ev["in_ready"])
        _lib.copy_many([(self.q_idx_in, st_qi), (self.q_in, st_q), (self.rows_in, new_rows)])
        ev["in_free"].record(main)
        self.graph.replay()
        self.history += 1
        main.wait_event(ev["out_free"])        # previous D2H from this slot finished
        st_out.copy_(self.out)
        ev["out_ready"].record(main)
        ds.wait_event(ev["out_ready"])
        with torch.cuda.stream(ds):
            h_out.copy_(st_out, non_blocking=True)
            ev["out_free"].record(ds)

    def _step_host_serial(self, h_q_idx, h_q, new_rows, h_out) -> None:
        d = self.device
        if getattr(self, "_cs", None) is None:
            self._cs = torch.cuda.Stream(d)    # H2D copies
            self._ds = torch.cuda.Stream(d)    # D2H copies (other PCIe direction)
            self._slot = 0
        main, cs, ds = torch.cuda.current_stream(d), self._cs, self._ds
        k = self._slot
        self._slot ^= 1
        S, P = self._hslots[k], self._hslots[k ^ 1]
        cs.wait_event(S["in_free"])       # the graph that last read slot k has finished
        P["gathered"].wait(cs)            # the previous step's gathers are off the link
        with torch.cuda.stream(cs):
            S["qi"].copy_(h_q_idx, non_blocking=True)
            S["qi_ready"].record(cs)
            S["q"].copy_(h_q, non_blocking=True)
            S["uploaded"].record(cs)      # graph k's gathers and attention wait on this
        main.wait_event(S["qi_ready"])    # the indexer needs only the indexer queries
        main.wait_event(S["out_free"])    # the D2H of slot k's previous output is done
        _lib.copy_many([(self.rows_in, new_rows)])
        S["graph"].replay()
        self.history += 1
        S["in_free"].record(main)
        S["done"].record(main)
        ds.wait_event(S["done"])
        with torch.cuda.stream(ds):
            h_out.copy_(S["out"], non_blocking=True)
            S["out_free"].record(ds)

    def host_sync(self) -> None:
        """Wait for every outstanding step_host transfer."""
        for s in ("_cs", "_ds"):
            if getattr(self, s, None) is not None:
                getattr(self, s).synchronize()
        torch.cuda.synchronize(self.device)

    def step_counts(self) -> torch.Tensor:
        """[B, 4] access counts of the last step (hits, misses, evicted, transient)."""
        return self.acc.counts

    def append_token(self, new_rows: torch.Tensor | None = None, new_keys: torch.Tensor | None = None):
        """Each request admits its generated token (cache.py:191-195 order: grow, append)."""
        B, d = self.B, self.device
        steps = self.history - self.ctx + 1   # tokens generated after this one
        self.history += 1
        self.pool.grow([pool_capacity(self.rho, n + steps) for n in self.ctx_lens])
        if getattr(self, "_ids", None) is None:
            self._ids = torch.empty((B, 1), dtype=torch.int32, device=d)
            self._one = torch.ones(B, dtype=torch.int32, device=d)
        self._ids.copy_(self.lens.view(B, 1))  # the new id of request b is its history length
        slots = self.pool.append(self._ids, self._one)
        if new_rows is None:
            new_rows = random_latent_rows(B, d, self.gen).view(B, 1, ROW)
        write_generated(self.pool, self.store, self._ids, self._one, slots, new_rows)
        if new_keys is not None:
            self.k_cache[torch.arange(B, device=d), self.lens.long()] = new_keys
        self.lens += 1

    def close(self):
        self.pool.close()
        self.store.close()


class DSADecodeModel:
    """The attention path of a full decode step (BASELINE configs[2], "C3"): ``num_layers``
    DSA layers back to back, each with its own indexer key cache, LRU pools, slot store
    and host latent store (one pool per (request, layer)).  Layer l+1
    starts only once layer l's attention output exists (its inputs would be computed
    from it in the real model), so overlap stays inside a layer (DA / DBA); the whole
    step is one CUDA graph.  Projections, MoE and the dense MLP are outside this path
    (DESIGN.md §12); every layer's queries are synthetic inputs."""

    def __init__(self, num_layers: int, batch: int, context_len: int, sparse_ratio: float,
                 topk_k: int = 2048, max_new_tokens: int = 64, device=None, seed: int = 0,
                 drift=0.97, hugepages: bool = True):
        """``drift``: one query-drift coefficient for every layer, or one per layer (real
        models' layers differ in step-to-step selection similarity, hence in misses —
        what the layer-wise plan keys on)."""
        drifts = list(drift) if isinstance(drift, (list, tuple, np.ndarray)) else [drift] * num_layers
        if len(drifts) != num_layers:
            raise ValueError(f"{len(drifts)} drift values for {num_layers} layers")
        self.layers = [DSADecodeLayer(batch, context_len, sparse_ratio, topk_k, max_new_tokens,
                                      device=device, seed=seed + 7919 * i, drift=float(drifts[i]),
                                      hugepages=hugepages) for i in range(num_layers)]
        self.B, self.device = batch, self.layers[0].device
        self.plan = None

    def set_schedule(self, micro: int = 2, first_frac: float | None = None) -> None:
        for layer in self.layers:
            layer.micro, layer.first_frac = micro, first_frac

    def prefill_warmup(self, windows: int = 32) -> None:
        for layer in self.layers:
            layer.prefill_warmup(windows=windows)

    def next_queries(self):
        return [layer.next_queries() for layer in self.layers]

    def capture(self, overlap: str = "dba", gather_ctas: int = 32, plan=None) -> None:
        """One eager step (advances the state), then the whole step captured as a graph.

        ``plan`` (a ``plan.LayerPlan``, pipeline.py:177-195): each layer is recorded with
        its own strategy — ``"dba"`` micro-batched with the schedule's ``micro``,
        ``"da"`` one batch, ``"none"`` sequential — instead of ``overlap`` for all."""
        d = self.device
        if plan is not None:
            plan.check(len(self.layers))
        self.plan = plan
        ovs = list(plan.strategies) if plan is not None else [overlap] * len(self.layers)
        for layer in self.layers:
            layer._alloc_static()
        s = torch.cuda.Stream(d)
        s.wait_stream(torch.cuda.current_stream(d))
        with torch.cuda.stream(s):
            for layer, ov in zip(self.layers, ovs):
                layer._device_step(ov, gather_ctas)
        torch.cuda.current_stream(d).wait_stream(s)
        torch.cuda.synchronize(d)
        for layer in self.layers:
            layer.history += 1
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            for layer, ov in zip(self.layers, ovs):
                layer._device_step(ov, gather_ctas)
        self._overlaps = ovs

    def plan_layers(self, threshold: float, meter=None, source: str = "live miss means"):
        """The layer-wise plan from the model's running miss means (``plan.MissMeter``:
        the pools' own counters since its snapshot), pipeline.py:190-195."""
        from .plan import MissMeter, plan_from_means
        meter = meter if meter is not None else MissMeter(self)
        return plan_from_means(meter.means(), threshold, source)

    def launches_per_step(self) -> int:
        """This library's kernel nodes in the captured step (each layer's own schedule)."""
        return sum(layer.launches_per_step(ov) for layer, ov in zip(self.layers, self._overlaps))

    def step(self, queries, new_rows) -> None:
        """queries: per layer (q_idx, q); new_rows: per layer [B, 1, 656] (or one shared)."""
        for layer in self.layers:
            layer._check_room()
        pairs = []
        for i, (layer, (q_idx, q)) in enumerate(zip(self.layers, queries)):
            pairs += [(layer.q_idx_in, q_idx), (layer.q_in, q),
                      (layer.rows_in, new_rows[i] if isinstance(new_rows, (list, tuple)) else new_rows)]
        _lib.copy_many(pairs)  # every layer's inputs: one SM copy kernel per 64 tensors
        self.graph.replay()
        for layer in self.layers:
            layer.history += 1

    def access_totals(self) -> tuple[int, int]:
        h = m = 0
        for layer in self.layers:
            a, b = layer.access_totals()
            h, m = h + a, m + b
        return h, m

    def check(self, what: str = "model") -> None:
        for i, layer in enumerate(self.layers):
            layer.pool.check(f"{what} layer {i}")

    def close(self) -> None:
        for layer in self.layers:
            layer.close()


class SelectionRecorder:
    """Live K2 selections -> ESSTRACE v1 (format trace.py:238-287,
    SPEC.md:194).  Attach one recorder to the decode layers of a model (one trace
    layer per DSADecodeLayer); after each decode step ``record()`` copies every
    request's selection set to the host.  ``trace(b)`` is request b's AccessTrace, so
    ``offsim trace stats`` computes the Eq. (1) step-to-step similarity
    (trace.py:164-196) of model-driven runs and ``offsim simulate --trace`` / ``replay``
    re-run the cache manager on them.  Diagnostic / export path: it synchronises, so
    it stays outside timed regions."""

    def __init__(self, layers):
        self.layers = list(layers)
        if not self.layers:
            raise ValueError("no layers to record")
        l0 = self.layers[0]
        self.B, self.ctx, self.K = l0.B, l0.ctx, l0.K
        if any((l.B, l.ctx, l.K) != (self.B, self.ctx, self.K) for l in self.layers):
            raise ValueError("layers must share batch, context and top-k")
        self.steps = [[] for _ in range(self.B)]       # [b][t] -> list over layers
        self.windows = None                              # [b][layer][window]

    def prefill(self, windows_per_layer) -> None:
        """``windows_per_layer[l]`` = DSADecodeLayer.prefill_warmup(record=True) of layer l."""
        if len(windows_per_layer) != len(self.layers):
            raise ValueError("one window list per layer")
        self.windows = [[[np.asarray(w[b], dtype=np.int64) for w in windows_per_layer[l]]
                         for l in range(len(self.layers))] for b in range(self.B)]

    def record(self) -> None:
        """Append the selections of the step just run (one accepted token per step)."""
        sel = [(l.idx.cpu().numpy(), l.cnt.cpu().numpy()) for l in self.layers]
        for b in range(self.B):
            self.steps[b].append([idx[b, :cnt[b]].astype(np.int64) for idx, cnt in sel])

    def trace(self, b: int):
        from .trace import AccessTrace, StepAccess
        tr = AccessTrace(num_layers=len(self.layers), context_len=self.layers[0].ctx_lens[b], topk=self.K,
                         steps=[StepAccess(layers=s, tokens_accepted=1) for s in self.steps[b]],
                         prefill_windows=self.windows[b] if self.windows is not None else None)
        tr.check()
        return tr

    def write(self, b: int, path) -> None:
        from .trace import write_trace
        write_trace(self.trace(b), path)
