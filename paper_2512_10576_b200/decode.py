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
from dataclasses import dataclass, field

import torch

from . import _lib
from .attention import DEFAULT_SM_SCALE, sparse_mla
from .cache import PoolSet, pool_capacity
from .indexer import indexer_logits, topk
from .transfer import HostLatentStore, gather, write_generated

ROW = 656


def _e4m3(x: torch.Tensor) -> torch.Tensor:
    return x.clamp(-448.0, 448.0).to(torch.float8_e4m3fn).view(torch.uint8)


def random_latent_rows(n: int, device, gen=None) -> torch.Tensor:
    """[n, 656] latent rows: e4m3 NoPE (values ~N(0,1)*32 quantised), positive
    group scales ~1/32, bf16 RoPE ~N(0,1)."""
    nope = _e4m3(torch.randn((n, 512), device=device, generator=gen) * 32.0)
    scales = (torch.rand((n, 4), device=device, generator=gen) * 0.5 + 0.75) / 32.0
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

    def __init__(self, batch: int, context_len: int, sparse_ratio: float, topk_k: int = 2048,
                 max_new_tokens: int = 64, device=None, seed: int = 0, drift: float = 0.95,
                 sm_scale: float = DEFAULT_SM_SCALE):
        _lib.require_cuda()
        self.device = torch.device(device if device is not None else "cuda")
        self.B, self.ctx, self.rho, self.K = batch, context_len, sparse_ratio, topk_k
        self.drift, self.sm_scale = drift, sm_scale
        self.Lmax = ((context_len + max_new_tokens + 127) // 128) * 128
        self.gen = torch.Generator(device=self.device).manual_seed(seed)
        d, g, B = self.device, self.gen, batch
        self.lens = torch.full((B,), context_len, dtype=torch.int32, device=d)
        self.history = context_len
        # indexer key cache (HBM): e4m3 keys + f32 per-token scale
        self.k_cache = _e4m3(torch.randn((B, self.Lmax, 128), device=d, generator=g) * 8.0)
        self.k_scale = torch.rand((B, self.Lmax), device=d, generator=g) * 0.5 + 0.75
        # host latent store (pinned, mapped) + GPU slot pool
        self.store = HostLatentStore(B, self.Lmax)
        for b in range(B):  # fill through the GPU: random rows copied into pinned memory
            self.store.host[b].copy_(random_latent_rows(self.Lmax, d, g), non_blocking=False)
        self.cap0 = pool_capacity(sparse_ratio, context_len)
        self.cap_max = pool_capacity(sparse_ratio, self.Lmax)
        staging = topk_k if self.cap0 < topk_k else 0
        self.pool = PoolSet(B, self.Lmax, self.cap_max, self.cap0, row_bytes=_lib.SLOT_ROW_BYTES,
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
        order, n = self.pool.lru_order()
        order = order[:, :self.cap_max].contiguous()
        slots = torch.stack([self.pool.lookup(b, order[b].clamp_min(0)) for b in range(self.B)])
        counts = torch.zeros((self.B, 4), dtype=torch.int32, device=self.device)
        counts[:, 1] = n
        from .cache import AccessBatch
        gather(self.pool, self.store, AccessBatch(counts=counts, sel_row=None, miss_ids=order,
                                                  miss_row=slots.contiguous()), max_ctas=148)
        self.pool.check("prefill_warmup")
        return rec

    # -- the decode step -------------------------------------------------------------------
    def attend(self, q_idx, q, gather_ctas: int = 32):
        """K1..K5 for every request of the layer."""
        indexer_logits(q_idx, self.w, self.k_cache, self.k_scale, self.lens, out=self.logits)
        topk(self.logits, self.lens, self.K, out=self.idx, count=self.cnt)
        self.acc = self.pool.access(self.idx, self.cnt, out=self.acc)
        gather(self.pool, self.store, self.acc, max_ctas=gather_ctas)
        sparse_mla(self.pool, q, self.acc.sel_row, self.cnt, self.sm_scale, out=self.out, lse=self.lse)
        return self.out, self.lse

    def append_token(self, new_rows: torch.Tensor | None = None, new_keys: torch.Tensor | None = None):
        """Each request admits its generated token (cache.py:191-195 order: grow, append)."""
        B, d = self.B, self.device
        pos = self.history
        self.history += 1
        self.pool.grow(pool_capacity(self.rho, self.history))
        ids = torch.full((B, 1), pos, dtype=torch.int32, device=d)
        one = torch.ones(B, dtype=torch.int32, device=d)
        slots = self.pool.append(ids, one)
        if new_rows is None:
            new_rows = random_latent_rows(B, d, self.gen).view(B, 1, ROW)
        write_generated(self.pool, self.store, ids, one, slots, new_rows)
        if new_keys is not None:
            self.k_cache[:, pos] = new_keys
        self.lens += 1

    def close(self):
        self.pool.close()
        self.store.close()
