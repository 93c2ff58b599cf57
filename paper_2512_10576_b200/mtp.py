"""MTP decode: ``mtp + 1`` query tokens per request and step through K1 -> K5.

With multi-token prediction each decode step verifies ``qtok = mtp + 1`` tokens per
request (the main token and its drafts): the reference sizes the indexer at
``effective_token_width(mtp) * batch`` rows (costmodel.py:34-36, pipeline.py:213-215)
and appends ``tokens_accepted`` ids per step, Poisson(mean - 1) + 1
(trace.py:127, cache.py:191-195); the paper's Table 2 runs at MTP = 2 and 4
(PAPER.md:420-450).  On device:

  K1  one pass over each request's cached keys for all qtok tokens: tcgen05 MMA with
      N = 64 * qtok (``ess_indexer_logits_mtp``) — the indexer's HBM bytes do not grow
      with the MTP width;
  K2  one top-k row per (request, token) over the request's cached history
      (``ess_topk_mtp``; the selection universe is the cache history, trace.py:151-154 —
      the drafts' own KV is in the step's activations, not the offloaded cache);
  K3  the qtok sets taken as consecutive access_steps in one launch
      (``ess_pool_access_mtp``): recency is updated by every selected set (SPEC.md:298,
      the spec's stated choice for the paper's open question), misses of all sets
      appended into one per-request miss list;
  K4  one gather per micro-batch over those lists (a row missed by several tokens is
      fetched once: the later sets hit it);
  K5  attention over B * qtok query rows, row (b, j) over its own selection in pool b
      (``ESS_MLA_QTOK_SHIFT``);
  tail  admission of each request's accepted ids h .. h+m-1 (``ess_pool_admit`` with
      per-request m), their rows written back to host.

Every pool must hold all its tokens' selections at once (floor(rho * ctx) >= qtok * K),
so a later set's evictions never take a row an earlier token attends this step; the
C1-style oversize regime (cap < K) is served by the single-token layer.
"""

from __future__ import annotations

import math
import os
from types import SimpleNamespace

import numpy as np
import torch

from . import _lib
from .attention import SplitWorkspace, sparse_mla
from .cache import AccessBatch
from .decode import ROW, DSADecodeLayer, _e4m3, random_latent_rows
from .indexer import indexer_logits, indexer_logits_mtp, topk, topk_mtp
from .transfer import gather, gather_stream


class MTPDecodeLayer(DSADecodeLayer):
    """One offloaded DSA layer decoding ``mtp + 1`` query tokens per request and step."""

    def __init__(self, batch: int, context_len, sparse_ratio: float, topk_k: int = 2048,
                 mtp: int = 2, max_new_tokens: int = 16, device=None, seed: int = 0,
                 drift: float = 0.95, hugepages: bool = True):
        qtok = int(mtp) + 1
        if not 2 <= qtok <= _lib.MAX_QTOK:
            raise ValueError(f"mtp must be in [1, {_lib.MAX_QTOK - 1}]")
        # history headroom: up to qtok accepted ids per step
        super().__init__(batch, context_len, sparse_ratio, topk_k, max_new_tokens=max_new_tokens * qtok,
                         device=device, seed=seed, drift=drift, hugepages=hugepages, slot_format="f16")
        if self.cap0 < qtok * topk_k:
            raise ValueError(f"MTP needs every pool to hold all {qtok} tokens' selections: "
                             f"floor(rho * ctx) = {self.cap0} < {qtok} * {topk_k}")
        self.qtok, self.mtp = qtok, int(mtp)
        self.early_gather = False
        # streamed gathers (launched after each micro-batch's indexer, taking requests as
        # the cache manager publishes them): correct, but the spinning CTAs cost the later
        # indexer / top-k SMs (523 vs 490 us at C2 MTP = 2), so off by default
        self.stream_gather = os.environ.get("ESS_MTP_STREAM_GATHER", "0") == "1"
        B, d, g, Q = self.B, self.device, self.gen, qtok
        self._zi = torch.randn((B, Q, 64, 128), device=d, generator=g)
        self._za = torch.randn((B, Q, 128, 576), device=d, generator=g)
        # head weights: per request, the same for every position (as the single-token
        # layer keeps them across steps), so a position's selection does not depend on
        # which token slot of a step it occupies
        self.w = (torch.randn((B, 1, 64), device=d, generator=g) / 8.0).expand(B, Q, 64).contiguous()
        self.logits = torch.empty((B, Q, self.Lmax), dtype=torch.float32, device=d)
        self.idx = torch.empty((B, Q, topk_k), dtype=torch.int32, device=d)
        self.cnt = torch.empty((B, Q), dtype=torch.int32, device=d)
        self.sel_row = torch.empty((B, Q, topk_k), dtype=torch.int32, device=d)
        self.out = torch.empty((B, Q, 128, 512), dtype=torch.bfloat16, device=d)
        self.lse = torch.empty((B, Q, 128), dtype=torch.float32, device=d)
        # prefill windows: one query per position (token 0's indexer)
        self._logits1 = torch.empty((B, self.Lmax), dtype=torch.float32, device=d)
        self._idx1 = torch.empty((B, topk_k), dtype=torch.int32, device=d)
        self._cnt1 = torch.empty(B, dtype=torch.int32, device=d)

    def next_queries(self, advance=None):
        """(q_idx [B, qtok, 64, 128] e4m3, q [B, qtok, 128, 576] bf16) of the next step.

        The qtok tokens of a step are consecutive positions and a query is a function of
        its position, drifting between adjacent positions as consecutive decode steps do
        (Eq. (1)): q(p+1) = a q(p) + sqrt(1-a^2) eps.  A step starts ``advance[b]`` positions
        after the previous one (the previous step's accepted tokens, default 1): its first
        qtok - advance tokens are the previous step's last ones (same positions, same
        queries), the rest continue the chain."""
        B, Q, d = self.B, self.qtok, self.device
        adv = torch.ones(B, dtype=torch.long, device=d) if advance is None else \
            torch.as_tensor(np.asarray(advance), dtype=torch.long).to(d)
        if adv.shape != (B,) or int(adv.min()) < 1 or int(adv.max()) > Q:
            raise ValueError(f"advance must hold one value in [1, {Q}] per request")
        a = self.drift
        s = math.sqrt(max(0.0, 1.0 - a * a))
        rows = torch.arange(B, device=d)
        out = []
        for old in (self._zi, self._za):
            new = torch.empty_like(old)
            prev = old[:, Q - 1]
            for j in range(Q):
                src = j + adv
                chain = a * prev + s * torch.randn(prev.shape, device=d, generator=self.gen)
                keep = (src < Q).view(B, *([1] * (old.dim() - 2)))
                new[:, j] = torch.where(keep, old[rows, src.clamp(max=Q - 1)], chain)
                prev = new[:, j]
            out.append(new)
        self._zi, self._za = out
        return _e4m3(self._zi * 4.0), (self._za * 0.5).to(torch.bfloat16)

    def prefill_warmup(self, windows: int = 32, record: bool = False):
        rec = []
        w0 = self.w[:, 0].contiguous()
        for _ in range(windows):
            q_idx, _q = self.next_queries()
            indexer_logits(q_idx[:, 0].contiguous(), w0, self.k_cache, self.k_scale, self.lens,
                           out=self._logits1)
            topk(self._logits1, self.lens, self.K, out=self._idx1, count=self._cnt1)
            self.pool.warmup(self._idx1, self._cnt1)
            if record:
                rec.append([self._idx1[b, :int(self._cnt1[b])].cpu().numpy() for b in range(self.B)])
        self._fill_resident()
        return rec

    # -- the decode step -------------------------------------------------------------------
    def _view(self, a, b):
        acc = self.acc
        return AccessBatch(counts=acc.counts[a:b], sel_row=None, miss_ids=acc.miss_ids[a:b],
                           miss_row=acc.miss_row[a:b], hit_row=acc.hit_row[a:b])

    def attend(self, q_idx, q, gather_ctas: int = 32, overlap: str = "dba", new_rows=None,
               micro: int = 2):
        """K1..K5 for the qtok query tokens of every request.  ``overlap="dba"``: the
        requests in ``micro`` micro-batches; micro-batch i's gather (side stream) overlaps
        micro-batch i+1's indexer, whose grid leaves the gather its SMs.
        Attention is the paper's DA split per (request, token) row:
        pass 1 over the rows its selection found resident while the gathers run, pass 2
        over the rows fetched this step (by its own set or an earlier token's) once they
        have landed, merged through the workspace.  ``"da"``: one micro-batch.
        ``"none"``: K1 -> K2 -> K3 -> K4 -> K5 in order, one attention pass."""
        B, Q, K = self.B, self.qtok, self.K
        if self.acc is None:
            z = lambda: torch.empty((B, Q * K), dtype=torch.int32, device=self.device)  # noqa: E731
            self.acc = AccessBatch(counts=torch.empty((B, 4), dtype=torch.int32, device=self.device),
                                   sel_row=None, miss_ids=z(), miss_row=z(), hit_row=z())
            t = lambda: torch.empty((B, Q, K), dtype=torch.int32, device=self.device)  # noqa: E731
            self.tok_split = (t(), t(), torch.empty((B, Q, 2), dtype=torch.int32, device=self.device))
            self._ws = SplitWorkspace(B * Q, self.device)
        if overlap not in ("none", "da", "dba"):
            raise ValueError(f"unknown overlap schedule {overlap!r}")
        main = torch.cuda.current_stream(self.device)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device, priority=-1)
            self._sel = torch.cuda.Stream(self.device)
            self._attn = torch.cuda.Stream(self.device)
        side, sel, attn = self._side, self._sel, self._attn
        split = overlap != "none"
        qv, ov, lv = q.view(B * Q, 128, 576), self.out.view(B * Q, 128, 512), self.lse.view(B * Q, 128)
        if split:
            th, tf, tc = self.tok_split
            th, tf, tc = th.view(B * Q, K), tf.view(B * Q, K), tc.view(B * Q, 2)
        sms = torch.cuda.get_device_properties(self.device).multi_processor_count
        ranges = self.micro_batches(micro if overlap == "dba" else 1)
        # streamed gathers: each micro-batch's gather is launched as soon as its indexer is
        # done and takes each request's misses the moment the cache manager publishes them
        # (ready flags), so its CTAs are resident before that micro-batch's attention floods
        # the SMs (launched after the cache manager, a gather queued behind 2 x qtok
        # attention CTAs per request and ran at ~25 GB/s)
        streamed = split and self.stream_gather
        if streamed:
            if getattr(self, "_gsync", None) is None:
                self._gsync = torch.zeros(2 * B, dtype=torch.int32, device=self.device)  # ready | claim
                self._gsides = []
            while len(self._gsides) < len(ranges):
                self._gsides.append(torch.cuda.Stream(self.device, priority=-1))
            self._gsync.zero_()
            gready, gclaim = self._gsync[:B], self._gsync[B:]
        prev = 0
        for i, (a, b) in enumerate(ranges):
            # later micro-batches' indexer leaves SMs to the running gather and to the
            # previous micro-batch's top-k / cache manager (one CTA per request row)
            ctas = 0 if i == 0 else max(16, sms - max(gather_ctas, self.early_gather_sms) - prev)
            indexer_logits_mtp(q_idx[a:b], self.w[a:b], self.k_cache[a:b], self.k_scale[a:b],
                               self.lens[a:b], out=self.logits[a:b], max_ctas=ctas)
            scored = torch.cuda.Event()
            scored.record(main)
            g = gather_ctas if i == len(ranges) - 1 else max(gather_ctas, self.early_gather_sms)
            if streamed:
                gs = self._gsides[i]
                gs.wait_event(scored)
                with torch.cuda.stream(gs):
                    gather_stream(self.pool, self.store, self._view(a, b), gready[a:b], gclaim[a:b], None,
                                  begin=a, max_ctas=g)
                    fetched = torch.cuda.Event()
                    fetched.record(gs)
                side.wait_event(fetched)
            sel.wait_event(scored)
            with torch.cuda.stream(sel):
                topk_mtp(self.logits[a:b], self.lens[a:b], K, out=self.idx[a:b], count=self.cnt[a:b])
                self.pool.access_mtp(self.idx[a:b], self.cnt[a:b], begin=a, out=self._view(a, b),
                                     sel_row=self.sel_row[a:b],
                                     tok_split=None if overlap == "none" else
                                     tuple(x[a:b] for x in self.tok_split),
                                     ready=gready[a:b] if streamed else None)
                ready = torch.cuda.Event()
                ready.record(sel)
            if not streamed:
                side.wait_event(ready)
                with torch.cuda.stream(side):
                    # exclusive SMs: the host-link loads must not share an SM's miss
                    # tracking with the indexer or attention CTAs
                    gather(self.pool, self.store, self._view(a, b), begin=a, max_ctas=g, exclusive=True)
                    fetched = torch.cuda.Event()
                    fetched.record(side)
            if split:
                # this micro-batch's attention on its own stream, while later micro-batches
                # select and gather: pass 1 over its resident rows right after its cache
                # manager, pass 2 over its fetched rows once its gather has landed them
                r0, r1 = a * Q, b * Q
                ws = SimpleNamespace(o=self._ws.o[r0:r1], ml=self._ws.ml[r0:r1], splits=1)
                attn.wait_event(ready)
                with torch.cuda.stream(attn):
                    sparse_mla(self.pool, qv[r0:r1], th[r0:r1], tc[r0:r1, 0], self.sm_scale, pool_begin=a,
                               workspace=ws, mode="partial", qtok=Q)
                attn.wait_event(fetched)
                with torch.cuda.stream(attn):
                    sparse_mla(self.pool, qv[r0:r1], tf[r0:r1], tc[r0:r1, 1], self.sm_scale, pool_begin=a,
                               out=ov[r0:r1], lse=lv[r0:r1], workspace=ws, mode="resume", qtok=Q)
            prev = b - a   # one SM per request for its qtok top-k rows (in waves) and K3
        done = torch.cuda.Event()
        done.record(side)
        if not split:
            main.wait_event(done)
            sparse_mla(self.pool, qv, self.sel_row.view(B * Q, K), self.cnt.view(B * Q), self.sm_scale,
                       out=ov, lse=lv, qtok=Q)
            return self.out, self.lse
        attended = torch.cuda.Event()
        attended.record(attn)
        main.wait_event(attended)
        main.wait_event(done)
        return self.out, self.lse

    def step_counts(self) -> torch.Tensor:
        """[B, 4] access counts of the last step, summed over the qtok sets."""
        return self.acc.counts

    def _admit(self, new_rows: torch.Tensor, accepted: torch.Tensor) -> None:
        """The step's tail on device: per request grow to floor(rho * (h + m)), admit ids
        h..h+m-1 (m = accepted[b]), write their rows back to host and into their slots."""
        _lib.check(_lib.load().ess_pool_admit(
            self.pool.handle, 0, self.B, self.lens.data_ptr(), accepted.data_ptr(), float(self.rho),
            new_rows.data_ptr(), new_rows.stride(0) // ROW, self.store.pool_ptr(0),
            self.store.rows_per_pool, None, _lib.stream_handle()), "ess_pool_admit")

    def append_tokens(self, accepted, new_rows: torch.Tensor | None = None) -> None:
        """Eager tail: each request admits its ``accepted[b]`` (1..qtok) verified tokens."""
        acc = torch.as_tensor(accepted, dtype=torch.int32).to(self.device)
        if acc.shape != (self.B,) or int(acc.min()) < 1 or int(acc.max()) > self.qtok:
            raise ValueError(f"accepted must hold one count in [1, {self.qtok}] per request")
        self._check_room(int(acc.max()))
        if new_rows is None:
            new_rows = random_latent_rows(self.B * self.qtok, self.device, self.gen).view(self.B, self.qtok, ROW)
        self._admit(new_rows, acc)
        self.history += int(acc.max())

    def _check_room(self, m: int = None) -> None:
        m = self.qtok if m is None else m
        if self.history + m > self.Lmax:
            raise ValueError(f"decode step exceeds max_new_tokens: history {self.history} + {m} > Lmax {self.Lmax}")

    # -- whole-step CUDA graph ------------------------------------------------------------
    def _alloc_static(self) -> None:
        B, Q, d = self.B, self.qtok, self.device
        self.q_idx_in = torch.empty((B, Q, 64, 128), dtype=torch.uint8, device=d)
        self.q_in = torch.empty((B, Q, 128, 576), dtype=torch.bfloat16, device=d)
        self.rows_in = torch.zeros((B, Q, ROW), dtype=torch.uint8, device=d)
        self.accept_in = torch.ones(B, dtype=torch.int32, device=d)
        q_idx, q = self.next_queries()
        self.q_idx_in.copy_(q_idx)
        self.q_in.copy_(q)

    def _device_step(self, overlap: str, gather_ctas: int) -> None:
        self.attend(self.q_idx_in, self.q_in, gather_ctas=gather_ctas, overlap=overlap, micro=self.micro)
        self._admit(self.rows_in, self.accept_in)

    def launches_per_step(self, overlap: str) -> int:
        """K1, K2, K3, K4 per micro-batch, K5 (two passes per micro-batch unless "none"), and
        the admission."""
        micro = len(self.micro_batches(self.micro if overlap == "dba" else 1))
        return 4 * micro + (1 if overlap == "none" else 2 * micro) + 1

    def capture(self, overlap: str = "dba", gather_ctas: int = 32, accepted=None):
        """One eager step with ``accepted`` (default: qtok for every request), then the
        step recorded as a CUDA graph; ``step`` replays it."""
        d = self.device
        self._alloc_static()
        if accepted is not None:
            self.accept_in.copy_(torch.as_tensor(accepted, dtype=torch.int32))
        else:
            self.accept_in.fill_(self.qtok)
        m = int(self.accept_in.max())
        self._check_room(m)
        s = torch.cuda.Stream(d)
        s.wait_stream(torch.cuda.current_stream(d))
        with torch.cuda.stream(s):
            self._device_step(overlap, gather_ctas)
        torch.cuda.current_stream(d).wait_stream(s)
        torch.cuda.synchronize(d)
        eager_counts = self.step_counts().clone()
        self.history += m
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._device_step(overlap, gather_ctas)
        return eager_counts

    def step(self, q_idx: torch.Tensor, q: torch.Tensor, new_rows: torch.Tensor, accepted: torch.Tensor,
             max_accepted: int | None = None):
        """One MTP decode step through the captured graph.  ``accepted`` [B] int32 (device
        or pinned host): verified tokens per request, 1..qtok; ``max_accepted`` (its max,
        if the caller knows it without a sync) keeps the host's room check exact."""
        m = self.qtok if max_accepted is None else int(max_accepted)
        if not 1 <= m <= self.qtok:
            raise ValueError(f"max_accepted must be in [1, {self.qtok}]")
        if isinstance(accepted, torch.Tensor) and not accepted.is_cuda:
            if accepted.shape != (self.B,) or int(accepted.min()) < 1 or int(accepted.max()) > m:
                raise ValueError(f"accepted must hold one count in [1, {m}] per request")
        # device-resident counts are checked by the admission kernel (m > qtok latches
        # ESS_ERR_ARG; read by pool.check())
        self._check_room(m)
        pairs = [(self.q_idx_in, q_idx), (self.q_in, q), (self.rows_in, new_rows)]
        if isinstance(accepted, torch.Tensor) and accepted.is_cuda:
            pairs.append((self.accept_in, accepted))
        else:
            self.accept_in.copy_(torch.as_tensor(accepted, dtype=torch.int32), non_blocking=True)
        _lib.copy_many(pairs)
        self.graph.replay()
        self.history += m
        return self.out, self.lse


def draw_accepted(rng, batch: int, mean_accept: float, qtok: int):
    """Accepted tokens per request: Poisson(mean - 1) + 1 (trace.py:127), capped at the
    qtok tokens a step verifies."""
    a = rng.poisson(max(0.0, mean_accept - 1.0), size=batch).astype(np.int32) + 1
    return np.minimum(a, qtok).astype(np.int32)


__all__ = ["MTPDecodeLayer", "draw_accepted"]
