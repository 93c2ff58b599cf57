"""The CPU oracle chain that a decode layer's device state is mirrored against, step by
step (test infrastructure; oracle/ is the checker):

  * top-k: oracle/dsa.topk_indices on the GPU's own logits (bit-exact)
  * cache manager: the C restatement of offsim's SparsePool (oracle/lru_oracle.c),
    driven with the same selections — hit / miss counts every step, LRU order at the end
  * attention: fp64 sparse MLA over the HOST store's rows of the selected ids (so the
    gather / settle / admission path is covered too), on a sample of requests
  * indexer: fp64 logits on a sample of requests (rel 1e-3 of the row's max |logit|)
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import dsa
from oracle import lru as olru


class OracleChain:
    def __init__(self, layer, lens, windows, attn_sample=(), logit_sample=(), rel_tol=1e-2):
        from paper_2512_10576_b200.cache import pool_capacity
        self.layer, self.hist = layer, list(lens)
        self.rho, self.K = layer.rho, layer.K
        self.pool_capacity = pool_capacity
        self.orc = [olru.OraclePool(pool_capacity(self.rho, n)) for n in self.hist]
        for w in windows or []:
            for b, o in enumerate(self.orc):
                o.warmup([w[b].tolist()])
        self.attn_sample, self.logit_sample, self.rel_tol = list(attn_sample), list(logit_sample), rel_tol
        self.steps = 0
        self.hits = self.misses = 0

    def mirror(self, q=None, q_idx=None, counts=None):
        """Check the step that just ran (q / q_idx: its queries, for the sampled
        attention / indexer checks; counts: the access counts, default the layer's)."""
        L = self.layer
        torch.cuda.synchronize()
        logits = L.logits.cpu().numpy()
        idx, cnt = L.idx.cpu().numpy(), L.cnt.cpu().numpy()
        counts = (L.step_counts() if counts is None else counts).cpu().numpy()
        host = L.store.host.numpy() if (q is not None and self.attn_sample) else None
        for b in range(L.B):
            want = dsa.topk_indices(logits[b], self.hist[b], self.K)
            assert cnt[b] == len(want), (self.steps, b)
            np.testing.assert_array_equal(idx[b, :cnt[b]], want, err_msg=f"top-k step {self.steps} req {b}")
            r = self.orc[b].access_step(want.tolist())
            assert counts[b, 0] == len(r.hit_ids) and counts[b, 1] == len(r.miss_ids), \
                (self.steps, b, counts[b].tolist(), len(r.hit_ids), len(r.miss_ids))
            self.hits += len(r.hit_ids)
            self.misses += len(r.miss_ids)
            if q is not None and b in self.attn_sample:
                ref_o, ref_l = dsa.sparse_mla(q[b].float().cpu().numpy(), host[b, want], L.sm_scale)
                o = L.out[b].float().cpu().numpy()
                rel = np.linalg.norm(o - ref_o) / np.linalg.norm(ref_o)
                assert rel <= self.rel_tol, (self.steps, b, rel)
                assert np.abs(L.lse[b].cpu().numpy() - ref_l).max() <= 1e-2, (self.steps, b)
            if q_idx is not None and b in self.logit_sample:
                n = self.hist[b]
                ref = dsa.indexer_logits(q_idx[b].cpu().numpy(), L.w[b].cpu().numpy(),
                                         L.k_cache[b].cpu().numpy(), L.k_scale[b].cpu().numpy(), n)
                tol = 1e-3 * float(np.abs(ref).max()) + 1e-5
                assert np.abs(logits[b, :n] - ref).max() <= tol, (self.steps, b)
        for b, o in enumerate(self.orc):  # the step's tail: grow, then admit the new token
            self.hist[b] += 1
            o.grow_capacity(self.pool_capacity(self.rho, self.hist[b]))
            o.append_generated([self.hist[b] - 1])
        self.steps += 1

    def check_final(self):
        L = self.layer
        L.pool.check("oracle chain")
        out, cnt = L.pool.lru_order()
        out, cnt = out.cpu().numpy(), cnt.cpu().numpy()
        for b, o in enumerate(self.orc):
            assert out[b, :int(cnt[b])].tolist() == o.lru_order(), f"LRU order of request {b}"
        assert L.lens.tolist() == self.hist
