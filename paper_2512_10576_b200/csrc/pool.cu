// K3: on-device LRU latent-cache manager, plus K4 zero-copy miss gather and the
// generated-row write-back.  Replaces offsim.cache.SparsePool
// (/root/reference/pkg/src/offsim/cache.py:29-134) for P independent pools at once.
//
// Parallel contract (verified bit-exact against the reference):
//   * every pool keeps key[slot]: a free slot has key == slot index (< cap_max), a
//     resident slot a stamp from a strictly increasing clock (>= ESS_CLOCK_BASE);
//   * access, n <= cap (cache.py:112-118): hits (requested order) get stamps
//     clk.., then the nmiss smallest keys are selected (radix select) — free slots
//     first, then the least-recent residents that were NOT requested (hits were
//     just re-stamped above every old stamp) — and the j-th miss takes the j-th
//     selected slot (ascending slot index) with stamp clk+nhit+j;
//   * access, n > cap (cache.py:103-111): keep = requested[n-cap:], every other
//     resident is evicted (counted), kept misses take the freed slots, requested
//     ids before keep are transient (served from per-pool staging rows);
//   * warm-up (cache.py:73-88): same machinery with stamps in window order and
//     uncounted evictions; windows longer than cap get the exact "inserted" count
//     from a reuse-distance test;
//   * append (cache.py:122-134): per new id, the smallest key is either a free
//     slot or the LRU resident (evicted, counted).
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace {

constexpr int NT = 1024;                 // threads per pool CTA
constexpr int MAXR = ESS_MAX_REQUEST;    // 2048 ids per call
constexpr int EPT = MAXR / NT;           // elements per thread (contiguous)
constexpr int ROW_CHUNKS = ESS_LATENT_ROW_BYTES / 16;  // 41 x 16 B
#ifdef ESS_POOL_PROF  // scratch builds: per-phase globaltimer stamps of K3 (thread 0)
__device__ unsigned long long g_pool_prof[256][16];
#define PPROF(i)                                                              \
  do {                                                                        \
    __syncthreads();                                                          \
    if (threadIdx.x == 0 && blockIdx.x < 256) {                               \
      unsigned long long tt;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                  \
      g_pool_prof[blockIdx.x][i] = tt;                                        \
    }                                                                         \
  } while (0)
#else
#define PPROF(i) \
  do {           \
  } while (0)
#endif
constexpr int POOL_STAGED = 1 << 30;     // internal access flag: stage keys/slot ids in smem
constexpr size_t STAGE_SMEM_MAX = 180 * 1024;


enum { MODE_ACCESS = 0, MODE_WARMUP = 1 };

// MTP attention split (ess_pool_access_mtp): per selection set (request b, token j), the
// rows resident before the step ("hit", attention pass 1 beside the gather) and the rows
// fetched this step by this set or an earlier set of the request ("fresh", pass 2 after
// the gather), each in requested order; cnt [num][qtok][2].  Marks live in a per-launch
// shared-memory bitmap over the pool's slots.
struct TokSplit {
  int32_t *hit_row = nullptr;
  int32_t *fresh_row = nullptr;
  int32_t *cnt = nullptr;
  int32_t *ready = nullptr;  // per pool: set to 1 (release) once its lists and counts are out
};

struct StepSmem {
  int id[MAXR];
  int slot[MAXR];      // old slot (-1 = not resident), later the final row
  int sel[MAXR];       // selected / free slots, ascending
  int ev[MAXR];        // evicted ids (unsorted, then optionally sorted)
  unsigned char mark[MAXR];
  int hist[256];
  int warp[32];
  int scal[8];
};

struct PoolView {
  PoolMeta *meta;
  int32_t *slot_of;
  int32_t *slot_id;
  uint32_t *key;
  uint8_t *rows;
  int32_t *status;
  int64_t max_ids;
  int32_t cap_max;
  int32_t row_bytes;
  int32_t staging;
  int64_t rows_per_pool;
};

PoolView view(const ess_pool *p) {
  return PoolView{p->meta,   p->slot_of,   p->slot_id, p->key,     p->rows,         p->status,
                  p->max_ids, p->cap_max, p->row_bytes, p->staging, p->rows_per_pool};
}

// Histogram add with warp aggregation: lanes hitting the same bin add once (popc).
// Stamps are clustered (a recent clock window), so the high-digit passes would
// otherwise serialise 1024 shared-memory atomics on one or two bins.
__device__ __forceinline__ void hist_add_warp(int *hist, uint32_t bin, bool active) {
  const unsigned am = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  const unsigned peers = __match_any_sync(am, bin);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
}

// k-th smallest (1-based) of keys[0:cnt) — keys are unique, so exactly kth keys
// are <= the result.  4 passes of 8-bit digits, histogram in shared memory.
__device__ uint32_t select_kth_smallest(const uint32_t *__restrict__ keys, int cnt, int kth,
                                        StepSmem &sm) {
  uint32_t prefix = 0, mask = 0;
  int rem = kth;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += NT) sm.hist[i] = 0;
    __syncthreads();
    for (int s0 = 0; s0 < cnt; s0 += NT) {  // uniform trip count: warp-collective adds
      const int s = s0 + threadIdx.x;
      const uint32_t k = s < cnt ? keys[s] : 0u;
      hist_add_warp(sm.hist, (k >> shift) & 255u, s < cnt && (k & mask) == prefix);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int loc[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        loc[j] = sm.hist[lane * 8 + j];
        sum += loc[j];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int c = incl - sum;
      if (c < rem && rem <= incl) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
          if (c + loc[j] >= rem) {
            sm.scal[0] = lane * 8 + j;
            sm.scal[1] = rem - c;
            break;
          }
          c += loc[j];
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)sm.scal[0] << shift;
    mask |= 0xFFu << shift;
    rem = sm.scal[1];
    __syncthreads();
  }
  return prefix;
}

// k-th smallest (1-based) of the unique keys[0:cnt) via two passes of 11-bit digits
// over a narrow key range.  Free slots (key = slot index < ESS_CLOCK_BASE) come first
// in key order; they are counted, and the select then runs over whichever class holds
// the k-th key: the free slots (range < cap) or the residents, whose stamps span a
// recent clock window.  2048-bin histograms live in `h` (2048 ints of shared memory).
// Returns false (T untouched) when that class spans 2^22 or more; the caller then
// falls back to select_kth_smallest.
__device__ bool select_kth_narrow(const uint32_t *__restrict__ keys, int cnt, int kth, StepSmem &sm,
                                  int *h, uint32_t *T) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint32_t mn = 0xFFFFFFFFu, mx = 0u;
  int nfree = 0;
#pragma unroll 8
  for (int s = t; s < cnt; s += NT) {  // unrolled: keys may be in global memory (big pools)
    const uint32_t k = keys[s];
    if (k < ESS_CLOCK_BASE) {
      nfree++;
    } else {
      mn = min(mn, k);
      mx = max(mx, k);
    }
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  nfree = __reduce_add_sync(0xffffffffu, nfree);
  uint32_t *red = reinterpret_cast<uint32_t *>(sm.hist);  // [0,32) min, [32,64) max, [64,96) free
  if (lane == 0) {
    red[warp] = mn;
    red[32 + warp] = mx;
    red[64 + warp] = (uint32_t)nfree;
  }
  __syncthreads();
  mn = __reduce_min_sync(0xffffffffu, red[lane]);
  mx = __reduce_max_sync(0xffffffffu, red[32 + lane]);
  nfree = (int)__reduce_add_sync(0xffffffffu, red[64 + lane]);
  __syncthreads();  // red aliases the histogram zeroed below
  // the class holding the k-th key: [lo, hi] and the rank inside it
  uint32_t lo, hi;
  int rem = kth;
  if (kth <= nfree) {
    lo = 0;
    hi = ESS_CLOCK_BASE - 1;
    mx = (uint32_t)cnt;  // free keys are slot indices < cnt
  } else {
    lo = mn;
    hi = 0xFFFFFFFFu;
    rem = kth - nfree;
  }
  const uint32_t range = kth <= nfree ? (uint32_t)cnt : mx - mn;
  if (range >> 22) return false;  // uniform: every thread read the same values
  const int bits = 32 - __clz((int)(range | 1u));
  const int shift = bits > 11 ? bits - 11 : 0;
  uint32_t prefix = 0;
  for (int pass = 0; pass < (shift ? 2 : 1); pass++) {
    for (int i = t; i < 2048; i += NT) h[i] = 0;
    __syncthreads();
#pragma unroll 8
    for (int s = t; s < cnt; s += NT) {
      const uint32_t k = keys[s];
      const uint32_t rel = k - lo;
      const bool in = k >= lo && k <= hi;
      const bool on = in && (pass == 0 || (rel >> shift) == prefix);
      // plain atomics: 2048 bins spread the clustered stamps enough (merging equal-bin
      // lane runs or match_any aggregation measured slower here)
      if (on) atomicAdd(&h[pass == 0 ? rel >> shift : rel & ((1u << shift) - 1u)], 1);
    }
    __syncthreads();
    const int v0 = h[2 * t], v1 = h[2 * t + 1];
    int tot;
    const int ex = block_exclusive_scan<NT>(v0 + v1, sm.warp, &tot);
    if (ex < rem && rem <= ex + v0 + v1) {
      const bool first = rem <= ex + v0;
      sm.scal[0] = 2 * t + (first ? 0 : 1);
      sm.scal[1] = rem - ex - (first ? 0 : v0);
    }
    __syncthreads();
    prefix = pass == 0 ? (uint32_t)sm.scal[0] : (prefix << shift) | (uint32_t)sm.scal[0];
    rem = sm.scal[1];
    __syncthreads();
  }
  *T = lo + prefix;
  return true;
}

// Ascending slot indices s < cnt with keys[s] <= T into out[0:MAXR): warp ballots per
// 32-slot group, one block scan over the (chunk, warp) counts (in `c`, 2048 ints), a
// second ballot pass writes.  cnt <= 64 * NT.
__device__ void compact_le(const uint32_t *__restrict__ keys, int cnt, uint32_t T, StepSmem &sm,
                           int *c, int *out) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nch = (cnt + NT - 1) / NT;
  for (int ch = 0; ch < nch; ch++) {
    const int s = ch * NT + t;
    const unsigned bal = __ballot_sync(0xffffffffu, s < cnt && keys[s] <= T);
    if (lane == 0) c[ch * 32 + warp] = __popc(bal);
  }
  for (int i = nch * 32 + t; i < 2048; i += NT) c[i] = 0;
  __syncthreads();
  const int v0 = c[2 * t], v1 = c[2 * t + 1];
  int tot;
  const int ex = block_exclusive_scan<NT>(v0 + v1, sm.warp, &tot);
  c[2 * t] = ex;
  c[2 * t + 1] = ex + v0;
  __syncthreads();
  for (int ch = 0; ch < nch; ch++) {
    const int s = ch * NT + t;
    const bool f = s < cnt && keys[s] <= T;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const int pos = c[ch * 32 + warp] + __popc(bal & ((1u << lane) - 1u));
    if (f && pos < MAXR) out[pos] = s;
  }
}

// Ascending bitonic sort of sm.ev[0:n), n <= MAXR.
__device__ void sort_ids(StepSmem &sm, int n) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + threadIdx.x; i < m; i += NT) sm.ev[i] = 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += NT) {
        int l = i ^ j;
        if (l > i) {
          int a = sm.ev[i], b = sm.ev[l];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            sm.ev[i] = b;
            sm.ev[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ void copy_row(const uint8_t *src, uint8_t *dst, int lane, int bytes) {
  // every load of the row first, then the stores: one memory round trip per row, not
  // one per 512-B chunk (rows up to 1536 B; longer rows loop)
  const int n16 = bytes / 16;
  for (int c0 = 0; c0 < n16; c0 += 96) {
    uint4 v[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const int c = c0 + lane + 32 * k;
      if (c < n16) v[k] = __ldcg(reinterpret_cast<const uint4 *>(src) + c);
    }
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const int c = c0 + lane + 32 * k;
      if (c < n16) reinterpret_cast<uint4 *>(dst)[c] = v[k];
    }
  }
}

// One 656-B latent row held by a warp (lane l: chunk l in v0; lanes 0..8: chunk
// 32+l in v1 — lane 0 has the four f32 group scales, lanes 1..8 the RoPE) ->
// the 1152-B f16 slot row.  NoPE: f16(f32(e4m3) * scale), RoPE: f16(bf16) — both
// single roundings, so the slot row is a pure function of the latent row.
__device__ __forceinline__ bool dequant_row_to_slot(uint4 v0, uint4 v1, int lane, uint8_t *dst) {
  const float s0 = __uint_as_float(__shfl_sync(0xffffffffu, v1.x, 0));
  const float s1 = __uint_as_float(__shfl_sync(0xffffffffu, v1.y, 0));
  const float s2 = __uint_as_float(__shfl_sync(0xffffffffu, v1.z, 0));
  const float s3 = __uint_as_float(__shfl_sync(0xffffffffu, v1.w, 0));
  const int g = lane >> 3;
  const float s = g == 0 ? s0 : g == 1 ? s1 : g == 2 ? s2 : s3;
  uint4 a, c;
  a.x = e4m3x2_scaled_f16x2((uint16_t)(v0.x & 0xFFFF), s);
  a.y = e4m3x2_scaled_f16x2((uint16_t)(v0.x >> 16), s);
  a.z = e4m3x2_scaled_f16x2((uint16_t)(v0.y & 0xFFFF), s);
  a.w = e4m3x2_scaled_f16x2((uint16_t)(v0.y >> 16), s);
  c.x = e4m3x2_scaled_f16x2((uint16_t)(v0.z & 0xFFFF), s);
  c.y = e4m3x2_scaled_f16x2((uint16_t)(v0.z >> 16), s);
  c.z = e4m3x2_scaled_f16x2((uint16_t)(v0.w & 0xFFFF), s);
  c.w = e4m3x2_scaled_f16x2((uint16_t)(v0.w >> 16), s);
  st_v4(dst + lane * 32, a);
  st_v4(dst + lane * 32 + 16, c);
  bool bad = f16x8_nonfinite(a) | f16x8_nonfinite(c);
  if (lane >= 1 && lane <= 8) {
    const uint4 r = cvt8_bf16_f16(v1);
    st_v4(dst + 1024 + (lane - 1) * 16, r);
    bad |= f16x8_nonfinite(r);
  }
  return bad;  // this lane wrote a value outside the f16 range
}

// The slot row of a 656-B latent row held by a warp, in the pool's slot format: the raw
// row (ESS_SLOT_ROW_BYTES_FP8: K5 dequantises in shared memory) or the dequantised f16
// row (ESS_SLOT_ROW_BYTES).
// Returns true if this lane stored an f16 value outside the f16 range (the caller
// latches ESS_ERR_RANGE).
__device__ __forceinline__ bool store_slot_row(uint4 v0, uint4 v1, int lane, uint8_t *dst, int row_bytes) {
  if (row_bytes == ESS_SLOT_ROW_BYTES_FP8) {
    st_v4(dst + lane * 16, v0);
    if (lane + 32 < ESS_LATENT_ROW_BYTES / 16) st_v4(dst + (lane + 32) * 16, v1);
    return false;
  }
  return dequant_row_to_slot(v0, v1, lane, dst);
}

template <int MODE>
__global__ void __launch_bounds__(NT, 1)
    pool_step_kernel(PoolView pv, int begin, const int32_t *__restrict__ req,
                     const int32_t *__restrict__ req_n, int req_stride, int32_t *hit_out,
                     int32_t *miss_out, int32_t *ev_out, int32_t *sel_row_out,
                     int32_t *hit_row_out, int32_t *miss_row_out, int32_t *counts_out,
                     int out_stride, int flags,
                     int64_t *inserted_out, int qtok, int sel_stride, TokSplit ts) {
  __shared__ StepSmem sm;
  extern __shared__ uint32_t stage_smem[];  // [cap_max] keys (STAGED)
  const int t = threadIdx.x;
  const int b = blockIdx.x;
  const int p = begin + b;
  PoolMeta *meta = pv.meta + p;
  int32_t *slot_of = pv.slot_of + (int64_t)p * pv.max_ids;
  int32_t *slot_id = pv.slot_id + (int64_t)p * pv.cap_max;
  uint32_t *key = pv.key + (int64_t)p * pv.cap_max;
  // MTP (qtok > 1): the pool takes its request's qtok selection sets one after another,
  // each a full access_step (recency updated by every selected set); the
  // hit / miss / evicted lists of the sets are appended per pool, the counts summed.
  int acc_hit = 0, acc_miss = 0, acc_ev = 0, acc_tr = 0;
  uint32_t *fresh_bits = stage_smem + ((flags & POOL_STAGED) ? pv.cap_max : 0);  // TokSplit marks
  if (ts.hit_row) {
    for (int w = t; w < (pv.cap_max + 31) / 32; w += NT) fresh_bits[w] = 0u;
    __syncthreads();
  }
  for (int jq = 0; jq < qtok; jq++) {
  const int n = req_n[(int64_t)b * qtok + jq];
  const int32_t *reqj = req + ((int64_t)b * qtok + jq) * req_stride;
  const int cap = meta->cap;
  const int size0 = meta->size;
  const uint32_t clk = meta->clk;
  const int64_t out_base = (int64_t)b * out_stride;
  const int64_t sel_base = ((int64_t)b * qtok + jq) * sel_stride;
  PPROF(0);
  // STAGED: the pool's keys are copied to shared memory once, so the victim
  // select's passes and its compaction read on-chip
  // instead of paying an HBM round trip per pass (the state is evicted from L2 by
  // the indexer stream between steps).  Global copies stay authoritative: every
  // write below goes to both.
  const bool staged = (flags & POOL_STAGED) != 0;
  uint32_t *skey = stage_smem;
  const uint32_t *kread = staged ? skey : key;
  const int32_t *sread = slot_id;

  // ---- load + validate -------------------------------------------------------
  bool bad = n < 0 || n > MAXR || (uint64_t)clk + (uint64_t)n > 0xFFFFFF00ull;
  int hflag[EPT], xs[EPT];
#pragma unroll
  for (int e = 0; e < EPT; e++) {
    const int i = t * EPT + e;
    xs[e] = (!bad && i < n) ? reqj[i] : 0;
  }
  // the key staging loads go out while the requested ids are in flight
  if (staged && jq == 0) {
#pragma unroll 4
    for (int s2 = t; s2 < cap; s2 += NT) skey[s2] = key[s2];
  }
#pragma unroll
  for (int e = 0; e < EPT; e++) {
    int i = t * EPT + e;
    hflag[e] = 0;
    if (!bad && i < n) {
      int x = xs[e];
      if (x < 0 || x >= pv.max_ids) {
        bad = true;
      } else {
        sm.id[i] = x;
        int s = slot_of[x];
        sm.slot[i] = s;
        hflag[e] = s >= 0;
      }
    }
  }
  if (__syncthreads_or(bad)) {
    if (t == 0) ess_set_status(pv.status, (n > MAXR || n < 0) ? ESS_ERR_ARG
                                          : ((uint64_t)clk + (uint64_t)n > 0xFFFFFF00ull)
                                              ? ESS_ERR_CLOCK
                                              : ESS_ERR_ARG);
    if (ts.ready && t == 0) {  // a waiting gather must not spin: publish an empty list
      if (counts_out) counts_out[b * 4 + 1] = 0;
      __threadfence();
      ess_st_release(ts.ready + b, 1);
    }
    return;
  }

  PPROF(1);
  // ---- hit / miss split in requested order (cache.py:98-99) ---------------------
  int nh_local = 0;
#pragma unroll
  for (int e = 0; e < EPT; e++) nh_local += hflag[e];
  int nhit;
  int hr = block_exclusive_scan<NT>(nh_local, sm.warp, &nhit);
  const int nmiss = n - nhit;
  int hrank[EPT], mrank[EPT];
#pragma unroll
  for (int e = 0; e < EPT; e++) {
    int i = t * EPT + e;
    hrank[e] = hr;
    mrank[e] = i - hr;
    if (i < n) {
      if (hflag[e]) {
        if (MODE == MODE_ACCESS && hit_out) hit_out[out_base + acc_hit + hr] = sm.id[i];
        hr++;
      } else if (MODE == MODE_ACCESS && miss_out) {
        miss_out[out_base + acc_miss + (i - hrank[e])] = sm.id[i];
      }
    }
  }

  PPROF(2);
  int nev = 0;
  int64_t inserted = 0;
  if (MODE == MODE_WARMUP) {
    // Warm-up touches in window order (cache.py:79-87), so a resident x at window
    // position i may be evicted by the earlier touches before its own: that happens
    // iff the distinct ids touched after x's old stamp fill the pool, i.e.
    //   r_x < i - B_x - free      r_x = #residents older than x (LRU rank)
    //                             B_x = #{j < i : W[j] resident and newer than x}
    //                             free = cap - size
    // and x then counts as inserted.  Only ranks below D = n-1-free matter, so the
    // D oldest residents are located by radix select and ranked by brute force.
    const int free0 = cap - size0;
    const int D = n - 1 - free0;
    int extra = 0;
    if (D > 0 && nhit > 0 && size0 > 0) {
      const int kk = D < size0 ? D : size0;
      const uint32_t Tstar = select_kth_smallest(key, cap, free0 + kk, sm);
      uint32_t *cand = reinterpret_cast<uint32_t *>(sm.ev);   // <= kk resident stamps
      uint32_t *pkey = reinterpret_cast<uint32_t *>(sm.sel);  // old stamp by position
      int base = 0;
      for (int s0 = 0; s0 < cap; s0 += NT) {
        int s = s0 + t;
        uint32_t k = s < cap ? key[s] : 0xFFFFFFFFu;
        int f = (s < cap && k <= Tstar && slot_id[s] >= 0) ? 1 : 0;
        int tot;
        int pos = block_exclusive_scan<NT>(f, sm.warp, &tot);
        if (f && base + pos < MAXR) cand[base + pos] = k;
        base += tot;
      }
      const int ncand = base < MAXR ? base : MAXR;
#pragma unroll
      for (int e = 0; e < EPT; e++) {
        int i = t * EPT + e;
        if (i < n) pkey[i] = hflag[e] ? key[sm.slot[i]] : 0u;
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < EPT; e++) {
        int i = t * EPT + e;
        if (i >= n || !hflag[e] || i - free0 <= 0) continue;
        const uint32_t sx = pkey[i];
        if (sx > Tstar) continue;  // rank >= D: cannot be evicted in this window
        int r = 0, B = 0;
        for (int c = 0; c < ncand; c++) r += cand[c] < sx;
        for (int j = 0; j < i; j++) B += pkey[j] > sx;
        extra += (r < i - B - free0);
      }
      __syncthreads();
    }
    int tot;
    block_exclusive_scan<NT>(extra, sm.warp, &tot);
    inserted = (int64_t)nmiss + tot;
  }
  if (n <= cap) {
    // ---- normal path (cache.py:112-118; warm-up windows <= cap, cache.py:79-87) --
#pragma unroll
    for (int e = 0; e < EPT; e++) {
      int i = t * EPT + e;
      if (i < n && hflag[e]) {
        const uint32_t st = (MODE == MODE_ACCESS) ? clk + hrank[e] : clk + i;
        key[sm.slot[i]] = st;
        if (staged) skey[sm.slot[i]] = st;
      }
    }
    __syncthreads();
    PPROF(3);
    if (nmiss > 0) {
      // sm.ev is free until the victims are listed: it serves as the 2048-bin
      // histogram of the narrow select and the count table of the compaction
      uint32_t T;
      if (!select_kth_narrow(kread, cap, nmiss, sm, sm.ev, &T)) T = select_kth_smallest(kread, cap, nmiss, sm);
      PPROF(4);
      // the nmiss selected slots in ascending order (exactly nmiss keys are <= T)
      if (cap <= 64 * NT) {
        compact_le(kread, cap, T, sm, sm.ev, sm.sel);
      } else {  // very large pools: contiguous runs per thread, still one block scan
        const int per = (cap + NT - 1) / NT;
        const int s0 = min(cap, t * per), s1 = min(cap, s0 + per);
        int f = 0;
#pragma unroll 8
        for (int s2 = s0; s2 < s1; s2++) f += kread[s2] <= T;
        int tot;
        int pos = block_exclusive_scan<NT>(f, sm.warp, &tot);
        for (int s2 = s0; s2 < s1 && f > 0; s2++) {
          if (kread[s2] <= T) {
            if (pos < MAXR) sm.sel[pos] = s2;
            pos++;
            f--;
          }
        }
      }
      __syncthreads();
      PPROF(5);
      // victims: selected slots that were occupied (least recent first is not needed:
      // the set is what matters, evicted_ids is reported sorted, cache.py:120)
      int ef[EPT], eid[EPT], ne_local = 0;
#pragma unroll
      for (int e = 0; e < EPT; e++) {
        int j = t * EPT + e;
        ef[e] = 0;
        if (j < nmiss) {
          int old = sread[sm.sel[j]];
          eid[e] = old;
          ef[e] = old >= 0;
          ne_local += ef[e];
        }
      }
      int epos = block_exclusive_scan<NT>(ne_local, sm.warp, &nev);
#pragma unroll
      for (int e = 0; e < EPT; e++) {
        if (ef[e]) {
          sm.ev[epos++] = eid[e];
          slot_of[eid[e]] = -1;
        }
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < EPT; e++) {
        int i = t * EPT + e;
        if (i < n && !hflag[e]) {
          int j = mrank[e];
          int s = sm.sel[j];
          slot_of[sm.id[i]] = s;
          slot_id[s] = sm.id[i];
          const uint32_t st = (MODE == MODE_ACCESS) ? clk + nhit + j : clk + i;
          key[s] = st;
          if (staged) skey[s] = st;  // the staged copy stays exact for the next MTP set
          if (ts.hit_row) atomicOr(&fresh_bits[s >> 5], 1u << (s & 31));
          sm.slot[i] = s;
          if (MODE == MODE_ACCESS && miss_row_out) miss_row_out[out_base + acc_miss + j] = s;
        }
      }
    }
  } else {
    // ---- oversize path: keep requested[n-cap:] (cache.py:103-111) -----------------
    const int keep0 = n - cap;  // cap < n <= MAXR, so every slot index < MAXR
    if (MODE == MODE_ACCESS && pv.rows && keep0 > pv.staging && t == 0)
      ess_set_status(pv.status, ESS_ERR_ARG);  // not enough staging rows for transients
    for (int s = t; s < MAXR; s += NT) sm.mark[s] = 0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < EPT; e++) {
      int i = t * EPT + e;
      if (i >= keep0 && i < n && hflag[e]) sm.mark[sm.slot[i]] = 1;
    }
    __syncthreads();
    // transient requested-but-not-kept residents: preserve their rows in staging
    // before their slots are reused (the attention kernel reads them this step)
    if (MODE == MODE_ACCESS && pv.rows) {
      const int warp = t >> 5, lane = t & 31;
      uint8_t *rbase = pv.rows + (int64_t)p * pv.rows_per_pool * pv.row_bytes;
      for (int i = warp; i < keep0; i += NT / 32) {
        int s = sm.slot[i];
        if (s >= 0)
          copy_row(rbase + (int64_t)s * pv.row_bytes,
                   rbase + (int64_t)(pv.cap_max + i) * pv.row_bytes, lane, pv.row_bytes);
      }
    }
    // evict every resident outside keep; the freed slots (ascending) host kept misses
    int ebase = 0, fbase = 0;
    for (int s0 = 0; s0 < cap; s0 += NT) {
      int s = s0 + t;
      int freef = (s < cap && !sm.mark[s]) ? 1 : 0;
      int old = freef ? slot_id[s] : -1;
      int evf = old >= 0 ? 1 : 0;
      int etot, ftot;
      int ep = block_exclusive_scan<NT>(evf, sm.warp, &etot);
      int fp = block_exclusive_scan<NT>(freef, sm.warp, &ftot);
      if (evf) {
        sm.ev[ebase + ep] = old;
        slot_of[old] = -1;
        slot_id[s] = -1;
      }
      if (freef) sm.sel[fbase + fp] = s;
      ebase += etot;
      fbase += ftot;
    }
    nev = ebase;
    __syncthreads();
    int km_local = 0;
#pragma unroll
    for (int e = 0; e < EPT; e++) {
      int i = t * EPT + e;
      km_local += (i >= keep0 && i < n && !hflag[e]);
    }
    int kmtot;
    int km = block_exclusive_scan<NT>(km_local, sm.warp, &kmtot);
#pragma unroll
    for (int e = 0; e < EPT; e++) {
      int i = t * EPT + e;
      if (i >= n) continue;
      if (i >= keep0) {
        int s;
        if (hflag[e]) {
          s = sm.slot[i];
        } else {
          s = sm.sel[km++];
          slot_of[sm.id[i]] = s;
          slot_id[s] = sm.id[i];
          if (ts.hit_row) atomicOr(&fresh_bits[s >> 5], 1u << (s & 31));
        }
        const uint32_t st = (MODE == MODE_ACCESS) ? clk + (i - keep0) : clk + i;
        key[s] = st;
        if (staged) skey[s] = st;
        sm.slot[i] = s;
      } else {
        sm.slot[i] = pv.cap_max + i;  // transient: staging row
      }
      if (MODE == MODE_ACCESS && miss_row_out && !hflag[e]) miss_row_out[out_base + acc_miss + mrank[e]] = sm.slot[i];
    }
  }
  __syncthreads();

  PPROF(6);
  // ---- outputs + counters -----------------------------------------------------
  if (MODE == MODE_ACCESS && ts.hit_row) {  // MTP attention split of this set
    int fr[EPT], nf = 0, nh = 0;
#pragma unroll
    for (int e = 0; e < EPT; e++) {
      const int i = t * EPT + e;
      fr[e] = 0;
      if (i < n) {
        const int sl = sm.slot[i];
        // staging rows (oversize transients) were fetched this step too
        fr[e] = sl >= pv.cap_max ? 1 : (int)((fresh_bits[sl >> 5] >> (sl & 31)) & 1u);
        nf += fr[e];
        nh += 1 - fr[e];
      }
    }
    int tot;
    const int ex = block_exclusive_scan<NT>(nh | (nf << 16), sm.warp, &tot);
    int ph = ex & 0xFFFF, pf = ex >> 16;
    const int64_t rb = ((int64_t)b * qtok + jq) * sel_stride;
#pragma unroll
    for (int e = 0; e < EPT; e++) {
      const int i = t * EPT + e;
      if (i < n) {
        if (fr[e]) ts.fresh_row[rb + pf++] = sm.slot[i];
        else ts.hit_row[rb + ph++] = sm.slot[i];
      }
    }
    if (t == 0) {
      ts.cnt[((int64_t)b * qtok + jq) * 2 + 0] = tot & 0xFFFF;
      ts.cnt[((int64_t)b * qtok + jq) * 2 + 1] = tot >> 16;
    }
  }
  if (MODE == MODE_ACCESS) {
    if (sel_row_out) {
#pragma unroll
      for (int e = 0; e < EPT; e++) {
        int i = t * EPT + e;
        if (i < n) sel_row_out[sel_base + i] = sm.slot[i];
      }
    }
    if (hit_row_out) {  // rows already resident before this step (attention pass 1)
#pragma unroll
      for (int e = 0; e < EPT; e++) {
        int i = t * EPT + e;
        if (i < n && hflag[e]) hit_row_out[out_base + acc_hit + hrank[e]] = sm.slot[i];
      }
    }
    if (ev_out) {
      if (flags & ESS_ACCESS_SORT_EVICTED) sort_ids(sm, nev);
      for (int j = t; j < nev; j += NT) ev_out[out_base + acc_ev + j] = sm.ev[j];
    }
  }
  PPROF(7);
  if (t == 0) {
    if (MODE == MODE_ACCESS) {
      meta->hits += nhit;
      meta->misses += nmiss;
      meta->evictions += nev;
      if (counts_out && jq == qtok - 1) {
        counts_out[b * 4 + 0] = acc_hit + nhit;
        counts_out[b * 4 + 1] = acc_miss + nmiss;
        counts_out[b * 4 + 2] = acc_ev + nev;
        counts_out[b * 4 + 3] = acc_tr + (n > cap ? n - cap : 0);
      }
    } else if (inserted_out) {
      inserted_out[b] += inserted;
    }
    if (n <= cap) {
      meta->clk = clk + n;
      meta->size = size0 + nmiss - nev;
    } else {
      meta->clk = clk + n;
      meta->size = cap;
    }
  }
  acc_hit += nhit;
  acc_miss += nmiss;
  acc_ev += nev;
  acc_tr += n > cap ? n - cap : 0;
  __syncthreads();  // the next set reads the pool state (meta, keys) this one wrote
  }  // jq
  if (ts.ready) {  // a concurrent streamed gather takes this pool's misses from here on
    __threadfence();
    __syncthreads();
    if (t == 0) ess_st_release(ts.ready + b, 1);
  }
}

__global__ void pool_reset_kernel(PoolView pv, int begin, int num, const int32_t *cap) {
  // grid: (num, y) — y-blocks stride over the per-pool arrays
  const int b = blockIdx.x, p = begin + b;
  const int c = cap[b];
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    if (c < 1 || c > pv.cap_max) {
      ess_set_status(pv.status, ESS_ERR_CAPACITY);
    }
    PoolMeta m;
    memset(&m, 0, sizeof(m));
    m.cap = (c < 1 || c > pv.cap_max) ? 1 : c;
    m.clk = ESS_CLOCK_BASE;
    m.watermark = -1;
    pv.meta[p] = m;
  }
  int32_t *so = pv.slot_of + (int64_t)p * pv.max_ids;
  for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < pv.max_ids;
       i += (int64_t)gridDim.y * blockDim.x)
    so[i] = -1;
  int32_t *sid = pv.slot_id + (int64_t)p * pv.cap_max;
  uint32_t *k = pv.key + (int64_t)p * pv.cap_max;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < pv.cap_max; i += gridDim.y * blockDim.x) {
    sid[i] = -1;
    k[i] = (uint32_t)i;
  }
}

__global__ void pool_grow_kernel(PoolView pv, int begin, int num, const int32_t *cap) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= num) return;
  PoolMeta *m = pv.meta + begin + b;
  int c = cap[b];
  if (c < m->cap) {
    ess_set_status(pv.status, ESS_ERR_SHRINK);
  } else if (c > pv.cap_max) {
    ess_set_status(pv.status, ESS_ERR_CAPACITY);
  } else {
    m->cap = c;
  }
}

constexpr int NTA = 256;

// block-wide argmin of key[0:cap) -> slot (keys unique)
__device__ int argmin_key(const uint32_t *key, int cap, unsigned long long *red) {
  // 16-B loads, several in flight per thread: the scan is latency-bound otherwise
  // (the key array sits in HBM; the indexer stream evicts it from L2 every step).
  // Plain (coherent) loads: thread 0 rewrites a key between the scans of one launch.
  unsigned long long best = ~0ull;
  const int head = min(cap, (int)((4 - ((reinterpret_cast<uintptr_t>(key) >> 2) & 3)) & 3));
  const int body = (cap - head) & ~3;
  if ((int)threadIdx.x < head) {
    unsigned long long v = ((unsigned long long)key[threadIdx.x] << 32) | threadIdx.x;
    best = v < best ? v : best;
  }
  const uint4 *k4 = reinterpret_cast<const uint4 *>(key + head);
#pragma unroll 4
  for (int j = threadIdx.x * 4; j < body; j += NTA * 4) {
    const uint4 q = k4[j >> 2];
    const unsigned s = (unsigned)(head + j);
    const unsigned long long v0 = ((unsigned long long)q.x << 32) | s;
    const unsigned long long v1 = ((unsigned long long)q.y << 32) | (s + 1);
    const unsigned long long v2 = ((unsigned long long)q.z << 32) | (s + 2);
    const unsigned long long v3 = ((unsigned long long)q.w << 32) | (s + 3);
    const unsigned long long a = v0 < v1 ? v0 : v1, c = v2 < v3 ? v2 : v3;
    const unsigned long long m = a < c ? a : c;
    best = m < best ? m : best;
  }
  for (int s = head + body + threadIdx.x; s < cap; s += NTA) {
    unsigned long long v = ((unsigned long long)key[s] << 32) | (unsigned)s;
    best = v < best ? v : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y < best ? y : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long v = red[0];
    for (int w = 1; w < NTA / 32; w++) v = red[w] < v ? red[w] : v;
    red[NTA / 32] = v;
  }
  __syncthreads();
  int s = (int)(red[NTA / 32] & 0xffffffffu);
  __syncthreads();
  return s;
}

// cache.py:122-134 — validation of all ids first, then per id: evict the LRU if
// full (counted), touch.  Sequential over the (few) generated ids of a step.
__global__ void __launch_bounds__(NTA) pool_append_kernel(PoolView pv, int begin,
                                                         const int32_t *ids, const int32_t *m,
                                                         int stride, int32_t *slot_out) {
  __shared__ unsigned long long red[NTA / 32 + 1];
  const int b = blockIdx.x, p = begin + b;
  const int M = m[b];
  PoolMeta *meta = pv.meta + p;
  int32_t *slot_of = pv.slot_of + (int64_t)p * pv.max_ids;
  int32_t *slot_id = pv.slot_id + (int64_t)p * pv.cap_max;
  uint32_t *key = pv.key + (int64_t)p * pv.cap_max;
  const int64_t wm = meta->watermark;
  uint32_t clk = meta->clk;
  int code = 0;
  if (M < 0 || (uint64_t)clk + (uint64_t)(M < 0 ? 0 : M) > 0xFFFFFF00ull) code = ESS_ERR_ARG;
  for (int i = threadIdx.x; code == 0 && i < M; i += NTA) {
    int x = ids[(int64_t)b * stride + i];
    if (x < 0 || x >= pv.max_ids) code = ESS_ERR_ARG;
    else if (slot_of[x] >= 0 || (int64_t)x <= wm) code = ESS_ERR_DUPLICATE;
  }
  if (__syncthreads_or(code != 0)) {
    if (code && threadIdx.x == 0) ess_set_status(pv.status, code);
    if (code) ess_set_status(pv.status, code);
    return;
  }
  const int cap = meta->cap;
  int size = meta->size;
  int64_t evictions = 0, w = wm;
  for (int i = 0; i < M; i++) {
    const int x = ids[(int64_t)b * stride + i];
    int s = -1;
    if (size >= cap) {
      s = argmin_key(key, cap, reinterpret_cast<unsigned long long *>(red));
      if (threadIdx.x == 0) {
        int old = slot_id[s];
        slot_of[old] = -1;
        slot_id[s] = -1;
        key[s] = (uint32_t)s;
      }
      size--;
      evictions++;
      __syncthreads();
    }
    int cur = slot_of[x];
    __syncthreads();
    if (cur >= 0) {  // duplicate inside this call: refresh only (cache.py:132 touch)
      if (threadIdx.x == 0) key[cur] = clk;
      s = cur;
    } else {
      if (s < 0) s = argmin_key(key, cap, reinterpret_cast<unsigned long long *>(red));
      if (threadIdx.x == 0) {
        slot_of[x] = s;
        slot_id[s] = x;
        key[s] = clk;
      }
      size++;
    }
    clk++;
    if (x > w) w = x;
    if (slot_out && threadIdx.x == 0) slot_out[(int64_t)b * stride + i] = s;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    meta->size = size;
    meta->clk = clk;
    meta->watermark = w;
    meta->evictions += evictions;
  }
}

// rank of each resident by stamp = its LRU position (cache.py:55-57)
__global__ void pool_lru_order_kernel(PoolView pv, int begin, int32_t *out, int32_t *count) {
  __shared__ uint32_t tile[256];
  const int b = blockIdx.x, p = begin + b;
  const int cap = pv.meta[p].cap;
  const int32_t *slot_id = pv.slot_id + (int64_t)p * pv.cap_max;
  const uint32_t *key = pv.key + (int64_t)p * pv.cap_max;
  const int s = blockIdx.y * 256 + threadIdx.x;
  const bool valid = s < cap && slot_id[s] >= 0;
  const uint32_t mk = valid ? key[s] : 0xFFFFFFFFu;
  int rank = 0;
  for (int t0 = 0; t0 < cap; t0 += 256) {
    int u = t0 + threadIdx.x;
    tile[threadIdx.x] = (u < cap && slot_id[u] >= 0) ? key[u] : 0xFFFFFFFFu;
    __syncthreads();
    int lim = min(256, cap - t0);
    for (int j = 0; j < lim; j++) rank += tile[j] < mk;
    __syncthreads();
  }
  if (valid) out[(int64_t)b * pv.cap_max + rank] = slot_id[s];
  if (blockIdx.y == 0 && threadIdx.x == 0) count[b] = pv.meta[p].size;
}

// ---- early-gather split of K3 -----------------------------------------------------
// "K3a": the hit/miss split alone (read-only on the LRU state: one slot_of lookup per
// requested id).  Misses are pointed at per-pool staging rows cap_max + j, so the host
// link gather can start before victim selection; the full access ("K3b") then updates
// the LRU state exactly as one access would and reports each miss's final slot, and a
// settle pass moves the fetched rows from staging into those slots.  Victims are never
// requested ids (n <= cap), so K5 reads hits in place and misses from staging while
// the settle writes only victim slots.
__global__ void __launch_bounds__(NT) pool_split_kernel(PoolView pv, int begin,
                                                        const int32_t *__restrict__ req,
                                                        const int32_t *__restrict__ req_n,
                                                        int req_stride, int32_t *hit_row_out,
                                                        int32_t *miss_out, int32_t *miss_row_out,
                                                        int32_t *counts_out, int out_stride) {
  __shared__ int wbuf[NT / 32];
  const int t = threadIdx.x, b = blockIdx.x, p = begin + b;
  const int n = min(max(req_n[b], 0), MAXR);
  const int32_t *slot_of = pv.slot_of + (int64_t)p * pv.max_ids;
  int x[EPT], s[EPT], h = 0;
#pragma unroll
  for (int e = 0; e < EPT; e++) {
    const int i = t * EPT + e;
    x[e] = i < n ? req[(int64_t)b * req_stride + i] : -1;
  }
#pragma unroll
  for (int e = 0; e < EPT; e++) {
    s[e] = (x[e] >= 0 && x[e] < pv.max_ids) ? slot_of[x[e]] : -1;  // bad ids: K3b flags them
    h += (t * EPT + e < n) && s[e] >= 0;
  }
  int nhit;
  int hr = block_exclusive_scan<NT>(h, wbuf, &nhit);
  const int64_t ob = (int64_t)b * out_stride;
#pragma unroll
  for (int e = 0; e < EPT; e++) {
    const int i = t * EPT + e;
    if (i >= n) continue;
    if (s[e] >= 0) {
      hit_row_out[ob + hr++] = s[e];
    } else {
      const int j = i - hr;
      miss_out[ob + j] = x[e];
      miss_row_out[ob + j] = pv.cap_max + j;
    }
  }
  if (t == 0) {
    counts_out[b * 4 + 0] = nhit;
    counts_out[b * 4 + 1] = n - nhit;
    counts_out[b * 4 + 2] = 0;
    counts_out[b * 4 + 3] = 0;
  }
}

// settle: staging row cap_max + j -> final slot slot[j] (< 0: not admitted), one warp
// per row, for the counts[b*4+1] misses of each pool
#ifndef ESS_SETTLE_CTAS
#define ESS_SETTLE_CTAS 8  // CTAs per pool (8 warps each, one row per warp at a time)
#endif
__global__ void pool_settle_kernel(PoolView pv, int begin, const int32_t *__restrict__ slot,
                                   const int32_t *__restrict__ counts, int stride) {
  const int b = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = counts[b * 4 + 1];
  uint8_t *base = pv.rows + (int64_t)(begin + b) * pv.rows_per_pool * pv.row_bytes;
  for (int j = blockIdx.y * (blockDim.x / 32) + warp; j < m; j += gridDim.y * (blockDim.x / 32)) {
    const int s = slot[(int64_t)b * stride + j];
    if (s >= 0) copy_row(base + (int64_t)(pv.cap_max + j) * pv.row_bytes, base + (int64_t)s * pv.row_bytes,
                         lane, pv.row_bytes);
  }
}

__global__ void pool_counters_kernel(PoolView pv, int begin, int num, int64_t *out) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= num) return;
  const PoolMeta m = pv.meta[begin + b];
  int64_t *o = out + (int64_t)b * 8;
  o[0] = m.cap;
  o[1] = m.size;
  o[2] = m.hits;
  o[3] = m.misses;
  o[4] = m.evictions;
  o[5] = m.clk;
  o[6] = m.watermark;
  o[7] = 0;
}

// ---- K4: zero-copy gather of miss rows ------------------------
#ifndef ESS_GATHER_LD256
#define ESS_GATHER_LD256 0
#endif
__device__ __forceinline__ uint4 shfl_v4(uint4 x, int src) {
  return make_uint4(__shfl_sync(0xffffffffu, x.x, src), __shfl_sync(0xffffffffu, x.y, src),
                    __shfl_sync(0xffffffffu, x.z, src), __shfl_sync(0xffffffffu, x.w, src));
}
#ifndef ESS_GATHER_NTG
#define ESS_GATHER_NTG 256
#endif
constexpr int NTG = ESS_GATHER_NTG;
#ifndef ESS_GATHER_GROWS
#define ESS_GATHER_GROWS 4
#endif
constexpr int GROWS = ESS_GATHER_GROWS;  // rows per warp iteration -> 8 x 16-B loads in flight per lane

__global__ void __launch_bounds__(NTG) gather_kernel(PoolView pv, int begin, int num,
                                                     const uint8_t *host, int64_t host_stride,
                                                     const int32_t *__restrict__ miss_ids,
                                                     const int32_t *__restrict__ miss_row,
                                                     const int32_t *__restrict__ counts,
                                                     int stride, int32_t *landed) {
  extern __shared__ int pref[];  // [num + 1]
  __shared__ int wbuf[NTG / 32];
  ess_pdl_trigger();
  ess_pdl_wait();  // PDL-launched: the split's miss lists complete and visible
  int run = 0;
  for (int c0 = 0; c0 < num; c0 += NTG) {
    int i = c0 + threadIdx.x;
    int v = i < num ? counts[i * 4 + 1] : 0;
    int tot;
    int ex = block_exclusive_scan<NTG>(v, wbuf, &tot);
    if (i < num) pref[i] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0) pref[num] = run;
  __syncthreads();
  const int total = run;
  const int lane = threadIdx.x & 31;
  const int gwarp = blockIdx.x * (NTG / 32) + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * (NTG / 32);
  const int64_t rb = pv.row_bytes;
  // each warp owns a contiguous run of the flattened miss list (it spans few pools),
  // so arrival counts are published once per pool change and at the end: one fence
  // each instead of one per iteration, which would stall the host-link pipeline
  const int per = (total + nwarps - 1) / nwarps;
  const int gbeg = min(total, gwarp * per), gend = min(total, gbeg + per);
  int cur_pool = -1, tally = 0;
  auto publish = [&]() {
    if (landed && tally > 0) {
      __threadfence();  // every lane's slot stores before the release add
      __syncwarp();
      if (lane == 0)
        asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(landed + cur_pool), "r"(tally)
                     : "memory");
    }
    if (lane == 0 && tally > 0) SPROF_MAX(begin + cur_pool, 2);
    tally = 0;
  };
  for (int g0 = gbeg; g0 < gend; g0 += GROWS) {
    const uint8_t *src[GROWS];
    uint8_t *dst[GROWS];
    int pool_of[GROWS];
#pragma unroll
    for (int r = 0; r < GROWS; r++) {
      int g = g0 + r;
      src[r] = nullptr;
      pool_of[r] = 0;
      if (g < gend) {
        int lo = 0, hi = num - 1;  // last pool with pref <= g
        while (lo < hi) {
          int mid = (lo + hi + 1) >> 1;
          if (pref[mid] <= g) lo = mid; else hi = mid - 1;
        }
        int j = g - pref[lo];
        int id = miss_ids[(int64_t)lo * stride + j];
        int row = miss_row[(int64_t)lo * stride + j];
        src[r] = host + ((int64_t)lo * host_stride + id) * ESS_HOST_ROW_PITCH;
        dst[r] = pv.rows + ((int64_t)(begin + lo) * pv.rows_per_pool + row) * rb;
        pool_of[r] = lo;
      }
    }
    // all PCIe loads of the warp's rows in flight first, then dequantise
    uint4 v[GROWS][2];
#if ESS_GATHER_LD256
    // 32-B loads (lanes 0-19 two chunks each, lane 20 the last chunk), then shuffles put
    // chunk l in lane l (v0) and chunk 32+l in lane l (v1) as the dequant expects
#pragma unroll
    for (int r = 0; r < GROWS; r++) {
      uint4 a0 = make_uint4(0, 0, 0, 0), a1 = make_uint4(0, 0, 0, 0);
      if (src[r]) {
        if (lane < ROW_CHUNKS / 2) ld_host_v8(src[r] + lane * 32, a0, a1);
        else if (lane == ROW_CHUNKS / 2) a0 = ld_host_v4(src[r] + lane * 32);
      }
      const int s0 = lane >> 1, s1 = 16 + (lane >> 1);
      const uint4 t0 = shfl_v4(a0, s0), t1 = shfl_v4(a1, s0);
      const uint4 u0 = shfl_v4(a0, s1), u1 = shfl_v4(a1, s1);
      v[r][0] = (lane & 1) ? t1 : t0;
      v[r][1] = (lane + 32 < ROW_CHUNKS) ? ((lane & 1) ? u1 : u0) : make_uint4(0, 0, 0, 0);
    }
#else
#pragma unroll
    for (int r = 0; r < GROWS; r++) {
      v[r][1] = make_uint4(0, 0, 0, 0);
      if (src[r]) {
        v[r][0] = ld_host_v4(src[r] + lane * 16);
        if (lane + 32 < ROW_CHUNKS) v[r][1] = ld_host_v4(src[r] + (lane + 32) * 16);
      }
    }
#endif
#pragma unroll
    for (int r = 0; r < GROWS; r++) {
      if (!src[r]) continue;
      if (pool_of[r] != cur_pool) {  // rows of the previous pool are all stored
        publish();
        cur_pool = pool_of[r];
      }
      if (store_slot_row(v[r][0], v[r][1], lane, dst[r], (int)rb)) ess_set_status(pv.status, ESS_ERR_RANGE);
      tally++;
    }
  }
  publish();
}

// K4, streamed form: the gather starts with the step and takes each request as soon as
// the streamed top-k published its split (ready[b], acquire): warps claim GROWS-row
// chunks of request b's miss list from claim[b] (atomic tickets, requests in order), so
// every warp works on the earliest request that still has rows.  Each chunk's rows are
// published on landed[b] (release) for the fused DA attention.  The lists were written
// by a concurrent kernel: read through L2 (ld.global.cg).
__global__ void __launch_bounds__(NTG) gather_stream_kernel(PoolView pv, int begin, int num,
                                                            const uint8_t *host, int64_t host_stride,
                                                            const int32_t *miss_ids, const int32_t *miss_row,
                                                            const int32_t *counts, int stride,
                                                            const int32_t *ready, int32_t *claim,
                                                            int32_t *landed) {
  const int lane = threadIdx.x & 31;
  const int64_t rb = pv.row_bytes;
  int b = 0, nmiss = -1;
  while (b < num) {
    if (nmiss < 0) {
      ess_warp_wait_geq(ready + b, 1);
      nmiss = __ldcg(counts + (int64_t)b * 4 + 1);
    }
    int j0 = 0;
    if (lane == 0) j0 = atomicAdd(claim + b, GROWS);
    j0 = __shfl_sync(0xffffffffu, j0, 0);
    if (j0 >= nmiss) {
      b++;
      nmiss = -1;
      continue;
    }
    const int nr = min(GROWS, nmiss - j0);
    const uint8_t *src[GROWS];
    uint8_t *dst[GROWS];
#pragma unroll
    for (int r = 0; r < GROWS; r++) {
      src[r] = nullptr;
      if (r < nr) {
        const int id = __ldcg(miss_ids + (int64_t)b * stride + j0 + r);
        const int row = __ldcg(miss_row + (int64_t)b * stride + j0 + r);
        src[r] = host + ((int64_t)b * host_stride + id) * ESS_HOST_ROW_PITCH;
        dst[r] = pv.rows + ((int64_t)(begin + b) * pv.rows_per_pool + row) * rb;
      }
    }
    uint4 v[GROWS][2];
#pragma unroll
    for (int r = 0; r < GROWS; r++) {
      v[r][1] = make_uint4(0, 0, 0, 0);
      if (src[r]) {
        v[r][0] = ld_host_v4(src[r] + lane * 16);
        if (lane + 32 < ROW_CHUNKS) v[r][1] = ld_host_v4(src[r] + (lane + 32) * 16);
      }
    }
#pragma unroll
    for (int r = 0; r < GROWS; r++)
      if (src[r] && store_slot_row(v[r][0], v[r][1], lane, dst[r], (int)rb)) ess_set_status(pv.status, ESS_ERR_RANGE);
    if (landed) {
      __threadfence();  // every lane's slot stores before the release add
      __syncwarp();
      if (lane == 0) ess_red_release_add(landed + b, nr);
    }
    if (lane == 0) SPROF_MAX(begin + b, 2);
  }
}

// K4, bulk-copy form (ESS_GATHER_BULK): each warp streams its contiguous run of the
// flattened miss list through a ring of GB_RING 656-B shared-memory row buffers filled
// by one-instruction `cp.async.bulk` copies straight from the mapped host store (one
// 656-B request per row instead of 41 x 16-B loads), then dequantises from shared
// memory into the slot rows.  Same outputs and arrival counters as gather_kernel.
constexpr int GB_RING = 8;
constexpr int GB_ROW = ESS_LATENT_ROW_BYTES;  // 656 = 41 x 16 B

__device__ __forceinline__ int gather_locate(const int *pref, int num, int g) {
  int lo = 0, hi = num - 1;  // last pool with pref <= g
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(NTG) gather_bulk_kernel(PoolView pv, int begin, int num,
                                                          const uint8_t *host, int64_t host_stride,
                                                          const int32_t *__restrict__ miss_ids,
                                                          const int32_t *__restrict__ miss_row,
                                                          const int32_t *__restrict__ counts,
                                                          int stride, int32_t *landed) {
  extern __shared__ __align__(128) uint8_t gsm[];
  constexpr int NW = NTG / 32;
  uint8_t *ring = gsm;                                                   // [NW][GB_RING][656]
  uint64_t *bars = reinterpret_cast<uint64_t *>(gsm + NW * GB_RING * GB_ROW);  // [NW][GB_RING]
  int *pref = reinterpret_cast<int *>(bars + NW * GB_RING);             // [num + 1]
  __shared__ int wbuf[NW];
  int run = 0;
  for (int c0 = 0; c0 < num; c0 += NTG) {
    int i = c0 + threadIdx.x;
    int v = i < num ? counts[i * 4 + 1] : 0;
    int tot;
    int ex = block_exclusive_scan<NTG>(v, wbuf, &tot);
    if (i < num) pref[i] = run + ex;
    run += tot;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t *myring = ring + warp * GB_RING * GB_ROW;
  uint64_t *mybar = bars + warp * GB_RING;
  if (threadIdx.x == 0) pref[num] = run;
  if (lane == 0) {
    for (int k = 0; k < GB_RING; k++) mbar_init(&mybar[k], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int total = run;
  const int gwarp = blockIdx.x * NW + warp;
  const int nwarps = gridDim.x * NW;
  const int64_t rb = pv.row_bytes;
  const int per = (total + nwarps - 1) / nwarps;
  const int gbeg = min(total, gwarp * per), gend = min(total, gbeg + per);
  const int n = gend - gbeg;
  auto issue = [&](int k) {  // lane 0: row gbeg + k -> ring buffer k % GB_RING
    const int g = gbeg + k;
    const int lo = gather_locate(pref, num, g);
    const int id = miss_ids[(int64_t)lo * stride + (g - pref[lo])];
    uint64_t *bar = &mybar[k % GB_RING];
    mbar_arrive_expect_tx(bar, GB_ROW);
    bulk_load(myring + (k % GB_RING) * GB_ROW, host + ((int64_t)lo * host_stride + id) * ESS_HOST_ROW_PITCH,
              GB_ROW, bar);
  };
  if (lane == 0)
    for (int k = 0; k < min(n, GB_RING); k++) issue(k);
  int cur_pool = -1, tally = 0;
  auto publish = [&]() {
    if (landed && tally > 0) {
      __threadfence();
      __syncwarp();
      if (lane == 0)
        asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(landed + cur_pool), "r"(tally)
                     : "memory");
    }
    tally = 0;
  };
  for (int k = 0; k < n; k++) {
    const int slot = k % GB_RING;
    const int g = gbeg + k;
    const int lo = gather_locate(pref, num, g);
    const int row = miss_row[(int64_t)lo * stride + (g - pref[lo])];
    mbar_wait(&mybar[slot], (k / GB_RING) & 1);
    const uint4 *buf = reinterpret_cast<const uint4 *>(myring + slot * GB_ROW);
    const uint4 v0 = buf[lane];
    const uint4 v1 = lane + 32 < ROW_CHUNKS ? buf[lane + 32] : make_uint4(0, 0, 0, 0);
    __syncwarp();
    if (lane == 0 && k + GB_RING < n) issue(k + GB_RING);
    if (lo != cur_pool) {
      publish();
      cur_pool = lo;
    }
    if (store_slot_row(v0, v1, lane, pv.rows + ((int64_t)(begin + lo) * pv.rows_per_pool + row) * rb, (int)rb)) ess_set_status(pv.status, ESS_ERR_RANGE);
    tally++;
  }
  publish();
}

// generated rows (656-B latent format) -> host store (D2H through the mapped alias)
// and, dequantised, their slots
__global__ void write_generated_kernel(PoolView pv, int begin, const int32_t *ids,
                                       const int32_t *m, const int32_t *slot, int stride,
                                       const uint8_t *src, uint8_t *host, int64_t host_stride) {
  const int b = blockIdx.x;
  const int M = m[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int64_t LB = ESS_LATENT_ROW_BYTES;
  for (int j = warp; j < M; j += blockDim.x / 32) {
    const int id = ids[(int64_t)b * stride + j];
    const int s = slot ? slot[(int64_t)b * stride + j] : -1;
    const uint8_t *sr = src + ((int64_t)b * stride + j) * LB;
    uint4 v0 = reinterpret_cast<const uint4 *>(sr)[lane];
    uint4 v1 = lane + 32 < ROW_CHUNKS ? reinterpret_cast<const uint4 *>(sr)[lane + 32] : make_uint4(0, 0, 0, 0);
    if (host) {
      uint8_t *h = host + ((int64_t)b * host_stride + id) * ESS_HOST_ROW_PITCH;
      st_v4(h + lane * 16, v0);
      if (lane + 32 < ROW_CHUNKS) st_v4(h + (lane + 32) * 16, v1);
    }
    if (s >= 0)
      if (store_slot_row(v0, v1, lane, pv.rows + ((int64_t)(begin + b) * pv.rows_per_pool + s) * pv.row_bytes,
                     pv.row_bytes)) ess_set_status(pv.status, ESS_ERR_RANGE);
  }
}

// The decode step's tail for one pool in one launch (cache.py:191-195 order): grow the
// capacity to max(1, floor(rho * (h + m))) (cache.py:137-138, f64 as in Python), admit
// the m generated ids h..h+m-1 at top recency (evicting LRU, counted; cache.py:122-134),
// write each new 656-B row back to the host store (D2H) and, dequantised,
// into its slot, and advance the history h (the request's length) by m.
__global__ void __launch_bounds__(NTA) pool_admit_kernel(PoolView pv, int begin, int32_t *hist,
                                                        const int32_t *m_arr, double rho,
                                                        const uint8_t *src, int src_stride,
                                                        uint8_t *host, int64_t host_stride,
                                                        int32_t *slot_out) {
  __shared__ unsigned long long red[NTA / 32 + 1];
  __shared__ int slots[64];
  const int b = blockIdx.x, p = begin + b;
  PoolMeta *meta = pv.meta + p;
  int32_t *slot_of = pv.slot_of + (int64_t)p * pv.max_ids;
  int32_t *slot_id = pv.slot_id + (int64_t)p * pv.cap_max;
  uint32_t *key = pv.key + (int64_t)p * pv.cap_max;
  const int h = hist[b];
  const int M = m_arr ? m_arr[b] : 1;
  const int64_t want = (int64_t)floor(rho * (double)(h + M));
  const int newcap = (int)(want < 1 ? 1 : want);
  int code = 0;
  // M rows per pool are read from the source: never more than its row stride holds
  if (M < 0 || M > 64 || M > src_stride || (int64_t)h + M > pv.max_ids) code = ESS_ERR_ARG;
  else if (newcap < meta->cap) code = ESS_ERR_SHRINK;
  else if (newcap > pv.cap_max) code = ESS_ERR_CAPACITY;
  else if ((int64_t)h <= meta->watermark) code = ESS_ERR_DUPLICATE;
  if (code) {
    if (threadIdx.x == 0) ess_set_status(pv.status, code);
    return;
  }
  const int cap = newcap;
  int size = meta->size;
  uint32_t clk = meta->clk;
  int64_t evictions = 0;
  for (int i = 0; i < M; i++) {
    int s;
    if (size >= cap) {  // LRU resident -> evicted; its slot takes the new id
      s = argmin_key(key, cap, red);
      if (threadIdx.x == 0) slot_of[slot_id[s]] = -1;
      evictions++;
    } else {            // smallest free slot (free keys == slot index < any stamp)
      s = argmin_key(key, cap, red);
      size++;
    }
    if (threadIdx.x == 0) {
      slot_of[h + i] = s;
      slot_id[s] = h + i;
      key[s] = clk;
      slots[i] = s;
    }
    clk++;
    __syncthreads();
  }
  // rows: host write-back + dequantised slot fill, one warp per row
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = warp; i < M; i += NTA / 32) {
    const uint8_t *sr = src + ((int64_t)b * src_stride + i) * ESS_LATENT_ROW_BYTES;
    uint4 v0 = reinterpret_cast<const uint4 *>(sr)[lane];
    uint4 v1 = lane + 32 < ROW_CHUNKS ? reinterpret_cast<const uint4 *>(sr)[lane + 32] : make_uint4(0, 0, 0, 0);
    if (host) {
      uint8_t *hp = host + ((int64_t)b * host_stride + h + i) * ESS_HOST_ROW_PITCH;
      st_v4(hp + lane * 16, v0);
      if (lane + 32 < ROW_CHUNKS) st_v4(hp + (lane + 32) * 16, v1);
    }
    if (pv.rows)
      if (store_slot_row(v0, v1, lane, pv.rows + ((int64_t)p * pv.rows_per_pool + slots[i]) * pv.row_bytes,
                     pv.row_bytes)) ess_set_status(pv.status, ESS_ERR_RANGE);
    if (slot_out && lane == 0) slot_out[(int64_t)b * src_stride + i] = slots[i];
  }
  if (threadIdx.x == 0) {
    meta->cap = cap;
    meta->size = size;
    meta->clk = clk;
    meta->watermark = h + M - 1 > meta->watermark ? h + M - 1 : meta->watermark;
    meta->evictions += evictions;
    hist[b] = h + M;
  }
}

__global__ void pool_lookup_kernel(PoolView pv, int p, const int32_t *ids, int n, int32_t *out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int x = ids[i];
  out[i] = (x >= 0 && x < pv.max_ids) ? pv.slot_of[(int64_t)p * pv.max_ids + x] : -1;
}

// dst pools [dst_begin, +num) <- src pools [src_begin, +num); dst may be larger in
// max_ids / cap_max (the extra ids are absent, the extra slots free)
__global__ void pool_copy_kernel(PoolView d, int dst_begin, PoolView s, int src_begin) {
  const int b = blockIdx.x;
  const int pd = dst_begin + b, ps = src_begin + b;
  if (blockIdx.y == 0 && threadIdx.x == 0) d.meta[pd] = s.meta[ps];
  const int64_t stride = (int64_t)gridDim.y * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < d.max_ids; i += stride)
    d.slot_of[(int64_t)pd * d.max_ids + i] = i < s.max_ids ? s.slot_of[(int64_t)ps * s.max_ids + i] : -1;
  for (int64_t i = i0; i < d.cap_max; i += stride) {
    bool in = i < s.cap_max;
    d.slot_id[(int64_t)pd * d.cap_max + i] = in ? s.slot_id[(int64_t)ps * s.cap_max + i] : -1;
    d.key[(int64_t)pd * d.cap_max + i] = in ? s.key[(int64_t)ps * s.cap_max + i] : (uint32_t)i;
  }
  if (d.rows && s.rows) {
    const int64_t nb = (int64_t)(s.cap_max < d.cap_max ? s.cap_max : d.cap_max) * s.row_bytes / 16;
    const uint4 *src = reinterpret_cast<const uint4 *>(s.rows + (int64_t)ps * s.rows_per_pool * s.row_bytes);
    uint4 *dst = reinterpret_cast<uint4 *>(d.rows + (int64_t)pd * d.rows_per_pool * d.row_bytes);
    for (int64_t i = i0; i < nb; i += stride) dst[i] = src[i];
  }
}

thread_local int g_last_cuda_error = 0;

bool range_ok(const ess_pool *p, int begin, int num) {
  return p && begin >= 0 && num >= 0 && (int64_t)begin + num <= p->P;
}

}  // namespace

int ess_record_cuda_error(cudaError_t e) {
  g_last_cuda_error = (int)e;
  return ESS_ERR_CUDA;
}

extern "C" {

int ess_pool_create(ess_pool **out, int32_t num_pools, int64_t max_ids, int32_t cap_max,
                    int32_t row_bytes, int32_t staging_rows) {
  if (!out || num_pools < 1 || max_ids < 1 || max_ids > 0x7fffffff || cap_max < 1 ||
      cap_max > 0x00ffffff || staging_rows < 0 || row_bytes < 0 ||
      (row_bytes && row_bytes != ESS_SLOT_ROW_BYTES && row_bytes != ESS_SLOT_ROW_BYTES_FP8))
    return ESS_ERR_ARG;
  // 64-B alignment for the embedded CUtensorMap
  ess_pool *p = (ess_pool *)aligned_alloc(64, (sizeof(ess_pool) + 63) & ~size_t(63));
  if (!p) return ESS_ERR_NOMEM;
  memset(p, 0, sizeof(ess_pool));
  p->P = num_pools;
  p->max_ids = max_ids;
  p->cap_max = cap_max;
  p->row_bytes = row_bytes;
  p->staging = staging_rows;
  p->rows_per_pool = (int64_t)cap_max + staging_rows;
  cudaGetDevice(&p->device);
  cudaError_t e = cudaSuccess;
  e = cudaMalloc(&p->meta, sizeof(PoolMeta) * num_pools);
  if (e == cudaSuccess) e = cudaMalloc(&p->slot_of, sizeof(int32_t) * num_pools * max_ids);
  if (e == cudaSuccess) e = cudaMalloc(&p->slot_id, sizeof(int32_t) * num_pools * (int64_t)cap_max);
  if (e == cudaSuccess) e = cudaMalloc(&p->key, sizeof(uint32_t) * num_pools * (int64_t)cap_max);
  if (e == cudaSuccess) e = cudaMalloc(&p->status, sizeof(int32_t));
  if (e == cudaSuccess && row_bytes)
    e = cudaMalloc(&p->rows, (size_t)num_pools * p->rows_per_pool * row_bytes);
  if (e == cudaSuccess) e = cudaMemset(p->status, 0, sizeof(int32_t));
  if (e == cudaSuccess && row_bytes)
    e = cudaMemset(p->rows, 0, (size_t)num_pools * p->rows_per_pool * row_bytes);
  if (e != cudaSuccess) {
    ess_pool_destroy(p);
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? ESS_ERR_NOMEM : ess_record_cuda_error(e);
  }
  // initial state: every pool empty at capacity cap_max
  int32_t *caps = nullptr;
  e = cudaMalloc(&caps, sizeof(int32_t) * num_pools);
  if (e == cudaSuccess) {
    int32_t *h = (int32_t *)malloc(sizeof(int32_t) * num_pools);
    for (int i = 0; i < num_pools; i++) h[i] = cap_max;
    cudaMemcpy(caps, h, sizeof(int32_t) * num_pools, cudaMemcpyHostToDevice);
    free(h);
    int rc = ess_pool_reset(p, 0, num_pools, caps, nullptr);
    cudaDeviceSynchronize();
    cudaFree(caps);
    if (rc) {
      ess_pool_destroy(p);
      return rc;
    }
  }
  *out = p;
  return ESS_OK;
}

int ess_pool_destroy(ess_pool *p) {
  if (!p) return ESS_ERR_ARG;
  cudaFree(p->meta);
  cudaFree(p->slot_of);
  cudaFree(p->slot_id);
  cudaFree(p->key);
  cudaFree(p->rows);
  cudaFree(p->status);
  free(p);
  return ESS_OK;
}

int ess_pool_reset(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_capacity,
                   void *stream) {
  if (!range_ok(p, begin, num) || !d_capacity) return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  int64_t per = p->max_ids > p->cap_max ? p->max_ids : p->cap_max;
  int gy = (int)((per + 256 * 8 - 1) / (256 * 8));
  if (gy > 64) gy = 64;
  dim3 grid(num, gy);
  pool_reset_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(view(p), begin, num, d_capacity);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_grow(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_capacity,
                  void *stream) {
  if (!range_ok(p, begin, num) || !d_capacity) return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  pool_grow_kernel<<<(num + 255) / 256, 256, 0, (cudaStream_t)stream>>>(view(p), begin, num,
                                                                         d_capacity);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_warmup(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_ids,
                    const int32_t *d_n, int32_t stride, int64_t *d_inserted, void *stream) {
  if (!range_ok(p, begin, num) || !d_ids || !d_n || stride < 0) return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  pool_step_kernel<MODE_WARMUP><<<num, NT, 0, (cudaStream_t)stream>>>(
      view(p), begin, d_ids, d_n, stride, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
      nullptr, 0, 0, d_inserted, 1, 0, TokSplit{});
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_split(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_req, const int32_t *d_n,
                   int32_t req_stride, int32_t *d_hit_row, int32_t *d_miss_ids, int32_t *d_miss_row,
                   int32_t *d_counts, int32_t out_stride, void *stream) {
  if (!range_ok(p, begin, num) || !d_req || !d_n || !d_hit_row || !d_miss_ids || !d_miss_row ||
      !d_counts || out_stride < 1 || req_stride < 0 || p->staging < MAXR)
    return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  pool_split_kernel<<<num, NT, 0, (cudaStream_t)stream>>>(view(p), begin, d_req, d_n, req_stride,
                                                           d_hit_row, d_miss_ids, d_miss_row,
                                                           d_counts, out_stride);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_settle(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_slot,
                    const int32_t *d_counts, int32_t stride, void *stream) {
  if (!range_ok(p, begin, num) || !p->rows || !d_slot || !d_counts || stride < 1) return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  pool_settle_kernel<<<dim3(num, ESS_SETTLE_CTAS), 256, 0, (cudaStream_t)stream>>>(view(p), begin, d_slot, d_counts,
                                                                     stride);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

static int pool_access_launch(ess_pool *p, int32_t begin, int32_t num, int32_t qtok,
                              const int32_t *d_req, const int32_t *d_n, int32_t req_stride,
                              int32_t *d_hit_ids, int32_t *d_miss_ids, int32_t *d_evicted_ids,
                              int32_t *d_sel_row, int32_t sel_stride, int32_t *d_hit_row,
                              int32_t *d_miss_row, int32_t *d_counts, int32_t out_stride,
                              int32_t flags, void *stream, TokSplit ts = TokSplit{}) {
  if (!range_ok(p, begin, num) || !d_req || !d_n || req_stride < 0) return ESS_ERR_ARG;
  if ((d_hit_ids || d_miss_ids || d_evicted_ids || d_sel_row || d_hit_row || d_miss_row) &&
      out_stride < 1)
    return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  if (flags & POOL_STAGED) return ESS_ERR_ARG;
  const size_t stage = (size_t)p->cap_max * 4;
  const size_t bits = ts.hit_row ? (size_t)(p->cap_max + 31) / 32 * 4 : 0;
  size_t smem = bits;
  if (stage + bits <= STAGE_SMEM_MAX) {
    smem = stage + bits;
    flags |= POOL_STAGED;
  }
  if (smem)
    if (int rc = ess_smem_optin((const void *)pool_step_kernel<MODE_ACCESS>, smem)) return rc;
  pool_step_kernel<MODE_ACCESS><<<num, NT, smem, (cudaStream_t)stream>>>(
      view(p), begin, d_req, d_n, req_stride, d_hit_ids, d_miss_ids, d_evicted_ids, d_sel_row,
      d_hit_row, d_miss_row, d_counts, out_stride, flags, nullptr, qtok, sel_stride, ts);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_access(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_req,
                    const int32_t *d_n, int32_t req_stride, int32_t *d_hit_ids,
                    int32_t *d_miss_ids, int32_t *d_evicted_ids, int32_t *d_sel_row,
                    int32_t *d_hit_row, int32_t *d_miss_row, int32_t *d_counts,
                    int32_t out_stride, int32_t flags, void *stream) {
  return pool_access_launch(p, begin, num, 1, d_req, d_n, req_stride, d_hit_ids, d_miss_ids,
                            d_evicted_ids, d_sel_row, out_stride, d_hit_row, d_miss_row, d_counts,
                            out_stride, flags, stream);
}

int ess_pool_access_mtp(ess_pool *p, int32_t begin, int32_t num, int32_t qtok, const int32_t *d_req,
                        const int32_t *d_n, int32_t req_stride, int32_t *d_hit_ids,
                        int32_t *d_miss_ids, int32_t *d_evicted_ids, int32_t *d_sel_row,
                        int32_t *d_hit_row, int32_t *d_miss_row, int32_t *d_counts,
                        int32_t out_stride, int32_t *d_tok_hit_row, int32_t *d_tok_fresh_row,
                        int32_t *d_tok_counts, int32_t *d_ready, int32_t flags, void *stream) {
  if (qtok < 1 || qtok > ESS_INDEXER_MAX_QTOK) return ESS_ERR_ARG;
  if ((d_tok_hit_row || d_tok_fresh_row || d_tok_counts) && !(d_tok_hit_row && d_tok_fresh_row && d_tok_counts))
    return ESS_ERR_ARG;
  TokSplit ts;
  ts.hit_row = d_tok_hit_row;
  ts.fresh_row = d_tok_fresh_row;
  ts.cnt = d_tok_counts;
  ts.ready = d_ready;
  if ((d_hit_ids || d_miss_ids || d_evicted_ids || d_hit_row || d_miss_row) &&
      (int64_t)out_stride < (int64_t)qtok * req_stride)
    return ESS_ERR_ARG;  // the appended lists of qtok sets must fit a pool's row
  return pool_access_launch(p, begin, num, qtok, d_req, d_n, req_stride, d_hit_ids, d_miss_ids,
                            d_evicted_ids, d_sel_row, req_stride, d_hit_row, d_miss_row, d_counts,
                            out_stride, flags, stream, ts);
}

#ifdef ESS_POOL_PROF
int ess_debug_pool_prof(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, g_pool_prof, sizeof(g_pool_prof)) == cudaSuccess ? 0 : -7;
}
#endif

int ess_pool_append(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_ids,
                    const int32_t *d_m, int32_t stride, int32_t *d_slot_out, void *stream) {
  if (!range_ok(p, begin, num) || !d_ids || !d_m || stride < 0) return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  pool_append_kernel<<<num, NTA, 0, (cudaStream_t)stream>>>(view(p), begin, d_ids, d_m, stride,
                                                            d_slot_out);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_lru_order(ess_pool *p, int32_t begin, int32_t num, int32_t *d_out,
                       int32_t *d_count, void *stream) {
  if (!range_ok(p, begin, num) || !d_out || !d_count) return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  dim3 grid(num, (p->cap_max + 255) / 256);
  pool_lru_order_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(view(p), begin, d_out, d_count);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_counters(ess_pool *p, int32_t begin, int32_t num, int64_t *d_out, void *stream) {
  if (!range_ok(p, begin, num) || !d_out) return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  pool_counters_kernel<<<(num + 127) / 128, 128, 0, (cudaStream_t)stream>>>(view(p), begin, num,
                                                                            d_out);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_status(ess_pool *p, int32_t *status_out) {
  if (!p || !status_out) return ESS_ERR_ARG;
  int32_t h = 0;
  ESS_CUDA_TRY(cudaMemcpy(&h, p->status, sizeof(int32_t), cudaMemcpyDeviceToHost));
  ESS_CUDA_TRY(cudaMemset(p->status, 0, sizeof(int32_t)));
  *status_out = h;
  return ESS_OK;
}

int ess_pool_info(ess_pool *p, int32_t *num_pools, int64_t *max_ids, int32_t *cap_max,
                  int32_t *row_bytes, int64_t *rows_per_pool, void **d_rows) {
  if (!p) return ESS_ERR_ARG;
  if (num_pools) *num_pools = p->P;
  if (max_ids) *max_ids = p->max_ids;
  if (cap_max) *cap_max = p->cap_max;
  if (row_bytes) *row_bytes = p->row_bytes;
  if (rows_per_pool) *rows_per_pool = p->rows_per_pool;
  if (d_rows) *d_rows = p->rows;
  return ESS_OK;
}

int ess_pool_lookup(ess_pool *p, int32_t pool, const int32_t *d_ids, int32_t n,
                    int32_t *d_slot_out, void *stream) {
  if (!p || pool < 0 || pool >= p->P || n < 0 || (n && (!d_ids || !d_slot_out))) return ESS_ERR_ARG;
  if (n == 0) return ESS_OK;
  pool_lookup_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(view(p), pool, d_ids, n,
                                                                        d_slot_out);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_copy_state(ess_pool *dst, int32_t dst_begin, ess_pool *src, int32_t src_begin,
                        int32_t num, void *stream) {
  if (!range_ok(dst, dst_begin, num) || !range_ok(src, src_begin, num) ||
      dst->max_ids < src->max_ids || dst->cap_max < src->cap_max ||
      dst->row_bytes != src->row_bytes)
    return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  dim3 grid(num, 32);
  pool_copy_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(view(dst), dst_begin, view(src), src_begin);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_gather(ess_pool *p, int32_t begin, int32_t num, const void *d_host_rows,
               int64_t host_pool_stride_rows, const int32_t *d_miss_ids,
               const int32_t *d_miss_row, const int32_t *d_counts, int32_t stride,
               int32_t max_ctas, int32_t flags, void *stream) {
  return ess_gather_signal(p, begin, num, d_host_rows, host_pool_stride_rows, d_miss_ids,
                           d_miss_row, d_counts, stride, nullptr, max_ctas, flags, stream);
}

int ess_gather_signal(ess_pool *p, int32_t begin, int32_t num, const void *d_host_rows,
                      int64_t host_pool_stride_rows, const int32_t *d_miss_ids,
                      const int32_t *d_miss_row, const int32_t *d_counts, int32_t stride,
                      int32_t *d_landed, int32_t max_ctas, int32_t flags, void *stream) {
  if (!range_ok(p, begin, num) || !p->rows || !d_host_rows || !d_miss_ids || !d_miss_row ||
      !d_counts || stride < 1 || max_ctas < 1)
    return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  const bool bulk = (flags & ESS_GATHER_BULK) != 0;
  const size_t ring = bulk ? (size_t)(NTG / 32) * GB_RING * (GB_ROW + 8) : 0;
  size_t smem = ring + sizeof(int) * (num + 1);
  // ESS_GATHER_EXCLUSIVE_SM: reserve enough shared memory that a gather CTA can never
  // share an SM with a K5 CTA (~205 KB), so the long-latency host-link loads do not
  // compete with attention for the SM's L1 miss tracking — the gather runs on the SMs
  // attention leaves idle.
  if ((flags & ESS_GATHER_EXCLUSIVE_SM) && smem < ESS_GATHER_EXCLUSIVE_SMEM)
    smem = ESS_GATHER_EXCLUSIVE_SMEM;
  if (bulk && (flags & ESS_LAUNCH_PDL)) return ESS_ERR_ARG;  // the bulk form has no PDL wait
  auto kern = bulk ? gather_bulk_kernel : gather_kernel;
  if (int rc = ess_smem_optin((const void *)kern, smem)) return rc;
  ESS_CUDA_TRY(ess_launch(kern, dim3(max_ctas), dim3(NTG), smem, (cudaStream_t)stream, 1,
                          (flags & ESS_LAUNCH_PDL) != 0, view(p), (int)begin, (int)num,
                          (const uint8_t *)d_host_rows, host_pool_stride_rows, d_miss_ids, d_miss_row,
                          d_counts, (int)stride, d_landed));
  return ESS_OK;
}

int ess_gather_stream(ess_pool *p, int32_t begin, int32_t num, const void *d_host_rows,
                      int64_t host_pool_stride_rows, const int32_t *d_miss_ids,
                      const int32_t *d_miss_row, const int32_t *d_counts, int32_t stride,
                      const int32_t *d_ready, int32_t *d_claim, int32_t *d_landed, int32_t max_ctas,
                      int32_t flags, void *stream) {
  if (!range_ok(p, begin, num) || !p->rows || !d_host_rows || !d_miss_ids || !d_miss_row ||
      !d_counts || stride < 1 || max_ctas < 1 || !d_ready || !d_claim || (flags & ESS_GATHER_BULK))
    return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  size_t smem = 0;
  if (flags & ESS_GATHER_EXCLUSIVE_SM) smem = ESS_GATHER_EXCLUSIVE_SMEM;
  if (int rc = ess_smem_optin((const void *)gather_stream_kernel, smem)) return rc;
  gather_stream_kernel<<<max_ctas, NTG, smem, (cudaStream_t)stream>>>(
      view(p), begin, num, (const uint8_t *)d_host_rows, host_pool_stride_rows, d_miss_ids, d_miss_row,
      d_counts, stride, d_ready, d_claim, d_landed);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_pool_admit(ess_pool *p, int32_t begin, int32_t num, int32_t *d_hist, const int32_t *d_m,
                   double rho, const void *d_src_rows, int32_t src_stride, void *d_host_rows,
                   int64_t host_pool_stride_rows, int32_t *d_slot_out, void *stream) {
  if (!range_ok(p, begin, num) || !d_hist || !d_src_rows || src_stride < 1 || !(rho > 0.0) ||
      rho > 1.0)
    return rho > 0.0 && rho <= 1.0 ? ESS_ERR_ARG : ESS_ERR_RATIO;
  if (num == 0) return ESS_OK;
  pool_admit_kernel<<<num, NTA, 0, (cudaStream_t)stream>>>(
      view(p), begin, d_hist, d_m, rho, (const uint8_t *)d_src_rows, src_stride,
      (uint8_t *)d_host_rows, host_pool_stride_rows, d_slot_out);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_write_generated(ess_pool *p, int32_t begin, int32_t num, const int32_t *d_ids,
                        const int32_t *d_m, const int32_t *d_slot, int32_t stride,
                        const void *d_src_rows, void *d_host_rows,
                        int64_t host_pool_stride_rows, void *stream) {
  if (!range_ok(p, begin, num) || !p->rows || !d_ids || !d_m || !d_src_rows || stride < 1)
    return ESS_ERR_ARG;
  if (num == 0) return ESS_OK;
  write_generated_kernel<<<num, 128, 0, (cudaStream_t)stream>>>(
      view(p), begin, d_ids, d_m, d_slot, stride, (const uint8_t *)d_src_rows,
      (uint8_t *)d_host_rows, host_pool_stride_rows);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

}  // extern "C"

#ifdef ESS_STREAM_PROF
ESS_STREAM_PROF_READER(ess_debug_stream_prof_gather)
#endif

int ess_preload_pool() {  // see ess_preload_indexer
  cudaFuncAttributes a;
  const void *k[] = {(const void *)pool_step_kernel<MODE_ACCESS>, (const void *)pool_step_kernel<MODE_WARMUP>,
                     (const void *)pool_reset_kernel, (const void *)pool_grow_kernel,
                     (const void *)pool_append_kernel, (const void *)pool_lru_order_kernel,
                     (const void *)pool_split_kernel, (const void *)pool_settle_kernel,
                     (const void *)pool_counters_kernel, (const void *)gather_kernel,
                     (const void *)gather_bulk_kernel, (const void *)gather_stream_kernel,
                     (const void *)write_generated_kernel, (const void *)pool_admit_kernel,
                     (const void *)pool_lookup_kernel, (const void *)pool_copy_kernel};
  for (const void *f : k) ESS_CUDA_TRY(cudaFuncGetAttributes(&a, f));
  return ESS_OK;
}
