// K2: per-row top-k radix select (op "indexer_topk", costmodel.py:18-27).
//
// Contract (the reference's generator has no tie rule, trace.py:107-112):
//   select the k largest logits[b][0:len) ordered by (score desc, index asc) and
//   emit them ascending by index — the canonical selection-set form of
//   AccessTrace (trace.py:31-46).  len <= k returns 0..len-1 (scenario.py:110-112).
//
// One CLN-CTA thread-block cluster per row (CLN in {1,2,4,8}, the smallest whose slice
// fits shared memory: 1 up to 40K tokens, 4 at 128K); CTA r owns the r-th
// contiguous slice of the row, staged once as order-preserving u32 keys in shared
// memory (-0.0 canonicalised to +0.0 so IEEE-equal scores are equal keys).
//
// Exact k-th largest key T in three radix digits, 12 + 10 + 10 bits:
//   1. the 12-bit histogram (sign, exponent, 3 mantissa bits) is built while the slice
//      is staged; every CTA pushes its nonzero bins into every rank's summed histogram
//      (distributed shared memory reductions) and all agree on the digit d1 without a
//      global round trip;
//   2. the keys whose first digit is >= d1 (the < k keys above the bin plus the bin
//      itself, about k per row) are appended in one pass to per-warp u16 list segments
//      (in warp order = row order); a segment overflow falls back to one contiguous list;
//   3. the two 10-bit passes and the ordered emit (per warp segment) touch only the list.
// Full-slice passes: stage, list.  A list longer than LCAP (mass ties) makes that CTA
// fall back to full-slice passes.  The emit takes every key > T plus the first
// (k - #greater) keys == T in index order; CTA r's output offset is the cluster prefix
// of the (greater, equal) counts of CTAs 0..r-1.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

#ifdef ESS_TOPK_PROF  // scratch builds: per-phase globaltimer stamps (thread 0 of each CTA)
__device__ unsigned long long g_topk_prof[1024][12];
#define KPROF(i)                                                             \
  do {                                                                       \
    __syncthreads();                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                             \
      unsigned long long tt;                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                 \
      g_topk_prof[blockIdx.x][i] = tt;                                       \
    }                                                                        \
  } while (0)
extern "C" int ess_debug_topk_prof(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, g_topk_prof, sizeof(g_topk_prof)) == cudaSuccess ? 0 : -7;
}
#else
#define KPROF(i) \
  do {           \
  } while (0)
#endif

namespace {

#ifndef ESS_TOPK_LIST_UNROLL
#define ESS_TOPK_LIST_UNROLL 2
#endif
constexpr int LIST_UNROLL = ESS_TOPK_LIST_UNROLL;
constexpr int NT = 1024;                  // threads per CTA
constexpr int NW = NT / 32;
constexpr int VEC = 4;
constexpr int SLICE_MAX = 40 * 1024;      // keys per CTA (160 KB of shared memory)
constexpr int LCAP = 12 * 1024;           // list entries per CTA (u16, 24 KB)
constexpr int RCAP = LCAP / (NT / 32);    // per-warp list segment (one-pass list)
constexpr int D1_BITS = 12, D1_BINS = 1 << D1_BITS, D1_SHIFT = 32 - D1_BITS;
constexpr int DR_BITS = 10, DR_BINS = 1 << DR_BITS;
static_assert(DR_BINS == NT, "one 10-bit bin per thread");

__device__ __forceinline__ uint32_t score_key(float f) {
  uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// (greater, equal) counts packed as g | q << 16 in an unsigned word: g < k <= 65535 and
// a CTA holds at most SLICE_MAX (40K) keys, so neither field carries into the other and
// the logical >> 16 never sign-extends (a signed pack broke at 32K equal keys).
__device__ __forceinline__ uint32_t pack_gq(uint32_t g, uint32_t q) { return g | (q << 16); }
static_assert(SLICE_MAX < 65536, "equal-count field of pack_gq");

template <int CLN>
__device__ __forceinline__ void cluster_sync() {
  if constexpr (CLN > 1) cg::this_cluster().sync();
  else __syncthreads();
}

// Cluster rows sum their histograms by pushing: every CTA adds its counts into every
// rank's `csum` with remote shared-memory reductions (only nonzero bins for the 12-bit
// digit, one add per candidate key for the 10-bit digits), then each CTA picks from its
// own csum.  Pulling every bin of every peer (4 B DSMEM loads) cost 4 / 10 us at 2 / 4
// CTAs per row; pushes are fire-and-forget and skip the empty bins.
__device__ __forceinline__ uint32_t cluster_addr(const void *p, int rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}
__device__ __forceinline__ void cluster_red_add(uint32_t addr, int v) {
  asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Digit holding the rem-th largest key of a histogram (bins scanned from the top);
// thread t owns NB/NT consecutive bins.  Leaves (digit, rank inside the bin)
// in scal and syncs the CTA.
template <int NB>
__device__ __forceinline__ void pick_digit(int *hist, int rem, int *wbuf, int *scal) {
  constexpr int BPT = NB / NT;
  int loc[BPT], sum = 0;
#pragma unroll
  for (int j = 0; j < BPT; j++) {
    loc[j] = hist[NB - 1 - (threadIdx.x * BPT + j)];
    sum += loc[j];
  }
  int tot;
  int c = block_exclusive_scan<NT>(sum, wbuf, &tot);
  if (c < rem && rem <= c + sum) {
#pragma unroll
    for (int j = 0; j < BPT; j++) {
      if (c + loc[j] >= rem) {
        scal[0] = NB - 1 - (threadIdx.x * BPT + j);
        scal[1] = rem - c;
        break;
      }
      c += loc[j];
    }
  }
  __syncthreads();
}

// Fallback helpers over warp-contiguous runs [lo, hi) of the staged slice.
__device__ __forceinline__ void run_counts(const uint32_t *skey, int lo, int hi, uint32_t T,
                                           int &g, int &q) {
  const int lane = threadIdx.x & 31;
  g = 0;
  q = 0;
  for (int i = lo; i < hi; i += 32) {
    const int j = i + lane;
    const uint32_t key = j < hi ? skey[j] : 0u;
    g += __popc(__ballot_sync(0xffffffffu, j < hi && key > T));
    q += __popc(__ballot_sync(0xffffffffu, j < hi && key == T));
  }
}

__device__ __forceinline__ void run_emit(const uint32_t *skey, int lo, int hi, uint32_t T,
                                         int need_eq, int gb, int eb, int idx_base,
                                         int32_t *__restrict__ o) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  for (int i = lo; i < hi; i += 32) {
    const int j = i + lane;
    const uint32_t key = j < hi ? skey[j] : 0u;
    const bool gt = j < hi && key > T, eq = j < hi && key == T;
    const uint32_t mg = __ballot_sync(0xffffffffu, gt), me = __ballot_sync(0xffffffffu, eq);
    const int e = eb + __popc(me & lt);
    if (gt || (eq && e < need_eq)) o[gb + __popc(mg & lt) + min(e, need_eq)] = idx_base + j;
    gb += __popc(mg);
    eb += __popc(me);
  }
}

template <int CLN>
__host__ __device__ __forceinline__ int64_t slice_cap(int64_t ld) {  // keys, 4-aligned
  return (((ld + CLN - 1) / CLN) + 3) & ~3LL;
}

// Optional fused epilogue: the early-gather hit/miss split of the cache
// manager (ess_pool_split) on the selection this CTA just emitted, saving a launch and
// the id reload.  slot_of already points at the first pool of the batch.
struct SplitArgs {
  const int32_t *slot_of;  // nullptr: no split
  int64_t max_ids;
  int32_t cap_max;
  int32_t *hit_row, *miss_ids, *miss_row, *counts;
  int32_t out_stride;
  int32_t len_div = 1;  // MTP: rows b*len_div .. b*len_div+len_div-1 share len[b]
  int32_t prof_base = 0;  // ESS_STREAM_PROF: pool index of row 0
};

__device__ __forceinline__ void split_tail(int b, const int32_t *o, int n, const SplitArgs &sp,
                                           int *wbuf) {
  __syncthreads();  // the emitted ids (global, this CTA's writes) are visible block-wide
  const int t = threadIdx.x;
  const int32_t *so = sp.slot_of + (int64_t)b * sp.max_ids;
  int x[2], sl[2], h = 0;
#pragma unroll
  for (int e = 0; e < 2; e++) {
    const int i = t * 2 + e;
    x[e] = i < n ? o[i] : -1;
  }
#pragma unroll
  for (int e = 0; e < 2; e++) {
    sl[e] = (x[e] >= 0 && x[e] < sp.max_ids) ? so[x[e]] : -1;
    h += (t * 2 + e < n) && sl[e] >= 0;
  }
  int nhit;
  int hr = block_exclusive_scan<NT>(h, wbuf, &nhit);
  const int64_t ob = (int64_t)b * sp.out_stride;
#pragma unroll
  for (int e = 0; e < 2; e++) {
    const int i = t * 2 + e;
    if (i >= n) continue;
    if (sl[e] >= 0) {
      sp.hit_row[ob + hr++] = sl[e];
    } else {
      const int j = i - hr;
      sp.miss_ids[ob + j] = x[e];
      sp.miss_row[ob + j] = sp.cap_max + j;  // per-pool staging row
    }
  }
  if (t == 0) {
    sp.counts[b * 4 + 0] = nhit;
    sp.counts[b * 4 + 1] = n - nhit;
    sp.counts[b * 4 + 2] = 0;
    sp.counts[b * 4 + 3] = 0;
  }
}

// One row (b) of the top-k on this CTA (cluster).  STREAM: the row's logits are being
// written by a concurrent indexer launch (ess_indexer_logits_stream) and were published
// with a release; they are read through L2 (ld.global.cg), not the non-coherent path.
template <int CLN, bool STREAM>
__device__ __forceinline__ void topk_row(const int b, const float *__restrict__ logits, int64_t ld,
                                         const int32_t *__restrict__ lens, int k,
                                         int32_t *__restrict__ out, int out_ld,
                                         int32_t *__restrict__ counts, const SplitArgs &sp) {
  extern __shared__ uint32_t skey[];  // slice_cap keys, then LCAP u16 list entries + NT trash
  uint16_t *list = reinterpret_cast<uint16_t *>(skey + slice_cap<CLN>(ld));
  __shared__ int hist[D1_BINS];
  __shared__ int csum[CLN > 1 ? D1_BINS : 1];  // cluster rows: histogram summed over ranks
  __shared__ int wbuf[NW];
  uint32_t *uwbuf = reinterpret_cast<uint32_t *>(wbuf);  // packed-count scans
  __shared__ int scal[2];
  __shared__ int part[2];  // this CTA's (greater, equal) totals
  __shared__ int pre[2];   // cluster rows: (greater, equal) totals of the lower ranks (pushed)
  int rank = 0;
  if constexpr (CLN > 1) rank = (int)cg::this_cluster().block_rank();
  const int len = (int)min((int64_t)lens[b / sp.len_div], ld);  // a len past the row stride reads no further
  const float *row = logits + (int64_t)b * ld;
  int32_t *o = out + (int64_t)b * out_ld;
  const int chunk = (((len + CLN - 1) / CLN) + 3) & ~3;
  const int beg = min(len, rank * chunk), end = min(len, beg + chunk);
  const int n = end - beg;
  if (len <= k) {  // whole row, ascending (uniform across the cluster: no cluster sync)
    for (int i = beg + threadIdx.x; i < end; i += NT) o[i] = i;
    if (rank == 0 && threadIdx.x == 0) counts[b] = len < 0 ? 0 : len;
    if (sp.slot_of) {
      if constexpr (CLN > 1) {
        cg::this_cluster().sync();  // every rank's ids written (release / acquire)
        if (rank == 0) split_tail(b, o, max(len, 0), sp, wbuf);
      } else {
        split_tail(b, o, max(len, 0), sp, wbuf);
      }
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  KPROF(0);
  for (int i = threadIdx.x; i < D1_BINS; i += NT) hist[i] = 0;
  if constexpr (CLN > 1) {
    for (int i = threadIdx.x; i < D1_BINS; i += NT) csum[i] = 0;
    if (threadIdx.x < 2) pre[threadIdx.x] = 0;
    cluster_arrive();  // csum / pre zeroed; peers push into them after the matching wait
  }
  __syncthreads();

  // ---- stage the slice as keys + first-digit histogram (8 loads in flight) ----------
  const float *src = row + beg;
  const bool vec_ok = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(logits) & 15) == 0);
  {
    constexpr int U = 8;
    const int n4 = vec_ok ? (n & ~3) : 0;
    for (int i0 = threadIdx.x * VEC; i0 < n4; i0 += NT * VEC * U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int i = i0 + u * NT * VEC;
        if (i < n4) {
          if constexpr (STREAM) v[u] = __ldcg(reinterpret_cast<const float4 *>(src + i));
          else v[u] = __ldg(reinterpret_cast<const float4 *>(src + i));
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int i = i0 + u * NT * VEC;
        if (i < n4) {
          const uint4 kk = make_uint4(score_key(v[u].x), score_key(v[u].y), score_key(v[u].z),
                                      score_key(v[u].w));
          *reinterpret_cast<uint4 *>(skey + i) = kk;
          atomicAdd(&hist[kk.x >> D1_SHIFT], 1);
          atomicAdd(&hist[kk.y >> D1_SHIFT], 1);
          atomicAdd(&hist[kk.z >> D1_SHIFT], 1);
          atomicAdd(&hist[kk.w >> D1_SHIFT], 1);
        }
      }
    }
    for (int i = n4 + threadIdx.x; i < n; i += NT) {
      const uint32_t key = score_key(STREAM ? __ldcg(src + i) : src[i]);
      skey[i] = key;
      atomicAdd(&hist[key >> D1_SHIFT], 1);
    }
  }
  KPROF(1);
  if constexpr (CLN > 1) {
    __syncthreads();  // this slice's histogram complete
    cluster_wait();   // every rank's csum zeroed
    uint32_t rb[CLN];
#pragma unroll
    for (int r = 0; r < CLN; r++) rb[r] = cluster_addr(csum, r);
    for (int i = threadIdx.x; i < D1_BINS; i += NT) {
      const int v = hist[i];
      if (v) {
#pragma unroll
        for (int r = 0; r < CLN; r++) cluster_red_add(rb[r] + 4 * i, v);
      }
    }
    cluster_sync<CLN>();  // every push landed
    pick_digit<D1_BINS>(csum, k, wbuf, scal);
  } else {
    __syncthreads();
    pick_digit<D1_BINS>(hist, k, wbuf, scal);
  }
  const uint32_t d1 = (uint32_t)scal[0];
  int rem = scal[1];

  KPROF(2);
  // ---- list = slice keys with first digit >= d1, in row order -----------------------
  const int cw = (((n + NW - 1) / NW) + 31) & ~31;
  const int lo = min(n, warp * cw), hi = min(n, lo + cw);
  // the list pass: warp-contiguous runs of whole 128-key chunks (n rounds up to a
  // multiple of 4 inside the slice allocation; keys past n are masked by hi4 = n)
  const int cw4 = (((n + NW - 1) / NW) + 127) & ~127;
  const int lo4 = min(n, warp * cw4), hi4 = min(n, lo4 + cw4);
  // One pass: each warp appends its run's candidates to its own segment of the list
  // (RCAP entries), so no block-wide scan or second pass is needed; segments in warp
  // order are in row order.  128-key chunks: each lane reads 4 consecutive keys with
  // one 16-B shared load and the 4 ballots give every key's rank in row order.
  uint16_t *myseg = list + warp * RCAP;
  const int trash = LCAP + threadIdx.x - warp * RCAP;  // list[LCAP + thread], relative to myseg
  int cnt = 0;
#pragma unroll LIST_UNROLL
  for (int i = lo4; i < hi4; i += 128) {
    const int j = i + lane * 4;
    // lanes past the run read nothing (slice_cap is 4-aligned, so j < hi4 keeps the
    // 16-B read inside the staged slice, never into the list behind it)
    const uint4 kv = j < hi4 ? *reinterpret_cast<const uint4 *>(skey + j) : make_uint4(0, 0, 0, 0);
    const bool c0 = j + 0 < hi4 && (kv.x >> D1_SHIFT) >= d1;
    const bool c1 = j + 1 < hi4 && (kv.y >> D1_SHIFT) >= d1;
    const bool c2 = j + 2 < hi4 && (kv.z >> D1_SHIFT) >= d1;
    const bool c3 = j + 3 < hi4 && (kv.w >> D1_SHIFT) >= d1;
    const uint32_t b0 = __ballot_sync(0xffffffffu, c0), b1 = __ballot_sync(0xffffffffu, c1);
    const uint32_t b2 = __ballot_sync(0xffffffffu, c2), b3 = __ballot_sync(0xffffffffu, c3);
    // branch-free: non-candidates (and overflow) store to this thread's trash entry
    const int p0 = cnt + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
    const int p1 = p0 + c0, p2 = p1 + c1, p3 = p2 + c2;
    myseg[c0 && p0 < RCAP ? p0 : trash] = (uint16_t)(j + 0);
    myseg[c1 && p1 < RCAP ? p1 : trash] = (uint16_t)(j + 1);
    myseg[c2 && p2 < RCAP ? p2 : trash] = (uint16_t)(j + 2);
    myseg[c3 && p3 < RCAP ? p3 : trash] = (uint16_t)(j + 3);
    cnt += __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
  }
  KPROF(8);
  // a segment overflowed (candidates bunched in one run, e.g. sorted rows): one
  // contiguous list from the per-warp counts (scan + second pass), or, past LCAP
  // entries (mass ties), full-slice passes
  const bool seg = !__syncthreads_or(cnt > RCAP);
  int m = 0;
  bool use_l = true;
  if (!seg) {
    int base = block_exclusive_scan<NT>(lane ? 0 : cnt, wbuf, &m);
    base = __shfl_sync(0xffffffffu, base, 0);
    use_l = m <= LCAP;
    if (use_l) {
#pragma unroll LIST_UNROLL
      for (int i = lo4; i < hi4; i += 128) {
        const int j = i + lane * 4;
        const uint4 kv = j < hi4 ? *reinterpret_cast<const uint4 *>(skey + j) : make_uint4(0, 0, 0, 0);
        const bool c0 = j + 0 < hi4 && (kv.x >> D1_SHIFT) >= d1;
        const bool c1 = j + 1 < hi4 && (kv.y >> D1_SHIFT) >= d1;
        const bool c2 = j + 2 < hi4 && (kv.z >> D1_SHIFT) >= d1;
        const bool c3 = j + 3 < hi4 && (kv.w >> D1_SHIFT) >= d1;
        const uint32_t b0 = __ballot_sync(0xffffffffu, c0), b1 = __ballot_sync(0xffffffffu, c1);
        const uint32_t b2 = __ballot_sync(0xffffffffu, c2), b3 = __ballot_sync(0xffffffffu, c3);
        int pos = base + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
        if (c0) list[pos++] = (uint16_t)(j + 0);
        if (c1) list[pos++] = (uint16_t)(j + 1);
        if (c2) list[pos++] = (uint16_t)(j + 2);
        if (c3) list[pos++] = (uint16_t)(j + 3);
        base += __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
      }
    }
  }
#ifdef ESS_TOPK_PROF
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_topk_prof[blockIdx.x][7] = (unsigned long long)(seg ? 0 : m);
#endif
  KPROF(9);
  // the candidates: this warp's segment (seg), the contiguous list, or the whole slice
  const int len2 = seg ? cnt : (use_l ? m : n);
  const int i0 = seg ? lane : threadIdx.x, istep = seg ? 32 : NT;
  auto cand = [&](int i) -> int { return seg ? myseg[i] : (use_l ? list[i] : i); };

  KPROF(3);
  // ---- two 10-bit digits inside bin d1 ------------------------------------------------
  uint32_t prefix = d1 << D1_SHIFT, mask = ~0u << D1_SHIFT;
  if constexpr (CLN > 1) {
    // both 10-bit passes' sums (csum[0:1024], csum[1024:2048]) zeroed after this CTA's
    // first-digit pick; one cluster barrier covers the zeroing and every rank's pick
    csum[threadIdx.x] = 0;
    csum[DR_BINS + threadIdx.x] = 0;
    cluster_sync<CLN>();
  }
  for (int shift = DR_BITS; shift >= 0; shift -= DR_BITS) {
    if constexpr (CLN > 1) {
      int *dsum = csum + (shift ? 0 : DR_BINS);  // this pass's buffer (no peer reads it yet)
      uint32_t rb[CLN];
#pragma unroll
      for (int r = 0; r < CLN; r++) rb[r] = cluster_addr(dsum, r);
      for (int i = i0; i < len2; i += istep) {
        const uint32_t key = skey[cand(i)];
        if ((key & mask) == prefix) {
          const uint32_t off = 4u * ((key >> shift) & (DR_BINS - 1));
#pragma unroll
          for (int r = 0; r < CLN; r++) cluster_red_add(rb[r] + off, 1);
        }
      }
      cluster_sync<CLN>();  // every push landed
      pick_digit<DR_BINS>(dsum, rem, wbuf, scal);
    } else {
      hist[threadIdx.x] = 0;
      __syncthreads();
      for (int i = i0; i < len2; i += istep) {
        const uint32_t key = skey[cand(i)];
        if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & (DR_BINS - 1)], 1);
      }
      __syncthreads();
      pick_digit<DR_BINS>(hist, rem, wbuf, scal);
    }
    prefix |= (uint32_t)scal[0] << shift;
    mask |= (uint32_t)(DR_BINS - 1) << shift;
    rem = scal[1];
  }
  const uint32_t T = prefix;
  const int need_eq = rem;  // keys == T to take, in index order over the whole row

  KPROF(4);
  // ---- this slice's (greater, equal) counts and their cluster prefix ------------------
  int gb = 0, eb = 0;
  uint32_t fb_ex = 0;  // packed (greater, equal) prefix of the lower warps
  if (seg) {  // per-warp counts; their prefix orders the segments' emits
    int g = 0, q = 0;
    for (int i = lane; i < cnt; i += 32) {
      const uint32_t key = skey[myseg[i]];
      g += key > T;
      q += key == T;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      g += __shfl_xor_sync(0xffffffffu, g, d);
      q += __shfl_xor_sync(0xffffffffu, q, d);
    }
    uint32_t tot;
    fb_ex = block_exclusive_scan<NT>(lane ? 0u : pack_gq(g, q), uwbuf, &tot);
    fb_ex = __shfl_sync(0xffffffffu, fb_ex, 0);
    if (threadIdx.x == 0) {
      part[0] = (int)(tot & 0xFFFFu);
      part[1] = (int)(tot >> 16);
    }
  } else if (use_l) {
    if constexpr (CLN > 1) {
      int g = 0, q = 0;
      for (int i = threadIdx.x; i < m; i += NT) {
        const uint32_t key = skey[list[i]];
        g += key > T;
        q += key == T;
      }
      uint32_t tot;
      block_exclusive_scan<NT>(pack_gq(g, q), uwbuf, &tot);
      if (threadIdx.x == 0) {
        part[0] = (int)(tot & 0xFFFFu);
        part[1] = (int)(tot >> 16);
      }
    }
  } else {
    int g, q;
    uint32_t tot;
    run_counts(skey, lo, hi, T, g, q);
    fb_ex = block_exclusive_scan<NT>(lane ? 0u : pack_gq(g, q), uwbuf, &tot);
    fb_ex = __shfl_sync(0xffffffffu, fb_ex, 0);
    if (threadIdx.x == 0) {
      part[0] = (int)(tot & 0xFFFFu);
      part[1] = (int)(tot >> 16);
    }
  }
  if constexpr (CLN > 1) {
    // add this slice's totals into every higher rank's prefix, one barrier, read ours
    __syncthreads();  // part written
    if (threadIdx.x == 0) {
      for (int r = rank + 1; r < CLN; r++) {
        const uint32_t a = cluster_addr(pre, r);
        cluster_red_add(a, part[0]);
        cluster_red_add(a + 4, part[1]);
      }
    }
    cluster_sync<CLN>();
    gb = pre[0];
    eb = pre[1];
  }

  KPROF(5);
  // ---- ordered emit: every key > T and the first need_eq keys == T --------------------
  if (seg) {
    int gw = gb + (int)(fb_ex & 0xFFFFu), ew = eb + (int)(fb_ex >> 16);
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int i = c0 + lane;
      const int j = i < cnt ? myseg[i] : 0;
      const uint32_t key = i < cnt ? skey[j] : 0u;
      const bool gt = i < cnt && key > T, eq = i < cnt && key == T;
      const uint32_t mg = __ballot_sync(0xffffffffu, gt), me = __ballot_sync(0xffffffffu, eq);
      const int e = ew + __popc(me & lt);
      if (gt || (eq && e < need_eq)) o[gw + __popc(mg & lt) + min(e, need_eq)] = beg + j;
      gw += __popc(mg);
      ew += __popc(me);
    }
  } else if (use_l) {
    for (int c0 = 0; c0 < m; c0 += NT) {
      const int i = c0 + threadIdx.x;
      const int j = i < m ? list[i] : 0;
      const uint32_t key = i < m ? skey[j] : 0u;
      const bool gt = i < m && key > T, eq = i < m && key == T;
      uint32_t tot;
      const uint32_t ex = block_exclusive_scan<NT>(pack_gq(gt, eq), uwbuf, &tot);
      const int e = eb + (int)(ex >> 16);
      if (gt || (eq && e < need_eq)) o[gb + (int)(ex & 0xFFFFu) + min(e, need_eq)] = beg + j;
      gb += (int)(tot & 0xFFFFu);
      eb += (int)(tot >> 16);
    }
  } else {
    run_emit(skey, lo, hi, T, need_eq, gb + (int)(fb_ex & 0xFFFFu), eb + (int)(fb_ex >> 16), beg, o);
  }
  KPROF(6);
  if (rank == 0 && threadIdx.x == 0) counts[b] = k;
  if (sp.slot_of) {
    if constexpr (CLN > 1) {
      cg::this_cluster().sync();  // every rank's part of the selection written
      if (rank == 0) split_tail(b, o, k, sp, wbuf);
    } else {
      split_tail(b, o, k, sp, wbuf);
    }
    if (threadIdx.x == 0 && rank == 0) SPROF(sp.prof_base + b, 1);
  }
  KPROF(10);
}

template <int CLN>
__global__ void __launch_bounds__(NT, 1)
    topk_kernel(const float *__restrict__ logits, int64_t ld, const int32_t *__restrict__ lens,
                int k, int32_t *__restrict__ out, int out_ld, int32_t *__restrict__ counts,
                SplitArgs sp) {
  ess_pdl_trigger();  // a PDL-launched consumer (the gather) may become resident now
  ess_pdl_wait();     // PDL-launched: the indexer's logits complete and visible
  topk_row<CLN, false>(blockIdx.x / CLN, logits, ld, lens, k, out, out_ld, counts, sp);
}

// Streamed step (K2 + K3a): a persistent grid walks the requests in order (CTA c takes
// c, c + grid, ...); row b starts once the concurrent indexer has published all its
// logits (done[b] == min(len, ld)); after the top-k and the hit/miss split the CTA
// publishes ready[b] = 1 (release) for the streamed gather.  CLN-CTA clusters per row
// (CLN = 2 halves a row's latency: the first rows gate the host link).
template <int CLN>
__global__ void __launch_bounds__(NT, 1)
    topk_stream_kernel(const float *__restrict__ logits, int64_t ld, const int32_t *__restrict__ lens,
                       int B, int k, int32_t *__restrict__ out, int out_ld,
                       int32_t *__restrict__ counts, SplitArgs sp, const int32_t *done, int32_t *ready) {
  const int nclu = gridDim.x / CLN;
  for (int b = blockIdx.x / CLN; b < B; b += nclu) {
    __syncthreads();  // the previous row's shared-memory readers are done
    if (threadIdx.x < 32) ess_warp_wait_geq(done + b, (int)min((int64_t)lens[b], ld));
    __syncthreads();
    if (threadIdx.x == 0) SPROF(sp.prof_base + b, 0);
    topk_row<CLN, true>(b, logits, ld, lens, k, out, out_ld, counts, sp);
    __threadfence();  // this thread's selection / split outputs, before the flag
    if constexpr (CLN > 1) cg::this_cluster().sync();  // every rank's part (rank 0 split)
    else __syncthreads();
    if (threadIdx.x == 0 && (CLN == 1 || cg::this_cluster().block_rank() == 0)) {
      ess_st_release(ready + b, 1);
      SPROF(sp.prof_base + b, 1);
    }
  }
}

template <int CLN>
int launch_topk(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch, int32_t k,
                int32_t *d_idx, int32_t idx_ld, int32_t *d_count, cudaStream_t stream,
                SplitArgs sp = SplitArgs{}, bool pdl = false) {
  const size_t smem = (size_t)slice_cap<CLN>(ld) * sizeof(uint32_t) + (LCAP + NT) * sizeof(uint16_t);
  // per (instantiation, device): opt in to the largest slice
  if (int rc = ess_smem_optin((const void *)topk_kernel<CLN>,
                              SLICE_MAX * sizeof(uint32_t) + (LCAP + NT) * sizeof(uint16_t)))
    return rc;
  ESS_CUDA_TRY(ess_launch(topk_kernel<CLN>, dim3((unsigned)batch * CLN), dim3(NT), smem, stream, CLN, pdl,
                          d_logits, ld, d_len, (int)k, d_idx, (int)idx_ld, d_count, sp));
  return ESS_OK;
}

}  // namespace

namespace {

int topk_rows(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t rows, int32_t len_div,
              int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count, void *stream) {
  if (!d_logits || !d_len || !d_idx || !d_count || rows < 0 || k < 1 || k > ESS_TOPK_MAX_K ||
      idx_ld < k || ld < 1 || len_div < 1)
    return ESS_ERR_ARG;
  if (rows == 0) return ESS_OK;
  // Cluster size: the smallest that fits a slice in shared memory.  Growing it to fill
  // idle SMs does not pay: 1024-thread CTAs are register-limited to one per SM and the
  // DSMEM histogram sums cost more than the shorter slices save (profiles/README.md).
  int cln = 1;
  while (cln < 8 && (ld + cln - 1) / cln > SLICE_MAX) cln *= 2;
  // A/B switch (scratch timing): a minimum cluster size per row
  static const int min_cln = [] {
    const char *e = getenv("ESS_TOPK_MIN_CLUSTER");
    int v = e ? atoi(e) : 1;
    return v == 2 || v == 4 || v == 8 ? v : 1;
  }();
  while (cln < min_cln) cln *= 2;
  if ((ld + cln - 1) / cln > SLICE_MAX) return ESS_ERR_ARG;  // rows longer than 320K tokens
  cudaStream_t s = (cudaStream_t)stream;
  SplitArgs sp{};
  sp.slot_of = nullptr;
  sp.len_div = len_div;
  int rc;
  switch (cln) {
    case 1: rc = launch_topk<1>(d_logits, ld, d_len, rows, k, d_idx, idx_ld, d_count, s, sp); break;
    case 2: rc = launch_topk<2>(d_logits, ld, d_len, rows, k, d_idx, idx_ld, d_count, s, sp); break;
    case 4: rc = launch_topk<4>(d_logits, ld, d_len, rows, k, d_idx, idx_ld, d_count, s, sp); break;
    default: rc = launch_topk<8>(d_logits, ld, d_len, rows, k, d_idx, idx_ld, d_count, s, sp); break;
  }
  if (rc != ESS_OK) return rc;
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

}  // namespace

extern "C" int ess_topk(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch,
                        int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count,
                        void *stream) {
  return topk_rows(d_logits, ld, d_len, batch, 1, k, d_idx, idx_ld, d_count, stream);
}

// MTP: batch * qtok rows (request-major), row b*qtok + j scored over len[b] tokens.
extern "C" int ess_topk_mtp(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch,
                            int32_t qtok, int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count,
                            void *stream) {
  if (qtok < 1 || qtok > ESS_INDEXER_MAX_QTOK || batch < 0) return ESS_ERR_ARG;
  return topk_rows(d_logits, ld, d_len, batch * qtok, qtok, k, d_idx, idx_ld, d_count, stream);
}

// Top-k fused with the early-gather hit/miss split (ess_pool_split) of pools
// [pool_begin, pool_begin + batch) in one launch (cluster rows: rank 0 splits after a
// cluster barrier).
extern "C" int ess_topk_split(const float *d_logits, int64_t ld, const int32_t *d_len,
                              int32_t batch, int32_t k, int32_t *d_idx, int32_t idx_ld,
                              int32_t *d_count, ess_pool *pool, int32_t pool_begin,
                              int32_t *d_hit_row, int32_t *d_miss_ids, int32_t *d_miss_row,
                              int32_t *d_counts, int32_t out_stride, void *stream) {
  return ess_topk_split_ex(d_logits, ld, d_len, batch, k, d_idx, idx_ld, d_count, pool, pool_begin,
                           d_hit_row, d_miss_ids, d_miss_row, d_counts, out_stride, 0, stream);
}

extern "C" int ess_topk_split_ex(const float *d_logits, int64_t ld, const int32_t *d_len,
                                 int32_t batch, int32_t k, int32_t *d_idx, int32_t idx_ld,
                                 int32_t *d_count, ess_pool *pool, int32_t pool_begin,
                                 int32_t *d_hit_row, int32_t *d_miss_ids, int32_t *d_miss_row,
                                 int32_t *d_counts, int32_t out_stride, int32_t flags, void *stream) {
  if (flags & ~ESS_LAUNCH_PDL) return ESS_ERR_ARG;
  const bool pdl = (flags & ESS_LAUNCH_PDL) != 0;
  if (!pool || pool_begin < 0 || (int64_t)pool_begin + batch > pool->P || !d_hit_row ||
      !d_miss_ids || !d_miss_row || !d_counts || out_stride < 1 || k > 2 * NT ||
      pool->staging < k)
    return ESS_ERR_ARG;
  if (!d_logits || !d_len || !d_idx || !d_count || batch < 0 || k < 1 || idx_ld < k || ld < 1)
    return ESS_ERR_ARG;
  if (batch == 0) return ESS_OK;
  int cln = 1;
  while (cln < 8 && (ld + cln - 1) / cln > SLICE_MAX) cln *= 2;
  if ((ld + cln - 1) / cln > SLICE_MAX) return ESS_ERR_ARG;
  SplitArgs sp;
  sp.slot_of = pool->slot_of + (int64_t)pool_begin * pool->max_ids;
  sp.max_ids = pool->max_ids;
  sp.cap_max = pool->cap_max;
  sp.hit_row = d_hit_row;
  sp.miss_ids = d_miss_ids;
  sp.miss_row = d_miss_row;
  sp.counts = d_counts;
  sp.out_stride = out_stride;
  sp.prof_base = pool_begin;
  // cluster rows: rank 0 of each cluster runs the split after a cluster barrier
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  switch (cln) {
    case 1: rc = launch_topk<1>(d_logits, ld, d_len, batch, k, d_idx, idx_ld, d_count, st, sp, pdl); break;
    case 2: rc = launch_topk<2>(d_logits, ld, d_len, batch, k, d_idx, idx_ld, d_count, st, sp, pdl); break;
    case 4: rc = launch_topk<4>(d_logits, ld, d_len, batch, k, d_idx, idx_ld, d_count, st, sp, pdl); break;
    default: rc = launch_topk<8>(d_logits, ld, d_len, batch, k, d_idx, idx_ld, d_count, st, sp, pdl); break;
  }
  if (rc != ESS_OK) return rc;
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

// Streamed K2 + K3a (see topk_stream_kernel): rows <= 40K tokens (one CTA per row),
// `ctas` persistent CTAs; d_done from ess_indexer_logits_stream, d_ready [batch] zero
// at launch, set to 1 per request once its selection, split rows and counts are stored.
extern "C" int ess_topk_split_stream(const float *d_logits, int64_t ld, const int32_t *d_len,
                                     int32_t batch, int32_t k, int32_t *d_idx, int32_t idx_ld,
                                     int32_t *d_count, ess_pool *pool, int32_t pool_begin,
                                     int32_t *d_hit_row, int32_t *d_miss_ids, int32_t *d_miss_row,
                                     int32_t *d_counts, int32_t out_stride, const int32_t *d_done,
                                     int32_t *d_ready, int32_t ctas, void *stream) {
  if (!pool || pool_begin < 0 || (int64_t)pool_begin + batch > pool->P || !d_hit_row ||
      !d_miss_ids || !d_miss_row || !d_counts || out_stride < 1 || k > 2 * NT ||
      pool->staging < k || !d_done || !d_ready || ctas == 0)
    return ESS_ERR_ARG;
  if (!d_logits || !d_len || !d_idx || !d_count || batch < 0 || k < 1 || idx_ld < k || ld < 1 ||
      (ld + 7) / 8 > SLICE_MAX)
    return ESS_ERR_ARG;
  if (batch == 0) return ESS_OK;
  SplitArgs sp{};
  sp.slot_of = pool->slot_of + (int64_t)pool_begin * pool->max_ids;
  sp.max_ids = pool->max_ids;
  sp.cap_max = pool->cap_max;
  sp.hit_row = d_hit_row;
  sp.miss_ids = d_miss_ids;
  sp.miss_row = d_miss_row;
  sp.counts = d_counts;
  sp.out_stride = out_stride;
  sp.prof_base = pool_begin;
  // cluster size per row: the smallest whose slice fits shared memory (rows > 40K tokens
  // take 2-8 CTAs, as ess_topk); ctas < 0 forces at least CTA pairs.  `ctas` counts rows
  // worked on at once (clusters).
  int cln = 1;
  while (cln < 8 && (ld + cln - 1) / cln > SLICE_MAX) cln *= 2;
  if (ctas < 0 && cln < 2) cln = 2;
  int nclu = ctas < 0 ? -ctas : ctas;
  if (nclu > batch) nclu = batch;
  const size_t smem = (size_t)(cln == 1 ? slice_cap<1>(ld) : cln == 2 ? slice_cap<2>(ld)
                               : cln == 4 ? slice_cap<4>(ld) : slice_cap<8>(ld)) * sizeof(uint32_t) +
                      (LCAP + NT) * sizeof(uint16_t);
  const void *kern = cln == 1 ? (const void *)topk_stream_kernel<1> : cln == 2 ? (const void *)topk_stream_kernel<2>
                     : cln == 4 ? (const void *)topk_stream_kernel<4> : (const void *)topk_stream_kernel<8>;
  if (int rc = ess_smem_optin(kern, SLICE_MAX * sizeof(uint32_t) + (LCAP + NT) * sizeof(uint16_t))) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclu * cln));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cln;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (cln) {
    case 1:
      ESS_CUDA_TRY(cudaLaunchKernelEx(&cfg, topk_stream_kernel<1>, d_logits, ld, d_len, (int)batch, (int)k, d_idx,
                                      (int)idx_ld, d_count, sp, d_done, d_ready));
      break;
    case 2:
      ESS_CUDA_TRY(cudaLaunchKernelEx(&cfg, topk_stream_kernel<2>, d_logits, ld, d_len, (int)batch, (int)k, d_idx,
                                      (int)idx_ld, d_count, sp, d_done, d_ready));
      break;
    case 4:
      ESS_CUDA_TRY(cudaLaunchKernelEx(&cfg, topk_stream_kernel<4>, d_logits, ld, d_len, (int)batch, (int)k, d_idx,
                                      (int)idx_ld, d_count, sp, d_done, d_ready));
      break;
    default:
      ESS_CUDA_TRY(cudaLaunchKernelEx(&cfg, topk_stream_kernel<8>, d_logits, ld, d_len, (int)batch, (int)k, d_idx,
                                      (int)idx_ld, d_count, sp, d_done, d_ready));
      break;
  }
  return ESS_OK;
}

#ifdef ESS_STREAM_PROF
ESS_STREAM_PROF_READER(ess_debug_stream_prof_topk)
#endif

int ess_preload_topk() {  // see ess_preload_indexer
  cudaFuncAttributes a;
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_kernel<1>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_kernel<2>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_kernel<4>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_kernel<8>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_stream_kernel<1>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_stream_kernel<2>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_stream_kernel<4>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)topk_stream_kernel<8>));
  return ESS_OK;
}
