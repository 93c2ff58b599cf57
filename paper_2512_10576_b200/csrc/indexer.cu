// K1: lightning indexer (op "indexer_logits", costmodel.py:18-27).
//
//   logits[b][s] = kscale[b][s] * sum_h w[b][h] * relu(q[b][h] . k[b][s])
//
// The head contraction is a real GEMM per 128-token tile: D[128 tok][64 heads] =
// K_tile[128 x 128 e4m3] . Q[64 x 128 e4m3]^T, issued as tcgen05.mma kind::f8f6f4
// (M=128, N=64, 4 x K=32) by one thread into TMEM.  The pipeline moves 256-token
// UNITS (two MMA tiles, one 32-KB ring stage, one barrier round, one TMEM
// accumulator of 128 columns): with 128-token units the per-unit barrier / commit /
// TMEM hand-off chain, not HBM, set the rate (K1 scaled linearly with the number of
// SMs; profiles/README.md), and doubling the unit took C2 from 68 to 55 us and C4
// from 228 to 178 us (98% of the measured copy bandwidth).  TMA (SWIZZLE_128B)
// streams K tiles through a 5-stage ring; q is loaded once per request into one of
// two slots.  The kernel is persistent (one CTA per SM, contiguous unit ranges) and
// HBM-bound: 132 B/token in, 4 B out.
//
// Warp roles (320 threads): w0 TMA producer, w1 TMEM alloc + MMA issuer,
// w2..w9 epilogue in two groups taking alternate units (TMEM lane quarter =
// warp % 4); head weights stay in registers while the request does not change.
#include <cuda.h>

#include "common.cuh"

namespace {

#ifndef ESS_K1_SUB
#define ESS_K1_SUB 2
#endif
#ifndef ESS_K1_MTP_STAGES  // MTP instantiations (QT > 1); 0 = per-QT default
#define ESS_K1_MTP_STAGES 0
#endif
#ifndef ESS_K1_STAGES
#define ESS_K1_STAGES (ESS_K1_SUB == 1 ? 10 : 3)
#endif
constexpr int TILE_M = 128;                 // tokens per MMA tile (M)
constexpr int HEADS = ESS_INDEXER_HEADS;    // 64 heads per query token
constexpr int DIM = ESS_INDEXER_DIM;        // 128 = K (bytes, e4m3)
constexpr int KT_BYTES = TILE_M * DIM;      // 16 KB per MMA tile
constexpr int NEPI = 8;                     // epilogue warps: 2 groups x 4 lane quarters
constexpr int NTHREADS = 32 * (2 + NEPI);
constexpr int MAX_BATCH = 4096;

// Per query-token count QT (1 = plain decode; QT = mtp + 1 query tokens per request,
// pipeline.py:213-215): the QT tokens of a request share its key stream, so one MMA
// with N = 64 * QT (all tokens' heads) consumes each key tile once — the indexer reads
// the keys once per request whatever the MTP width.  QT = 1 keeps the 256-token units
// (two MMA tiles per stage); QT > 1 has QT x the epilogue work per tile, so one tile
// per unit already amortises the barrier chain.
template <int QT>
struct K1Cfg {
  static constexpr int SUB = QT == 1 ? ESS_K1_SUB : 1;         // MMA tiles per unit
  static constexpr int UNIT_M = SUB * TILE_M;                  // tokens per unit
  static constexpr int STAGES = QT == 1 ? ESS_K1_STAGES : ESS_K1_MTP_STAGES > 0 ? ESS_K1_MTP_STAGES : (QT == 2 ? 10 : 8);
  static constexpr int N = HEADS * QT;                         // MMA N (all tokens' heads)
  static constexpr int UT_BYTES = SUB * KT_BYTES;
  static constexpr int QT_BYTES = N * DIM;                     // one request's q (x2 slots)
  static constexpr int ACC_COLS = SUB * N;                     // TMEM columns per unit
  static constexpr int NACC = 512 / ACC_COLS < 4 ? 512 / ACC_COLS : 4;
  static constexpr int TMEM_USED = NACC * ACC_COLS;
  static constexpr int TMEM_COLS = TMEM_USED <= 32 ? 32 : TMEM_USED <= 64 ? 64 : TMEM_USED <= 128 ? 128
                                   : TMEM_USED <= 256 ? 256 : 512;
  static constexpr uint32_t IDESC = make_idesc(0 /*e4m3*/, 0 /*e4m3*/, TILE_M, N, 0, 0);
  struct Ctrl {
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint64_t qfull[2];
    uint64_t qempty[2];
    uint64_t tfull[NACC];
    uint64_t tempty[NACC];
    uint32_t tmem;
    int pref[MAX_BATCH + 1];
    alignas(16) float wq[2][QT > 1 ? QT * HEADS : 4];  // QT > 1: each epilogue group's head weights
  };
  static constexpr size_t SMEM_BYTES =
      1024 /*align slack*/ + (size_t)STAGES * UT_BYTES + 2 * QT_BYTES + sizeof(Ctrl);
  static_assert(SMEM_BYTES <= 232448, "K1 shared memory over the sm_100 limit");
  static_assert(N <= 256 && N % 16 == 0, "MMA N out of range");
};

#ifdef ESS_K1_PROF  // scratch builds: per-CTA globaltimer stamps (entry, setup, first unit, end)
__device__ unsigned long long g_k1_prof[160][6];
__device__ __forceinline__ void k1_stamp(int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#ifdef ESS_K1_PROF_FULLGRID  // the latest full-grid launch (the step's first micro-batch)
  if (blockIdx.x < 160 && gridDim.x >= 148) g_k1_prof[blockIdx.x][i] = t;
#else  // first launch after a reset wins (the step launches K1 once per micro-batch)
  if (blockIdx.x < 160 && g_k1_prof[blockIdx.x][i] == 0) g_k1_prof[blockIdx.x][i] = t;
#endif
}
#define K1PROF(i) k1_stamp(i)
#else
#define K1PROF(i) \
  do {            \
  } while (0)
#endif

// Walk the flattened (request, unit) sequence.
struct TileCursor {
  int b, t;
  __device__ void seek(const int *pref, int B, int idx) {
    int lo = 0, hi = B - 1;
    while (lo < hi) {  // last b with pref[b] <= idx
      int mid = (lo + hi + 1) >> 1;
      if (pref[mid] <= idx) lo = mid; else hi = mid - 1;
    }
    b = lo;
    t = idx - pref[lo];
  }
  __device__ void next(const int *pref, int B) {
    t++;
    while (b < B && pref[b] + t >= pref[b + 1]) {
      t = t - (pref[b + 1] - pref[b]);
      b++;
    }
  }
};

// The CTA's share of the flattened (request, unit) sequence.  Requests form groups of
// `rg` (rg >= B: one group, the plain persistent split); the CTA takes its contiguous
// slice of every group's units, group after group, so the whole grid finishes the
// requests of group 0 first — the streamed step's top-k starts on them while the
// indexer still runs (per-request completion counters, ess_indexer_logits_stream).
struct UnitSeq {
  int g, ngroups, rg, rg0, B, grid, cta, idx, end;
  TileCursor cur;
  // group gg: requests [b0, b1) — the first group has rg0 requests, the others rg
  __device__ int group_begin(int gg) const { return gg == 0 ? 0 : min(B, rg0 + (gg - 1) * rg); }
  __device__ bool slice(const int *pref, int gg, int &s, int &e) const {
    const int b0 = group_begin(gg), b1 = group_begin(gg + 1);
    const int u0 = pref[b0], tot = pref[b1] - u0;
    s = u0 + (int)((int64_t)tot * cta / grid);
    e = u0 + (int)((int64_t)tot * (cta + 1) / grid);
    return s < e;
  }
  __device__ void open(const int *pref) {  // the first non-empty slice from group g on
    for (; g < ngroups; g++) {
      int s0, e0;
      if (slice(pref, g, s0, e0)) {
        idx = s0;
        end = e0;
        cur.seek(pref, B, s0);
        return;
      }
    }
  }
  __device__ void start(const int *pref, int B_, int rg_, int rg0_) {
    B = B_;
    rg = rg_;
    rg0 = rg0_ < rg_ ? rg0_ : rg_;
    ngroups = 1 + (B - rg0 + rg - 1) / rg;
    cta = blockIdx.x;
    grid = gridDim.x;
    g = 0;
    open(pref);
  }
  __device__ int count(const int *pref) const {
    int n = 0;
    for (int gg = 0; gg < ngroups; gg++) {
      int s0, e0;
      if (slice(pref, gg, s0, e0)) n += e0 - s0;
    }
    return n;
  }
  __device__ void next(const int *pref) {
    if (++idx < end) {
      cur.next(pref, B);
    } else {
      g++;
      open(pref);
    }
  }
};

__device__ __forceinline__ void group_bar(int g) {  // the 128 threads of epilogue group g
  asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
}

template <int QT>
__global__ void __launch_bounds__(NTHREADS, 1)
    indexer_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_q,
                   const float *__restrict__ w, const float *__restrict__ kscale,
                   const int32_t *__restrict__ lens, int B, int64_t k_ld, float *__restrict__ logits,
                   int rg, int32_t *done) {
  using C = K1Cfg<QT>;
  constexpr int SUB = C::SUB, UNIT_M = C::UNIT_M, STAGES = C::STAGES, NACC = C::NACC;
  constexpr int UT_BYTES = C::UT_BYTES, QT_BYTES = C::QT_BYTES, ACC_COLS = C::ACC_COLS;
  extern __shared__ uint8_t smem_raw[];
  // offset from the shared array itself (keeps the shared address space: LDS/STS, not generic)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *qbuf = smem + (size_t)STAGES * UT_BYTES;
  typename C::Ctrl &c = *reinterpret_cast<typename C::Ctrl *>(qbuf + 2 * QT_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) K1PROF(0);
  ess_pdl_trigger();  // a PDL-launched consumer (K2 + K3a) may take the SMs K1 leaves

  // unit prefix over requests (every CTA computes it): warp 0, 32 requests per round
  // (a serial loop of dependent-latency loads cost ~27 ns per request)
  if (warp == 0) {
    int acc = 0;
    for (int b0 = 0; b0 < B; b0 += 32) {
      const int b = b0 + lane;
      const int L = b < B ? min(__ldg(lens + b), (int)k_ld) : 0;
      const int u = L > 0 ? (L + UNIT_M - 1) / UNIT_M : 0;
      int x = u;  // inclusive warp scan
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (b < B) c.pref[b] = acc + x - u;
      acc += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) c.pref[B] = acc;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&c.full[s], 1);
      mbar_init(&c.empty[s], 1);
    }
    for (int s = 0; s < 2; s++) {
      mbar_init(&c.qfull[s], 1);
      mbar_init(&c.qempty[s], 1);
    }
    for (int a = 0; a < NACC; a++) {
      mbar_init(&c.tfull[a], 1);
      mbar_init(&c.tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&c.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) K1PROF(1);
  const uint32_t tmem = c.tmem;
  UnitSeq seq0;
  seq0.start(c.pref, B, rg & 0xFFFF, rg >> 16 ? rg >> 16 : rg & 0xFFFF);
  const int ntiles = seq0.count(c.pref);

  if (ntiles > 0) {
    if (warp == 0) {
      // ---- TMA producer: q once per request (2 slots), K units through the ring ----
      if (elect_one()) {
        prefetch_tmap(&tm_k);
        prefetch_tmap(&tm_q);
        const uint64_t kpol = l2_policy_evict_first();
        UnitSeq seq = seq0;
        const TileCursor &cur = seq.cur;
        int qs = 1, prev_b = -1, len_b = 0;
        uint32_t quse[2] = {0, 0};
        for (int it = 0; it < ntiles; it++) {
          if (cur.b != prev_b) {
            qs ^= 1;
            mbar_wait(&c.qempty[qs], (quse[qs] & 1) ^ 1);
            mbar_arrive_expect_tx(&c.qfull[qs], QT_BYTES);
            tma_load_2d(qbuf + qs * QT_BYTES, &tm_q, &c.qfull[qs], 0, cur.b * C::N);
            quse[qs]++;
            prev_b = cur.b;
            len_b = min(__ldg(lens + cur.b), (int)k_ld);
          }
          const int s = it % STAGES;
          // MMA tiles of this unit that hold tokens (the last unit may be short; its
          // missing tile is never loaded — the MMA reads stale rows, masked below)
          const int rem = len_b - cur.t * UNIT_M;
          const int nsub = rem >= UNIT_M ? SUB : (rem + TILE_M - 1) / TILE_M;
          mbar_wait(&c.empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&c.full[s], nsub * KT_BYTES);
          for (int j = 0; j < nsub; j++)
#ifndef ESS_K1_NO_EVICT_FIRST
            // keys are streamed once: evict-first keeps L2 for the logits K2 reads next
            tma_load_2d_hint(smem + (size_t)s * UT_BYTES + j * KT_BYTES, &tm_k, &c.full[s], 0,
                             (int32_t)(cur.b * k_ld + (int64_t)cur.t * UNIT_M + j * TILE_M), kpol);
#else
            tma_load_2d(smem + (size_t)s * UT_BYTES + j * KT_BYTES, &tm_k, &c.full[s], 0,
                        (int32_t)(cur.b * k_ld + (int64_t)cur.t * UNIT_M + j * TILE_M));
#endif
          seq.next(c.pref);
        }
      }
    } else if (warp == 1) {
      // ---- MMA issuer ---------------------------------------------------------------
      if (elect_one()) {
        UnitSeq seq = seq0;
        const TileCursor &cur = seq.cur;
        int qs = 1, prev_b = -1;
        uint32_t quse[2] = {0, 0};
        for (int it = 0; it < ntiles; it++) {
          if (cur.b != prev_b) {
            if (prev_b >= 0) tc_commit(&c.qempty[qs]);  // after the last MMA reading it
            qs ^= 1;
            mbar_wait(&c.qfull[qs], quse[qs] & 1);
            quse[qs]++;
            prev_b = cur.b;
          }
          const int s = it % STAGES;
          const int a = it % NACC;
          mbar_wait(&c.tempty[a], ((it / NACC) & 1) ^ 1);
          mbar_wait(&c.full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t qaddr = smem_u32(qbuf + qs * QT_BYTES);
#pragma unroll
          for (int j = 0; j < SUB; j++) {
            const uint32_t kaddr = smem_u32(smem + (size_t)s * UT_BYTES + j * KT_BYTES);
#pragma unroll
            for (int kk = 0; kk < DIM / 32; kk++) {
              uint64_t ad = sw128_desc(kaddr + kk * 32, 16, 1024);
              uint64_t bd = sw128_desc(qaddr + kk * 32, 16, 1024);
              mma_f8f6f4_ss(tmem + a * ACC_COLS + j * C::N, ad, bd, C::IDESC, kk > 0 ? 1u : 0u);
            }
          }
          tc_commit(&c.empty[s]);
          tc_commit(&c.tfull[a]);
          seq.next(c.pref);
        }
      }
    } else {
      // ---- epilogue: group g = units it % 2 == g; warp % 4 = TMEM lane quarter ------
      const int e = warp - 2;
      const int g = e >> 2;
      const int quarter = warp & 3;
      const int row = quarter * 32 + lane;
      UnitSeq seq = seq0;
      const TileCursor &cur = seq.cur;
      if (g == 1) seq.next(c.pref);
      int wb = -1, len_b = 0;
      int acc_b = seq.cur.b, acc_n = 0;  // streamed step: rows stored for request acc_b
      float wr[QT == 1 ? HEADS : 1];  // QT = 1: head weights in registers
      for (int it = g; it < ntiles; it += 2) {
        const int b = cur.b;
        if (b != wb) {  // head weights of this request
          if constexpr (QT == 1) {
            const float4 *src = reinterpret_cast<const float4 *>(w + (int64_t)b * HEADS);
#pragma unroll
            for (int h4 = 0; h4 < HEADS / 4; h4++) {
              float4 v = __ldg(src + h4);
              wr[4 * h4] = v.x;
              wr[4 * h4 + 1] = v.y;
              wr[4 * h4 + 2] = v.z;
              wr[4 * h4 + 3] = v.w;
            }
          } else {  // QT x 64 weights: the group's shared-memory copy (broadcast reads)
            group_bar(g);  // every thread of the group is done with the previous request
            for (int i = (e - 4 * g) * 32 + lane; i < QT * HEADS; i += 128)
              c.wq[g][i] = __ldg(w + (int64_t)b * QT * HEADS + i);
            group_bar(g);
          }
          len_b = min(__ldg(lens + b), (int)k_ld);
          wb = b;
        }
        int64_t off[SUB];
        bool valid[SUB];
        float ks[SUB];
#pragma unroll
        for (int j = 0; j < SUB; j++) {
          const int64_t tok = (int64_t)cur.t * UNIT_M + j * TILE_M + row;
          valid[j] = tok < len_b;
          off[j] = (int64_t)b * k_ld + tok;
          ks[j] = valid[j] ? __ldg(kscale + off[j]) : 0.f;
        }
        const int a = it % NACC;
        mbar_wait(&c.tfull[a], (it / NACC) & 1);
        tc_fence_after();
        if (it == 0 && threadIdx.x == 64) K1PROF(2);
        if constexpr (QT == 1) {
#pragma unroll
          for (int j = 0; j < SUB; j++) {
            uint32_t r[64];
            tmem_ld_32x32b_x64(tmem + ((uint32_t)(quarter * 32) << 16) + a * ACC_COLS + j * HEADS, r);
            tmem_ld_wait();
            if (j == SUB - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&c.tempty[a]);
            }
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
            for (int h = 0; h < HEADS; h += 4) {
              a0 = fmaf(wr[h + 0], fmaxf(__uint_as_float(r[h + 0]), 0.f), a0);
              a1 = fmaf(wr[h + 1], fmaxf(__uint_as_float(r[h + 1]), 0.f), a1);
              a2 = fmaf(wr[h + 2], fmaxf(__uint_as_float(r[h + 2]), 0.f), a2);
              a3 = fmaf(wr[h + 3], fmaxf(__uint_as_float(r[h + 3]), 0.f), a3);
            }
            if (valid[j]) logits[off[j]] = ((a0 + a1) + (a2 + a3)) * ks[j];
          }
        } else {
          // one MMA tile per unit: token jq's 64 heads are columns [jq*64, jq*64+64);
          // logits row (b, jq) of [B][QT][k_ld].  The 2*QT 32-column chunks are loaded
          // one ahead (two register buffers): chunk c+1's tcgen05.ld is in flight while
          // chunk c is folded, so the TMEM load latency hides behind the FMAs.
          const float4 *wq = reinterpret_cast<const float4 *>(c.wq[g]);
          const int64_t tok = (int64_t)cur.t * UNIT_M + row;
          const uint32_t tbase = tmem + ((uint32_t)(quarter * 32) << 16) + a * ACC_COLS;
          constexpr int NCH = 2 * QT;
          uint32_t rbuf[2][32];
          tmem_ld_32x32b_x32(tbase, rbuf[0]);
          tmem_ld_wait();
          float acc4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int ch = 0; ch < NCH; ch++) {
            if (ch + 1 < NCH) tmem_ld_32x32b_x32(tbase + (ch + 1) * 32, rbuf[(ch + 1) & 1]);
            const uint32_t(&r)[32] = rbuf[ch & 1];
            const int jq = ch >> 1, h0 = (ch & 1) * 32;
#pragma unroll
            for (int h = 0; h < 32; h += 4) {
              const float4 wv = wq[jq * (HEADS / 4) + (h0 + h) / 4];
              acc4[0] = fmaf(wv.x, fmaxf(__uint_as_float(r[h + 0]), 0.f), acc4[0]);
              acc4[1] = fmaf(wv.y, fmaxf(__uint_as_float(r[h + 1]), 0.f), acc4[1]);
              acc4[2] = fmaf(wv.z, fmaxf(__uint_as_float(r[h + 2]), 0.f), acc4[2]);
              acc4[3] = fmaf(wv.w, fmaxf(__uint_as_float(r[h + 3]), 0.f), acc4[3]);
            }
            if (ch & 1) {  // token jq complete
              if (valid[0])
                logits[((int64_t)b * QT + jq) * k_ld + tok] = ((acc4[0] + acc4[1]) + (acc4[2] + acc4[3])) * ks[0];
              acc4[0] = acc4[1] = acc4[2] = acc4[3] = 0.f;
            }
            tmem_ld_wait();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&c.tempty[a]);
        }
        if (done) {  // streamed step: count this warp's stored rows of request b
#pragma unroll
          for (int j = 0; j < SUB; j++) acc_n += __popc(__ballot_sync(0xffffffffu, valid[j]));
        }
        seq.next(c.pref);
        seq.next(c.pref);
        if (done && seq.cur.b != acc_b) {
          // the warp leaves request acc_b (its slice is contiguous, so it never returns):
          // publish its rows once (one release = one wait for the warp's stores, per
          // request instead of per unit)
          __syncwarp();
          if (lane == 0 && acc_n) {
            ess_red_release_add(done + acc_b, acc_n);
            SPROF_MAX(acc_b, 3);
          }
          acc_b = seq.cur.b;
          acc_n = 0;
        }
      }
      if (done) {  // the warp's last request
        __syncwarp();
        if (lane == 0 && acc_n) {
          ess_red_release_add(done + acc_b, acc_n);
          SPROF_MAX(acc_b, 3);
        }
      }
    }
  }
  if (threadIdx.x == 64) K1PROF(3);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<C::TMEM_COLS>(tmem);
  if (threadIdx.x == 32) K1PROF(4);
}

// 2D uint8 tensor [rows][128 B], box [box_rows][128 B], 128-B swizzle.  The last
// encoded maps are cached: the decode loop calls with the same buffers every step.
struct MapCache {
  const void *base = nullptr;
  uint64_t rows = 0;
  uint32_t box = 0;
  CUtensorMap map;
};

bool make_map(CUtensorMap *m, const void *base, uint64_t rows, uint32_t box_rows, MapCache &cache) {
  if (cache.base == base && cache.rows == rows && cache.box == box_rows) {
    *m = cache.map;
    return true;
  }
  if (!ess_make_tmap_2d(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, 128, rows, 128, 128, box_rows,
                        CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  cache.base = base;
  cache.rows = rows;
  cache.box = box_rows;
  cache.map = *m;
  return true;
}

}  // namespace

#ifdef ESS_K1_PROF
extern "C" int ess_debug_k1_prof(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, g_k1_prof, sizeof(g_k1_prof)) == cudaSuccess ? 0 : -7;
}
extern "C" int ess_debug_k1_prof_reset() {
  static unsigned long long zero[160][6];
  return cudaMemcpyToSymbol(g_k1_prof, zero, sizeof(zero)) == cudaSuccess ? 0 : -7;
}
#endif

extern "C" int ess_indexer_logits(const void *d_q, const float *d_w, const void *d_k,
                                  const float *d_kscale, const int32_t *d_len, int32_t batch,
                                  int64_t k_ld, float *d_logits, void *stream) {
  return ess_indexer_logits_ex(d_q, d_w, d_k, d_kscale, d_len, batch, k_ld, d_logits, 0, stream);
}

namespace {

template <int QT>
int launch_indexer(const void *d_q, const float *d_w, const void *d_k, const float *d_kscale,
                   const int32_t *d_len, int32_t batch, int64_t k_ld, float *d_logits,
                   int32_t max_ctas, int32_t group, int32_t *d_done, void *stream) {
  using C = K1Cfg<QT>;
  static thread_local MapCache kc, qc;
  alignas(64) CUtensorMap tk;
  alignas(64) CUtensorMap tq;
  if (!make_map(&tk, d_k, (uint64_t)batch * (uint64_t)k_ld, TILE_M, kc)) return ESS_ERR_CUDA;
  if (!make_map(&tq, d_q, (uint64_t)batch * C::N, C::N, qc)) return ESS_ERR_CUDA;
  if (int rc = ess_smem_optin((const void *)indexer_kernel<QT>, C::SMEM_BYTES)) return rc;
  const bool pdl = (max_ctas & ESS_LAUNCH_PDL) != 0;
  max_ctas &= ~ESS_LAUNCH_PDL;
  const int ctas = max_ctas > 0 && max_ctas < ess_sm_count() ? max_ctas : ess_sm_count();
  ESS_CUDA_TRY(ess_launch(indexer_kernel<QT>, dim3(ctas), dim3(NTHREADS), C::SMEM_BYTES, (cudaStream_t)stream,
                          1, pdl, tk, tq, d_w, d_kscale, d_len, (int)batch, k_ld, d_logits,
                          (int)((group & 0xFFFF) ? group : ((group & ~0xFFFF) | (batch & 0xFFFF))), d_done));
  return ESS_OK;
}

}  // namespace

extern "C" int ess_indexer_logits_ex(const void *d_q, const float *d_w, const void *d_k,
                                     const float *d_kscale, const int32_t *d_len, int32_t batch,
                                     int64_t k_ld, float *d_logits, int32_t max_ctas,
                                     void *stream) {
  return ess_indexer_logits_mtp(d_q, d_w, d_k, d_kscale, d_len, batch, 1, k_ld, d_logits, max_ctas,
                                stream);
}

extern "C" int ess_indexer_logits_mtp(const void *d_q, const float *d_w, const void *d_k,
                                      const float *d_kscale, const int32_t *d_len, int32_t batch,
                                      int32_t qtok, int64_t k_ld, float *d_logits, int32_t max_ctas,
                                      void *stream) {
  if (max_ctas < 0 || qtok < 1 || qtok > ESS_INDEXER_MAX_QTOK) return ESS_ERR_ARG;
  if (!d_q || !d_w || !d_k || !d_kscale || !d_len || !d_logits || batch < 0 ||
      batch > MAX_BATCH || k_ld < TILE_M || (k_ld % TILE_M) != 0 ||
      (reinterpret_cast<uintptr_t>(d_k) & 15) || (reinterpret_cast<uintptr_t>(d_q) & 15) ||
      (reinterpret_cast<uintptr_t>(d_w) & 15))
    return ESS_ERR_ARG;
  if (batch == 0) return ESS_OK;
  switch (qtok) {
    case 1: return launch_indexer<1>(d_q, d_w, d_k, d_kscale, d_len, batch, k_ld, d_logits, max_ctas, 0, nullptr, stream);
    case 2: return launch_indexer<2>(d_q, d_w, d_k, d_kscale, d_len, batch, k_ld, d_logits, max_ctas, 0, nullptr, stream);
    case 3: return launch_indexer<3>(d_q, d_w, d_k, d_kscale, d_len, batch, k_ld, d_logits, max_ctas, 0, nullptr, stream);
    default: return launch_indexer<4>(d_q, d_w, d_k, d_kscale, d_len, batch, k_ld, d_logits, max_ctas, 0, nullptr, stream);
  }
}

// Streamed step: requests in groups of `group`, the whole grid finishing each group
// before the next; after storing its logits rows of a unit every epilogue warp adds the
// number of rows it stored to d_done[b] (release, GPU scope), so d_done[b] reaches
// min(len[b], k_ld) exactly when request b's logits are complete.  d_done [batch] must be
// zero at launch.
extern "C" int ess_indexer_logits_stream(const void *d_q, const float *d_w, const void *d_k,
                                         const float *d_kscale, const int32_t *d_len, int32_t batch,
                                         int64_t k_ld, float *d_logits, int32_t max_ctas, int32_t group,
                                         int32_t *d_done, void *stream) {
  // group: requests per group (low 16 bits; 0 = one group), first group (high 16 bits)
  if (max_ctas < 0 || group < 0 || !d_done) return ESS_ERR_ARG;
  if (!d_q || !d_w || !d_k || !d_kscale || !d_len || !d_logits || batch < 0 ||
      batch > MAX_BATCH || k_ld < TILE_M || (k_ld % TILE_M) != 0 ||
      (reinterpret_cast<uintptr_t>(d_k) & 15) || (reinterpret_cast<uintptr_t>(d_q) & 15) ||
      (reinterpret_cast<uintptr_t>(d_w) & 15))
    return ESS_ERR_ARG;
  if (batch == 0) return ESS_OK;
  return launch_indexer<1>(d_q, d_w, d_k, d_kscale, d_len, batch, k_ld, d_logits, max_ctas, group, d_done,
                           stream);
}

#ifdef ESS_STREAM_PROF
ESS_STREAM_PROF_READER(ess_debug_stream_prof_k1)
#endif

// Load every kernel of this file now (lazy module loading would otherwise load a kernel
// at its first launch, which waits for the device: a deadlock when a running kernel
// spins on work the not-yet-loaded one produces — the streamed hand-offs).
int ess_preload_indexer() {
  cudaFuncAttributes a;
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)indexer_kernel<1>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)indexer_kernel<2>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)indexer_kernel<3>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)indexer_kernel<4>));
  return ESS_OK;
}
