// K5, FP8 slot rows: sparse MLA decode over 656-B latent rows (op "sparse_mla",
// costmodel.py:18-27) on a CTA pair with cta_group::2 MMAs.
//
// Why a second K5.  The f16-slot kernel (mla.cu) runs a request on two CTAs that each
// own 256 output dims and BOTH compute the full 128-head score tile (1.53x the
// algorithmic MMA work), and it reads 1152-B dequantised rows (1.76x the 656-B wire
// bytes; the slot store costs 1.76x the latent bytes it caches).  Here:
//   * the slot store keeps the raw 656-B row (512 e4m3 NoPE, 4 f32 group scales,
//     64 bf16 RoPE, scenario.py:25) — a 25% pool costs 25% of the latent bytes — and
//     the kernel dequantises in shared memory: f16(e4m3) x f16(scale) in one HMUL2
//     (exact for the power-of-two group scales of DeepSeek-V3.2's FP8 cache; for other
//     scales one f16 rounding of the scale, < 1 f16 ulp from oracle.dsa.slot_rows);
//   * the pair splits the HEADS (CTA r owns heads 64r..64r+63) and every MMA is
//     cta_group::2 with M = 128: S = Q K^T has each CTA supply its 64 q rows and half
//     of the tile's 32 K rows (N = 32), so each score is computed once; O += P V has
//     each CTA supply its 64 P rows and half of each 256-dim V block (N = 256, two
//     instructions for 512 dims).  Per-SM tensor work is the algorithmic 285 MFLOP per
//     request instead of 436.
//
// TMEM per CTA (cta_group::2 "2x2" layout: a 64 x N accumulator spans 128 lanes x N/2
// columns, lanes 64..127 holding columns N/2..N-1):
//   O   [0,256)    two 64 x 256 accumulators (dims 0..255, 256..511)
//   S   [256,320)  four 64 x 32 score buffers (16 columns each): S(i+3) issues before PV(i)
//   Q   [320,512)  q dims 0..383 as f16 pairs, duplicated over both lane halves (the
//                  A-from-TMEM layout of cta_group::2)
// Thread t of the softmax warps owns head 64r + t%64 and tile tokens [16u, 16u+16),
// u = t/64; the pair's two threads of a head exchange their tile max through shared
// memory.  Shared memory per CTA: q dims 384..575 (3 SW128 blocks), a 3-deep staging
// ring of raw rows (own 16 rows whole + the other 16 rows' V bytes of this CTA's dims),
// 3 S tiles [16 rows][576] and 4 V tiles [32 rows][256 dims] in SW128 f16, 4 P tiles
// [64 heads][32 tokens].
//
// Warp roles (320 threads): w0-3 softmax + epilogue, w4 TMEM alloc + MMA issue (rank 0
// only issues), w5 row loader (cp.async.bulk per row / row part), w6-9 dequantisers.
// The rank-0 CTA's barriers gate the MMAs: the peer's dequantisers and softmax warps
// arrive on them remotely; MMA completion is multicast to both CTAs' barriers.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int HEADS = ESS_MLA_HEADS;   // 128 = M of every MMA (64 per CTA)
constexpr int HH = HEADS / 2;          // heads per CTA
constexpr int NB = 32;                 // tokens per tile (N of S)
constexpr int NH = NB / 2;             // tokens per CTA half
constexpr int NBLK = ESS_MLA_QK_DIM / 64;  // 9 dim-blocks of 64
constexpr int QT_BLKS = 6;             // q blocks in TMEM (dims 0..383)
constexpr int QS_BLKS = NBLK - QT_BLKS;    // 3 in shared memory (384..575)
constexpr int NSB = 4;                 // TMEM S buffers / P tiles
#ifndef ESS_MLA2_KSS  // ring depths (scratch builds sweep them; smem-bound)
#define ESS_MLA2_KSS 2
#define ESS_MLA2_KSV 4
#define ESS_MLA2_NST 4
#endif
#ifndef ESS_MLA2_DEQ_LAG
#define ESS_MLA2_DEQ_LAG 1
#endif
constexpr int DEQ_LAG = ESS_MLA2_DEQ_LAG;  // S dequantisation leads V by this many tiles
constexpr int KSS = ESS_MLA2_KSS;      // S tiles
constexpr int KSV = ESS_MLA2_KSV;      // V tiles
constexpr int NST = ESS_MLA2_NST;      // staging stages
constexpr int ROW = ESS_LATENT_ROW_BYTES;  // 656
constexpr int OTHER = 272;             // other half's row part: 2 x 128 B NoPE + 16 B scales
constexpr int STG_OWN = NH * ROW;      // 10496
constexpr int STG_BYTES = STG_OWN + NH * OTHER;  // 14848
constexpr int QBLK = HH * 128;         // [64 heads][64 dims] f16 = 8 KB
constexpr int S_BLK = NH * 128;        // [16 rows][64 dims] = 2 KB
constexpr int S_TILE = NBLK * S_BLK;   // 18 KB
constexpr int V_BLK = NB * 128;        // [32 rows][64 dims] = 4 KB
constexpr int V_TILE = 4 * V_BLK;      // 16 KB: this CTA's 256 of the 512 V dims
constexpr int P_TILE = HH * 128;       // [64 heads][32 tokens] f16 in 128-B SW128 rows
#ifndef ESS_MLA2_NLOAD
#define ESS_MLA2_NLOAD 4
#endif
constexpr int NSOFT = 4, MMA_WARP = 4, LOAD0 = 5, NLOAD = ESS_MLA2_NLOAD, CONV0 = LOAD0 + NLOAD, NCONV = 4;
constexpr int NTHREADS = 32 * (CONV0 + NCONV);  // 416
constexpr int NLT = NLOAD * 32;                 // loader threads
constexpr int OWN_CHUNKS = ROW / 16;            // 41 16-B chunks per own row
constexpr int OTHER_CHUNKS = OTHER / 16;        // 17 per other row
constexpr uint32_t TM_O = 0, TM_S = 256, TM_Q = 320;
static_assert(TM_Q + QT_BLKS * 32 <= 512, "TMEM budget");
static_assert(NST > DEQ_LAG, "staging ring must hold the V-lagged tiles");
constexpr float RESCALE_THRESHOLD = 8.0f;
constexpr int MLA_AWAIT = 4;           // internal flag (as in mla.cu)
constexpr int LANDED_TAG = 1 << 24;
constexpr uint32_t IDESC_S = make_idesc(0, 0, HEADS, NB, 0, 0);
constexpr uint32_t IDESC_PV = make_idesc(0, 0, HEADS, 256, 0, 1 /* B MN-major */);

// f16 slot rows (1152 B, dequantised on admission): no staging or dequantisers; the
// loaders cp.async each CTA's 16 own rows straight into an S tile and its 256 V dims of
// all 32 rows into a V tile (one stage = both), 4 stages
constexpr int F_NST = 4, F_NLOAD = 4;
constexpr int F_NTHREADS = 32 * (LOAD0 + F_NLOAD);  // 288
constexpr int F_ROW = ESS_SLOT_ROW_BYTES;           // 1152
constexpr int MAXR = 4;                              // barrier array size of every ring
static_assert(KSS <= MAXR && KSV <= MAXR && NST <= MAXR && F_NST <= MAXR, "ring barrier arrays");
struct Ctrl {
  uint64_t stg_full[MAXR], stg_empty[MAXR];
  uint64_t s_full[MAXR], s_empty[MAXR];   // s_full/v_full/p_full: rank 0's gate the MMAs
  uint64_t v_full[MAXR], v_empty[MAXR];
  uint64_t ld_full[MAXR];                 // f16 rows: this CTA's cp.async of a stage landed
  uint64_t s_ready[NSB], p_full[NSB], pv_done[NSB];
  uint64_t o_done, q_full;
  uint32_t tmem;
  float xm[2][2][HH];                   // pair max / sum exchange (double-buffered)
};
constexpr size_t OFF_Q = 0;
constexpr size_t OFF_S = OFF_Q + QS_BLKS * QBLK;
constexpr size_t OFF_V = OFF_S + KSS * S_TILE;
constexpr size_t OFF_P = OFF_V + KSV * V_TILE;
constexpr size_t OFF_STG = OFF_P + NSB * P_TILE;
constexpr size_t OFF_CTRL = OFF_STG + NST * STG_BYTES;
constexpr size_t SMEM_BYTES = 1024 + OFF_CTRL + sizeof(Ctrl);
static_assert(SMEM_BYTES <= 232448, "K5 (FP8) shared memory over the sm_100 limit");
static_assert(QT_BLKS * QBLK <= KSV * V_TILE, "q staging for TMEM fits the V ring");
static_assert(OFF_S % 1024 == 0 && OFF_V % 1024 == 0 && OFF_P % 1024 == 0, "SW128 alignment");
constexpr size_t F_OFF_V = OFF_S + F_NST * S_TILE;
constexpr size_t F_OFF_P = F_OFF_V + F_NST * V_TILE;
constexpr size_t F_OFF_CTRL = F_OFF_P + NSB * P_TILE;
constexpr size_t F_SMEM_BYTES = 1024 + F_OFF_CTRL + sizeof(Ctrl);
static_assert(F_SMEM_BYTES <= 232448, "K5 (f16 pair) shared memory over the sm_100 limit");
static_assert(QT_BLKS * QBLK <= F_NST * V_TILE && F_OFF_V % 1024 == 0 && F_OFF_P % 1024 == 0, "f16 layout");

// ---- cta_group::2 PTX --------------------------------------------------------------
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// completion of every prior tcgen05 op of this thread -> arrive on the barrier at the
// same shared-memory offset in both CTAs of the pair
__device__ __forceinline__ void commit2(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t *dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst))
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive (release, cluster scope) on the barrier at the same offset in CTA `rank`
__device__ __forceinline__ void arrive_on(uint64_t *bar, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void softmax_bar() {  // the 4 softmax warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&r)[32]) { tmem_st_32x32b_x32(taddr, r); }
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// bf16 pair -> f16 pair, saturating at +-65504 (no silent inf from the narrower range)
__device__ __forceinline__ uint32_t bf16x2_to_f16x2_sat(uint32_t v) {
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(v & 0xFFFF0000u)),
      "f"(__uint_as_float(v << 16)));
  return r;
}
__device__ __forceinline__ uint4 cvt8_bf16_f16_sat(uint4 x) {
  return make_uint4(bf16x2_to_f16x2_sat(x.x), bf16x2_to_f16x2_sat(x.y), bf16x2_to_f16x2_sat(x.z),
                    bf16x2_to_f16x2_sat(x.w));
}
// 16 e4m3 (one uint4) x f16 scale pair -> 16 f16 (two uint4): exact e4m3 -> f16, one HMUL2
__device__ __forceinline__ void deq16(uint4 v, uint32_t s2, uint4 &a, uint4 &c) {
  const __half2 sc = *reinterpret_cast<const __half2 *>(&s2);
  auto m = [&](uint32_t w16) {
    uint32_t h = cvt_e4m3x2_f16x2((uint16_t)w16);
    __half2 r = __hmul2(*reinterpret_cast<__half2 *>(&h), sc);
    return *reinterpret_cast<uint32_t *>(&r);
  };
  a = make_uint4(m(v.x & 0xFFFF), m(v.x >> 16), m(v.y & 0xFFFF), m(v.y >> 16));
  c = make_uint4(m(v.z & 0xFFFF), m(v.z >> 16), m(v.w & 0xFFFF), m(v.w >> 16));
}
__device__ __forceinline__ uint32_t scale_f16x2(float s) {
  __half2 h = __float2half2_rn(s);
  return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
// arrive on the mbarrier once every cp.async this thread issued so far has completed
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_landed(const int32_t *p, int target) {
  if ((threadIdx.x & 31) == 0) {
    uint32_t spins = 0;
    while ((ld_acquire(p) & (LANDED_TAG - 1)) < target) {
      if (++spins > ESS_SPIN_LIMIT) __trap();
      __nanosleep(256);
    }
  }
  __syncwarp();
  (void)ld_acquire(p);
  fence_proxy_async_global();  // the gather's generic-proxy stores -> our bulk-copy reads
}

#ifdef ESS_MLA2_TRACE  // scratch builds: per-tile globaltimer stamps of request 0's CTA pair
__device__ unsigned long long g_mla2_trace[2][10][72];
#define M2TRACE(ev, i)                                                                 \
  do {                                                                                 \
    if (blockIdx.y == 0 && (i) < 72) {                                                 \
      unsigned long long tt;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                           \
      g_mla2_trace[r][ev][i] = tt;                                                     \
    }                                                                                  \
  } while (0)
#else
#define M2TRACE(ev, i) \
  do {                 \
  } while (0)
#endif

template <bool F16>
__global__ void __launch_bounds__(F16 ? F_NTHREADS : NTHREADS, 1)
    sparse_mla_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const uint8_t *__restrict__ rows,
                          int64_t rows_per_pool, int pool_begin, const int32_t *__restrict__ sel_row,
                          const int32_t *__restrict__ sel2, int32_t *landed, int sel_stride,
                          const int32_t *__restrict__ counts, int count_stride, float sm_scale,
                          uint16_t *__restrict__ out, float *__restrict__ lse, float *__restrict__ ws_o,
                          float *__restrict__ ws_ml, int flags, int nsplit, int32_t *status) {
  extern __shared__ uint8_t smem_raw[];
  // offset from the shared array itself (keeps the shared address space: LDS/STS, not generic)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int KS_S = F16 ? F_NST : KSS, KS_V = F16 ? F_NST : KSV;  // S / V tile rings
  constexpr int NTH = F16 ? F_NTHREADS : NTHREADS;
  uint8_t *sq = smem + OFF_Q, *sS = smem + OFF_S, *sV = smem + (F16 ? F_OFF_V : OFF_V);
  uint8_t *sP = smem + (F16 ? F_OFF_P : OFF_P);
  uint8_t *stg = smem + OFF_STG;
  Ctrl &c = *reinterpret_cast<Ctrl *>(smem + (F16 ? F_OFF_CTRL : OFF_CTRL));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = cluster_rank();         // 0: issues the MMAs
  const int split = blockIdx.y % nsplit;
  const int b = blockIdx.y / nsplit;
  const bool partial = flags & ESS_MLA_PARTIAL, resume = flags & ESS_MLA_RESUME;
  const bool to_ws = partial || nsplit > 1;
  const bool await = flags & MLA_AWAIT;
  const int n1t = min(counts[(int64_t)b * count_stride], ESS_MAX_REQUEST);
  const int n2t = await ? min(counts[(int64_t)b * count_stride + 1], ESS_MAX_REQUEST - n1t) : 0;
  const int h0 = n1t * split / nsplit, h1 = n1t * (split + 1) / nsplit;
  const int m0 = n2t * split / nsplit, m1 = n2t * (split + 1) / nsplit;
  const int n1 = h1 - h0;
  const int n = n1 + (m1 - m0);
  const bool fetched = m1 > m0;
  const int ntiles = (n + NB - 1) / NB;

  if (threadIdx.x == 0 && F16) {
    for (int i = 0; i < F_NST; i++) {
      mbar_init(&c.ld_full[i], F_NLOAD * 32);  // one cp.async completion arrive per loader thread
      mbar_init(&c.s_full[i], 1);              // rank 0: the peer's relay (its stage landed)
      mbar_init(&c.v_empty[i], 1);             // PV(i) done: stage free in both CTAs
    }
  }
  if (threadIdx.x == 0 && !F16) {
    for (int i = 0; i < NST; i++) {
      mbar_init(&c.stg_full[i], NLOAD * 32);  // one cp.async completion arrive per loader thread
      mbar_init(&c.stg_empty[i], NCONV);
    }
    for (int i = 0; i < KSS; i++) {
      mbar_init(&c.s_full[i], 2 * NCONV);
      mbar_init(&c.s_empty[i], 1);
    }
    for (int i = 0; i < KSV; i++) {
      mbar_init(&c.v_full[i], 2 * NCONV);
      mbar_init(&c.v_empty[i], 1);
    }
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSB; i++) {
      mbar_init(&c.s_ready[i], 1);
      mbar_init(&c.p_full[i], 2 * NSOFT);
      mbar_init(&c.pv_done[i], 1);
    }
    mbar_init(&c.o_done, 1);
    mbar_init(&c.q_full, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc2(&c.tmem);

  // ---- prologue: this CTA's 64 q rows -> TMEM (dims 0..383, duplicated over both lane
  // halves) and shared memory (384..575); TMA boxes of [64 heads][64 dims] bf16 -------
  __syncthreads();  // barriers initialised (q_full is waited on below)
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&c.q_full, HH * ESS_MLA_QK_DIM * 2);
    for (int blk = 0; blk < NBLK; blk++)
      tma_load_2d(blk < QT_BLKS ? sV + blk * QBLK : sq + (blk - QT_BLKS) * QBLK, &tm_q, &c.q_full, blk * 64,
                  b * HEADS + (int)r * HH);
  }
  mbar_wait(&c.q_full, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = c.tmem;
  if (warp < NSOFT) {
    const int h = (warp * 32 + lane) & (HH - 1);
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
#pragma unroll 1
    for (int cc = 0; cc < QT_BLKS; cc++) {
      const uint8_t *rowp = sV + cc * QBLK + h * 128;
      uint32_t v[32];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const uint4 x = *reinterpret_cast<const uint4 *>(rowp + ((k ^ (h & 7)) << 4));
        bad |= bf16x8_over_f16(x);
        const uint4 y = cvt8_bf16_f16_sat(x);
        v[4 * k] = y.x;
        v[4 * k + 1] = y.y;
        v[4 * k + 2] = y.z;
        v[4 * k + 3] = y.w;
      }
      tmem_st_x32(tmem + lane_base + TM_Q + cc * 32, v);
      if (bad) ess_set_status(status, ESS_ERR_RANGE);  // q saturated: outside the f16 range
    }
    tmem_st_wait();
  } else {
    uint4 *qs = reinterpret_cast<uint4 *>(sq);
    bool bad = false;
    for (int u = threadIdx.x - NSOFT * 32; u < QS_BLKS * QBLK / 16; u += NTH - NSOFT * 32)
    {
      bad |= bf16x8_over_f16(qs[u]);
      qs[u] = cvt8_bf16_f16_sat(qs[u]);
    }
    if (bad) ess_set_status(status, ESS_ERR_RANGE);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();   // the V ring (q staging) is free again
  cluster_sync_all();  // both CTAs: barriers initialised, q in TMEM / smem
  tc_fence_after();
  const float scale_log2 = sm_scale * 1.4426950408889634f;

  if (warp < NSOFT) {
    // ================= softmax / epilogue: thread = (head, token half) ===============
    const int t = warp * 32 + lane;
    const int h = t & (HH - 1), u = t >> 6;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int64_t hrow = (int64_t)b * HEADS + (int)r * HH + h;
    const int64_t wrow = (int64_t)(b * nsplit + split) * HEADS + (int)r * HH + h;
    float *wso = ws_o ? ws_o + wrow * ESS_MLA_V_DIM : nullptr;
    float m_run = -INFINITY, l_run = 0.f;
    for (int i = 0; i < ntiles; i++) {
      const int sb = i % NSB;
      mbar_wait(&c.s_ready[sb], (i / NSB) & 1);
      if (t == 0) M2TRACE(4, i);
      if (i >= NSB) mbar_wait(&c.pv_done[sb], ((i - NSB) / NSB) & 1);  // P tile sb free
      tc_fence_after();
      uint32_t sr[NH];
      tmem_ld_x16(tmem + lane_base + TM_S + sb * NH, sr);
      tmem_ld_wait();
      float x[NH];
      const int lim = n - i * NB - u * NH;  // valid tokens of this half
#pragma unroll
      for (int j = 0; j < NH; j++) x[j] = j < lim ? __uint_as_float(sr[j]) : -INFINITY;
      float mx = fmaxf(x[0], x[1]);
#pragma unroll
      for (int j = 2; j < NH; j++) mx = fmaxf(mx, x[j]);
      c.xm[i & 1][u][h] = mx;
      softmax_bar();
      const float mt = fmaxf(mx, c.xm[i & 1][u ^ 1][h]) * scale_log2;
      // both threads of a head see the same (mt, m_run): the pair and the two warps
      // holding the same heads (w, w+2) take the same, warp-uniform decision
      if (__any_sync(0xffffffffu, mt > m_run + RESCALE_THRESHOLD) || i == 0) {
        const float m_new = fmaxf(mt, m_run);
        const float alpha = exp2f(m_run - m_new);
        l_run *= alpha;
        if (i > 0) {
          mbar_wait(&c.pv_done[(i - 1) % NSB], ((i - 1) / NSB) & 1);  // O holds PV(i-1)
          tc_fence_after();
#pragma unroll 1
          for (int cc = 0; cc < 8; cc++) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j++) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
            tmem_st_x32(tmem + lane_base + TM_O + cc * 32, o);
          }
          tmem_st_wait();
        }
        m_run = m_new;
      }
      uint32_t p[NH / 2];
      float ls0 = 0.f, ls1 = 0.f;
      const float nm = -m_run;
#pragma unroll
      for (int e = 0; e < NH / 2; e++) {
        const float e0 = fast_exp2(fmaf(x[2 * e], scale_log2, nm));
        const float e1 = fast_exp2(fmaf(x[2 * e + 1], scale_log2, nm));
        p[e] = pack_f16x2(e0, e1);
        ls0 += e0;
        ls1 += e1;
      }
      l_run += ls0 + ls1;
      // P row h, tokens [16u, 16u+16): logical 16-B chunks 2u, 2u+1 of the SW128 row
      uint8_t *prow = sP + sb * P_TILE + h * 128;
      *reinterpret_cast<uint4 *>(prow + (((2 * u) ^ (h & 7)) << 4)) = make_uint4(p[0], p[1], p[2], p[3]);
      *reinterpret_cast<uint4 *>(prow + (((2 * u + 1) ^ (h & 7)) << 4)) = make_uint4(p[4], p[5], p[6], p[7]);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_on(&c.p_full[sb], 0);
      if (t == 0) M2TRACE(5, i);
    }
    // ---------------- epilogue ----------------------------------------------------
    const bool have_o = ntiles > 0;
    if (have_o) {
      mbar_wait(&c.o_done, 0);
      for (int k = max(0, ntiles - NSB); k < ntiles; k++) mbar_wait(&c.pv_done[k % NSB], (k / NSB) & 1);
      tc_fence_after();
    }
    c.xm[ntiles & 1][u][h] = l_run;  // the pair's sums
    softmax_bar();
    const float l_pair = l_run + c.xm[ntiles & 1][u ^ 1][h];
    // this thread's 256 dims: columns [0,128) = dims 128u + c, [128,256) = 256 + 128u + c
    auto dim_of = [&](int col) { return col < 128 ? 128 * u + col : 256 + 128 * u + (col - 128); };
    if (to_ws) {
#pragma unroll 1
      for (int cc = 0; cc < 8; cc++) {
        uint32_t o[32];
        if (have_o) {
          tmem_ld_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; j++) o[j] = 0u;
        }
        float *dst = wso + dim_of(cc * 32);
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4 *>(dst + j) = make_float4(__uint_as_float(o[j]), __uint_as_float(o[j + 1]),
                                                             __uint_as_float(o[j + 2]), __uint_as_float(o[j + 3]));
      }
      if (u == 0) {
        ws_ml[wrow * 2 + 0] = m_run;
        ws_ml[wrow * 2 + 1] = l_pair;
      }
    } else {
      float m = m_run, l = l_pair, a0 = 0.f, a1 = have_o ? 1.f : 0.f;
      if (resume) {
        const float mp = ws_ml[hrow * 2 + 0], lp = ws_ml[hrow * 2 + 1];
        m = fmaxf(mp, m_run);
        a0 = mp == -INFINITY ? 0.f : exp2f(mp - m);
        a1 = (have_o && m_run != -INFINITY) ? exp2f(m_run - m) : 0.f;
        l = lp * a0 + l_pair * a1;
      }
      uint16_t *ob = out + hrow * ESS_MLA_V_DIM;
      const float *wsr = resume ? ws_o + hrow * ESS_MLA_V_DIM : nullptr;
      // every lane runs the epilogue (tcgen05.ld is .sync.aligned; see mla.cu):
      // l == 0 -> zeros, lse -inf; l NaN (out-of-range operands) -> NaN
      {
        const bool pos = l > 0.f;
        const float inv = 1.f / l;
        const float c0 = pos ? a0 * inv : (l == l ? 0.f : l), c1 = pos ? a1 * inv : c0;
#pragma unroll 1
        for (int cc = 0; cc < 8; cc++) {
          uint32_t o[32];
          if (have_o) {
            tmem_ld_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int j = 0; j < 32; j++) o[j] = 0u;
          }
          const int d0 = dim_of(cc * 32);
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            float w[8];
#pragma unroll
            for (int e = 0; e < 8; e++) w[e] = resume ? wsr[d0 + j + e] : 0.f;
            uint4 pk;
            uint32_t *pw = reinterpret_cast<uint32_t *>(&pk);
#pragma unroll
            for (int e = 0; e < 4; e++) {
              __nv_bfloat162 tt = __floats2bfloat162_rn(__uint_as_float(o[j + 2 * e]) * c1 + w[2 * e] * c0,
                                                        __uint_as_float(o[j + 2 * e + 1]) * c1 + w[2 * e + 1] * c0);
              pw[e] = *reinterpret_cast<uint32_t *>(&tt);
            }
            *reinterpret_cast<uint4 *>(ob + d0 + j) = pk;
          }
        }
        if (u == 0) lse[hrow] = pos ? (m + log2f(l)) * 0.6931471805599453f : (l == l ? -INFINITY : l);
      }
    }
  } else if (warp == MMA_WARP) {
    // ================= MMA issue (rank 0; its instructions drive both SMs) ===========
    if (r == 0 && elect_one() && ntiles > 0) {
      const uint64_t qbase = sw128_desc(smem_u32(sq), 16, 1024);
      const uint64_t sbase = sw128_desc(smem_u32(sS), 16, 1024);
      const uint64_t vbase = sw128_desc(smem_u32(sV), V_BLK, 1024);
      const uint64_t pbase = sw128_desc(smem_u32(sP), 16, 1024);
      auto issue_s = [&](int i) {
        const int ks = i % KS_S, sb = i % NSB;
        tc_fence_after();  // s_full[ks] observed: both CTAs' halves of tile i in shared memory
        const uint32_t d = tmem + TM_S + sb * NH;
#pragma unroll
        for (int blk = 0; blk < NBLK; blk++) {
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            const uint64_t bd = sbase + (uint64_t)((ks * S_TILE + blk * S_BLK + kk * 32) >> 4);
            const uint32_t acc = (blk | kk) ? 1u : 0u;
            if (blk < QT_BLKS) mma2_ts(d, tmem + TM_Q + (blk * 4 + kk) * 8, bd, IDESC_S, acc);
            else mma2_ss(d, qbase + (uint64_t)(((blk - QT_BLKS) * QBLK + kk * 32) >> 4), bd, IDESC_S, acc);
          }
        }
        commit2(&c.s_ready[sb]);
        if (!F16) commit2(&c.s_empty[ks]);  // f16: the stage frees with its V tile (after PV)
      };
      auto issue_pv = [&](int i) {
        const int sb = i % NSB, kv = i % KS_V;
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 2; kk++) {
          const uint64_t ad = pbase + (uint64_t)((sb * P_TILE + kk * 32) >> 4);
#pragma unroll
          for (int hf = 0; hf < 2; hf++) {
            const uint64_t bd = vbase + (uint64_t)((kv * V_TILE + 2 * hf * V_BLK + kk * 16 * 128) >> 4);
            mma2_ss(tmem + TM_O + hf * 128, ad, bd, IDESC_PV, (i | kk) ? 1u : 0u);
          }
        }
        commit2(&c.pv_done[sb]);
        commit2(&c.v_empty[kv]);
        if (i == ntiles - 1) commit2(&c.o_done);
      };
      // Issue whichever MMA group is ready, S ahead of PV by up to NSB tiles: S(ns) needs
      // its dequantised K rows and a free TMEM S buffer (P(ns - NSB) seen, i.e.
      // PV(ns - NSB) issued); PV(np) needs P(np) and V(np).  A fixed "S(i+3), then PV(i)"
      // order made PV wait on rows three tiles ahead (and V dequantisation on PV).
      int ns = 0, np = 0;
      uint32_t spins = 0;
      while (np < ntiles) {
        bool progress = false;
        if (ns < ntiles && ns < np + NSB && mbar_test_wait(&c.s_full[ns % KS_S], (ns / KS_S) & 1) &&
            (!F16 || mbar_test_wait(&c.ld_full[ns % KS_S], (ns / KS_S) & 1))) {
          M2TRACE(6, ns);
          if (F16) fence_proxy_async_smem();  // this CTA's cp.async rows -> tensor-core reads
          issue_s(ns++);
          progress = true;
        }
        if (np < ns && mbar_test_wait(&c.p_full[np % NSB], (np / NSB) & 1)) {
          M2TRACE(7, np);
          if (F16 || mbar_test_wait(&c.v_full[np % KSV], (np / KSV) & 1)) {
            M2TRACE(8, np);
            issue_pv(np++);
            progress = true;
          }
        }
        if (progress) spins = 0;
        else if (++spins > ESS_SPIN_LIMIT) __trap();
      }
    } else if (F16 && r == 1 && elect_one()) {
      // relay: each stage this CTA's loaders filled -> rank 0's s_full (the MMA reads
      // both CTAs' tiles); the proxy fence orders the cp.async writes before the MMA reads
      for (int i = 0; i < ntiles; i++) {
        mbar_wait(&c.ld_full[i % F_NST], (i / F_NST) & 1);
        fence_proxy_async_smem();
        arrive_on(&c.s_full[i % F_NST], 0);
      }
    }
  } else if (F16) {
    // ================= f16 rows: 4 loader warps, cp.async straight into the tiles ===
    // Per tile: the 16 own rows whole (72 chunks of 8 dims) -> S tile [16][9 x 64 dims];
    // this CTA's 256 V dims (chunks 16r..16r+15 and 32+16r..32+16r+15) of all 32 rows ->
    // V tile [32][4 x 64 dims]; SW128 positions (8 lanes = one 128-B row: no conflicts)
    const int lt = threadIdx.x - LOAD0 * 32;  // 0..127
    const uint8_t *pool_rows = rows + (int64_t)(pool_begin + b / (((flags >> ESS_MLA_QTOK_SHIFT) & 7) + 1)) * rows_per_pool * F_ROW;
    const int32_t *selh = sel_row + (int64_t)b * sel_stride + h0;
    const int32_t *selm = await ? sel2 + (int64_t)b * sel_stride + m0 : nullptr;
    const uint32_t sS0 = smem_u32(sS), sV0 = smem_u32(sV);
    bool pending = fetched && n2t > 0;
    auto row_id = [&](int i) {
      const int tl = i * NB + lane;
      const int jl = tl < n ? tl : 0;
      return jl < n1 ? __ldg(selh + jl) : (pending ? 0 : __ldg(selm + (jl - n1)));
    };
    int sid_next = ntiles > 0 && !(pending && NB > n1) ? row_id(0) : 0;
    for (int i = 0; i < ntiles; i++) {
      const int st = i % F_NST;
      mbar_wait(&c.v_empty[st], ((i / F_NST) & 1) ^ 1);
      int sidl = sid_next;
      if (pending && (i + 1) * NB > n1) {
        wait_landed(landed + b, n2t);
        pending = false;
        sidl = row_id(i);
      }
      if (lt == 0) M2TRACE(0, i);
      if (i + 1 < ntiles && !(pending && (i + 2) * NB > n1)) sid_next = row_id(i + 1);
      const uint32_t sd = sS0 + st * S_TILE, vd = sV0 + st * V_TILE;
#pragma unroll
      for (int k = 0; k < NH * 72 / 128; k++) {  // 9
        const int it = lt + 128 * k;
        const int row = it / 72, ch = it - row * 72;
        const int tok = (int)r * NH + row;
        const int sid = __shfl_sync(0xffffffffu, sidl, tok);
        cp_async16(sd + (ch >> 3) * S_BLK + row * 128 + (((ch & 7) ^ (row & 7)) << 4),
                   pool_rows + (int64_t)sid * F_ROW + ch * 16, i * NB + tok < n ? 16u : 0u);
      }
#pragma unroll
      for (int k = 0; k < NB * 32 / 128; k++) {  // 8
        const int it = lt + 128 * k;
        const int tok = it >> 5, cc = it & 31;
        const int sid = __shfl_sync(0xffffffffu, sidl, tok);
        const int ch = (cc < 16 ? 16 * (int)r : 32 + 16 * (int)r) + (cc & 15);
        cp_async16(vd + (cc >> 3) * V_BLK + tok * 128 + (((cc & 7) ^ (tok & 7)) << 4),
                   pool_rows + (int64_t)sid * F_ROW + ch * 16, i * NB + tok < n ? 16u : 0u);
      }
      cp_async_arrive_noinc(&c.ld_full[st]);
      if (lt == 0) M2TRACE(9, i);
    }
    cp_async_wait_all();
  } else if (warp < LOAD0 + NLOAD) {
    // ================= row loaders (2 warps): 16-B cp.async per chunk ===============
    // Per tile this CTA stages its 16 own rows whole (41 chunks) and, of the other 16
    // rows, the 17 chunks of its V dims (2 x 128 B NoPE + the 16-B scales).  Each
    // thread's completion arrives on stg_full by itself (cp.async.mbarrier.arrive), so
    // no loader waits on its own copies.  (One cp.async.bulk per row part throttled on
    // the bulk-copy unit: 64 small copies per tile took 2.7 us.)
    const int lt = threadIdx.x - LOAD0 * 32;  // 0..NLT-1
    const uint8_t *pool_rows = rows + (int64_t)(pool_begin + b / (((flags >> ESS_MLA_QTOK_SHIFT) & 7) + 1)) * rows_per_pool * ROW;
    const int32_t *selh = sel_row + (int64_t)b * sel_stride + h0;
    const int32_t *selm = await ? sel2 + (int64_t)b * sel_stride + m0 : nullptr;
    const uint32_t stg0 = smem_u32(stg);
    bool pending = fetched && n2t > 0;
    // lane l holds the slot row of tile token l (padding tokens: row 0, zero-filled);
    // the next tile's ids are loaded one tile ahead, off the copy issue's critical path
    auto row_id = [&](int i) {
      const int tl = i * NB + lane;
      const int jl = tl < n ? tl : 0;
      return jl < n1 ? __ldg(selh + jl) : (pending ? 0 : __ldg(selm + (jl - n1)));
    };
    int sid_next = ntiles > 0 && !(pending && NB > n1) ? row_id(0) : 0;
    for (int i = 0; i < ntiles; i++) {
      const int st = i % NST;
      mbar_wait(&c.stg_empty[st], ((i / NST) & 1) ^ 1);
      int sidl = sid_next;
      if (pending && (i + 1) * NB > n1) {
        wait_landed(landed + b, n2t);  // the fetched rows' slot ids are final only now
        pending = false;
        sidl = row_id(i);
      }
      if (lt == 0) M2TRACE(0, i);
      if (i + 1 < ntiles && !(pending && (i + 2) * NB > n1)) sid_next = row_id(i + 1);
      const uint32_t dst = stg0 + st * STG_BYTES;
#pragma unroll
      for (int k = 0; k < (NH * OWN_CHUNKS + NLT - 1) / NLT; k++) {
        const int it = lt + NLT * k;
        const int row = it < NH * OWN_CHUNKS ? it / OWN_CHUNKS : 0;
        const int ch = it - row * OWN_CHUNKS;
        const int tok = (int)r * NH + row;
        const int sid = __shfl_sync(0xffffffffu, sidl, tok);
        if (it < NH * OWN_CHUNKS)
          cp_async16(dst + row * ROW + ch * 16, pool_rows + (int64_t)sid * ROW + ch * 16,
                     i * NB + tok < n ? 16u : 0u);
      }
#pragma unroll
      for (int k = 0; k < (NH * OTHER_CHUNKS + NLT - 1) / NLT; k++) {
        const int it = lt + NLT * k;
        const int row = it < NH * OTHER_CHUNKS ? it / OTHER_CHUNKS : 0;
        const int ch = it - row * OTHER_CHUNKS;
        const int tok = (1 - (int)r) * NH + row;
        const int sid = __shfl_sync(0xffffffffu, sidl, tok);
        const int soff = ch < 8 ? 128 * (int)r + 16 * ch : (ch < 16 ? 256 + 128 * (int)r + 16 * (ch - 8) : 512);
        if (it < NH * OTHER_CHUNKS)
          cp_async16(dst + STG_OWN + row * OTHER + ch * 16, pool_rows + (int64_t)sid * ROW + soff,
                     i * NB + tok < n ? 16u : 0u);
      }
      cp_async_arrive_noinc(&c.stg_full[st]);
      if (lt == 0) M2TRACE(9, i);
    }
    cp_async_wait_all();
  } else if (!F16) {
    // ================= dequantisers (4 warps): staging -> S tile, V tile ==============
    // Loads of an item group are issued together before any convert / store, and the
    // two 16-B halves of each dequantised chunk are stored in lane-dependent order so a
    // quarter warp's SW128 stores hit 8 distinct bank groups.
    const int ct = threadIdx.x - CONV0 * 32;  // 0..127
    const int wq = ct >> 5;                   // 0..3
    const uint32_t stg0 = smem_u32(stg), sS0 = smem_u32(sS), sV0 = smem_u32(sV);
    // S rows of tile j are dequantised DEQ_LAG tiles ahead of its V rows, so the score
    // MMAs never wait behind a V tile that waits on an earlier PV
    auto deq_s = [&](int i) {
      const int st = i % NST, ks = i % KSS;
      mbar_wait(&c.stg_full[st], (i / NST) & 1);
      if (ct == 0) M2TRACE(1, i);
      if (i >= KSS) mbar_wait(&c.s_empty[ks], ((i - KSS) / KSS) & 1);
      const uint32_t src = stg0 + st * STG_BYTES;
      const uint32_t sd = sS0 + ks * S_TILE;
      {  // own rows' NoPE: rows wq + 4k, chunk = lane (16 dims); RoPE: row ct / 8, chunk ct % 8
        uint4 v[4];
        float sc[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const uint32_t rp = src + (wq + 4 * k) * ROW;
          v[k] = lds128(rp + lane * 16);
          sc[k] = lds_f32(rp + 512 + 4 * (lane >> 3));
        }
        const int rrow = ct >> 3, rc = ct & 7;
        const uint4 rv = lds128(src + rrow * ROW + 528 + rc * 16);
        const int blk = lane >> 2, c0 = (lane & 3) * 2, odd = blk & 1;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int row = wq + 4 * k;
          uint4 lo, hi;
          deq16(v[k], scale_f16x2(sc[k]), lo, hi);
          const uint32_t dr = sd + blk * S_BLK + row * 128;
          const uint32_t a0 = dr + ((c0 ^ (row & 7)) << 4), a1 = dr + (((c0 + 1) ^ (row & 7)) << 4);
          sts128(odd ? a1 : a0, odd ? hi : lo);
          sts128(odd ? a0 : a1, odd ? lo : hi);
        }
        sts128(sd + 8 * S_BLK + rrow * 128 + ((rc ^ (rrow & 7)) << 4), cvt8_bf16_f16_sat(rv));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) arrive_on(&c.s_full[ks], 0);
      if (ct == 0) M2TRACE(2, i);
    };
    auto deq_v = [&](int i) {
      const int st = i % NST, kv = i % KSV;
      const uint32_t src = stg0 + st * STG_BYTES;
      // V: 32 tokens x this CTA's 256 NoPE dims (16 chunks) -> V tile [32][4 x 64] SW128;
      // item k: token (ct / 16) + 8k (tokens 16r..16r+15 are this CTA's own rows), chunk ct % 16
      if (i >= KSV) mbar_wait(&c.v_empty[kv], ((i - KSV) / KSV) & 1);
      const uint32_t vd = sV0 + kv * V_TILE;
      const int ch = ct & 15;
      {
        uint4 v[4];
        float sc[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int tok = (ct >> 4) + 8 * k;
          const int jr = tok & (NH - 1);
          if ((tok >> 4) == (int)r) {  // warp-uniform
            const int cabs = (ch < 8 ? 8 * (int)r : 16 + 8 * (int)r) + (ch & 7);
            const uint32_t rp = src + jr * ROW;
            v[k] = lds128(rp + cabs * 16);
            sc[k] = lds_f32(rp + 512 + 4 * (cabs >> 3));
          } else {
            const uint32_t rp = src + STG_OWN + jr * OTHER;
            v[k] = lds128(rp + ch * 16);
            sc[k] = lds_f32(rp + 256 + 4 * (ch < 8 ? (int)r : 2 + (int)r));
          }
        }
        const int vb = ch >> 2, c0 = (ch & 3) * 2, odd = vb & 1;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int tok = (ct >> 4) + 8 * k;
          uint4 lo, hi;
          deq16(v[k], scale_f16x2(sc[k]), lo, hi);
          const uint32_t dr = vd + vb * V_BLK + tok * 128;
          const uint32_t a0 = dr + ((c0 ^ (tok & 7)) << 4), a1 = dr + (((c0 + 1) ^ (tok & 7)) << 4);
          sts128(odd ? a1 : a0, odd ? hi : lo);
          sts128(odd ? a0 : a1, odd ? lo : hi);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        arrive_on(&c.v_full[kv], 0);
        mbar_arrive(&c.stg_empty[st]);
      }
      if (ct == 0) M2TRACE(3, i);
    };
    for (int it = 0; it < ntiles + DEQ_LAG; it++) {
      if (it < ntiles) deq_s(it);
      if (it >= DEQ_LAG) deq_v(it - DEQ_LAG);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (await && threadIdx.x == 0) {
    if (atomicAdd(landed + b, LANDED_TAG) >= (2 * nsplit - 1) * LANDED_TAG) atomicExch(landed + b, 0);
  }
  cluster_sync_all();  // no more remote arrives / peer operand reads; then free TMEM
  tc_fence_after();
  if (warp == MMA_WARP) tmem_dealloc2(tmem);
}

}  // namespace

#ifdef ESS_MLA2_TRACE
extern "C" int ess_debug_mla2_trace(unsigned long long *dst) {
  return cudaMemcpyFromSymbol(dst, g_mla2_trace, sizeof(g_mla2_trace)) == cudaSuccess ? 0 : -1;
}
#endif

// launched by mla.cu's entry points: the FP8 kernel for 656-B slot rows, the f16 pair
// kernel for 1152-B rows
int ess_launch_mla_pair(ess_pool *pool, int32_t pool_begin, const void *d_q, const int32_t *d_sel_row,
                        const int32_t *d_sel2, int32_t *d_landed, int32_t sel_stride,
                        const int32_t *d_count, int32_t count_stride, int32_t batch, float sm_scale,
                        void *d_out, float *d_lse, float *d_ws_o, float *d_ws_ml, int32_t flags,
                        int32_t nsplit, void *stream) {
  // q as a [batch * 128 heads][576] bf16 tensor, boxes of [64 heads][64 dims], SW128
  struct QMap {
    const void *base = nullptr;
    int32_t batch = 0;
    int dev = -1;
    CUtensorMap map;
  };
  static thread_local QMap qm;
  int dev = 0;
  ESS_CUDA_TRY(cudaGetDevice(&dev));
  alignas(64) CUtensorMap tq;
  if (qm.base == d_q && qm.batch == batch && qm.dev == dev) {
    tq = qm.map;
  } else {
    if (!ess_make_tmap_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, d_q, ESS_MLA_QK_DIM, (uint64_t)batch * HEADS,
                          ESS_MLA_QK_DIM * 2, 64, HH, CU_TENSOR_MAP_SWIZZLE_128B))
      return ESS_ERR_CUDA;
    qm.base = d_q;
    qm.batch = batch;
    qm.dev = dev;
    qm.map = tq;
  }
  const bool f16 = pool->row_bytes == ESS_SLOT_ROW_BYTES;
  const void *fn = f16 ? (const void *)sparse_mla_pair_kernel<true> : (const void *)sparse_mla_pair_kernel<false>;
  const size_t smem = f16 ? F_SMEM_BYTES : SMEM_BYTES;
  if (int rc = ess_smem_optin(fn, smem)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2, (unsigned)(batch * nsplit));
  cfg.blockDim = dim3(f16 ? F_NTHREADS : NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (f16)
    ESS_CUDA_TRY(cudaLaunchKernelEx(&cfg, sparse_mla_pair_kernel<true>, tq, (const uint8_t *)pool->rows,
                                    pool->rows_per_pool, (int)pool_begin, d_sel_row, d_sel2, d_landed,
                                    (int)sel_stride, d_count, (int)count_stride, sm_scale, (uint16_t *)d_out,
                                    d_lse, d_ws_o, d_ws_ml, (int)flags, (int)nsplit, pool->status));
  else
    ESS_CUDA_TRY(cudaLaunchKernelEx(&cfg, sparse_mla_pair_kernel<false>, tq, (const uint8_t *)pool->rows,
                                    pool->rows_per_pool, (int)pool_begin, d_sel_row, d_sel2, d_landed,
                                    (int)sel_stride, d_count, (int)count_stride, sm_scale, (uint16_t *)d_out,
                                    d_lse, d_ws_o, d_ws_ml, (int)flags, (int)nsplit, pool->status));
  return ESS_OK;
}

int ess_preload_mla2() {  // see ess_preload_indexer
  cudaFuncAttributes a;
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)sparse_mla_pair_kernel<true>));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)sparse_mla_pair_kernel<false>));
  return ESS_OK;
}
