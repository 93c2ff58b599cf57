// K5: sparse MLA decode over the selected slot rows (op "sparse_mla",
// costmodel.py:18-27).
//
// out[h] = softmax_j(q[h] . K[j] * sm_scale) V[j], K[j] = NoPE ++ RoPE (576 f16),
// V[j] = NoPE (512 f16), over the count[b] slot rows sel_row[b][:].  Slot rows are
// attention-ready f16 (dequantised once on admission by K4), so this kernel is a
// pure row-gather + tensor-core kernel.
//
// TMEM budget drives the split: the fp32 output of 128 heads x 512 dims is 256 KB,
// the whole TMEM of one SM, so each request runs on two CTAs that own 256 output
// dims each and both compute the full score tile S.  Per CTA (512 TMEM columns):
//   O      [0,256)    fp32 accumulator, 128 heads x 256 dims
//   S0..S2 [256,352)  fp32 scores, 32 rows each; P (f16) overwrites the first 16
//                     columns of its S buffer and feeds PV straight from TMEM
//   Qt     [352,512)  q dims 0..319 as f16 pairs: the A operand of S from TMEM
// Three S buffers let the MMA warp issue S(i+1) and S(i+2) before PV(i), so the
// softmax of tile i and the p_full -> PV hand-off hide behind two score tiles on
// the tensor pipe (with two buffers that per-tile round trip set K5's rate).
// Shared memory: q dims 320..575 (SW128 K-major, 64 KB), a 4-deep ring of KV tiles
// (32 rows x 576 f16, SW128: 9 blocks of [32 rows][64 dims]) filled by 16-B
// cp.async straight into the swizzled positions (TMA tile::gather4 moves only
// 4 x 128 B per instruction and was instruction-rate bound here), and the
// request's slot ids.
//
// Warp roles (288 threads): w0-3 softmax (thread = head; online softmax in exp2
// domain with lazy O rescaling when the running max grows by > 8), w4 TMEM alloc +
// MMA issuer (S = Q K^T: M=128, N=32, 36 x K=16; O += P V: M=128, N=256, V read as
// the MN-major view of the same tile), w5-8 row loaders.
#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

#ifdef ESS_MLA_TRACE  // scratch builds: per-tile globaltimer stamps of CTA (0, 0)
__device__ unsigned long long g_mla_trace[8][72];
#define MTRACE(ev, i)                                                                  \
  do {                                                                                 \
    if (blockIdx.x == 0 && blockIdx.y == 0 && (i) < 72) {                              \
      unsigned long long tt;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                           \
      g_mla_trace[ev][i] = tt;                                                         \
    }                                                                                  \
  } while (0)
extern "C" int ess_debug_mla_trace(unsigned long long *host) {
  return cudaMemcpyFromSymbol(host, g_mla_trace, sizeof(g_mla_trace)) == cudaSuccess ? 0 : -7;
}
#else
#define MTRACE(ev, i) \
  do {                \
  } while (0)
#endif

namespace {

constexpr int HEADS = ESS_MLA_HEADS;      // 128 = M
constexpr int QK_DIM = ESS_MLA_QK_DIM;    // 576
constexpr int V_HALF = 256;               // output dims per CTA
#ifndef ESS_MLA_NB
#define ESS_MLA_NB 32
#endif
constexpr int NB = ESS_MLA_NB;            // KV rows per tile (32, or 64: half the tiles)
constexpr int NBLK = QK_DIM / 64;         // 9 dim-blocks of 64 (128 B of f16)
#ifndef ESS_MLA_NSB
#define ESS_MLA_NSB 2
#endif
#ifndef ESS_MLA_QT_BLKS
#define ESS_MLA_QT_BLKS (ESS_MLA_NB == 64 ? 4 : 6)
#endif
constexpr int QT_BLKS = ESS_MLA_QT_BLKS;  // q blocks held in TMEM (dims 0..64*QT_BLKS-1)
constexpr int QS_BLKS = NBLK - QT_BLKS;   // q blocks in shared memory (dims 320..575)
constexpr int NSB = ESS_MLA_NSB;          // S/P buffers: S(i+NSB-1) is issued before PV(i)
constexpr int LOOKAHEAD = NSB - 1;
constexpr int QBLK_BYTES = HEADS * 128;            // one [128 heads][64 dims] block
constexpr int QS_BYTES = QS_BLKS * QBLK_BYTES;     // 65536
constexpr int KV_BLK_BYTES = NB * 128;             // 4096
constexpr int KV_BYTES = NBLK * KV_BLK_BYTES;      // 36864
constexpr int KS = NB == 64 ? 2 : 4;               // KV ring depth
// 64-row tiles: the selected slot ids are read from global memory per tile (no room
// for the 8-KB id copy in shared memory)
constexpr bool SSEL_SMEM = NB != 64;
// Loader completion: 1 = each thread's cp.async completion arrives on the tile barrier
// (cp.async.mbarrier.arrive.noinc); 0 = wait_group + proxy fence + one arrive per warp,
// the form compute-sanitizer's racecheck models (same speed at two S buffers).
#ifndef ESS_MLA_SPIN  // 1: spin with test_wait on the per-tile S / P hand-offs
#define ESS_MLA_SPIN 0
#endif
#ifndef ESS_MLA_ASYNC_ARRIVE
#define ESS_MLA_ASYNC_ARRIVE (ESS_MLA_NB == 64 ? 1 : 0)
#endif
#ifndef ESS_MLA_DBG_NOLOAD  // timing-only switches for scratch builds (scripts/variant_lib.sh)
#define ESS_MLA_DBG_NOLOAD 0
#endif
#ifndef ESS_MLA_DBG_NOMMA
#define ESS_MLA_DBG_NOMMA 0
#endif
#ifndef ESS_MLA_DBG_ALLSS
#define ESS_MLA_DBG_ALLSS 0
#endif
#ifndef ESS_MLA_DBG_NOSOFT
#define ESS_MLA_DBG_NOSOFT 0
#endif
// the MMA warp issues S(i+LOOKAHEAD) before PV(i) frees slot i: the ring must hold
// tiles i..i+LOOKAHEAD at once
static_assert(KS >= LOOKAHEAD + 1, "KV ring too shallow for the S lookahead");
// wait_group loader: tile j is signalled after tile j+1 is issued, i.e. once slot
// (j+1) % KS is free; S(i+LOOKAHEAD) must not wait for PV(i) -> KS >= LOOKAHEAD + 3
static_assert(ESS_MLA_ASYNC_ARRIVE || KS >= LOOKAHEAD + 3, "KV ring too shallow for the lagged loader");
constexpr int MAX_N = ESS_MAX_REQUEST;
constexpr int NSOFT = 4, NLOAD = 4;
constexpr int MMA_WARP = NSOFT, LOAD0 = NSOFT + 1;
constexpr int NTHREADS = 32 * (NSOFT + 1 + NLOAD);  // 288
constexpr int ROWS_PER_LOADER = NB / NLOAD;         // 8
constexpr int SLOT_CHUNKS = ESS_SLOT_ROW_BYTES / 16; // 72
constexpr uint32_t TM_O = 0, TM_S = 256, TM_Q = TM_S + NSB * NB;  // Q: [352, 512)
static_assert(TM_Q + QT_BLKS * 32 <= 512, "TMEM budget");
constexpr float RESCALE_THRESHOLD = 8.0f;
constexpr int MLA_AWAIT = 4;  // internal flag of ess_sparse_mla_da
#ifndef ESS_MLA_DBG_SN
#define ESS_MLA_DBG_SN NB
#endif
constexpr uint32_t IDESC_S = make_idesc(0 /*f16*/, 0 /*f16*/, HEADS, ESS_MLA_DBG_SN, 0, 0);
constexpr uint32_t IDESC_PV = make_idesc(0, 0, HEADS, V_HALF, 0, 1 /*B MN-major*/);

struct Ctrl {
  uint64_t kv_full[KS], kv_empty[KS];
  uint64_t s_full[NSB], p_full[NSB], pv_done[NSB], o_done, q_full;
  uint32_t tmem;
};
constexpr size_t SMEM_BYTES = 1024 + QS_BYTES + KS * KV_BYTES + (SSEL_SMEM ? MAX_N * 4 : 0) + sizeof(Ctrl);
static_assert(SMEM_BYTES <= 232448, "K5 shared memory over the sm_100 limit");

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 2^x in one MUFU op (ftz: subnormal results flush to 0, far below f16 P's range)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// (lo, hi) -> f16x2, round to nearest, one instruction
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// 16-B async global -> shared copy (L1 bypass); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// arrive on an mbarrier when every cp.async this thread issued so far has completed
// (the arrive counts toward the barrier's expected count)
[[maybe_unused]] __device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Arrival counter of the fused DA schedule: the low 24 bits count rows the gather has
// landed (release adds); each of the request's two CTAs adds LANDED_TAG once it no
// longer needs the counter, and the second one resets it to 0 for the next step (the
// next gather starts only after this kernel completed).
constexpr int LANDED_TAG = 1 << 24;
__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// One lane polls (acquire, GPU scope) until target rows landed, then every lane
// acquires once itself, so the slot rows published before the gather's release adds
// are visible to its cp.async.cg loads.
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
}

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_mla_kernel(const __grid_constant__ CUtensorMap tm_q, const uint8_t *__restrict__ rows,
                      int64_t rows_per_pool, int pool_begin, const int32_t *__restrict__ sel_row,
                      const int32_t *__restrict__ sel2, int32_t *landed,
                      int sel_stride, const int32_t *__restrict__ counts, int count_stride,
                      float sm_scale, uint16_t *__restrict__ out, float *__restrict__ lse,
                      float *__restrict__ ws_o, float *__restrict__ ws_ml, int flags, int nsplit,
                      int32_t *status) {
  extern __shared__ uint8_t smem_raw[];
  // offset from the shared array itself (keeps the shared address space: LDS/STS, not generic)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sq = smem;                        // q dims 320..575, 4 SW128 blocks
  uint8_t *skv = sq + QS_BYTES;              // KS f16 KV tiles
  int32_t *ssel = reinterpret_cast<int32_t *>(skv + KS * KV_BYTES);
  Ctrl &c = *reinterpret_cast<Ctrl *>(ssel + (SSEL_SMEM ? MAX_N : 0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v = blockIdx.x;  // output half
  const int split = blockIdx.y % nsplit;     // KV split: one share of the rows
  const int b = blockIdx.y / nsplit;
  const bool partial = flags & ESS_MLA_PARTIAL, resume = flags & ESS_MLA_RESUME;
  // split CTAs leave unnormalised partial states in the workspace; a combine kernel
  // merges them (small batches: 2 * nsplit CTAs per request fill the GPU)
  const bool to_ws = partial || nsplit > 1;
  // fused DA: rows sel_row[0:n1t) are resident, sel2[0:n2t) land during the kernel
  const bool await = flags & MLA_AWAIT;
  const int n1t = min(counts[(int64_t)b * count_stride], MAX_N);
  const int n2t = await ? min(counts[(int64_t)b * count_stride + 1], MAX_N - n1t) : 0;
  // Each share takes an equal slice of the resident rows AND of the fetched rows (its list is
  // [hits h0..h1) ++ [misses m0..m1)), so every share overlaps its own hits with the gather
  // and the post-arrival tail is ~n2t/nsplit rows instead of all of them in the last share.
  const int h0 = n1t * split / nsplit, h1 = n1t * (split + 1) / nsplit;
  const int m0 = n2t * split / nsplit, m1 = n2t * (split + 1) / nsplit;
  const int n1 = h1 - h0;                    // resident rows of this share
  const int n = n1 + (m1 - m0);
  const bool fetched = m1 > m0;              // the share holds fetched rows
  const int ntiles = (n + NB - 1) / NB;

  if (threadIdx.x == 0) {
    for (int i = 0; i < KS; i++) {
      // async-arrive: one cp.async completion arrive per loader thread; else one per warp
      mbar_init(&c.kv_full[i], ESS_MLA_ASYNC_ARRIVE ? NLOAD * 32 : NLOAD);
      mbar_init(&c.kv_empty[i], 1);
    }
    for (int i = 0; i < NSB; i++) {
      mbar_init(&c.s_full[i], 1);
      mbar_init(&c.p_full[i], NSOFT);
      mbar_init(&c.pv_done[i], 1);
    }
    mbar_init(&c.o_done, 1);
    mbar_init(&c.q_full, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc<512>(&c.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = c.tmem;

  // ---- prologue: q -> TMEM (dims 0..319) and smem (320..575); slot ids -> smem ----
  // Nine TMA box loads of [128 heads][64 dims] bf16 (SW128): blocks 5..8 land in their
  // final shared-memory place and are converted to f16 in place; blocks 0..4 land in
  // the still-empty KV ring, where each head's 128-B row is read bank-conflict free
  // (the swizzle spreads the 8 lanes of a phase over 8 chunks) and stored to TMEM.
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&c.q_full, HEADS * QK_DIM * 2);
    for (int blk = 0; blk < NBLK; blk++)
      tma_load_2d(blk < QT_BLKS ? skv + blk * QBLK_BYTES : sq + (blk - QT_BLKS) * QBLK_BYTES, &tm_q,
                  &c.q_full, blk * 64, b * HEADS);
  }
  if (SSEL_SMEM && warp >= LOAD0) {
    const int32_t *sel = sel_row + (int64_t)b * sel_stride;
    const int32_t *s2 = await ? sel2 + (int64_t)b * sel_stride : nullptr;
    for (int j = threadIdx.x - LOAD0 * 32; j < n; j += NLOAD * 32) {
      ssel[j] = j < n1 ? __ldg(sel + h0 + j) : __ldg(s2 + m0 + (j - n1));
    }
  }
  mbar_wait(&c.q_full, 0);
  if (warp < NSOFT) {
    const int h = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
#pragma unroll 1
    for (int cc = 0; cc < QT_BLKS; cc++) {  // 64 dims = 32 columns per block
      const uint8_t *rowp = skv + cc * QBLK_BYTES + h * 128;
      uint32_t r[32];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint4 y = cvt8_bf16_f16(*reinterpret_cast<const uint4 *>(rowp + ((k ^ (h & 7)) << 4)));
        bad |= f16x8_nonfinite(y);
        r[4 * k] = y.x;
        r[4 * k + 1] = y.y;
        r[4 * k + 2] = y.z;
        r[4 * k + 3] = y.w;
      }
      tmem_st_32x32b_x32(tmem + lane_base + TM_Q + cc * 32, r);
#ifndef ESS_NO_RANGE_LATCH
      if (bad) ess_set_status(status, ESS_ERR_RANGE);  // q outside the f16 range
#endif
    }
    tmem_st_wait();
  } else {
    // warps 4-8: q dims 320..575 to f16 in place (16-B units keep their SW128 position)
    constexpr int NT = NTHREADS - NSOFT * 32;
    uint4 *qs = reinterpret_cast<uint4 *>(sq);
    bool bad = false;
    for (int u = threadIdx.x - NSOFT * 32; u < QS_BYTES / 16; u += NT) {
      const uint4 y = cvt8_bf16_f16(qs[u]);
      bad |= f16x8_nonfinite(y);
      qs[u] = y;
    }
#ifndef ESS_NO_RANGE_LATCH
    if (bad) ess_set_status(status, ESS_ERR_RANGE);
#endif
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const float scale_log2 = sm_scale * 1.4426950408889634f;

  if (warp < NSOFT) {
    // ---------------- softmax / epilogue warps: thread = head --------------------
    const int h = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const int64_t hrow = (int64_t)b * HEADS + h;
    const int64_t wrow = (int64_t)(b * nsplit + split) * HEADS + h;  // workspace row
    float *wso = ws_o ? ws_o + wrow * ESS_MLA_V_DIM + v * V_HALF : nullptr;
    float m_run = -INFINITY, l_run = 0.f;  // resume starts a fresh partial, merged at the end
    for (int i = 0; i < ntiles; i++) {
      const int sb = i % NSB;
#if ESS_MLA_SPIN
      mbar_spin(&c.s_full[sb], (i / NSB) & 1);
#else
      mbar_wait(&c.s_full[sb], (i / NSB) & 1);
#endif
      if (threadIdx.x == 0) MTRACE(2, i);  // softmax sees S(i)
      // observe PV(i - NSB)'s pv_done phase: s_full(i) tracks it (issued before S(i)), so
      // this never stalls; every phase gets a waiter (compute-sanitizer synccheck)
      if (i >= NSB) mbar_wait(&c.pv_done[sb], ((i - NSB) / NSB) & 1);
      tc_fence_after();
#if ESS_MLA_DBG_NOSOFT
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.p_full[sb]);
      continue;
#endif
      uint32_t s[NB];
      if constexpr (NB == 64) tmem_ld_32x32b_x64(tmem + lane_base + TM_S + sb * NB, *reinterpret_cast<uint32_t(*)[64]>(s));
      else tmem_ld_32x32b_x32(tmem + lane_base + TM_S + sb * NB, *reinterpret_cast<uint32_t(*)[32]>(s));
      tmem_ld_wait();
      // raw scores; the scale folds into the exp2 argument (one FFMA per score)
      float x[NB];
      const int lim = n - i * NB;  // valid columns of this tile (uniform)
#pragma unroll
      for (int j = 0; j < NB; j++) x[j] = j < lim ? __uint_as_float(s[j]) : -INFINITY;
      float m0 = fmaxf(x[0], x[1]), m1 = fmaxf(x[2], x[3]);
#pragma unroll
      for (int j = 4; j < NB; j += 4) {
        m0 = fmaxf(m0, fmaxf(x[j], x[j + 1]));
        m1 = fmaxf(m1, fmaxf(x[j + 2], x[j + 3]));
      }
      const float mt = fmaxf(m0, m1) * scale_log2;
      // warp-uniform decision (tcgen05.ld/st are .sync.aligned); a lane whose own
      // max did not grow rescales by alpha = 1
      if (__any_sync(0xffffffffu, mt > m_run + RESCALE_THRESHOLD) || i == 0) {
        const float m_new = fmaxf(mt, m_run);
        const float alpha = exp2f(m_run - m_new);  // 0 when m_run = -inf
        l_run *= alpha;
        // PV(i-1) accumulates into O: wait for it before O is rescaled.  Only rescale
        // tiles wait, keeping the MMA round trip off the per-tile path.  pv_done[k % 3]
        // completes its phase k / 3 when PV(k) is done; the parity is unambiguous: the
        // s_full(i) commit tracks every MMA issued before S(i), PV(i-3) included, so
        // that barrier's previous phase (PV(i-4)) is complete, and PV(i+2) needs a P
        // this warp has not produced yet.
        if (i > 0) {
          mbar_wait(&c.pv_done[(i - 1) % NSB], ((i - 1) / NSB) & 1);
          tc_fence_after();
        }
        if (i > 0) {  // O holds PV(i-1)
#pragma unroll 1
          for (int cc = 0; cc < V_HALF / 32; cc++) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; j++) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
            tmem_st_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
          }
        }
        m_run = m_new;
      }
      // P (f16 pairs) over the first 16 columns of this S buffer: p = 2^(x*scale - m)
      // (ex2.approx, one MUFU op), packed two per cvt; l sums the unrounded values in
      // four independent chains (the f16 rounding of P is below the tolerance budget)
      uint32_t p[NB / 2];
      float ls0 = 0.f, ls1 = 0.f, ls2 = 0.f, ls3 = 0.f;
      const float nm = -m_run;
#pragma unroll
      for (int e = 0; e < NB / 2; e += 2) {
        const float e0 = fast_exp2(fmaf(x[2 * e], scale_log2, nm));
        const float e1 = fast_exp2(fmaf(x[2 * e + 1], scale_log2, nm));
        const float e2 = fast_exp2(fmaf(x[2 * e + 2], scale_log2, nm));
        const float e3 = fast_exp2(fmaf(x[2 * e + 3], scale_log2, nm));
        p[e] = pack_f16x2(e0, e1);
        p[e + 1] = pack_f16x2(e2, e3);
        ls0 += e0;
        ls1 += e1;
        ls2 += e2;
        ls3 += e3;
      }
      l_run += (ls0 + ls1) + (ls2 + ls3);
      if constexpr (NB == 64) tmem_st_32x32b_x32(tmem + lane_base + TM_S + sb * NB, *reinterpret_cast<const uint32_t(*)[32]>(p));
      else tmem_st_32x32b_x16(tmem + lane_base + TM_S + sb * NB, *reinterpret_cast<const uint32_t(*)[16]>(p));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.p_full[sb]);
      if (threadIdx.x == 0) MTRACE(3, i);  // softmax warp 0 arrived P(i)
    }
    // ---------------- epilogue ---------------------------------------------------
    const bool have_o = ntiles > 0;  // TMEM O holds a valid accumulator
    if (ntiles > 0) {
      mbar_wait(&c.o_done, 0);
      for (int k = max(0, ntiles - NSB); k < ntiles; k++)  // the last PV phases (all done)
        mbar_wait(&c.pv_done[k % NSB], (k / NSB) & 1);
      tc_fence_after();
    }
    if (to_ws) {
      // pass 1 of the split attention / a KV split: unnormalised O and (max, sum) to
      // the workspace
#pragma unroll 1
      for (int cc = 0; cc < V_HALF / 32; cc++) {
        uint32_t o[32];
        if (have_o) {
          tmem_ld_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int j = 0; j < 32; j++) o[j] = 0u;
        }
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4 *>(wso + cc * 32 + j) =
              make_float4(__uint_as_float(o[j]), __uint_as_float(o[j + 1]),
                          __uint_as_float(o[j + 2]), __uint_as_float(o[j + 3]));
      }
      if (v == 0) {
        ws_ml[wrow * 2 + 0] = m_run;
        ws_ml[wrow * 2 + 1] = l_run;
      }
    } else {
      // final output.  Resume mode merges this pass's O (TMEM) with pass 1's
      // unnormalised state from the workspace, streamed with a one-chunk prefetch:
      // out = (O0 a0 + O1 a1) / (l0 a0 + l1 a1), a_k = 2^(m_k - max(m0, m1)).
      float m = m_run, l = l_run, a0 = 0.f, a1 = have_o ? 1.f : 0.f;
      if (resume) {
        const float m0 = ws_ml[hrow * 2 + 0], l0 = ws_ml[hrow * 2 + 1];
        m = fmaxf(m0, m_run);
        a0 = m0 == -INFINITY ? 0.f : exp2f(m0 - m);
        a1 = (have_o && m_run != -INFINITY) ? exp2f(m_run - m) : 0.f;
        l = l0 * a0 + l_run * a1;
      }
      uint16_t *ob = out + hrow * ESS_MLA_V_DIM + v * V_HALF;
      // Every lane runs the epilogue (tcgen05.ld is .sync.aligned: a per-lane branch
      // around it would leave a partial warp — a hang when one head's l is NaN from an
      // out-of-range operand).  l == 0 (no rows): zeros, lse -inf; l NaN: NaN out.
      {
        const bool pos = l > 0.f;
        const float inv = 1.f / l;
        const float c0 = pos ? a0 * inv : (l == l ? 0.f : l), c1 = pos ? a1 * inv : c0;
        // pass 1's unnormalised state of this head (1 KB) is staged through the q
        // tile's shared memory (free once o_done fired: every S MMA has completed; never
        // touched by the row loaders) in two 512-B halves, [16-B unit][head], each half's
        // 32 copies in flight at once.  A thread stages and reads only its own head.
        const uint4 *wst = reinterpret_cast<const uint4 *>(sq);
#pragma unroll 1
        for (int cc = 0; cc < V_HALF / 32; cc++) {
          if (resume && (cc & 3) == 0) {
            const uint32_t st = smem_u32(sq);
            const int u0 = (cc >> 2) * 32;
#pragma unroll 8
            for (int k = 0; k < 32; k++) cp_async16(st + (k * HEADS + h) * 16, wso + 4 * (u0 + k), 16u);
            cp_async_commit();
            cp_async_wait<0>();
          }
          float4 w[8];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            if (resume) {
              const uint4 u = wst[((cc & 3) * 8 + j) * HEADS + h];
              w[j] = make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z),
                                 __uint_as_float(u.w));
            } else {
              w[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          uint32_t o[32];
          if (have_o) {
            tmem_ld_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int j = 0; j < 32; j++) o[j] = 0u;
          }
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            const float4 p = w[j / 4], q4 = w[j / 4 + 1];
            __nv_bfloat162 t0 = __floats2bfloat162_rn(__uint_as_float(o[j]) * c1 + p.x * c0,
                                                      __uint_as_float(o[j + 1]) * c1 + p.y * c0);
            __nv_bfloat162 t1 = __floats2bfloat162_rn(__uint_as_float(o[j + 2]) * c1 + p.z * c0,
                                                      __uint_as_float(o[j + 3]) * c1 + p.w * c0);
            __nv_bfloat162 t2 = __floats2bfloat162_rn(__uint_as_float(o[j + 4]) * c1 + q4.x * c0,
                                                      __uint_as_float(o[j + 5]) * c1 + q4.y * c0);
            __nv_bfloat162 t3 = __floats2bfloat162_rn(__uint_as_float(o[j + 6]) * c1 + q4.z * c0,
                                                      __uint_as_float(o[j + 7]) * c1 + q4.w * c0);
            uint4 pk;
            pk.x = *reinterpret_cast<uint32_t *>(&t0);
            pk.y = *reinterpret_cast<uint32_t *>(&t1);
            pk.z = *reinterpret_cast<uint32_t *>(&t2);
            pk.w = *reinterpret_cast<uint32_t *>(&t3);
            *reinterpret_cast<uint4 *>(ob + cc * 32 + j) = pk;
          }
        }
        if (v == 0) lse[hrow] = pos ? (m + log2f(l)) * 0.6931471805599453f : (l == l ? -INFINITY : l);
      }
    }
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer --------------------------------------------------
    if (elect_one() && ntiles > 0) {
      const uint64_t abase = sw128_desc(smem_u32(sq), 16, 1024);
      auto issue_s = [&](int i) {
        const int kb = i % KS, sb = i % NSB;
        // S(i) overwrites S/P buffer sb, last read by PV(i-3) as its A operand.  No
        // wait: softmax(i-3) finished with the buffer before p_full(i-3), PV(i-3) was
        // issued before this S(i), and one thread's tcgen05.mma ops execute in issue
        // order — waiting for PV(i-3) to complete would idle the tensor pipe each tile.
        mbar_wait(&c.kv_full[kb], (i / KS) & 1);
        MTRACE(0, i);  // tile i rows in smem (MMA view)
        fence_proxy_async_smem();  // cp.async (generic proxy) rows -> tensor-core reads
        tc_fence_after();
        const uint32_t d = tmem + TM_S + sb * NB;
        // descriptors as base + compile-time offsets (the 14-bit address field cannot
        // carry: shared memory ends below 2^18 B), so the fully unrolled 36-MMA
        // sequence issues back to back instead of rebuilding each descriptor
        const uint64_t bbase = sw128_desc(smem_u32(skv + kb * KV_BYTES), 16, 1024);
#pragma unroll
        for (int blk = 0; blk < NBLK; blk++) {
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            const uint64_t bd = bbase + (uint64_t)((blk * KV_BLK_BYTES + kk * 32) >> 4);
            const uint32_t acc = (blk | kk) ? 1u : 0u;
            if (ESS_MLA_DBG_NOMMA) continue;
            if (ESS_MLA_DBG_ALLSS || blk >= QT_BLKS) {
              const int qb = ESS_MLA_DBG_ALLSS ? blk % QS_BLKS : blk - QT_BLKS;
              mma_f16_ss(d, abase + (uint64_t)((qb * HEADS * 128 + kk * 32) >> 4), bd, IDESC_S, acc);
            } else {
              mma_f16_ts(d, tmem + TM_Q + (blk * 4 + kk) * 8, bd, IDESC_S, acc);
            }
          }
        }
        tc_commit(&c.s_full[sb]);
        MTRACE(1, i);  // S(i) issued
      };
      // two score tiles in flight ahead of PV: the softmax of tile i and the
      // p_full -> PV hand-off overlap S(i+1) and S(i+2) on the tensor pipe
      for (int i = 0; i < LOOKAHEAD && i < ntiles; i++) issue_s(i);
      for (int i = 0; i < ntiles; i++) {
        if (i + LOOKAHEAD < ntiles) issue_s(i + LOOKAHEAD);
        const int kb = i % KS, sb = i % NSB;
#if ESS_MLA_SPIN
        mbar_spin(&c.p_full[sb], (i / NSB) & 1);
#else
        mbar_wait(&c.p_full[sb], (i / NSB) & 1);
#endif
        MTRACE(4, i);  // MMA sees P(i)
        tc_fence_after();
        const uint32_t vaddr = smem_u32(skv + kb * KV_BYTES) + (uint32_t)(4 * v) * KV_BLK_BYTES;
#pragma unroll
        for (int kk = 0; kk < NB / 16; kk++) {
          uint64_t bd = sw128_desc(vaddr + kk * 16 * 128, KV_BLK_BYTES, 1024);
          if (!ESS_MLA_DBG_NOMMA)
            mma_f16_ts(tmem + TM_O, tmem + TM_S + sb * NB + kk * 8, bd, IDESC_PV, (i | kk) ? 1u : 0u);
        }
        tc_commit(&c.pv_done[sb]);
        MTRACE(5, i);  // PV(i) issued
        tc_commit(&c.kv_empty[kb]);
        if (i == ntiles - 1) tc_commit(&c.o_done);
      }
    }
  } else {
    // ---------------- row loaders: warp w owns rows 8w..8w+7 of every tile; each lane
    // copies 16-B chunks (lane, lane+32, lane+64 < 72) of those rows with cp.async
    // straight into the SW128 position; one commit group per tile, signalled one
    // tile later (wait_group 1) so two tiles are in flight per warp ----------------
    const int w = warp - LOAD0;
    const uint8_t *pool_rows = rows + (int64_t)(pool_begin + b / (((flags >> ESS_MLA_QTOK_SHIFT) & 7) + 1)) * rows_per_pool * ESS_SLOT_ROW_BYTES;
    const uint32_t kv0 = smem_u32(skv);
    [[maybe_unused]] auto signal = [&](int i) {
      fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.kv_full[i % KS]);
    };
    bool pending = fetched && n2t > 0;  // fetched rows not yet known to have landed
    for (int i = 0; i < ntiles; i++) {
      const int kb = i % KS;
      mbar_wait(&c.kv_empty[kb], ((i / KS) & 1) ^ 1);
      if (pending && (i + 1) * NB > n1) {  // first tile holding fetched rows
        wait_landed(landed + b, n2t);
        pending = false;
      }
      const uint32_t kv = kv0 + kb * KV_BYTES;
#pragma unroll
      for (int rr = 0; rr < ROWS_PER_LOADER; rr++) {
        const int r = w * ROWS_PER_LOADER + rr;
        const int j = i * NB + r;
        const bool ok = j < n;
        int sid;
        if constexpr (SSEL_SMEM) {
          sid = ssel[ok ? j : 0];
        } else {  // the id straight from global (L2-resident; warp-uniform per row)
          const int jj = ok ? j : 0;
          sid = jj < n1 ? __ldg(sel_row + (int64_t)b * sel_stride + h0 + jj)
                        : __ldg(sel2 + (int64_t)b * sel_stride + m0 + (jj - n1));
        }
        const uint8_t *src = pool_rows + (int64_t)sid * ESS_SLOT_ROW_BYTES;
#pragma unroll
        for (int k = 0; k < 3; k++) {
          const int ch = lane + 32 * k;
          if (ch < SLOT_CHUNKS && !ESS_MLA_DBG_NOLOAD)
            cp_async16(kv + (ch >> 3) * KV_BLK_BYTES + r * 128 + (((ch & 7) ^ (r & 7)) << 4),
                       src + ch * 16, ok ? 16u : 0u);
        }
      }
#if ESS_MLA_ASYNC_ARRIVE
      // tile i is full once every loader thread's copies landed: each thread's
      // completion arrives on kv_full by itself, so no loader waits on its own copies
      // and the ring runs as far ahead as the free slots allow
      cp_async_arrive_noinc(&c.kv_full[kb]);
#else
      // one commit group per tile, signalled one tile later (wait_group 1: two tiles
      // in flight per warp); the generic->async proxy fence precedes the arrive
      cp_async_commit();
      if (i >= 1) {
        cp_async_wait<1>();
        signal(i - 1);
      }
#endif
    }
    cp_async_wait<0>();
#if !ESS_MLA_ASYNC_ARRIVE
    if (ntiles > 0) signal(ntiles - 1);
#endif
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (await && threadIdx.x == 0) {  // this CTA's loaders are past their waits
    // the request's last CTA (of 2 * nsplit) to get here resets the counter
    if (atomicAdd(landed + b, LANDED_TAG) >= (2 * nsplit - 1) * LANDED_TAG) atomicExch(landed + b, 0);
  }
  if (warp == MMA_WARP) tmem_dealloc<512>(tmem);
}

// KV-split merge (the reference's merge_attn, costmodel.py:26): per (request, head),
// out = sum_s 2^(m_s - m) O_s / sum_s 2^(m_s - m) l_s with m = max_s m_s (exp2 domain,
// as the kernel's online softmax), lse = (m + log2 l) ln 2.  One warp per head, each
// lane 16 of the 512 output dims.
__global__ void __launch_bounds__(128) mla_combine_kernel(const float *__restrict__ ws_o,
                                                          const float *__restrict__ ws_ml, int nsplit,
                                                          uint16_t *__restrict__ out,
                                                          float *__restrict__ lse) {
  const int b = blockIdx.x, h = blockIdx.y * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  float ms[ESS_MLA_MAX_SPLIT], ls[ESS_MLA_MAX_SPLIT];
  float m = -INFINITY;
#pragma unroll
  for (int s = 0; s < ESS_MLA_MAX_SPLIT; s++) {
    if (s < nsplit) {
      const int64_t r = (int64_t)(b * nsplit + s) * HEADS + h;
      ms[s] = ws_ml[r * 2];
      ls[s] = ws_ml[r * 2 + 1];
      if (ls[s] > 0.f) m = fmaxf(m, ms[s]);
    }
  }
  float l = 0.f, wgt[ESS_MLA_MAX_SPLIT];
#pragma unroll
  for (int s = 0; s < ESS_MLA_MAX_SPLIT; s++) {
    wgt[s] = (s < nsplit && ls[s] > 0.f) ? exp2f(ms[s] - m) : 0.f;
    if (s < nsplit) l += ls[s] * wgt[s];
  }
  const int64_t hrow = (int64_t)b * HEADS + h;
  uint16_t *ob = out + hrow * ESS_MLA_V_DIM + lane * 16;
  if (!(l > 0.f)) {
    reinterpret_cast<uint4 *>(ob)[0] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4 *>(ob)[1] = make_uint4(0, 0, 0, 0);
    if (lane == 0) lse[hrow] = -INFINITY;
    return;
  }
  const float inv = 1.f / l;
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; j++) acc[j] = 0.f;
#pragma unroll
  for (int s = 0; s < ESS_MLA_MAX_SPLIT; s++) {
    if (s >= nsplit || wgt[s] == 0.f) continue;
    const float4 *src = reinterpret_cast<const float4 *>(
        ws_o + ((int64_t)(b * nsplit + s) * HEADS + h) * ESS_MLA_V_DIM + lane * 16);
#pragma unroll
    for (int q4 = 0; q4 < 4; q4++) {
      const float4 x = src[q4];
      acc[4 * q4 + 0] += x.x * wgt[s];
      acc[4 * q4 + 1] += x.y * wgt[s];
      acc[4 * q4 + 2] += x.z * wgt[s];
      acc[4 * q4 + 3] += x.w * wgt[s];
    }
  }
  uint32_t pk[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    __nv_bfloat162 t = __floats2bfloat162_rn(acc[2 * j] * inv, acc[2 * j + 1] * inv);
    pk[j] = *reinterpret_cast<uint32_t *>(&t);
  }
  reinterpret_cast<uint4 *>(ob)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  reinterpret_cast<uint4 *>(ob)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
  if (lane == 0) lse[hrow] = (m + log2f(l)) * 0.6931471805599453f;
}

}  // namespace

int ess_launch_mla_pair(ess_pool *pool, int32_t pool_begin, const void *d_q, const int32_t *d_sel_row,
                        const int32_t *d_sel2, int32_t *d_landed, int32_t sel_stride,
                        const int32_t *d_count, int32_t count_stride, int32_t batch, float sm_scale,
                        void *d_out, float *d_lse, float *d_ws_o, float *d_ws_ml, int32_t flags,
                        int32_t nsplit, void *stream);  // mla2.cu

namespace {

int launch_mla(ess_pool *pool, int32_t pool_begin, const void *d_q, const int32_t *d_sel_row,
               const int32_t *d_sel2, int32_t *d_landed, int32_t sel_stride,
               const int32_t *d_count, int32_t count_stride, int32_t batch, float sm_scale,
               void *d_out, float *d_lse, float *d_ws_o, float *d_ws_ml, int32_t flags,
               int32_t nsplit, void *stream) {
  // raw-row (FP8) slots: the CTA-pair kernel; f16 slots: the CTA pair when ESS_K5_PAIR=1
  static const bool pair_f16 = [] {
    const char *e = getenv("ESS_K5_PAIR");
    return e && e[0] == '1';
  }();
  if (pool->row_bytes == ESS_SLOT_ROW_BYTES_FP8 || pair_f16) {
    int rc = ess_launch_mla_pair(pool, pool_begin, d_q, d_sel_row, d_sel2, d_landed, sel_stride, d_count,
                                count_stride, batch, sm_scale, d_out, d_lse, d_ws_o, d_ws_ml, flags, nsplit,
                                stream);
    if (rc != ESS_OK) return rc;
    if (nsplit > 1) {
      mla_combine_kernel<<<dim3(batch, HEADS / 4), 128, 0, (cudaStream_t)stream>>>(
          d_ws_o, d_ws_ml, nsplit, (uint16_t *)d_out, d_lse);
      ESS_CUDA_TRY(cudaGetLastError());
    }
    return ESS_OK;
  }
  // q as a [batch * 128 heads][576] bf16 tensor, boxes of [128 heads][64 dims], SW128
  struct QMap {
    const void *base = nullptr;
    int32_t batch = 0;
    CUtensorMap map;
  };
  static thread_local QMap qm;
  alignas(64) CUtensorMap tq;
  if (qm.base == d_q && qm.batch == batch) {
    tq = qm.map;
  } else {
    if (!ess_make_tmap_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, d_q, QK_DIM, (uint64_t)batch * HEADS,
                          QK_DIM * 2, 64, HEADS, CU_TENSOR_MAP_SWIZZLE_128B))
      return ESS_ERR_CUDA;
    qm.base = d_q;
    qm.batch = batch;
    qm.map = tq;
  }
  if (int rc = ess_smem_optin((const void *)sparse_mla_kernel, SMEM_BYTES)) return rc;
  dim3 grid(2, batch * nsplit);
  sparse_mla_kernel<<<grid, NTHREADS, SMEM_BYTES, (cudaStream_t)stream>>>(
      tq, pool->rows, pool->rows_per_pool, pool_begin, d_sel_row, d_sel2, d_landed, sel_stride,
      d_count, count_stride, sm_scale, (uint16_t *)d_out, d_lse, d_ws_o, d_ws_ml, flags, nsplit,
      pool->status);
  ESS_CUDA_TRY(cudaGetLastError());
  if (nsplit > 1) {
    mla_combine_kernel<<<dim3(batch, HEADS / 4), 128, 0, (cudaStream_t)stream>>>(
        d_ws_o, d_ws_ml, nsplit, (uint16_t *)d_out, d_lse);
    ESS_CUDA_TRY(cudaGetLastError());
  }
  return ESS_OK;
}

bool pool_ok(ess_pool *pool, int32_t pool_begin, int32_t batch) {
  return pool && pool->rows &&
         (pool->row_bytes == ESS_SLOT_ROW_BYTES || pool->row_bytes == ESS_SLOT_ROW_BYTES_FP8) && batch >= 0 &&
         pool_begin >= 0 && (int64_t)pool_begin + batch <= pool->P;
}

}  // namespace

extern "C" int ess_sparse_mla(ess_pool *pool, int32_t pool_begin, const void *d_q,
                              const int32_t *d_sel_row, int32_t sel_stride, const int32_t *d_count,
                              int32_t count_stride, int32_t batch, float sm_scale, void *d_out,
                              float *d_lse, float *d_ws_o, float *d_ws_ml, int32_t flags,
                              void *stream) {
  const int nsplit = ((flags >> ESS_MLA_SPLIT_SHIFT) & 0xF) + 1;
  const int qtok = ((flags >> ESS_MLA_QTOK_SHIFT) & 7) + 1;
  flags &= ~(0xF << ESS_MLA_SPLIT_SHIFT);
  flags &= ~(7 << ESS_MLA_QTOK_SHIFT);
  if (qtok > ESS_INDEXER_MAX_QTOK || batch % qtok) return ESS_ERR_ARG;
  if (nsplit > ESS_MLA_MAX_SPLIT) return ESS_ERR_ARG;
  if ((flags & (ESS_MLA_PARTIAL | ESS_MLA_RESUME)) && (!d_ws_o || !d_ws_ml)) return ESS_ERR_ARG;
  if ((flags & ESS_MLA_PARTIAL) && (flags & ESS_MLA_RESUME)) return ESS_ERR_ARG;
  if (flags & ~(ESS_MLA_PARTIAL | ESS_MLA_RESUME)) return ESS_ERR_ARG;
  if (nsplit > 1 && (flags || !d_ws_o || !d_ws_ml)) return ESS_ERR_ARG;  // split: full mode only
  if (!pool_ok(pool, pool_begin, batch / qtok) || !d_q || !d_sel_row || !d_count || count_stride < 1 ||
      (!(flags & ESS_MLA_PARTIAL) && (!d_out || !d_lse)) || sel_stride < 1 ||
      (reinterpret_cast<uintptr_t>(d_q) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15))
    return ESS_ERR_ARG;
  if (batch == 0) return ESS_OK;
  return launch_mla(pool, pool_begin, d_q, d_sel_row, nullptr, nullptr, sel_stride, d_count,
                    count_stride, batch, sm_scale, d_out, d_lse, d_ws_o, d_ws_ml,
                    flags | ((qtok - 1) << ESS_MLA_QTOK_SHIFT), nsplit, stream);
}

extern "C" int ess_sparse_mla_da(ess_pool *pool, int32_t pool_begin, const void *d_q,
                                 const int32_t *d_hit_row, const int32_t *d_miss_row,
                                 int32_t row_stride, const int32_t *d_counts, int32_t count_stride,
                                 int32_t *d_landed, int32_t batch, float sm_scale,
                                 void *d_out, float *d_lse, void *stream) {
  return ess_sparse_mla_da_split(pool, pool_begin, d_q, d_hit_row, d_miss_row, row_stride, d_counts,
                                 count_stride, d_landed, batch, sm_scale, d_out, d_lse, nullptr,
                                 nullptr, 1, stream);
}

extern "C" int ess_sparse_mla_da_split(ess_pool *pool, int32_t pool_begin, const void *d_q,
                                       const int32_t *d_hit_row, const int32_t *d_miss_row,
                                       int32_t row_stride, const int32_t *d_counts,
                                       int32_t count_stride, int32_t *d_landed, int32_t batch,
                                       float sm_scale, void *d_out, float *d_lse, float *d_ws_o,
                                       float *d_ws_ml, int32_t nsplit, void *stream) {
  if (!pool_ok(pool, pool_begin, batch) || !d_q || !d_hit_row || !d_miss_row || !d_counts ||
      !d_landed || !d_out || !d_lse || row_stride < 1 || count_stride < 2 ||
      (reinterpret_cast<uintptr_t>(d_q) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15) ||
      nsplit < 1 || nsplit > ESS_MLA_MAX_SPLIT || (nsplit > 1 && (!d_ws_o || !d_ws_ml)))
    return ESS_ERR_ARG;
  if (batch == 0) return ESS_OK;
  // every CTA may spin on the arrival counters: all of them and the gather must fit at once
  if (2 * batch * nsplit > ess_sm_count() - 8) return ESS_ERR_ARG;
  return launch_mla(pool, pool_begin, d_q, d_hit_row, d_miss_row, d_landed, row_stride, d_counts,
                    count_stride, batch, sm_scale, d_out, d_lse, d_ws_o, d_ws_ml, MLA_AWAIT,
                    nsplit, stream);
}

int ess_preload_mla() {  // see ess_preload_indexer
  cudaFuncAttributes a;
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)sparse_mla_kernel));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)mla_combine_kernel));
  return ESS_OK;
}
