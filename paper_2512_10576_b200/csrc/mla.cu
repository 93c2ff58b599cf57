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
//   S0/S1  [256,320)  fp32 scores, 32 rows each; P (f16) overwrites the first 16
//                     columns of its S buffer and feeds PV straight from TMEM
//   Qt     [320,512)  q dims 0..383 as f16 pairs: the A operand of S from TMEM
// Shared memory: q dims 384..575 (SW128 K-major, 48 KB), a 4-deep ring of KV tiles
// (32 rows x 576 f16, SW128: 9 blocks of [32 rows][64 dims]) filled by 16-B
// cp.async straight into the swizzled positions (TMA tile::gather4 moves only
// 4 x 128 B per instruction and was instruction-rate bound here), and the
// request's slot ids.
//
// Warp roles (288 threads): w0-3 softmax (thread = head; online softmax in exp2
// domain with lazy O rescaling when the running max grows by > 8), w4 TMEM alloc +
// MMA issuer (S = Q K^T: M=128, N=32, 36 x K=16; O += P V: M=128, N=256, V read as
// the MN-major view of the same tile), w5-8 row loaders.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int HEADS = ESS_MLA_HEADS;      // 128 = M
constexpr int QK_DIM = ESS_MLA_QK_DIM;    // 576
constexpr int V_HALF = 256;               // output dims per CTA
constexpr int NB = 32;                    // KV rows per tile
constexpr int NBLK = QK_DIM / 64;         // 9 dim-blocks of 64 (128 B of f16)
constexpr int QT_BLKS = 6;                // q blocks held in TMEM (dims 0..383)
constexpr int QS_BLKS = NBLK - QT_BLKS;   // q blocks in shared memory (dims 384..575)
constexpr int QS_BYTES = QS_BLKS * HEADS * 128;    // 49152
constexpr int KV_BLK_BYTES = NB * 128;             // 4096
constexpr int KV_BYTES = NBLK * KV_BLK_BYTES;      // 36864
constexpr int KS = 4;                              // KV ring depth
#ifndef ESS_MLA_LOAD_LAG
#define ESS_MLA_LOAD_LAG 1
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
constexpr int LOAD_LAG = ESS_MLA_LOAD_LAG;         // tiles in flight per loader beyond the newest
// the MMA warp issues S(i+1) before PV(i) frees slot i, so a loader may run at most
// KS - 2 tiles ahead of its newest complete tile
static_assert(LOAD_LAG >= 1 && LOAD_LAG <= KS - 2, "loader lag must leave the MMA a lookahead slot");
constexpr int MAX_N = ESS_MAX_REQUEST;
constexpr int NSOFT = 4, NLOAD = 4;
constexpr int MMA_WARP = NSOFT, LOAD0 = NSOFT + 1;
constexpr int NTHREADS = 32 * (NSOFT + 1 + NLOAD);  // 288
constexpr int ROWS_PER_LOADER = NB / NLOAD;         // 8
constexpr int SLOT_CHUNKS = ESS_SLOT_ROW_BYTES / 16; // 72
constexpr uint32_t TM_O = 0, TM_S = 256, TM_Q = 320;
constexpr float RESCALE_THRESHOLD = 8.0f;
#ifndef ESS_MLA_DBG_SN
#define ESS_MLA_DBG_SN NB
#endif
constexpr uint32_t IDESC_S = make_idesc(0 /*f16*/, 0 /*f16*/, HEADS, ESS_MLA_DBG_SN, 0, 0);
constexpr uint32_t IDESC_PV = make_idesc(0, 0, HEADS, V_HALF, 0, 1 /*B MN-major*/);

struct Ctrl {
  uint64_t kv_full[KS], kv_empty[KS];
  uint64_t s_full[2], p_full, p_empty, o_done;
  uint32_t tmem;
};
constexpr size_t SMEM_BYTES = 1024 + QS_BYTES + KS * KV_BYTES + MAX_N * 4 + sizeof(Ctrl);

__device__ __forceinline__ uint32_t sw128(uint32_t o) { return o ^ (((o >> 7) & 7u) << 4); }

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

// 16-B async global -> shared copy (L1 bypass); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

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
    sparse_mla_kernel(const uint8_t *__restrict__ rows, const uint16_t *__restrict__ q,
                      int64_t rows_per_pool, int pool_begin, const int32_t *__restrict__ sel_row,
                      int sel_stride, const int32_t *__restrict__ counts, int count_stride,
                      float sm_scale, uint16_t *__restrict__ out, float *__restrict__ lse,
                      float *__restrict__ ws_o, float *__restrict__ ws_ml, int flags) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sq = smem;                        // q dims 384..575, 3 SW128 blocks
  uint8_t *skv = sq + QS_BYTES;              // KS f16 KV tiles
  int32_t *ssel = reinterpret_cast<int32_t *>(skv + KS * KV_BYTES);
  Ctrl &c = *reinterpret_cast<Ctrl *>(ssel + MAX_N);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v = blockIdx.x;  // output half
  const int b = blockIdx.y;
  const int n = min(counts[(int64_t)b * count_stride], MAX_N);
  const bool partial = flags & ESS_MLA_PARTIAL, resume = flags & ESS_MLA_RESUME;
  const int ntiles = (n + NB - 1) / NB;
  const uint16_t *qb = q + (int64_t)b * HEADS * QK_DIM;

  if (threadIdx.x == 0) {
    for (int i = 0; i < KS; i++) {
      mbar_init(&c.kv_full[i], NLOAD);
      mbar_init(&c.kv_empty[i], 1);
    }
    for (int i = 0; i < 2; i++) mbar_init(&c.s_full[i], 1);
    mbar_init(&c.p_full, NSOFT);
    mbar_init(&c.p_empty, 1);
    mbar_init(&c.o_done, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc<512>(&c.tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = c.tmem;

  // ---- prologue: q -> TMEM (dims 0..383) and smem (384..575); slot ids -> smem ----
  if (warp < NSOFT) {
    const int h = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint4 *src = reinterpret_cast<const uint4 *>(qb + (int64_t)h * QK_DIM);
#pragma unroll 1
    for (int cc = 0; cc < QT_BLKS; cc++) {  // 64 dims = 32 columns per chunk
      uint32_t r[32];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        uint4 y = cvt8_bf16_f16(__ldg(src + cc * 8 + k));
        r[4 * k] = y.x;
        r[4 * k + 1] = y.y;
        r[4 * k + 2] = y.z;
        r[4 * k + 3] = y.w;
      }
      tmem_st_32x32b_x32(tmem + lane_base + TM_Q + cc * 32, r);
    }
    tmem_st_wait();
  } else {
    // warps 4-8: slot ids, then q dims 384..575 into SW128 smem
    constexpr int NT = NTHREADS - NSOFT * 32;
    const int t = threadIdx.x - NSOFT * 32;
    const int32_t *sel = sel_row + (int64_t)b * sel_stride;
    for (int j = t; j < n; j += NT) ssel[j] = __ldg(sel + j);
    for (int it = t; it < HEADS * QS_BLKS * 8; it += NT) {
      const int h = it / (QS_BLKS * 8), ch = it % (QS_BLKS * 8);  // 8-element chunk
      uint4 y = cvt8_bf16_f16(__ldg(reinterpret_cast<const uint4 *>(qb + (int64_t)h * QK_DIM + 384) + ch));
      *reinterpret_cast<uint4 *>(sq + (ch >> 3) * (HEADS * 128) + sw128((uint32_t)h * 128 + (ch & 7) * 16)) = y;
    }
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
    float *wso = ws_o ? ws_o + hrow * ESS_MLA_V_DIM + v * V_HALF : nullptr;
    float m_run = -INFINITY, l_run = 0.f;
    if (resume) {  // continue from pass 1: running max / sum and this CTA's O half
      m_run = ws_ml[hrow * 2 + 0];
      l_run = ws_ml[hrow * 2 + 1];
#pragma unroll 1
      for (int cc = 0; cc < V_HALF / 32; cc++) {
        uint32_t o[32];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 f = *reinterpret_cast<const float4 *>(wso + cc * 32 + j);
          o[j] = __float_as_uint(f.x);
          o[j + 1] = __float_as_uint(f.y);
          o[j + 2] = __float_as_uint(f.z);
          o[j + 3] = __float_as_uint(f.w);
        }
        tmem_st_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
      }
      tmem_st_wait();
    }
    for (int i = 0; i < ntiles; i++) {
      const int sb = i & 1;
      mbar_wait(&c.s_full[sb], (i >> 1) & 1);
      tc_fence_after();
#if ESS_MLA_DBG_NOSOFT
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.p_full);
      continue;
#endif
      uint32_t s[32];
      tmem_ld_32x32b_x32(tmem + lane_base + TM_S + sb * NB, s);
      tmem_ld_wait();
      float x[32];
      float mt = -INFINITY;
#pragma unroll
      for (int j = 0; j < NB; j++) {
        x[j] = (i * NB + j < n) ? __uint_as_float(s[j]) * scale_log2 : -INFINITY;
        mt = fmaxf(mt, x[j]);
      }
      // warp-uniform decision (tcgen05.ld/st are .sync.aligned); a lane whose own
      // max did not grow rescales by alpha = 1
      if (__any_sync(0xffffffffu, mt > m_run + RESCALE_THRESHOLD) || (i == 0 && !resume)) {
        const float m_new = fmaxf(mt, m_run);
        const float alpha = exp2f(m_run - m_new);  // 0 when m_run = -inf
        l_run *= alpha;
        // PV(i-1) accumulates into O: wait for it before O is rescaled.  Only rescale
        // tiles wait, keeping the MMA round trip off the per-tile path.  The parity
        // is unambiguous: the s_full(i) commit tracks every earlier MMA, PV(i-2)
        // included, and PV(i) needs this tile's P, so p_empty has completed phase
        // i-2 and not phase i.
        if (i > 0) {
          mbar_wait(&c.p_empty, (i & 1) ^ 1);
          tc_fence_after();
        }
        if (i > 0 || resume) {  // O holds PV(i-1) or the resumed state
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
      // P (f16 pairs) over the first 16 columns of this S buffer
      uint32_t p[16];
      float lsum = 0.f;
#pragma unroll
      for (int e = 0; e < 16; e++) {
        __half2 p2 = __floats2half2_rn(exp2f(x[2 * e] - m_run), exp2f(x[2 * e + 1] - m_run));
        float2 f = __half22float2(p2);
        lsum += f.x + f.y;
        p[e] = *reinterpret_cast<uint32_t *>(&p2);
      }
      l_run += lsum;
      tmem_st_32x32b_x16(tmem + lane_base + TM_S + sb * NB, p);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.p_full);
    }
    // ---------------- epilogue ---------------------------------------------------
    const bool have_o = ntiles > 0 || resume;  // TMEM O holds a valid accumulator
    if (ntiles > 0) {
      mbar_wait(&c.o_done, 0);
      tc_fence_after();
    }
    if (partial) {
      // pass 1 of the split attention: unnormalised O and (max, sum) to the workspace
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
        ws_ml[hrow * 2 + 0] = m_run;
        ws_ml[hrow * 2 + 1] = l_run;
      }
    } else {
      uint16_t *ob = out + hrow * ESS_MLA_V_DIM + v * V_HALF;
      if (have_o && l_run > 0.f) {
        const float inv = 1.f / l_run;
#pragma unroll 1
        for (int cc = 0; cc < V_HALF / 32; cc++) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(tmem + lane_base + TM_O + cc * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 pk;
            __nv_bfloat162 t0 = __floats2bfloat162_rn(__uint_as_float(o[j]) * inv, __uint_as_float(o[j + 1]) * inv);
            __nv_bfloat162 t1 = __floats2bfloat162_rn(__uint_as_float(o[j + 2]) * inv, __uint_as_float(o[j + 3]) * inv);
            __nv_bfloat162 t2 = __floats2bfloat162_rn(__uint_as_float(o[j + 4]) * inv, __uint_as_float(o[j + 5]) * inv);
            __nv_bfloat162 t3 = __floats2bfloat162_rn(__uint_as_float(o[j + 6]) * inv, __uint_as_float(o[j + 7]) * inv);
            pk.x = *reinterpret_cast<uint32_t *>(&t0);
            pk.y = *reinterpret_cast<uint32_t *>(&t1);
            pk.z = *reinterpret_cast<uint32_t *>(&t2);
            pk.w = *reinterpret_cast<uint32_t *>(&t3);
            *reinterpret_cast<uint4 *>(ob + cc * 32 + j) = pk;
          }
        }
        if (v == 0) lse[hrow] = (m_run + log2f(l_run)) * 0.6931471805599453f;
      } else {
        for (int j = 0; j < V_HALF; j += 8) *reinterpret_cast<uint4 *>(ob + j) = make_uint4(0, 0, 0, 0);
        if (v == 0) lse[hrow] = -INFINITY;
      }
    }
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer --------------------------------------------------
    if (elect_one() && ntiles > 0) {
      const uint32_t qsaddr = smem_u32(sq);
      auto issue_s = [&](int i) {
        const int kb = i % KS, sb = i & 1;
        // S(i) overwrites S/P buffer sb, last read by PV(i-2) as its A operand.  No
        // wait: softmax(i-2) finished with the buffer before p_full(i-2), PV(i-2) was
        // issued before this S(i), and one thread's tcgen05.mma ops execute in issue
        // order — waiting for PV(i-2) to complete would idle the tensor pipe each tile.
        mbar_wait(&c.kv_full[kb], (i / KS) & 1);
        tc_fence_after();
        const uint32_t kvaddr = smem_u32(skv + kb * KV_BYTES);
        const uint32_t d = tmem + TM_S + sb * NB;
#pragma unroll 1
        for (int blk = 0; blk < QT_BLKS; blk++) {
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            uint64_t bd = sw128_desc(kvaddr + blk * KV_BLK_BYTES + kk * 32, 16, 1024);
#if ESS_MLA_DBG_ALLSS
            mma_f16_ss(d, sw128_desc(qsaddr + (blk % QS_BLKS) * (HEADS * 128) + kk * 32, 16, 1024), bd,
                       IDESC_S, (blk | kk) ? 1u : 0u);
#else
            if (!ESS_MLA_DBG_NOMMA)
              mma_f16_ts(d, tmem + TM_Q + (blk * 4 + kk) * 8, bd, IDESC_S, (blk | kk) ? 1u : 0u);
#endif
          }
        }
#pragma unroll 1
        for (int blk = QT_BLKS; blk < NBLK; blk++) {
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            uint64_t ad = sw128_desc(qsaddr + (blk - QT_BLKS) * (HEADS * 128) + kk * 32, 16, 1024);
            uint64_t bd = sw128_desc(kvaddr + blk * KV_BLK_BYTES + kk * 32, 16, 1024);
            if (!ESS_MLA_DBG_NOMMA) mma_f16_ss(d, ad, bd, IDESC_S, 1u);
          }
        }
        tc_commit(&c.s_full[sb]);
      };
      issue_s(0);
      for (int i = 0; i < ntiles; i++) {
        if (i + 1 < ntiles) issue_s(i + 1);
        const int kb = i % KS, sb = i & 1;
        mbar_wait(&c.p_full, i & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_u32(skv + kb * KV_BYTES) + (uint32_t)(4 * v) * KV_BLK_BYTES;
#pragma unroll
        for (int kk = 0; kk < NB / 16; kk++) {
          uint64_t bd = sw128_desc(vaddr + kk * 16 * 128, KV_BLK_BYTES, 1024);
          if (!ESS_MLA_DBG_NOMMA)
            mma_f16_ts(tmem + TM_O, tmem + TM_S + sb * NB + kk * 8, bd, IDESC_PV,
                       (i | kk) || resume ? 1u : 0u);
        }
        tc_commit(&c.p_empty);
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
    const uint8_t *pool_rows = rows + (int64_t)(pool_begin + b) * rows_per_pool * ESS_SLOT_ROW_BYTES;
    const uint32_t kv0 = smem_u32(skv);
    auto signal = [&](int i) {
      fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.kv_full[i % KS]);
    };
    for (int i = 0; i < ntiles; i++) {
      const int kb = i % KS;
      mbar_wait(&c.kv_empty[kb], ((i / KS) & 1) ^ 1);
      const uint32_t kv = kv0 + kb * KV_BYTES;
#pragma unroll
      for (int rr = 0; rr < ROWS_PER_LOADER; rr++) {
        const int r = w * ROWS_PER_LOADER + rr;
        const int j = i * NB + r;
        const bool ok = j < n;
        const uint8_t *src = pool_rows + (int64_t)ssel[ok ? j : 0] * ESS_SLOT_ROW_BYTES;
#pragma unroll
        for (int k = 0; k < 3; k++) {
          const int ch = lane + 32 * k;
          if (ch < SLOT_CHUNKS && !ESS_MLA_DBG_NOLOAD)
            cp_async16(kv + (ch >> 3) * KV_BLK_BYTES + r * 128 + (((ch & 7) ^ (r & 7)) << 4),
                       src + ch * 16, ok ? 16u : 0u);
        }
      }
      cp_async_commit();
      if (i >= LOAD_LAG) {
        cp_async_wait<LOAD_LAG>();
        signal(i - LOAD_LAG);
      }
    }
    cp_async_wait<0>();
    for (int i = max(0, ntiles - LOAD_LAG); i < ntiles; i++) signal(i);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == MMA_WARP) tmem_dealloc<512>(tmem);
}

}  // namespace

extern "C" int ess_sparse_mla(ess_pool *pool, int32_t pool_begin, const void *d_q,
                              const int32_t *d_sel_row, int32_t sel_stride, const int32_t *d_count,
                              int32_t count_stride, int32_t batch, float sm_scale, void *d_out,
                              float *d_lse, float *d_ws_o, float *d_ws_ml, int32_t flags,
                              void *stream) {
  if ((flags & (ESS_MLA_PARTIAL | ESS_MLA_RESUME)) && (!d_ws_o || !d_ws_ml)) return ESS_ERR_ARG;
  if ((flags & ESS_MLA_PARTIAL) && (flags & ESS_MLA_RESUME)) return ESS_ERR_ARG;
  if (!pool || !pool->rows || pool->row_bytes != ESS_SLOT_ROW_BYTES || !d_q || !d_sel_row ||
      !d_count || count_stride < 1 || (!(flags & ESS_MLA_PARTIAL) && (!d_out || !d_lse)) ||
      batch < 0 || pool_begin < 0 ||
      (int64_t)pool_begin + batch > pool->P || sel_stride < 1 ||
      (reinterpret_cast<uintptr_t>(d_q) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15))
    return ESS_ERR_ARG;
  if (batch == 0) return ESS_OK;
  static bool attr = false;
  if (!attr) {
    ESS_CUDA_TRY(cudaFuncSetAttribute(sparse_mla_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)SMEM_BYTES));
    attr = true;
  }
  dim3 grid(2, batch);
  sparse_mla_kernel<<<grid, NTHREADS, SMEM_BYTES, (cudaStream_t)stream>>>(
      pool->rows, (const uint16_t *)d_q, pool->rows_per_pool, pool_begin, d_sel_row,
      sel_stride, d_count, count_stride, sm_scale, (uint16_t *)d_out, d_lse, d_ws_o, d_ws_ml,
      flags);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}
