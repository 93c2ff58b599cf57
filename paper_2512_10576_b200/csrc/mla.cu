// K5: sparse MLA decode over the selected latent rows (op "sparse_mla",
// costmodel.py:18-27).
//
// out[h] = softmax_j(q[h] . K[j] * sm_scale) V[j], K[j] = dequant(NoPE) ++ RoPE (576),
// V[j] = dequant(NoPE) (512), over the count[b] slot-store rows sel_row[b][:].
//
// TMEM budget drives the split: the fp32 output of 128 heads x 512 dims is 256 KB,
// the whole TMEM of one SM, so each request runs on two CTAs that own 256 output
// dims each and both compute the full score tile S.  Per CTA (512 TMEM columns):
//   O      [0,256)    fp32 accumulator, 128 heads x 256 dims
//   S0/S1  [256,320)  fp32 scores, 32 rows each; P (f16) overwrites the first 16
//                     columns of its S buffer and feeds PV straight from TMEM
//   Qt     [320,512)  q dims 0..383 as f16 pairs: the A operand of S from TMEM
// Shared memory: q dims 384..575 (SW128, 48 KB), a 4-deep ring of raw 656-B rows
// filled by the TMA engine (one cp.async.bulk per row, mbarrier tx-count), a 2-deep
// ring of dequantised f16 KV tiles (SW128, 36 KB each) and the request's slot ids.
//
// Warp roles (448 threads): w0-3 softmax (thread = head; online softmax in exp2
// domain with lazy O rescaling when the running max grows by > 8), w4 TMEM alloc +
// MMA issuer (S = Q K^T: M=128, N=32, 36 x K=16; O += P V: M=128, N=256, V read as
// the MN-major view of the same tile), w5 row gather (bulk copies), w6-13 dequant
// (e4m3 x group scale -> f16, RoPE bf16 -> f16, smem -> smem).
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
constexpr int ROW = ESS_LATENT_ROW_BYTES;          // 656
constexpr int RAW_BYTES = NB * ROW;                // 20992
constexpr int KS = 2, RS = 4;                      // ring depths
constexpr int MAX_N = ESS_MAX_REQUEST;
constexpr int NSOFT = 4, NDEQ = 8;
constexpr int MMA_WARP = NSOFT, GATHER_WARP = NSOFT + 1, DEQ0 = NSOFT + 2;
constexpr int NTHREADS = 32 * (NSOFT + 2 + NDEQ);  // 448
constexpr uint32_t TM_O = 0, TM_S = 256, TM_Q = 320;
constexpr float RESCALE_THRESHOLD = 8.0f;
constexpr uint32_t IDESC_S = make_idesc(0 /*f16*/, 0 /*f16*/, HEADS, NB, 0, 0);
constexpr uint32_t IDESC_PV = make_idesc(0, 0, HEADS, V_HALF, 0, 1 /*B MN-major*/);

struct Ctrl {
  uint64_t raw_full[RS], raw_empty[RS], kv_full[KS], kv_empty[KS];
  uint64_t s_full[2], s_free[2], p_full, p_empty, o_done;
  uint32_t tmem;
};
constexpr size_t SMEM_BYTES =
    1024 + QS_BYTES + KS * KV_BYTES + RS * RAW_BYTES + MAX_N * 4 + sizeof(Ctrl);

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

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

__device__ __forceinline__ uint32_t cvt_e4m3x2_f16x2(uint16_t v) {
  uint32_t r;
  asm("{\n\t.reg .b16 t;\n\tmov.b16 t, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, t;\n\t}" : "=r"(r) : "h"(v));
  return r;
}

__device__ __forceinline__ uint32_t hmul2_u32(uint32_t a, __half2 s) {
  __half2 x = *reinterpret_cast<__half2 *>(&a);
  x = __hmul2(x, s);
  return *reinterpret_cast<uint32_t *>(&x);
}

__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t v) {
  float lo = __uint_as_float(v << 16), hi = __uint_as_float(v & 0xFFFF0000u);
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ uint4 cvt8_bf16_f16(uint4 x) {
  return make_uint4(bf16x2_to_f16x2(x.x), bf16x2_to_f16x2(x.y), bf16x2_to_f16x2(x.z),
                    bf16x2_to_f16x2(x.w));
}

__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_mla_kernel(const uint16_t *__restrict__ q, const uint8_t *__restrict__ rows,
                      int64_t rows_per_pool, int pool_begin, const int32_t *__restrict__ sel_row,
                      int sel_stride, const int32_t *__restrict__ counts, float sm_scale,
                      uint16_t *__restrict__ out, float *__restrict__ lse) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sq = smem;                        // q dims 384..575, 3 SW128 blocks
  uint8_t *skv = sq + QS_BYTES;              // KS dequantised tiles
  uint8_t *sraw = skv + KS * KV_BYTES;       // RS raw row tiles
  int32_t *ssel = reinterpret_cast<int32_t *>(sraw + RS * RAW_BYTES);
  Ctrl &c = *reinterpret_cast<Ctrl *>(ssel + MAX_N);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v = blockIdx.x;  // output half
  const int b = blockIdx.y;
  const int n = min(counts[b], MAX_N);
  const int ntiles = (n + NB - 1) / NB;
  const uint16_t *qb = q + (int64_t)b * HEADS * QK_DIM;

  if (threadIdx.x == 0) {
    for (int i = 0; i < RS; i++) {
      mbar_init(&c.raw_full[i], 1);
      mbar_init(&c.raw_empty[i], NDEQ);
    }
    for (int i = 0; i < KS; i++) {
      mbar_init(&c.kv_full[i], NDEQ);
      mbar_init(&c.kv_empty[i], 1);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(&c.s_full[i], 1);
      mbar_init(&c.s_free[i], 1);
    }
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
  } else if (warp == GATHER_WARP) {
    const int32_t *sel = sel_row + (int64_t)b * sel_stride;
    for (int j = lane; j < n; j += 32) ssel[j] = __ldg(sel + j);
  } else if (warp >= DEQ0) {
    const int gt = threadIdx.x - DEQ0 * 32;
    for (int it = gt; it < HEADS * QS_BLKS * 8; it += NDEQ * 32) {
      const int h = it / (QS_BLKS * 8), ch = it % (QS_BLKS * 8);  // 8-element chunk of dims 384..
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
    float m_run = -INFINITY, l_run = 0.f;
    for (int i = 0; i < ntiles; i++) {
      const int sb = i & 1;
      mbar_wait(&c.s_full[sb], (i >> 1) & 1);
      tc_fence_after();
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
      // PV(i-1) must be done before O is rescaled
      mbar_wait(&c.p_empty, (i & 1) ^ 1);
      tc_fence_after();
      // warp-uniform decision (tcgen05.ld/st are .sync.aligned); a lane whose own
      // max did not grow rescales by alpha = 1
      if (__any_sync(0xffffffffu, mt > m_run + RESCALE_THRESHOLD) || i == 0) {
        const float m_new = fmaxf(mt, m_run);
        const float alpha = exp2f(m_run - m_new);  // 0 when m_run = -inf
        l_run *= alpha;
        if (i > 0) {
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
    // ---------------- final normalisation ---------------------------------------
    uint16_t *ob = out + ((int64_t)b * HEADS + h) * ESS_MLA_V_DIM + v * V_HALF;
    if (ntiles > 0) {
      mbar_wait(&c.o_done, 0);
      tc_fence_after();
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
      if (v == 0) lse[(int64_t)b * HEADS + h] = (m_run + log2f(l_run)) * 0.6931471805599453f;
    } else {
      for (int j = 0; j < V_HALF; j += 8) *reinterpret_cast<uint4 *>(ob + j) = make_uint4(0, 0, 0, 0);
      if (v == 0) lse[(int64_t)b * HEADS + h] = -INFINITY;
    }
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer --------------------------------------------------
    if (elect_one() && ntiles > 0) {
      const uint32_t qsaddr = smem_u32(sq);
      auto issue_s = [&](int i) {
        const int kb = i % KS, sb = i & 1;
        mbar_wait(&c.kv_full[kb], (i / KS) & 1);
        mbar_wait(&c.s_free[sb], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t kvaddr = smem_u32(skv + kb * KV_BYTES);
        const uint32_t d = tmem + TM_S + sb * NB;
#pragma unroll 1
        for (int blk = 0; blk < QT_BLKS; blk++) {
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            uint64_t bd = sw128_desc(kvaddr + blk * KV_BLK_BYTES + kk * 32, 16, 1024);
            mma_f16_ts(d, tmem + TM_Q + (blk * 4 + kk) * 8, bd, IDESC_S, (blk | kk) ? 1u : 0u);
          }
        }
#pragma unroll 1
        for (int blk = QT_BLKS; blk < NBLK; blk++) {
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            uint64_t ad = sw128_desc(qsaddr + (blk - QT_BLKS) * (HEADS * 128) + kk * 32, 16, 1024);
            uint64_t bd = sw128_desc(kvaddr + blk * KV_BLK_BYTES + kk * 32, 16, 1024);
            mma_f16_ss(d, ad, bd, IDESC_S, 1u);
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
          mma_f16_ts(tmem + TM_O, tmem + TM_S + sb * NB + kk * 8, bd, IDESC_PV, (i | kk) ? 1u : 0u);
        }
        tc_commit(&c.p_empty);
        tc_commit(&c.kv_empty[kb]);
        tc_commit(&c.s_free[sb]);
        if (i == ntiles - 1) tc_commit(&c.o_done);
      }
    }
  } else if (warp == GATHER_WARP) {
    // ---------------- row gather: one bulk copy (TMA engine) per selected row ----
    const uint8_t *pool_rows = rows + (int64_t)(pool_begin + b) * rows_per_pool * ROW;
    for (int i = 0; i < ntiles; i++) {
      const int rs = i % RS;
      const int nvalid = min(NB, n - i * NB);
      mbar_wait(&c.raw_empty[rs], ((i / RS) & 1) ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&c.raw_full[rs], (uint32_t)(nvalid * ROW));
      __syncwarp();
      if (lane < nvalid)
        bulk_load(sraw + rs * RAW_BYTES + lane * ROW, pool_rows + (int64_t)ssel[i * NB + lane] * ROW,
                  ROW, &c.raw_full[rs]);
    }
  } else {
    // ---------------- dequant warps: raw rows -> f16 SW128 KV tile ----------------
    const int gt = threadIdx.x - DEQ0 * 32;  // 0..255
    for (int i = 0; i < ntiles; i++) {
      const int rs = i % RS, kb = i % KS;
      mbar_wait(&c.raw_full[rs], (i / RS) & 1);
      mbar_wait(&c.kv_empty[kb], ((i / KS) & 1) ^ 1);
      const uint8_t *raw = sraw + rs * RAW_BYTES;
      uint8_t *kv = skv + kb * KV_BYTES;
      // NoPE: 32 rows x 32 chunks of 16 e4m3 -> 2 x 16 B of f16
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int item = gt + 256 * k;
        const int r = item >> 5, ch = item & 31;
        uint4 y0 = make_uint4(0, 0, 0, 0), y1 = y0;
        if (i * NB + r < n) {
          const uint8_t *src = raw + r * ROW;
          const uint4 x = *reinterpret_cast<const uint4 *>(src + ch * 16);
          const __half2 s2 = __float2half2_rn(*reinterpret_cast<const float *>(src + 512 + 4 * (ch >> 3)));
          y0.x = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.x & 0xFFFF)), s2);
          y0.y = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.x >> 16)), s2);
          y0.z = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.y & 0xFFFF)), s2);
          y0.w = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.y >> 16)), s2);
          y1.x = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.z & 0xFFFF)), s2);
          y1.y = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.z >> 16)), s2);
          y1.z = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.w & 0xFFFF)), s2);
          y1.w = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.w >> 16)), s2);
        }
        // dims [16ch, 16ch+16): block ch/4, 16-B chunks 2(ch%4) and 2(ch%4)+1
        const int blk = ch >> 2, c0 = (ch & 3) * 2;
        uint8_t *base = kv + blk * KV_BLK_BYTES;
        *reinterpret_cast<uint4 *>(base + sw128((uint32_t)r * 128 + c0 * 16)) = y0;
        *reinterpret_cast<uint4 *>(base + sw128((uint32_t)r * 128 + (c0 + 1) * 16)) = y1;
      }
      // RoPE: 32 rows x 8 chunks of 8 bf16 -> 8 f16 (dim-block 8)
      {
        const int r = gt >> 3, ch = gt & 7;
        uint4 y = make_uint4(0, 0, 0, 0);
        if (i * NB + r < n) y = cvt8_bf16_f16(*reinterpret_cast<const uint4 *>(raw + r * ROW + 528 + ch * 16));
        *reinterpret_cast<uint4 *>(kv + 8 * KV_BLK_BYTES + sw128((uint32_t)r * 128 + ch * 16)) = y;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&c.raw_empty[rs]);
        mbar_arrive(&c.kv_full[kb]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == MMA_WARP) tmem_dealloc<512>(tmem);
}

}  // namespace

extern "C" int ess_sparse_mla(ess_pool *pool, int32_t pool_begin, const void *d_q,
                              const int32_t *d_sel_row, int32_t sel_stride, const int32_t *d_count,
                              int32_t batch, float sm_scale, void *d_out, float *d_lse,
                              void *stream) {
  if (!pool || !pool->rows || pool->row_bytes != ROW || !d_q || !d_sel_row || !d_count ||
      !d_out || !d_lse || batch < 0 || pool_begin < 0 || (int64_t)pool_begin + batch > pool->P ||
      sel_stride < 1 || (reinterpret_cast<uintptr_t>(d_q) & 15) ||
      (reinterpret_cast<uintptr_t>(d_out) & 15))
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
      (const uint16_t *)d_q, pool->rows, pool->rows_per_pool, pool_begin, d_sel_row, sel_stride,
      d_count, sm_scale, (uint16_t *)d_out, d_lse);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}
