// K5: sparse MLA decode over the selected latent rows (op "sparse_mla",
// costmodel.py:18-27).
//
// out[h] = softmax_j(q[h] . K[j] * sm_scale) V[j], K[j] = dequant(NoPE) ++ RoPE (576),
// V[j] = dequant(NoPE) (512), over the count[b] slot-store rows sel_row[b][:].
//
// TMEM budget drives the split: the fp32 output of 128 heads x 512 dims is 256 KB,
// the whole TMEM of one SM, so each request runs on two CTAs that own 256 output
// dims each (O = 256 columns) and both compute the full score tile S (32 columns,
// double-buffered).  Per CTA:
//   * Q (bf16 -> f16) resident in shared memory, SW128 K-major, 144 KB;
//   * 8 "gather" warps pull the 656-B rows by slot index (16-B loads), dequantise
//     e4m3 x group-scale -> f16 and RoPE bf16 -> f16 straight into the SW128 KV
//     tile (32 rows x 576, double-buffered) — the TMA-gather role, done with LSU
//     loads because every row also needs a dequant pass before the tensor core;
//   * 1 MMA thread: S = Q K^T (M=128, N=32, 36 x K=16) then O += P V
//     (M=128, N=256, V as the MN-major view of the same tile);
//   * 4 softmax warps (one head per TMEM lane): online softmax in exp2 domain with
//     lazy O rescaling (only when the running max grows by > 8), P -> f16 (SW64).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int HEADS = ESS_MLA_HEADS;      // 128 = M
constexpr int QK_DIM = ESS_MLA_QK_DIM;    // 576
constexpr int V_HALF = 256;               // output dims per CTA
constexpr int NB = 32;                    // KV rows per tile
constexpr int NBLK = QK_DIM / 64;         // 9 dim-blocks of 64 (128 B of f16)
constexpr int Q_BYTES = HEADS * QK_DIM * 2;        // 147456
constexpr int KV_BLK_BYTES = NB * 128;             // 4096
constexpr int KV_BYTES = NBLK * KV_BLK_BYTES;      // 36864
constexpr int P_BYTES = HEADS * NB * 2;            // 8192
constexpr int NSOFT = 4, NMMA = 1, NGATHER = 8;
constexpr int NTHREADS = 32 * (NSOFT + NMMA + NGATHER);  // 416
constexpr int MMA_WARP = NSOFT;
constexpr int G0 = NSOFT + NMMA;  // first gather warp
constexpr int ROW = ESS_LATENT_ROW_BYTES;
constexpr uint32_t TM_O = 0, TM_S = 256;  // TMEM column bases
constexpr float RESCALE_THRESHOLD = 8.0f;
constexpr uint32_t IDESC_S = make_idesc(0 /*f16*/, 0 /*f16*/, HEADS, NB, 0, 0);
constexpr uint32_t IDESC_PV = make_idesc(0, 0, HEADS, V_HALF, 0, 1 /*B MN-major*/);

struct Ctrl {
  uint64_t kv_full[2], kv_empty[2], s_full[2], s_empty[2], p_full, p_empty, o_done;
  uint32_t tmem;
};
constexpr size_t SMEM_BYTES = 1024 + Q_BYTES + 2 * KV_BYTES + P_BYTES + sizeof(Ctrl);

__device__ __forceinline__ uint32_t sw128(uint32_t o) { return o ^ (((o >> 7) & 7u) << 4); }
__device__ __forceinline__ uint32_t sw64(uint32_t o) { return o ^ (((o >> 7) & 3u) << 4); }

__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;  // LBO 16 B (unused for swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_mla_kernel(const uint16_t *__restrict__ q, const uint8_t *__restrict__ rows,
                      int64_t rows_per_pool, int pool_begin, const int32_t *__restrict__ sel_row,
                      int sel_stride, const int32_t *__restrict__ counts, float sm_scale,
                      uint16_t *__restrict__ out, float *__restrict__ lse) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sq = smem;
  uint8_t *skv = smem + Q_BYTES;
  uint8_t *sp = skv + 2 * KV_BYTES;
  Ctrl &c = *reinterpret_cast<Ctrl *>(sp + P_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v = blockIdx.x;  // output half
  const int b = blockIdx.y;
  const int n = counts[b];
  const int ntiles = (n + NB - 1) / NB;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      mbar_init(&c.kv_full[i], NGATHER);
      mbar_init(&c.kv_empty[i], 1);
      mbar_init(&c.s_full[i], 1);
      mbar_init(&c.s_empty[i], NSOFT);
    }
    mbar_init(&c.p_full, NSOFT);
    mbar_init(&c.p_empty, 1);
    mbar_init(&c.o_done, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc<512>(&c.tmem);
  // Q: bf16 -> f16, SW128 K-major, 9 blocks of [128 heads][64 dims]
  {
    const uint4 *qg = reinterpret_cast<const uint4 *>(q + (int64_t)b * HEADS * QK_DIM);
    for (int it = threadIdx.x; it < HEADS * QK_DIM / 8; it += NTHREADS) {
      const int h = it / (QK_DIM / 8), ch = it % (QK_DIM / 8);  // ch: 8-element chunk
      uint4 x = __ldg(qg + it);
      uint4 y;
      y.x = bf16x2_to_f16x2(x.x);
      y.y = bf16x2_to_f16x2(x.y);
      y.z = bf16x2_to_f16x2(x.z);
      y.w = bf16x2_to_f16x2(x.w);
      const uint32_t o = (uint32_t)(ch >> 3) * (HEADS * 128) + sw128((uint32_t)h * 128 + (ch & 7) * 16);
      *reinterpret_cast<uint4 *>(sq + o) = y;
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = c.tmem;
  const float scale_log2 = sm_scale * 1.4426950408889634f;

  if (warp < NSOFT) {
    // ---------------- softmax / epilogue warps: thread = head --------------------
    const int h = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    for (int i = 0; i < ntiles; i++) {
      const int kb = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      mbar_wait(&c.s_full[kb], ph);
      tc_fence_after();
      uint32_t s[32];
      tmem_ld_32x32b_x32(tmem + lane_base + TM_S + kb * NB, s);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.s_empty[kb]);
      float x[32];
      float mt = -INFINITY;
#pragma unroll
      for (int j = 0; j < NB; j++) {
        x[j] = (i * NB + j < n) ? __uint_as_float(s[j]) * scale_log2 : -INFINITY;
        mt = fmaxf(mt, x[j]);
      }
      // PV(i-1) must be done before P is overwritten or O rescaled
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
          tmem_st_wait();
        }
        m_run = m_new;
      }
      // P (f16) -> SW64 K-major [128 heads][32 rows]
      float lsum = 0.f;
#pragma unroll
      for (int ch = 0; ch < 4; ch++) {
        uint32_t w4[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
          __half2 p2 = __floats2half2_rn(exp2f(x[ch * 8 + 2 * e] - m_run), exp2f(x[ch * 8 + 2 * e + 1] - m_run));
          float2 f = __half22float2(p2);
          lsum += f.x + f.y;
          w4[e] = *reinterpret_cast<uint32_t *>(&p2);
        }
        const uint32_t o = (uint32_t)(h >> 3) * 512 + sw64((uint32_t)(h & 7) * 64 + ch * 16);
        *reinterpret_cast<uint4 *>(sp + o) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
      l_run += lsum;
      fence_proxy_async_smem();
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
      const uint32_t qaddr = smem_u32(sq), paddr = smem_u32(sp);
      auto issue_s = [&](int i) {
        const int kb = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        mbar_wait(&c.kv_full[kb], ph);
        mbar_wait(&c.s_empty[kb], ph ^ 1);
        tc_fence_after();
        const uint32_t kvaddr = smem_u32(skv + kb * KV_BYTES);
#pragma unroll 1
        for (int blk = 0; blk < NBLK; blk++) {
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            uint64_t ad = sw128_desc(qaddr + blk * (HEADS * 128) + kk * 32, 16, 1024);
            uint64_t bd = sw128_desc(kvaddr + blk * KV_BLK_BYTES + kk * 32, 16, 1024);
            mma_f16_ss(tmem + TM_S + kb * NB, ad, bd, IDESC_S, (blk | kk) ? 1u : 0u);
          }
        }
        tc_commit(&c.s_full[kb]);
      };
      issue_s(0);
      for (int i = 0; i < ntiles; i++) {
        if (i + 1 < ntiles) issue_s(i + 1);
        const int kb = i & 1;
        mbar_wait(&c.p_full, i & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_u32(skv + kb * KV_BYTES) + (uint32_t)(4 * v) * KV_BLK_BYTES;
#pragma unroll
        for (int kk = 0; kk < NB / 16; kk++) {
          uint64_t ad = sw64_desc(paddr + kk * 32, 512);
          uint64_t bd = sw128_desc(vaddr + kk * 16 * 128, KV_BLK_BYTES, 1024);
          mma_f16_ss(tmem + TM_O, ad, bd, IDESC_PV, (i | kk) ? 1u : 0u);
        }
        tc_commit(&c.p_empty);
        tc_commit(&c.kv_empty[kb]);
        if (i == ntiles - 1) tc_commit(&c.o_done);
      }
    }
  } else {
    // ---------------- gather + dequant warps --------------------------------------
    const int gt = threadIdx.x - G0 * 32;  // 0..255
    const uint8_t *pool_rows = rows + (int64_t)(pool_begin + b) * rows_per_pool * ROW;
    const int32_t *sel = sel_row + (int64_t)b * sel_stride;
    for (int i = 0; i < ntiles; i++) {
      const int kb = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      mbar_wait(&c.kv_empty[kb], ph ^ 1);
      uint8_t *kv = skv + kb * KV_BYTES;
      // NoPE: 32 rows x 32 chunks of 16 e4m3 -> 2 x 16 B of f16
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const int item = gt + 256 * k;
        const int r = item >> 5, ch = item & 31;
        const int j = i * NB + r;
        uint4 y0 = make_uint4(0, 0, 0, 0), y1 = y0;
        if (j < n) {
          const uint8_t *src = pool_rows + (int64_t)sel[j] * ROW;
          const uint4 x = ld_nc_v4(src + ch * 16);
          const float sc = __ldg(reinterpret_cast<const float *>(src + 512) + (ch >> 3));
          const __half2 s2 = __float2half2_rn(sc);
          y0.x = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.x & 0xFFFF)), s2);
          y0.y = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.x >> 16)), s2);
          y0.z = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.y & 0xFFFF)), s2);
          y0.w = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.y >> 16)), s2);
          y1.x = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.z & 0xFFFF)), s2);
          y1.y = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.z >> 16)), s2);
          y1.z = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.w & 0xFFFF)), s2);
          y1.w = hmul2_u32(cvt_e4m3x2_f16x2((uint16_t)(x.w >> 16)), s2);
        }
        // dims [16ch, 16ch+16): block 16ch/64, 16-B chunks (2ch)%8 and (2ch+1)%8
        const int blk = ch >> 2, c0 = (ch & 3) * 2;
        uint8_t *base = kv + blk * KV_BLK_BYTES;
        *reinterpret_cast<uint4 *>(base + sw128((uint32_t)r * 128 + c0 * 16)) = y0;
        *reinterpret_cast<uint4 *>(base + sw128((uint32_t)r * 128 + (c0 + 1) * 16)) = y1;
      }
      // RoPE: 32 rows x 8 chunks of 8 bf16 -> 8 f16 (dim-block 8)
      {
        const int r = gt >> 3, ch = gt & 7;
        const int j = i * NB + r;
        uint4 y = make_uint4(0, 0, 0, 0);
        if (j < n) {
          const uint4 x = ld_nc_v4(pool_rows + (int64_t)sel[j] * ROW + 528 + ch * 16);
          y.x = bf16x2_to_f16x2(x.x);
          y.y = bf16x2_to_f16x2(x.y);
          y.z = bf16x2_to_f16x2(x.z);
          y.w = bf16x2_to_f16x2(x.w);
        }
        *reinterpret_cast<uint4 *>(kv + 8 * KV_BLK_BYTES + sw128((uint32_t)r * 128 + ch * 16)) = y;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.kv_full[kb]);
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
