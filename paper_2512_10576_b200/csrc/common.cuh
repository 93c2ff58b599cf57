// Shared device/host helpers for libess_b200 (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/ess_b200.h"

#define ESS_CUDA_TRY(expr)                                  \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ess_record_cuda_error(_e); \
  } while (0)

int ess_record_cuda_error(cudaError_t e);

// Host: 2D tiled tensor map (driver entry point fetched through the runtime, so
// the library does not link libcuda).  inner/box_inner in elements.
bool ess_make_tmap_2d(CUtensorMap *m, CUtensorMapDataType dtype, const void *base,
                      uint64_t inner, uint64_t rows, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swizzle);
int ess_sm_count();  // of the current device
// raise `func`'s dynamic shared-memory limit to >= bytes on the current device (cached)
int ess_smem_optin(const void *func, size_t bytes);

// Per-pool mutable scalars (one 64-byte record per pool).  Recency is a strictly
// increasing 32-bit clock; free slots carry key == slot index (< cap_max) and
// resident slots carry a stamp >= ESS_CLOCK_BASE, so "the v smallest keys" is
// exactly "free slots first, then least-recent residents" (no ties).
struct PoolMeta {
  int32_t cap;
  int32_t size;
  uint32_t clk;
  int32_t pad0;
  int64_t watermark;  // cache.py:44 _append_watermark
  int64_t hits;       // cache.py:41-43
  int64_t misses;
  int64_t evictions;
  int64_t pad1;
  int64_t pad2;
};
static_assert(sizeof(PoolMeta) == 64, "PoolMeta layout");

struct ess_pool {
  int32_t P;
  int64_t max_ids;
  int32_t cap_max;
  int32_t row_bytes;
  int32_t staging;
  int64_t rows_per_pool;
  int device;
  PoolMeta *meta;     // [P]
  int32_t *slot_of;   // [P][max_ids]  id -> slot or -1
  int32_t *slot_id;   // [P][cap_max]  slot -> id or -1
  uint32_t *key;      // [P][cap_max]  recency key (see PoolMeta)
  uint8_t *rows;      // [P][rows_per_pool][row_bytes] slot store (+ staging rows)
  int32_t *status;    // device status word (first error wins)
};

__device__ __forceinline__ void ess_set_status(int32_t *status, int32_t code) {
  atomicCAS(status, 0, code);
}

// Exclusive block scan over NT threads (NT multiple of 32, <= 1024).
// `warp_buf` needs NT/32 ints.  All threads must call.  Returns exclusive prefix;
// *total gets the block sum.
// T = int, or uint32_t for packed multi-field counts (modular adds, logical shifts).
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T *warp_buf, T *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_buf[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T s = lane < NT / 32 ? warp_buf[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) warp_buf[lane] = s;
  }
  __syncthreads();
  T base = warp ? warp_buf[warp - 1] : T(0);
  *total = warp_buf[NT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

// ---- number formats ---------------------------------------------------------------
__device__ __forceinline__ uint32_t cvt_e4m3x2_f16x2(uint16_t v) {  // exact
  uint32_t r;
  asm("{\n\t.reg .b16 t;\n\tmov.b16 t, %1;\n\tcvt.rn.f16x2.e4m3x2 %0, t;\n\t}" : "=r"(r) : "h"(v));
  return r;
}

// f16(f32(e4m3) * s) for two packed e4m3 values (one rounding)
__device__ __forceinline__ uint32_t e4m3x2_scaled_f16x2(uint16_t v, float s) {
  uint32_t h = cvt_e4m3x2_f16x2(v);
  float2 f = __half22float2(*reinterpret_cast<__half2 *>(&h));
  __half2 r = __floats2half2_rn(f.x * s, f.y * s);
  return *reinterpret_cast<uint32_t *>(&r);
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

// Range guard of the f16 operands (K5 computes in f16 on the tensor cores): a packed
// f16 pair holding an inf / NaN — a bf16 source value of magnitude >= 65520 rounds to
// inf — flags ESS_ERR_RANGE in the pool's status word instead of passing silently.
__device__ __forceinline__ bool f16x2_nonfinite(uint32_t h) {
  return ((h & 0x7C00u) == 0x7C00u) | ((h & 0x7C000000u) == 0x7C000000u);
}
__device__ __forceinline__ bool f16x8_nonfinite(uint4 v) {
  return f16x2_nonfinite(v.x) | f16x2_nonfinite(v.y) | f16x2_nonfinite(v.z) | f16x2_nonfinite(v.w);
}
// a bf16 pair with a magnitude >= 65536 (or inf / NaN): outside what f16 represents
__device__ __forceinline__ bool bf16x2_over_f16(uint32_t v) {
  return ((v & 0x7FFFu) >= 0x4780u) | (((v >> 16) & 0x7FFFu) >= 0x4780u);
}
__device__ __forceinline__ bool bf16x8_over_f16(uint4 v) {
  return bf16x2_over_f16(v.x) | bf16x2_over_f16(v.y) | bf16x2_over_f16(v.z) | bf16x2_over_f16(v.w);
}

// Cross-kernel hand-off flags of the streamed step (GPU scope): a producer kernel
// publishes with a release add / store after its data stores, a consumer kernel polls
// with acquire loads (one lane, bounded: trap instead of a hang) and then reads the data
// through L2 (ld.global.cg), never through the non-coherent path.
__device__ __forceinline__ int ess_ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ess_red_release_add(int32_t *p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void ess_st_release(int32_t *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Programmatic dependent launch (ESS_LAUNCH_PDL): a kernel launched with programmatic
// stream serialization may start before the previous kernel on its stream completes —
// its CTAs become resident as the previous kernel's CTAs leave the SMs — and waits
// with ess_pdl_wait() until that kernel has completed and its stores are visible.
// ess_pdl_trigger() lets the NEXT kernel launch early.  Both are no-ops in a kernel
// launched without the attribute.
__device__ __forceinline__ void ess_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void ess_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Launch with optional thread-block cluster (cluster > 1) and programmatic stream
// serialization (pdl).
template <typename... KArgs, typename... Args>
inline cudaError_t ess_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, int cluster, bool pdl, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = (unsigned)cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    n++;
  }
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    n++;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Bounded mbarrier / flag spin: trap instead of hanging the GPU on a protocol bug.
#ifndef ESS_SPIN_LIMIT
#define ESS_SPIN_LIMIT (1u << 26)
#endif

// Scratch builds (-DESS_STREAM_PROF): per-request globaltimer stamps of the streamed
// step — [b][0] top-k start, [1] split published, [2] last gather chunk landed — read
// by scripts/stream_timeline.py through ess_debug_stream_prof_{topk,gather}.
#ifdef ESS_STREAM_PROF
#define ESS_STREAM_PROF_READER(name)                                                           \
  extern "C" int name(unsigned long long *host, int reset) {                                   \
    if (reset) {                                                                               \
      static unsigned long long zero[1024][4];                                                 \
      return cudaMemcpyToSymbol(g_stream_prof, zero, sizeof(zero)) == cudaSuccess ? 0 : -7;    \
    }                                                                                          \
    return cudaMemcpyFromSymbol(host, g_stream_prof, sizeof(g_stream_prof)) == cudaSuccess ? 0 \
                                                                                          : -7; \
  }
#endif
#ifdef ESS_STREAM_PROF
static __device__ unsigned long long g_stream_prof[1024][4];  // one copy per translation unit
__device__ __forceinline__ unsigned long long ess_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SPROF(b, i) (g_stream_prof[(b)][(i)] = ess_gtimer())
#define SPROF_MAX(b, i) atomicMax(&g_stream_prof[(b)][(i)], ess_gtimer())
#else
#define SPROF(b, i) \
  do {              \
  } while (0)
#define SPROF_MAX(b, i) \
  do {                  \
  } while (0)
#endif

// One lane polls (acquire, GPU scope, bounded) until *p >= target; then every lane
// acquires once itself, so the producer's released stores are visible to the warp.
// Exponential back-off (64 ns .. 1 us): many warps polling one flag must not turn its
// L2 slice into a hot spot for the concurrent HBM-bound indexer.
__device__ __forceinline__ void ess_warp_wait_geq(const int32_t *p, int target) {
  if ((threadIdx.x & 31) == 0) {
    uint32_t spins = 0, ns = 64;
    while (ess_ld_acquire(p) < target) {
      if (++spins > ESS_SPIN_LIMIT) __trap();
      __nanosleep(ns);
      ns = ns < 1024 ? 2 * ns : 1024;
    }
  }
  __syncwarp();
  (void)ess_ld_acquire(p);
}

// ---------------------------------------------------------------------------------
// PTX wrappers: mbarrier, TMA, tcgen05 (sm_100a)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// non-suspending probe: a spin on test_wait wakes as soon as the phase flips (try_wait
// may park the warp for a hardware-chosen interval)
__device__ __forceinline__ bool mbar_test_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_test_wait(bar, parity)) {
    if (++spins > 16u * ESS_SPIN_LIMIT) __trap();
  }
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++spins > ESS_SPIN_LIMIT) __trap();
  }
}

// 2D TMA tile load global -> shared, completion on an mbarrier (bytes counted).
__device__ __forceinline__ void tma_load_2d(void *dst, const void *tmap, uint64_t *bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Same with an L2 cache-policy hint (e.g. evict_first for data streamed exactly once).
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const void *tmap, uint64_t *bar,
                                                 int32_t c0, int32_t c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 1D bulk copy global -> shared (16-B aligned, size % 16 == 0), mbarrier tx completion.
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// tcgen05 -------------------------------------------------------------------------
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t *smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_dst)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// MMA completion -> mbarrier arrive (implicitly fences before_thread_sync)
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f8f6f4 (e4m3 x e4m3 -> f32)
__device__ __forceinline__ void mma_f8f6f4_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// kind::f16 (f16/bf16 x f16/bf16 -> f32)
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_128B canonical layout, sm_100 version 1.
//   start address (>>4) bits [0,14), LBO (>>4) [16,30), SBO (>>4) [32,46),
//   version [46,48) = 1, base offset [49,52) = 0, layout type [61,64) = 2 (SW128).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo_bytes,
                                               uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor (kind::f16 / kind::f8f6f4 dense):
//   c_format [4,6) (1 = f32), a_format [7,10), b_format [10,13),
//   a_major bit 15, b_major bit 16 (0 = K-major, 1 = MN-major),
//   n >> 3 at [17,23), m >> 4 at [24,29).
__host__ __device__ constexpr uint32_t make_idesc(uint32_t a_fmt, uint32_t b_fmt, uint32_t m,
                                                  uint32_t n, uint32_t a_mn_major,
                                                  uint32_t b_mn_major) {
  return (1u << 4) | (a_fmt << 7) | (b_fmt << 10) | (a_mn_major << 15) | (b_mn_major << 16) |
         ((n >> 3) << 17) | ((m >> 4) << 24);
}

// TMEM -> registers: 32 lanes x 32 bit, 64 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
      "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),
        "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]),
        "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
        "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]),
        "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

// 32 columns per thread
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// 128-bit loads/stores
__device__ __forceinline__ uint4 ld_nc_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
#ifndef ESS_HOST_PREFETCH
#define ESS_HOST_PREFETCH "L2::256B"
#endif
// host-link (zero-copy) variant: the L2 fetch-size hint turns a warp's 16-B lane loads
// into fewer, larger PCIe read requests
__device__ __forceinline__ uint4 ld_host_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate." ESS_HOST_PREFETCH ".v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// 32-B host-link load (sm_100 256-bit LDG)
__device__ __forceinline__ void ld_host_v8(const void *p, uint4 &a, uint4 &b) {
  asm volatile("ld.global.nc.L1::no_allocate." ESS_HOST_PREFETCH ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ uint4 ld_volatile_v4(const void *p) {
  // system-scope data (mapped host memory): bypass L1, no caching assumptions
  uint4 r;
  asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(void *p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
