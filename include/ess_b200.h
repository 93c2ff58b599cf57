/*
 * ess_b200.h — C ABI of the B200-native ESS decode hot path (libess_b200.so).
 *
 * Plain pointers and sizes only: every d_* argument is a device pointer (or a
 * device-mapped pointer to cudaHostRegister'd memory), every call is
 * asynchronous on the caller's cudaStream_t (passed as void*), nothing
 * allocates on the hot path, and every function returns an ESS_* status.
 * Errors that can only be detected on the device (the reference's ValueError
 * classes) are latched in a per-pool status word read by ess_pool_status().
 *
 * The reference (offsim, /root/reference/pkg/src/offsim) is pure Python and
 * has no FFI; each entry point below names the Python interface it replaces,
 * i.e. what an `offsim` maintainer would bind with ctypes.
 *
 * Data layouts:
 *   latent row   656 B = [0,512) e4m3 NoPE | [512,528) 4 x f32 group scales |
 *                [528,656) 64 x bf16 RoPE          (scenario.py:25, costmodel.py:31)
 *                — the host store and every H2D/D2H transfer use this format
 *   slot row     one of two formats, chosen per pool set at ess_pool_create:
 *                656 B  (ESS_SLOT_ROW_BYTES_FP8) the latent row itself — the slot store
 *                       costs exactly the latent bytes it caches; K5 dequantises in
 *                       shared memory (FP8 sparse MLA on a cta_group::2 CTA pair)
 *                1152 B (ESS_SLOT_ROW_BYTES) 576 x f16: dequantised NoPE (e4m3 x scale)
 *                       ++ RoPE, dequantised once on admission
 *   indexer key  128 B e4m3 + f32 scale per token (separate arrays)
 *                                                   (scenario.py:26, :30-33)
 *   pools        P = layers x requests independent LRU pools, pool id = l*B + b
 *                (one pool per (request, layer): SPEC.md:281, cache.py:176-177)
 */
#ifndef ESS_B200_H
#define ESS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESS_LATENT_ROW_BYTES 656
/* host latent store row pitch: 656-B rows on 64-B boundaries.  The host link moves
 * 64-B read requests; an unaligned 656-B row straddles 12 of them, an aligned one 11
 * (+6% zero-copy gather bandwidth, measured; profiles/README.md).  Rows of the host
 * store are addressed as d_host_rows + (pool * host_pool_stride_rows + id) * pitch. */
#ifndef ESS_HOST_ROW_PITCH  /* scratch builds may override (A/B of the host layout) */
#define ESS_HOST_ROW_PITCH 704
#endif
#define ESS_SLOT_ROW_BYTES 1152 /* 576 x f16: the dequantised slot format */
#define ESS_SLOT_ROW_BYTES_FP8 656 /* the raw latent row as the slot format (K5 dequantises on chip) */
#define ESS_NOPE_DIM 512
#define ESS_ROPE_DIM 64
#define ESS_INDEXER_HEADS 64
#define ESS_INDEXER_DIM 128
#define ESS_MLA_HEADS 128
#define ESS_MLA_QK_DIM 576
#define ESS_MLA_V_DIM 512
#define ESS_MAX_REQUEST 2048 /* max ids per pool per access/warm-up call (top-k 2048, scenario.py:24) */

/* status codes; the negative ones mirror the reference's ValueError classes */
#define ESS_OK 0
#define ESS_ERR_CAPACITY (-1)  /* capacity < 1 (cache.py:37-38) or > cap_max          */
#define ESS_ERR_SHRINK (-2)    /* "capacity may only grow" (cache.py:60-61)            */
#define ESS_ERR_DUPLICATE (-3) /* "duplicate generated entry id" (cache.py:127-128)    */
#define ESS_ERR_NOMEM (-4)
#define ESS_ERR_RATIO (-5)     /* sparse_ratio not in (0, 1] (cache.py:174-175)        */
#define ESS_ERR_ARG (-6)       /* id out of [0, max_ids), request too long, bad sizes  */
#define ESS_ERR_CUDA (-7)      /* CUDA runtime / driver failure                        */
#define ESS_ERR_CLOCK (-8)     /* 32-bit recency clock exhausted (> 4e9 touches)       */
#define ESS_ERR_RANGE (-9)     /* a K5 operand (q, or a slot row's dequantised value)
                                  outside the f16 range (|x| >= 65520): latched, the
                                  output of that launch is not valid                  */

/* Launch flag (OR-ed into ess_indexer_logits_ex's max_ctas, ess_gather(_signal)'s flags,
 * ess_topk_split_ex's flags): programmatic dependent launch — the kernel may start while
 * the previous kernel on the same stream is finishing (its prologue and launch latency
 * hide under that kernel's tail) and waits on the device for it to complete before
 * reading its outputs (griddepcontrol).  For back-to-back dependent launches on one
 * stream, e.g. the first micro-batch's K1 -> K2 + K3a -> K4 chain. */
#define ESS_LAUNCH_PDL (1 << 30)
#define ESS_CLOCK_BASE (1u << 24)   /* recency stamps start here; free slots key = slot index */

#define ESS_ACCESS_SORT_EVICTED 1 /* emit evicted ids sorted ascending (cache.py:120) */

typedef struct ess_pool ess_pool;

/* ---- library ---------------------------------------------------------------- */
const char *ess_version(void);
const char *ess_status_string(int status);
/* load every kernel of the library on the current device now (first call per device;
 * lazy module loading would load a kernel at its first launch, which waits for the
 * device — a deadlock when a running kernel spins on work a not-yet-loaded kernel
 * produces, as in the streamed hand-offs) */
int ess_preload(void);
/* ESS_HOST_ROW_PITCH as compiled into this library */
int ess_host_row_pitch(void);
/* cudaHostRegister(mapped) + device alias: the host latent store (UVA gather source) */
int ess_host_register(void *host_ptr, size_t bytes, void **d_alias);
int ess_host_unregister(void *host_ptr);
/* allocate + register the host latent store: 2-MB aligned, transparent huge pages
 * (ESS_HOST_HUGEPAGES), bound to numa_node when >= 0; *placed reports which of the
 * flags took effect.  ESS_HOST_VMM: one host-located VMM allocation (cuMemCreate,
 * CU_MEM_LOCATION_TYPE_HOST_NUMA) mapped at one VA for device and CPU (*host_ptr ==
 * *d_alias), falling back to the registered store when the driver has no host VMM.
 * Free with ess_host_free(host_ptr, bytes). */
#define ESS_HOST_HUGEPAGES 1
#define ESS_HOST_NUMA_BOUND 2
#define ESS_HOST_VMM 4
int ess_host_alloc(size_t bytes, int32_t flags, int32_t numa_node, void **host_ptr, void **d_alias,
                   int32_t *placed);
int ess_host_free(void *host_ptr, size_t bytes);
/* diagnostic: write the device global timer (ns) to *d_dst in stream order; works
 * inside captured CUDA graphs (step timelines) */
int ess_timestamp(uint64_t *d_dst, void *stream);
/* up to ESS_COPY_MAX device-to-device copies (pointers 16-B aligned, sizes multiples of
 * 16 B) in one SM kernel: the decode step's input staging (copy-engine D2D copies ran at
 * ~0.4 TB/s with microseconds of latency each, in front of every step) */
#define ESS_COPY_MAX 64
int ess_copy_many(int32_t n, void *const *d_dst, const void *const *d_src, const int64_t *bytes,
                  void *stream);

/* ---- K3 cache manager: replaces offsim.cache.SparsePool (cache.py:29-134) ------ */
/* num_pools pools over ids [0, max_ids), each with up to cap_max slots.  When
 * row_bytes is ESS_SLOT_ROW_BYTES_FP8 or ESS_SLOT_ROW_BYTES the pool also owns its GPU
 * slot store in that format: per pool
 * cap_max slot rows + staging_rows transient rows (oversize requests,
 * cache.py:103-111).  row_bytes == 0: bookkeeping only (replay). */
int ess_pool_create(ess_pool **out, int32_t num_pools, int64_t max_ids, int32_t cap_max,
                    int32_t row_bytes, int32_t staging_rows);
int ess_pool_destroy(ess_pool *pool);
/* empty pools [begin, begin+num) with capacity d_capacity[i]   (SparsePool(capacity)) */
int ess_pool_reset(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_capacity,
                   void *stream);
/* capacity may only grow                                      (SparsePool.grow_capacity) */
int ess_pool_grow(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_capacity,
                  void *stream);
/* one warm-up window per pool (<= ESS_MAX_REQUEST ids, duplicate-free); adds the
 * number of newly inserted ids to d_inserted[i]                   (SparsePool.warmup) */
int ess_pool_warmup(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_ids,
                    const int32_t *d_n, int32_t stride, int64_t *d_inserted, void *stream);
/* one selection set per pool (unique ids, any order, n <= ESS_MAX_REQUEST)
 *                                                            (SparsePool.access_step)
 * outputs, each [num][out_stride] (any may be NULL):
 *   d_hit_ids, d_miss_ids   in requested order (cache.py:98-99)
 *   d_evicted_ids           ascending if flags & ESS_ACCESS_SORT_EVICTED
 *   d_sel_row               slot-store row of every requested id (attention input)
 *   d_hit_row               row of every hit, in hit order (attention over the
 *                           resident rows while the misses are in flight)
 *   d_miss_row              destination row of every miss (gather input)
 *   d_counts [num][4]       nhit, nmiss (= h2d_blocks), nevicted, ntransient      */
int ess_pool_access(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_req,
                    const int32_t *d_n, int32_t req_stride, int32_t *d_hit_ids,
                    int32_t *d_miss_ids, int32_t *d_evicted_ids, int32_t *d_sel_row,
                    int32_t *d_hit_row, int32_t *d_miss_row, int32_t *d_counts,
                    int32_t out_stride, int32_t flags, void *stream);
/* MTP (qtok = mtp + 1 selection sets per pool per step: recency is updated
 * by every selected set): pool i takes sets r = i*qtok + j, j = 0..qtok-1 (d_req row r at
 * d_req + r*req_stride, n = d_n[r]) as qtok consecutive access_steps in one launch.
 * d_sel_row is laid out like d_req (row r: the slot row of each id of set r); the
 * hit / miss / evicted id and row lists of a pool's sets are appended in set order in
 * its [out_stride >= qtok * req_stride] row; d_counts [num][4] are the sums.
 * Optional attention split per set (all three or none), laid out like d_req: the rows
 * of the set resident before the step (d_tok_hit_row) and those fetched this step by
 * this set or an earlier one (d_tok_fresh_row), each in requested order, with
 * d_tok_counts [num * qtok][2] = (resident, fetched).  d_ready [num] (optional): set to 1
 * (release) per pool once its lists and counts are stored — a concurrently running
 * ess_gather_stream takes the pool's misses from then on. */
int ess_pool_access_mtp(ess_pool *pool, int32_t begin, int32_t num, int32_t qtok,
                        const int32_t *d_req, const int32_t *d_n, int32_t req_stride,
                        int32_t *d_hit_ids, int32_t *d_miss_ids, int32_t *d_evicted_ids,
                        int32_t *d_sel_row, int32_t *d_hit_row, int32_t *d_miss_row,
                        int32_t *d_counts, int32_t out_stride, int32_t *d_tok_hit_row,
                        int32_t *d_tok_fresh_row, int32_t *d_tok_counts, int32_t *d_ready,
                        int32_t flags, void *stream);
/* Early-gather split of ess_pool_access (needs staging_rows >= 2048 and n <= capacity):
 * ess_pool_split is the read-only hit/miss split — hit rows, miss ids and STAGING rows
 * (cap_max + j) for the misses, counts (hits, misses) — so the host-link gather can
 * start at once; ess_pool_access with d_miss_row = a settle-slot buffer then updates
 * the LRU state and reports each miss's final slot; ess_pool_settle copies the fetched
 * rows from staging into those slots (after the gather, concurrently with attention). */
int ess_pool_split(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_req,
                   const int32_t *d_n, int32_t req_stride, int32_t *d_hit_row, int32_t *d_miss_ids,
                   int32_t *d_miss_row, int32_t *d_counts, int32_t out_stride, void *stream);
int ess_pool_settle(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_slot,
                    const int32_t *d_counts, int32_t stride, void *stream);
/* admit generated ids at top recency; d_slot_out [num][stride] gets each id's
 * slot (may be NULL)                                     (SparsePool.append_generated) */
int ess_pool_append(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_ids,
                    const int32_t *d_m, int32_t stride, int32_t *d_slot_out, void *stream);
/* the decode step's tail in one launch (cache.py:191-195, :137-138, :122-134): per pool,
 * with h = d_hist[i] (history length) and m = d_m ? d_m[i] : 1 generated tokens
 * (m <= src_stride, else ESS_ERR_ARG is latched):
 * grow capacity to max(1, floor(rho * (h + m))), admit ids h..h+m-1 at top recency
 * (LRU evictions counted), write each 656-B source row (d_src_rows [num][src_stride])
 * to the host store (D2H) and, dequantised, to its slot; d_hist[i] += m.              */
int ess_pool_admit(ess_pool *pool, int32_t begin, int32_t num, int32_t *d_hist,
                   const int32_t *d_m, double rho, const void *d_src_rows, int32_t src_stride,
                   void *d_host_rows, int64_t host_pool_stride_rows, int32_t *d_slot_out,
                   void *stream);
/* least- to most-recent resident ids: d_out [num][cap_max], d_count [num]
 *                                                 (SparsePool.lru_order, cache.py:55-57) */
int ess_pool_lru_order(ess_pool *pool, int32_t begin, int32_t num, int32_t *d_out,
                       int32_t *d_count, void *stream);
/* d_out [num][8] int64: capacity, size, hits, misses, evictions, clock, watermark, 0 */
int ess_pool_counters(ess_pool *pool, int32_t begin, int32_t num, int64_t *d_out, void *stream);
/* slot of each id in pool `pool` (-1 = not resident)         (SparsePool.__contains__) */
int ess_pool_lookup(ess_pool *pool, int32_t pool_index, const int32_t *d_ids, int32_t n,
                    int32_t *d_slot_out, void *stream);
/* copy pool state (and slot rows) into another pool set with >= max_ids / cap_max;
 * used to grow a pool past its allocated cap_max            (SparsePool.grow_capacity) */
int ess_pool_copy_state(ess_pool *dst, int32_t dst_begin, ess_pool *src, int32_t src_begin,
                        int32_t num, void *stream);
/* synchronous: read and clear the pool's device status word */
int ess_pool_status(ess_pool *pool, int32_t *status_out);
int ess_pool_info(ess_pool *pool, int32_t *num_pools, int64_t *max_ids, int32_t *cap_max,
                  int32_t *row_bytes, int64_t *rows_per_pool, void **d_rows);

/* ---- K4 FlashTrans-style zero-copy gather (replaces the
 *      transfer_time(..., "h2d") cost term, costmodel.py:173-186) ------------------ */
/* copies every miss row host_rows[pool][miss_id] -> slot store[pool][miss_row]
 * with 16-B loads through the device alias of registered host memory.  Pool i
 * of the range reads host rows at d_host_rows + (i*host_pool_stride_rows + id)*704. */
#define ESS_GATHER_EXCLUSIVE_SM 1        /* run only on SMs no attention CTA occupies */
#define ESS_GATHER_EXCLUSIVE_SMEM (64 * 1024)
#define ESS_GATHER_BULK 2                /* rows via cp.async.bulk into a smem ring, not 16-B loads */
/* flags may also carry ESS_LAUNCH_PDL (ess_gather / ess_gather_signal) */
int ess_gather(ess_pool *pool, int32_t begin, int32_t num, const void *d_host_rows,
               int64_t host_pool_stride_rows, const int32_t *d_miss_ids,
               const int32_t *d_miss_row, const int32_t *d_counts, int32_t stride,
               int32_t max_ctas, int32_t flags, void *stream);
/* as ess_gather, and every landed row also adds 1 (release, GPU scope) to
 * d_landed[pool - begin] — the per-request arrival counters ess_sparse_mla_da
 * waits on.  The caller zeroes d_landed [num] before the launch. */
int ess_gather_signal(ess_pool *pool, int32_t begin, int32_t num, const void *d_host_rows,
                      int64_t host_pool_stride_rows, const int32_t *d_miss_ids,
                      const int32_t *d_miss_row, const int32_t *d_counts, int32_t stride,
                      int32_t *d_landed, int32_t max_ctas, int32_t flags, void *stream);
/* The streamed step's gather: launched with the step, it takes request b once
 * d_ready[b] != 0 (ess_topk_split_stream), warps claiming chunks of its miss list from
 * d_claim[b] (zero at launch), every landed chunk added to d_landed[b] (release; may be
 * NULL).  Requests are taken in order; rows as in ess_gather.  No ESS_GATHER_BULK. */
int ess_gather_stream(ess_pool *pool, int32_t begin, int32_t num, const void *d_host_rows,
                      int64_t host_pool_stride_rows, const int32_t *d_miss_ids,
                      const int32_t *d_miss_row, const int32_t *d_counts, int32_t stride,
                      const int32_t *d_ready, int32_t *d_claim, int32_t *d_landed, int32_t max_ctas,
                      int32_t flags, void *stream);
/* D2H write-back + slot fill of generated rows (cache.py:122-134):
 * src rows [num][stride][656] -> host_rows[pool][id] and slot store[pool][slot] */
int ess_write_generated(ess_pool *pool, int32_t begin, int32_t num, const int32_t *d_ids,
                        const int32_t *d_m, const int32_t *d_slot, int32_t stride,
                        const void *d_src_rows, void *d_host_rows,
                        int64_t host_pool_stride_rows, void *stream);

/* ---- K1 lightning indexer (op "indexer_logits", costmodel.py:18-27) ------------- */
/* logits[b][s] = kscale[b][s] * sum_h w[b][h] * relu(q[b][h] . k[b][s]), s < len[b]
 * q [B][64][128] e4m3, w [B][64] f32, k [B][k_ld][128] e4m3 (k_ld % 128 == 0),
 * kscale [B][k_ld] f32, logits [B][k_ld] f32.  tcgen05 kind::f8f6f4 + TMA.       */
int ess_indexer_logits(const void *d_q, const float *d_w, const void *d_k,
                       const float *d_kscale, const int32_t *d_len, int32_t batch,
                       int64_t k_ld, float *d_logits, void *stream);
/* same, on at most max_ctas SMs (0 = all): leaves SMs free for a concurrent
 * host-link gather (the DBA micro-batch schedule); max_ctas may carry
 * ESS_LAUNCH_PDL (K1 reads only its inputs, so it never waits for the previous kernel) */
int ess_indexer_logits_ex(const void *d_q, const float *d_w, const void *d_k,
                          const float *d_kscale, const int32_t *d_len, int32_t batch,
                          int64_t k_ld, float *d_logits, int32_t max_ctas, void *stream);

/* MTP decode (mtp + 1 = qtok query tokens per request, pipeline.py:213-215):
 * q [B][qtok][64][128] e4m3, w [B][qtok][64] f32, logits [B][qtok][k_ld] f32; every token
 * of request b scores the same len[b] cached keys (the selection universe is the cache
 * history, trace.py:151-154).  The keys are read once per request: one tcgen05 MMA with
 * N = 64 * qtok per key tile.  1 <= qtok <= ESS_INDEXER_MAX_QTOK; qtok = 1 is
 * ess_indexer_logits_ex. */
#define ESS_INDEXER_MAX_QTOK 4
int ess_indexer_logits_mtp(const void *d_q, const float *d_w, const void *d_k,
                           const float *d_kscale, const int32_t *d_len, int32_t batch,
                           int32_t qtok, int64_t k_ld, float *d_logits, int32_t max_ctas,
                           void *stream);

/* The streamed step (one CUDA graph, three concurrent kernels with per-request hand-off
 * counters instead of micro-batches): the indexer processes requests in groups of
 * `group` with the whole grid, and after storing its logits rows of request b every
 * epilogue warp adds their number to d_done[b] (release).  group: requests per group in
 * its low 16 bits, the first group's size in the high 16 bits (0: the same; a small first
 * group starts the host link sooner).  d_done reaches min(len[b],
 * k_ld) when b's logits are complete.  d_done [batch] zero at launch.  max_ctas must
 * leave SMs for the concurrent ess_topk_split_stream and ess_gather_stream grids (all
 * three must be co-resident). */
int ess_indexer_logits_stream(const void *d_q, const float *d_w, const void *d_k,
                              const float *d_kscale, const int32_t *d_len, int32_t batch,
                              int64_t k_ld, float *d_logits, int32_t max_ctas, int32_t group,
                              int32_t *d_done, void *stream);

/* ---- K2 top-k (op "indexer_topk") ---------------------------------------------- */
/* per row: the k largest logits[b][0:len[b]) by (score desc, index asc), written
 * ascending to d_idx [B][idx_ld]; d_count[b] = min(k, len[b]) (scenario.py:110-112);
 * 1 <= k <= ESS_TOPK_MAX_K */
#define ESS_TOPK_MAX_K 65535
int ess_topk(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch,
             int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count, void *stream);
/* MTP: batch * qtok rows (request-major: row b*qtok + j is token j of request b), each
 * the top-k of logits[row][0:len[b]) — the K2 half of ess_indexer_logits_mtp */
int ess_topk_mtp(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch,
                 int32_t qtok, int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count,
                 void *stream);
/* top-k fused with ess_pool_split on the emitted selection, one launch (for cluster
 * rows > 40K tokens, rank 0 of each cluster splits): pools [pool_begin, pool_begin+batch) */
int ess_topk_split(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch,
                   int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count, ess_pool *pool,
                   int32_t pool_begin, int32_t *d_hit_row, int32_t *d_miss_ids,
                   int32_t *d_miss_row, int32_t *d_counts, int32_t out_stride, void *stream);
/* same with launch flags (ESS_LAUNCH_PDL) */
int ess_topk_split_ex(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch,
                      int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count, ess_pool *pool,
                      int32_t pool_begin, int32_t *d_hit_row, int32_t *d_miss_ids,
                      int32_t *d_miss_row, int32_t *d_counts, int32_t out_stride, int32_t flags,
                      void *stream);

/* Streamed K2 + K3a: `ctas` persistent CTAs (ctas < 0: -ctas two-CTA clusters, one row
 * per pair) take the requests in order; row b starts
 * once d_done[b] == min(len[b], ld) (ess_indexer_logits_stream), then the top-k and the
 * early-gather split of ess_topk_split run and d_ready[b] is set to 1 (release).  Rows
 * up to 40K tokens (one CTA each); d_ready [batch] zero at launch. */
int ess_topk_split_stream(const float *d_logits, int64_t ld, const int32_t *d_len, int32_t batch,
                          int32_t k, int32_t *d_idx, int32_t idx_ld, int32_t *d_count, ess_pool *pool,
                          int32_t pool_begin, int32_t *d_hit_row, int32_t *d_miss_ids,
                          int32_t *d_miss_row, int32_t *d_counts, int32_t out_stride,
                          const int32_t *d_done, int32_t *d_ready, int32_t ctas, void *stream);

/* ---- K5 sparse MLA decode (ops "sparse_mla" + "merge_attn") --------------------- */
/* out[b][h] = softmax_j(q[b][h] . K[j] * sm_scale) V[j] over the rows
 * sel_row[b][0:count) (count = d_count[b * count_stride]) of pool (pool_begin + b)'s
 * slot store; K = NoPE ++ RoPE (576), V = NoPE (512).  q [B][128][576] bf16,
 * out [B][128][512] bf16, lse [B][128] f32 (natural log).
 * The paper's split attention is two calls sharing a workspace
 * (d_ws_o [B][128][512] f32, d_ws_ml [B][128][2] f32):
 *   ESS_MLA_PARTIAL  write the unnormalised state (O, running max, sum) to the
 *                    workspace instead of out/lse            (Attn0: resident rows)
 *   ESS_MLA_RESUME   start from the workspace state and finish (Attn1: fetched rows
 *                    + the merge)                                                   */
#define ESS_MLA_PARTIAL 1
#define ESS_MLA_SPLIT_SHIFT 8   /* flags bits 8..11: KV splits - 1 (full mode; ws sized batch*splits) */
#define ESS_MLA_MAX_SPLIT 8
#define ESS_MLA_QTOK_SHIFT 12   /* flags bits 12..14: qtok - 1 (MTP): batch = pools * qtok query-token
                                  rows, row r attends in pool pool_begin + r / qtok (q row r, out row r) */
#define ESS_MLA_RESUME 2
int ess_sparse_mla(ess_pool *pool, int32_t pool_begin, const void *d_q,
                   const int32_t *d_sel_row, int32_t sel_stride, const int32_t *d_count,
                   int32_t count_stride, int32_t batch, float sm_scale, void *d_out,
                   float *d_lse, float *d_ws_o, float *d_ws_ml, int32_t flags, void *stream);
/* The DA schedule in one launch: attention over the resident rows d_hit_row[b][0:h)
 * and then, once d_landed[b] reaches m, over the fetched rows d_miss_row[b][0:m)
 * (h, m = d_counts[b * count_stride + 0 / 1], the access counts of
 * ess_pool_access), while ess_gather_signal lands those rows on other SMs.  Same
 * out / lse as ess_sparse_mla over the union.  Its 2 * batch CTAs spin on the
 * counters, so the gather must be co-resident: batch <= (SMs - 8) / 2, with the
 * gather given the remaining SMs (ESS_GATHER_EXCLUSIVE_SM).  d_landed [batch] must
 * be zero at the first call; the kernel leaves it zero again for the next step.  */
int ess_sparse_mla_da(ess_pool *pool, int32_t pool_begin, const void *d_q,
                      const int32_t *d_hit_row, const int32_t *d_miss_row, int32_t row_stride,
                      const int32_t *d_counts, int32_t count_stride, int32_t *d_landed,
                      int32_t batch, float sm_scale, void *d_out, float *d_lse, void *stream);
/* same with the rows of each request split into nsplit shares, each an equal slice of the
 * resident rows and of the fetched rows (2 * nsplit CTAs per request; small batches),
 * partial states in d_ws_o [batch*nsplit][128][512] f32 / d_ws_ml [batch*nsplit][128][2]
 * f32, merged by a combine kernel on the stream.
 * nsplit = 1 is ess_sparse_mla_da.  2 * batch * nsplit <= SMs - 8.                */
int ess_sparse_mla_da_split(ess_pool *pool, int32_t pool_begin, const void *d_q,
                            const int32_t *d_hit_row, const int32_t *d_miss_row,
                            int32_t row_stride, const int32_t *d_counts, int32_t count_stride,
                            int32_t *d_landed, int32_t batch, float sm_scale, void *d_out,
                            float *d_lse, float *d_ws_o, float *d_ws_ml, int32_t nsplit,
                            void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ESS_B200_H */
