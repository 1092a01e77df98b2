/* wlbcp.h -- C ABI of the B200-native WLB-LLM context-parallel hot path.
 *
 * One shared library, `paper_2503_17924_b200/libwlbcp.so`, built for sm_100a.
 * Plain pointers and sizes only (no torch types).  Pointers documented as
 * "device" must be CUDA device memory; `stream` is a cudaStream_t (may be 0).
 * Every entry point returns WLB_OK or an error code; wlb_last_error() gives
 * the message.  All device work is stream-ordered and asynchronous.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/balsim/...).  The reference's FFI boundary is the
 * `balsim._kernels` module (_kernels/__init__.py:35-61), which the drop-in
 * Python layer (paper_2503_17924_b200/_native.py) binds with ctypes.
 */
#ifndef WLBCP_H
#define WLBCP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WLB_OK 0
#define WLB_EINVAL 22      /* bad argument: maps to Python ValueError */
#define WLB_ENODEV 19      /* no usable sm_100 device */
#define WLB_ECUDA 1000     /* CUDA runtime / driver failure */

#define WLB_STRATEGY_PER_SEQUENCE 0
#define WLB_STRATEGY_PER_DOCUMENT 1
#define WLB_POLICY_ADAPTIVE 2
#define WLB_POLICY_MEASURED 3   /* adaptive, priced by the B200 tile model */
#define WLB_TILE_MODEL_LEN 14

/* In-kernel CP synchronisation on per-peer arrival flags (see wlb_cp_signal /
 * wlb_cp_wait): the attention kernels can wait for, and publish, head-group
 * completion themselves, so one launch covers all heads and each head group
 * still starts as soon as its peers' rows have landed.
 *   wait_flags   device [n_groups][cp] int32 flags of THIS rank (the K/V
 *                arrival flags of one exchange slot); a forward CTA waits
 *                until the flags of its KV head's group are >= epoch before
 *                loading K/V.  NULL: no wait.
 *   signal_bases device [cp] peer-mapped flag-buffer bases; when the last
 *                work unit of a head group has stored its dK/dV partials,
 *                the backward stores epoch at byte offset signal_off + 4*cp*g
 *                of every peer (system-scope release).  NULL: no signal.
 *   counters     device [n_groups] int32, zeroed before the backward launch.
 *   kv_per_group KV heads per group (groups are contiguous, equal ranges). */
typedef struct WlbCpSync {
  const int32_t* wait_flags;
  const uint64_t* signal_bases;
  int64_t signal_off;
  int32_t* counters;
  int32_t cp;
  int32_t kv_per_group;
  int32_t epoch;
  int32_t pad_;
} WlbCpSync;

int32_t wlb_abi_version(void);
const char* wlb_last_error(void);
/* 0 when a compute-capability-10.x device is visible, else WLB_ENODEV. */
int wlb_device_check(void);

/* ---------------------------------------------------------------- host ---
 * Longest-first min-W bin placement (bit-identical fp64 expression order).
 * Replaces _kernels.heuristic_fill (_kernels/__init__.py:53-61,
 * _compiled.pyx:50-86).  lengths host [n], sorted descending; out host [n],
 * bin index or -1 for "fits nowhere under l_max". */
int wlb_heuristic_fill(const int64_t* lengths, int64_t n, int32_t n_mb, int64_t l_max,
                       double attn_coeff, double linear_coeff, int32_t* out);

/* -------------------------------------------------------------- device ---
 * Batched CP shard builder + adaptive selector.  Replaces
 * sharding.per_sequence_shard / per_document_shard / strategy_latencies /
 * adaptive_select (sharding.py:86-188) and _kernels.kernel_latency_sum
 * (_kernels/__init__.py:45-50) for n_mb micro-batches in ONE launch.
 *
 * Inputs (device): mb_doc_off[n_mb+1] doc offsets, doc_len[mb_doc_off[n_mb]],
 *   mb_tok_off[n_mb+1] token offsets, curve_q[n_curve], curve_v[n_curve].
 * policy: WLB_STRATEGY_PER_SEQUENCE / _PER_DOCUMENT / WLB_POLICY_ADAPTIVE.
 * Outputs (device):
 *   choice[n_mb]               strategy used (0 seq, 1 doc); -1 if T % 2cp != 0
 *   rank_latency[n_mb][2][cp]  fp64 model latency per strategy and rank,
 *                              bit-identical to worker_attention_latency
 *   rank_pairs[n_mb][cp]       causal pairs per rank (chosen strategy)
 *   seg_count[n_mb][2][cp]     canonical range count per strategy and rank
 *   segs[n_mb][2][cp][max_segs][3]  (doc pos, start, end), canonical order
 *   rowset_off[n_mb][cp][max_docs+1] local row offset of each doc (chosen)
 *   gather_index[mb_tok_off[n_mb]], positions[...] (may be NULL): for rank r
 *     of micro-batch b, local row i lives at mb_tok_off[b] + r*T_b/cp + i and
 *     holds the micro-batch-global token index / in-document position.
 * max_segs must be >= 4*max_docs+2; max_docs >= docs of any micro-batch. */
int wlb_shard_plan(int32_t n_mb, const int32_t* mb_doc_off, const int64_t* doc_len,
                   const int64_t* mb_tok_off, int32_t cp, int32_t policy,
                   int64_t tile, const int64_t* curve_q, const double* curve_v,
                   int32_t n_curve, double op_scale, int32_t max_segs, int32_t max_docs,
                   int32_t* choice, double* rank_latency, int64_t* rank_pairs,
                   int32_t* seg_count, int32_t* segs, int32_t* rowset_off,
                   int32_t* gather_index, int32_t* positions, void* stream);

/* wlb_shard_plan with the MEASURED-latency selector (north-star item 4;
 * PAPER.md:425-429 selects with profiled kernel latency; the reference's
 * CostProfile form, sharding.py:151-188, prices dense q x kv rectangles).
 * Both strategies are priced from the work lists the attention kernels will
 * run: forward 128-row query tiles (pairs) x 128-key KV steps, backward
 * 128-key KV tiles x 64- or 128-query steps, per (strategy, rank).
 * policy: WLB_STRATEGY_PER_SEQUENCE / _PER_DOCUMENT (features and latencies
 *   still computed) or WLB_POLICY_MEASURED (per-sequence if its slowest rank
 *   is predicted no slower, else per-document).
 * model (device) [WLB_TILE_MODEL_LEN] fp64: {SMs, Hq, Hkv, fwd_item_s,
 *   fwd_step_s, bwd_item_s (64-query kernel), bwd_step64_s, bwd_step128_s,
 *   v3_min_rows, const_s, d_is_128, bwd_item128_s (128-query kernel),
 *   fwd_tail, bwd_tail (list-scheduling tail weights)},
 *   calibrated on B200 (paper_2503_17924_b200/calibrate.py).
 * rank_latency receives the predicted seconds [n_mb][2][cp]; features (may
 *   be NULL) [n_mb][2][cp][8] int64: fwd items, fwd steps, max fwd item
 *   steps, bwd items, bwd 64-q steps, bwd 128-q steps, max bwd item steps
 *   (64, 128).  Other arguments as wlb_shard_plan; cp <= 64. */
int wlb_shard_plan_measured(int32_t n_mb, const int32_t* mb_doc_off, const int64_t* doc_len,
                            const int64_t* mb_tok_off, int32_t cp, int32_t policy,
                            const double* model, int32_t max_segs, int32_t max_docs,
                            int32_t* choice, double* rank_latency, int64_t* rank_pairs,
                            int32_t* seg_count, int32_t* segs, int32_t* rowset_off,
                            int32_t* gather_index, int32_t* positions, int64_t* features,
                            void* stream);

/* Tile-padded model latency of arbitrary (q, kv) ranges, summed in order
 * (replaces _kernels.kernel_latency_sum, _compiled.pyx:30-47).  All device;
 * out[0] receives the fp64 sum. */
int wlb_kernel_latency_sum(const int64_t* q_lens, const int64_t* kv_lens, int64_t n,
                           int64_t tile, const int64_t* curve_q, const double* curve_v,
                           int32_t n_curve, double op_scale, double* out, void* stream);

/* Attention work list for one rank: query tiles of <= 128 rows cut from each
 * (rank, doc) row-set, back-aligned (optimal for the doc-prefix cost), paired
 * from the end of the row-set (a pair shares K/V tiles) and sorted by
 * descending KV extent.  rowset_off[n_docs+1], positions[rows] and
 * doc_start[n_docs+1] (global KV offsets) are device arrays.
 * tiles[4*max_tiles][4] int32: item i occupies rows 2i, 2i+1 =
 * {rowX0, nrowsX, kv_begin, kv_endX}, {rowY0, nrowsY, kv_endY, 0} (X is the
 * later tile; nrowsY = 0 when unpaired); the second half is scratch.
 * n_tiles[0] receives the item count.  block_m must be 128. */
int wlb_attn_tiles(int32_t n_docs, const int32_t* rowset_off, const int32_t* positions,
                   const int32_t* doc_start, int32_t block_m, int32_t max_tiles,
                   int32_t* tiles, int32_t* n_tiles, void* stream);

/* Document-prefix causal attention forward, tcgen05/TMEM/TMA on sm_100a.
 * q[Tl][Hq][D], k/v[T][Hkv][D] bf16 (document order), o[Tl][Hq][D] bf16,
 * lse[Hq][Tl] fp32 (natural-log logsumexp of scaled scores).
 * Row i attends keys [kv_begin, kv_begin + positions[i] + 1) of its item.
 * D in {64, 128}; Hq % Hkv == 0. */
int wlb_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                 const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                 const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                 int32_t Hkv, int32_t D, float scale, void* stream);

/* wlb_attn_fwd restricted to KV heads [kv_head_begin, +kv_head_count) and
 * their query heads (the CP exchange's head-group pipeline: attention on a
 * head group starts as soon as that group's K/V rows have landed). */
int wlb_attn_fwd_heads(const void* q, const void* k, const void* v, void* o, float* lse,
                       const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                       const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv,
                       int32_t D, float scale, int32_t kv_head_begin, int32_t kv_head_count,
                       void* stream);

/* wlb_attn_fwd, all heads in one launch, each CTA gated on sync->wait_flags
 * of its KV head's group (sync may be NULL: plain wlb_attn_fwd). */
int wlb_attn_fwd_sync(const void* q, const void* k, const void* v, void* o, float* lse,
                      const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                      const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv,
                      int32_t D, float scale, const WlbCpSync* sync, void* stream);

/* Backward.  do_[Tl][Hq][D] bf16, o and lse from the forward.  Writes
 * dq[Tl][Hq][D] bf16 and dK/dV partials over the full document-ordered
 * sequence, dk/dv[T][Hkv][D] fp32 (summed over ranks by the CP
 * reduce-scatter).  rowset_off[n_docs+1] / positions[Tl] as produced by
 * wlb_shard_plan for this rank, doc_start[n_docs+1] global KV offsets.
 * ws: device workspace of wlb_attn_bwd_workspace() bytes. */
size_t wlb_attn_bwd_workspace(int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv, int32_t D,
                              int32_t n_docs);
int wlb_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                 const void* do_, const float* lse, void* dq, float* dk, float* dv,
                 const int32_t* rowset_off, const int32_t* doc_start, int32_t n_docs,
                 const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                 int32_t Hkv, int32_t D, float scale, void* ws, void* stream);
/* wlb_attn_bwd with flags: WLB_BWD_DKV_BF16 writes the dK/dV partials as
 * bf16 [T][Hkv][D] (the symmetric CP exchange then moves half the bytes and
 * sums them in fp32, wlb_cp_dkv_pull_ex); WLB_BWD_COVERED_ONLY skips the
 * zero fill of uncovered rows; 0 is wlb_attn_bwd. */
#define WLB_BWD_DKV_BF16 1
/* WLB_BWD_COVERED_ONLY: write only the dK/dV partial rows this rank's KV
 * tiles cover (keys below roundup128(last local position + 1) of each
 * document); the rest are left untouched instead of zero-filled.  For
 * consumers that read covered rows only (wlb_cp_dkv_pull_cov). */
#define WLB_BWD_COVERED_ONLY 2
/* WLB_PULL_OUT_BF16 (wlb_cp_dkv_pull_* flags): store the fp32 sums as bf16
 * (round to nearest even) rows of the full head width, e.g. straight into a
 * host-bound bf16 buffer without a conversion pass. */
#define WLB_PULL_OUT_BF16 4
int wlb_attn_bwd_ex(const void* q, const void* k, const void* v, const void* o,
                    const void* do_, const float* lse, void* dq, void* dk, void* dv,
                    const int32_t* rowset_off, const int32_t* doc_start, int32_t n_docs,
                    const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                    int32_t Hkv, int32_t D, float scale, void* ws, int32_t flags, void* stream);
/* wlb_attn_bwd_ex restricted to KV heads [kv_head_begin, +kv_head_count)
 * (dQ of their query heads, dK/dV partial columns of those KV heads).
 * Successive calls over disjoint head ranges may share one workspace. */
int wlb_attn_bwd_heads(const void* q, const void* k, const void* v, const void* o,
                       const void* do_, const float* lse, void* dq, void* dk, void* dv,
                       const int32_t* rowset_off, const int32_t* doc_start, int32_t n_docs,
                       const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv,
                       int32_t D, float scale, void* ws, int32_t flags, int32_t kv_head_begin,
                       int32_t kv_head_count, void* stream);
/* wlb_attn_bwd_ex, all heads in one launch, signalling every peer per head
 * group through sync->signal_bases once the group's partials are stored
 * (sync may be NULL: plain wlb_attn_bwd_ex). */
int wlb_attn_bwd_sync(const void* q, const void* k, const void* v, const void* o,
                      const void* do_, const float* lse, void* dq, void* dk, void* dv,
                      const int32_t* rowset_off, const int32_t* doc_start, int32_t n_docs,
                      const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv,
                      int32_t D, float scale, void* ws, int32_t flags, const WlbCpSync* sync,
                      void* stream);
/* Backward kernel selection for D = 128: the 128-query-tile kernel (v3) runs
 * when Tl >= v3_min_rows * n_docs, else the 64-query kernel (v2).  Negative
 * restores the default (1: always for D = 128); returns the previous threshold.  Process-wide
 * tuning knob (no reference analogue). */
int32_t wlb_attn_bwd_select(int32_t v3_min_rows);
/* v3 as 2-CTA clusters (KV tiles 2q, 2q+1 of a document share query tiles and
 * exchange dQ halves over distributed shared memory, halving the dQ
 * reductions).  Experimental, measured slower: 1 on, 0 off (default),
 * negative = default; returns the previous setting. */
int32_t wlb_attn_bwd_pairs(int32_t on);

/* 64-query (v2) backward scheduling: 1 = persistent (one CTA per SM taking
 * (KV tile, KV head) units from a dynamic queue), 0 = one CTA per unit;
 * negative = default.  Returns the previous setting.  Process-wide knob. */
int32_t wlb_attn_bwd_persistent(int32_t on);

/* SMs the persistent backward kernels leave free for concurrent kernels on
 * other streams (the CP exchange's push / pull): grid = SMs - n (n >= 0;
 * negative = 0, the default).  Returns the previous value.  No reference
 * analogue (a B200 scheduling knob). */
int32_t wlb_attn_bwd_reserve_sms(int32_t n);

/* Persistent 128-query backward: L2 prefetch of the next work unit's K / V
 * tile and first Q / dO tile while the current unit drains (1 on, 0 off,
 * negative = build default).  Returns the previous setting. */
int32_t wlb_attn_bwd_l2_prefetch(int32_t on);

/* Split a fused QKV projection y[Tl][Hq+2*Hkv][D] (bf16) into THD q / k / v
 * and apply rotate-half rotary embeddings at the IN-DOCUMENT positions the
 * shard builder emits (positions[Tl], TokenRange coordinates,
 * workload.py:33-45), theta_i = base^(-2i/D).  The step before the path
 * (SURVEY.md 8f row 3); no reference analogue (the reference does not model
 * the projection). */
int wlb_qkv_rope(const void* y, void* q, void* k, void* v, const int32_t* positions,
                 int32_t Tl, int32_t Hq, int32_t Hkv, int32_t D, float base, void* stream);

/* The projection and RoPE fused into ONE tcgen05 GEMM (D = 128): for local
 * row i, y = x[rows ? rows[i] : i] @ w (x [x_rows][hidden] bf16, w
 * [hidden][(Hq + 2 Hkv) * D] bf16, the x @ W orientation), then q / k get
 * rotate-half RoPE at positions[i] (in-document, as wlb_qkv_rope) and v is
 * y's value heads; q [Tl][Hq][D], k / v [Tl][Hkv][D] bf16.  rows (device
 * [Tl], may be NULL) is the rank's gather_local when x holds the
 * micro-batch's global rows (TMA gather4 loads them).  hidden % 64 == 0,
 * ((Hq + 2 Hkv) * D) % 256 == 0.  Replaces cuBLAS + wlb_qkv_rope (SURVEY.md
 * 8f row 3). */
int wlb_qkv_proj_rope(const void* x, int32_t x_rows, const int32_t* rows, const void* w,
                      void* q, void* k, void* v, const int32_t* positions, int32_t Tl,
                      int32_t hidden, int32_t Hq, int32_t Hkv, int32_t D, float base,
                      void* stream);

/* Row permutations for the CP exchange (rows of row_bytes, 16-B aligned).
 * scatter: dst[index[i]] = src[i];  gather: dst[i] = src[index[i]]. */
int wlb_rows_scatter(const void* src, void* dst, const int32_t* index, int64_t n_rows,
                     int64_t row_bytes, void* stream);
int wlb_rows_gather(const void* src, void* dst, const int32_t* index, int64_t n_rows,
                    int64_t row_bytes, void* stream);

/* Fused CP exchange over NVLink peer memory (symmetric buffers; replaces NCCL
 * all-gather + un-permute and permute + reduce-scatter).
 * peer_bases: device array [cp] of peer-mapped base addresses (same layout on
 * every rank).  kv_push stores local row i of K / V at row gather_local[i] of
 * EVERY rank's document-ordered buffers (base + k_off / v_off).  dkv_pull
 * writes dk[i] = sum_r partial_dk_r[gather_local[i]] (fp32, row_bytes per row),
 * same for dv.  Cross-rank ordering is the caller's (symmetric-memory
 * barriers on the same stream). */
int wlb_cp_kv_push(const void* k_local, const void* v_local, const int32_t* gather_local,
                   int64_t n_rows, int64_t row_bytes, const uint64_t* peer_bases,
                   int64_t k_off, int64_t v_off, int32_t cp, void* stream);
int wlb_cp_dkv_pull(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                    const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                    float* dk, float* dv, int32_t cp, void* stream);
/* As wlb_cp_dkv_pull; with WLB_BWD_DKV_BF16 the peers' partials are bf16
 * (row_bytes = the bf16 row) and are summed in fp32 into fp32 dk / dv. */
int wlb_cp_dkv_pull_ex(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                       const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                       float* dk, float* dv, int32_t cp, int32_t flags, void* stream);
/* As wlb_cp_dkv_pull_ex, reading a peer's partial row only where that peer's
 * backward covered it: rank p covers document d's keys below
 * min(len_d, roundup128(last local position of p in d + 1)), the rest are the
 * zeros the backward writes, so the sums are identical.  rowset_all:
 * [cp][rowset_stride] row-set offsets of every rank (the shard plan's
 * rowset_off for this micro-batch); positions_all: [cp][n_rows] in-document
 * positions of every rank's local rows; doc_start: [n_docs+1]. */
/* As wlb_cp_kv_push, storing local row i only into the ranks that load it:
 * the coverage rule of wlb_cp_dkv_pull_cov, plus the rows a rank's last
 * 128-key tile of an earlier document reads past that document's end (up to
 * 127 rows, under the mask).  Every row any rank's tiles load is therefore
 * rewritten by this micro-batch; rows no tile loads keep earlier contents.
 * cp <= 32 (the coverage mask is a warp ballot). */
int wlb_cp_kv_push_cov(const void* k_local, const void* v_local, const int32_t* gather_local,
                       int64_t n_rows, int64_t row_bytes, const uint64_t* peer_bases,
                       int64_t k_off, int64_t v_off, int32_t cp, const int32_t* rowset_all,
                       int32_t rowset_stride, const int32_t* positions_all,
                       const int32_t* doc_start, int32_t n_docs, void* stream);
int wlb_cp_dkv_pull_cov(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                        const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                        float* dk, float* dv, int32_t cp, int32_t flags,
                        const int32_t* rowset_all, int32_t rowset_stride,
                        const int32_t* positions_all, const int32_t* doc_start, int32_t n_docs,
                        void* stream);

/* General forms of the push / pull above: columns [col_off, col_off +
 * col_bytes) of every row only (a range of KV heads; 16-B aligned), and the
 * covered variant when rowset_all != NULL (else every rank / every row).
 * For the pull, row_bytes / col_* count the partial rows (bf16 with
 * WLB_BWD_DKV_BF16), and dk / dv are fp32 rows of the full head width
 * (bf16 with WLB_PULL_OUT_BF16). */
int wlb_cp_kv_push_part(const void* k_local, const void* v_local, const int32_t* gather_local,
                        int64_t n_rows, int64_t row_bytes, int64_t col_off, int64_t col_bytes,
                        const uint64_t* peer_bases, int64_t k_off, int64_t v_off, int32_t cp,
                        const int32_t* rowset_all, int32_t rowset_stride,
                        const int32_t* positions_all, const int32_t* doc_start, int32_t n_docs,
                        void* stream);
int wlb_cp_dkv_pull_part(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                         const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                         int64_t col_off, int64_t col_bytes, float* dk, float* dv, int32_t cp,
                         int32_t flags, const int32_t* rowset_all, int32_t rowset_stride,
                         const int32_t* positions_all, const int32_t* doc_start, int32_t n_docs,
                         void* stream);
/* The K/V push on the COPY ENGINES: runs (host [n_runs][3] int64: local
 * row, global row, rows) of this rank's local rows, columns [col_off,
 * col_off + col_bytes) of every row, copied (2-D, pitch row_bytes) into every
 * rank's buffer (peer_bases: HOST [cp] peer-mapped addresses) at k_off /
 * v_off.  No SMs: the attention kernels keep every SM while K/V move, and
 * attention CTAs waiting on the arrival flags inside the kernel
 * (wlb_attn_fwd_sync) cannot starve the push. */
int wlb_cp_kv_push_dma(const void* k_local, const void* v_local, const int64_t* runs,
                       int32_t n_runs, int64_t row_bytes, int64_t col_off, int64_t col_bytes,
                       const uint64_t* peer_bases, int64_t k_off, int64_t v_off, int32_t cp,
                       void* stream);

/* Per-peer arrival flags on symmetric memory (replace whole-slot barriers on
 * the data path).  wlb_cp_signal: once the work before it on `stream` is
 * complete, store `value` (system-scope release) at byte offset flag_off of
 * every rank's flag buffer (flag_bases: device [cp] peer-mapped addresses).
 * wlb_cp_wait: work after it on `stream` starts once all n int32 flags
 * (device, this rank's buffer) are >= value (system-scope acquire).  Values
 * are increasing epochs; a wait longer than 60 s traps. */
int wlb_cp_signal(const uint64_t* flag_bases, int64_t flag_off, int32_t cp, int32_t value,
                  void* stream);
int wlb_cp_wait(const int32_t* flags, int32_t n, int32_t value, void* stream);
/* The same as stream memory operations (cuStreamWriteValue32 /
 * cuStreamWaitValue32 GEQ), executed by the GPU front end without an SM, so
 * they make progress while kernels hold every SM (flag_bases: HOST [cp]). */
int wlb_cp_signal_memop(const uint64_t* flag_bases, int64_t flag_off, int32_t cp, int32_t value,
                        void* stream);
int wlb_cp_wait_memop(const int32_t* flags, int32_t n, int32_t value, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WLBCP_H */
