// Document-prefix causal attention, backward, on sm_100a tensor cores.
//
// Work item = (KV tile, KV head g): 128 consecutive keys of ONE document
// (in-document positions [k0, k0+128)) and every local query row of the
// (rank, doc) row-set that can see them (position >= k0: a suffix of the
// row-set, found by binary search), for every query head of the GQA group.
// The rows are walked in query tiles of BM = 64; per tile i:
//
//   S^T  = K Q^T,  dP^T = V dO^T     TMEM, lanes = keys, double-buffered
//   P^T  = exp2(S^T*scale*log2e - LSE2[q]);  dS^T = P^T (dP^T - Delta[q])
//          (8 compute warps: key row = TMEM lane, 32 query columns each;
//           P^T -> TMEM over S^T, dS^T -> TMEM over dP^T AND SMEM, bf16)
//   dV  += P^T dO,  dK += dS^T Q     TS MMAs (A read from TMEM), TMEM accumulators
//   dQ^T = K^T dS^T                  TMEM, aliases dP^T of the same buffer;
//          drained by a dedicated warpgroup with warp-coalesced fp32
//          reductions (lane = head-dim index, so each red covers 128
//          contiguous bytes).
//
// The MMA warp issues S/dP for tile i+1 before the dV/dK/dQ group of tile i,
// so the tensor pipe runs while the compute warps work on the previous tile.
// dK/dV are written once per work item as fp32 partials over the full
// document-ordered sequence (the CP reduce-scatter sums them over ranks);
// keys no work item covers are zero-filled separately.  For short row-sets a
// CTA walks several KV heads of its tile in one flat tile sequence.  This is
// the "v2" kernel (any D); the 128-query "v3" kernel below takes over for
// long row-sets at D = 128 (wlb_attn_bwd_select).
#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

#ifndef WLB_HPC_ROWS
#define WLB_HPC_ROWS 4096   // several heads per CTA below this many local rows per document
                           // (2048-row documents: fwd +5%, bwd +3% vs a 2048 threshold;
                           //  8192 cost a 6-document 32K sequence 7% in the forward)
#endif

#include <algorithm>

// Query-tile order inside a KV work item for GQA (Hq > Hkv): 0 (default) =
// head by head; 1 = the group's query heads innermost (a row block's heads
// back to back).  1 was meant to keep the fp32 dQ accumulator lines of a row
// block L2-resident across heads, but measured 5x the DRAM traffic of the v3
// backward (132 vs 27 GB per GQA bench step) and 881 vs 926-932 TFLOP/s
// (profiles/r02_ab_gqa_head_order.txt).  No effect for Hq = Hkv.
#ifndef WLB_BWD_HEAD_INNER
#define WLB_BWD_HEAD_INNER 0
#endif

namespace wlb {
using namespace sm100;

#ifdef WLB_TRACE
// development aid: per-iteration clock64 stamps of the first two CTAs
__device__ long long g_bwd_trace[2][8][128];
#define TRACE(ev, i)                                                            \
  do {                                                                          \
    if (blockIdx.x < 2 && (i) < 128 && (threadIdx.x & 31) == 0 &&               \
        (threadIdx.x >> 5) == ((ev) < 3 ? 1 : (ev) < 6 ? 4 : 12))               \
      g_bwd_trace[blockIdx.x][ev][i] = clock64();                               \
  } while (0)
#else
#define TRACE(ev, i) \
  do {               \
  } while (0)
#endif

template <int D, int NCW = 2>
struct BwdCfg {
  static_assert(NCW == 2, "two compute warpgroups (one 32-query half each)");
  static constexpr int BM = 64, BN = 128;   // queries per tile, keys per tile
  static constexpr int SLABS = D / 64;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int T_BYTES = BN * BM * 2;   // P^T / dS^T tile: 128 rows x 128 B
  static constexpr int Q_SLAB = BM * 128, KV_SLAB = BN * 128;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV_BYTES;
  static constexpr int QS = 3;                          // Q/dO + query-vector ring depth
  static constexpr int OFF_Q = OFF_V + KV_BYTES;        // QS stages
  static constexpr int OFF_DO = OFF_Q + QS * Q_BYTES;   // QS stages
  static constexpr int OFF_DS = OFF_DO + QS * Q_BYTES;  // 2 buffers (dS^T for the dQ MMA)
  static constexpr int OFF_VEC = OFF_DS + 2 * T_BYTES;  // QS x {lse2, delta, pos-k0}[BM]
  static constexpr int OFF_BAR = OFF_VEC + QS * 3 * BM * 4;
  // The dynamic-SMEM window starts 1024-B aligned on sm_100 (checked at run
  // time), so no alignment slack is reserved (D = 128: 194.75 KB).
  // (A second K buffer, so the next KV head's K lands early, measured 3-10%
  //  SLOWER on the same box: profiles/r02_ab_bwd_kdb.txt; the 227 KB carve-out
  //  leaves almost no L1 for the per-query vector loads.)
  // (the dK/dV epilogue transposes through the dS^T buffers, 4 KB per compute
  //  warp: a separate 32 KB region left almost no L1 and cost the vector
  //  loads of short per-sequence ranks 4-8 %)
  static constexpr int SMEM = OFF_BAR + 512;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t COL_S = 0;      // S^T[b] at b*64
  static constexpr uint32_t COL_DP = 128;   // dP^T[b] at 128 + b*64 (later dQ^T[b])
  static constexpr uint32_t COL_DV = 256;
  static constexpr uint32_t COL_DK = 256 + D;
  static constexpr uint32_t IDESC_ST = idesc_bf16(BN, BM, 0, 0);
  static constexpr uint32_t IDESC_ACC = idesc_bf16(BN, D, 0, 1);   // dV, dK
  static constexpr uint32_t IDESC_DQT = idesc_bf16(D, BM, 1, 1);   // dQ^T
  static constexpr int THREADS = 128 + 128 * NCW + 128;   // + dQ drain warpgroup
};

// Work units reach the roles through a small ring: the producer warp takes
// the next unit (dynamically, from a global counter, when persistent) and
// publishes its index; every consumer warp reads it and releases the slot.
constexpr int kUnitRing = 4;

struct BwdBars {  // 268 bytes; OFF_BAR reserves 512
  uint64_t kv_full, kv_empty;
  uint64_t q_full[3], q_empty[3];
  uint64_t s_full[2], p_full[2], mma2_done[2], s_free[2];
  uint64_t vec_full[3], vec_empty[3];
  uint64_t acc_done;
  uint64_t unit_full[kUnitRing], unit_empty[kUnitRing];
  int unit_id[kUnitRing];
  uint32_t tmem_base;
};
static_assert(sizeof(BwdBars) <= 512, "barrier block");
static_assert(BwdCfg<128>::SMEM <= 232448, "bwd v2 exceeds the 227 KB SMEM window");
static_assert(2 * BwdCfg<128>::T_BYTES >= 8 * 4096, "epilogue staging fits the dS^T buffers");

// dV and dK (scaled) of a warp's 32 key rows x 32 head-dims (one TMEM load
// each, lane = key row) stored through a 4 KB per-warp shared-memory
// transpose, so every store instruction writes whole 128-B lines (fp32: 8
// lanes per row, 4 rows per instruction; bf16: 4 lanes per row, 8 rows).
// Storing straight from the TMEM layout put 32 rows into each instruction,
// 16 B per line: the per-KV-head epilogue of short documents then took more
// SM time than their query tiles.  `off0` is the element offset of head-dim
// 0 of key row 0 of the block, `ld` the row stride in elements; rows at or
// past `n_rows` (keys past the tile) are not stored.
__device__ __forceinline__ void store_dkv_block(void* dv, void* dk, size_t off0, size_t ld,
                                                int n_rows, const uint32_t (&a)[32],
                                                const uint32_t (&bb)[32], float scale, bool bf16,
                                                uint4* stg) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int tsel = 0; tsel < 2; ++tsel) {
    const uint32_t(&v)[32] = tsel ? bb : a;
    const float sc = tsel ? scale : 1.f;
    void* dst = tsel ? dk : dv;
    __syncwarp();
    if (bf16) {
      // row = 16 packed bf16 pairs = 4 x 16 B chunks, chunk j at j ^ (row & 3)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        stg[lane * 4 + (j ^ (lane & 3))] =
            make_uint4(pack_bf16(__uint_as_float(v[8 * j]) * sc, __uint_as_float(v[8 * j + 1]) * sc),
                       pack_bf16(__uint_as_float(v[8 * j + 2]) * sc, __uint_as_float(v[8 * j + 3]) * sc),
                       pack_bf16(__uint_as_float(v[8 * j + 4]) * sc, __uint_as_float(v[8 * j + 5]) * sc),
                       pack_bf16(__uint_as_float(v[8 * j + 6]) * sc, __uint_as_float(v[8 * j + 7]) * sc));
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = 8 * k + (lane >> 2), c = lane & 3;
        const uint4 x = stg[r * 4 + (c ^ (r & 3))];
        if (r < n_rows)
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(dst) + off0 + r * ld + 8 * c) = x;
      }
    } else {
      // row = 8 x 16 B chunks, chunk j at j ^ (row & 7)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        stg[lane * 8 + (j ^ (lane & 7))] =
            make_uint4(__float_as_uint(__uint_as_float(v[4 * j]) * sc),
                       __float_as_uint(__uint_as_float(v[4 * j + 1]) * sc),
                       __float_as_uint(__uint_as_float(v[4 * j + 2]) * sc),
                       __float_as_uint(__uint_as_float(v[4 * j + 3]) * sc));
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int r = 4 * k + (lane >> 3), c = lane & 7;
        const uint4 x = stg[r * 8 + (c ^ (r & 7))];
        if (r < n_rows)
          *reinterpret_cast<uint4*>(reinterpret_cast<float*>(dst) + off0 + r * ld + 4 * c) = x;
      }
    }
  }
  __syncwarp();
}

// kv_tiles[2i] = {kv_begin (global), kv_len, row_first, row_end}, kv_tiles[2i+1].x = k0
//
// Work unit u = (KV tile item, KV-head group): item u % n_slots, KV heads
// [g0, g0 + nh) with g0 = (u / n_slots) * hpc (head-major unit order, LPT
// within a head: resident CTAs share one head's Q / dO / dQ in L2).  The query
// tiles of a unit's heads form one flat sequence, and the sequences of all
// the units a CTA runs are concatenated: every ring stage and barrier phase
// runs on a CTA-global tile counter, so one unit's tail (its last dK/dV
// epilogue, the next K/V load) overlaps the next unit's start.
//   persistent = 0: one unit per CTA (unit = blockIdx.x);
//   persistent = 1: one CTA per SM takes units from a global counter until
//                   none are left (dynamic list scheduling in unit order).
template <int D, int NCW>
__global__ void __launch_bounds__(256 + 128 * NCW, 1)
attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                const float* __restrict__ lse, const float* __restrict__ delta,
                float* __restrict__ dq_acc, void* __restrict__ dk, void* __restrict__ dv,
                const int4* __restrict__ kv_tiles, const int* __restrict__ n_kv_tiles,
                const int* __restrict__ positions, int Tl, int Hq, int Hkv, int n_slots, int hpc,
                int n_units, int* __restrict__ sched, int persistent, int g_begin, int g_end,
                float scale, float scale_log2, int dkv_bf16, const CpSync sync) {
  using C = BwdCfg<D, NCW>;
  extern __shared__ uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023) __trap();   // SW128 tiles need 1024-B alignment
  uint8_t* smem = smem_raw;
  const int n_items = n_kv_tiles[0];
  const int group = Hq / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  BwdBars* bars = reinterpret_cast<BwdBars*>(smem + C::OFF_BAR);
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sDO = smem + C::OFF_DO;
  uint8_t* sDS = smem + C::OFF_DS;
  float* sVec = reinterpret_cast<float*>(smem + C::OFF_VEC);

  if (threadIdx.x == 0) {
    mbar_init(&bars->kv_full, 1);
    mbar_init(&bars->kv_empty, 1);
    for (int i = 0; i < C::QS; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], 1);
      mbar_init(&bars->vec_full[i], 32);
      mbar_init(&bars->vec_empty[i], 128 * NCW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], 128 * NCW);
      mbar_init(&bars->mma2_done[i], 1);
      mbar_init(&bars->s_free[i], 128);
    }
    mbar_init(&bars->acc_done, 1);
    for (int i = 0; i < kUnitRing; ++i) {
      mbar_init(&bars->unit_full[i], 1);
      // consumers: MMA warp, vector warp, 4 drain warps, 4 * NCW compute warps
      mbar_init(&bars->unit_empty[i], 2 + 4 + 4 * NCW);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&bars->tmem_base, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  // unit geometry (every role derives the same from the unit index)
  struct Unit {
    int4 kt;        // {kv_begin, kv_len, row_first, row_end}
    int k0, g0, nh, qt_per_head, n_iter, n_all;
  };
  auto geom = [&](int u) {
    Unit U;
    const int item = u % n_slots;
    U.kt = kv_tiles[2 * item];
    U.k0 = kv_tiles[2 * item + 1].x;   // in-document position of key 0 of the tile
    U.g0 = g_begin + (u / n_slots) * hpc;   // KV heads [g_begin, g_end) of this launch
    U.nh = min(hpc, g_end - U.g0);
    U.qt_per_head = (U.kt.w - U.kt.z + C::BM - 1) / C::BM;
    U.n_iter = U.qt_per_head * group;  // query tiles per KV head
    // unit invariants: a non-empty row suffix inside [0, Tl), 1..128 keys of
    // one document from position k0, KV heads inside the launch's range
    WLB_DCHECK(U.kt.z >= 0 && U.kt.z < U.kt.w && U.kt.w <= Tl);
    WLB_DCHECK(U.kt.y >= 1 && U.kt.y <= C::BN && U.kt.x >= 0 && U.k0 >= 0);
    WLB_DCHECK(U.g0 >= g_begin && U.nh >= 1 && U.g0 + U.nh <= g_end && g_end <= Hkv);
    U.n_all = U.n_iter * U.nh;
    return U;
  };
  // unit-local flat tile I -> (KV head, query head, first row)
  auto tile_g = [&](const Unit& U, int I) { return U.g0 + I / U.n_iter; };
  auto tile_h = [&](const Unit& U, int I) {
    return tile_g(U, I) * group + (WLB_BWD_HEAD_INNER ? (I % U.n_iter) % group
                                                      : (I % U.n_iter) / U.qt_per_head);
  };
  auto tile_row = [&](const Unit& U, int I) {
    return U.kt.z + (WLB_BWD_HEAD_INNER ? (I % U.n_iter) / group
                                        : (I % U.n_iter) % U.qt_per_head) * C::BM;
  };
  // consumer side of the unit ring (whole warp; lane 0 releases the slot)
  auto next_unit = [&](int seq) {
    const int st = seq % kUnitRing;
    mbar_wait(&bars->unit_full[st], (seq / kUnitRing) & 1);
    const int u = *reinterpret_cast<volatile int*>(&bars->unit_id[st]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->unit_empty[st]);
    return u;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer --
    // whole warp; one elected lane issues.  I0 / G0: tiles / KV heads of the
    // units this CTA already ran (ring stages and barrier phases run on).
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmDO);
    int I0 = 0, G0 = 0;
    for (int seq = 0;; ++seq) {
      int u = -1;
      if (lane == 0) {
        if (persistent) {
          do {
            u = atomicAdd(sched, 1);
          } while (u < n_units && u % n_slots >= n_items);
          if (u >= n_units) u = -1;
        } else if (seq == 0 && (int)blockIdx.x % n_slots < n_items) {
          u = blockIdx.x;
        }
        const int st = seq % kUnitRing;
        mbar_wait(&bars->unit_empty[st], ((seq / kUnitRing) & 1) ^ 1);
        bars->unit_id[st] = u;
        mbar_arrive(&bars->unit_full[st]);
      }
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u < 0) break;
      const Unit U = geom(u);
      for (int I = 0; I < U.n_all; ++I) {
        if (I % U.n_iter == 0) {            // next KV head: K/V once the last reader is done
          const int gl = I / U.n_iter, G = G0 + gl;
          if (G > 0) mbar_wait(&bars->kv_empty, (G - 1) & 1);
          mbar_expect_tx_w(&bars->kv_full, 2 * C::KV_BYTES);
          for (int s = 0; s < C::SLABS; ++s) {
            tma_load_3d_w(sK + s * C::KV_SLAB, &tmK, &bars->kv_full, s * 64, U.g0 + gl, U.kt.x);
            tma_load_3d_w(sV + s * C::KV_SLAB, &tmV, &bars->kv_full, s * 64, U.g0 + gl, U.kt.x);
          }
        }
        const int Ig = I0 + I, st = Ig % C::QS;
        const int h = tile_h(U, I), row = tile_row(U, I);
        mbar_wait(&bars->q_empty[st], ((Ig / C::QS) & 1) ^ 1);
        mbar_expect_tx_w(&bars->q_full[st], 2 * C::Q_BYTES);
        for (int s = 0; s < C::SLABS; ++s) {
          tma_load_3d_w(sQ + st * C::Q_BYTES + s * C::Q_SLAB, &tmQ, &bars->q_full[st], s * 64, h, row);
          tma_load_3d_w(sDO + st * C::Q_BYTES + s * C::Q_SLAB, &tmDO, &bars->q_full[st], s * 64, h,
                        row);
        }
      }
      I0 += U.n_all;
      G0 += U.nh;
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer --
    // whole warp; one elected lane issues
    const uint32_t k_b = smem_u32(sK), v_b = smem_u32(sV), q_b = smem_u32(sQ),
                   do_b = smem_u32(sDO), ds_b = smem_u32(sDS);
    int I0 = 0, G0 = 0;
    for (int seq = 0;; ++seq) {
      const int u = next_unit(seq);
      if (u < 0) break;
      const Unit U = geom(u);
      // S^T / dP^T of tile I (first MMA group)
      auto first_half = [&](int I) {
        const int Ig = I0 + I;
        const int b = Ig & 1, st = Ig % C::QS;
        mbar_wait(&bars->q_full[st], (Ig / C::QS) & 1);
        TRACE(0, Ig);
        tc_fence_after();
        const uint32_t qs = q_b + st * C::Q_BYTES, dos = do_b + st * C::Q_BYTES;
        // S^T[b] was last read by the compute warps of tile I-2 (before p_full,
        // already waited); dP^T[b] also held dQ^T of tile I-2, so only the dP
        // half waits for the drain warps.
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {   // contract over D: K-major both
          const uint32_t ko = (kk >> 2) * C::KV_SLAB + (kk & 3) * 32;
          const uint32_t qo = (kk >> 2) * C::Q_SLAB + (kk & 3) * 32;
          mma_ss_w(tmem + C::COL_S + b * 64, sdesc_sw128(k_b + ko, 16, 1024),
                   sdesc_sw128(qs + qo, 16, 1024), C::IDESC_ST, kk > 0);
        }
        if (Ig >= 2) mbar_wait_fast(&bars->s_free[b], ((Ig - 2) >> 1) & 1);
        TRACE(1, Ig);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * C::KV_SLAB + (kk & 3) * 32;
          const uint32_t qo = (kk >> 2) * C::Q_SLAB + (kk & 3) * 32;
          mma_ss_w(tmem + C::COL_DP + b * 64, sdesc_sw128(v_b + ko, 16, 1024),
                   sdesc_sw128(dos + qo, 16, 1024), C::IDESC_ST, kk > 0);
        }
        mma_commit_w(&bars->s_full[b]);
      };
      // dQ^T, dV, dK of tile J (second MMA group)
      auto second_half = [&](int J) {
        const int Jg = I0 + J;
        const int b = Jg & 1, st = Jg % C::QS, j = J % U.n_iter;
        mbar_wait_fast(&bars->p_full[b], (Jg >> 1) & 1);
        TRACE(2, Jg);
        tc_fence_after();
        const uint32_t qs = q_b + st * C::Q_BYTES, dos = do_b + st * C::Q_BYTES;
        const uint32_t dss = ds_b + b * C::T_BYTES;
        // dQ^T first: it lands in the dP^T[b] columns (free once the compute
        // warps loaded dP^T), so the drain of tile J overlaps dV/dK(J) and
        // S(J+2) instead of stalling dP(J+2).
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {   // contract over keys
          mma_ss_w(tmem + C::COL_DP + b * 64, sdesc_sw128(k_b + kk * 2048, C::KV_SLAB, 1024),
                   sdesc_sw128(dss + kk * 2048, C::KV_SLAB, 1024), C::IDESC_DQT, kk > 0);
        }
        mma_commit_w(&bars->mma2_done[b]);
        // P^T / dS^T (packed bf16) sit in the S^T[b] columns: queries
        // [32c, 32c+32) at column 32c (P) and 32c+16 (dS), 8 columns per K16
#pragma unroll
        for (int kk = 0; kk < C::BM / 16; ++kk) {   // contract over queries (A from TMEM)
          const uint32_t acc = (j > 0) || (kk > 0);
          const uint32_t ca = C::COL_S + b * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
          mma_ts_w(tmem + C::COL_DV, tmem + ca,
                   sdesc_sw128(dos + kk * 2048, C::Q_SLAB, 1024), C::IDESC_ACC, acc);
          mma_ts_w(tmem + C::COL_DK, tmem + ca + 16,
                   sdesc_sw128(qs + kk * 2048, C::Q_SLAB, 1024), C::IDESC_ACC, acc);
        }
        mma_commit_w(&bars->q_empty[st]);
        if (j == U.n_iter - 1) {                  // last tile of this KV head
          mma_commit_w(&bars->acc_done);
          mma_commit_w(&bars->kv_empty);
        }
      };
      // Pipelined one tile deep (S/dP of tile I before dQ/dV/dK of tile I-1),
      // except across a KV-head (or unit) boundary: tile I of the next head
      // needs the new K/V, which may only land after the last reader of the
      // old ones.
      for (int I = 0; I <= U.n_all; ++I) {
        const bool head_start = I < U.n_all && I % U.n_iter == 0;
        if (I < U.n_all && !head_start) first_half(I);
        if (I >= 1) second_half(I - 1);
        if (head_start) {
          mbar_wait(&bars->kv_full, (G0 + I / U.n_iter) & 1);
          first_half(I);
        }
      }
      I0 += U.n_all;
      G0 += U.nh;
    }
  } else if (warp == 3) {
    // ------------------------------------------------- per-query vectors --
    int I0 = 0;
    for (int seq = 0;; ++seq) {
      const int u = next_unit(seq);
      if (u < 0) break;
      const Unit U = geom(u);
      for (int I = 0; I < U.n_all; ++I) {
        const int Ig = I0 + I, b = Ig % C::QS;
        const int h = tile_h(U, I), row0 = tile_row(U, I);
        mbar_wait(&bars->vec_empty[b], ((Ig / C::QS) & 1) ^ 1);
        float* vec = sVec + b * 3 * C::BM;
#pragma unroll
        for (int e = lane; e < C::BM; e += 32) {
          const int row = row0 + e;
          const bool ok = row < U.kt.w;
          vec[e] = ok ? lse[(size_t)h * Tl + row] * 1.4426950408889634f : 0.f;
          vec[C::BM + e] = ok ? delta[(size_t)h * Tl + row] : 0.f;
          reinterpret_cast<int*>(vec)[2 * C::BM + e] = ok ? positions[row] - U.k0 : -1;
        }
        mbar_arrive(&bars->vec_full[b]);
      }
      I0 += U.n_all;
    }
  } else if (warp >= 4 + 4 * NCW) {
    // ------------------------------------------------------------ dQ drain --
    // dQ^T lanes are head-dim rows (lane = d for D = 128; for D = 64 the M=64
    // accumulator uses lanes 0-15 of each quarter).  Each warp-wide RED covers
    // 32 consecutive floats of one query row.  Kept off the compute warps so
    // their proxy fences never wait on outstanding global reductions.
    const int lg = warp & 3;
    const uint32_t lane_base = tmem + ((uint32_t)(lg * 32) << 16);
    const int d = D == 128 ? lg * 32 + lane : lg * 16 + lane;
    const size_t stride = (size_t)Hq * D;
    int I0 = 0;
    for (int seq = 0;; ++seq) {
      const int u = next_unit(seq);
      if (u < 0) break;
      const Unit U = geom(u);
      for (int J = 0; J < U.n_all; ++J) {
        const int Jg = I0 + J, b = Jg & 1;
        const int h = tile_h(U, J), row0 = tile_row(U, J);
        mbar_wait(&bars->mma2_done[b], (Jg >> 1) & 1);
        TRACE(6, Jg);
        tc_fence_after();
        uint32_t v[64];
        tmem_ld32(lane_base + C::COL_DP + b * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
        tmem_ld32(lane_base + C::COL_DP + b * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars->s_free[b]);
        TRACE(7, Jg);
        if (D == 128 || lane < 16) {
          float* ptr = dq_acc + ((size_t)row0 * Hq + h) * D + d;
          const int nvalid = min(C::BM, U.kt.w - row0);
          if (nvalid == C::BM) {
#pragma unroll
            for (int q = 0; q < C::BM; ++q, ptr += stride) atomicAdd(ptr, __uint_as_float(v[q]) * scale);
          } else {
#pragma unroll
            for (int q = 0; q < C::BM; ++q, ptr += stride)
              if (q < nvalid) atomicAdd(ptr, __uint_as_float(v[q]) * scale);
          }
        }
      }
      I0 += U.n_all;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- compute --
    const int lg = warp & 3;                 // TMEM lane quarter
    const int ch = (warp - 4) >> 2;          // which 32-column half of the 64 queries
    const int t = lg * 32 + lane;            // key row in the tile
    const uint32_t lane_base = tmem + ((uint32_t)(lg * 32) << 16);
    int I0 = 0, G0 = 0;
    for (int seq = 0;; ++seq) {
      const int u = next_unit(seq);
      if (u < 0) break;
      const Unit U = geom(u);
      const bool key_ok = t < U.kt.y;
      for (int I = 0; I < U.n_all; ++I) {
        const int Ig = I0 + I;
        const int b = Ig & 1, vb = Ig % C::QS;
        mbar_wait(&bars->vec_full[vb], (Ig / C::QS) & 1);
        mbar_wait(&bars->s_full[b], (Ig >> 1) & 1);
        TRACE(3, Ig);
        tc_fence_after();
        uint32_t us[32], ud[32];
        tmem_ld32(lane_base + C::COL_S + b * 64 + ch * 32, us);
        tmem_ld32(lane_base + C::COL_DP + b * 64 + ch * 32, ud);
        const float* vec = sVec + vb * 3 * C::BM + ch * 32;
        const float4* vl4 = reinterpret_cast<const float4*>(vec);
        const float4* vd4 = reinterpret_cast<const float4*>(vec + C::BM);
        const int4* vp4 = reinterpret_cast<const int4*>(vec + 2 * C::BM);
        // Unmasked fast path: every query of this half sees every key of the tile
        // (rows are position-sorted, so the first and last columns bound them).
        const bool full = U.kt.y == C::BN && vp4[0].x >= C::BN - 1 && vp4[7].w >= C::BN - 1;
        tmem_ld_wait();
        TRACE(4, Ig);
        uint32_t pk[16], dk2[16];
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          const float4 l4 = vl4[e4], d4 = vd4[e4];
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dv4[4] = {d4.x, d4.y, d4.z, d4.w};
          float pp[4], dd[4];
          if (full) {
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              pp[x] = ex2(fmaf(__uint_as_float(us[4 * e4 + x]), scale_log2, -lv[x]));
              dd[x] = pp[x] * (__uint_as_float(ud[4 * e4 + x]) - dv4[x]);
            }
          } else {
            const int4 p4 = vp4[e4];
            const int pv[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const bool allowed = key_ok && pv[x] >= t;   // key position k0+t <= query position
              const float y = fmaf(__uint_as_float(us[4 * e4 + x]), scale_log2, -lv[x]);
              pp[x] = allowed ? ex2(y) : 0.f;
              dd[x] = pp[x] * (__uint_as_float(ud[4 * e4 + x]) - dv4[x]);
            }
          }
          pk[2 * e4] = pack_bf16(pp[0], pp[1]);
          pk[2 * e4 + 1] = pack_bf16(pp[2], pp[3]);
          dk2[2 * e4] = pack_bf16(dd[0], dd[1]);
          dk2[2 * e4 + 1] = pack_bf16(dd[2], dd[3]);
        }
        tc_fence_before();
        mbar_arrive(&bars->vec_empty[vb]);
        // P^T and dS^T (packed bf16) over THIS warp's own 32 S^T columns (no
        // other warp reads them): A operands of the TS dV / dK MMAs.  The
        // previous readers (dV/dK of tile I-2) finished before MMA1(I)
        // (s_full implies it).  dP^T[b] is free once loaded: dQ^T(I) goes
        // there.  dS^T also goes to SMEM as the B operand of dQ^T = K^T dS^T.
        tmem_st16(lane_base + C::COL_S + b * 64 + ch * 32, pk);
        tmem_st16(lane_base + C::COL_S + b * 64 + ch * 32 + 16, dk2);
        uint8_t* drow = sDS + b * C::T_BYTES + t * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int off = (((ch * 4 + c) ^ (t & 7)) << 4);
          *reinterpret_cast<uint4*>(drow + off) = make_uint4(dk2[4 * c], dk2[4 * c + 1], dk2[4 * c + 2], dk2[4 * c + 3]);
        }
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        TRACE(5, Ig);
        mbar_arrive(&bars->p_full[b]);
        if (I % U.n_iter == U.n_iter - 1) {
          // -------------------------------------------------------- epilogue --
          // the last MMA group of this KV head wrote dV / dK; the next head's
          // (or unit's) first dV/dK MMA (accumulate = 0) waits for this warp's
          // next p_full, i.e. for these TMEM loads
          const int g = tile_g(U, I);
          mbar_wait(&bars->acc_done, (G0 + I / U.n_iter) & 1);
          tc_fence_after();
          // TMEM loads are warp-collective: issue converged, predicate the stores.
          // the warp's 32 key rows from the block's first (lg * 32)
          const size_t off = ((size_t)(U.kt.x + lg * 32) * Hkv + g) * D + ch * (D / 2);
          // staging: the dS^T buffers (their last reader, this head's last dQ^T
          // MMA, completed before acc_done; the next tile's dS^T is written
          // after this epilogue, by these warps)
          uint4* stg = reinterpret_cast<uint4*>(sDS + (warp - 4) * 4096);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) {
            uint32_t a[32], bb[32];
            tmem_ld32(lane_base + C::COL_DV + ch * (D / 2) + c * 32, a);
            tmem_ld32(lane_base + C::COL_DK + ch * (D / 2) + c * 32, bb);
            tmem_ld_wait();
            store_dkv_block(dv, dk, off + c * 32, (size_t)Hkv * D, U.kt.y - lg * 32, a, bb, scale,
                            dkv_bf16 != 0, stg);
          }
          tc_fence_before();
          if (sync.signal_bases && I == U.n_all - 1) {
            // CP: the unit's partials are stored (all compute warps); count it
            // toward its head group and publish the group when complete
            named_bar_sync(1, 128 * NCW);
            if (warp == 4 && lane == 0)
              cp_sync_unit_done(sync, U.g0 / sync.kv_per_group,
                                n_items * (sync.kv_per_group / hpc));
          }
        }
      }
      I0 += U.n_all;
      G0 += U.nh;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, C::TMEM_COLS);
}

// ---------------------------------------------------------------------------
// v3 (D = 128): 128-query tiles, every MMA N = 128.
//
// The v2 kernel above is bound by shared-memory operand bandwidth (128 B/clk
// per SM): its N = 64 SS MMAs re-read the 32 KB K / V / K^T operands once per
// 64 queries.  Here a tile has 128 queries, so each of S^T, dP^T and dQ is
// one M=128 N=128 MMA chain (full rate) and the A operands are re-read half as
// often.  TMEM (512 columns) then holds exactly one S^T and one dP^T:
//
//   [0,128)   S^T (fp32) -> P^T (bf16, columns 64c..64c+32 for query half c,
//             written by the warps that read those S^T columns)
//   [128,256) dP^T (fp32) -> dQ (fp32, lanes = queries) once the compute
//             warps have read dP^T
//   [256,384) dV, [384,512) dK accumulators
//   dS^T lives in SMEM only (B of dQ = dS K, A of dK += dS^T Q).
//
// Tensor-pipe order (see the MMA issuer): ... dV(i-1) | S(i) | dQ(i-1) |
// dK(i-1) | dP(i) | dV(i) | S(i+1) ...  With no double buffering the compute
// warps hide inside it instead:
//   * P(i) is computed under dQ(i-1), dK(i-1) and dP(i), and handed over in
//     two 32-query chunks (p_full[c]) so dV(i) starts on chunk 0;
//   * dS(i) is computed under dV(i) and S(i+1), again in two chunks;
//   * the dQ drain warps load dQ(i-1) under dK(i-1) (s_free gates dP(i)) and
//     pace its 16-B reductions over the next tile.
// PAIR = true is the experimental 2-CTA-cluster variant (off by default).
// ---------------------------------------------------------------------------
#ifdef WLB_TRACE
__device__ long long g_bwd3_trace[2][16][128];   // CTAs 0 and 1 (a cluster pair)
#define TRACE3(ev, i)                                                             \
  do {                                                                            \
    if (blockIdx.x < 2 && (i) < 128 && (threadIdx.x & 31) == 0)                   \
      g_bwd3_trace[blockIdx.x][ev][i] = clock64();                                \
  } while (0)
#else
#define TRACE3(ev, i) \
  do {                \
  } while (0)
#endif

struct Bwd3Cfg {
  static constexpr int D = 128, BM = 128, BN = 128;
  static constexpr int KV_BYTES = BN * D * 2, Q_BYTES = BM * D * 2, T_BYTES = BN * BM * 2;
  static constexpr int SLAB = 128 * 128;   // 128 rows x 128 B (64 bf16) swizzle slab
  static constexpr int QS = 2;             // Q/dO + query-vector ring depth
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV_BYTES;
  static constexpr int OFF_Q = OFF_V + KV_BYTES;
  static constexpr int OFF_DO = OFF_Q + QS * Q_BYTES;
  static constexpr int OFF_DS = OFF_DO + QS * Q_BYTES;              // dS^T, 2 query slabs
  static constexpr int OFF_VEC = OFF_DS + T_BYTES;                  // QS x {-lse2, delta}[BM] f32
  static constexpr int OFF_POS = OFF_VEC + QS * 2 * BM * 4;         // QS x rel. position[BM] i8
  static constexpr int OFF_BAR = OFF_POS + QS * BM;
  static constexpr int SMEM = OFF_BAR + 512;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 384;
  static constexpr uint32_t IDESC_ST = idesc_bf16(BN, BM, 0, 0);    // S^T, dP^T
  static constexpr uint32_t IDESC_ACC = idesc_bf16(BN, D, 0, 1);    // dV, dK
  static constexpr uint32_t IDESC_DQ = idesc_bf16(BM, D, 1, 1);     // dQ
  static constexpr int THREADS = 512;
};
static_assert(Bwd3Cfg::SMEM <= 232448, "bwd v3 exceeds the 227 KB SMEM window");

struct Bwd3Bars {
  uint64_t kv_full, kv_empty;
  uint64_t unit_full[kUnitRing], unit_empty[kUnitRing];
  int unit_id[kUnitRing];
  uint64_t q_full[2], q_empty[2], vec_full[2], vec_empty[2];
  uint64_t s_full, dp_full, p_full[2], ds_full[2], dq_full, s_free, acc_done;
  uint64_t do_full, do_empty, rx_full[4], peer_free;   // PAIR: single dO buffer, dQ exchange
  uint32_t tmem_base;
};
static_assert(sizeof(Bwd3Bars) <= 512, "barrier block");

#ifndef WLB_BWD_V3
#define WLB_BWD_V3 1     // 0: D = 128 always uses the v2 (64-query) kernel
#endif
// v3 wins on long row-sets and, since its dQ partials leave by TMA
// reduce-adds (TRED), both kernels store dK/dV as whole lines and v3 runs as a
// persistent kernel, on every document length measured (128-row documents 98
// vs 93 TFLOP/s, 256: 189 vs 156, 384: 271 vs 216; GQA 256: 254 vs 203;
// config-5 short ranks +15 %: profiles/r02_ab_bwd3_persistent.txt), so D = 128
// always uses it (threshold 1 local row per document); the 64-query kernel
// serves D = 64 and remains selectable (wlb_attn_bwd_select).
#ifndef WLB_BWD_V3_MIN_ROWS
#define WLB_BWD_V3_MIN_ROWS 1
#endif
#ifndef WLB_RED_B0          // dQ reduction batches (v4 REDs per thread, of 32)
#define WLB_RED_B0 8
#endif
#ifndef WLB_RED_B1
#define WLB_RED_B1 8
#endif
#ifndef WLB_RED_B2
#define WLB_RED_B2 8
#endif
#ifndef WLB_RED_PACE
#define WLB_RED_PACE 0   // 0: dQ reductions paced by pipeline barriers; N: N batches + nanosleep
#endif
#ifndef WLB_RED_SLEEP
#define WLB_RED_SLEEP 150
#endif
#ifndef WLB_TRED_PACE
#define WLB_TRED_PACE 1   // TMA dQ reduces paced by the next tile's barriers (0: at once)
#endif
#ifndef WLB_BWD_POLY
#define WLB_BWD_POLY 0   // column pairs (of every 8) whose exp2 runs on the FMA pipe
#endif

// P for one 32-query chunk of one key row: p = exp2(s * scale_log2 + nl[q]),
// zero where the key is past the row's position (MASK) -> packed bf16 pairs
// (pk: the A operand of dV += P^T dO) and packed fp16 pairs (ph: kept in
// registers for dS = P (dP - Delta)).  P is in [0, 1], where fp16 keeps 3
// more mantissa bits than bf16: forming dS from the bf16 P rounded P twice
// (P, then dS) and put the GQA dK (summed over 8 query heads x 32K queries)
// past the 2e-2 + 1e-2|ref| bar; with fp16 P its error matches the 64-query
// kernel's, which multiplies the fp32 P.
template <bool MASK, bool P16>
__device__ __forceinline__ void bwd3_p_chunk(const uint32_t (&us)[32], const float* nl,
                                             const int8_t* rp, int t, bool key_ok,
                                             float scale_log2, uint32_t (&pk)[16],
                                             uint32_t (&ph)[16]) {
  const float2 sc2 = make_float2(scale_log2, scale_log2);
  const float4* n4 = reinterpret_cast<const float4*>(nl);
  int8_t pos[32];
  if (MASK) {
    *reinterpret_cast<int4*>(pos) = reinterpret_cast<const int4*>(rp)[0];
    *reinterpret_cast<int4*>(pos + 16) = reinterpret_cast<const int4*>(rp)[1];
  }
#pragma unroll
  for (int e4 = 0; e4 < 8; ++e4) {
    const float4 l4 = n4[e4];
#pragma unroll
    for (int u2 = 0; u2 < 2; ++u2) {
      const int e = 4 * e4 + 2 * u2;
      const float2 x = ffma2(make_float2(__uint_as_float(us[e]), __uint_as_float(us[e + 1])), sc2,
                             u2 ? make_float2(l4.z, l4.w) : make_float2(l4.x, l4.y));
      float2 pp;
      if (((e >> 1) & 7) < WLB_BWD_POLY) {
        pp = ex2_poly2(x);
      } else {
        pp.x = ex2(x.x);
        pp.y = ex2(x.y);
      }
      if (MASK) {
        pp.x = (key_ok && pos[e] >= t) ? pp.x : 0.f;
        pp.y = (key_ok && pos[e + 1] >= t) ? pp.y : 0.f;
      }
      pk[e >> 1] = pack_bf16(pp.x, pp.y);
      ph[e >> 1] = P16 ? pack_f16(pp.x, pp.y) : pk[e >> 1];
    }
  }
}

// P16: dS from the fp16 copy of P (GQA, where dK sums over the group's query
// heads and the bf16 double rounding of P failed the bar); otherwise from the
// bf16 P the dV MMA reads (one conversion fewer per pair on the compute warps,
// within the bar for Hq = Hkv: tests/test_gpu_scale.py).
// TRED: the dQ drain stages each warp's 32 x 128 fp32 partial in shared memory
// (the second dO stage: dO is single-buffered as in PAIR) and reduces it into
// dq_acc with TMA tile reduce-adds (4 boxes of 32 rows x 32 head-dims per
// warp and tile) instead of 32 per-thread RED.v4, taking the reduction off the
// SM's load/store queues that the compute warps' TMEM loads share.
template <bool PAIR, bool P16, bool TRED = false>
__global__ void __launch_bounds__(512, 1)
attn_bwd3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                 const __grid_constant__ CUtensorMap tmDQ,
                 const float* __restrict__ lse, const float* __restrict__ delta,
                 float* __restrict__ dq_acc, void* __restrict__ dk, void* __restrict__ dv,
                 const int4* __restrict__ kv_tiles, const int* __restrict__ n_kv_tiles,
                 const int* __restrict__ positions, int Tl, int Hq, int Hkv, int n_slots,
                 int g_begin, float scale, float scale_log2, int dkv_bf16, int n_units,
                 int* __restrict__ sched, int persistent, const CpSync sync) {
  using C = Bwd3Cfg;
  constexpr int D = C::D;
  extern __shared__ uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023) __trap();
  uint8_t* smem = smem_raw;
  // PAIR: a 2-CTA cluster runs KV tiles 2q and 2q+1 of one document over the
  // same query tiles (kv_tiles holds pair items: {kv_begin, kv_len, row_first,
  // row_end} of tile 2q, then {k0, kv_begin', kv_len', k0'} with kv_begin' < 0
  // for a lone last tile); each CTA reduces half of the pair's summed dQ.
  const int cta = PAIR ? (int)cluster_ctarank() : 0;
  const int n_items = n_kv_tiles[0];
  const int group = Hq / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Work unit u = (KV tile item u % n_slots, KV head g_begin + u / n_slots):
  // one per CTA (blockIdx.x; PAIR: per cluster), or, persistent, one CTA per
  // SM taking units from a global counter (dynamic list scheduling in unit
  // order, LPT within a head) and publishing them to its warps through a
  // ring; every ring stage and barrier phase runs on CTA-global tile / unit
  // counters, so a unit's epilogue overlaps the next unit's loads and first
  // MMAs instead of a CTA teardown and launch.
  bool paired = false;
  if (PAIR) {
    const int item = (int)(blockIdx.x >> 1) % n_slots;
    if (item >= n_items) return;
    paired = kv_tiles[2 * item + 1].y >= 0;
    if (!paired && cta == 1) return;         // lone tile: CTA 1 idles, CTA 0 runs solo
  } else if (!persistent && (int)blockIdx.x % n_slots >= n_items) {
    return;
  }
  struct Unit3 {
    int4 kt;   // {kv_begin, kv_len, row_first, row_end}
    int k0, g, qt, n_iter;
  };
  // PAIR: a 2-CTA cluster runs KV tiles 2q and 2q+1 of one document over the
  // same query tiles (kv_tiles holds pair items: {kv_begin, kv_len, row_first,
  // row_end} of tile 2q, then {k0, kv_begin', kv_len', k0'} with kv_begin' < 0
  // for a lone last tile); each CTA reduces half of the pair's summed dQ.
  auto geom = [&](int u) {
    Unit3 U;
    const int item = u % n_slots;
    U.g = g_begin + u / n_slots;
    U.kt = kv_tiles[2 * item];
    U.k0 = kv_tiles[2 * item + 1].x;
    if (PAIR && cta == 1) {
      const int4 t2 = kv_tiles[2 * item + 1];
      U.kt.x = t2.y;
      U.kt.y = t2.z;
      U.k0 = t2.w;
    }
    WLB_DCHECK(U.kt.z >= 0 && U.kt.z < U.kt.w && U.kt.w <= Tl && U.kt.y >= 1 && U.kt.y <= 128 &&
               U.k0 >= 0);
    WLB_DCHECK(U.g >= 0 && U.g < Hkv);
    U.qt = (U.kt.w - U.kt.z + C::BM - 1) / C::BM;
    U.n_iter = U.qt * group;
    return U;
  };
  const int first_unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;

  Bwd3Bars* bars = reinterpret_cast<Bwd3Bars*>(smem + C::OFF_BAR);
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sDO = smem + C::OFF_DO;
  uint8_t* sDS = smem + C::OFF_DS;
  float* sVec = reinterpret_cast<float*>(smem + C::OFF_VEC);
  int8_t* sPos = reinterpret_cast<int8_t*>(smem + C::OFF_POS);

  if (threadIdx.x == 0) {
    mbar_init(&bars->kv_full, 1);
    for (int i = 0; i < C::QS; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], 1);
      mbar_init(&bars->vec_full[i], 32);
      mbar_init(&bars->vec_empty[i], 256);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    for (int c = 0; c < 2; ++c) {
      mbar_init(&bars->p_full[c], 256);
      mbar_init(&bars->ds_full[c], 256);
    }
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->s_free, 128);
    mbar_init(&bars->acc_done, 1);
    mbar_init(&bars->do_full, 1);
    mbar_init(&bars->do_empty, 1);
    for (int c = 0; c < 4; ++c) mbar_init(&bars->rx_full[c], 128);
    mbar_init(&bars->peer_free, 128);
    mbar_init(&bars->kv_empty, 1);
    for (int i = 0; i < kUnitRing; ++i) {
      mbar_init(&bars->unit_full[i], 1);
      // consumers: MMA warp, vector warp, 4 drain warps, 8 compute warps
      mbar_init(&bars->unit_empty[i], 14);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&bars->tmem_base, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  if (PAIR && paired) cluster_sync();       // peer barriers initialised before remote use

  // consumer side of the unit ring (whole warp; lane 0 releases the slot)
  auto next_unit = [&](int seq) {
    const int st = seq % kUnitRing;
    mbar_wait(&bars->unit_full[st], (seq / kUnitRing) & 1);
    const int u = *reinterpret_cast<volatile int*>(&bars->unit_id[st]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->unit_empty[st]);
    return u;
  };
  if (warp < 4) setmaxnreg_dec<80>();   // TMA / MMA / alloc / vector warps
  if (warp == 0) {
    // ------------------------------------------------------------ producer --
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmDO);
    int I0 = 0;
    for (int seq = 0;; ++seq) {
    int u = -1;
    if (lane == 0) {
      if (persistent) {
        do {
          u = atomicAdd(sched, 1);
        } while (u < n_units && u % n_slots >= n_items);
        if (u >= n_units) u = -1;
      } else if (seq == 0) {
        u = first_unit;
      }
      const int st = seq % kUnitRing;
      mbar_wait(&bars->unit_empty[st], ((seq / kUnitRing) & 1) ^ 1);
      bars->unit_id[st] = u;
      mbar_arrive(&bars->unit_full[st]);
      if (!PAIR) TRACE3(14, I0);   // unit fetched (trace builds)
    }
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u < 0) break;
    const Unit3 U = geom(u);
    const int4 kt = U.kt;
    const int g = U.g, qt_per_head = U.qt, n_iter = U.n_iter;
    // (persistent & 2) this unit is taken ~2 query tiles before the previous
    // one ends: warm L2 with its K / V tile and first Q / dO tile, so the loads
    // issued after kv_empty hit L2 instead of HBM at the unit boundary
    if (seq > 0 && (persistent & 2)) {
      for (int s = 0; s < 2; ++s) {
        tma_prefetch_3d_w(&tmK, s * 64, g, kt.x);
        tma_prefetch_3d_w(&tmV, s * 64, g, kt.x);
        tma_prefetch_3d_w(&tmQ, s * 64, g * group, kt.z);
        tma_prefetch_3d_w(&tmDO, s * 64, g * group, kt.z);
      }
    }
    // K/V of this unit once the previous unit's last MMAs have read the old
    if (seq > 0) mbar_wait(&bars->kv_empty, (seq - 1) & 1);
    if (!PAIR) TRACE3(12, I0);   // K / V buffers free (trace builds)
    mbar_expect_tx_w(&bars->kv_full, 2 * C::KV_BYTES);
    for (int s = 0; s < 2; ++s) {
      tma_load_3d_w(sK + s * C::SLAB, &tmK, &bars->kv_full, s * 64, g, kt.x);
      tma_load_3d_w(sV + s * C::SLAB, &tmV, &bars->kv_full, s * 64, g, kt.x);
    }
    for (int i = 0; i < n_iter; ++i) {
      const int Ig = I0 + i;
      const int st = Ig % C::QS;
      const int h = g * group + (WLB_BWD_HEAD_INNER ? i % group : i / qt_per_head);
      const int row = kt.z + (WLB_BWD_HEAD_INNER ? i / group : i % qt_per_head) * C::BM;
      mbar_wait(&bars->q_empty[st], ((Ig / C::QS) & 1) ^ 1);
      if (PAIR || TRED) {
        // dO single-buffered (its second stage is the dQ exchange buffer): it
        // is read by dP(i) and dV(i) only, and dO(i+1) has S(i+1), dQ(i) and
        // dK(i) to land in
        mbar_expect_tx_w(&bars->q_full[st], C::Q_BYTES);
        for (int s = 0; s < 2; ++s)
          tma_load_3d_w(sQ + st * C::Q_BYTES + s * C::SLAB, &tmQ, &bars->q_full[st], s * 64, h, row);
        mbar_wait(&bars->do_empty, (Ig & 1) ^ 1);
        mbar_expect_tx_w(&bars->do_full, C::Q_BYTES);
        for (int s = 0; s < 2; ++s)
          tma_load_3d_w(sDO + s * C::SLAB, &tmDO, &bars->do_full, s * 64, h, row);
      } else {
        mbar_expect_tx_w(&bars->q_full[st], 2 * C::Q_BYTES);
        for (int s = 0; s < 2; ++s) {
          tma_load_3d_w(sQ + st * C::Q_BYTES + s * C::SLAB, &tmQ, &bars->q_full[st], s * 64, h, row);
          tma_load_3d_w(sDO + st * C::Q_BYTES + s * C::SLAB, &tmDO, &bars->q_full[st], s * 64, h, row);
        }
      }
    }
    I0 += n_iter;
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer --
    // Tensor-pipe order (steady state):
    //   ... dV(i-1) | S(i) | dQ(i-1) | dK(i-1) | dP(i) | dV(i) | S(i+1) | ...
    // so P(i) is computed under dQ(i-1), dK(i-1) and dP(i), dS(i) under dV(i)
    // and S(i+1), and the dQ(i-1) drain under dK(i-1).  S(i) may overwrite the
    // S^T columns as soon as dV(i-1) has read P^T(i-1) (same in-order pipe):
    // dS^T lives only in SMEM, and dK reads it from there (SS MMA).
    const uint32_t k_b = smem_u32(sK), v_b = smem_u32(sV), q_b = smem_u32(sQ),
                   do_b = smem_u32(sDO), ds_b = smem_u32(sDS);
    // descriptor offsets (16-B units) of the 8 K16 steps: K-major operands step
    // 32 B within a 128-B swizzle row and a slab every 4; MN-major ones 16 rows
    uint32_t kmaj_off[8], mn_off[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      kmaj_off[kk] = ((kk >> 2) * C::SLAB + (kk & 3) * 32) >> 4;
      mn_off[kk] = (kk * 2048) >> 4;
    }
    int I0 = 0;
    for (int seq = 0;; ++seq) {
    const int u = next_unit(seq);
    if (u < 0) break;
    const int n_iter = geom(u).n_iter;
    mbar_wait(&bars->kv_full, seq & 1);
    if (!PAIR) TRACE3(15, I0);   // K / V of this unit landed (trace builds)
    for (int i = 0; i <= n_iter; ++i) {
      const int Ig = I0 + i;
      if (i < n_iter) {
        const int st = Ig % C::QS;
        const uint32_t qs = q_b + st * C::Q_BYTES;
        mbar_wait(&bars->q_full[st], (Ig / C::QS) & 1);
        TRACE3(0, Ig);
        if (!PAIR && i == 0) TRACE3(4, Ig);   // unit start (trace builds)
        tc_fence_after();
        // S^T = K Q^T (contract over D; K-major both); 8-MMA chains under one
        // elect.sync keep the MMA warp's issue slots off its SMSP's compute warps
        mma_ss8_w(tmem + C::COL_S, sdesc_sw128(k_b, 16, 1024), sdesc_sw128(qs, 16, 1024), kmaj_off,
                  kmaj_off, C::IDESC_ST, 0);
        mma_commit_w(&bars->s_full);
      }
      if (i >= 1) {
        const int j = i - 1, Jg = Ig - 1, st = Jg % C::QS;
        const uint32_t qs = q_b + st * C::Q_BYTES;
        mbar_wait_fast(&bars->ds_full[0], Jg & 1);
        mbar_wait_fast(&bars->ds_full[1], Jg & 1);
        TRACE3(5, Jg);
        tc_fence_after();
        const uint32_t dsb = ds_b;
        // dQ = dS K (contract over keys; A = dS from the dS^T buffer and B = K,
        // both MN-major): lanes = queries, so the drain emits 16-B reductions
        mma_ss8_w(tmem + C::COL_DP, sdesc_sw128(dsb, C::SLAB, 1024), sdesc_sw128(k_b, C::SLAB, 1024),
                  mn_off, mn_off, C::IDESC_DQ, 0);
        mma_commit_w(&bars->dq_full);
        // dK += dS^T Q (contract over queries; A = dS^T K-major from SMEM)
        mma_ss8_w(tmem + C::COL_DK, sdesc_sw128(dsb, 16, 1024), sdesc_sw128(qs, C::SLAB, 1024),
                  kmaj_off, mn_off, C::IDESC_ACC, j > 0);
        mma_commit_w(&bars->q_empty[st]);
        if (j == n_iter - 1) mma_commit_w(&bars->acc_done);
      }
      if (i < n_iter) {
        const int st = Ig % C::QS;
        const uint32_t dos = (PAIR || TRED) ? do_b : do_b + st * C::Q_BYTES;
        const uint32_t ph = Ig & 1;
        if (PAIR || TRED) mbar_wait(&bars->do_full, ph);
        // dP^T = V dO^T into the columns dQ(i-1) (or the previous unit's last
        // dQ) occupied: wait for the drain
        if (Ig >= 1) mbar_wait_fast(&bars->s_free, (Ig - 1) & 1);
        TRACE3(1, Ig);
        tc_fence_after();
        mma_ss8_w(tmem + C::COL_DP, sdesc_sw128(v_b, 16, 1024), sdesc_sw128(dos, 16, 1024), kmaj_off,
                  kmaj_off, C::IDESC_ST, 0);
        mma_commit_w(&bars->dp_full);
        // dV += P^T dO, contract over queries, A = P^T from TMEM; chunk c holds
        // queries [32c, 32c+32) of both 64-query halves
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          mbar_wait_fast(&bars->p_full[c], ph);
          TRACE3(2 + c, Ig);
          tc_fence_after();
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
              const int kk = hf * 4 + c * 2 + sub;   // queries [16kk, 16kk+16)
              mma_ts_w(tmem + C::COL_DV, tmem + C::COL_S + 64 * hf + 16 * c + 8 * sub,
                       sdesc_sw128(dos + kk * 2048, C::SLAB, 1024), C::IDESC_ACC,
                       (i > 0) || (c | hf | sub));
            }
        }
        if (PAIR || TRED) mma_commit_w(&bars->do_empty);   // single dO buffer: dV(i) was its last reader
      }
    }
    mma_commit_w(&bars->kv_empty);   // this unit's last K / V readers issued
    I0 += n_iter;
    }
  } else if (warp == 3) {
    // ------------------------------------------------- per-query vectors --
    int I0 = 0;
    for (int seq = 0;; ++seq) {
    const int u = next_unit(seq);
    if (u < 0) break;
    const Unit3 U = geom(u);
    const int4 kt = U.kt;
    const int k0 = U.k0, g = U.g, qt_per_head = U.qt, n_iter = U.n_iter;
    for (int i = 0; i < n_iter; ++i) {
      const int Ig = I0 + i;
      const int b = Ig % C::QS;
      const int h = g * group + (WLB_BWD_HEAD_INNER ? i % group : i / qt_per_head);
      const int row0 = kt.z + (WLB_BWD_HEAD_INNER ? i / group : i % qt_per_head) * C::BM;
      mbar_wait(&bars->vec_empty[b], ((Ig / C::QS) & 1) ^ 1);
      float* vec = sVec + b * 2 * C::BM;
      int8_t* rp = sPos + b * C::BM;
#pragma unroll
      for (int e = lane; e < C::BM; e += 32) {
        const int row = row0 + e;
        const bool ok = row < kt.w;
        vec[e] = ok ? -lse[(size_t)h * Tl + row] * 1.4426950408889634f : 0.f;
        vec[C::BM + e] = ok ? delta[(size_t)h * Tl + row] : 0.f;
        rp[e] = (int8_t)(ok ? min(positions[row] - k0, 127) : -1);
      }
      mbar_arrive(&bars->vec_full[b]);
    }
    I0 += n_iter;
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------ dQ drain --
    const int lg = warp & 3;             // TMEM lane quarter = 32 query rows
    const uint32_t lane_base = tmem + ((uint32_t)(lg * 32) << 16);
    // dq_acc layout [Hq][D/4][Tl][4]: the warp's 32 query rows of one 4-float
    // column block are 512 contiguous bytes -> one coalesced 16-B-per-lane RED.
    // The whole 128-column dQ row is loaded at once (192 registers via
    // setmaxnreg), so the dP^T/dQ columns are released right away; the 32
    // reductions are then paced over the next tile (after dp_full, ds_full[0],
    // ds_full[1] of tile j+1) instead of bursting into L2 at once: a burst
    // backed up the SM's memory queues and stalled the compute warps' TMEM
    // loads.  (dp_full / ds_full of tile j+2 need s_free(j+1) from this warp,
    // so those waits cannot alias a later phase.)
    setmaxnreg_inc<160>();
    const size_t blk = (size_t)Tl * 4;
    int I0 = 0;
    for (int seq = 0;; ++seq) {
    const int u = next_unit(seq);
    if (u < 0) break;
    const Unit3 U = geom(u);
    const int4 kt = U.kt;
    const int g = U.g, qt_per_head = U.qt, n_iter = U.n_iter;
    for (int j = 0; j < n_iter; ++j) {
      const int Jg = I0 + j;
      const int h = g * group + (WLB_BWD_HEAD_INNER ? j % group : j / qt_per_head);
      const int row = kt.z + (WLB_BWD_HEAD_INNER ? j / group : j % qt_per_head) * C::BM + lg * 32 + lane;
#ifdef WLB_EXP_NORED
      const bool ok = false;   // timing experiment: no dQ reductions (wrong dQ)
#else
      const bool ok = row < kt.w;
#endif
      float* base = dq_acc + (size_t)h * (D / 4) * blk + (size_t)row * 4;
#ifdef WLB_EXP_NORED
      const bool ok_tile = false;
#else
      const bool ok_tile = true;
#endif
      mbar_wait(&bars->dq_full, Jg & 1);
      // (trace event 12 is the producer's kv_empty, above)
      tc_fence_after();
      uint32_t u[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_ld32(lane_base + C::COL_DP + c * 32, *reinterpret_cast<uint32_t(*)[32]>(u + 32 * c));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&bars->s_free);
      // (trace event 13 is the compute warps' dK / dV epilogue end, below)
      const bool last = j + 1 == n_iter;   // (no pacing across units)
      const uint32_t nph = (Jg + 1) & 1;
      if (PAIR && paired) {
        // Exchange halves with the peer CTA: keep head-dims [64*cta, 64*cta+64),
        // send the other 64 (st.async into the peer's exchange buffer, row q,
        // 16-B chunks XOR-swizzled by q so a quarter-warp's loads hit distinct
        // banks), add the peer's, reduce half as many bytes into dq_acc.
        const int q = lg * 32 + lane, peer = cta ^ 1;
        // kept half -> u[0, 64), sent half -> u[64, 128) (register selects, no
        // dynamic indexing)
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const uint32_t lo = u[e], hi = u[64 + e];
          u[e] = cta ? hi : lo;
          u[64 + e] = cta ? lo : hi;
        }
        // The exchange runs in 4 quarters of 16 head-dims, paced like the
        // reductions (a 32 KB st.async burst jammed the SM's memory queue and
        // stalled the compute warps' loads).  Quarter c of row q sits at
        // rx + c*8K + q*64, its 16-B chunks XOR-swizzled by (q>>1)&3.
        uint8_t* rx = sDO + C::Q_BYTES;     // the unused second dO stage
        const uint32_t rx_row = smem_u32(rx) + q * 64;
        const uint32_t prow = mapa_shared(rx_row, peer);
        const int sw = (q >> 1) & 3;
        // (CTA-scope waits: a cluster-scope acquire invalidates the SM's L1 on
        //  every completion; the peer's loads of its buffer are complete before
        //  its release-arrive, and st.async data is visible through the
        //  rx_full transaction counts)
        mbar_wait_fast(&bars->peer_free, (Jg & 1) ^ 1);     // peer consumed tile j-1
        if (warp == 12) TRACE3(4, Jg);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (!last) {
            if (c == 1) mbar_wait(&bars->dp_full, nph);
            if (c == 2) mbar_wait(&bars->ds_full[0], nph);
            if (c == 3) mbar_wait(&bars->ds_full[1], nph);
          }
          mbar_expect_tx(&bars->rx_full[c], 64);
          const uint32_t pbar = mapa_shared(smem_u32(&bars->rx_full[c]), peer);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            st_async_v4(prow + c * 8192 + ((e ^ sw) << 4), pbar, u[64 + 16 * c + 4 * e],
                        u[64 + 16 * c + 4 * e + 1], u[64 + 16 * c + 4 * e + 2],
                        u[64 + 16 * c + 4 * e + 3]);
          // (no suspend hint: a remote completion wakes a suspended waiter late)
          mbar_wait_fast(&bars->rx_full[c], Jg & 1);
          if (warp == 12 && c == 0) TRACE3(14, Jg);
          if (warp == 12 && c == 3) TRACE3(15, Jg);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint4 r = *reinterpret_cast<const uint4*>(rx + c * 8192 + q * 64 + ((e ^ sw) << 4));
            const int dd = 16 * c + 4 * e;          // kept head-dims 64*cta + dd
            if (ok)
              red_add_v4(base + (size_t)(16 * cta + dd / 4) * blk,
                         (__uint_as_float(u[dd]) + __uint_as_float(r.x)) * scale,
                         (__uint_as_float(u[dd + 1]) + __uint_as_float(r.y)) * scale,
                         (__uint_as_float(u[dd + 2]) + __uint_as_float(r.z)) * scale,
                         (__uint_as_float(u[dd + 3]) + __uint_as_float(r.w)) * scale);
          }
        }
        fence_proxy_async_smem();           // loads done before the peer's next st.async
        mbar_arrive_remote(mapa_shared(smem_u32(&bars->peer_free), peer));
        continue;
      }
      if (TRED) {
        // 4 rounds of 8 column blocks (32 head-dims): staging [8][32 rows][4]
        // fp32 = 4 KB, two buffers per warp in the unused second dO stage;
        // rounds paced like the reductions below.  Rows past the document
        // (masked: exact zeros) add 0; rows past Tl are clipped by the map.
        uint8_t* stg = sDO + C::Q_BYTES + (warp - 12) * 8192;
        const int row0 = row - lane;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (!last && WLB_TRED_PACE) {
            if (r == 1) mbar_wait(&bars->dp_full, nph);
            if (r == 2) mbar_wait(&bars->ds_full[0], nph);
            if (r == 3) mbar_wait(&bars->ds_full[1], nph);
          }
          uint8_t* buf = stg + (r & 1) * 4096;
          if (lane == 0) bulk_wait_group_read<1>();   // this buffer's previous reduce has read it
          __syncwarp();
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int q = 8 * r + e;
            *reinterpret_cast<float4*>(buf + e * 512 + lane * 16) =
                make_float4(__uint_as_float(u[4 * q]) * scale, __uint_as_float(u[4 * q + 1]) * scale,
                            __uint_as_float(u[4 * q + 2]) * scale,
                            __uint_as_float(u[4 * q + 3]) * scale);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && ok_tile) {
            tma_reduce_add_3d(&tmDQ, buf, 4 * row0, 8 * r, h);
            bulk_commit_group();
          }
        }
        continue;
      }
#if WLB_RED_PACE == 0
      // 32 16-B reductions per thread: the first WLB_RED_B0 right away, then
      // batches after dp_full, ds_full[0] and ds_full[1] of the next tile
      constexpr int T1 = WLB_RED_B0, T2 = T1 + WLB_RED_B1, T3 = T2 + WLB_RED_B2;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        if (!last) {
          if (e == T1 && T1 < 32) mbar_wait(&bars->dp_full, nph);
          if (e == T2 && T2 < 32) mbar_wait(&bars->ds_full[0], nph);
          if (e == T3 && T3 < 32) mbar_wait(&bars->ds_full[1], nph);
        }
        if (ok)
          red_add_v4(base + (size_t)e * blk, __uint_as_float(u[4 * e]) * scale,
                     __uint_as_float(u[4 * e + 1]) * scale, __uint_as_float(u[4 * e + 2]) * scale,
                     __uint_as_float(u[4 * e + 3]) * scale);
      }
#else
      (void)last;
      (void)nph;
#pragma unroll
      for (int c = 0; c < WLB_RED_PACE; ++c) {
        if (c > 0) __nanosleep(WLB_RED_SLEEP);
        if (ok) {
#pragma unroll
          for (int e = 0; e < 32 / WLB_RED_PACE; ++e) {
            const int q = c * (32 / WLB_RED_PACE) + e;
            red_add_v4(base + (size_t)q * blk, __uint_as_float(u[4 * q]) * scale,
                       __uint_as_float(u[4 * q + 1]) * scale, __uint_as_float(u[4 * q + 2]) * scale,
                       __uint_as_float(u[4 * q + 3]) * scale);
          }
        }
      }
#endif
    }
    I0 += n_iter;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- compute --
    setmaxnreg_inc<136>();
    const int lg = warp & 3;                 // TMEM lane quarter
    const int hf = (warp - 4) >> 2;          // query half [64hf, 64hf+64)
    const int t = lg * 32 + lane;            // key row in the tile
    const uint32_t lane_base = tmem + ((uint32_t)(lg * 32) << 16);
    int I0 = 0;
    for (int seq = 0;; ++seq) {
    const int u = next_unit(seq);
    if (u < 0) break;
    const Unit3 U = geom(u);
    const int4 kt = U.kt;
    const int g = U.g, n_iter = U.n_iter;
    const bool key_ok = t < kt.y;
    for (int i = 0; i < n_iter; ++i) {
      const int Ig = I0 + i;
      const int vb = Ig % C::QS;
      const uint32_t ph = Ig & 1;
      uint8_t* drow = sDS + hf * C::SLAB + t * 128;
      const float* nl = sVec + vb * 2 * C::BM + 64 * hf;
      const float* dl = nl + C::BM;
      const int8_t* rp = sPos + vb * C::BM + 64 * hf;
      mbar_wait(&bars->vec_full[vb], (Ig / C::QS) & 1);
      mbar_wait(&bars->s_full, ph);
      if (warp == 4) TRACE3(6, Ig);
      tc_fence_after();
      uint32_t p16[2][16];   // P (fp16 pairs with P16, else bf16), kept for dS
      // ---- P^T = exp2(S^T * scale * log2e - lse2), per 32-query chunk
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t us[32];
        tmem_ld32(lane_base + C::COL_S + 64 * hf + 32 * c, us);
        const bool full = kt.y == C::BN && rp[32 * c] >= C::BN - 1 && rp[32 * c + 31] >= C::BN - 1;
        tmem_ld_wait();

        uint32_t pk[16];
        if (full)
          bwd3_p_chunk<false, P16>(us, nl + 32 * c, rp + 32 * c, t, key_ok, scale_log2, pk, p16[c]);
        else
          bwd3_p_chunk<true, P16>(us, nl + 32 * c, rp + 32 * c, t, key_ok, scale_log2, pk, p16[c]);

        // over S^T columns this warp already loaded (chunk 0's 32 columns)
        tmem_st16(lane_base + C::COL_S + 64 * hf + 16 * c, pk);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars->p_full[c]);
        if (warp == 4) TRACE3(7 + c, Ig);
      }
      // ---- dS^T = P^T (dP^T - Delta), per chunk, into SMEM (for dQ and dK)
      // (the buffer's previous readers, dQ(i-1) and dK(i-1), were issued
      //  before dP(i): dp_full(i) implies they completed)
      mbar_wait(&bars->dp_full, ph);
      if (warp == 4) TRACE3(9, Ig);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t ud[32];
        tmem_ld32(lane_base + C::COL_DP + 64 * hf + 32 * c, ud);
        const float4* d4p = reinterpret_cast<const float4*>(dl + 32 * c);
        tmem_ld_wait();
        uint32_t dk2[16];
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          const float4 d4 = d4p[e4];
#pragma unroll
          for (int u2 = 0; u2 < 2; ++u2) {
            const int e = 4 * e4 + 2 * u2;
            const uint32_t pp = p16[c][e >> 1];
            const float2 pf = P16 ? __half22float2(*reinterpret_cast<const __half2*>(&pp))
                                  : make_float2(__uint_as_float(pp << 16), __uint_as_float(pp & 0xffff0000u));
            const float2 dd = fadd2(make_float2(__uint_as_float(ud[e]), __uint_as_float(ud[e + 1])),
                                    u2 ? make_float2(-d4.z, -d4.w) : make_float2(-d4.x, -d4.y));
            const float2 ds = fmul2(pf, dd);
            dk2[e >> 1] = pack_bf16(ds.x, ds.y);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int chunk = 4 * c + j;   // 16-B chunk (8 queries) within the 128-B row
          *reinterpret_cast<uint4*>(drow + ((chunk ^ (t & 7)) << 4)) =
              make_uint4(dk2[4 * j], dk2[4 * j + 1], dk2[4 * j + 2], dk2[4 * j + 3]);
        }
        fence_proxy_async_smem();
        mbar_arrive(&bars->ds_full[c]);
        if (warp == 4) TRACE3(10 + c, Ig);
      }
      mbar_arrive(&bars->vec_empty[vb]);
    }
    mbar_wait(&bars->acc_done, seq & 1);   // this unit's last MMA group wrote dV / dK
    tc_fence_after();
    // ------------------------------------------------------------ epilogue --
    // (the dS^T buffer is free: acc_done follows the last dK MMA, its last reader)
    const size_t off = ((size_t)(kt.x + lg * 32) * Hkv + g) * D + hf * 64;
    uint4* stg = reinterpret_cast<uint4*>(sDS + (warp - 4) * 4096);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t a[32], bb[32];
      tmem_ld32(lane_base + C::COL_DV + hf * 64 + c * 32, a);
      tmem_ld32(lane_base + C::COL_DK + hf * 64 + c * 32, bb);
      tmem_ld_wait();
      store_dkv_block(dv, dk, off + c * 32, (size_t)Hkv * D, kt.y - lg * 32, a, bb, scale,
                      dkv_bf16 != 0, stg);
    }
    if (warp == 4 && !PAIR) TRACE3(13, I0 + n_iter);   // epilogue issued (trace builds)
    if (!PAIR && sync.signal_bases) {
      // CP: this (KV tile, head) unit's partials are stored; count it toward
      // its head group and publish the group when complete
      named_bar_sync(1, 256);
      if (warp == 4 && lane == 0)
        cp_sync_unit_done(sync, g / sync.kv_per_group, n_kv_tiles[0] * sync.kv_per_group);
    }
    I0 += n_iter;
    }
  }
  if (TRED && warp >= 12 && lane == 0) bulk_wait_group<0>();   // reduces done with the staging
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, C::TMEM_COLS);
  if (PAIR && paired) cluster_sync();       // no CTA leaves while its peer may write it
}

// Delta[h][i] = sum_d dO[i,h,d] * O[i,h,d] (fp32).  D/8 lanes per (row, head),
// 16 B of O and dO per lane; each thread keeps 4 (row, head) pairs in flight
// (one pair per warp and a dependent reduction ran at ~3.7 TB/s).
template <int D>
__global__ void __launch_bounds__(256) bwd_delta_kernel(const __nv_bfloat16* __restrict__ o,
                                                        const __nv_bfloat16* __restrict__ dout,
                                                        float* __restrict__ delta, int Tl, int Hq,
                                                        int h_begin, int h_count,
                                                        uint4* __restrict__ dq_zero) {
  constexpr int LPR = D / 8;                 // lanes per (row, head)
  constexpr int U = 4;                       // pairs in flight per thread
  const long long n = (long long)Tl * h_count;   // (row, head) pairs, heads [h_begin, +h_count)
  const int sub = threadIdx.x % LPR;
  const long long lanes = (long long)gridDim.x * blockDim.x / LPR;
  for (long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPR; w0 < n;
       w0 += U * lanes) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long w = w0 + u * lanes;
      if (w < n) {
        const long long rh = h_count == Hq ? w : (w / h_count) * Hq + h_begin + w % h_count;
        a[u] = reinterpret_cast<const uint4*>(o + rh * D)[sub];
        b[u] = reinterpret_cast<const uint4*>(dout + rh * D)[sub];
        if (dq_zero) {   // the (row, head)'s fp32 dQ accumulator slice, [Tl][Hq][D] layout
          dq_zero[rh * (D / 4) + 2 * sub] = make_uint4(0, 0, 0, 0);
          dq_zero[rh * (D / 4) + 2 * sub + 1] = make_uint4(0, 0, 0, 0);
        }
      } else {
        a[u] = b[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
      const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&b[u]);
      float sum = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 xf = __bfloat1622float2(x[e]), yf = __bfloat1622float2(y[e]);
        sum = fmaf(xf.x, yf.x, fmaf(xf.y, yf.y, sum));
      }
#pragma unroll
      for (int off = LPR / 2; off; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      const long long w = w0 + u * lanes;
      if (sub == 0 && w < n) {
        const unsigned uw = (unsigned)w;          // Tl * Hq < 2^31
        delta[(size_t)(h_begin + uw % (unsigned)h_count) * Tl + uw / (unsigned)h_count] = sum;
      }
    }
  }
}

// v3 dQ accumulator [Hq][D/4][Tl][4] fp32 -> dq [Tl][Hq][D] bf16, heads
// [h_begin, h_begin + h_count).  32-bit index math with D a template
// constant (a 64-bit division per element cost ~6% of a short rank's step).
template <int D>
__global__ void __launch_bounds__(256) dq_convert3_kernel(const float4* __restrict__ acc,
                                                          uint2* __restrict__ dq, int Tl, int Hq,
                                                          int h_begin, int h_count) {
  // one block per (32 rows, head): coalesced 512-B reads along rows of each
  // 4-float column block, a shared-memory transpose, coalesced row writes
  // (the flat output-ordered loop read 16 B per 32-B sector: ~3.9 TB/s)
  constexpr int DB = D / 4, R = 32;
  __shared__ float4 tile[R][DB + 1];
  const int row0 = (int)(blockIdx.x % (unsigned)((Tl + R - 1) / R)) * R;
  const int h = h_begin + (int)(blockIdx.x / (unsigned)((Tl + R - 1) / R));
  const float4* src = acc + (size_t)h * DB * Tl;
#pragma unroll
  for (int k = 0; k < (R * DB + 255) / 256; ++k) {
    const int idx = k * 256 + (int)threadIdx.x;
    if (idx < R * DB) {
      const int db = idx / R, r = idx % R;
      tile[r][db] = row0 + r < Tl ? src[(size_t)db * Tl + row0 + r] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < (R * DB + 255) / 256; ++k) {
    const int idx = k * 256 + (int)threadIdx.x;
    if (idx < R * DB) {
      const int r = idx / DB, db = idx % DB;
      if (row0 + r < Tl) {
        const float4 v = tile[r][db];
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
        dq[((size_t)(row0 + r) * Hq + h) * DB + db] =
            make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
      }
    }
  }
}

// v2 dQ accumulator [Tl][Hq][D] fp32 -> dq bf16, heads [h_begin, h_begin +
// h_count); all heads (the common case) is one flat pass.
template <int D>
__global__ void dq_convert_kernel(const float4* __restrict__ acc, __nv_bfloat162* __restrict__ dq,
                                  int Tl, int Hq, int h_begin, int h_count) {
  constexpr unsigned DB = D / 4;
  const unsigned n = (unsigned)Tl * (unsigned)h_count * DB;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    size_t j = i;
    if (h_count != Hq) {
      const unsigned rh = i / DB;
      j = ((size_t)(rh / (unsigned)h_count) * Hq + h_begin + rh % (unsigned)h_count) * DB + i % DB;
    }
    const float4 v = acc[j];
    dq[2 * j] = __floats2bfloat162_rn(v.x, v.y);
    dq[2 * j + 1] = __floats2bfloat162_rn(v.z, v.w);
  }
}

// KV-tile work list: for each document with local rows, 128-key tiles up to the
// largest local position; the query rows of a tile are the row-set suffix with
// position >= k0 (binary search).  Sorted by descending query-row count.
constexpr int kKvThreads = 1024;
constexpr int kKvBins = 2048;
__global__ void __launch_bounds__(kKvThreads)
bwd_kv_tiles_kernel(int nd, const int* __restrict__ rowset_off, const int* __restrict__ positions,
                    const int* __restrict__ doc_start, int max_items, int4* __restrict__ out,
                    int* __restrict__ n_out, int4* __restrict__ scratch, int pairs) {
  __shared__ long long warp_tot[kKvThreads / 32 + 1];
  __shared__ int hist[kKvBins];
  __shared__ int maxkey_s;
  // pass 1 (parallel over documents): KV-tile count and item offset of each
  // document (doc_base lives past the item scratch); pass 2 expands the items
  // in parallel over items (a serial per-document loop cost ~250 us per call).
  int* doc_base = reinterpret_cast<int*>(scratch + 2 * (size_t)max_items);   // [nd + 1]
  long long carry = 0;
  for (int base = 0; base < nd; base += blockDim.x) {
    const int p = base + threadIdx.x;
    int nt = 0;
    if (p < nd) {
      const int r0 = rowset_off[p], r1 = rowset_off[p + 1];
      if (r1 > r0) nt = (positions[r1 - 1] + 128) / 128;
      if (pairs) nt = (nt + 1) / 2;            // items = tile pairs (2q, 2q+1)
    }
    long long tot;
    const long long off = carry + block_exclusive_scan(nt, warp_tot, &tot);
    if (p < nd) doc_base[p] = (int)off;
    carry += tot;
  }
  if (threadIdx.x == 0) doc_base[nd] = (int)carry;
  __syncthreads();
  const int n_items = carry < max_items ? (int)carry : max_items;
  // pass 2 (parallel over items): owning document by binary search over the
  // bases, first visible row by binary search over the row-set positions.
  for (int it = threadIdx.x; it < n_items; it += blockDim.x) {
    int lo = 0, hi = nd;                      // largest p with doc_base[p] <= it
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (doc_base[mid] <= it) lo = mid;
      else hi = mid;
    }
    const int p = lo, t = (it - doc_base[p]) * (pairs ? 2 : 1), k0 = t * 128;
    const int r0 = rowset_off[p], r1 = rowset_off[p + 1];
    int a = r0, b = r1;                       // first row with position >= k0
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (positions[mid] >= k0) b = mid;
      else a = mid + 1;
    }
    const int dl = doc_start[p + 1] - doc_start[p];
    const int len = dl - k0;
    scratch[2 * it] = make_int4(doc_start[p] + k0, len < 128 ? len : 128, a, r1);
    if (pairs) {                              // second tile of the pair, if it exists
      const int k1 = k0 + 128;
      const bool has = r1 > r0 && k1 <= positions[r1 - 1];
      scratch[2 * it + 1] = make_int4(k0, has ? doc_start[p] + k1 : -1,
                                      has ? min(128, dl - k1) : 0, k1);
    } else {
      scratch[2 * it + 1] = make_int4(k0, p, 0, 0);
    }
  }
  __syncthreads();
  const int total = n_items;
  int mk = 0;
  for (int i = threadIdx.x; i < total; i += blockDim.x)
    mk = max(mk, (scratch[2 * i].w - scratch[2 * i].z + 127) >> 7);
  for (int o = 16; o; o >>= 1) mk = max(mk, __shfl_xor_sync(0xffffffffu, mk, o));
  if (threadIdx.x == 0) maxkey_s = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicMax(&maxkey_s, mk);
  __syncthreads();
  int shift = 0;
  while ((maxkey_s >> shift) >= kKvBins) ++shift;
  for (int i = threadIdx.x; i < kKvBins; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x)
    atomicAdd(&hist[kKvBins - 1 - (((scratch[2 * i].w - scratch[2 * i].z + 127) >> 7) >> shift)], 1);
  __syncthreads();
  const long long a0 = hist[2 * threadIdx.x], a1 = hist[2 * threadIdx.x + 1];
  long long tot;
  const long long ex = block_exclusive_scan(a0 + a1, warp_tot, &tot);
  hist[2 * threadIdx.x] = (int)ex;
  hist[2 * threadIdx.x + 1] = (int)(ex + a0);
  __syncthreads();
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int key = kKvBins - 1 - (((scratch[2 * i].w - scratch[2 * i].z + 127) >> 7) >> shift);
    const int slot = atomicAdd(&hist[key], 1);
    out[2 * slot] = scratch[2 * i];
    out[2 * slot + 1] = scratch[2 * i + 1];
  }
  if (threadIdx.x == 0) n_out[0] = total;
}

static int g_bwd_v3_min_rows = WLB_BWD_V3_MIN_ROWS;
#ifndef WLB_HPC
#define WLB_HPC 4   // KV heads per CTA for short row-sets (2 the same, 8 up to 4% slower)
#endif
static int g_bwd_hpc_short = WLB_HPC;
// v3 as 2-CTA clusters exchanging dQ halves over DSMEM (experimental, off):
// it halves the dQ reduction bytes but adds the same number of DSMEM bytes to
// the SM's outbound memory path, which is what bounds the reductions (plain
// stores instead of reductions measured the same as reductions), and the
// pair's exchange couples the two CTAs' pipelines: 650-725 vs 960-980 TFLOP/s
// on a 32K document (profiles/r01_bwd3_pairs_trace.txt).
#ifndef WLB_BWD_PAIRS
#define WLB_BWD_PAIRS 0
#endif
static int g_bwd_pairs = WLB_BWD_PAIRS;
// 128-query backward: dQ partials reduced by TMA tile reduce-adds from shared
// memory (1) or by per-thread RED.v4 (0)
#ifndef WLB_BWD_TRED
#define WLB_BWD_TRED 1
#endif
static int g_bwd_tred = WLB_BWD_TRED;
// 128-query backward as a persistent kernel (one CTA per SM, unit queue)
#ifndef WLB_BWD3_PERSIST
#define WLB_BWD3_PERSIST 1
#endif
static int g_bwd3_persistent = WLB_BWD3_PERSIST;
// SMs the persistent backward kernels leave free (grid = SMs - reserve), so
// the CP exchange's pull / push kernels on the communication stream find SMs
// while a head group's backward runs (0: every SM; set by the CP pipeline)
static int g_bwd_reserve_sms = 0;
// persistent 128-query backward: L2 prefetch of the next unit's K / V and
// first Q / dO tile while the current unit drains
#ifndef WLB_BWD3_L2PF
#define WLB_BWD3_L2PF 0
#endif
static int g_bwd3_l2pf = WLB_BWD3_L2PF;
// v2 backward as a persistent kernel (one CTA per SM, dynamic unit queue)
#ifndef WLB_BWD_PERSIST
#define WLB_BWD_PERSIST 1
#endif
static int g_bwd_persistent = WLB_BWD_PERSIST;

// Zero the dK/dV rows no KV tile covers: in document p, keys at in-document
// positions >= 128 * ceil((last local position + 1) / 128) (all of p when this
// rank holds none of its rows); same tile rule as bwd_kv_tiles_kernel.  Block b
// owns global rows [b*ZR, (b+1)*ZR) and walks the documents overlapping them.
constexpr int kZeroRows = 64;
__global__ void zero_uncovered_kernel(const int* __restrict__ rowset_off,
                                      const int* __restrict__ positions,
                                      const int* __restrict__ doc_start, int n_docs,
                                      uint4* __restrict__ dk, uint4* __restrict__ dv,
                                      int row_f4,     // row length in 16-B units
                                      int col_f4, int ncol_f4) {   // the KV heads' columns
  const int a0 = blockIdx.x * kZeroRows, a1 = min(a0 + kZeroRows, doc_start[n_docs]);
  int lo = 0, hi = n_docs;                   // last document with doc_start <= a0
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (doc_start[mid] <= a0) lo = mid;
    else hi = mid;
  }
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (int p = lo; p < n_docs && doc_start[p] < a1; ++p) {
    const int r0 = rowset_off[p], r1 = rowset_off[p + 1];
    const int len = doc_start[p + 1] - doc_start[p];
    const int covered = r1 > r0 ? min(len, (positions[r1 - 1] + 128) / 128 * 128) : 0;
    const int z0 = max(a0, doc_start[p] + covered), z1 = min(a1, doc_start[p + 1]);
    if (z0 >= z1) continue;
    const long long n = (long long)(z1 - z0) * ncol_f4;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      const long long e = (long long)(z0 + i / ncol_f4) * row_f4 + col_f4 + i % ncol_f4;
      dk[e] = z;
      dv[e] = z;
    }
  }
}

struct BwdWorkspace {
  float* dq_acc;
  float* delta;
  int4* kv_tiles;   // [2*max_items] sorted + [2*max_items] scratch
  int* n_kv;
  int* sched;       // persistent kernel's unit counter
  size_t bytes;
};

static BwdWorkspace carve(void* base, int Tl, int T, int Hq, int D, int n_docs) {
  BwdWorkspace w;
  const size_t max_items = (size_t)T / 128 + n_docs + 1;
  uint8_t* p = (uint8_t*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* r = p ? p + off : nullptr;
    off += (bytes + 255) & ~(size_t)255;
    return r;
  };
  w.dq_acc = (float*)take((size_t)Tl * Hq * D * 4);
  w.delta = (float*)take((size_t)Hq * Tl * 4);
  w.kv_tiles = (int4*)take(4 * max_items * sizeof(int4) + (n_docs + 1) * sizeof(int));
  w.n_kv = (int*)take(16);
  w.sched = (int*)take(16);
  w.bytes = off;
  return w;
}

template <int D>
static int launch_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                      const float* lse, void* dq, void* dk, void* dv, const int32_t* rowset_off,
                      const int32_t* doc_start, int32_t n_docs, const int32_t* positions,
                      int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv, float scale, void* ws,
                      int dkv_bf16, bool covered_only, int g_begin, int g_count,
                      const CpSync& sync, cudaStream_t stream) {
  using C = BwdCfg<D>;
  BwdWorkspace w = carve(ws, Tl, T, Hq, D, n_docs);
  const int max_items = T / 128 + n_docs + 1;
  const int group = Hq / Hkv, h_begin = g_begin * group, h_count = g_count * group;
#if WLB_BWD_V3
  const bool v3 = D == 128 && (long long)Tl >= (long long)g_bwd_v3_min_rows * (n_docs > 0 ? n_docs : 1);
  const bool pairs = v3 && g_bwd_pairs && !sync.signal_bases;   // (pairs do not signal)
#else
  const bool v3 = false, pairs = false;
#endif
  // dQ accumulator of this launch's query heads: [Hq][D/4][Tl][4] (v3) keeps
  // a head contiguous, [Tl][Hq][D] (v2) strides it
  // the 64-query kernel's [Tl][Hq][D] accumulator is zeroed by the Delta pass
  // (same rows and heads, one launch fewer: ~12 us of a short rank's step);
  // the 128-query kernel's [Hq][D/4][Tl][4] one keeps a head range contiguous
  if (v3)
    WLB_CUDA_TRY(cudaMemsetAsync(w.dq_acc + (size_t)h_begin * D * Tl, 0,
                                 (size_t)Tl * h_count * D * 4, stream));
  // dK/dV rows of every KV tile are stored whole by the kernel; only the keys
  // no KV tile covers (past a document's last local query position) are zeroed
  // here, instead of clearing 2 x T x Hkv x D x 4 bytes up front.
  if (n_docs > 0 && !covered_only) {
    const int hf4 = D * (dkv_bf16 ? 2 : 4) / 16;    // one KV head's columns in 16-B units
    zero_uncovered_kernel<<<(unsigned)((T + kZeroRows - 1) / kZeroRows), 256, 0, stream>>>(
        rowset_off, positions, doc_start, n_docs, (uint4*)dk, (uint4*)dv, Hkv * hf4,
        g_begin * hf4, g_count * hf4);
    WLB_LAUNCH_CHECK();
  }
  {
    const long long lanes = (long long)Tl * h_count * (D / 8);
    const unsigned blocks = (unsigned)std::min<long long>((lanes + 255) / 256, 148 * 8);
    bwd_delta_kernel<D><<<blocks, 256, 0, stream>>>(
        (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, w.delta, Tl, Hq, h_begin, h_count,
        v3 ? nullptr : reinterpret_cast<uint4*>(w.dq_acc));
    WLB_LAUNCH_CHECK();
  }
  if (sync.signal_bases)
    WLB_CUDA_TRY(cudaMemsetAsync(sync.counters, 0, sizeof(int) * (Hkv / sync.kv_per_group), stream));
  bwd_kv_tiles_kernel<<<1, kKvThreads, 0, stream>>>(n_docs, rowset_off, positions, doc_start,
                                                     max_items, w.kv_tiles, w.n_kv,
                                                     w.kv_tiles + 2 * max_items, pairs ? 1 : 0);
  WLB_LAUNCH_CHECK();
  CUtensorMap tq, tk, tv, tdo, tdq;
  int rc;
#if WLB_BWD_V3
  if (v3) {
    using C3 = Bwd3Cfg;
    if ((rc = make_dq_acc_tmap(&tdq, w.dq_acc, Tl, Hq, D))) return rc;
    if ((rc = make_thd_tmap(&tq, q, Tl, Hq, D, C3::BM))) return rc;
    if ((rc = make_thd_tmap(&tdo, dout, Tl, Hq, D, C3::BM))) return rc;
    if ((rc = make_thd_tmap(&tk, k, T, Hkv, D, C3::BN))) return rc;
    if ((rc = make_thd_tmap(&tv, v, T, Hkv, D, C3::BN))) return rc;
    const bool p16 = Hq != Hkv;
    WLB_SMEM_ATTR((attn_bwd3_kernel<false, false>), C3::SMEM);
    WLB_SMEM_ATTR((attn_bwd3_kernel<false, true>), C3::SMEM);
    WLB_SMEM_ATTR((attn_bwd3_kernel<true, false>), C3::SMEM);
    WLB_SMEM_ATTR((attn_bwd3_kernel<true, true>), C3::SMEM);
    WLB_SMEM_ATTR((attn_bwd3_kernel<false, false, true>), C3::SMEM);
    WLB_SMEM_ATTR((attn_bwd3_kernel<false, true, true>), C3::SMEM);
    const float sl2 = scale * 1.4426950408889634f;
    if (pairs) {
      // 2-CTA clusters: one pair of KV tiles per cluster
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(2 * max_items * g_count));
      cfg.blockDim = dim3(C3::THREADS);
      cfg.dynamicSmemBytes = C3::SMEM;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      WLB_CUDA_TRY(cudaLaunchKernelEx(&cfg, p16 ? attn_bwd3_kernel<true, true> : attn_bwd3_kernel<true, false>, tq, tk, tv, tdo, tdq, lse,
                                      (const float*)w.delta, w.dq_acc, dk, dv,
                                      (const int4*)w.kv_tiles, (const int*)w.n_kv, positions, Tl,
                                      Hq, Hkv, max_items, g_begin, scale, sl2, dkv_bf16,
                                      max_items * g_count, w.sched, 0, sync));
    } else {
      auto kern = g_bwd_tred ? (p16 ? attn_bwd3_kernel<false, true, true>
                                    : attn_bwd3_kernel<false, false, true>)
                             : (p16 ? attn_bwd3_kernel<false, true> : attn_bwd3_kernel<false, false>);
      const int n_units = max_items * g_count;
      unsigned grid = (unsigned)n_units;
      if (g_bwd3_persistent) {
        // one CTA per SM over the unit queue (a unit's epilogue overlaps the
        // next unit's K/V load and first MMAs)
        int dev = 0, sms = 148;
        WLB_CUDA_TRY(cudaGetDevice(&dev));
        WLB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        WLB_CUDA_TRY(cudaMemsetAsync(w.sched, 0, sizeof(int), stream));
        grid = (unsigned)std::min(n_units, std::max(1, sms - g_bwd_reserve_sms));
      }
      kern<<<grid, C3::THREADS, C3::SMEM, stream>>>(
          tq, tk, tv, tdo, tdq, lse, w.delta, w.dq_acc, dk, dv, w.kv_tiles, w.n_kv, positions, Tl, Hq,
          Hkv, max_items, g_begin, scale, sl2, dkv_bf16, n_units, w.sched,
          g_bwd3_persistent ? (1 | (g_bwd3_l2pf ? 2 : 0)) : 0, sync);
    }
    WLB_LAUNCH_CHECK();
  } else
#endif
  {
  if ((rc = make_thd_tmap(&tq, q, Tl, Hq, D, C::BM))) return rc;
  if ((rc = make_thd_tmap(&tdo, dout, Tl, Hq, D, C::BM))) return rc;
  if ((rc = make_thd_tmap(&tk, k, T, Hkv, D, C::BN))) return rc;
  if ((rc = make_thd_tmap(&tv, v, T, Hkv, D, C::BN))) return rc;
  // (A 128-query, single-buffered variant with all-N=128 MMAs measured 1.5x
  //  slower: the S/dP -> compute -> dV/dK/dQ serialisation costs more than the
  //  SMEM bandwidth it saves.)
  WLB_SMEM_ATTR((attn_bwd_kernel<D, 2>), C::SMEM);
  // several KV heads per unit for short row-sets (< WLB_HPC_ROWS local rows
  // per document on average): a unit's heads run back to back (only with >= 6
  // waves of units: Tl/128 bounds the KV tiles from below)
  int hpc = (g_count % g_bwd_hpc_short == 0 && (long long)Tl < (long long)WLB_HPC_ROWS * (n_docs > 0 ? n_docs : 1) &&
             (long long)(Tl / 128) * g_count >= 6LL * 148 * g_bwd_hpc_short)
                ? g_bwd_hpc_short : 1;
  if (sync.signal_bases && sync.kv_per_group % hpc) hpc = 1;   // units inside one head group
  const int n_units = max_items * ((g_count + hpc - 1) / hpc);
  if (g_bwd_persistent) {
    // one CTA per SM taking units from a global counter: a unit's tail
    // (dK/dV epilogue, next K/V load) overlaps the next unit instead of a CTA
    // teardown + launch, and the SMs stay busy to the end
    int dev = 0, sms = 148;
    WLB_CUDA_TRY(cudaGetDevice(&dev));
    WLB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    WLB_CUDA_TRY(cudaMemsetAsync(w.sched, 0, sizeof(int), stream));
    attn_bwd_kernel<D, 2><<<(unsigned)std::min(n_units, std::max(1, sms - g_bwd_reserve_sms)),
                            C::THREADS, C::SMEM, stream>>>(
        tq, tk, tv, tdo, lse, w.delta, w.dq_acc, dk, dv, w.kv_tiles, w.n_kv, positions, Tl, Hq,
        Hkv, max_items, hpc, n_units, w.sched, 1, g_begin, g_begin + g_count, scale,
        scale * 1.4426950408889634f, dkv_bf16, sync);
  } else {
    attn_bwd_kernel<D, 2><<<(unsigned)n_units, C::THREADS, C::SMEM, stream>>>(
        tq, tk, tv, tdo, lse, w.delta, w.dq_acc, dk, dv, w.kv_tiles, w.n_kv, positions, Tl, Hq,
        Hkv, max_items, hpc, n_units, w.sched, 0, g_begin, g_begin + g_count, scale,
        scale * 1.4426950408889634f, dkv_bf16, sync);
  }
  WLB_LAUNCH_CHECK();
  }
  const long long n4 = (long long)Tl * h_count * D / 4;
  const unsigned cblocks = (unsigned)std::min<long long>((n4 + 255) / 256, 148 * 16);
  if (v3) {
    const unsigned tblocks = (unsigned)((Tl + 31) / 32) * (unsigned)h_count;
    dq_convert3_kernel<D><<<tblocks, 256, 0, stream>>>((const float4*)w.dq_acc, (uint2*)dq, Tl, Hq,
                                                        h_begin, h_count);
    WLB_LAUNCH_CHECK();
    return WLB_OK;
  }
  dq_convert_kernel<D><<<cblocks, 256, 0, stream>>>((const float4*)w.dq_acc, (__nv_bfloat162*)dq,
                                                    Tl, Hq, h_begin, h_count);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

}  // namespace wlb

#ifdef WLB_TRACE
extern "C" int wlb_debug_bwd3_trace(void* host) {
  WLB_CUDA_TRY(cudaMemcpyFromSymbol(host, wlb::g_bwd3_trace, sizeof(wlb::g_bwd3_trace)));
  return WLB_OK;
}
extern "C" int wlb_debug_bwd_trace(void* host) {
  WLB_CUDA_TRY(cudaMemcpyFromSymbol(host, wlb::g_bwd_trace, sizeof(wlb::g_bwd_trace)));
  return WLB_OK;
}
#endif

extern "C" int32_t wlb_attn_bwd_pairs(int32_t on) {
  const int32_t prev = wlb::g_bwd_pairs;
  wlb::g_bwd_pairs = on < 0 ? WLB_BWD_PAIRS : (on != 0);
  return prev;
}

extern "C" int32_t wlb_attn_bwd_persistent(int32_t on) {
  const int32_t prev = wlb::g_bwd_persistent;
  wlb::g_bwd_persistent = on < 0 ? WLB_BWD_PERSIST : (on != 0);
  return prev;
}

extern "C" int32_t wlb_attn_bwd_l2_prefetch(int32_t on) {
  const int32_t prev = wlb::g_bwd3_l2pf;
  wlb::g_bwd3_l2pf = on < 0 ? WLB_BWD3_L2PF : (on != 0);
  return prev;
}

extern "C" int32_t wlb_attn_bwd_reserve_sms(int32_t n) {
  const int32_t prev = wlb::g_bwd_reserve_sms;
  wlb::g_bwd_reserve_sms = n < 0 ? 0 : n;
  return prev;
}

extern "C" int32_t wlb_attn_bwd_select(int32_t v3_min_rows) {
  const int32_t prev = wlb::g_bwd_v3_min_rows;
  wlb::g_bwd_v3_min_rows = v3_min_rows < 0 ? WLB_BWD_V3_MIN_ROWS : v3_min_rows;
  return prev;
}

extern "C" size_t wlb_attn_bwd_workspace(int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv, int32_t D,
                                         int32_t n_docs) {
  (void)Hkv;
  return wlb::carve(nullptr, Tl, T, Hq, D, n_docs).bytes;
}

extern "C" int wlb_attn_bwd_heads(const void* q, const void* k, const void* v, const void* o,
                                  const void* do_, const float* lse, void* dq, void* dk, void* dv,
                                  const int32_t* rowset_off, const int32_t* doc_start,
                                  int32_t n_docs, const int32_t* positions, int32_t Tl, int32_t T,
                                  int32_t Hq, int32_t Hkv, int32_t D, float scale, void* ws,
                                  int32_t flags, int32_t kv_head_begin, int32_t kv_head_count,
                                  void* stream) {
  WLB_REQUIRE(D == 64 || D == 128, "head dim %d unsupported (64 or 128)", D);
  WLB_REQUIRE(Hq > 0 && Hkv > 0 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  WLB_REQUIRE(Tl >= 0 && T > 0 && n_docs >= 0 && ws != nullptr, "bad sizes");
  WLB_REQUIRE((flags & ~(WLB_BWD_DKV_BF16 | WLB_BWD_COVERED_ONLY)) == 0,
              "unknown backward flags 0x%x", flags);
  WLB_REQUIRE(kv_head_begin >= 0 && kv_head_count >= 0 && kv_head_begin + kv_head_count <= Hkv,
              "KV head range [%d, %d) outside [0, %d)", kv_head_begin,
              kv_head_begin + kv_head_count, Hkv);
  if (kv_head_count == 0) return WLB_OK;
  const int bf = (flags & WLB_BWD_DKV_BF16) != 0;
  const bool cov = (flags & WLB_BWD_COVERED_ONLY) != 0;
  const wlb::CpSync none = wlb::cp_sync_none();
  if (D == 64)
    return wlb::launch_bwd<64>(q, k, v, o, do_, lse, dq, dk, dv, rowset_off, doc_start, n_docs,
                               positions, Tl, T, Hq, Hkv, scale, ws, bf, cov, kv_head_begin,
                               kv_head_count, none, (cudaStream_t)stream);
  return wlb::launch_bwd<128>(q, k, v, o, do_, lse, dq, dk, dv, rowset_off, doc_start, n_docs,
                              positions, Tl, T, Hq, Hkv, scale, ws, bf, cov, kv_head_begin,
                              kv_head_count, none, (cudaStream_t)stream);
}

extern "C" int wlb_attn_bwd_sync(const void* q, const void* k, const void* v, const void* o,
                                 const void* do_, const float* lse, void* dq, void* dk, void* dv,
                                 const int32_t* rowset_off, const int32_t* doc_start,
                                 int32_t n_docs, const int32_t* positions, int32_t Tl, int32_t T,
                                 int32_t Hq, int32_t Hkv, int32_t D, float scale, void* ws,
                                 int32_t flags, const WlbCpSync* sync, void* stream) {
  WLB_REQUIRE(D == 64 || D == 128, "head dim %d unsupported (64 or 128)", D);
  WLB_REQUIRE(Hq > 0 && Hkv > 0 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  WLB_REQUIRE(Tl >= 0 && T > 0 && n_docs >= 0 && ws != nullptr, "bad sizes");
  WLB_REQUIRE((flags & ~(WLB_BWD_DKV_BF16 | WLB_BWD_COVERED_ONLY)) == 0,
              "unknown backward flags 0x%x", flags);
  WLB_REQUIRE(!sync || (sync->cp >= 1 && sync->kv_per_group >= 1 &&
                        Hkv % sync->kv_per_group == 0 && sync->counters),
              "bad CP sync descriptor");
  const int bf = (flags & WLB_BWD_DKV_BF16) != 0;
  const bool cov = (flags & WLB_BWD_COVERED_ONLY) != 0;
  const wlb::CpSync s = wlb::cp_sync_from(sync);
  if (D == 64)
    return wlb::launch_bwd<64>(q, k, v, o, do_, lse, dq, dk, dv, rowset_off, doc_start, n_docs,
                               positions, Tl, T, Hq, Hkv, scale, ws, bf, cov, 0, Hkv, s,
                               (cudaStream_t)stream);
  return wlb::launch_bwd<128>(q, k, v, o, do_, lse, dq, dk, dv, rowset_off, doc_start, n_docs,
                              positions, Tl, T, Hq, Hkv, scale, ws, bf, cov, 0, Hkv, s,
                              (cudaStream_t)stream);
}

extern "C" int wlb_attn_bwd_ex(const void* q, const void* k, const void* v, const void* o,
                               const void* do_, const float* lse, void* dq, void* dk, void* dv,
                               const int32_t* rowset_off, const int32_t* doc_start, int32_t n_docs,
                               const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                               int32_t Hkv, int32_t D, float scale, void* ws, int32_t flags,
                               void* stream) {
  return wlb_attn_bwd_heads(q, k, v, o, do_, lse, dq, dk, dv, rowset_off, doc_start, n_docs,
                            positions, Tl, T, Hq, Hkv, D, scale, ws, flags, 0, Hkv, stream);
}

extern "C" int wlb_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                            const void* do_, const float* lse, void* dq, float* dk, float* dv,
                            const int32_t* rowset_off, const int32_t* doc_start, int32_t n_docs,
                            const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                            int32_t Hkv, int32_t D, float scale, void* ws, void* stream) {
  return wlb_attn_bwd_ex(q, k, v, o, do_, lse, dq, dk, dv, rowset_off, doc_start, n_docs,
                         positions, Tl, T, Hq, Hkv, D, scale, ws, 0, stream);
}
