// Document-prefix causal attention, forward, on sm_100a tensor cores.
//
// The reference only PRICES this computation (sharding.py:19-21 -- a local
// query range [s, e) of a document attends that document's causal prefix
// [0, e); block-diagonal causal mask, workload.py:3-4).  Here it is executed.
//
// Work item = (tile pair, query head).  A tile pair is two adjacent <= 128-row
// query tiles X (later rows, longer KV extent) and Y (earlier rows; may be
// absent) of one (rank, document) row-set (built by wlb_attn_tiles).  Row i
// attends keys [kv_begin, kv_begin + pos_i + 1) of the document-ordered K/V;
// only KV tiles below X's largest position are visited (per-document block
// skipping) and each K/V tile is loaded ONCE for both query tiles.
//
// Warp roles (384 threads, 1 CTA / SM):
//   warp 0       TMA producer: Q_X, Q_Y once, then K_j / V_j (2-stage rings)
//   warp 1       MMA issuer (warp-uniform, elected lane):
//                  S_X = Q_X K_j^T, S_Y = Q_Y K_j^T          (SS, M=128 N=128)
//                  O_X += P_X V_j,  O_Y += P_Y V_j            (TS: P read from TMEM)
//                ordered PV(j-1) -> QK(j) per tile so the two tiles ping-pong
//   warp 2       TMEM allocator
//   warps 4..7   softmax of tile X, warps 8..11 softmax of tile Y: one query
//                row per thread (TMEM lane); exp2-domain online softmax with
//                lazy O rescaling (only when a row max grows by > 2^8); P is
//                written back as packed bf16 over the first 64 columns of its
//                own S (tcgen05.st) and consumed by the TS MMA.
// TMEM: S_X [0,128)  S_Y [128,256)  O_X [256,256+D)  O_Y [256+D,256+2D)
#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

#ifndef WLB_HPC_ROWS
#define WLB_HPC_ROWS 4096   // several heads per CTA below this many local rows per document
                           // (2048-row documents: fwd +5%, bwd +3% vs a 2048 threshold;
                           //  8192 cost a 6-document 32K sequence 7% in the forward;
                           //  N=4 128K bench: 2048/4096/8192 within noise,
                           //  profiles/r01c_ab_hpc_rows_n4.txt)
#endif

#include <algorithm>

#ifndef WLB_FWD_TURNS
#define WLB_FWD_TURNS 0   // 1: strict X/Y alternation of the softmax warpgroups
                          //    (measured 7% slower: a lone softmax warp is
                          //    issue/MUFU-latency bound, not contended)
#endif
#ifndef WLB_FWD_MMA8
#define WLB_FWD_MMA8 1   // 8-MMA chains under one elect.sync (fewer issue slots on the MMA warp's SMSP)
#endif
#ifndef WLB_FWD_POLY
#define WLB_FWD_POLY 3   // column pairs (of every 8) whose exp2 runs on the FMA pipe
#endif

namespace wlb {
using namespace sm100;

#ifdef WLB_TRACE
// development aid: per-KV-step clock64 stamps of the first CTA
__device__ long long g_fwd_trace[12][256];
#define FTRACE(ev, j)                                                           \
  do {                                                                          \
    if (blockIdx.x == 0 && (j) < 256 && (threadIdx.x & 31) == 0 &&              \
        (threadIdx.x >> 5) == ((ev) < 2 || (ev) == 8 ? 1 : (ev) < 5 || (ev) > 8 ? 4 : 8))   \
      g_fwd_trace[ev][j] = clock64();                                           \
  } while (0)
#else
#define FTRACE(ev, j) \
  do {                \
  } while (0)
#endif

template <int D>
struct FwdCfg {
  static constexpr int BM = 128, BN = 128, STAGES = 2;
  static constexpr int SLABS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int OFF_Q = 0;                            // Q_X | Q_Y
  static constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + STAGES * KV_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t COL_S = 0;       // + tile * 128
  static constexpr uint32_t COL_O = 256;     // + tile * D
  static constexpr uint32_t IDESC_QK = idesc_bf16(BM, BN, 0, 0);
  static constexpr uint32_t IDESC_PV = idesc_bf16(BM, D, 0, 1);
  static constexpr int THREADS = 384;
};

struct FwdBars {
  uint64_t q_full, q_empty;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_full[2], pv_done[2];   // per query tile (X = 0, Y = 1)
  uint32_t tmem_base;
};

template <int D>
__global__ void __launch_bounds__(384, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out,
                float* __restrict__ lse, const int4* __restrict__ items,
                const int* __restrict__ n_items, const int* __restrict__ positions, int Tl,
                int Hq, int Hkv, int n_slots, int hpc, int h_begin, int h_end, float scale_log2,
                const CpSync sync) {
  using C = FwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  // head-major order (LPT within a head): resident CTAs share one head's K/V in L2.
  // A CTA runs heads [h0, h0 + nh) of its tile pair back to back (hpc > 1 for
  // short row-sets): the next head's Q and K/V loads and its first QK overlap
  // this head's last PV and epilogue instead of a CTA teardown + launch.
  // Query heads [h_begin, h_end) of the launch (all heads, or one head group
  // of the CP exchange's head-group pipeline).
  const int item = blockIdx.x % n_slots, h0 = h_begin + (blockIdx.x / n_slots) * hpc;
  if (item >= n_items[0]) return;
  const int nh = min(hpc, h_end - h0);
  const int4 tx = items[2 * item], ty = items[2 * item + 1];
  // item invariants: rows inside [0, Tl), tile Y directly before X, KV
  // extents past kv_begin
  WLB_DCHECK(tx.x >= 0 && tx.y >= 1 && tx.y <= 128 && tx.x + tx.y <= Tl);
  WLB_DCHECK(ty.y == 0 || (ty.y <= 128 && ty.x >= 0 && ty.x + ty.y == tx.x));
  WLB_DCHECK(tx.w > tx.z && (ty.y == 0 || (ty.z > tx.z && ty.z <= tx.w)));
  WLB_DCHECK(h0 >= 0 && h0 < h_end && h_end <= Hq);
  // tile 0 = X {row0, nrows, kv_end}, tile 1 = Y
  const int kv_begin = tx.z;
  const int n_kv[2] = {(tx.w - kv_begin + C::BN - 1) / C::BN,
                       ty.y ? (ty.z - kv_begin + C::BN - 1) / C::BN : 0};
  const int group = Hq / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  FwdBars* bars = reinterpret_cast<FwdBars*>(smem + C::OFF_BAR);
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], 128);
      mbar_init(&bars->pv_done[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&bars->tmem_base, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer --
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    int waited = -1;                 // head group whose peers' K/V are known landed
    for (int hh = 0; hh < nh; ++hh) {
      const int h = h0 + hh, kvh = h / group;
      if (kvh / sync.kv_per_group != waited) {   // CP: the group's K/V rows have landed
        waited = kvh / sync.kv_per_group;
        cp_sync_wait_group(sync, waited, lane);
      }
      if (hh > 0) mbar_wait(&bars->q_empty, (hh - 1) & 1);   // last QK of head hh-1 done
      mbar_expect_tx_w(&bars->q_full, (ty.y ? 2 : 1) * C::Q_BYTES);
      for (int s = 0; s < C::SLABS; ++s) {
        tma_load_3d_w(sQ + s * C::BM * 128, &tmQ, &bars->q_full, s * 64, h, tx.x);
        if (ty.y)
          tma_load_3d_w(sQ + C::Q_BYTES + s * C::BM * 128, &tmQ, &bars->q_full, s * 64, h, ty.x);
      }
      for (int j = 0; j < n_kv[0]; ++j) {
        const int jj = hh * n_kv[0] + j;          // K/V ring position across heads
        const int st = jj % C::STAGES;
        const uint32_t ph = (jj / C::STAGES) & 1;
        const int row = kv_begin + j * C::BN;
        mbar_wait(&bars->k_empty[st], ph ^ 1);
        mbar_expect_tx_w(&bars->k_full[st], C::KV_BYTES);
        for (int s = 0; s < C::SLABS; ++s)
          tma_load_3d_w(sK + st * C::KV_BYTES + s * C::BN * 128, &tmK, &bars->k_full[st], s * 64,
                        kvh, row);
        mbar_wait(&bars->v_empty[st], ph ^ 1);
        mbar_expect_tx_w(&bars->v_full[st], C::KV_BYTES);
        for (int s = 0; s < C::SLABS; ++s)
          tma_load_3d_w(sV + st * C::KV_BYTES + s * C::BN * 128, &tmV, &bars->v_full[st], s * 64,
                        kvh, row);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer --
    const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
#if WLB_FWD_MMA8
    // one elect.sync per 8-MMA chain, descriptors as base + constant offsets
    uint32_t koff[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) koff[kk] = ((kk >> 2) * C::BN * 128 + (kk & 3) * 32) >> 4;
    auto qk = [&](int t, int jj) {           // S_t = Q_t K_jj^T
      const int st = jj % C::STAGES;
      static_assert(D == 128 || D == 64, "head dim");
      if (D == 128) {
        uint32_t qoff[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) qoff[kk] = ((kk >> 2) * C::BM * 128 + (kk & 3) * 32) >> 4;
        mma_ss8_w(tmem + C::COL_S + t * 128, sdesc_sw128(q_base + t * C::Q_BYTES, 16, 1024),
                  sdesc_sw128(k_base + st * C::KV_BYTES, 16, 1024), qoff, koff, C::IDESC_QK, 0);
      } else {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t qo = t * C::Q_BYTES + (kk >> 2) * C::BM * 128 + (kk & 3) * 32;
          const uint32_t ko = st * C::KV_BYTES + (kk >> 2) * C::BN * 128 + (kk & 3) * 32;
          mma_ss_w(tmem + C::COL_S + t * 128, sdesc_sw128(q_base + qo, 16, 1024),
                   sdesc_sw128(k_base + ko, 16, 1024), C::IDESC_QK, kk > 0);
        }
      }
      mma_commit_w(&bars->s_full[t]);
    };
    auto pv = [&](int t, int j, int jj) {   // O_t += P_t V_jj, P_t packed bf16 in TMEM
      const int st = jj % C::STAGES;
      mma_ts8_w(tmem + C::COL_O + t * D, tmem + C::COL_S + t * 128, 8,
                sdesc_sw128(v_base + st * C::KV_BYTES, C::BN * 128, 1024), 2048 >> 4, C::IDESC_PV,
                j > 0);
      mma_commit_w(&bars->pv_done[t]);
    };
#else
    auto qk = [&](int t, int jj) {           // S_t = Q_t K_jj^T
      const int st = jj % C::STAGES;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t qo = t * C::Q_BYTES + (kk >> 2) * C::BM * 128 + (kk & 3) * 32;
        const uint32_t ko = st * C::KV_BYTES + (kk >> 2) * C::BN * 128 + (kk & 3) * 32;
        mma_ss_w(tmem + C::COL_S + t * 128, sdesc_sw128(q_base + qo, 16, 1024),
                 sdesc_sw128(k_base + ko, 16, 1024), C::IDESC_QK, kk > 0);
      }
      mma_commit_w(&bars->s_full[t]);
    };
    auto pv = [&](int t, int j, int jj) {   // O_t += P_t V_jj, P_t packed bf16 in TMEM
      const int st = jj % C::STAGES;
#pragma unroll
      for (int kk = 0; kk < C::BN / 16; ++kk)
        mma_ts_w(tmem + C::COL_O + t * D, tmem + C::COL_S + t * 128 + kk * 8,
                 sdesc_sw128(v_base + st * C::KV_BYTES + kk * 2048, C::BN * 128, 1024),
                 C::IDESC_PV, (j > 0) || (kk > 0));
      mma_commit_w(&bars->pv_done[t]);
    };
#endif
    for (int hh = 0; hh < nh; ++hh) {
      const int kb = hh * n_kv[0];            // K/V ring base of this head
      const int sb[2] = {hh * n_kv[0], hh * n_kv[1]};   // per-tile step base
      mbar_wait(&bars->q_full, hh & 1);
      mbar_wait(&bars->k_full[kb % C::STAGES], (kb / C::STAGES) & 1);
      tc_fence_after();
      qk(0, kb);
      if (n_kv[1] > 0) qk(1, kb);
      mma_commit_w(&bars->k_empty[kb % C::STAGES]);
      if (n_kv[0] == 1) mma_commit_w(&bars->q_empty);
      for (int j = 1; j <= n_kv[0]; ++j) {
        const int jp = kb + j - 1, jn = kb + j;
        const int sp = jp % C::STAGES;
        mbar_wait(&bars->v_full[sp], (jp / C::STAGES) & 1);
        if (j < n_kv[0]) mbar_wait(&bars->k_full[jn % C::STAGES], (jn / C::STAGES) & 1);
        FTRACE(8, j - 1);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (j - 1 < n_kv[t]) {
            mbar_wait_fast(&bars->p_full[t], (sb[t] + j - 1) & 1);
            FTRACE(t, j - 1);
            tc_fence_after();
            pv(t, j - 1, jp);                    // reads P_t before QK overwrites S_t
            if (j < n_kv[t]) qk(t, jn);
          }
        }
        mma_commit_w(&bars->v_empty[sp]);
        if (j < n_kv[0]) mma_commit_w(&bars->k_empty[jn % C::STAGES]);
        if (j == n_kv[0] - 1) mma_commit_w(&bars->q_empty);   // last QK of this head issued
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax --
    const int t = (warp - 4) >> 2;           // 0: tile X, 1: tile Y
    const int nkv = n_kv[t];
    if (nkv > 0) {
      const int4 tt = t ? ty : tx;
      const int wq = warp & 3;
      const int r = wq * 32 + lane;
      const bool valid = r < tt.y;
      const int row = tt.x + r;
      const int lim0 = (valid ? positions[row] : 0) + 1;   // allowed keys from kv_begin
      WLB_DCHECK(!valid || lim0 <= nkv * C::BN);
      const uint32_t lane_base = tmem + ((uint32_t)(wq * 32) << 16);
      const uint32_t s_col = lane_base + C::COL_S + t * 128;
      const uint32_t o_col = lane_base + C::COL_O + t * D;
      for (int hh = 0; hh < nh; ++hh) {
      const int h = h0 + hh, sb = hh * nkv;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&bars->s_full[t], (sb + j) & 1);
        FTRACE(2 + 3 * t, j);
        tc_fence_after();
        // all 128 scores of this row in registers (one TMEM wait per tile:
        // a chunked two-pass variant re-reading S measured ~40% slower)
        float sv[C::BN];
#pragma unroll
        for (int c = 0; c < C::BN / 32; ++c) {
          uint32_t u[32];
          tmem_ld32(s_col + c * 32, u);
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(u[i]);
        }
        tmem_ld_wait();
        // Softmax turns: Y(j) runs after X(j), X(j+1) after Y(j), so each
        // warpgroup's exp2 work has the SMSP pipes to itself while the tensor
        // pipe works on the other tile (overlapping them stretched both).
        if (WLB_FWD_TURNS) {
          if (t == 1)
            named_bar_sync(1, 256);
          else if (j >= 1 && j - 1 < n_kv[1])
            named_bar_sync(2, 256);
        }
        FTRACE(3 + 3 * t, j);
        const int lim = lim0 - j * C::BN;
        const bool full = __all_sync(0xffffffffu, lim >= C::BN);
        // row max as 4 independent chains (a single 128-long dependent
        // FMNMX chain sat on the softmax critical path)
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (full) {
#pragma unroll
          for (int c = 0; c < C::BN; ++c) mx[c & 3] = fmaxf(mx[c & 3], sv[c]);
        } else {
#pragma unroll
          for (int c = 0; c < C::BN; ++c) {
            sv[c] = c < lim ? sv[c] : -INFINITY;
            mx[c & 3] = fmaxf(mx[c & 3], sv[c]);
          }
        }
        const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        if (t == 0) FTRACE(9, j);
        const float m_new = fmaxf(m_run, mt * scale_log2);
        const bool rescale = __any_sync(0xffffffffu, m_new > m_run + 8.f);
        const float m_use = rescale ? m_new : m_run;
        const float alpha = ex2(m_run - m_use);
        // P = exp2(S*scale - m), written back as packed bf16 over the first 64
        // columns of S (P chunk c lands in S columns [16c, 16c+16), already
        // consumed).
        // Packed pairs: x = S*scale - m by FFMA2, row sums by FADD2 (two
        // independent accumulators), WLB_FWD_POLY of every 8 column pairs take
        // the FMA-pipe polynomial exp2, the rest the MUFU.
        float2 ls[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m_use, -m_use);
#pragma unroll
        for (int c = 0; c < C::BN / 32; ++c) {
          uint32_t p[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = c * 32 + 2 * i;
            const float2 x = ffma2(make_float2(sv[col], sv[col + 1]), sc2, nm2);
            float2 pp;
            if ((i & 7) < WLB_FWD_POLY) {
              pp = ex2_poly2(x);
            } else {
              pp.x = ex2(x.x);
              pp.y = ex2(x.y);
            }
            ls[i & 1] = fadd2(ls[i & 1], pp);
            p[i] = pack_bf16(pp.x, pp.y);
          }
          tmem_st16(s_col + c * 16, p);
        }
        if (t == 0) FTRACE(10, j);
        l_run = l_run * alpha + ((ls[0].x + ls[0].y) + (ls[1].x + ls[1].y));
        if (rescale && j > 0) {                // PV(j-1) complete (ordered before QK(j))
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t u[32];
            tmem_ld32(o_col + c * 32, u);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
            tmem_st32(o_col + c * 32, u);
          }
        }
        tmem_st_wait();
        if (t == 0) FTRACE(11, j);
        tc_fence_before();
        FTRACE(4 + 3 * t, j);
        mbar_arrive(&bars->p_full[t]);
        if (WLB_FWD_TURNS) {
          if (t == 0 && j < n_kv[1])
            named_bar_arrive(1, 256);
          else if (t == 1 && j + 1 < n_kv[0])
            named_bar_arrive(2, 256);
        }
        m_run = m_use;
      }
      // ---------------------------------------------------------- epilogue --
      mbar_wait(&bars->pv_done[t], (sb + nkv - 1) & 1);
      tc_fence_after();
      const float inv_l = 1.f / l_run;
      __nv_bfloat16* orow = out + ((size_t)row * Hq + h) * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(o_col + c * 32, u);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = pack_bf16(__uint_as_float(u[2 * i]) * inv_l, __uint_as_float(u[2 * i + 1]) * inv_l);
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        }
      }
      if (valid) lse[(size_t)h * Tl + row] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
      // (the next head's first PV overwrites O_t only after this warpgroup's
      //  p_full of that head's first step, i.e. after these TMEM loads)
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, C::TMEM_COLS);
}

#ifndef WLB_HPC
#define WLB_HPC 4   // heads per CTA for short row-sets (2 measured the same, 8 up to 17% slower)
#endif
static int g_fwd_hpc_short = WLB_HPC;

template <int D>
static int launch_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                      const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                      const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv,
                      int32_t h_begin, int32_t h_count, float scale, const CpSync& sync,
                      cudaStream_t stream) {
  using C = FwdCfg<D>;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_thd_tmap(&tq, q, Tl, Hq, D, C::BM))) return rc;
  if ((rc = make_thd_tmap(&tk, k, T, Hkv, D, C::BN))) return rc;
  if ((rc = make_thd_tmap(&tv, v, T, Hkv, D, C::BN))) return rc;
  WLB_SMEM_ATTR(attn_fwd_kernel<D>, C::SMEM);
  const float scale_log2 = scale * 1.4426950408889634f;
  // Heads per CTA: max_tiles = Tl/256 + n_docs + 1 (attention.py), so its excess
  // over Tl/256 counts the documents.  Short row-sets (< 2048 local rows per
  // document on average) get 4 heads per CTA to amortise the per-CTA latency.
  // Only when that still leaves >= 6 waves of CTAs (a small rank's few tiles
  // need the parallelism more: config-5 ranks of ~4K rows lost 10% with it).
  const long long docs = std::max<long long>(1, (long long)max_tiles - Tl / (2 * C::BM) - 1);
  const int hpc = (h_count % g_fwd_hpc_short == 0 && (long long)Tl < (long long)WLB_HPC_ROWS * docs &&
                   (long long)max_tiles * h_count >= 6LL * 148 * g_fwd_hpc_short)
                      ? g_fwd_hpc_short : 1;
  attn_fwd_kernel<D><<<(unsigned)max_tiles * ((h_count + hpc - 1) / hpc), C::THREADS, C::SMEM,
                       stream>>>(
      tq, tk, tv, (__nv_bfloat16*)o, lse, (const int4*)tiles, n_tiles, positions, Tl, Hq, Hkv,
      max_tiles, hpc, h_begin, h_begin + h_count, scale_log2, sync);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

}  // namespace wlb

#ifdef WLB_TRACE
extern "C" int wlb_debug_fwd_trace(void* host) {
  WLB_CUDA_TRY(cudaMemcpyFromSymbol(host, wlb::g_fwd_trace, sizeof(wlb::g_fwd_trace)));
  return WLB_OK;
}
#endif

extern "C" int wlb_attn_fwd_heads(const void* q, const void* k, const void* v, void* o, float* lse,
                                  const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                                  const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                                  int32_t Hkv, int32_t D, float scale, int32_t kv_head_begin,
                                  int32_t kv_head_count, void* stream) {
  WLB_REQUIRE(D == 64 || D == 128, "head dim %d unsupported (64 or 128)", D);
  WLB_REQUIRE(Hq > 0 && Hkv > 0 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  WLB_REQUIRE(Tl >= 0 && T > 0 && max_tiles >= 0, "bad sizes");
  WLB_REQUIRE(kv_head_begin >= 0 && kv_head_count >= 0 && kv_head_begin + kv_head_count <= Hkv,
              "KV head range [%d, %d) outside [0, %d)", kv_head_begin,
              kv_head_begin + kv_head_count, Hkv);
  if (Tl == 0 || max_tiles == 0 || kv_head_count == 0) return WLB_OK;
  const int g = Hq / Hkv;
  if (D == 64)
    return wlb::launch_fwd<64>(q, k, v, o, lse, tiles, n_tiles, max_tiles, positions, Tl, T, Hq,
                               Hkv, kv_head_begin * g, kv_head_count * g, scale,
                               wlb::cp_sync_none(), (cudaStream_t)stream);
  return wlb::launch_fwd<128>(q, k, v, o, lse, tiles, n_tiles, max_tiles, positions, Tl, T, Hq,
                              Hkv, kv_head_begin * g, kv_head_count * g, scale,
                              wlb::cp_sync_none(), (cudaStream_t)stream);
}

extern "C" int wlb_attn_fwd_sync(const void* q, const void* k, const void* v, void* o, float* lse,
                                 const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                                 const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                                 int32_t Hkv, int32_t D, float scale, const WlbCpSync* sync,
                                 void* stream) {
  WLB_REQUIRE(D == 64 || D == 128, "head dim %d unsupported (64 or 128)", D);
  WLB_REQUIRE(Hq > 0 && Hkv > 0 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  WLB_REQUIRE(Tl >= 0 && T > 0 && max_tiles >= 0, "bad sizes");
  WLB_REQUIRE(!sync || (sync->cp >= 1 && sync->kv_per_group >= 1 &&
                        Hkv % sync->kv_per_group == 0),
              "bad CP sync descriptor");
  if (Tl == 0 || max_tiles == 0) return WLB_OK;
  const wlb::CpSync s = wlb::cp_sync_from(sync);
  if (D == 64)
    return wlb::launch_fwd<64>(q, k, v, o, lse, tiles, n_tiles, max_tiles, positions, Tl, T, Hq,
                               Hkv, 0, Hq, scale, s, (cudaStream_t)stream);
  return wlb::launch_fwd<128>(q, k, v, o, lse, tiles, n_tiles, max_tiles, positions, Tl, T, Hq,
                              Hkv, 0, Hq, scale, s, (cudaStream_t)stream);
}

extern "C" int wlb_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                            const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                            const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                            int32_t Hkv, int32_t D, float scale, void* stream) {
  return wlb_attn_fwd_heads(q, k, v, o, lse, tiles, n_tiles, max_tiles, positions, Tl, T, Hq, Hkv,
                            D, scale, 0, Hkv, stream);
}
