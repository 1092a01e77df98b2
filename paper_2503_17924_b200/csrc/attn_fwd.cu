// Document-prefix causal attention, forward, on sm_100a tensor cores.
//
// The reference only PRICES this computation (sharding.py:19-21 — a local
// query range [s, e) of a document attends that document's causal prefix
// [0, e); block-diagonal causal mask, workload.py:3-4).  Here it is executed:
//
//   work item = (query tile, query head).  A query tile is <= 128 local rows of
//   one (rank, document) row-set (built by wlb_attn_tiles); row i may attend
//   keys [kv_begin, kv_begin + pos_i + 1) of the document-ordered K/V.
//   Only KV tiles below the tile's largest position are visited (per-document
//   block skipping); per-row masks are applied only where a row's causal
//   limit falls inside the KV tile.
//
// Warp roles (256 threads, 1 CTA / SM):
//   warp 0      TMA producer: Q once, then K_j / V_j into 2-stage rings
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into TMEM (double
//               buffered), O += P_{j-1} V_{j-1} with O resident in TMEM
//   warp 2      TMEM allocator
//   warps 4..7  softmax: one query row per thread (TMEM lane), online softmax
//               in the exp2 domain with lazy O rescaling (only when a row max
//               grows by > 2^8), P written to SMEM (128-B swizzle, K-major) as
//               the A operand of the P.V MMA; final normalisation + store.
#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace wlb {
using namespace sm100;

template <int D>
struct FwdCfg {
  static constexpr int BM = 128, BN = 128, STAGES = 2;
  static constexpr int SLABS = D / 64;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int KV_BYTES = BN * D * 2;
  static constexpr int P_BYTES = BM * BN * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * KV_BYTES;
  static constexpr int OFF_P = OFF_V + STAGES * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 512;   // S0 | S1 | O
  static constexpr uint32_t COL_O = 2 * BN;
  static constexpr uint32_t IDESC_QK = idesc_bf16(BM, BN, 0, 0);
  static constexpr uint32_t IDESC_PV = idesc_bf16(BM, D, 0, 1);
};

struct FwdBars {
  uint64_t q_full;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2];
  uint64_t p_full, pv_done;
  uint32_t tmem_base;
};

template <int D>
__global__ void __launch_bounds__(256, 1)
attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out,
                float* __restrict__ lse, const int4* __restrict__ tiles,
                const int* __restrict__ n_tiles, const int* __restrict__ positions, int Tl,
                int Hq, int Hkv, float scale_log2) {
  using C = FwdCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int tile_idx = blockIdx.x / Hq, h = blockIdx.x % Hq;
  if (tile_idx >= n_tiles[0]) return;
  const int4 tile = tiles[tile_idx];   // {row0, nrows, kv_begin, kv_end}
  const int kvh = h / (Hq / Hkv);
  const int n_kv = (tile.w - tile.z + C::BN - 1) / C::BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  FwdBars* bars = reinterpret_cast<FwdBars*>(smem + C::OFF_BAR);
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sK = smem + C::OFF_K;
  uint8_t* sV = smem + C::OFF_V;
  uint8_t* sP = smem + C::OFF_P;

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
      mbar_init(&bars->s_full[i], 1);
    }
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&bars->tmem_base, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer --
    {   // whole warp; one elected lane issues
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      mbar_expect_tx_w(&bars->q_full, C::Q_BYTES);
      for (int s = 0; s < C::SLABS; ++s)
        tma_load_3d_w(sQ + s * C::BM * 128, &tmQ, &bars->q_full, s * 64, h, tile.x);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % C::STAGES;
        const uint32_t ph = (j / C::STAGES) & 1;
        const int row = tile.z + j * C::BN;
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
    {   // whole warp; one elected lane issues
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV),
                     p_base = smem_u32(sP);
      mbar_wait(&bars->q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= n_kv; ++j) {
        if (j < n_kv) {
          const int st = j % C::STAGES;
          mbar_wait(&bars->k_full[st], (j / C::STAGES) & 1);
          tc_fence_after();
          const uint32_t s_tmem = tmem + (j & 1) * C::BN;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * C::BM * 128 + (kk & 3) * 32;
            const uint32_t koff = (kk >> 2) * C::BN * 128 + (kk & 3) * 32;
            mma_ss_w(s_tmem, sdesc_sw128(q_base + off, 16, 1024),
                   sdesc_sw128(k_base + st * C::KV_BYTES + koff, 16, 1024), C::IDESC_QK, kk > 0);
          }
          mma_commit_w(&bars->s_full[j & 1]);
          mma_commit_w(&bars->k_empty[st]);
        }
        if (j >= 1) {
          const int jj = j - 1, st = jj % C::STAGES;
          mbar_wait(&bars->p_full, jj & 1);
          mbar_wait(&bars->v_full[st], (jj / C::STAGES) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < C::BN / 16; ++kk) {
            const uint32_t poff = (kk >> 2) * C::BM * 128 + (kk & 3) * 32;
            const uint32_t voff = st * C::KV_BYTES + kk * 16 * 128;
            mma_ss_w(tmem + C::COL_O, sdesc_sw128(p_base + poff, 16, 1024),
                   sdesc_sw128(v_base + voff, C::BN * 128, 1024), C::IDESC_PV, (jj > 0) || (kk > 0));
          }
          mma_commit_w(&bars->pv_done);
          mma_commit_w(&bars->v_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------- softmax --
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const bool valid = r < tile.y;
    const int row = tile.x + r;
    const int lim0 = (valid ? positions[row] : 0) + 1;   // allowed keys from kv_begin
    const uint32_t lane_base = tmem + ((uint32_t)(wq * 32) << 16);
    float m_run = -INFINITY, l_run = 0.f;
    uint8_t* p_row = sP + r * 128;
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&bars->s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float s[C::BN];
#pragma unroll
      for (int c = 0; c < C::BN / 32; ++c) {
        uint32_t u[32];
        tmem_ld32(lane_base + (j & 1) * C::BN + c * 32, u);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(u[i]);
      }
      const int lim = lim0 - j * C::BN;
      float mt = -INFINITY;
      if (__all_sync(0xffffffffu, lim >= C::BN)) {
#pragma unroll
        for (int c = 0; c < C::BN; ++c) {
          s[c] *= scale_log2;
          mt = fmaxf(mt, s[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < C::BN; ++c) {
          s[c] = c < lim ? s[c] * scale_log2 : -INFINITY;
          mt = fmaxf(mt, s[c]);
        }
      }
      const float m_new = fmaxf(m_run, mt);
      const bool rescale = __any_sync(0xffffffffu, m_new > m_run + 8.f);
      const float m_use = rescale ? m_new : m_run;
      const float alpha = ex2(m_run - m_use);
      float lsum = 0.f;
      uint32_t p[C::BN / 2];
#pragma unroll
      for (int c = 0; c < C::BN / 2; ++c) {
        const float p0 = ex2(s[2 * c] - m_use), p1 = ex2(s[2 * c + 1] - m_use);
        lsum += p0 + p1;
        p[c] = pack_bf16(p0, p1);
      }
      l_run = l_run * alpha + lsum;
      if (j >= 1) {
        mbar_wait(&bars->pv_done, (j - 1) & 1);   // O final for j-1, P buffer free
        tc_fence_after();
        if (rescale) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t u[32];
            tmem_ld32(lane_base + C::COL_O + c * 32, u);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * alpha);
            tmem_st32(lane_base + C::COL_O + c * 32, u);
          }
          tmem_st_wait();
        }
      }
#pragma unroll
      for (int c = 0; c < C::BN / 8; ++c) {   // 16-B chunks of 8 keys
        const int slab = c >> 3, cc = c & 7;
        uint4 v = make_uint4(p[4 * c], p[4 * c + 1], p[4 * c + 2], p[4 * c + 3]);
        *reinterpret_cast<uint4*>(p_row + slab * C::BM * 128 + ((cc ^ (r & 7)) << 4)) = v;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->p_full);
      m_run = m_use;
    }
    // ------------------------------------------------------------ epilogue --
    mbar_wait(&bars->pv_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l_run;
    __nv_bfloat16* orow = out + ((size_t)row * Hq + h) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t u[32];
      tmem_ld32(lane_base + C::COL_O + c * 32, u);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        pk[i] = pack_bf16(__uint_as_float(u[2 * i]) * inv_l, __uint_as_float(u[2 * i + 1]) * inv_l);
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
    if (valid) lse[(size_t)h * Tl + row] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, C::TMEM_COLS);
}

template <int D>
static int launch_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                      const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                      const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv,
                      float scale, cudaStream_t stream) {
  using C = FwdCfg<D>;
  CUtensorMap tq, tk, tv;
  int rc;
  if ((rc = make_thd_tmap(&tq, q, Tl, Hq, D, C::BM))) return rc;
  if ((rc = make_thd_tmap(&tk, k, T, Hkv, D, C::BN))) return rc;
  if ((rc = make_thd_tmap(&tv, v, T, Hkv, D, C::BN))) return rc;
  static bool attr = false;
  if (!attr) {
    WLB_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      C::SMEM));
    attr = true;
  }
  const float scale_log2 = scale * 1.4426950408889634f;
  attn_fwd_kernel<D><<<(unsigned)max_tiles * Hq, 256, C::SMEM, stream>>>(
      tq, tk, tv, (__nv_bfloat16*)o, lse, (const int4*)tiles, n_tiles, positions, Tl, Hq, Hkv,
      scale_log2);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

}  // namespace wlb

extern "C" int wlb_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                            const int32_t* tiles, const int32_t* n_tiles, int32_t max_tiles,
                            const int32_t* positions, int32_t Tl, int32_t T, int32_t Hq,
                            int32_t Hkv, int32_t D, float scale, void* stream) {
  WLB_REQUIRE(D == 64 || D == 128, "head dim %d unsupported (64 or 128)", D);
  WLB_REQUIRE(Hq > 0 && Hkv > 0 && Hq % Hkv == 0, "Hq must be a multiple of Hkv");
  WLB_REQUIRE(Tl >= 0 && T > 0 && max_tiles >= 0, "bad sizes");
  if (Tl == 0 || max_tiles == 0) return WLB_OK;
  if (D == 64)
    return wlb::launch_fwd<64>(q, k, v, o, lse, tiles, n_tiles, max_tiles, positions, Tl, T, Hq,
                               Hkv, scale, (cudaStream_t)stream);
  return wlb::launch_fwd<128>(q, k, v, o, lse, tiles, n_tiles, max_tiles, positions, Tl, T, Hq,
                              Hkv, scale, (cudaStream_t)stream);
}
