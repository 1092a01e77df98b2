// The step before the path as ONE tcgen05 kernel: the
// fused QKV projection of a CP rank's local tokens with rotary embeddings at
// the builder's IN-DOCUMENT positions applied in the epilogue.
//
//   y[i, :] = x[rows[i], :] @ W            (rows = the rank's gather_local, or
//                                           identity for already-local x)
//   q / k  = rotate-half RoPE(y's query / key heads) at positions[i]
//   v      = y's value heads
//
// x [R][hidden] bf16, W [hidden][N] bf16 (N = (Hq + 2 Hkv) * D, the
// `x @ W` orientation, so W is the MN-major B operand), q [Tl][Hq][D],
// k / v [Tl][Hkv][D] bf16.  Positions are TokenRange coordinates
// (workload.py:33-45): every document starts at rotary position 0 on every
// rank, whichever chunks it was cut into.
//
// Persistent kernel, one CTA per SM, 128 x 256 output tiles (two D = 128
// heads), K in 64-element steps through a 4-stage TMA ring:
//   warp 0      TMA producer: A rows by tile::gather4 (4 arbitrary rows per
//               instruction, 32 per stage) or one 2-D box; W as 4 MN-major slabs
//   warp 1      MMA issuer: M=128 N=256 K=16 tcgen05 (SS), accumulators double
//               buffered in TMEM (2 x 256 columns) so tile t's epilogue overlaps
//               tile t+1's main loop
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: one output row per thread (TMEM lane), RoPE with the
//               angle pos * theta_i formed in fp64 (theta_i from a per-CTA table)
//               and reduced mod 2 pi before an fp32 sincos (angles reach 1.3e5
//               rad at 128K positions), bf16 16-B stores into THD q / k / v
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace wlb {
using namespace sm100;

namespace proj {
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, D = 128;
constexpr int A_BYTES = BM * BK * 2;          // 16 KB: 128 rows x 128 B (K-major SW128)
constexpr int B_SLAB = BK * 128;              // 8 KB: 64 K-rows x 64 N (MN-major SW128)
constexpr int B_BYTES = (BN / 64) * B_SLAB;   // 32 KB
constexpr int OFF_A = 0;
constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
constexpr int OFF_BAR = OFF_B + STAGES * B_BYTES;
constexpr int SMEM = OFF_BAR + 1024;
constexpr uint32_t IDESC = idesc_bf16(BM, BN, 0, 1);
constexpr int THREADS = 256;
static_assert(SMEM <= 232448, "projection GEMM exceeds the SMEM window");
}  // namespace proj

struct ProjBars {
  uint64_t full[proj::STAGES], empty[proj::STAGES];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
  double theta[proj::D / 2];     // rotary frequencies base^(-2i/D)
};

// per-thread (not elected): every lane of the producer warp gathers its own 4 rows
__device__ __forceinline__ void tma_gather4(void* dst, const void* tmap, uint64_t* bar, int col,
                                            int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_w(void* dst, const void* tmap, uint64_t* bar, int c0,
                                              int c1) {
  asm volatile(
      "{\n\t.reg .pred P;\n\t" WLB_ELECT
      "@P cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n\t}" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// tile t -> (m tile, n tile): n-major sweeps inside groups of GM m-tiles, so
// the CTAs resident at once share a few A row blocks and W column blocks in L2
__device__ __forceinline__ void proj_tile(int t, int mt, int nt, int& m, int& n) {
  constexpr int GM = 16;
  const int group = t / (GM * nt);
  const int first = group * GM;
  const int rows = min(GM, mt - first);
  const int r = t - group * GM * nt;
  m = first + r % rows;
  n = r / rows;
}

__global__ void __launch_bounds__(proj::THREADS, 1)
qkv_proj_rope_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                     const int* __restrict__ rows, int gather, const int* __restrict__ positions,
                     __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                     __nv_bfloat16* __restrict__ v, int Tl, int hidden, int Hq, int Hkv,
                     double log2_base) {
  using namespace proj;
  extern __shared__ uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023) __trap();   // SW128 tiles need 1024-B alignment
  uint8_t* smem = smem_raw;
  ProjBars* bars = reinterpret_cast<ProjBars*>(smem + OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = Hq + 2 * Hkv;
  const int mt = (Tl + BM - 1) / BM, nt = H * D / BN, n_tiles = mt * nt, kb_n = hidden / BK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&bars->full[i], 1);
      mbar_init(&bars->empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->acc_full[i], 1);
      mbar_init(&bars->acc_empty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(&bars->tmem_base, 512);
  if (threadIdx.x >= 128 && threadIdx.x < 128 + D / 2)
    bars->theta[threadIdx.x - 128] = exp2(-(double)(2 * (threadIdx.x - 128)) / D * log2_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ producer --
    tma_prefetch(&tmA);
    tma_prefetch(&tmW);
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      int m, n;
      proj_tile(t, mt, nt, m, n);
      const int m0 = m * BM, n0 = n * BN;
      // this lane's 4 source rows of every gather4 (rows past Tl repeat the
      // last one; their outputs are not stored)
      int src[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = min(m0 + 4 * lane + j, Tl - 1);
        src[j] = gather ? rows[r] : r;
      }
      for (int kb = 0; kb < kb_n; ++kb, ++it) {
        const int st = it % STAGES;
        mbar_wait(&bars->empty[st], ((it / STAGES) & 1) ^ 1);
        mbar_expect_tx_w(&bars->full[st], A_BYTES + B_BYTES);
        uint8_t* sa = smem + OFF_A + st * A_BYTES;
        if (gather) {
          // 32 x 4 rows: lane g's rows land at rows 4g..4g+3 of the slab (the
          // SW128 swizzle follows the shared-memory address, so 512-B pieces
          // compose into the 1024-B atoms of a K-major slab)
          __syncwarp();
          tma_gather4(sa + lane * 4 * 128, &tmA, &bars->full[st], kb * BK, src[0], src[1], src[2],
                      src[3]);
          __syncwarp();
        } else {
          tma_load_2d_w(sa, &tmA, &bars->full[st], kb * BK, m0);
        }
        uint8_t* sb = smem + OFF_B + st * B_BYTES;
        for (int s = 0; s < BN / 64; ++s)
          tma_load_2d_w(sb + s * B_SLAB, &tmW, &bars->full[st], n0 + s * 64, kb * BK);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer --
    const uint32_t a_base = smem_u32(smem + OFF_A), b_base = smem_u32(smem + OFF_B);
    int it = 0, tc = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tc) {
      const int ab = tc & 1;
      mbar_wait(&bars->acc_empty[ab], ((tc >> 1) & 1) ^ 1);   // epilogue drained this buffer
      tc_fence_after();
      const uint32_t acc = tmem + ab * BN;
      for (int kb = 0; kb < kb_n; ++kb, ++it) {
        const int st = it % STAGES;
        mbar_wait_fast(&bars->full[st], (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t a = a_base + st * A_BYTES, b = b_base + st * B_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)   // A K-major: 32 B per K16; B MN-major: 16 rows
          mma_ss_w(acc, sdesc_sw128(a + kk * 32, 16, 1024), sdesc_sw128(b + kk * 2048, B_SLAB, 1024),
                   IDESC, (kb | kk) != 0);
        mma_commit_w(&bars->empty[st]);
      }
      mma_commit_w(&bars->acc_full[ab]);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue --
    const int lg = warp & 3;
    const uint32_t lane_base = tmem + ((uint32_t)(lg * 32) << 16);
    int tc = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tc) {
      int m, n;
      proj_tile(t, mt, nt, m, n);
      const int row = m * BM + lg * 32 + lane;
      const bool valid = row < Tl;
      const int ab = tc & 1;
      const int pos = valid ? positions[row] : 0;
      mbar_wait(&bars->acc_full[ab], (tc >> 1) & 1);
      tc_fence_after();
      // the tile's two heads share every row's rotation angles: cos / sin of
      // 32 frequencies at a time, then both heads' column pairs (i, i + D/2)
      const int h_first = n * (BN / D);
      const bool any_rope = h_first < Hq + Hkv;
#pragma unroll 1
      for (int c = 0; c < D / 2; c += 32) {
        float cs[32], sn[32];
        if (any_rope) {
          constexpr double two_pi = 6.283185307179586, inv_two_pi = 0.15915494309189535;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const double g = (double)pos * bars->theta[c + e];
            sincosf((float)fma(-rint(g * inv_two_pi), two_pi, g), &sn[e], &cs[e]);
          }
        }
#pragma unroll 1
        for (int hh = 0; hh < BN / D; ++hh) {
          const int h = h_first + hh;               // head among q | k | v
          const uint32_t col = lane_base + ab * BN + hh * D;
          __nv_bfloat16* dst;
          if (h < Hq) dst = q + ((size_t)row * Hq + h) * D;
          else if (h < Hq + Hkv) dst = k + ((size_t)row * Hkv + (h - Hq)) * D;
          else dst = v + ((size_t)row * Hkv + (h - Hq - Hkv)) * D;
          const bool rope = h < Hq + Hkv;
          uint32_t lo[32], hi[32];
          tmem_ld32(col + c, lo);
          tmem_ld32(col + c + D / 2, hi);
          tmem_ld_wait();
          uint32_t plo[16], phi[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float a0 = __uint_as_float(lo[2 * e]), a1 = __uint_as_float(lo[2 * e + 1]);
            float b0 = __uint_as_float(hi[2 * e]), b1 = __uint_as_float(hi[2 * e + 1]);
            if (rope) {
              // rotate-half: x'[i] = x[i] cos - x[i+D/2] sin, x'[i+D/2] = x[i+D/2] cos + x[i] sin
              const float c0 = cs[2 * e], s0 = sn[2 * e], c1 = cs[2 * e + 1], s1 = sn[2 * e + 1];
              const float x0 = a0 * c0 - b0 * s0, y0 = b0 * c0 + a0 * s0;
              const float x1 = a1 * c1 - b1 * s1, y1 = b1 * c1 + a1 * s1;
              a0 = x0; b0 = y0; a1 = x1; b1 = y1;
            }
            plo[e] = pack_bf16(a0, a1);
            phi[e] = pack_bf16(b0, b1);
          }
          if (valid) {
            uint4* dlo = reinterpret_cast<uint4*>(dst + c);
            uint4* dhi = reinterpret_cast<uint4*>(dst + c + D / 2);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              dlo[e] = make_uint4(plo[4 * e], plo[4 * e + 1], plo[4 * e + 2], plo[4 * e + 3]);
              dhi[e] = make_uint4(phi[4 * e], phi[4 * e + 1], phi[4 * e + 2], phi[4 * e + 3]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->acc_empty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

static int make_2d_tmap(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                        uint32_t box_inner, uint32_t box_outer) {
  auto enc = tmap_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return WLB_ECUDA;
  }
  cuuint64_t gdim[2] = {inner, outer};
  cuuint64_t gstride[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride,
                   box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) for a %llu x %llu map", (int)r,
              (unsigned long long)outer, (unsigned long long)inner);
    return WLB_ECUDA;
  }
  return WLB_OK;
}

}  // namespace wlb

extern "C" int wlb_qkv_proj_rope(const void* x, int32_t x_rows, const int32_t* rows,
                                 const void* w, void* q, void* k, void* v,
                                 const int32_t* positions, int32_t Tl, int32_t hidden, int32_t Hq,
                                 int32_t Hkv, int32_t D, float base, void* stream) {
  using namespace wlb;
  WLB_REQUIRE(D == proj::D, "head dim %d unsupported (128)", D);
  WLB_REQUIRE(Hq > 0 && Hkv > 0 && Tl >= 0 && x_rows > 0, "bad projection sizes");
  WLB_REQUIRE(hidden > 0 && hidden % proj::BK == 0, "hidden (%d) must be a multiple of %d", hidden,
              proj::BK);
  WLB_REQUIRE(((Hq + 2 * Hkv) * D) % proj::BN == 0, "(Hq + 2 Hkv) * D must be a multiple of %d",
              proj::BN);
  WLB_REQUIRE(rows != nullptr || x_rows >= Tl, "x has %d rows for %d local rows", x_rows, Tl);
  WLB_REQUIRE(base > 1.f, "rope base must be > 1");
  WLB_REQUIRE((((uintptr_t)q | (uintptr_t)k | (uintptr_t)v) & 15) == 0, "outputs must be 16-B aligned");
  if (Tl == 0) return WLB_OK;
  CUtensorMap ta, tw;
  int rc;
  // gather4 boxes are 1 row (4 rows per instruction); the tile load takes 128
  if ((rc = make_2d_tmap(&ta, x, (uint64_t)hidden, (uint64_t)x_rows, proj::BK,
                         rows ? 1 : proj::BM)))
    return rc;
  const int N = (Hq + 2 * Hkv) * D;
  if ((rc = make_2d_tmap(&tw, w, (uint64_t)N, (uint64_t)hidden, 64, proj::BK))) return rc;
  WLB_SMEM_ATTR(qkv_proj_rope_kernel, proj::SMEM);
  int dev = 0, sms = 148;
  WLB_CUDA_TRY(cudaGetDevice(&dev));
  WLB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int tiles = ((Tl + proj::BM - 1) / proj::BM) * (N / proj::BN);
  qkv_proj_rope_kernel<<<std::min(tiles, sms), proj::THREADS, proj::SMEM, (cudaStream_t)stream>>>(
      ta, tw, rows, rows ? 1 : 0, positions, (__nv_bfloat16*)q, (__nv_bfloat16*)k,
      (__nv_bfloat16*)v, Tl, hidden, Hq, Hkv, log2((double)base));
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}
