// Fused CP exchange over NVLink / NVSwitch peer memory (symmetric buffers).
//
// The reference has no collectives; the paper's CP exchange is an
// all-gather of K/V in the forward and a reduce-scatter of dK/dV in the
// backward.  With NCCL that is all-gather -> un-permute to
// document order (an extra HBM pass) and gather-permute -> reduce-scatter.
// Here both are ONE kernel each, on peer-mapped symmetric buffers:
//
//   kv_push   every local row i of K and V is stored straight into EVERY rank's
//             document-ordered full K/V buffer at row gather_local[i]
//             (NVLink stores; the un-permute is free: the destination index
//             is the permutation).
//   dkv_pull  each rank sums, for its own rows, the fp32 dK/dV partials of all
//             ranks (NVLink loads), replacing the permute + reduce-scatter.
//
// One warp per row, 16-byte vectors; cross-rank ordering is done by the
// caller's symmetric-memory barriers on the same stream.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace wlb {

// Coverage test shared by the covered push / pull: does rank `lane` (< cp)
// read (forward K/V) or write (backward dK/dV partials) global row g?  Rank p
// touches document d's keys below min(len_d, roundup128(last local position
// of p in d + 1)): the forward's and the backward's KV tiles are 128 keys
// from the document start.  With SPILL (the push), a rank's last tile of an
// EARLIER document also reads rows past that document's end (up to 127 rows
// into the following documents, under the mask): those rows are pushed too,
// so every row a tile loads belongs to the current micro-batch.  A stale row
// left by an earlier micro-batch would otherwise reach O and dQ as 0 * Inf =
// NaN through the masked P.V / dS products.  (The backward writes dK/dV only
// for keys inside the document, so the pull takes SPILL = false.)  Returns
// the warp's mask of such ranks.
template <bool SPILL>
__device__ __forceinline__ unsigned covering_ranks(int g, int lane, int cp,
                                                   const int* __restrict__ rowset_all, int rs,
                                                   const int* __restrict__ pos_all, long long tl,
                                                   const int* __restrict__ doc_start, int n_docs) {
  int lo = 0, hi = n_docs;                     // last document with doc_start <= g
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (doc_start[mid] <= g) lo = mid;
    else hi = mid;
  }
  bool covers = false;
  if (lane < cp) {
    for (int d = lo; d >= 0; --d) {
      // a tile of document d reaches at most roundup128(len_d) <= len_d + 127
      // rows past its start: documents ending 127+ rows before g cannot
      if (d < lo && doc_start[d + 1] + 127 <= g) break;
      const int r0 = rowset_all[lane * rs + d], r1 = rowset_all[lane * rs + d + 1];
      if (r1 > r0) {
        const int len = doc_start[d + 1] - doc_start[d];
        const int tiles = (pos_all[lane * tl + r1 - 1] + 128) / 128 * 128;
        const int cov = SPILL ? tiles : min(len, tiles);
        if (g - doc_start[d] < cov) {
          covers = true;
          break;
        }
      }
      if (!SPILL) break;
    }
  }
  return __ballot_sync(0xffffffffu, covers);
}

// Push: local row i of K and V (columns [col0, col0 + ncol) of the row, in
// 16-B units: a range of KV heads) is stored at row gather_local[i] of the
// document-ordered buffers of every rank (COVERED: only of the ranks whose
// attention loads it, including a last tile's reads past its document's end).
template <bool COVERED>
__global__ void kv_push_kernel(const int4* __restrict__ k, const int4* __restrict__ v,
                               const int* __restrict__ gidx, long long n_rows, long long row_vecs,
                               long long col0, long long ncol,
                               const unsigned long long* __restrict__ bases, long long k_off,
                               long long v_off, int cp, const int* __restrict__ rowset_all, int rs,
                               const int* __restrict__ pos_all, const int* __restrict__ doc_start,
                               int n_docs) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps) {
    const long long g = gidx[r];
    WLB_DCHECK(g >= 0 && g < n_rows * cp);      // every rank holds T / cp rows
    const unsigned mask = COVERED ? covering_ranks<true>((int)g, lane, cp, rowset_all, rs, pos_all,
                                                         n_rows, doc_start, n_docs)
                                  : 0xffffffffu;
    for (long long c = col0 + lane; c < col0 + ncol; c += 32) {
      const int4 kv = k[r * row_vecs + c], vv = v[r * row_vecs + c];
      for (int p = 0; p < cp; ++p) {
        if (COVERED && !((mask >> p) & 1u)) continue;
        char* base = reinterpret_cast<char*>(bases[p]);
        reinterpret_cast<int4*>(base + k_off)[g * row_vecs + c] = kv;
        reinterpret_cast<int4*>(base + v_off)[g * row_vecs + c] = vv;
      }
    }
  }
}

// Pull: dk[i] = sum over ranks of their dK partial row gather_local[i]
// (columns [col0, col0 + ncol) of the partial row, 16-B units), same for dV,
// summed in fp32 in rank order (deterministic).  BF16: the partials are bf16
// and the fp32 outputs have twice the row bytes.  COVERED: a peer's row is
// read only where that peer's backward wrote it; rank p covers document d's
// keys below min(len_d, roundup128(last local position of p in d + 1)), every
// key past that is an exact zero, so the sums are the same and fewer bytes
// cross NVLink (most under per-sequence shards, where a short document lives
// in one rank's chunk).  rowset_all: [cp][rs] per-rank row-set offsets per
// document; pos_all: [cp][tl] per-rank in-document positions.  OUT16: the
// fp32 sums are stored as bf16 (round to nearest even), half the output bytes.
template <bool COVERED, bool BF16, bool OUT16>
__global__ void dkv_pull_kernel(const unsigned long long* __restrict__ bases, long long dk_off,
                                long long dv_off, const int* __restrict__ gidx, long long n_rows,
                                long long row_vecs, long long col0, long long ncol,
                                void* __restrict__ dk_out, void* __restrict__ dv_out, int cp,
                                const int* __restrict__ rowset_all, int rs,
                                const int* __restrict__ pos_all, long long tl,
                                const int* __restrict__ doc_start, int n_docs) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps) {
    const int g = gidx[r];
    WLB_DCHECK(g >= 0 && g < n_rows * cp);
    const unsigned mask = COVERED ? covering_ranks<false>(g, lane, cp, rowset_all, rs, pos_all, tl,
                                                          doc_start, n_docs)
                                  : 0xffffffffu;
    for (long long c = col0 + lane; c < col0 + ncol; c += 32) {
      float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, b[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int p = 0; p < cp; ++p) {
        if (COVERED && !((mask >> p) & 1u)) continue;
        const char* base = reinterpret_cast<const char*>(bases[p]);
        if (BF16) {
          const uint4 x = reinterpret_cast<const uint4*>(base + dk_off)[g * row_vecs + c];
          const uint4 y = reinterpret_cast<const uint4*>(base + dv_off)[g * row_vecs + c];
          const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&x);
          const __nv_bfloat162* y2 = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 xf = __bfloat1622float2(x2[e]), yf = __bfloat1622float2(y2[e]);
            a[2 * e] += xf.x; a[2 * e + 1] += xf.y;
            b[2 * e] += yf.x; b[2 * e + 1] += yf.y;
          }
        } else {
          const float4 x = reinterpret_cast<const float4*>(base + dk_off)[g * row_vecs + c];
          const float4 y = reinterpret_cast<const float4*>(base + dv_off)[g * row_vecs + c];
          a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
          b[0] += y.x; b[1] += y.y; b[2] += y.z; b[3] += y.w;
        }
      }
      if (OUT16) {
        // one 16-B input vector of fp32 partials (4 values) -> 8 output bytes;
        // of bf16 partials (8 values) -> 16
        uint32_t ka[4], vb[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 x = __floats2bfloat162_rn(a[2 * e], a[2 * e + 1]);
          __nv_bfloat162 y = __floats2bfloat162_rn(b[2 * e], b[2 * e + 1]);
          ka[e] = *reinterpret_cast<uint32_t*>(&x);
          vb[e] = *reinterpret_cast<uint32_t*>(&y);
        }
        if (BF16) {
          reinterpret_cast<uint4*>(dk_out)[r * row_vecs + c] = make_uint4(ka[0], ka[1], ka[2], ka[3]);
          reinterpret_cast<uint4*>(dv_out)[r * row_vecs + c] = make_uint4(vb[0], vb[1], vb[2], vb[3]);
        } else {
          reinterpret_cast<uint2*>(dk_out)[r * row_vecs + c] = make_uint2(ka[0], ka[1]);
          reinterpret_cast<uint2*>(dv_out)[r * row_vecs + c] = make_uint2(vb[0], vb[1]);
        }
      } else if (BF16) {
        float4* dk = reinterpret_cast<float4*>(dk_out);
        float4* dv = reinterpret_cast<float4*>(dv_out);
        dk[(r * row_vecs + c) * 2] = make_float4(a[0], a[1], a[2], a[3]);
        dk[(r * row_vecs + c) * 2 + 1] = make_float4(a[4], a[5], a[6], a[7]);
        dv[(r * row_vecs + c) * 2] = make_float4(b[0], b[1], b[2], b[3]);
        dv[(r * row_vecs + c) * 2 + 1] = make_float4(b[4], b[5], b[6], b[7]);
      } else {
        reinterpret_cast<float4*>(dk_out)[r * row_vecs + c] = make_float4(a[0], a[1], a[2], a[3]);
        reinterpret_cast<float4*>(dv_out)[r * row_vecs + c] = make_float4(b[0], b[1], b[2], b[3]);
      }
    }
  }
}

// Per-peer arrival flags (one int per (slot, kind, head group, source rank) in
// every rank's symmetric flag buffer).  signal: after this rank's stores of a
// head group have completed (the previous kernel on the stream), publish
// `value` into slot flag_off of every peer with a system-scope release.
// wait: spin until the n local flags reach `value` (system-scope acquire),
// so the next kernel on the stream sees every peer's rows.  Values are
// monotonically increasing epochs, so no flag is ever reset.  A wait that
// exceeds 60 s traps (a lost peer must not hang the GPU).
__global__ void signal_kernel(const unsigned long long* __restrict__ bases, long long flag_off,
                              int cp, int value) {
  __threadfence_system();
  for (int p = threadIdx.x; p < cp; p += blockDim.x) {
    int* f = reinterpret_cast<int*>(reinterpret_cast<char*>(bases[p]) + flag_off);
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(value) : "memory");
  }
}

__global__ void wait_kernel(const int* __restrict__ flags, int n, int value) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      int x;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(x) : "l"(flags + i) : "memory");
      if (x >= value) break;
      __nanosleep(128);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 60000000000ull) __trap();
    }
  }
  __syncthreads();
}

// Push/pull blocks (256 threads) per 8 SMs.  The exchange runs on its own
// stream beside the attention kernels, which hold one CTA per SM: a grid of
// 8 blocks per SM took SMs from the attention for the whole exchange (N=4
// bench 3688-3695 TFLOP/s); 2 per SM moves the same bytes under the compute
// with less interference (3746-3750); 1 per 4 SMs left the exchange exposed
// (3385).
#ifndef WLB_XCHG_BLOCKS_PER_SM
#define WLB_XCHG_BLOCKS_PER_SM 16
#endif
static bool aligned16(const void* a, const void* b) {
  return (((uintptr_t)a | (uintptr_t)b) & 15) == 0;
}

static int grid_for(long long n_rows) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long blocks = (n_rows + 7) / 8;
  const long long cap = (long long)sms * WLB_XCHG_BLOCKS_PER_SM / 8;
  if (blocks > cap) blocks = cap;
  return (int)(blocks > 0 ? blocks : 1);
}

}  // namespace wlb

using namespace wlb;

extern "C" int wlb_cp_kv_push_part(const void* k_local, const void* v_local,
                                   const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                                   int64_t col_off, int64_t col_bytes, const uint64_t* peer_bases,
                                   int64_t k_off, int64_t v_off, int32_t cp,
                                   const int32_t* rowset_all, int32_t rowset_stride,
                                   const int32_t* positions_all, const int32_t* doc_start,
                                   int32_t n_docs, void* stream) {
  WLB_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0 && k_off % 16 == 0 && v_off % 16 == 0,
              "rows and offsets must be 16-byte aligned");
  WLB_REQUIRE(col_off >= 0 && col_bytes >= 0 && col_off % 16 == 0 && col_bytes % 16 == 0 &&
                  col_off + col_bytes <= row_bytes,
              "column range [%lld, %lld) must be 16-byte aligned inside the %lld-byte row",
              (long long)col_off, (long long)(col_off + col_bytes), (long long)row_bytes);
  WLB_REQUIRE(aligned16(k_local, v_local), "k_local / v_local must be 16-byte aligned");
  WLB_REQUIRE(cp >= 1, "cp must be >= 1");
  const bool covered = rowset_all != nullptr;
  if (covered) {
    WLB_REQUIRE(cp <= 32, "the covered push needs cp in [1, 32]");
    WLB_REQUIRE(n_docs >= 1 && rowset_stride >= n_docs + 1,
                "bad row-set table (n_docs %d, stride %d)", n_docs, rowset_stride);
  }
  if (n_rows <= 0 || col_bytes == 0) return WLB_OK;
  auto kern = covered ? kv_push_kernel<true> : kv_push_kernel<false>;
  kern<<<grid_for(n_rows), 256, 0, (cudaStream_t)stream>>>(
      (const int4*)k_local, (const int4*)v_local, gather_local, n_rows, row_bytes / 16,
      col_off / 16, col_bytes / 16, (const unsigned long long*)peer_bases, k_off, v_off, cp,
      rowset_all, rowset_stride, positions_all, doc_start, n_docs);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

extern "C" int wlb_cp_dkv_pull_part(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                                    const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                                    int64_t col_off, int64_t col_bytes, float* dk, float* dv,
                                    int32_t cp, int32_t flags, const int32_t* rowset_all,
                                    int32_t rowset_stride, const int32_t* positions_all,
                                    const int32_t* doc_start, int32_t n_docs, void* stream) {
  WLB_REQUIRE((flags & ~(WLB_BWD_DKV_BF16 | WLB_PULL_OUT_BF16)) == 0, "unknown pull flags 0x%x",
              flags);
  WLB_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0 && dk_off % 16 == 0 && dv_off % 16 == 0,
              "rows and offsets must be 16-byte aligned");
  WLB_REQUIRE(col_off >= 0 && col_bytes >= 0 && col_off % 16 == 0 && col_bytes % 16 == 0 &&
                  col_off + col_bytes <= row_bytes,
              "column range [%lld, %lld) must be 16-byte aligned inside the %lld-byte row",
              (long long)col_off, (long long)(col_off + col_bytes), (long long)row_bytes);
  WLB_REQUIRE(aligned16(dk, dv), "dk / dv must be 16-byte aligned");
  WLB_REQUIRE(cp >= 1, "cp must be >= 1");
  const bool covered = rowset_all != nullptr;
  if (covered) {
    WLB_REQUIRE(cp <= 32, "the covered pull needs cp in [1, 32]");
    WLB_REQUIRE(n_docs >= 1 && rowset_stride >= n_docs + 1,
                "bad row-set table (n_docs %d, stride %d)", n_docs, rowset_stride);
  }
  if (n_rows <= 0 || col_bytes == 0) return WLB_OK;
  const bool bf = (flags & WLB_BWD_DKV_BF16) != 0, o16 = (flags & WLB_PULL_OUT_BF16) != 0;
  using K = decltype(&dkv_pull_kernel<true, true, true>);
  const K kerns[2][2][2] = {
      {{dkv_pull_kernel<false, false, false>, dkv_pull_kernel<false, false, true>},
       {dkv_pull_kernel<false, true, false>, dkv_pull_kernel<false, true, true>}},
      {{dkv_pull_kernel<true, false, false>, dkv_pull_kernel<true, false, true>},
       {dkv_pull_kernel<true, true, false>, dkv_pull_kernel<true, true, true>}}};
  // row_bytes / col_* count the partial rows; the local fp32 outputs are
  // twice as long for bf16 partials (bf16 outputs: half as long as fp32)
  kerns[covered][bf][o16]<<<grid_for(n_rows), 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)peer_bases, dk_off, dv_off, gather_local, n_rows, row_bytes / 16,
      col_off / 16, col_bytes / 16, dk, dv, cp, rowset_all, rowset_stride, positions_all, n_rows,
      doc_start, n_docs);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

extern "C" int wlb_cp_kv_push(const void* k_local, const void* v_local, const int32_t* gather_local,
                              int64_t n_rows, int64_t row_bytes, const uint64_t* peer_bases,
                              int64_t k_off, int64_t v_off, int32_t cp, void* stream) {
  return wlb_cp_kv_push_part(k_local, v_local, gather_local, n_rows, row_bytes, 0, row_bytes,
                             peer_bases, k_off, v_off, cp, nullptr, 0, nullptr, nullptr, 0, stream);
}

extern "C" int wlb_cp_kv_push_cov(const void* k_local, const void* v_local,
                                  const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                                  const uint64_t* peer_bases, int64_t k_off, int64_t v_off,
                                  int32_t cp, const int32_t* rowset_all, int32_t rowset_stride,
                                  const int32_t* positions_all, const int32_t* doc_start,
                                  int32_t n_docs, void* stream) {
  WLB_REQUIRE(rowset_all != nullptr, "rowset_all is required");
  return wlb_cp_kv_push_part(k_local, v_local, gather_local, n_rows, row_bytes, 0, row_bytes,
                             peer_bases, k_off, v_off, cp, rowset_all, rowset_stride,
                             positions_all, doc_start, n_docs, stream);
}

extern "C" int wlb_cp_dkv_pull(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                               const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                               float* dk, float* dv, int32_t cp, void* stream) {
  return wlb_cp_dkv_pull_part(peer_bases, dk_off, dv_off, gather_local, n_rows, row_bytes, 0,
                              row_bytes, dk, dv, cp, 0, nullptr, 0, nullptr, nullptr, 0, stream);
}

extern "C" int wlb_cp_dkv_pull_ex(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                                  const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                                  float* dk, float* dv, int32_t cp, int32_t flags, void* stream) {
  return wlb_cp_dkv_pull_part(peer_bases, dk_off, dv_off, gather_local, n_rows, row_bytes, 0,
                              row_bytes, dk, dv, cp, flags, nullptr, 0, nullptr, nullptr, 0,
                              stream);
}

extern "C" int wlb_cp_dkv_pull_cov(const uint64_t* peer_bases, int64_t dk_off, int64_t dv_off,
                                   const int32_t* gather_local, int64_t n_rows, int64_t row_bytes,
                                   float* dk, float* dv, int32_t cp, int32_t flags,
                                   const int32_t* rowset_all, int32_t rowset_stride,
                                   const int32_t* positions_all, const int32_t* doc_start,
                                   int32_t n_docs, void* stream) {
  WLB_REQUIRE(rowset_all != nullptr, "rowset_all is required");
  return wlb_cp_dkv_pull_part(peer_bases, dk_off, dv_off, gather_local, n_rows, row_bytes, 0,
                              row_bytes, dk, dv, cp, flags, rowset_all, rowset_stride,
                              positions_all, doc_start, n_docs, stream);
}

extern "C" int wlb_cp_kv_push_dma(const void* k_local, const void* v_local, const int64_t* runs,
                                  int32_t n_runs, int64_t row_bytes, int64_t col_off,
                                  int64_t col_bytes, const uint64_t* peer_bases, int64_t k_off,
                                  int64_t v_off, int32_t cp, void* stream) {
  WLB_REQUIRE(row_bytes > 0 && col_off >= 0 && col_bytes > 0 && col_off + col_bytes <= row_bytes,
              "bad column range [%lld, %lld) of a %lld-byte row", (long long)col_off,
              (long long)(col_off + col_bytes), (long long)row_bytes);
  WLB_REQUIRE(cp >= 1 && n_runs >= 0 && (n_runs == 0 || runs) && peer_bases, "bad push arguments");
  const char* ks = static_cast<const char*>(k_local);
  const char* vs = static_cast<const char*>(v_local);
  for (int32_t r = 0; r < n_runs; ++r) {
    const int64_t lr = runs[3 * r], gr = runs[3 * r + 1], n = runs[3 * r + 2];
    if (n <= 0) continue;
    for (int32_t p = 0; p < cp; ++p) {
      char* base = reinterpret_cast<char*>(peer_bases[p]);
      WLB_CUDA_TRY(cudaMemcpy2DAsync(base + k_off + gr * row_bytes + col_off, row_bytes,
                                     ks + lr * row_bytes + col_off, row_bytes, col_bytes, n,
                                     cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
      WLB_CUDA_TRY(cudaMemcpy2DAsync(base + v_off + gr * row_bytes + col_off, row_bytes,
                                     vs + lr * row_bytes + col_off, row_bytes, col_bytes, n,
                                     cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    }
  }
  return WLB_OK;
}

// Stream memory operations (executed by the GPU front end, no SM): signal and
// wait on the arrival flags even while attention CTAs hold every SM.
namespace {
typedef CUresult (*StreamValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamValue32Fn memop(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<StreamValue32Fn>(p);
}
}  // namespace

extern "C" int wlb_cp_signal_memop(const uint64_t* flag_bases, int64_t flag_off, int32_t cp,
                                   int32_t value, void* stream) {
  static StreamValue32Fn write = memop("cuStreamWriteValue32");
  WLB_REQUIRE(write != nullptr, "cuStreamWriteValue32 unavailable");
  WLB_REQUIRE(cp >= 1 && flag_off >= 0 && flag_off % 4 == 0 && flag_bases, "bad signal arguments");
  for (int32_t p = 0; p < cp; ++p) {
    // default flags: the write follows a memory barrier over the stream's prior work
    const CUresult r = write((CUstream)stream, (CUdeviceptr)(flag_bases[p] + flag_off),
                             (cuuint32_t)value, CU_STREAM_WRITE_VALUE_DEFAULT);
    WLB_REQUIRE(r == CUDA_SUCCESS, "cuStreamWriteValue32 failed (%d)", (int)r);
  }
  return WLB_OK;
}

extern "C" int wlb_cp_wait_memop(const int32_t* flags, int32_t n, int32_t value, void* stream) {
  static StreamValue32Fn wait = memop("cuStreamWaitValue32");
  WLB_REQUIRE(wait != nullptr, "cuStreamWaitValue32 unavailable");
  WLB_REQUIRE(n >= 0 && ((uintptr_t)flags & 3) == 0, "bad wait arguments");
  for (int32_t i = 0; i < n; ++i) {
    const CUresult r = wait((CUstream)stream, (CUdeviceptr)(flags + i), (cuuint32_t)value,
                            CU_STREAM_WAIT_VALUE_GEQ);
    WLB_REQUIRE(r == CUDA_SUCCESS, "cuStreamWaitValue32 failed (%d)", (int)r);
  }
  return WLB_OK;
}

extern "C" int wlb_cp_signal(const uint64_t* flag_bases, int64_t flag_off, int32_t cp,
                             int32_t value, void* stream) {
  WLB_REQUIRE(cp >= 1 && flag_off >= 0 && flag_off % 4 == 0, "bad signal arguments");
  signal_kernel<<<1, 32 * ((cp + 31) / 32 < 32 ? (cp + 31) / 32 : 32), 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)flag_bases, flag_off, cp, value);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

extern "C" int wlb_cp_wait(const int32_t* flags, int32_t n, int32_t value, void* stream) {
  WLB_REQUIRE(n >= 0 && ((uintptr_t)flags & 3) == 0, "bad wait arguments");
  if (n == 0) return WLB_OK;
  wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(flags, n, value);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}
