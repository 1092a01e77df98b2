// C-ABI plumbing: error state, device check, the host-side packer kernel and
// the row-permutation kernels used by the CP exchange.
#include <stdarg.h>
#include <string.h>

#include "common.cuh"

namespace wlb {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// 16-byte vector copies of whole rows; one warp per row keeps each row's
// 128-B lines coalesced (rows are Hkv*D*2 = 512..8192 bytes here).
__global__ void rows_permute_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                    const int* __restrict__ index, long long n_rows,
                                    long long row_vecs, int scatter) {
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_rows;
       r += warps) {
    const long long j = index[r];
    const int4* s = src + (scatter ? r : j) * row_vecs;
    int4* d = dst + (scatter ? j : r) * row_vecs;
    for (long long c = lane; c < row_vecs; c += 32) d[c] = s[c];
  }
}

static int rows_permute(const void* src, void* dst, const int32_t* index, int64_t n_rows,
                        int64_t row_bytes, void* stream, int scatter) {
  WLB_REQUIRE(row_bytes > 0 && row_bytes % 16 == 0, "row_bytes must be a positive multiple of 16");
  WLB_REQUIRE(((uintptr_t)src | (uintptr_t)dst) % 16 == 0, "rows must be 16-byte aligned");
  if (n_rows <= 0) return WLB_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long blocks = (n_rows + 7) / 8;
  if (blocks > sms * 16LL) blocks = sms * 16LL;
  rows_permute_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(
      (const int4*)src, (int4*)dst, index, n_rows, row_bytes / 16, scatter);
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}

}  // namespace wlb

using namespace wlb;

extern "C" int32_t wlb_abi_version(void) { return 1; }

extern "C" const char* wlb_last_error(void) { return g_err; }

extern "C" int wlb_device_check(void) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_error("no CUDA device visible (%s)", e == cudaSuccess ? "count 0" : cudaGetErrorString(e));
    return WLB_ENODEV;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    set_error("device %d has compute capability %d.x; this library is built for sm_100a", dev, major);
    return WLB_ENODEV;
  }
  return WLB_OK;
}

// Host: the packer stays on the CPU (north star), natively.  Same algorithm,
// integer widths and fp64 expression order as _compiled.pyx:50-86, so the
// placement is bit-identical (pinned by tests/golden/kernels.json.gz).
extern "C" int wlb_heuristic_fill(const int64_t* lengths, int64_t n, int32_t n_mb, int64_t l_max,
                                  double attn_coeff, double linear_coeff, int32_t* out) {
  WLB_REQUIRE(n_mb >= 1, "n_mb must be >= 1");
  WLB_REQUIRE(n >= 0, "n must be >= 0");
  long long* bin_len = new long long[2 * (size_t)n_mb]();
  long long* bin_pairs = bin_len + n_mb;
  for (int64_t i = 0; i < n; ++i) {
    const long long d = lengths[i];
    // lowest modeled latency W = attn_coeff*pairs + linear_coeff*len; ties -> lowest index
    int pick = 0;
    double best = attn_coeff * (double)bin_pairs[0] + linear_coeff * (double)bin_len[0];
    for (int j = 1; j < n_mb; ++j) {
      const double w = attn_coeff * (double)bin_pairs[j] + linear_coeff * (double)bin_len[j];
      if (w < best) {
        best = w;
        pick = j;
      }
    }
    if (bin_len[pick] + d > l_max) {
      // fallback: the shortest bin, if the document fits there
      int shortest = 0;
      for (int j = 1; j < n_mb; ++j)
        if (bin_len[j] < bin_len[shortest]) shortest = j;
      pick = bin_len[shortest] + d <= l_max ? shortest : -1;
    }
    out[i] = pick;
    if (pick >= 0) {
      bin_len[pick] += d;
      bin_pairs[pick] += d * (d + 1) / 2;
    }
  }
  delete[] bin_len;
  return WLB_OK;
}

extern "C" int wlb_rows_scatter(const void* src, void* dst, const int32_t* index, int64_t n_rows,
                                int64_t row_bytes, void* stream) {
  return rows_permute(src, dst, index, n_rows, row_bytes, stream, 1);
}

extern "C" int wlb_rows_gather(const void* src, void* dst, const int32_t* index, int64_t n_rows,
                               int64_t row_bytes, void* stream) {
  return rows_permute(src, dst, index, n_rows, row_bytes, stream, 0);
}
