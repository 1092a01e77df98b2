// Shared helpers for the wlbcp sm_100a library: error state, launch checks and
// block-wide scans.  PTX wrappers for TMA / mbarrier / tcgen05 live in sm100.cuh.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/wlbcp.h"

namespace wlb {

// Last error message (per host thread).
void set_error(const char* fmt, ...);

#define WLB_CUDA_TRY(expr)                                                        \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::wlb::set_error("%s failed at %s:%d: %s", #expr, __FILE__, __LINE__,       \
                       cudaGetErrorString(_e));                                   \
      return WLB_ECUDA;                                                           \
    }                                                                             \
  } while (0)

#define WLB_LAUNCH_CHECK() WLB_CUDA_TRY(cudaGetLastError())

#define WLB_REQUIRE(cond, ...)                                                    \
  do {                                                                            \
    if (!(cond)) {                                                                \
      ::wlb::set_error(__VA_ARGS__);                                              \
      return WLB_EINVAL;                                                          \
    }                                                                             \
  } while (0)

// Device-side bounds checks, compiled in with -DWLB_DEBUG_CHECKS (the
// checked build, tools/debug_checks.sh; compute-sanitizer is not available
// on the GPU pool): a violated invariant traps with its location.
#ifdef WLB_DEBUG_CHECKS
#define WLB_DCHECK(cond)                                                          \
  do {                                                                            \
    if (!(cond)) {                                                                \
      printf("WLB_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond,      \
             __FILE__, __LINE__, (int)blockIdx.x, (int)threadIdx.x);              \
      __trap();                                                                   \
    }                                                                             \
  } while (0)
#else
#define WLB_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per-device state, so the "done" flag is a bit per device
// of the calling thread's current device (up to 64 devices).
#define WLB_SMEM_ATTR(kernel, bytes)                                                   \
  do {                                                                                 \
    static unsigned long long _done = 0;                                               \
    int _dev = 0;                                                                      \
    WLB_CUDA_TRY(cudaGetDevice(&_dev));                                                \
    if (!((_done >> (_dev & 63)) & 1ull)) {                                            \
      WLB_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        (bytes)));                                     \
      _done |= 1ull << (_dev & 63);                                                    \
    }                                                                                  \
  } while (0)

// Device-side view of WlbCpSync (wlbcp.h): per-group arrival flags waited
// for by the forward and published by the backward.
struct CpSync {
  const int* wait_flags;
  const unsigned long long* signal_bases;
  long long signal_off;
  int* counters;
  int cp, kv_per_group, epoch;
};

__host__ __device__ __forceinline__ CpSync cp_sync_none() {
  return CpSync{nullptr, nullptr, 0, nullptr, 0, 1, 0};
}

// Spin (one warp) until the cp flags of group g are >= epoch, with a
// system-scope acquire; then order the async proxy (TMA) after it.  Traps
// after 20 s: waiting CTAs hold their SMs, so a caller that lets them start
// before the exchange kernels they wait for are resident can deadlock (see
// SymmExchange.fused_sync).
__device__ __forceinline__ void cp_sync_wait_group(const CpSync& s, int g, int lane) {
  if (!s.wait_flags) return;
  const int* f = s.wait_flags + (size_t)g * s.cp;
  for (int p = lane; p < s.cp; p += 32) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      int x;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(x) : "l"(f + p) : "memory");
      if (x >= s.epoch) break;
      __nanosleep(64);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      // spinning CTAs can starve the exchange kernels of SMs: never hang the GPU
      if (t - t0 > 20000000000ull) __trap();
    }
  }
  __syncwarp();
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// One work unit of head group g is complete (its partial stores issued by
// this CTA's threads, which have all passed a barrier before this call, made
// by one thread): count it; the unit completing the group publishes epoch to
// every peer.
__device__ __forceinline__ void cp_sync_unit_done(const CpSync& s, int g, int target) {
  if (!s.signal_bases) return;
  __threadfence();
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(s.counters + g) : "memory");
  if (old == target - 1) {
    __threadfence_system();
    for (int p = 0; p < s.cp; ++p) {
      int* f = reinterpret_cast<int*>(reinterpret_cast<char*>(s.signal_bases[p]) + s.signal_off +
                                      4ll * s.cp * g);
      asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(s.epoch) : "memory");
    }
  }
}

inline CpSync cp_sync_from(const WlbCpSync* s) {
  if (!s) return CpSync{nullptr, nullptr, 0, nullptr, 0, 1, 0};
  return CpSync{s->wait_flags, reinterpret_cast<const unsigned long long*>(s->signal_bases),
                s->signal_off, s->counters, s->cp, s->kv_per_group, s->epoch};
}

// Rotary angle of in-document position `pos` and frequency index i (of D/2):
// pos * base^(-2i/D) formed in fp64 and reduced to [-pi, pi] before the fp32
// sincos.  Positions reach 1.3e5 at 128K, where an fp32 product is already
// ~7e-3 rad off (a 3.7e-2 error on |q| ~ 4, past the bf16 bar).
__device__ __forceinline__ void rope_sincos(int pos, int i, int D, double log2_base, float* s,
                                            float* c) {
  const double ang = (double)pos * exp2(-(double)(2 * i) / D * log2_base);
  const double two_pi = 6.283185307179586;
  const float r = (float)(ang - rint(ang / two_pi) * two_pi);
  sincosf(r, s, c);
}

// Block-wide exclusive scan of one int64 per thread.  `warp_tot` must hold
// blockDim.x/32 + 1 entries of shared memory.  Returns the exclusive prefix and
// writes the block total to *total (all threads).
__device__ __forceinline__ long long block_exclusive_scan(long long v, long long* warp_tot,
                                                          long long* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    long long t = lane < nwarp ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nwarp) warp_tot[lane] = t;           // inclusive warp prefix
    if (lane == nwarp - 1) warp_tot[nwarp] = t;     // block total
  }
  __syncthreads();
  long long base = warp ? warp_tot[warp - 1] : 0;
  long long res = base + x - v;
  *total = warp_tot[nwarp];
  __syncthreads();
  return res;
}

}  // namespace wlb
