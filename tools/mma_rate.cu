// Development aid: raw tcgen05.mma throughput per shape / operand source on
// every SM at once (cycles per instruction, FLOP/clk/SM).  Groups of 8 MMAs
// are unrolled with constant offsets, as in the attention kernels; operand
// contents are whatever SMEM holds (zeros): only timing matters.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <stdio.h>

#include "../paper_2503_17924_b200/csrc/sm100.cuh"

using namespace wlb::sm100;

// MODE: 0 SS K-major | 1 TS (A from TMEM) | 2 SS MN-major A.  NACC chains
// interleaved (independent accumulators).
template <int MODE, int N, int NACC>
__global__ void __launch_bounds__(128, 1) rate(int groups, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t a_b = smem_u32(smem), b_b = smem_u32(smem) + 32 * 1024;
  constexpr uint32_t IDESC = idesc_bf16(128, N, MODE == 2 ? 1 : 0, 0);
  if (warp == 0) {
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
        for (int c = 0; c < NACC; ++c) {
          const uint32_t ko = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint64_t bd = sdesc_sw128(b_b + ko, 16, 1024);
          const uint32_t dst = tmem + c * N;
          if (MODE == 1)
            mma_ts_w(dst, tmem + 384 + kk * 8, bd, IDESC, 1);
          else if (MODE == 2)
            mma_ss_w(dst, sdesc_sw128(a_b + kk * 2048, 16384, 1024), bd, IDESC, 1);
          else
            mma_ss_w(dst, sdesc_sw128(a_b + ko, 16, 1024), bd, IDESC, 1);
        }
      }
    }
    long long t_issue = clock64();
    mma_commit_w(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      out[2 * blockIdx.x] = t1 - t0;
      out[2 * blockIdx.x + 1] = t_issue - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE, int N, int NACC>
static void run(const char* name, int sms, long long* d) {
  const int groups = 1024;
  cudaFuncSetAttribute(rate<MODE, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  rate<MODE, N, NACC><<<sms, 128, 100 * 1024>>>(groups, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  long long h[512];
  cudaMemcpy(h, d, 2 * sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0, iss = 0;
  for (int i = 0; i < sms; ++i) {
    mean += h[2 * i];
    iss += h[2 * i + 1];
  }
  mean /= sms;
  iss /= sms;
  const double n_instr = groups * 8.0 * NACC;
  const double cyc = mean / n_instr, flop = 2.0 * 128 * N * 16;
  const double operand = (MODE == 1 ? 0 : 128 * 16 * 2) + N * 16 * 2;
  printf("%-14s chains %d N=%3d: %6.1f clk/instr (issue %5.1f)  %5.0f FLOP/clk/SM (%3.0f%%)  smem %4.0f B/clk\n",
         name, NACC, N, cyc, iss / n_instr, flop / cyc, 100 * flop / cyc / 8192, operand / cyc);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, 2 * sms * sizeof(long long));
  run<0, 64, 1>("SS K-major", sms, d);
  run<0, 64, 2>("SS K-major", sms, d);
  run<0, 64, 4>("SS K-major", sms, d);
  run<0, 128, 1>("SS K-major", sms, d);
  run<0, 128, 2>("SS K-major", sms, d);
  run<0, 256, 1>("SS K-major", sms, d);
  run<1, 64, 1>("TS (A tmem)", sms, d);
  run<1, 64, 2>("TS (A tmem)", sms, d);
  run<1, 128, 1>("TS (A tmem)", sms, d);
  run<1, 128, 2>("TS (A tmem)", sms, d);
  run<1, 256, 1>("TS (A tmem)", sms, d);
  run<2, 64, 1>("SS MN-major A", sms, d);
  run<2, 64, 2>("SS MN-major A", sms, d);
  run<2, 128, 1>("SS MN-major A", sms, d);
  run<2, 256, 1>("SS MN-major A", sms, d);
  return 0;
}
