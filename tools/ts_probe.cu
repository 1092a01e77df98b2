// Standalone probe (development aid): validates the tcgen05 "TS" MMA form
// D[tmem] = A[tmem] * B[smem] with A = 128x64 bf16 written to TMEM as packed
// bf16 pairs by tcgen05.st, B = 64x64 (K x N) bf16 K-major in SW128 SMEM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o ts_probe ts_probe.cu
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>

#include "../paper_2503_17924_b200/csrc/sm100.cuh"

using namespace wlb::sm100;

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  __shared__ __align__(1024) uint8_t sB[64 * 128];   // 64 rows (n) x 64 k, 128 B rows, SW128
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // B^T rows: n = 0..63, each 64 k-values (128 B), swizzled 16-B chunks
  for (int i = t; i < 64 * 8; i += blockDim.x) {
    int n = i / 8, c = i % 8;
    const uint4* src = reinterpret_cast<const uint4*>(B + n * 64 + c * 8);   // B stored [n][k]
    *reinterpret_cast<uint4*>(sB + n * 128 + ((c ^ (n & 7)) << 4)) = *src;
  }
  fence_proxy_async_smem();
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&tbase, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  // A rows into TMEM columns [64, 96): row m -> lane m, 32 packed bf16 pairs
  {
    uint32_t r[32];
    const int m = t;   // 128 threads
    for (int i = 0; i < 32; ++i) {
      __nv_bfloat162 v = __halves2bfloat162(A[m * 64 + 2 * i], A[m * 64 + 2 * i + 1]);
      r[i] = *reinterpret_cast<uint32_t*>(&v);
    }
    tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 64, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16(128, 64, 0, 0);
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t bdesc = sdesc_sw128(smem_u32(sB) + kk * 32, 16, 1024);
      if (lane == 0) mma_ts(tmem, tmem + 64 + kk * 8, bdesc, idesc, kk > 0);
    }
    if (lane == 0) mma_commit(&bar);
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  for (int c = 0; c < 2; ++c) {
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c * 32, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) D[t * 64 + c * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

int main() {
  const int M = 128, N = 64, K = 64;
  __nv_bfloat16 *hA = new __nv_bfloat16[M * K], *hB = new __nv_bfloat16[N * K];
  float *fA = new float[M * K], *fB = new float[N * K];
  srand(1);
  for (int i = 0; i < M * K; ++i) { fA[i] = (rand() % 17 - 8) / 8.f; hA[i] = __float2bfloat16(fA[i]); }
  for (int i = 0; i < N * K; ++i) { fB[i] = (rand() % 17 - 8) / 8.f; hB[i] = __float2bfloat16(fB[i]); }
  __nv_bfloat16 *dA, *dB; float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
  float* hD = new float[M * N];
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += fA[m * K + k] * fB[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
    }
  printf("TS probe max abs err %.3e -> %s\n", maxerr, maxerr < 1e-3 ? "PASS" : "FAIL");
  return maxerr < 1e-3 ? 0 : 1;
}
