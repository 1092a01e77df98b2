// Development aid: MUFU ex2 and FMA-pipe throughput per SM (clock64 around
// unrolled independent chains; 148 CTAs x 128/256/512 threads).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, long long* clk, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (MODE == 1) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      else if (MODE == 3) {
        unsigned h = __float_as_uint(a[i]);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
        a[i] = __uint_as_float(h);
      }
      else {
        float2 v = make_float2(a[i], a[(i + 1) & 7]);
        asm volatile("{.reg .b64 r; mov.b64 r, {%0, %1}; fma.rn.f32x2 r, r, r, r; mov.b64 {%0, %1}, r;}" : "+f"(v.x), "+f"(v.y));
        a[i] = v.x;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 148 * 8);
  const char* names[4] = {"MUFU.EX2", "FFMA", "FFMA2", "EX2.F16x2"};
  for (int mode = 0; mode < 4; ++mode)
    for (int th = 128; th <= 512; th *= 2) {
      int iters = 4096;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, th>>>(out, clk, iters);
        else if (mode == 1) k<1><<<148, th>>>(out, clk, iters);
        else if (mode == 2) k<2><<<148, th>>>(out, clk, iters);
        else k<3><<<148, th>>>(out, clk, iters);
      }
      cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
      double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
      double ops = (double)th * iters * 8 * (mode >= 2 ? 2 : 1);
      printf("%-9s threads/SM %4d: %.2f results/clk/SM\n", names[mode], th, ops / c);
    }
  return 0;
}
