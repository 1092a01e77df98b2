// Development aid: SM -> L2 store / reduction bandwidth per SM (all 148 SMs,
// 16-B per lane, L2-resident footprint), B/clk/SM from clock64.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float4* buf, long long* clk, int iters, int footprint_f4) {
  float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  const int stride = gridDim.x * blockDim.x;
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float4* p = buf + idx;
    if (MODE == 0) *p = v;
    else asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    idx += stride;
    if (idx >= footprint_f4) idx -= footprint_f4;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  const int fp = 16 << 20;   // 16M float4 = 256 MB? use 64 MB footprint below
  float4* buf; long long* clk;
  cudaMalloc(&buf, (size_t)fp * 16); cudaMalloc(&clk, 148 * 8);
  for (int mode = 0; mode < 2; ++mode)
    for (int th = 128; th <= 1024; th *= 2)
      for (int foot : {1 << 20, 4 << 20}) {   // 16 MB, 64 MB
        int iters = 2048;
        for (int rep = 0; rep < 2; ++rep) {
          if (mode == 0) k<0><<<148, th>>>(buf, clk, iters, foot);
          else k<1><<<148, th>>>(buf, clk, iters, foot);
        }
        cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
        double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
        printf("%-6s threads %4d footprint %3d MB: %.1f B/clk/SM\n", mode ? "RED.v4" : "STG.128", th,
               foot * 16 >> 20, (double)th * iters * 16 / c);
      }
  return 0;
}
