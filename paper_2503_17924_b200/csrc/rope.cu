// The step before the path: split a fused QKV
// projection into THD Q / K / V and apply rotary position embeddings at the
// builder's IN-DOCUMENT positions (`positions` from wlb_shard_plan: each
// local row's offset inside its document, the TokenRange coordinates of
// workload.py:33-45), so every document starts at rotary position 0 whatever
// CP rank and chunk its rows landed on.  The projection itself is a plain
// GEMM (cuBLAS through torch); this kernel is its epilogue pass.
//
// y [Tl][Hq + 2*Hkv][D] bf16 (query heads, then key heads, then value heads)
// q [Tl][Hq][D], k/v [Tl][Hkv][D] bf16.  Rotate-half (GPT-NeoX / Llama) form:
//   x'[i]       = x[i] cos(t w_i) - x[i + D/2] sin(t w_i)
//   x'[i + D/2] = x[i + D/2] cos(t w_i) + x[i] sin(t w_i),  w_i = base^(-2i/D)
// with the angle formed in fp64 and reduced mod 2 pi (angles reach 1.3e5 rad
// at 128K positions, common.cuh rope_sincos).
#include <cuda_bf16.h>

#include "common.cuh"

namespace wlb {

__global__ void qkv_rope_kernel(const __nv_bfloat162* __restrict__ y, __nv_bfloat162* __restrict__ q,
                                __nv_bfloat162* __restrict__ k, __nv_bfloat162* __restrict__ v,
                                const int* __restrict__ positions, int Tl, int Hq, int Hkv, int D,
                                double log2_base) {
  // one thread per (row, head, pair of rotation indices {2j, 2j+1})
  const int H = Hq + 2 * Hkv, P = D / 4;     // bf16x2 pairs per half-head
  const long long n = (long long)Tl * H * P;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(t % P);
    const long long rh = t / P;
    const int h = (int)(rh % H);
    const int row = (int)(rh / H);
    const __nv_bfloat162* src = y + rh * (D / 2);
    const __nv_bfloat162 a = src[j], b = src[j + P];   // x[2j, 2j+1], x[2j+D/2, 2j+1+D/2]
    __nv_bfloat162* dst;
    if (h < Hq) dst = q + ((long long)row * Hq + h) * (D / 2);
    else if (h < Hq + Hkv) dst = k + ((long long)row * Hkv + (h - Hq)) * (D / 2);
    else {
      dst = v + ((long long)row * Hkv + (h - Hq - Hkv)) * (D / 2);
      dst[j] = a;
      dst[j + P] = b;
      continue;
    }
    const int pos = positions[row];
    const float2 x0 = __bfloat1622float2(a), x1 = __bfloat1622float2(b);
    float s0, c0, s1, c1;
    rope_sincos(pos, 2 * j, D, log2_base, &s0, &c0);       // i = 2j
    rope_sincos(pos, 2 * j + 1, D, log2_base, &s1, &c1);   // i = 2j+1
    dst[j] = __floats2bfloat162_rn(x0.x * c0 - x1.x * s0, x0.y * c1 - x1.y * s1);
    dst[j + P] = __floats2bfloat162_rn(x1.x * c0 + x0.x * s0, x1.y * c1 + x0.y * s1);
  }
}

}  // namespace wlb

extern "C" int wlb_qkv_rope(const void* y, void* q, void* k, void* v, const int32_t* positions,
                            int32_t Tl, int32_t Hq, int32_t Hkv, int32_t D, float base,
                            void* stream) {
  WLB_REQUIRE(Tl >= 0 && Hq > 0 && Hkv > 0 && D > 0 && D % 4 == 0, "bad qkv_rope sizes");
  WLB_REQUIRE(base > 1.f, "rope base must be > 1");
  if (Tl == 0) return WLB_OK;
  const long long n = (long long)Tl * (Hq + 2 * Hkv) * (D / 4);
  const unsigned blocks = (unsigned)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  wlb::qkv_rope_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat162*)y, (__nv_bfloat162*)q, (__nv_bfloat162*)k, (__nv_bfloat162*)v,
      positions, Tl, Hq, Hkv, D, log2((double)base));
  WLB_LAUNCH_CHECK();
  return WLB_OK;
}
