// Placeholder until the tcgen05 backward lands (next milestone).
#include "common.cuh"

extern "C" size_t wlb_attn_bwd_workspace(int32_t Tl, int32_t T, int32_t Hq, int32_t Hkv, int32_t D) {
  return (size_t)Tl * Hq * D * 4 + (size_t)Hq * Tl * 4;
}

extern "C" int wlb_attn_bwd(const void*, const void*, const void*, const void*, const void*,
                            const float*, void*, float*, float*, const int32_t*, const int32_t*,
                            int32_t, const int32_t*, const int32_t*, int32_t, const int32_t*,
                            int32_t, int32_t, int32_t, int32_t, int32_t, float, void*, void*) {
  wlb::set_error("wlb_attn_bwd: not built yet");
  return WLB_EINVAL;
}
