// prefill.cu — K3: branch-masked prefill attention (tcgen05 / TMEM / TMA). Work in progress.
#include "common.cuh"

using namespace mv;

extern "C" size_t mv_prefill_workspace_size(int32_t n, int32_t q_heads, int32_t kv_heads) {
  (void)q_heads;
  (void)kv_heads;
  return (size_t)n * 64 + 4096;
}

extern "C" mv_status mv_attn_prefill(const void*, const void*, const void*, const int32_t*, const int32_t*, int32_t,
                                     int32_t, int32_t, int32_t, double, void*, void*, size_t, mv_stream_t) {
  return fail(MV_ERR_INVALID_ARGUMENT, "mv_attn_prefill: not built yet");
}
