// Expert-parallel MoE routing / dispatch / combine (filled in below the GEMM milestone).
#include <cuda_runtime.h>

#include "tf_internal.h"
#include "tf_team.h"

using tf::fail;

extern "C" {
int tf_moe_topk(const float*, int64_t, int, int, int32_t*, float*, void*) {
  return fail(TF_ERR_CONFIG, "tf_moe_topk: not built yet");
}
int tf_moe_count(const int32_t*, int64_t, int, int, int32_t*, int32_t*, void*) {
  return fail(TF_ERR_CONFIG, "tf_moe_count: not built yet");
}
int tf_moe_dispatch(tf_team*, int, const void*, int64_t, int64_t, const int32_t*, int, int,
                    const int32_t*, const int32_t*, uint64_t, int, void*) {
  return fail(TF_ERR_CONFIG, "tf_moe_dispatch: not built yet");
}
int tf_moe_combine(tf_team*, int, uint64_t, int64_t, const int32_t*, const float*, int64_t, int,
                   int, const int32_t*, const int32_t*, void*, int, void*) {
  return fail(TF_ERR_CONFIG, "tf_moe_combine: not built yet");
}
}
