// gemm.cu -- tcgen05 GEMM for the prefill path (placeholder until the kernel lands).
#include "common.cuh"

namespace usk {
usk_status launch_gemm_bf16(const void*, const void*, void*, int32_t, int64_t, int64_t, int64_t, int64_t,
                            cudaStream_t) {
  return fail(USK_EUNSUPPORTED, "usk_linear: T > 1 tensor-core path not built yet");
}
}  // namespace usk
