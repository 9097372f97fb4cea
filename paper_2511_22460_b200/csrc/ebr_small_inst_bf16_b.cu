// Latency-path kernel instances (bf16_b); see ebr_small_kernel.cuh.
#include "ebr_small_kernel.cuh"

namespace ebr {
namespace small {
EBR_SMALL_INSTANTIATE(__nv_bfloat16, 16, 1)
EBR_SMALL_INSTANTIATE(__nv_bfloat16, 32, 1)
}  // namespace small
}  // namespace ebr
