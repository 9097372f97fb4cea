// Latency-path kernel instances (bf16_a); see ebr_small_kernel.cuh.
#include "ebr_small_kernel.cuh"

namespace ebr {
namespace small {
EBR_SMALL_INSTANTIATE(__nv_bfloat16, 4, 1)
EBR_SMALL_INSTANTIATE(__nv_bfloat16, 8, 1)
}  // namespace small
}  // namespace ebr
