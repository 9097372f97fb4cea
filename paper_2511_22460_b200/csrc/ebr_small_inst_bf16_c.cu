// Latency-path kernel instances (bf16_c); see ebr_small_kernel.cuh.
#include "ebr_small_kernel.cuh"

namespace ebr {
namespace small {
EBR_SMALL_INSTANTIATE(__nv_bfloat16, 32, 2)
EBR_SMALL_INSTANTIATE(__nv_bfloat16, 32, 4)
}  // namespace small
}  // namespace ebr
