// Latency-path kernel instances (f32_b); see ebr_small_kernel.cuh.
#include "ebr_small_kernel.cuh"

namespace ebr {
namespace small {
EBR_SMALL_INSTANTIATE(float, 16, 1)
EBR_SMALL_INSTANTIATE(float, 32, 1)
}  // namespace small
}  // namespace ebr
