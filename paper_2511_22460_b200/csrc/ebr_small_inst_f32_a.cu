// Latency-path kernel instances (f32_a); see ebr_small_kernel.cuh.
#include "ebr_small_kernel.cuh"

namespace ebr {
namespace small {
EBR_SMALL_INSTANTIATE(float, 4, 1)
EBR_SMALL_INSTANTIATE(float, 8, 1)
}  // namespace small
}  // namespace ebr
