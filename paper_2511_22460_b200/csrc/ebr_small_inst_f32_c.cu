// Latency-path kernel instances (f32_c); see ebr_small_kernel.cuh.
#include "ebr_small_kernel.cuh"

namespace ebr {
namespace small {
EBR_SMALL_INSTANTIATE(float, 32, 2)
EBR_SMALL_INSTANTIATE(float, 32, 4)
}  // namespace small
}  // namespace ebr
