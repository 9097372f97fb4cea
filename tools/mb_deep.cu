// Microbenchmark of the latency kernel's deep stream: per-CTA contiguous row ranges, 16 lanes per
// 256-byte row (fp32 d=64), U loads in flight per lane, dot + shuffle-reduce + store.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r;
}
template <int U, int NW, bool STORE, bool GRIDSTRIDE>
__global__ void __launch_bounds__(NW * 32, 1) k_deep(const char* A, int64_t n, float* out, const float* uvec) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lpr = 16, sub = lane / lpr, li = lane % lpr, rpw = 2;
    float u[4];
    for (int e = 0; e < 4; ++e) u[e] = uvec[li * 4 + e];
    int64_t r0, r1, step, base0;
    if (GRIDSTRIDE) { r0 = 0; r1 = n; step = (int64_t)gridDim.x * NW * rpw * U; base0 = ((int64_t)blockIdx.x * NW + warp) * rpw; }
    else { int64_t R = (n + gridDim.x - 1) / gridDim.x; r0 = blockIdx.x * R; r1 = min(n, r0 + R); step = (int64_t)NW * rpw * U; base0 = r0 + warp * rpw; }
    const int64_t qstride = GRIDSTRIDE ? (int64_t)gridDim.x * NW * rpw : (int64_t)NW * rpw;
    for (int64_t base = base0; base < r1; base += step) {
        uint4 av[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int64_t row = base + q * qstride + sub;
            av[q] = row < r1 ? ldg_stream(A + row * 256 + li * 16) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            float acc = __uint_as_float(av[q].x) * u[0] + __uint_as_float(av[q].y) * u[1] + __uint_as_float(av[q].z) * u[2] + __uint_as_float(av[q].w) * u[3];
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const int64_t row = base + q * qstride + sub;
            if (STORE) { if (li == 0 && row < r1) __stcg(&out[row], acc); }
            else if (acc == 1.2345f) out[0] = acc;
        }
    }
}
int main() {
    const int64_t n = 1000000; const size_t bytes = n * 256;
    char* a; float* out; float* uv; float* fl;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&out, n * 4)); CK(cudaMalloc(&uv, 256)); CK(cudaMalloc(&fl, 512ull << 20));
    CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(uv, 0, 256)); CK(cudaMemset(fl, 0, 512ull << 20));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // clean flush: read 512 MB
    auto flush = [&]() { k_deep<8, 16, false, true><<<sms, 512>>>((const char*)fl, (512ll << 20) / 256, out, uv); cudaDeviceSynchronize(); };
#define RUN(U, NW, ST, GS) { float best = 1e9; for (int r = 0; r < 7; ++r) { flush(); cudaEventRecord(e0); k_deep<U, NW, ST, GS><<<sms, NW * 32>>>(a, n, out, uv); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; } CK(cudaGetLastError()); printf("U=%2d warps=%2d store=%d gridstride=%d: %7.1f us %6.0f GB/s\n", U, NW, ST, GS, best * 1e3, bytes / (best * 1e-3) / 1e9); }
    RUN(8, 12, true, false) RUN(8, 12, false, false) RUN(8, 16, true, false) RUN(8, 16, false, false)
    RUN(16, 12, true, false) RUN(16, 16, true, false) RUN(8, 12, true, true) RUN(8, 16, true, true)
    RUN(16, 16, true, true) RUN(4, 32, true, false) RUN(8, 32, true, false) RUN(8, 32, true, true)
    return 0;
}
