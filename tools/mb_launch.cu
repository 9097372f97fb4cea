// Launch-overhead microbenchmark: device time (CUDA events) of an empty persistent-shaped kernel
// (148 CTAs x 512 threads, 100 KB dynamic smem) launched normally vs cooperatively, back to back
// and with a 256 MB L2-flushing read in between (bench.py's step shape).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void empty_k(int* out) { if (threadIdx.x == 0 && out[blockIdx.x] == 12345) out[0] = 1; }
__global__ void sync_k(int* out) { cg::this_grid().sync(); if (threadIdx.x == 0 && out[blockIdx.x] == 12345) out[0] = 1; }
__global__ void flush_k(const float4* p, size_t n, float* o) {
    float s = 0; for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) { float4 v = __ldcg(p + i); s += v.x; }
    if (s == 123.f) *o = s;
}
int main() {
    int* d; cudaMalloc(&d, 4096); cudaMemset(d, 0, 4096);
    float4* f; size_t nf = (256u << 20) / 16; cudaMalloc(&f, nf * 16); cudaMemset(f, 0, nf * 16); float* o; cudaMalloc(&o, 4);
    const int smem = 100 * 1024;
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sync_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 6; ++mode) {
        float tot = 0; int n = 200;
        for (int i = 0; i < n + 5; ++i) {
            if (mode >= 3) flush_k<<<148 * 4, 512>>>(f, nf, o);
            cudaEventRecord(a);
            void* args[] = {&d};
            int m = mode % 3;
            if (m == 0) empty_k<<<148, 512, smem>>>(d);
            else if (m == 1) cudaLaunchCooperativeKernel((void*)empty_k, 148, 512, args, smem, 0);
            else cudaLaunchCooperativeKernel((void*)sync_k, 148, 512, args, smem, 0);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 5) tot += ms;
        }
        const char* nm[] = {"regular", "cooperative", "coop+grid.sync"};
        printf("%s%s: %.2f us/launch\n", nm[mode % 3], mode >= 3 ? " (after flush)" : "", tot / n * 1000);
    }
    // launch-floor variants: tiny kernel, no smem, and a CUDA graph of the 148 x 512 x 100 KB kernel
    {
        cudaStream_t s; cudaStreamCreate(&s);
        auto timeit = [&](const char* nm, auto fn) {
            float tot = 0; int n = 200;
            for (int i = 0; i < n + 5; ++i) {
                cudaEventRecord(a, s); fn(); cudaEventRecord(b, s); cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 5) tot += ms;
            }
            printf("%s: %.2f us/launch\n", nm, tot / n * 1000);
        };
        timeit("1x32 no smem", [&] { empty_k<<<1, 32, 0, s>>>(d); });
        timeit("148x512 no smem", [&] { empty_k<<<148, 512, 0, s>>>(d); });
        timeit("148x512 100KB", [&] { empty_k<<<148, 512, smem, s>>>(d); });
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        void* args[] = {&d};
        cudaLaunchCooperativeKernel((void*)sync_k, 148, 512, args, smem, s);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        timeit("graph: coop+grid.sync 148x512 100KB", [&] { cudaGraphLaunch(ge, s); });
        timeit("direct: coop+grid.sync 148x512 100KB", [&] { cudaLaunchCooperativeKernel((void*)sync_k, 148, 512, args, smem, s); });
    }
    return 0;
}
