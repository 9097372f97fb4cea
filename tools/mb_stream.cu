// Microbenchmark: HBM streaming rate of (a) 16-byte non-allocating vector loads with unroll U,
// (b) a bulk-copy (TMA engine) shared-memory ring with S stages of B bytes, consumed by warps
// that read every staged byte.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(d)), "l"(s), "r"(n), "r"(smem_u32(b)) : "memory");
}

template <int U>
__global__ void __launch_bounds__(512, 1) k_ldg(const uint4* __restrict__ a, size_t n16, float* out) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(a + i + u * stride));
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __uint_as_float(v[u].x) + __uint_as_float(v[u].w);
    }
    for (; i < n16; i += stride) acc += __uint_as_float(a[i].x);
    if (acc == 1.2345f) out[0] = acc;
}

// contiguous per-CTA range, producer lane + (nw-1) consumer warps
__global__ void __launch_bounds__(512, 1) k_tma(const char* __restrict__ a, size_t bytes, int stages, int stage_bytes, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * stage_bytes);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nc = blockDim.x / 32 - 1;
    const size_t per = (bytes / gridDim.x + 4095) & ~(size_t)4095;
    const size_t b0 = per * blockIdx.x, b1 = min(bytes, b0 + per);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nc); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    if (warp == 0) {
        if (lane == 0) {
            uint32_t g = 0;
            for (size_t o = b0; o < b1; o += stage_bytes, ++g) {
                const int slot = g % stages;
                if (g >= (uint32_t)stages) mbar_wait(&empty[slot], ((g / stages) - 1) & 1);
                const uint32_t n = (uint32_t)min((size_t)stage_bytes, b1 - o);
                mbar_expect(&full[slot], n);
                bulk(sm + (size_t)slot * stage_bytes, a + o, n, &full[slot]);
            }
        }
    } else {
        uint32_t g = 0;
        for (size_t o = b0; o < b1; o += stage_bytes, ++g) {
            const int slot = g % stages;
            mbar_wait(&full[slot], (g / stages) & 1);
            const uint32_t n = (uint32_t)min((size_t)stage_bytes, b1 - o);
            const uint4* st = reinterpret_cast<const uint4*>(sm + (size_t)slot * stage_bytes);
            for (uint32_t i = (warp - 1) * 32 + lane; i < n / 16; i += nc * 32) { uint4 v = st[i]; acc += __uint_as_float(v.x); }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
    }
    if (acc == 1.2345f) out[0] = acc;
}

int main() {
    const size_t bytes = 256ull << 20;
    char* a; float* out; char* fl;
    CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&out, 4)); CK(cudaMalloc(&fl, 512ull << 20));
    CK(cudaMemset(a, 1, bytes));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int flush_mode = 0;
    auto flush = [&]() {
        if (flush_mode == 0) cudaMemset(fl, 0, 512ull << 20);
        else k_ldg<8><<<sms * 2, 512>>>((const uint4*)fl, (512ull << 20) / 16, out);
        cudaDeviceSynchronize();
    };
    auto report = [&](const char* name, float ms) { printf("%-40s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
    // a: ldg
    for (int blocks_per_sm : {1, 2, 4}) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            flush(); cudaEventRecord(e0);
            k_ldg<8><<<sms * blocks_per_sm, 512>>>((const uint4*)a, bytes / 16, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        char nm[64]; snprintf(nm, 64, "ldg U=8 x %d CTA/SM (512 thr)", blocks_per_sm); report(nm, best);
    }
    {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            flush(); cudaEventRecord(e0);
            k_ldg<16><<<sms * 2, 512>>>((const uint4*)a, bytes / 16, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        report("ldg U=16 x 2 CTA/SM", best);
    }
    // b: tma ring
    for (int sb : {8192, 16384, 32768}) for (int st : {4, 6, 8, 12}) {
        size_t smem = (size_t)st * sb + 2 * st * 8;
        if (smem > 220 * 1024) continue;
        CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            flush(); cudaEventRecord(e0);
            k_tma<<<sms, 512, smem>>>(a, bytes, st, sb, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        char nm[64]; snprintf(nm, 64, "tma ring %2d x %5d B", st, sb); report(nm, best);
    }
    flush_mode = 1;
    printf("--- clean (read) flush ---\n");
    {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            flush(); cudaEventRecord(e0);
            k_ldg<8><<<sms * 2, 512>>>((const uint4*)a, bytes / 16, out);
            cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        report("ldg U=8 x 2 CTA/SM, clean flush", best);
        for (int st : {6, 8}) {
            size_t smem = (size_t)st * 16384 + 2 * st * 8;
            CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            best = 1e9;
            for (int r = 0; r < 5; ++r) {
                flush(); cudaEventRecord(e0);
                k_tma<<<sms, 512, smem>>>(a, bytes, st, 16384, out);
                cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
            }
            char nm[64]; snprintf(nm, 64, "tma ring %d x 16K, clean flush", st); report(nm, best);
        }
    }
    // memset-flush vs read-flush effect on a plain copy
    {
        char* b; CK(cudaMalloc(&b, bytes));
        float best = 1e9;
        for (int r = 0; r < 5; ++r) { flush(); cudaEventRecord(e0); cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
        printf("%-40s %8.1f us  %7.0f GB/s (read+write)\n", "cudaMemcpy D2D 256MB after dirty flush", best * 1e3, 2 * bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}
