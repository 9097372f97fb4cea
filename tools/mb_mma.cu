// tcgen05.mma throughput microbenchmark (kind::f16, cta_group::1, M = 128): A from shared memory
// (SS) or from TMEM (TS), B from shared memory, N = 64 / 128 / 256, one CTA per SM, one issuing
// thread, accumulating into one TMEM accumulator.  Reports dense flop/clk/SM and the implied
// TFLOP/s over 148 SMs at the measured clock -- the rate the batched path's fused kernel can
// reach per tile.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_22460_b200/csrc \
//          -o tools/bin/mb_mma tools/mb_mma.cu -lcuda
#include <cstdio>
#include <cstdint>

#include "ebr_tc.cuh"

using namespace ebr;

struct Res { unsigned long long clk, ns; };

template <bool TS>
__global__ void __launch_bounds__(128, 1) mma_k(int iters, int n, Res* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    // A tile 128 x 64 bf16 (16 KB) and B tile 256 x 64 bf16 (32 KB), small values
    for (int i = tid; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3C003C00u;
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (tid < 32) tc::tmem_alloc(&tslot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = tslot;
    if (TS) {   // A operand in TMEM columns [256, 288): 128 lanes x 64 K (two bf16 per column)
        const int w = tid >> 5;
        uint32_t v[32];
        for (int j = 0; j < 32; ++j) v[j] = 0x3C003C00u;
        tc::tmem_st32(tbase + ((uint32_t)(w * 32) << 16) + 256u, v);
        tc::fence_before();
    }
    __syncthreads();
    tc::fence_after();
    unsigned long long c0 = 0, t0 = 0;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_bf16_m128(n);
        const uint64_t da = tc::sdesc_sw128(smem), db = tc::sdesc_sw128(smem + 16384);
        c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (TS) tc::umma_f16_ts(tbase, tbase + 256u + (uint32_t)(k * 8), db + (uint64_t)(k * 2), idesc, 1u);
                else tc::umma_f16(tbase, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc, 1u);
            }
        }
        tc::umma_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[blockIdx.x].clk = clock64() - c0;
        out[blockIdx.x].ns = t1 - t0;
    }
    tc::fence_before();
    __syncthreads();
    if (tid < 32) tc::tmem_dealloc(tbase, 512);
}

int main() {
    Res* d;
    cudaMalloc(&d, sizeof(Res) * 148);
    Res h[148];
    const int smem = 16384 + 32768 + 1024;
    cudaFuncSetAttribute(mma_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(mma_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int ts = 0; ts < 2; ++ts) {
        for (int n : {64, 128, 256}) {
            const int iters = 4096;
            auto k = ts ? mma_k<true> : mma_k<false>;
            k<<<148, 128, smem>>>(16, n, d);
            k<<<148, 128, smem>>>(iters, n, d);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            unsigned long long mc = 0, mn = 0;
            for (int i = 0; i < 148; ++i) { if (h[i].clk > mc) mc = h[i].clk; if (h[i].ns > mn) mn = h[i].ns; }
            const double flop = 2.0 * 128 * n * 16 * 4.0 * iters;
            printf("{\"bench\":\"tcgen05.mma kind::f16 M128\",\"A\":\"%s\",\"N\":%d,\"flop_per_clk_sm\":%.1f,"
                   "\"clk_per_mma\":%.1f,\"ghz\":%.3f,\"tflops_148sm\":%.1f,\"err\":\"%s\"}\n",
                   ts ? "tmem" : "smem", n, flop / mc, (double)mc / (4.0 * iters), (double)mc / mn,
                   flop * 148 / mn / 1e3, cudaGetErrorString(e));
        }
    }
    return 0;
}
