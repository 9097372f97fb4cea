// Microbenchmark of the one-CTA top-K selection (cta_select_topk) on n random unique keys.
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <functional>
#include "../paper_2511_22460_b200/csrc/ebr_device.cuh"
using namespace ebr;
__global__ void __launch_bounds__(512, 1) k_sel(const uint64_t* keys, int64_t n, int K, uint64_t* out, unsigned long long* tm, int smem_bytes) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t sScalar[8];
    const int P = pow2ceil_i(K);
    uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);
    uint32_t* shist = reinterpret_cast<uint32_t*>(sbuf + P);
    uint64_t* scand = reinterpret_cast<uint64_t*>(shist + kSelBins);
    const int64_t scap = (smem_bytes - (int64_t)((char*)scand - (char*)smem)) / 8;
    if (threadIdx.x == 0) { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); tm[3] = t; }
    const int nsel = cta_select_topk([keys](int64_t i) { return __ldcg(&keys[i]); }, n, K, sbuf, scand, scap, shist, sScalar, tm);
    for (int q = threadIdx.x; q < K; q += blockDim.x) out[q] = q < nsel ? sbuf[q] : 0;
    if (threadIdx.x == 0) { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); tm[4] = t; }
}
int main() {
    for (int64_t n : {701, 2000, 5000, 20000}) for (int K : {100, 500, 1000}) {
        std::vector<uint64_t> h(n); std::mt19937_64 rng(n * 7 + K);
        for (auto& x : h) x = (0xC0800000ull << 32) | (rng() & 0x00FFFFFFFFFFFFull);   // shared top bits, like a histogram bin
        uint64_t *d, *o; unsigned long long* tm;
        cudaMalloc(&d, n * 8); cudaMalloc(&o, K * 8); cudaMalloc(&tm, 64);
        cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
        int smem = 200 * 1024; cudaFuncSetAttribute(k_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        double best[5] = {1e9, 1e9, 1e9, 1e9, 1e9};
        for (int r = 0; r < 10; ++r) {
            cudaMemset(tm, 0, 64);
            k_sel<<<1, 512, smem>>>(d, n, K, o, tm, smem);
            unsigned long long t[5]; cudaMemcpy(t, tm, 40, cudaMemcpyDeviceToHost);
            double s = (t[4] - t[3]) / 1e3, st = t[0] ? (t[0] - t[3]) / 1e3 : 0, rd = (t[1] - t[3]) / 1e3, so = (t[2] - t[1]) / 1e3;
            if (s < best[0]) { best[0] = s; best[1] = st; best[2] = rd; best[3] = so; }
        }
        std::vector<uint64_t> out(K); cudaMemcpy(out.data(), o, K * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end(), std::greater<uint64_t>());
        bool ok = true; for (int q = 0; q < K && q < n; ++q) ok &= out[q] == h[q];
        printf("n=%6lld K=%5d total %7.2f us | staged %6.2f  radix-done %6.2f  sort %6.2f  %s\n", (long long)n, K, best[0], best[1], best[2], best[3], ok ? "ok" : "WRONG");
        cudaFree(d); cudaFree(o); cudaFree(tm);
    }
}
