// Unit-rate microbenchmarks for the batched path's design (R_scatter is to be
// measured, not assumed).  Every kernel runs one CTA per SM (148 CTAs) with `nw` warps and reports
// per-SM rates per SM clock (clock64 / globaltimer measured inside the kernel).
//
//   atoms_*   shared-memory integer / fp32 atomics (red.shared.add) with four address patterns:
//             lane-consecutive, random over 64 KB, a 257-word row stride (rows = ads, lanes = ads),
//             and "same row, lanes = users" (consecutive words)
//   rmw       plain LDS + IADD + STS (owner-computes, no atomic) on random addresses
//   ldtm      tcgen05.ld.32x32b.x{32,64} throughput with 4/8/16 warps
//   sttm      tcgen05.st.32x32b.x32 throughput
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mb_units tools/mb_units.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

struct Res { unsigned long long clk; unsigned long long ns; };

// ---------------------------------------------------------------------------------------------
// shared atomics.  The address stream is precomputed into registers (16 per lane) so the loop
// body is (almost) only the atomic.
// ---------------------------------------------------------------------------------------------
template <int PATTERN, bool F32>
__global__ void atoms_k(int iters, Res* out, uint32_t* sink) {
    extern __shared__ uint32_t sm[];   // 16384 words = 64 KB
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 16384; i += blockDim.x) sm[i] = 0;
    uint32_t addr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        uint32_t a;
        if (PATTERN == 0) a = (uint32_t)((warp * 16 + j) * 32 + lane) & 16383u;          // consecutive
        else if (PATTERN == 1) a = hash32(tid * 977 + j * 131 + blockIdx.x) & 16383u;    // random
        else if (PATTERN == 2) a = ((hash32(warp * 16 + j) & 63u) + lane) * 257u & 16383u; // rows x 257 (lanes = ads)
        else a = ((hash32(warp * 16 + j) & 63u) * 256u + (hash32(lane * 7 + j) & 255u)) & 16383u; // random users in a row
        addr[j] = a;
    }
    const uint32_t vi = (uint32_t)lane * 3u + 1u + (uint32_t)iters;
    const float vf = (float)vi;
    __syncthreads();
    unsigned long long c0 = clock64(), t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (F32) atomicAdd(reinterpret_cast<float*>(&sm[addr[j]]), vf);
            else atomicAdd(&sm[addr[j]], vi);
        }
    }
    __syncthreads();
    unsigned long long c1 = clock64(), t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (tid == 0) { out[blockIdx.x].clk = c1 - c0; out[blockIdx.x].ns = t1 - t0; }
    if (sm[tid] == 0xdeadbeef) sink[0] = 1;
}

// owner-computes read-modify-write without atomics (random addresses; results racy, rate only)
__global__ void rmw_k(int iters, Res* out, uint32_t* sink) {
    extern __shared__ uint32_t sm[];
    const int tid = threadIdx.x;
    for (int i = tid; i < 16384; i += blockDim.x) sm[i] = 0;
    uint32_t addr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) addr[j] = hash32(tid * 977 + j * 131 + blockIdx.x) & 16383u;
    __syncthreads();
    unsigned long long c0 = clock64(), t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            volatile uint32_t* p = &sm[addr[j]];
            *p = *p + (uint32_t)tid;
        }
    }
    __syncthreads();
    unsigned long long c1 = clock64(), t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (tid == 0) { out[blockIdx.x].clk = c1 - c0; out[blockIdx.x].ns = t1 - t0; }
    if (sm[tid] == 0xdeadbeef) sink[0] = 1;
}

// ---------------------------------------------------------------------------------------------
// TMEM
// ---------------------------------------------------------------------------------------------
template <int X>
__device__ __forceinline__ uint32_t ldtm(uint32_t taddr);
template <>
__device__ __forceinline__ uint32_t ldtm<32>(uint32_t taddr) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= r[i];
    return x;
}
template <>
__device__ __forceinline__ uint32_t ldtm<16>(uint32_t taddr) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= r[i];
    return x;
}

// two loads in flight before one wait
__device__ __forceinline__ uint32_t ldtm2x32(uint32_t taddr) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]),
          "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),
          "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),
          "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
          "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 64; ++i) x ^= r[i];
    return x;
}

template <int MODE>   // 0: x16, 1: x32, 2: x64, 3: st x32
__global__ void tmem_k(int iters, Res* out, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = slot;
    const int q = warp & 3, grp = warp >> 2, ngrp = blockDim.x / 128;
    uint32_t x = 0;
    unsigned long long c0 = clock64(), t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const int width = MODE == 0 ? 16 : MODE == 2 ? 64 : 32;
    const int per = 512 / width;                 // column blocks per pass
    for (int it = 0; it < iters; ++it) {
        for (int b = grp; b < per; b += ngrp) {
            const uint32_t a = base + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * width);
            if (MODE == 0) x ^= ldtm<16>(a);
            else if (MODE == 1) x ^= ldtm<32>(a);
            else if (MODE == 2) x ^= ldtm2x32(a);
            else {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                    "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
                    "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(a), "r"(it + lane)
                    : "memory");
            }
        }
        if (MODE == 3) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    unsigned long long c1 = clock64(), t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (tid == 0) { out[blockIdx.x].clk = c1 - c0; out[blockIdx.x].ns = t1 - t0; }
    if (x == 0xdeadbeef) sink[0] = x;
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512));
}

static Res run_and_max(Res* d, int n) {
    Res h[148];
    cudaMemcpy(h, d, sizeof(Res) * n, cudaMemcpyDeviceToHost);
    Res m{0, 0};
    for (int i = 0; i < n; ++i) { if (h[i].clk > m.clk) m.clk = h[i].clk; if (h[i].ns > m.ns) m.ns = h[i].ns; }
    return m;
}

int main() {
    Res* d; cudaMalloc(&d, sizeof(Res) * 148);
    uint32_t* sink; cudaMalloc(&sink, 64);
    const int smem = 64 * 1024;
    const char* pat[] = {"consecutive", "random64KB", "rows257_lanes=ads", "row_lanes=random_users"};
    auto atoms = [&](auto kern, const char* nm, int p, int nw) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = 256;
        kern<<<148, nw * 32, smem>>>(8, d, sink);
        kern<<<148, nw * 32, smem>>>(iters, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        Res r = run_and_max(d, 148);
        const double ops = (double)iters * 16 * nw * 32;      // lane-ops per SM
        printf("{\"bench\":\"%s\",\"pattern\":\"%s\",\"warps\":%d,\"lane_ops_per_clk_sm\":%.3f,\"ghz\":%.3f,\"err\":\"%s\"}\n",
               nm, p >= 0 ? pat[p] : "random64KB", nw, ops / r.clk, (double)r.clk / r.ns, cudaGetErrorString(e));
    };
    for (int nw : {8, 16, 32}) {
        atoms(atoms_k<0, false>, "atoms.u32", 0, nw);
        atoms(atoms_k<1, false>, "atoms.u32", 1, nw);
        atoms(atoms_k<2, false>, "atoms.u32", 2, nw);
        atoms(atoms_k<3, false>, "atoms.u32", 3, nw);
        atoms(atoms_k<1, true>, "atoms.f32", 1, nw);
        atoms(atoms_k<0, true>, "atoms.f32", 0, nw);
        atoms(rmw_k, "lds+sts rmw", -1, nw);
    }
    auto tm = [&](auto kern, const char* nm, int nw) {
        const int iters = 200;
        kern<<<148, nw * 32>>>(4, d, sink);
        kern<<<148, nw * 32>>>(iters, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        Res r = run_and_max(d, 148);
        const double bytes = (double)iters * 128 * 512 * 4;   // whole TMEM per pass
        printf("{\"bench\":\"%s\",\"warps\":%d,\"bytes_per_clk_sm\":%.2f,\"ghz\":%.3f,\"err\":\"%s\"}\n", nm, nw,
               bytes / r.clk, (double)r.clk / r.ns, cudaGetErrorString(e));
    };
    for (int nw : {4, 8, 16}) {
        tm(tmem_k<0>, "tcgen05.ld.32x32b.x16", nw);
        tm(tmem_k<1>, "tcgen05.ld.32x32b.x32", nw);
        tm(tmem_k<2>, "tcgen05.ld.32x32b.x64", nw);
        tm(tmem_k<3>, "tcgen05.st.32x32b.x32", nw);
    }
    return 0;
}
