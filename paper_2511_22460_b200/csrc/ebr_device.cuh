// ebr_device.cuh -- device helpers shared by the ebr kernels (sm_100a only).
//
// Citations "P:n" are /root/reference/PAPER.md lines; readings R1..R21 are in DESIGN.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "ebr_internal.h"

namespace ebr {

constexpr unsigned FULL = 0xFFFFFFFFu;

// ------------------------------------------------------------------------------------------
// A5: score -> order-preserving uint32, and the unique 64-bit ranking key
//     kappa = (ord(s) << 32) | (0xFFFFFFFF - global_id)
// so that "kappa descending" == "score descending, ties by ascending ad id" (reading R13).
// -0 is canonicalised to +0 first (reading R14).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ord_of(float s) {
    uint32_t u = __float_as_uint(s);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float float_of_ord(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}
__device__ __forceinline__ uint64_t kappa_of(float s, uint32_t gid) {
    return ((uint64_t)ord_of(s) << 32) | (uint64_t)(0xFFFFFFFFu - gid);
}
__device__ __forceinline__ uint32_t gid_of(uint64_t kappa) {
    return 0xFFFFFFFFu - (uint32_t)(kappa & 0xFFFFFFFFull);
}
__device__ __forceinline__ float score_of(uint64_t kappa) {
    return float_of_ord((uint32_t)(kappa >> 32));
}

// ------------------------------------------------------------------------------------------
// A2: warp-cooperative decode of one 32-posting chunk.
// Lane i >= 1 extracts its b-bit field (gap_i - 1); an inclusive warp scan of
// {first, gap_1, ..., gap_{n-1}} yields the n ascending shard-local ad ids.
// Replaces the paper's 24-bit header + 8-bit residual blocks (Alg. 2 l.355-357).
// All 32 lanes must call it; returns true on lanes holding a posting.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ bool decode_chunk(const uint2* __restrict__ hdr,
                                             const uint32_t* __restrict__ payload,
                                             uint32_t key_word_base, uint32_t c, int lane,
                                             uint32_t& id) {
    const uint2 h = __ldg(&hdr[c]);
    const uint32_t n = (h.y & 31u) + 1u;
    const uint32_t b = (h.y >> 5) & 31u;
    uint32_t g;
    if (lane == 0) {
        g = h.x;
    } else if ((uint32_t)lane < n) {
        uint32_t v = 0;
        if (b) {
            const uint32_t bit = (uint32_t)(lane - 1) * b;
            const uint32_t w = key_word_base + (h.y >> 10) + (bit >> 5);
            const uint64_t two = (uint64_t)__ldg(&payload[w]) | ((uint64_t)__ldg(&payload[w + 1]) << 32);
            v = (uint32_t)(two >> (bit & 31u)) & ((1u << b) - 1u);
        }
        g = v + 1u;
    } else {
        g = 0u;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, g, o);
        if (lane >= o) g += t;
    }
    id = g;
    return (uint32_t)lane < n;
}

// Number of chunks in [lo, hi) whose first id is <= x  (first ids ascending within a key);
// i.e. the index of the first chunk with first > x.  Warp-cooperative 32-ary search.
__device__ __forceinline__ uint32_t warp_upper_bound_first(const uint2* __restrict__ hdr,
                                                           uint32_t lo, uint32_t hi, uint32_t x,
                                                           int lane) {
    while (hi - lo > 32u) {
        const uint32_t step = (hi - lo + 31u) >> 5;
        const uint32_t p = lo + (uint32_t)lane * step;
        const bool pred = (p < hi) && (__ldg(&hdr[p]).x <= x);
        const uint32_t t = __popc(__ballot_sync(FULL, pred));
        if (t == 0u) return lo;
        const uint32_t nlo = lo + (t - 1u) * step + 1u;
        const uint32_t nhi = min(hi, lo + t * step);
        lo = nlo;
        hi = nhi;
    }
    const uint32_t p = lo + (uint32_t)lane;
    const bool pred = (p < hi) && (__ldg(&hdr[p]).x <= x);
    return lo + __popc(__ballot_sync(FULL, pred));
}

// fp32 add into shared memory.  (red.shared.add.f32 is a CAS loop on sm_100a; callers use it
// only where hits are few.)
__device__ __forceinline__ void smem_add(float* p, float v) { atomicAdd(p, v); }

// ------------------------------------------------------------------------------------------
// A6: exact top-K of a set of unique 64-bit keys, by one CTA.
//   1. radix select (8 passes of 8-bit digits) finds the K-th largest key exactly;
//   2. the keys >= it (exactly K, keys are unique) are gathered into shared memory;
//   3. bitonic sort descending.
// `get(i)` returns key i (global or shared memory).  sbuf holds >= pow2ceil(min(n,K)) keys.
// Returns the number of selected keys (min(n, K)) sorted descending in sbuf[0..).
// ------------------------------------------------------------------------------------------
template <typename Get>
__device__ int cta_select_topk(Get get, int64_t n, int K, uint64_t* sbuf, uint32_t* shist,
                               uint32_t* sscalar /* >= 4 words */) {
    const int tid = threadIdx.x, nt = blockDim.x;
    int nsel;
    if (n <= (int64_t)K) {
        nsel = (int)n;
        for (int i = tid; i < nsel; i += nt) sbuf[i] = get(i);
    } else {
        uint64_t prefix = 0;
        uint32_t need = (uint32_t)K;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += nt) shist[i] = 0;
            __syncthreads();
            const uint64_t hmask = (shift == 56) ? 0ull : (~0ull << (shift + 8));
            for (int64_t i = tid; i < n; i += nt) {
                const uint64_t x = get(i);
                if (((x ^ prefix) & hmask) == 0ull) atomicAdd(&shist[(x >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (tid < 32) {
                // warp 0: find digit t with count(>t) < need <= count(>=t), scanning 255..0
                uint32_t cnt[8];
                uint32_t local = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) { cnt[j] = shist[255 - (tid * 8 + j)]; local += cnt[j]; }
                uint32_t incl = local;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(FULL, incl, o);
                    if (tid >= o) incl += t;
                }
                uint32_t c = incl - local;  // count of digits above this lane's group
                int found = -1;
                uint32_t above = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (found < 0 && c < need && c + cnt[j] >= need) { found = 255 - (tid * 8 + j); above = c; }
                    c += cnt[j];
                }
                const unsigned m = __ballot_sync(FULL, found >= 0);
                const int src = __ffs(m) - 1;
                const int t = __shfl_sync(FULL, found, src);
                const uint32_t ab = __shfl_sync(FULL, above, src);
                if (tid == 0) { sscalar[0] = (uint32_t)t; sscalar[1] = ab; }
            }
            __syncthreads();
            prefix |= (uint64_t)sscalar[0] << shift;
            need -= sscalar[1];
            __syncthreads();
        }
        // prefix == the K-th largest key; gather keys >= prefix (exactly K of them)
        if (tid == 0) sscalar[2] = 0;
        __syncthreads();
        for (int64_t i = tid; i < n; i += nt) {
            const uint64_t x = get(i);
            if (x >= prefix) sbuf[atomicAdd(&sscalar[2], 1u)] = x;
        }
        __syncthreads();
        nsel = K;
    }
    int P = 1;
    while (P < nsel) P <<= 1;
    for (int i = nsel + tid; i < P; i += nt) sbuf[i] = 0ull;
    __syncthreads();
    // bitonic sort, descending
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = tid; i < (P >> 1); i += nt) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool desc = ((lo & size) == 0);
                const uint64_t a = sbuf[lo], b = sbuf[hi];
                if ((a < b) == desc) { sbuf[lo] = b; sbuf[hi] = a; }
            }
            __syncthreads();
        }
    }
    return nsel;
}

// Writes one user's sorted selection: ids/scores (or raw keys), padding (id -1, -inf) / 0.
__device__ __forceinline__ void cta_write_topk(const uint64_t* sbuf, int nsel, int K,
                                               int32_t* out_ids, float* out_scores,
                                               uint64_t* out_keys) {
    for (int q = threadIdx.x; q < K; q += blockDim.x) {
        const uint64_t x = (q < nsel) ? sbuf[q] : 0ull;   // 0 = padding (never a real kappa)
        if (out_keys) out_keys[q] = x;
        if (out_ids) out_ids[q] = x ? (int32_t)gid_of(x) : -1;
        if (out_scores) out_scores[q] = x ? score_of(x) : __int_as_float(0xFF800000);
    }
}

__host__ __device__ constexpr int pow2ceil_i(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

}  // namespace ebr
