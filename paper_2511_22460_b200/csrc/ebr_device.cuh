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

// Decodes chunks [cb, ce) (ce - cb <= 16) of one key in two memory round trips: lanes fetch the
// (up to) 16 chunk headers at once, then every lane issues its payload loads for all 16 chunks,
// then each chunk is unpacked + warp-scanned.  f(id) is called on every lane holding a posting.
template <typename F>
__device__ __forceinline__ void decode_unit16(const uint2* __restrict__ hdr,
                                              const uint32_t* __restrict__ payload, uint32_t kwb,
                                              uint32_t cb, uint32_t ce, int lane, F f) {
    const uint32_t nc = ce - cb;
    uint2 h = make_uint2(0u, 0u);
    if ((uint32_t)lane < nc) h = __ldg(&hdr[cb + lane]);
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        lo[q] = 0u;
        hi[q] = 0u;
        if ((uint32_t)q >= nc) break;                // warp-uniform: short units stop early
        const uint32_t meta = __shfl_sync(FULL, h.y, q);
        const uint32_t n = (meta & 31u) + 1u, b = (meta >> 5) & 31u;
        if ((uint32_t)q < nc && lane >= 1 && (uint32_t)lane < n && b) {
            const uint32_t bit = (uint32_t)(lane - 1) * b;
            const uint32_t w = kwb + (meta >> 10) + (bit >> 5);
            lo[q] = __ldg(&payload[w]);
            hi[q] = __ldg(&payload[w + 1]);
        }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        if ((uint32_t)q >= nc) break;
        const uint32_t meta = __shfl_sync(FULL, h.y, q);
        const uint32_t first = __shfl_sync(FULL, h.x, q);
        const uint32_t n = (meta & 31u) + 1u, b = (meta >> 5) & 31u;
        uint32_t g;
        if (lane == 0) {
            g = first;
        } else if ((uint32_t)lane < n) {
            uint32_t v = 0u;
            if (b) {
                const uint32_t bit = (uint32_t)(lane - 1) * b;
                v = (uint32_t)(((((uint64_t)hi[q]) << 32) | lo[q]) >> (bit & 31u)) & ((1u << b) - 1u);
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
        if ((uint32_t)lane < n) f(g);
    }
}

// decode_unit16 for warp-collective consumers: f(id, ok) is called on EVERY lane for each chunk
// (ok = the lane holds a posting), so f may use __match_any_sync / __shfl_sync over the full warp.
template <typename F>
__device__ __forceinline__ void decode_unit16_warp(const uint2* __restrict__ hdr,
                                                   const uint32_t* __restrict__ payload, uint32_t kwb,
                                                   uint32_t cb, uint32_t ce, int lane, F f) {
    const uint32_t nc = ce - cb;
    uint2 h = make_uint2(0u, 0u);
    if ((uint32_t)lane < nc) h = __ldg(&hdr[cb + lane]);
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        lo[q] = 0u;
        hi[q] = 0u;
        if ((uint32_t)q >= nc) break;                // warp-uniform
        const uint32_t meta = __shfl_sync(FULL, h.y, q);
        const uint32_t n = (meta & 31u) + 1u, b = (meta >> 5) & 31u;
        if (lane >= 1 && (uint32_t)lane < n && b) {
            const uint32_t bit = (uint32_t)(lane - 1) * b;
            const uint32_t w = kwb + (meta >> 10) + (bit >> 5);
            lo[q] = __ldg(&payload[w]);
            hi[q] = __ldg(&payload[w + 1]);
        }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        if ((uint32_t)q >= nc) break;
        const uint32_t meta = __shfl_sync(FULL, h.y, q);
        const uint32_t first = __shfl_sync(FULL, h.x, q);
        const uint32_t n = (meta & 31u) + 1u, b = (meta >> 5) & 31u;
        uint32_t g;
        if (lane == 0) {
            g = first;
        } else if ((uint32_t)lane < n) {
            uint32_t v = 0u;
            if (b) {
                const uint32_t bit = (uint32_t)(lane - 1) * b;
                v = (uint32_t)(((((uint64_t)hi[q]) << 32) | lo[q]) >> (bit & 31u)) & ((1u << b) - 1u);
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
        f(g, (uint32_t)lane < n);
    }
}

// Block-wide exclusive scan of one value per thread (blockDim.x <= 1024); returns the prefix and
// writes the total to *total.  `scratch` holds >= 33 words.  Contains __syncthreads().
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = (blockDim.x + 31) >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) scratch[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = (lane < nw) ? scratch[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, wi, o);
            if (lane >= o) wi += t;
        }
        scratch[lane] = wi - w;
        if (lane == 31) scratch[32] = wi;
    }
    __syncthreads();
    const uint32_t r = scratch[warp] + incl - v;
    *total = scratch[32];
    __syncthreads();
    return r;
}

// fp32 add into shared memory.  (red.shared.add.f32 is a CAS loop on sm_100a; callers use it
// only where hits are few.)
__device__ __forceinline__ void smem_add(float* p, float v) { atomicAdd(p, v); }

// ------------------------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine) helpers, sm_90+ PTX
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// the same wait with a suspend-time hint: the thread sleeps in the barrier (woken when the phase
// completes) instead of re-issuing try_wait, leaving issue slots to the warps that do the work
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
}
// the same wait by pure polling (mbarrier.test_wait never suspends the thread)
__device__ __forceinline__ void mbar_wait_poll(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// histogram increment aggregated over the lanes of a warp that hit the same bin
__device__ __forceinline__ void warp_hist_add(uint32_t* hist, uint32_t bin, bool active) {
    const unsigned act = __ballot_sync(FULL, active);
    if (!active) return;
    const unsigned peers = __match_any_sync(act, bin);
    if ((threadIdx.x & 31) == (__ffs(peers) - 1)) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}


// ------------------------------------------------------------------------------------------
// A6: exact top-K of a set of unique 64-bit keys, by one CTA.
//   1. the bits common to every key are skipped (AND/OR reduction);
//   2. radix select with 11-bit digits, MSB first, finds the K-th largest key; it stops early as
//      soon as the digit bucket holding the K-th is needed in full;
//   3. the keys >= the threshold (exactly K: keys are unique) are gathered into shared memory;
//   4. bitonic sort, descending (warp shuffles for strides < 32, registers for strides >= the
//      CTA size, shared memory in between).
// `get(i)` returns key i.  If n <= scand_cap the keys are first staged in scand (shared).
// sbuf holds >= pow2ceil(min(n,K)) keys; shist kSelBins words; sscalar 8 words.
// ------------------------------------------------------------------------------------------
constexpr int kSelBits = 11;
constexpr int kSelBins = 1 << kSelBits;

__device__ __forceinline__ uint64_t warp_and64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v &= __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(FULL, v, o);
    return v;
}

template <typename Get>
__device__ int cta_radix_select(Get get, int64_t n, int K, uint64_t* sbuf, uint32_t* shist,
                                uint32_t* sscalar) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    uint64_t* sred = reinterpret_cast<uint64_t*>(shist);   // 2 x 32 words of scratch
    // 1. common prefix of all keys
    uint64_t va = ~0ull, vo = 0ull;
    for (int64_t i = tid; i < n; i += nt) { const uint64_t x = get(i); va &= x; vo |= x; }
    va = warp_and64(va);
    vo = warp_or64(vo);
    if (lane == 0) { sred[warp] = va; sred[32 + warp] = vo; }
    __syncthreads();
    if (warp == 0) {
        const int nw = (nt + 31) >> 5;
        uint64_t a = lane < nw ? sred[lane] : ~0ull, o = lane < nw ? sred[32 + lane] : 0ull;
        a = warp_and64(a);
        o = warp_or64(o);
        if (lane == 0) { sred[0] = a; sred[1] = o; }
    }
    __syncthreads();
    const uint64_t kand = sred[0], kor = sred[1];
    __syncthreads();
    const uint64_t diff = kand ^ kor;                 // n > K >= 1 unique keys => diff != 0
    int hi = 63 - __clzll((long long)diff);
    uint64_t prefix = kand & ~((hi >= 63) ? ~0ull : ((2ull << hi) - 1ull));
    uint32_t need = (uint32_t)K;
    while (hi >= 0) {
        const int width = hi + 1 < kSelBits ? hi + 1 : kSelBits;
        const int shift = hi + 1 - width;
        const uint32_t nb = 1u << width;
        for (int i = tid; i < (int)nb; i += nt) shist[i] = 0;
        __syncthreads();
        const uint64_t hmask = (hi >= 63) ? 0ull : ~((2ull << hi) - 1ull);
        for (int64_t i = tid; i < n; i += nt) {
            const uint64_t x = get(i);
            if (((x ^ prefix) & hmask) == 0ull) atomicAdd(&shist[(uint32_t)(x >> shift) & (nb - 1u)], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            // digit t (scanning nb-1 .. 0): count(> t) < need <= count(>= t)
            const int per = (int)(nb + 31) >> 5;
            uint32_t local = 0;
            for (int j = 0; j < per; ++j) {
                const int d = (int)nb - 1 - (lane * per + j);
                if (d >= 0) local += shist[d];
            }
            uint32_t incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += t;
            }
            uint32_t c = incl - local;
            int found = -1;
            uint32_t above = 0, cnt_t = 0;
            if (c < need && c + local >= need) {
                for (int j = 0; j < per; ++j) {
                    const int d = (int)nb - 1 - (lane * per + j);
                    if (d < 0) break;
                    const uint32_t h = shist[d];
                    if (found < 0 && c < need && c + h >= need) { found = d; above = c; cnt_t = h; }
                    c += h;
                }
            }
            const unsigned m = __ballot_sync(FULL, found >= 0);
            const int src = __ffs(m) - 1;
            const int t = __shfl_sync(FULL, found, src);
            const uint32_t ab = __shfl_sync(FULL, above, src);
            const uint32_t ct = __shfl_sync(FULL, cnt_t, src);
            if (lane == 0) { sscalar[0] = (uint32_t)t; sscalar[1] = ab; sscalar[3] = ct; }
        }
        __syncthreads();
        prefix |= (uint64_t)sscalar[0] << shift;
        need -= sscalar[1];
        const bool done = (sscalar[3] == need);     // the whole bucket is needed: stop here
        __syncthreads();
        if (done) break;
        hi = shift - 1;
    }
    // gather the keys >= prefix (exactly K of them)
    if (tid == 0) sscalar[2] = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += nt) {
        const int64_t i = base + tid;
        uint64_t x = 0;
        bool take = false;
        if (i < n) { x = get(i); take = x >= prefix; }
        const unsigned m = __ballot_sync(FULL, take);
        uint32_t pos = 0;
        if (lane == 0 && m) pos = atomicAdd(&sscalar[2], (uint32_t)__popc(m));
        pos = __shfl_sync(FULL, pos, 0);
        if (take) sbuf[pos + __popc(m & ((1u << lane) - 1u))] = x;
    }
    __syncthreads();
    return K;
}

// Bitonic sort (descending) of sbuf[0..P), P = pow2ceil(nsel), entries >= nsel padded with 0.
// Element i lives in thread (i % nt), register (i / nt): strides < 32 use warp shuffles,
// strides >= nt stay in registers, the others go through shared memory.
template <int E>
__device__ __forceinline__ void cta_bitonic_fast(uint64_t* sbuf, int P) {
    const int tid = threadIdx.x, nt = blockDim.x;
    uint64_t v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) { const int i = tid + e * nt; v[e] = i < P ? sbuf[i] : 0ull; }
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= nt) {
                const int em = stride / nt;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int e2 = e ^ em;
                    if (e2 > e && e2 < E) {
                        const int i = tid + e * nt;
                        const bool desc = (i & size) == 0;
                        const uint64_t a = v[e], b = v[e2];
                        if ((a < b) == desc) { v[e] = b; v[e2] = a; }
                    }
                }
            } else if (stride >= 32) {
#pragma unroll
                for (int e = 0; e < E; ++e) { const int i = tid + e * nt; if (i < P) sbuf[i] = v[e]; }
                __syncthreads();
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = tid + e * nt;
                    if (i < P) {
                        const uint64_t o = sbuf[i ^ stride];
                        const bool lower = (i & stride) == 0, desc = (i & size) == 0;
                        const uint64_t mx = v[e] > o ? v[e] : o, mn = v[e] > o ? o : v[e];
                        v[e] = (lower == desc) ? mx : mn;
                    }
                }
                __syncthreads();
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = tid + e * nt;
                    const uint64_t o = __shfl_xor_sync(FULL, v[e], stride);
                    const bool lower = (i & stride) == 0, desc = (i & size) == 0;
                    const uint64_t mx = v[e] > o ? v[e] : o, mn = v[e] > o ? o : v[e];
                    v[e] = (lower == desc) ? mx : mn;
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) { const int i = tid + e * nt; if (i < P) sbuf[i] = v[e]; }
    __syncthreads();
}

__device__ __forceinline__ void cta_bitonic_desc(uint64_t* sbuf, int nsel) {
    const int tid = threadIdx.x, nt = blockDim.x;
    int P = 1;
    while (P < nsel) P <<= 1;
    for (int i = nsel + tid; i < P; i += nt) sbuf[i] = 0ull;
    __syncthreads();
    if (P <= nt) { cta_bitonic_fast<1>(sbuf, P); return; }
    if (P <= 2 * nt) { cta_bitonic_fast<2>(sbuf, P); return; }
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
}

__device__ __forceinline__ void stamp_max(unsigned long long* tm, int i) {
    if (tm && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        atomicMax(&tm[i], t);
    }
}

// Selects the min(n, K) largest keys, sorted descending into sbuf.  Returns that count.
template <typename Get>
__device__ int cta_select_topk(Get get, int64_t n, int K, uint64_t* sbuf, uint64_t* scand,
                               int64_t scand_cap, uint32_t* shist, uint32_t* sscalar,
                               unsigned long long* tm = nullptr) {
    const int tid = threadIdx.x, nt = blockDim.x;
    int nsel;
    if (n <= (int64_t)K) {
        nsel = (int)n;
        for (int i = tid; i < nsel; i += nt) sbuf[i] = get(i);
        __syncthreads();
    } else if (scand && n <= scand_cap) {
        for (int64_t i = tid; i < n; i += nt) scand[i] = get(i);
        __syncthreads();
        stamp_max(tm, 0);
        nsel = cta_radix_select([scand](int64_t i) { return scand[i]; }, n, K, sbuf, shist, sscalar);
    } else {
        nsel = cta_radix_select(get, n, K, sbuf, shist, sscalar);
    }
    stamp_max(tm, 1);
    cta_bitonic_desc(sbuf, nsel);
    stamp_max(tm, 2);
    return nsel;
}

// Writes one user's sorted selection: ids/scores (or raw keys), padding (id -1, -inf) / 0.
__device__ __forceinline__ void cta_write_topk(const uint64_t* sbuf, int nsel, int K,
                                               int32_t* out_ids, float* out_scores,
                                               uint64_t* out_keys) {
    for (int q = threadIdx.x; q < K; q += blockDim.x) {
        // keys below 2^32 are padding (0, or a merge sentinel): never a real kappa, whose
        // ord(s) >= 1 for every finite score
        uint64_t x = (q < nsel) ? sbuf[q] : 0ull;
        if (x < (1ull << 32)) x = 0ull;
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
