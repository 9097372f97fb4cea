// ebr_batch.cu -- the batched path (bf16 embeddings, user batch >= 16): the deep score is a dense
// contraction D[ads x users] = A . U^T (Eq. 1 / Eq. 8 for every (user, ad) pair) and runs on the
// 5th-generation tensor cores, together with the wide term of the hot keys (the longest posting
// lists, kept as dense one-hot columns H of L -- DESIGN.md R22): D = W + A U_deep^T + H U_hot^T,
// where U_hot holds each user's w~ as three exact bf16 terms and W is the cold keys' wide term
// decoded from the compressed inverted lists.  Per group of up to 128 users, one call runs:
//
//   1. plan_kernel     A1: hot slots -> U_hot (hi, mid, lo), cold slots -> work items, the per-user
//                      fixed-point scale, and the deep part of the bf16 user tile U
//   2. span_kernel     for every cold item and kWideR-ad range, the chunks holding ids in the range
//      wide_smem_kernel A2+A3 for cold keys: CTA (range, user) decodes the user's postings in the
//                      range and accumulates w~ in shared memory (Alg. 2 l.358), then writes W
//   3. gemm_kernel<0>  A4+A5 on a strided 1/16 sample of the ad tiles: s = W + deep + hot, stored
//   4. theta_kernel    A6a per user: theta_u = the K-th largest key among the sampled ads.  The
//                      sample is a subset of the inventory, so at least K ads have key >= theta_u
//                      and the top-K is contained in {key >= theta_u} -- exact, not heuristic.
//   5. gemm_kernel<1>  A4+A5+A6b on every tile: keys >= theta_u appended to the user's candidates
//   6. final_kernel    A6c per user: exact radix select + sort of the candidates
//   A user whose candidate list overflowed (possible only for massively tied scores) is recomputed
//   by the latency path after a single stream synchronisation at the end of the call.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ebr_tc.cuh"

namespace ebr {
ebr_status run_small(const QueryArgs& q, int b0, int B);

namespace batch {

constexpr int kGroup = 128;          // users per group (UMMA N)
constexpr int kTileM = 128;          // ads per tile (UMMA M)
constexpr int kBlockK = 64;          // bf16 elements per 128-byte swizzle row
constexpr int kSampleStride = 16;    // every 16th tile is sampled for theta
constexpr int kEpiWarps = 8;         // 2 per TMEM lane quadrant, two 32-column chunks each
constexpr int kEpiChunks = kGroup / 32 / (kEpiWarps / 4);
constexpr int kLoadWarps = 4;        // one per TMEM lane quadrant, every 32-column chunk in turn
constexpr int kEpiWarp0 = 4;
constexpr int kLoadWarp0 = kEpiWarp0 + kEpiWarps;
constexpr int kGemmThreads = 32 * (kLoadWarp0 + kLoadWarps);   // 0 TMA, 1 MMA, 2 TMEM alloc, 3 W bulk copies
constexpr int kAccStages = 4;        // TMEM: 4 x 128 columns = all 512
#ifndef EBR_WPF
#define EBR_WPF 4
#endif
constexpr int kWPrefetch = EBR_WPF;  // tiles of W streamed into L2 ahead of their bulk copies
constexpr int kHotPieces = 3;        // w~ = hi + mid + lo in bf16: 24 significant bits, exact (R22)
constexpr int kBlockBytes = kTileM * 128;   // one ring stage: 128 ads x 64 bf16 (one K block)

struct BItem {
    uint32_t key, c0, c1, u, kwb;
    float w;
};

struct BatchWs {   // workspace carve-up (device pointers)
    uint32_t* header;     // [0] n_items, [1] overflow users, [2] users short of K candidates
    BItem* items;         // [cap_items]
    uint64_t* chunk_off;  // [cap_items + 1]
    __nv_bfloat16* U;     // [kGroup][d_pad]
    float* W;             // [n_tiles][kGroup][128] tile-major: a tile's 32-user chunk is 16 KB contiguous
    float* samp;          // [kGroup][n_samp]
    uint64_t* theta;      // [kGroup]
    uint32_t* cand_count; // [kGroup]
    uint64_t* cand;       // [kGroup][cap]
    uint32_t* overflow;   // [kGroup]
    uint32_t* user_item;  // [kGroup + 1]  items of group user u: [user_item[u], user_item[u+1])
    int32_t* user_shift;  // [kGroup] fixed-point scale S_u of the user's cold wide sum
    uint32_t* span;       // [nj + 1][cap_items] first chunk of item i with first id >= j*R
    uint32_t* span_lo;    // [nj][cap_items]     first chunk of item i holding an id >= j*R
};

#ifndef EBR_WIDE_R
#define EBR_WIDE_R 16384
#endif
#ifndef EBR_WIDE_T
#define EBR_WIDE_T 384
#endif
constexpr int kWideR = EBR_WIDE_R;     // ads per shared-memory accumulation chunk (int32 each)

// ------------------------------------------------------------------------------------------
// 1. plan (one CTA)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) plan_kernel(const uint32_t* __restrict__ key_chunk_off,
                                                   const uint32_t* __restrict__ key_word_off,
                                                   const float* __restrict__ cross_w,
                                                   const int32_t* __restrict__ field_card,
                                                   const int32_t* __restrict__ field_base, int F, int S,
                                                   const int32_t* __restrict__ user_feat,
                                                   const float* __restrict__ user_x,
                                                   const uint16_t* __restrict__ user_emb, int d, int d_pad,
                                                   int nu, int nu_pad, const int32_t* __restrict__ hot_slot,
                                                   int n_hot, int u_cols, BatchWs ws, uint32_t* err) {
    extern __shared__ float sHot[];          // [nu_pad][n_hot] sum of w~ per (user, hot slot)
    __shared__ uint32_t sScan[40];
    __shared__ float sBound[kGroup];         // sum |w~| of each user's cold items
    __shared__ uint64_t sCarry;
    const int tid = threadIdx.x;
    uint16_t* U = reinterpret_cast<uint16_t*>(ws.U);
    // user tile, deep part (zero padded): U[u][0..d_pad)
    for (int i = tid; i < nu_pad * d_pad; i += blockDim.x) {
        const int u = i / d_pad, j = i - u * d_pad;
        const uint16_t v = (u < nu && j < d) ? user_emb[(size_t)u * d + j] : (uint16_t)0;
        U[(size_t)u * u_cols + j] = v;
    }
    for (int i = tid; i < nu_pad * n_hot; i += blockDim.x) sHot[i] = 0.f;
    for (int i = tid; i < kGroup; i += blockDim.x) sBound[i] = 0.f;
    __syncthreads();
    const int nslot = nu * F * S;
    uint32_t base = 0;
    if (tid == 0) sCarry = 0;
    __syncthreads();
    for (int s0 = 0; s0 < nslot; s0 += blockDim.x) {
        const int i = s0 + tid;
        BItem it{};
        bool ok = false;
        if (i < nslot) {
            const int f = (i / S) % F;
            const int32_t v = user_feat[i];
            if (v >= field_card[f]) atomicOr(err, 1u);
            else if (v >= 0) {
                const uint32_t key = (uint32_t)(field_base[f] + v);
                it.c0 = key_chunk_off[key];
                it.c1 = key_chunk_off[key + 1];
                it.key = key;
                it.u = (uint32_t)(i / (F * S));
                it.kwb = key_word_off[key];
                it.w = __fmul_rn(cross_w[key], user_x[i]);   // w~ = fl32(w x), never an FMA (R10)
                const int32_t h = n_hot ? hot_slot[key] : -1;
                if (h >= 0 && h < n_hot) atomicAdd(&sHot[it.u * n_hot + h], it.w);   // dense column (R22)
                else ok = it.c1 > it.c0;
                if (ok) atomicAdd(&sBound[it.u], fabsf(it.w));
            }
        }
        uint32_t tot;
        const uint32_t pos = block_exclusive_scan(ok ? 1u : 0u, sScan, &tot);
        uint32_t ctot;
        const uint32_t cpre = block_exclusive_scan(ok ? it.c1 - it.c0 : 0u, sScan, &ctot);
        if (ok) {
            ws.items[base + pos] = it;
            ws.chunk_off[base + pos] = sCarry + cpre;
        }
        __syncthreads();
        if (tid == 0) sCarry += ctot;
        base += tot;
        __syncthreads();
    }
    if (tid == 0) {
        ws.header[0] = base;
        ws.header[1] = 0;       // overflow users of this group
        ws.header[2] = 0;       // users with fewer than K candidates (theta rank below K)
        ws.chunk_off[base] = sCarry;
    }
    __syncthreads();
    // fixed-point scale of each user's cold wide sum: |sum| <= bound < 2^e, S = 30 - e keeps every
    // partial sum inside int32 (and int32 addition is modular anyway)
    for (int u = tid; u < kGroup; u += blockDim.x) {
        int e = 0;
        frexpf(sBound[u] * 1.0001f + 1e-30f, &e);
        ws.user_shift[u] = 30 - e;
    }
    // user tile, hot part: w~ of hot slot h as kHotPieces bf16 terms (hi, mid, lo; R22) in
    // U[u][d_pad + ((h/64)*kHotPieces + p)*64 + h%64] -- one 64-column K block per (block, piece)
    for (int i = tid; i < nu_pad * n_hot; i += blockDim.x) {
        const int u = i / n_hot, h = i - u * n_hot;
        float r = sHot[i];
        uint16_t* dst = U + (size_t)u * u_cols + d_pad + (size_t)(h >> 6) * kHotPieces * 64 + (h & 63);
#pragma unroll
        for (int p = 0; p < kHotPieces; ++p) {
            const __nv_bfloat16 b = __float2bfloat16_rn(r);
            dst[p * 64] = __bfloat16_as_ushort(b);
            r -= __bfloat162float(b);            // exact (Sterbenz-type cancellation of the top bits)
        }
    }
    // items are in slot order, i.e. grouped by user: first item of each user by binary search
    for (int u = tid; u <= nu; u += blockDim.x) {
        int lo = 0, hi = (int)base;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int)ws.items[mid].u < u) lo = mid + 1; else hi = mid;
        }
        ws.user_item[u] = (uint32_t)lo;
    }
}

// ------------------------------------------------------------------------------------------
// 2a. spans: for every item and every kWideR-ad chunk j, the item's posting chunks that hold an
//     id in [j*R, (j+1)*R): [span_lo[j][i], span[j+1][i]).  One warp per item, lanes binary-search
//     different boundaries over the chunk first ids; chunk_last decides whether the chunk that
//     straddles j*R reaches into the range (so an item with no posting there costs nothing).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) span_kernel(const uint2* __restrict__ hdr,
                                                   const uint32_t* __restrict__ chunk_last,
                                                   BatchWs ws, int nj, int cap_items) {
    const int lane = threadIdx.x & 31;
    const uint32_t n_items = __ldcg(&ws.header[0]);
    const uint32_t i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (i >= n_items) return;
    const BItem t = ws.items[i];
    for (int j = lane; j <= nj; j += 32) {
        const uint32_t x = (uint32_t)((int64_t)j * kWideR);
        uint32_t lo = t.c0, hi = t.c1;           // first chunk with first >= x
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(&hdr[mid]).x < x) lo = mid + 1; else hi = mid;
        }
        ws.span[(size_t)j * cap_items + i] = lo;
        if (j < nj) {
            const bool straddles = lo > t.c0 && __ldg(&chunk_last[lo - 1]) >= x;
            ws.span_lo[(size_t)j * cap_items + i] = straddles ? lo - 1 : lo;
        }
    }
}

// ------------------------------------------------------------------------------------------
// 2b. wide (cold keys): CTA (chunk j, user u) decodes the user's cold postings inside ads
//     [j*R, (j+1)*R) and accumulates w~ on chip (Alg. 2 l.355-358 with the per-ad accumulator in
//     shared memory).  Accumulation is 32-bit fixed point over native shared integer atomics: with
//     the user's scale S (plan_kernel: |any partial sum| <= sum |w~| < 2^(30-S)), each w~ becomes
//     rint(w~ 2^S); integer addition is exact and order-free (deterministic), and the one rounding
//     is the final int -> fp32 conversion (exact for the dyadic inputs of exact mode; otherwise the
//     quantisation error is <= 2^-31 of the user's bound per hit).  fp32 shared atomics are CAS
//     loops on sm_100a.  Units of 16 posting chunks are load-balanced over the CTA's warps by an
//     exclusive scan of the items' unit counts (the paper's ExclusiveScan + LoadBalance,
//     l.353-354).  W is written tile-major with coalesced 16-byte stores; nothing to re-zero.
// ------------------------------------------------------------------------------------------
constexpr int kWideThreads = EBR_WIDE_T;
constexpr int kWideItems = kWideThreads;   // items per pass of the unit scan
#ifndef EBR_BUNIT
#define EBR_BUNIT 8
#endif
constexpr int kBUnit = EBR_BUNIT;          // posting chunks per work unit (<= 32)
#ifndef EBR_UNIT_MAP
#define EBR_UNIT_MAP 1024
#endif
constexpr int kUnitMap = EBR_UNIT_MAP;     // units with a direct unit -> item entry (beyond: a walk)
constexpr int kWideMinBlocks = (2048 / kWideThreads) < (200 * 1024 / (kWideR * 4)) ? (2048 / kWideThreads)
                                                                                    : (200 * 1024 / (kWideR * 4));
__global__ void __launch_bounds__(kWideThreads, kWideMinBlocks > 0 ? kWideMinBlocks : 1) wide_smem_kernel(const uint2* __restrict__ hdr,
                                                                    const uint32_t* __restrict__ payload,
                                                                    BatchWs ws, int nj, int64_t n_pad,
                                                                    int cap_items) {
    extern __shared__ __align__(16) int32_t acc[];   // [kWideR]
    __shared__ uint32_t sLo[kWideItems], sHi[kWideItems], sUoff[kWideItems + 1], sScan[40], sCtr;
    __shared__ uint16_t sUnitItem[kUnitMap];
    __shared__ int32_t sF[kWideItems];
    __shared__ uint32_t sKwb[kWideItems];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = kWideThreads / 32;
    const int j = blockIdx.x, u = blockIdx.y;
    const int64_t a0 = (int64_t)j * kWideR;
    const int64_t a1 = (a0 + kWideR < n_pad) ? a0 + kWideR : n_pad;
    {
        int4* a4 = reinterpret_cast<int4*>(acc);
        for (int i = tid; i < kWideR / 4; i += kWideThreads) a4[i] = make_int4(0, 0, 0, 0);
    }
    const uint32_t i0 = __ldcg(&ws.user_item[u]), i1 = __ldcg(&ws.user_item[u + 1]);
    const int S = __ldcg(&ws.user_shift[u]);
    for (uint32_t ib = i0; ib < i1; ib += kWideItems) {
        const uint32_t ni = min((uint32_t)kWideItems, i1 - ib);
        uint32_t nu_units = 0, lo = 0;
        if ((uint32_t)tid < ni) {
            const uint32_t it = ib + tid;
            const BItem t = ws.items[it];
            lo = __ldcg(&ws.span_lo[(size_t)j * cap_items + it]);
            const uint32_t s1 = __ldcg(&ws.span[(size_t)(j + 1) * cap_items + it]);
            nu_units = s1 > lo ? (s1 - lo + kBUnit - 1) / kBUnit : 0;
            sF[tid] = (int32_t)__float2ll_rn(ldexpf(t.w, S));   // |w~ 2^S| < 2^30
            sHi[tid] = s1;
            sKwb[tid] = t.kwb;
        }
        uint32_t tot;
        const uint32_t pre = block_exclusive_scan(nu_units, sScan, &tot);
        if ((uint32_t)tid < ni) {
            sLo[tid] = lo;
            sUoff[tid] = pre;
            for (uint32_t v = pre; v < pre + nu_units && v < (uint32_t)kUnitMap; ++v) sUnitItem[v] = (uint16_t)tid;
        }
        if (tid == 0) { sUoff[ni] = tot; sCtr = 0u; }
        __syncthreads();
        // units of up to kBUnit chunks are claimed dynamically from a shared counter (load balance
        // across the CTA's warps; a warp's claims increase, so its item index walks forward) and
        // software-pipelined: the next unit's chunk headers are in flight while this unit's
        // payload words are extracted and scattered
        struct BUnit { uint32_t unit; int l; uint32_t cb, nc; uint2 h; };
        int lw = 0;
        auto start = [&]() -> BUnit {
            uint32_t unit = 0;
            if (lane == 0) unit = atomicAdd(&sCtr, 1u);
            BUnit r{__shfl_sync(FULL, unit, 0), 0, 0u, 0u, make_uint2(0u, 0u)};
            if (r.unit < tot) {
                if (r.unit < (uint32_t)kUnitMap) lw = sUnitItem[r.unit];       // unit -> item map
                else while (sUoff[lw + 1] <= r.unit) ++lw;
                r.l = lw;
                r.cb = sLo[lw] + (r.unit - sUoff[lw]) * kBUnit;
                r.nc = min(r.cb + kBUnit, sHi[lw]) - r.cb;
                if ((uint32_t)lane < r.nc) r.h = __ldg(&hdr[r.cb + lane]);
            }
            return r;
        };
        BUnit cur = start();
        while (cur.unit < tot) {
            const uint32_t kwb = sKwb[cur.l];
            uint32_t lo_w[kBUnit], hi_w[kBUnit];
#pragma unroll
            for (int qq = 0; qq < kBUnit; ++qq) {
                lo_w[qq] = 0u;
                hi_w[qq] = 0u;
                if ((uint32_t)qq >= cur.nc) break;             // warp-uniform
                const uint32_t meta = __shfl_sync(FULL, cur.h.y, qq);
                const uint32_t n = (meta & 31u) + 1u, bw = (meta >> 5) & 31u;
                if (lane >= 1 && (uint32_t)lane < n && bw) {
                    const uint32_t bit = (uint32_t)(lane - 1) * bw;
                    const uint32_t wi = kwb + (meta >> 10) + (bit >> 5);
                    lo_w[qq] = __ldg(&payload[wi]);
                    hi_w[qq] = __ldg(&payload[wi + 1]);
                }
            }
            const BUnit nxt = start();                       // overlaps this unit's payload round trip
            const int32_t Fv = sF[cur.l];
#pragma unroll
            for (int qq = 0; qq < kBUnit; ++qq) {
                if ((uint32_t)qq >= cur.nc) break;
                const uint32_t meta = __shfl_sync(FULL, cur.h.y, qq);
                const uint32_t first = __shfl_sync(FULL, cur.h.x, qq);
                const uint32_t n = (meta & 31u) + 1u, bw = (meta >> 5) & 31u;
                uint32_t g;
                if (lane == 0) {
                    g = first;
                } else if ((uint32_t)lane < n) {
                    uint32_t v = 0u;
                    if (bw) {
                        const uint32_t bit = (uint32_t)(lane - 1) * bw;
                        v = (uint32_t)(((((uint64_t)hi_w[qq]) << 32) | lo_w[qq]) >> (bit & 31u)) & ((1u << bw) - 1u);
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
                if ((uint32_t)lane < n && (int64_t)g >= a0 && (int64_t)g < a1) atomicAdd(&acc[g - a0], Fv);
            }
            cur = nxt;
        }
        __syncthreads();
    }
    const float inv = ldexpf(1.f, -S);
    const int64_t t0 = a0 / kTileM;
    // dense W[tile][u][row]: the chunk spans (a1 - a0) / 128 tiles; 32 float4 per (tile, user) row
    const int4* a4 = reinterpret_cast<const int4*>(acc);
    for (int64_t i = tid; i < (a1 - a0) / 4; i += kWideThreads) {
        const int4 v = a4[i];
        float4 o;
        o.x = v.x ? (float)v.x * inv : 0.f;          // int -> fp32: the one rounding; * 2^-S exact
        o.y = v.y ? (float)v.y * inv : 0.f;
        o.z = v.z ? (float)v.z * inv : 0.f;
        o.w = v.w ? (float)v.w * inv : 0.f;
        const int64_t t = t0 + (i >> 5);
        __stcg(reinterpret_cast<float4*>(ws.W + ((size_t)t * kGroup + u) * kTileM) + (i & 31), o);
    }
}

// ------------------------------------------------------------------------------------------
// 3/5. tcgen05 GEMM with the fused epilogue
// ------------------------------------------------------------------------------------------
struct GemmParams {
    int64_t n_ads, n_pad;
    uint32_t ad_begin;
    int d_pad, n_kb;       // deep K blocks of 64
    int n_hb;              // hot-key K blocks of 64 (A side: H; B side: kHotPieces blocks each)
    int u_blocks;          // K blocks of the user tile: n_kb + n_hb * kHotPieces
    int nu, nu_pad;        // users in this group (valid / padded to 32)
    int n_tiles;           // tiles to process in this launch
    int tile_stride;       // 1 (all tiles) or kSampleStride (sample)
    int n_samp;            // sample buffer row length (ads)
    int stages;            // A/H ring stages (16 KB each)
    int wstages;           // W ring stages (one 32-user x 128-ad fp32 chunk = 16 KB each)
    int64_t cap;           // candidate capacity per user
    BatchWs ws;
};

template <int MODE>   // 0: sample (store s), 1: filter (append keys >= theta)
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmH,
            const __grid_constant__ CUtensorMap tmU, const GemmParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u_bytes = p.nu_pad * 128 * p.u_blocks;
    const int nkt = p.n_kb + p.n_hb;                                // A-side K blocks per tile
    unsigned char* sU = smem;                                       // [u_blocks][nu_pad rows x 128 B]
    unsigned char* sA = smem + ((u_bytes + 1023) & ~1023);          // ring: [stages][128 x 128 B]
    float* sW = reinterpret_cast<float*>(sA + (size_t)p.stages * kBlockBytes);   // [wstages][32][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sA + (size_t)(p.stages + p.wstages) * kBlockBytes);
    uint64_t* full = bars;                       // [stages]
    uint64_t* empty = bars + p.stages;           // [stages]
    uint64_t* wfull = bars + 2 * p.stages;       // [wstages] W chunk landed
    uint64_t* wempty = wfull + p.wstages;        // [wstages] W chunk read by its 4 loader warps
    uint64_t* tfull = wempty + p.wstages;        // [kAccStages] MMA done -> epilogue
    uint64_t* tempty = tfull + kAccStages;       // [kAccStages] epilogue drained -> wide loaders
    uint64_t* wready = tempty + kAccStages;      // [kAccStages] wide term stored -> MMA
    uint64_t* ufull = wready + kAccStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ufull + 1);
    uint64_t* sTheta = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // [kGroup]
    float* sThetaS = reinterpret_cast<float*>(sTheta + kGroup);       // score part of theta, [kGroup]

    if (tid == 0) {
        for (int s = 0; s < p.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < p.wstages; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 4); }
        for (int s = 0; s < kAccStages; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kEpiWarps);
            mbar_init(&wready[s], kLoadWarps);
        }
        mbar_init(ufull, 1);
        fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc(tmem_slot, kAccStages * 128);     // kAccStages x 128 user columns
    if (MODE == 1)
        for (int i = tid; i < p.nu_pad; i += kGemmThreads) {
            sTheta[i] = __ldcg(&p.ws.theta[i]);
            sThetaS[i] = score_of(sTheta[i]);       // key >= theta implies score >= this
        }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            tc::tma_prefetch(&tmA);
            if (p.n_hb) tc::tma_prefetch(&tmH);
            tc::tma_prefetch(&tmU);
            mbar_arrive_expect_tx(ufull, (uint32_t)u_bytes);
            for (int kb = 0; kb < p.u_blocks; ++kb)
                tc::tma_load_2d(sU + (size_t)kb * p.nu_pad * 128, &tmU, kb * kBlockK, 0, ufull);
            uint32_t gb = 0;                                 // ring position (one K block per stage)
            const uint64_t pol = tc::policy_evict_first();   // A and H are read once per pass
            for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
                const int row0 = t * p.tile_stride * kTileM;
                for (int kb = 0; kb < nkt; ++kb, ++gb) {
                    const uint32_t slot = gb % p.stages, round = gb / p.stages;
                    if (round > 0) mbar_wait_sleep(&empty[slot], (round - 1) & 1);
                    mbar_arrive_expect_tx(&full[slot], (uint32_t)kBlockBytes);
                    if (kb < p.n_kb)
                        tc::tma_load_2d_hint(sA + (size_t)slot * kBlockBytes, &tmA, kb * kBlockK, row0, &full[slot], pol);
                    else
                        tc::tma_load_2d_hint(sA + (size_t)slot * kBlockBytes, &tmH, (kb - p.n_kb) * kBlockK, row0,
                                             &full[slot], pol);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (one thread) ----------------
            // The accumulator stage already holds the tile's wide term (stored by the loader warps),
            // so every MMA accumulates: D = W + A U^T (+ H (hi, mid, lo)^T).
            const uint32_t idesc = tc::idesc_bf16_m128(p.nu_pad);
            mbar_wait_sleep(ufull, 0);
            tc::fence_after();
            int it = 0;
            uint32_t gb = 0;
            for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
                const int acc = it % kAccStages;
                mbar_wait_sleep(&wready[acc], (it / kAccStages) & 1);
                tc::fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * 128);
                for (int kb = 0; kb < nkt; ++kb, ++gb) {
                    const uint32_t slot = gb % p.stages;
                    mbar_wait_sleep(&full[slot], (gb / p.stages) & 1);
                    tc::fence_after();
                    const uint64_t da0 = tc::sdesc_sw128(sA + (size_t)slot * kBlockBytes);
                    // deep block kb pairs with user block kb; hot block h with its kHotPieces
                    // user blocks (the same one-hot A tile times hi, mid and lo of w~)
                    const int np = kb < p.n_kb ? 1 : kHotPieces;
                    const int ub0 = kb < p.n_kb ? kb : p.n_kb + (kb - p.n_kb) * kHotPieces;
                    for (int pc = 0; pc < np; ++pc) {
                        const uint64_t db0 = tc::sdesc_sw128(sU + (size_t)(ub0 + pc) * p.nu_pad * 128);
#pragma unroll
                        for (int k = 0; k < kBlockK / 16; ++k)   // +32 bytes per K step inside the swizzle row
                            tc::umma_f16(d_tmem, da0 + (uint64_t)(k * 2), db0 + (uint64_t)(k * 2), idesc, 1u);
                    }
                    tc::umma_commit(&empty[slot]);     // ring stage free once these MMAs completed
                }
                tc::umma_commit(&tfull[acc]);      // accumulator ready for the epilogue
            }
        }
    } else if (warp == 3) {
        if (lane == 0) {
            // ---------------- W producer: the tile's 16 KB user chunks of W -> smem ring ----------------
            // (bulk copies, the blocks streamed into L2 kWPrefetch tiles ahead)
            const int nwc = p.nu_pad / 32;
            const uint64_t keep = tc::policy_evict_last(), drop = tc::policy_evict_first();
            auto prefetch = [&](int t) {     // held in L2 (evict_last) until its bulk copy reads it
                if (t < p.n_tiles)
                    tc::bulk_prefetch_l2_hint(p.ws.W + (size_t)t * p.tile_stride * kGroup * kTileM,
                                              (uint32_t)p.nu_pad * kTileM * 4, keep);
            };
            for (int k = 0; k < kWPrefetch; ++k) prefetch(blockIdx.x + k * gridDim.x);
            uint32_t g = 0;
            for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
                prefetch(t + kWPrefetch * gridDim.x);
                const float* src = p.ws.W + (size_t)t * p.tile_stride * kGroup * kTileM;
                for (int ch = 0; ch < nwc; ++ch, ++g) {
                    const uint32_t slot = g % p.wstages, round = g / p.wstages;
                    if (round > 0) mbar_wait_sleep(&wempty[slot], (round - 1) & 1);
                    mbar_arrive_expect_tx(&wfull[slot], (uint32_t)kBlockBytes);
                    tc::bulk_g2s_hint(sW + (size_t)slot * 32 * kTileM, src + (size_t)ch * 32 * kTileM,
                                      (uint32_t)kBlockBytes, &wfull[slot], drop);
                }
            }
        }
    } else if (warp >= kLoadWarp0) {
        // ---------------- wide loaders: W -> TMEM accumulator stage (before the MMA) ----------------
        // loader warp q owns TMEM lane quadrant q (rows q*32..q*32+31) and walks the tile's 32-user
        // chunks in ring order (the 4 loader warps are the only consumers of every W slot and take
        // them strictly in sequence, so mbarrier parities never alias): read its 32 x 32 block
        // from smem (conflict-free: lanes read consecutive rows), free the slot, and store the block
        // into the accumulator stage once the epilogue has drained it (kAccStages tiles earlier).
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int nwc = p.nu_pad / 32;
        int it = 0;
        uint32_t g = 0;
        for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
            const int acc = it % kAccStages;
            const int64_t tw = (int64_t)t * p.tile_stride;              // global tile index
            const bool valid = tw * kTileM + row < p.n_ads;
            for (int ch = 0; ch < nwc; ++ch, ++g) {
                const int c = ch * 32;
                const uint32_t slot = g % p.wstages;
                mbar_wait_sleep(&wfull[slot], (g / p.wstages) & 1);
                const float* w = sW + (size_t)slot * 32 * kTileM + row;
                uint32_t wf[32];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    wf[j] = (valid && c + j < p.nu) ? __float_as_uint(w[j * kTileM]) : 0u;
                __syncwarp();
                if (lane == 0) mbar_arrive(&wempty[slot]);
                if (ch == 0 && it >= kAccStages) mbar_wait_sleep(&tempty[acc], ((it / kAccStages) - 1) & 1);
                tc::fence_after();
                tc::tmem_st32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 128 + c), wf);
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&wready[acc]);
        }
    } else if (warp >= kEpiWarp0) {
        // ---------------- epilogue: TMEM -> registers, key, filter ----------------
        const int e = warp - kEpiWarp0;
        const int q = warp & 3;                    // TMEM lane quadrant of this warp
        const int row = q * 32 + lane;             // ad row inside the tile
        int it = 0;
        for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
            const int acc = it % kAccStages;
            const int64_t a = (int64_t)t * p.tile_stride * kTileM + row;   // shard-local ad
            const bool valid = a < p.n_ads;
            mbar_wait_sleep(&tfull[acc], (it / kAccStages) & 1);
            tc::fence_after();
#pragma unroll 1
            for (int ch = 0; ch < kEpiChunks; ++ch) {
                const int c = (e >> 2) * (32 * kEpiChunks) + ch * 32;   // this chunk's 32 users
                if (c >= p.nu_pad) break;
                uint32_t r[32];
                tc::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 128 + c), r);
                const int nuc = p.nu - c;                 // valid users in these 32 columns
                const uint32_t umask = nuc >= 32 ? 0xFFFFFFFFu : (nuc > 0 ? (1u << nuc) - 1u : 0u);
                if (MODE == 0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        float s = __uint_as_float(r[j]);
                        if (s == 0.f) s = 0.f;                       // -0 -> +0 (R14)
                        if ((umask >> j) & 1u)
                            p.ws.samp[(size_t)(c + j) * p.n_samp + (int64_t)t * kTileM + row] =
                                valid ? s : __int_as_float(0xFF800000);
                    }
                } else {
                    // branch-free pre-filter of all 32 columns, then the exact key compare only
                    // for the columns where some lane passed
                    uint32_t pass = 0;
                    const float4* th4 = reinterpret_cast<const float4*>(sThetaS + c);
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const float4 th = th4[j4];
                        pass |= (__uint_as_float(r[j4 * 4 + 0]) >= th.x ? 1u : 0u) << (j4 * 4 + 0);
                        pass |= (__uint_as_float(r[j4 * 4 + 1]) >= th.y ? 1u : 0u) << (j4 * 4 + 1);
                        pass |= (__uint_as_float(r[j4 * 4 + 2]) >= th.z ? 1u : 0u) << (j4 * 4 + 2);
                        pass |= (__uint_as_float(r[j4 * 4 + 3]) >= th.w ? 1u : 0u) << (j4 * 4 + 3);
                    }
                    pass &= valid ? umask : 0u;
                    // compact (not unrolled) loop over the columns where some lane passed: the
                    // unrolled form overflowed the instruction cache (ncu: no_instruction stalls)
                    uint32_t cols = __reduce_or_sync(FULL, pass);
#pragma unroll 1
                    while (cols) {
                        const int j = __ffs(cols) - 1;
                        cols &= cols - 1u;
                        {
                            const int u = c + j;
                            const bool maybe = (pass >> j) & 1u;
                            float s = 0.f;
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) s = (jj == j) ? __uint_as_float(r[jj]) : s;
                            if (s == 0.f) s = 0.f;                       // -0 -> +0 (R14)
                            const uint64_t key = maybe ? kappa_of(s, p.ad_begin + (uint32_t)a) : 0ull;
                            const bool take = maybe && key >= sTheta[u];
                            const unsigned m = __ballot_sync(FULL, take);
                            if (m) {
                                const int leader = __ffs(m) - 1;
                                uint32_t pos = 0;
                                if (lane == leader) pos = atomicAdd(&p.ws.cand_count[u], (uint32_t)__popc(m));
                                pos = __shfl_sync(FULL, pos, leader) + __popc(m & ((1u << lane) - 1u));
                                if (take && pos < p.cap) p.ws.cand[(size_t)u * p.cap + pos] = key;
                            }
                        }
                    }
                }
            }
            // every chunk of this stage is in registers (and consumed): hand it to the loaders
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    __syncwarp();
    tc::fence_before();
    __syncthreads();
    if (warp == 2) tc::tmem_dealloc(tmem_base, kAccStages * 128);
}

// ------------------------------------------------------------------------------------------
// 4. theta: the K-th largest key of each user's sampled ads
// ------------------------------------------------------------------------------------------
// Two histogram passes over ord(score) (11 + 11 bits; per-warp-group private histograms, 8-wide
// vector loads in flight) narrow the K-th largest down to a 22-bit score prefix T; the sampled keys
// with ord >= T (K plus the few in T's bucket) are compacted into shared memory and the exact K-th
// largest key is selected there.  Only if that bucket is huge (massive score ties) does the kernel
// fall back to the radix select over the whole sample in global memory.
constexpr int kThetaThreads = 1024;
constexpr int kThetaCopies = 8;    // private histograms (warps w and w+8, w+16, ... share one)

__device__ __forceinline__ uint32_t samp_ord(float s) { return ord_of(s); }

// Warp 0: the digit t with count(> t) < need <= count(>= t) in hist[0..2048); writes
// sScalar[0] = t, sScalar[1] = count(> t).
__device__ __forceinline__ void theta_find_digit(const uint32_t* hist, uint32_t need, uint32_t* sScalar) {
    const int lane = threadIdx.x & 31;
    constexpr int per = 2048 / 32;
    uint32_t local = 0;
    for (int j = 0; j < per; ++j) local += hist[2047 - (lane * per + j)];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
    }
    uint32_t c = incl - local;
    int found = -1;
    uint32_t above = 0;
    if (c < need && c + local >= need) {
        for (int j = 0; j < per; ++j) {
            const int d = 2047 - (lane * per + j);
            const uint32_t h = hist[d];
            if (found < 0 && c + h >= need) { found = d; above = c; }
            c += h;
        }
    }
    const unsigned m = __ballot_sync(FULL, found >= 0);
    const int src = m ? __ffs(m) - 1 : 0;
    const int t = __shfl_sync(FULL, found, src);
    const uint32_t ab = __shfl_sync(FULL, above, src);
    if (lane == 0) { sScalar[0] = m ? (uint32_t)t : 0u; sScalar[1] = m ? ab : 0u; }
}

__global__ void __launch_bounds__(kThetaThreads, 1) theta_kernel(BatchWs ws, int n_samp, int K, uint32_t ad_begin,
                                                                int nu, int scap) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t sScalar[8];
    const int u = blockIdx.x;
    if (u >= nu) return;
    const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5;
    const int P = pow2ceil_i(K);
    uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);                 // [P]
    uint32_t* hist = reinterpret_cast<uint32_t*>(sbuf + P);             // [kThetaCopies][2048]
    uint64_t* scand = reinterpret_cast<uint64_t*>(hist + kThetaCopies * 2048);   // [scap]
    uint32_t* myh = hist + (warp % kThetaCopies) * 2048;
    const float* sp = ws.samp + (size_t)u * n_samp;
    const float4* sp4 = reinterpret_cast<const float4*>(sp);
    const int n4 = n_samp / 4;                                          // n_samp is a multiple of 128
    auto ad_of = [](int64_t i) { return (i / kTileM) * kSampleStride * kTileM + (i % kTileM); };
    uint32_t prefix = 0, need = (uint32_t)K;
    for (int pass = 0; pass < 2; ++pass) {
        const int shift = pass == 0 ? 21 : 10;
        for (int i = tid; i < kThetaCopies * 2048; i += nt) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < n4; i += 2 * nt) {
            float4 v[2];
            v[0] = __ldcg(&sp4[i]);
            v[1] = (i + nt < n4) ? __ldcg(&sp4[i + nt]) : make_float4(0.f, 0.f, 0.f, 0.f);
            const int nv = (i + nt < n4) ? 2 : 1;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q >= nv) break;
                const float f[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint32_t o = samp_ord(f[r]);
                    if (pass == 0 || (o >> 21) == (prefix >> 21)) atomicAdd(&myh[(o >> shift) & 2047u], 1u);
                }
            }
        }
        __syncthreads();
        for (int b = tid; b < 2048; b += nt) {
            uint32_t s = 0;
#pragma unroll
            for (int c = 0; c < kThetaCopies; ++c) s += hist[c * 2048 + b];
            hist[b] = s;
        }
        __syncthreads();
        if (warp == 0) theta_find_digit(hist, need, sScalar);
        __syncthreads();
        prefix |= sScalar[0] << shift;
        need -= sScalar[1];
        // one pass is enough when every key in the digit's bin and above fits the compaction
        // buffer: then compact {ord >> 21 >= digit} directly (the second histogram pass is skipped)
        const bool done = pass == 0 && (uint64_t)sScalar[1] + hist[sScalar[0]] <= (uint64_t)scap;
        __syncthreads();
        if (done) break;
    }
    // keys with ord >= prefix: at least K of them; compact into shared memory
    if (tid == 0) sScalar[2] = 0;
    __syncthreads();
    for (int i = tid; i < n_samp; i += nt) {
        const float s = __ldcg(&sp[i]);
        if (samp_ord(s) >= prefix) {
            const uint32_t pos = atomicAdd(&sScalar[2], 1u);
            if ((int)pos < scap) scand[pos] = kappa_of(s, ad_begin + (uint32_t)ad_of(i));
        }
    }
    __syncthreads();
    const int64_t cnt = sScalar[2];
    __syncthreads();
    int nsel;
    if (cnt <= scap) {
        nsel = cta_select_topk([scand](int64_t i) { return scand[i]; }, cnt, K, sbuf, nullptr, 0, hist, sScalar);
    } else {
        auto get = [sp, ad_begin, ad_of](int64_t i) { return kappa_of(__ldcg(&sp[i]), ad_begin + (uint32_t)ad_of(i)); };
        nsel = cta_select_topk(get, n_samp, K, sbuf, nullptr, 0, hist, sScalar);
    }
    if (tid == 0) {
        ws.theta[u] = (nsel >= K) ? sbuf[K - 1] : 0ull;
        ws.cand_count[u] = 0;
    }
}

// ------------------------------------------------------------------------------------------
// 6. final: exact top-K of the candidates
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1) final_kernel(BatchWs ws, int64_t cap, int K, int nu, int32_t* out_ids,
                                                       float* out_scores, uint64_t* out_keys, int64_t scap) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t sScalar[8];
    const int u = blockIdx.x;
    if (u >= nu) return;
    const int64_t n = __ldcg(&ws.cand_count[u]);
    if (n > cap) {   // overflow: recomputed by the latency path
        if (threadIdx.x == 0) { ws.overflow[u] = 1; atomicAdd(&ws.header[1], 1u); }
        return;
    }
    // fewer than K ads reached theta (possible only when theta was taken at a rank below K of the
    // sample): the top-K is not guaranteed inside the candidates -- the host reruns the group with
    // rank K (inventories reaching this path hold >= 64 K ads, so n >= K otherwise)
    if (n < K) {
        if (threadIdx.x == 0) atomicAdd(&ws.header[2], 1u);
        return;
    }
    const int P = pow2ceil_i(K);
    uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);
    uint32_t* shist = reinterpret_cast<uint32_t*>(sbuf + P);
    uint64_t* scand = reinterpret_cast<uint64_t*>(shist + kSelBins);
    const uint64_t* cb = ws.cand + (size_t)u * cap;
    const int nsel = cta_select_topk([cb](int64_t i) { return __ldcg(&cb[i]); }, n, K, sbuf, scand, scap,
                                     shist, sScalar);
    cta_write_topk(sbuf, nsel, K, out_ids ? out_ids + (size_t)u * K : nullptr,
                   out_scores ? out_scores + (size_t)u * K : nullptr, out_keys ? out_keys + (size_t)u * K : nullptr);
}

// ------------------------------------------------------------------------------------------
// host
// ------------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult qres;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) == cudaSuccess &&
            qres == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

static bool encode_2d_bf16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                           uint32_t box_rows) {
    auto fn = get_encode();
    if (!fn) return false;
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {inner * 2};
    const cuuint32_t box[2] = {box_inner, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Layout {
    size_t header, items, chunk_off, U, W, samp, theta, count, cand, overflow, user_item, user_shift, span, span_lo, total;
    int64_t cap, n_samp, cap_items, nj;
};

static Layout layout(const ebr_index* idx, int32_t slots, int32_t k) {
    Layout L;
    auto al = [](size_t x) { return (x + 1023) & ~(size_t)1023; };
    const int64_t n_tiles = idx->n_pad / kTileM;
    L.n_samp = ((n_tiles + kSampleStride - 1) / kSampleStride) * kTileM;
    L.cap = std::max<int64_t>((int64_t)kSampleStride * k * 8, 1 << 16);
    L.cap_items = (int64_t)kGroup * idx->n_fields * slots;
    size_t o = 0;
    L.header = o;    o = al(o + 64);
    L.items = o;     o = al(o + (size_t)L.cap_items * sizeof(BItem));
    L.chunk_off = o; o = al(o + (size_t)(L.cap_items + 1) * 8);
    L.U = o;         o = al(o + (size_t)kGroup * (idx->d_pad + kHotPieces * idx->n_hot) * 2);
    L.W = o;         o = al(o + (size_t)kGroup * idx->n_pad * 4);
    L.samp = o;      o = al(o + (size_t)kGroup * L.n_samp * 4);
    L.theta = o;     o = al(o + (size_t)kGroup * 8);
    L.count = o;     o = al(o + (size_t)kGroup * 4);
    L.cand = o;      o = al(o + (size_t)kGroup * L.cap * 8);
    L.overflow = o;  o = al(o + (size_t)kGroup * 4);
    L.nj = (idx->n_pad + kWideR - 1) / kWideR;
    L.user_item = o; o = al(o + (size_t)(kGroup + 1) * 4);
    L.user_shift = o; o = al(o + (size_t)kGroup * 4);
    L.span = o;      o = al(o + (size_t)L.cap_items * (L.nj + 1) * 4);
    L.span_lo = o;   o = al(o + (size_t)L.cap_items * L.nj * 4);
    L.total = o;
    return L;
}

static BatchWs carve(char* base, const Layout& L) {
    BatchWs w;
    w.header = reinterpret_cast<uint32_t*>(base + L.header);
    w.items = reinterpret_cast<BItem*>(base + L.items);
    w.chunk_off = reinterpret_cast<uint64_t*>(base + L.chunk_off);
    w.U = reinterpret_cast<__nv_bfloat16*>(base + L.U);
    w.W = reinterpret_cast<float*>(base + L.W);
    w.samp = reinterpret_cast<float*>(base + L.samp);
    w.theta = reinterpret_cast<uint64_t*>(base + L.theta);
    w.cand_count = reinterpret_cast<uint32_t*>(base + L.count);
    w.cand = reinterpret_cast<uint64_t*>(base + L.cand);
    w.overflow = reinterpret_cast<uint32_t*>(base + L.overflow);
    w.user_item = reinterpret_cast<uint32_t*>(base + L.user_item);
    w.user_shift = reinterpret_cast<int32_t*>(base + L.user_shift);
    w.span = reinterpret_cast<uint32_t*>(base + L.span);
    w.span_lo = reinterpret_cast<uint32_t*>(base + L.span_lo);
    return w;
}

}  // namespace batch

using namespace batch;

bool batch_eligible(const ebr_index* idx, int32_t batch, int32_t k) {
    if (getenv("EBR_NO_BATCH_PATH")) return false;
    // small batches take the tensor-core path too on large inventories, where the latency path's
    // per-user wide scratch no longer fits L2 (C5 sweep: B=4 at 20 M ads 3.9 ms latency path)
    const bool big = idx->n_ads >= ((int64_t)1 << 21);
    return idx->dtype == EBR_BF16 && (batch >= 16 || (big && batch >= 4)) && idx->d_pad <= 256 &&
           idx->n_ads >= (int64_t)4 * kSampleStride * std::max(k, kTileM) && get_encode() != nullptr;
}

size_t batch_workspace_bytes(const ebr_index* idx, int32_t slots, int32_t k) {
    return layout(idx, slots, k).total + 1024;
}

// The workspace passed here is the batched region (after the latency path's region).
ebr_status run_batch(const QueryArgs& q, void* region, uint32_t* err_word) {
    const ebr_index* idx = q.idx;
    const Layout L = layout(idx, q.slots, q.k);
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(region) + 1023) & ~(uintptr_t)1023);
    BatchWs ws = carve(base, L);
    const int n_kb = idx->d_pad / kBlockK;
    const int n_tiles = (int)(idx->n_pad / kTileM);
    const int n_samp_tiles = (int)(L.n_samp / kTileM);
    cudaError_t e = cudaMemsetAsync(ws.overflow, 0, (size_t)kGroup * 4, q.stream);
    if (e != cudaSuccess) return cuda_check(e, "memset(overflow)");
    e = cudaFuncSetAttribute(wide_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWideR * 4);
    if (e != cudaSuccess) return cuda_check(e, "attr(wide)");
    CUtensorMap tmA, tmH;
    if (!encode_2d_bf16(&tmA, idx->A, (uint64_t)idx->d_pad, (uint64_t)idx->n_pad, kBlockK, kTileM))
        return set_error(EBR_ECUDA, "cuTensorMapEncodeTiled(A) failed");
    if (idx->n_hot > 0) {
        if (!encode_2d_bf16(&tmH, idx->H, (uint64_t)idx->n_hot, (uint64_t)idx->n_pad, kBlockK, kTileM))
            return set_error(EBR_ECUDA, "cuTensorMapEncodeTiled(H) failed");
    } else {
        tmH = tmA;   // unused
    }
    int max_smem = 0;
    e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, idx->device);
    if (e != cudaSuccess) return cuda_check(e, "attr(max smem)");
    e = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kGroup * kMaxHot * 4);
    if (e != cudaSuccess) return cuda_check(e, "attr(plan)");
    std::vector<int> overflow_users;
    // test hook: a smaller candidate capacity exercises the overflow -> latency-path fallback
    int64_t cap = L.cap;
    if (const char* c = getenv("EBR_TEST_CAND_CAP")) cap = std::min<int64_t>(cap, std::max(1, atoi(c)));
    for (int g0 = 0; g0 < q.batch; g0 += kGroup) {
        const int nu = std::min(kGroup, q.batch - g0);
        const int nu_pad = (nu + 31) & ~31;
        // hot K blocks: as many as fit next to the resident user tile with >= 4 ring stages
        const size_t fixed = 1024 + 512 + (size_t)kGroup * 12;
        const int wstages = 2;
        auto smem_of = [&](int hb, int st) {
            return fixed + (((size_t)nu_pad * 128 * (n_kb + kHotPieces * hb) + 1023) & ~(size_t)1023) +
                   (size_t)(st + wstages) * kBlockBytes;
        };
        // hot K blocks pay per ad (2 B x 64 keys of H) and save per (ad, user) hit; block b (in
        // decreasing coverage) pays off from ~2, 14, 30, 60 users: cap by group size
        int n_hb = idx->n_hot / 64;
        n_hb = std::min(n_hb, nu < 14 ? 1 : nu < 30 ? 2 : nu < 60 ? 3 : 4);
        if (getenv("EBR_NO_HOT")) n_hb = 0;
        while (n_hb > 0 && smem_of(n_hb, 4) > (size_t)max_smem) --n_hb;
        int stages = 4;
        while (stages < 8 && smem_of(n_hb, stages + 1) <= (size_t)max_smem) ++stages;
        const int u_blocks = n_kb + kHotPieces * n_hb;
        const int u_cols = u_blocks * kBlockK;
        CUtensorMap tmU;
        if (!encode_2d_bf16(&tmU, ws.U, (uint64_t)u_cols, (uint64_t)nu_pad, kBlockK, (uint32_t)nu_pad))
            return set_error(EBR_ECUDA, "cuTensorMapEncodeTiled(U) failed");
        plan_kernel<<<1, 1024, (size_t)nu_pad * n_hb * 64 * 4, q.stream>>>(
            idx->key_chunk_off, idx->key_word_off, idx->cross_w, idx->field_card, idx->field_base, idx->n_fields,
            q.slots, q.user_feat + (size_t)g0 * idx->n_fields * q.slots, q.user_x + (size_t)g0 * idx->n_fields * q.slots,
            reinterpret_cast<const uint16_t*>(q.user_emb) + (size_t)g0 * idx->d, idx->d, idx->d_pad, nu, nu_pad,
            idx->hot_slot, n_hb * 64, u_cols, ws, err_word);
        const int max_items = nu * idx->n_fields * q.slots;
        span_kernel<<<(max_items + 7) / 8, 256, 0, q.stream>>>(idx->chunk_hdr, idx->chunk_last, ws, (int)L.nj,
                                                               (int)L.cap_items);
        wide_smem_kernel<<<dim3((unsigned)L.nj, (unsigned)nu), kWideThreads, kWideR * 4, q.stream>>>(
            idx->chunk_hdr, idx->payload, ws, (int)L.nj, idx->n_pad, (int)L.cap_items);
        GemmParams gp;
        gp.n_ads = idx->n_ads; gp.n_pad = idx->n_pad; gp.ad_begin = (uint32_t)idx->ad_begin;
        gp.d_pad = idx->d_pad; gp.n_kb = n_kb; gp.n_hb = n_hb; gp.u_blocks = u_blocks;
        gp.nu = nu; gp.nu_pad = nu_pad;
        gp.n_samp = (int)L.n_samp; gp.stages = stages; gp.wstages = wstages; gp.cap = cap; gp.ws = ws;
        const size_t smem = smem_of(n_hb, stages);
        // sample pass
        gp.n_tiles = n_samp_tiles; gp.tile_stride = kSampleStride;
        e = cudaFuncSetAttribute(gemm_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_check(e, "attr(gemm0)");
        gemm_kernel<0><<<std::min(idx->sm_count, n_samp_tiles), kGemmThreads, smem, q.stream>>>(tmA, tmH, tmU, gp);
        // theta at sample rank r, the filter pass over every tile, the final select.  The sample
        // is every 16th tile, so ~K/16 sampled keys lie above the K-th largest overall: taking
        // theta at r = K/16 + 5 sqrt(K/16) + 8 (< K) instead of K cuts the candidates ~10x; a
        // user left with fewer than K candidates (counted by final_kernel) makes the group rerun
        // with r = K, which guarantees >= K candidates (exact either way)
        const size_t tsmem = 200 * 1024;
        const int tscap = (int)((tsmem - (size_t)pow2ceil_i(q.k) * 8 - kThetaCopies * 2048 * 4) / 8);
        e = cudaFuncSetAttribute(theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
        if (e != cudaSuccess) return cuda_check(e, "attr(theta)");
        e = cudaFuncSetAttribute(gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_check(e, "attr(gemm1)");
        const size_t fsmem = 200 * 1024;
        const int64_t scap = (int64_t)(fsmem - (size_t)pow2ceil_i(q.k) * 8 - kSelBins * 4) / 8;
        e = cudaFuncSetAttribute(final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem);
        if (e != cudaSuccess) return cuda_check(e, "attr(final)");
        const double ks = (double)q.k / kSampleStride;
        int rank = (int)std::ceil(ks + 5.0 * std::sqrt(ks) + 8.0);
        if (getenv("EBR_THETA_RANK")) rank = atoi(getenv("EBR_THETA_RANK"));   // test hook
        rank = std::max(1, std::min(rank, q.k));
        auto select_pass = [&](int r) {
            theta_kernel<<<nu, kThetaThreads, tsmem, q.stream>>>(ws, (int)L.n_samp, r, (uint32_t)idx->ad_begin, nu,
                                                                 tscap);
            gp.n_tiles = n_tiles; gp.tile_stride = 1;
            gemm_kernel<1><<<std::min(idx->sm_count, n_tiles), kGemmThreads, smem, q.stream>>>(tmA, tmH, tmU, gp);
            final_kernel<<<nu, 512, fsmem, q.stream>>>(ws, cap, q.k, nu,
                                                       q.out_ids ? q.out_ids + (size_t)g0 * q.k : nullptr,
                                                       q.out_scores ? q.out_scores + (size_t)g0 * q.k : nullptr,
                                                       q.out_keys ? q.out_keys + (size_t)g0 * q.k : nullptr, scap);
        };
        select_pass(rank);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_check(e, "launch(batch)");
        uint32_t hdr[3] = {0, 0, 0};
        e = cudaMemcpyAsync(hdr, ws.header, 12, cudaMemcpyDeviceToHost, q.stream);
        if (e != cudaSuccess) return cuda_check(e, "memcpy(header)");
        e = cudaStreamSynchronize(q.stream);
        if (e != cudaSuccess) return cuda_check(e, "sync(batch)");
        if (hdr[2] && rank < q.k) {
            // shortfall: the whole group again with theta at rank K (W and the sample are reused)
            e = cudaMemsetAsync(ws.overflow, 0, (size_t)kGroup * 4, q.stream);
            if (e == cudaSuccess) e = cudaMemsetAsync(ws.header + 1, 0, 8, q.stream);
            if (e != cudaSuccess) return cuda_check(e, "memset(rerun)");
            select_pass(q.k);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_check(e, "launch(batch rerun)");
            e = cudaMemcpyAsync(hdr, ws.header, 12, cudaMemcpyDeviceToHost, q.stream);
            if (e != cudaSuccess) return cuda_check(e, "memcpy(header)");
            e = cudaStreamSynchronize(q.stream);
            if (e != cudaSuccess) return cuda_check(e, "sync(batch)");
        }
        // overflowed users of this group: the exact latency path for them
        if (hdr[1]) {
            std::vector<uint32_t> of(nu);
            e = cudaMemcpy(of.data(), ws.overflow, (size_t)nu * 4, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return cuda_check(e, "memcpy(overflow)");
            for (int u = 0; u < nu; ++u)
                if (of[u]) overflow_users.push_back(g0 + u);
            e = cudaMemsetAsync(ws.overflow, 0, (size_t)kGroup * 4, q.stream);
            if (e != cudaSuccess) return cuda_check(e, "memset(overflow)");
        }
    }
    for (int u : overflow_users) {
        ebr_status st = run_small(q, u, 1);
        if (st != EBR_OK) return st;
    }
    return EBR_OK;
}

}  // namespace ebr
