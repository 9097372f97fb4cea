// ebr_small.cu -- the latency path (small user batch, B <= 8 per launch): ONE cooperative,
// persistent kernel per call that runs every step of the hot path:
//
//   phase 0  A1 plan     : each CTA turns the batch's user slots into work items
//                          (key i = base_f + v, w~ = w_i * x_i, the key's chunk span)  (P:277,
//                          Alg. 2 l.352 "k_length")
//   phase 1  per ad range [r0, r1) owned by the CTA, two warp roles run concurrently:
//            wide warps  A2+A3: locate each item's chunks overlapping the range (interpolation
//                          + 32-ary warp search), exclusive-scan the per-item piece counts and
//                          hand 16-chunk pieces to warps from a shared counter (the paper's
//                          ExclusiveScan + LoadBalance, Alg. 2 l.353-354), decode each
//                          chunk warp-cooperatively and add w~ into a shared-memory fp32 array
//                          (Alg. 2 l.358 AtomicAdd, but into SMEM instead of a global array)
//            deep warps  A4: stream A's rows once from HBM with 16-byte non-allocating loads,
//                          dot with the B user vectors held in registers (Eq. 1, fp32 FFMA)
//            then A5 fuse s = deep + wide, write s to an L2-resident scratch and build a
//            per-user 2048-bin histogram of ord(s)'s top 11 bits
//   grid sync
//   phase 3  A6a every CTA finds, per user, the histogram bin holding the K-th largest score
//   phase 4  A6b compaction: every (user, ad) whose bin >= that bin is appended as a 64-bit key
//   grid sync
//   phase 5  A6c one CTA per user: exact radix select + bitonic sort of the candidates, write the
//            sorted top-K (score desc, id asc; reading R13).
//
// The paper's design (T4: a global score array, 9 log2 groups, one global AtomicAdd per posting)
// is prior art; here the whole query is one launch whose HBM traffic is A (read once) plus the
// touched postings.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "ebr_device.cuh"

namespace cg = cooperative_groups;

namespace ebr {
namespace {

constexpr int kWideWarps = 8;
constexpr int kDeepWarps = 8;
static_assert((kWideWarps + kDeepWarps) * 32 == kThreads, "CTA layout");
constexpr int kPiece = 16;     // chunks per load-balanced work unit
constexpr int kDecodeU = 4;    // chunks decoded concurrently by one warp
constexpr int kUnroll = 8;     // row-groups in flight per deep warp

struct SmallParams {
    // index
    const void* A;
    int32_t d, d_pad, lpr;      // lpr: lanes per row (row bytes = lpr * vpl * 16)
    int64_t n_ads, n_pad;
    uint32_t ad_begin;
    const uint32_t* key_chunk_off;
    const uint32_t* key_word_off;
    const uint2* hdr;
    const uint32_t* payload;
    const float* cross_w;
    const int32_t* field_card;
    const int32_t* field_base;
    int32_t n_fields;
    // query (this launch's users)
    const void* U;              // [B][d]
    int32_t B, slots, K;
    const int32_t* user_feat;   // [B][F][S]
    const float* user_x;
    // workspace
    uint32_t* err;
    unsigned long long* timers;  // optional phase stamps (EBR_PHASE_TIMERS=1), else null
    uint32_t* ghist;            // [B][kHistBins]
    uint32_t* cand_count;       // [B]
    float* scores;              // [B][n_pad]
    uint64_t* cand;             // [B][n_pad]
    // outputs
    int32_t* out_ids;           // [B][K] (already offset to this launch's first user)
    float* out_scores;
    uint64_t* out_keys;
    // decomposition
    int32_t R;                  // ads per range
    int32_t n_ranges;
    int32_t items_cap;          // >= B * F * S
};

struct Item {
    uint32_t key, c0, c1, b;
    float w;
};

template <typename T> struct Vec;
template <> struct Vec<float> {
    static constexpr int E = 4;
    __device__ static void unpack(const uint4& v, float* o) {
        o[0] = __uint_as_float(v.x); o[1] = __uint_as_float(v.y);
        o[2] = __uint_as_float(v.z); o[3] = __uint_as_float(v.w);
    }
    __device__ static float elem(const void* p, int64_t i) { return ((const float*)p)[i]; }
};
template <> struct Vec<__nv_bfloat16> {
    static constexpr int E = 8;
    __device__ static void unpack(const uint4& v, float* o) {
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            o[2 * j] = __uint_as_float(w[j] << 16);
            o[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
        }
    }
    __device__ static float elem(const void* p, int64_t i) {
        return __uint_as_float(((uint32_t)((const uint16_t*)p)[i]) << 16);
    }
};

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define EBR_STAMP(i) do { if (p.timers && (tid & 31) == 0) atomicMax(&p.timers[i], gtimer()); } while (0)

__device__ __forceinline__ void wide_bar() {
    asm volatile("bar.sync 1, %0;" ::"n"(kWideWarps * 32));
}

// First chunk index in [c0, c1] whose first id is > x, guessing the position from x's relative
// place in the shard (ad ids of a key are spread over the shard) and checking a 32-chunk window
// before falling back to the 32-ary search.
__device__ __forceinline__ uint32_t locate(const uint2* hdr, uint32_t c0, uint32_t c1, uint32_t x,
                                          int64_t n_ads, int lane) {
    if (c1 <= c0) return c0;
    const uint32_t nch = c1 - c0;
    uint32_t g = c0 + (uint32_t)(((double)x / (double)n_ads) * (double)nch);
    g = min(g, c1 - 1u);
    const uint32_t lo = (g >= c0 + 16u) ? g - 16u : c0;
    const uint32_t hi = min(c1, lo + 32u);
    const uint32_t p = lo + (uint32_t)lane;
    const bool pred = (p < hi) && (__ldg(&hdr[p]).x <= x);
    const uint32_t t = __popc(__ballot_sync(FULL, pred));
    if ((t > 0u || lo == c0) && (t < hi - lo || hi == c1)) return lo + t;
    if (t == 0u) return warp_upper_bound_first(hdr, c0, lo, x, lane);
    return warp_upper_bound_first(hdr, hi, c1, x, lane);
}

template <typename T, int NB, int VPL>
__global__ void __launch_bounds__(kThreads, 1) small_kernel(const SmallParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int B = p.B, R = p.R;
    // ---- shared-memory carve-up (phase 1) ----
    float* sD = reinterpret_cast<float*>(smem);                         // [B][R] deep
    float* sW = sD + (size_t)B * R;                                     // [B][R] wide
    uint32_t* sHist = reinterpret_cast<uint32_t*>(sW + (size_t)B * R);  // [B][bins]
    Item* sItems = reinterpret_cast<Item*>(sHist + (size_t)B * kHistBins);
    uint32_t* sSpanLo = reinterpret_cast<uint32_t*>(sItems + p.items_cap);
    uint32_t* sSpanHi = sSpanLo + p.items_cap;
    uint32_t* sPieceOff = sSpanHi + p.items_cap;                        // [items_cap + 1]
    __shared__ uint32_t sNItems, sPieceCounter, sScalar[8];
    __shared__ uint32_t sBinStar[kSmallMaxB], sAbove[kSmallMaxB];

    // ---- phase 0: A1 plan (redundantly per CTA; B*F*S is small on this path) ----
    if (p.timers && blockIdx.x == 0 && tid == 0) p.timers[0] = gtimer();
    if (tid == 0) sNItems = 0;
    for (int i = tid; i < B * kHistBins; i += kThreads) sHist[i] = 0;
    __syncthreads();
    const int nslot = B * p.n_fields * p.slots;
    for (int i = tid; i < nslot; i += kThreads) {
        const int b = i / (p.n_fields * p.slots);
        const int f = (i / p.slots) % p.n_fields;
        const int32_t v = p.user_feat[i];
        if (v < 0) continue;
        if (v >= p.field_card[f]) {            // bounds error: skip the slot, raise the flag
            if (blockIdx.x == 0) atomicOr(p.err, 1u);
            continue;
        }
        const uint32_t key = (uint32_t)(p.field_base[f] + v);
        Item it;
        it.key = key;
        it.b = (uint32_t)b;
        it.w = __fmul_rn(__ldg(&p.cross_w[key]), p.user_x[i]);   // w~ = fl32(w x)  (R10)
        it.c0 = __ldg(&p.key_chunk_off[key]);
        it.c1 = __ldg(&p.key_chunk_off[key + 1]);
        if (it.c1 > it.c0) sItems[atomicAdd(&sNItems, 1u)] = it;
    }
    __syncthreads();
    const int n_items = (int)sNItems;
    EBR_STAMP(1);

    // user vectors -> registers (deep warps), zero-padded to d_pad
    using V = Vec<T>;
    constexpr int E = V::E;
    float u[NB][VPL][E];
    const int lpr = p.lpr;
    const int sub = lane / lpr, li = lane % lpr, rpw = 32 / lpr;
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int v = 0; v < VPL; ++v)
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int j = (li + v * lpr) * E + e;
                u[b][v][e] = (b < B && j < p.d) ? V::elem(p.U, (int64_t)b * p.d + j) : 0.f;
            }

    // ---- phase 1: ranges ----
    for (int range = blockIdx.x; range < p.n_ranges; range += gridDim.x) {
        const int64_t r0 = (int64_t)range * R;
        const int64_t r1 = ((r0 + R < p.n_ads) ? r0 + R : p.n_ads);
        const int rn = (int)(r1 - r0);
        for (int i = tid; i < B * R; i += kThreads) sW[i] = 0.f;
        if (tid == 0) sPieceCounter = 0;
        __syncthreads();
        if (warp < kWideWarps) {
            // ---------- wide: spans ----------
            for (int it = warp; it < n_items; it += kWideWarps) {
                const Item t = sItems[it];
                uint32_t lo = locate(p.hdr, t.c0, t.c1, (uint32_t)r0, p.n_ads, lane);
                if (lo > t.c0) lo -= 1u;                // chunk that may contain r0
                const uint32_t hi = locate(p.hdr, lo, t.c1, (uint32_t)(r1 - 1), p.n_ads, lane);
                if (lane == 0) { sSpanLo[it] = lo; sSpanHi[it] = hi; }
            }
            wide_bar();
            // ---------- exclusive scan of piece counts (warp 0) ----------
            if (warp == 0) {
                uint32_t carry = 0;
                for (int base = 0; base < n_items; base += 32) {
                    const int it = base + lane;
                    const uint32_t np = (it < n_items) ? (sSpanHi[it] - sSpanLo[it] + kPiece - 1) / kPiece : 0u;
                    uint32_t incl = np;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t x = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += x;
                    }
                    if (it < n_items) sPieceOff[it] = carry + incl - np;
                    carry += __shfl_sync(FULL, incl, 31);
                }
                if (lane == 0) sPieceOff[n_items] = carry;
            }
            wide_bar();
            const uint32_t total = sPieceOff[n_items];
            // ---------- load-balanced decode + accumulate ----------
            while (true) {
                uint32_t unit = 0;
                if (lane == 0) unit = atomicAdd(&sPieceCounter, 1u);
                unit = __shfl_sync(FULL, unit, 0);
                if (unit >= total) break;
                // item = last it with sPieceOff[it] <= unit
                int lo_i = 0, hi_i = n_items - 1;
                while (lo_i < hi_i) {
                    const int mid = (lo_i + hi_i + 1) >> 1;
                    if (sPieceOff[mid] <= unit) lo_i = mid; else hi_i = mid - 1;
                }
                const Item t = sItems[lo_i];
                const uint32_t cb = sSpanLo[lo_i] + (unit - sPieceOff[lo_i]) * kPiece;
                const uint32_t ce = min(cb + (uint32_t)kPiece, sSpanHi[lo_i]);
                const uint32_t kwb = __ldg(&p.key_word_off[t.key]);
                float* wrow = sW + (size_t)t.b * R;
                for (uint32_t c = cb; c < ce; c += kDecodeU) {
                    uint32_t ids[kDecodeU];
                    bool ok[kDecodeU];
#pragma unroll
                    for (int q = 0; q < kDecodeU; ++q) {
                        ok[q] = false;
                        ids[q] = 0;
                        if (c + q < ce) ok[q] = decode_chunk(p.hdr, p.payload, kwb, c + q, lane, ids[q]);
                    }
#pragma unroll
                    for (int q = 0; q < kDecodeU; ++q) {
                        if (ok[q] && ids[q] >= (uint32_t)r0 && ids[q] < (uint32_t)r1)
                            smem_add(&wrow[ids[q] - (uint32_t)r0], t.w);
                    }
                }
            }
            EBR_STAMP(2);
        } else {
            // ---------- deep: stream rows [r0, r1) ----------
            const int dw = warp - kWideWarps;
            const char* Abase = reinterpret_cast<const char*>(p.A);
            const int64_t row_bytes = (int64_t)p.d_pad * sizeof(T);
            const int64_t step = (int64_t)kDeepWarps * rpw * kUnroll;
            for (int64_t base = r0 + (int64_t)dw * rpw * kUnroll; base < r1; base += step) {
                uint4 av[kUnroll][VPL];
#pragma unroll
                for (int q = 0; q < kUnroll; ++q) {
                    const int64_t row = base + q * rpw + sub;
#pragma unroll
                    for (int v = 0; v < VPL; ++v) {
                        if (row < r1)
                            av[q][v] = ldg_stream(Abase + row * row_bytes + (int64_t)(li + v * lpr) * 16);
                        else
                            av[q][v] = make_uint4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int q = 0; q < kUnroll; ++q) {
                    float acc[NB];
#pragma unroll
                    for (int b = 0; b < NB; ++b) acc[b] = 0.f;
#pragma unroll
                    for (int v = 0; v < VPL; ++v) {
                        float a[E];
                        V::unpack(av[q][v], a);
#pragma unroll
                        for (int b = 0; b < NB; ++b)
#pragma unroll
                            for (int e = 0; e < E; ++e) acc[b] = fmaf(a[e], u[b][v][e], acc[b]);
                    }
#pragma unroll
                    for (int b = 0; b < NB; ++b)
                        for (int o = lpr >> 1; o > 0; o >>= 1) acc[b] += __shfl_xor_sync(FULL, acc[b], o);
                    const int64_t row = base + q * rpw + sub;
                    if (li == 0 && row < r1) {
#pragma unroll
                        for (int b = 0; b < NB; ++b)
                            if (b < B) sD[(size_t)b * R + (row - r0)] = acc[b];
                    }
                }
            }
            EBR_STAMP(3);
        }
        __syncthreads();
        // ---------- A5 fuse + histogram ----------
        for (int i = tid; i < B * R; i += kThreads) {
            const int b = i / R, r = i - b * R;
            if (r < rn) {
                float s = sD[i] + sW[i];
                if (s == 0.f) s = 0.f;                  // -0 -> +0 (R14)
                __stcg(&p.scores[(size_t)b * p.n_pad + r0 + r], s);
                atomicAdd(&sHist[b * kHistBins + (ord_of(s) >> (32 - kHistBits))], 1u);
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < B * kHistBins; i += kThreads) {
        const uint32_t c = sHist[i];
        if (c) atomicAdd(&p.ghist[i], c);
    }
    EBR_STAMP(4);

    cg::this_grid().sync();
    EBR_STAMP(5);

    // ---- phase 3: threshold bin per user (warp b handles user b) ----
    if (warp < B) {
        const uint32_t* h = p.ghist + (size_t)warp * kHistBins;
        constexpr int PER = kHistBins / 32;
        uint32_t local = 0;
        for (int j = 0; j < PER; ++j) local += __ldcg(&h[kHistBins - 1 - (lane * PER + j)]);
        uint32_t incl = local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += x;
        }
        uint32_t c = incl - local;
        int found = -1;
        uint32_t above = 0;
        const uint32_t K = (uint32_t)p.K;
        if (c < K && c + local >= K) {
            for (int j = 0; j < PER; ++j) {
                const int bin = kHistBins - 1 - (lane * PER + j);
                const uint32_t cnt = __ldcg(&h[bin]);
                if (found < 0 && c < K && c + cnt >= K) { found = bin; above = c; }
                c += cnt;
            }
        }
        const unsigned m = __ballot_sync(FULL, found >= 0);
        const int src = m ? __ffs(m) - 1 : 0;
        const int fb = __shfl_sync(FULL, found, src);
        const uint32_t ab = __shfl_sync(FULL, above, src);
        if (lane == 0) {
            sBinStar[warp] = m ? (uint32_t)fb : 0u;  // fewer than K ads: everything is a candidate
            sAbove[warp] = m ? ab : 0u;
        }
    }
    __syncthreads();

    // ---- phase 4: compaction of candidates ----
    for (int range = blockIdx.x; range < p.n_ranges; range += gridDim.x) {
        const int64_t r0 = (int64_t)range * R;
        const int64_t r1 = ((r0 + R < p.n_ads) ? r0 + R : p.n_ads);
        const int rn = (int)(r1 - r0);
        for (int i = tid; i < B * R; i += kThreads) {
            const int b = i / R, r = i - b * R;
            if (r < rn) {
                const float s = __ldcg(&p.scores[(size_t)b * p.n_pad + r0 + r]);
                if ((ord_of(s) >> (32 - kHistBits)) >= sBinStar[b]) {
                    const uint32_t pos = atomicAdd(&p.cand_count[b], 1u);
                    p.cand[(size_t)b * p.n_pad + pos] = kappa_of(s, p.ad_begin + (uint32_t)(r0 + r));
                }
            }
        }
    }

    EBR_STAMP(6);
    cg::this_grid().sync();
    EBR_STAMP(7);

    // ---- phase 5: exact selection, one CTA per user ----
    for (int b = blockIdx.x; b < B; b += gridDim.x) {
        uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);
        const int64_t n = (int64_t)__ldcg(&p.cand_count[b]);
        const uint64_t* cb = p.cand + (size_t)b * p.n_pad;
        const int nsel = cta_select_topk([cb](int64_t i) { return __ldcg(&cb[i]); }, n, p.K, sbuf,
                                         reinterpret_cast<uint32_t*>(sbuf + pow2ceil_i(p.K)), sScalar);
        cta_write_topk(sbuf, nsel, p.K, p.out_ids ? p.out_ids + (size_t)b * p.K : nullptr,
                       p.out_scores ? p.out_scores + (size_t)b * p.K : nullptr,
                       p.out_keys ? p.out_keys + (size_t)b * p.K : nullptr);
        __syncthreads();
        EBR_STAMP(8);
    }
}

// --------------------------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------------------------
typedef void (*kern_t)(const SmallParams);

template <typename T>
kern_t pick_kernel(int nb, int vpl) {
#define EBR_K(NB, VPL) if (nb == NB && vpl == VPL) return small_kernel<T, NB, VPL>;
    EBR_K(1, 1) EBR_K(2, 1) EBR_K(4, 1) EBR_K(8, 1)
    EBR_K(1, 2) EBR_K(2, 2) EBR_K(4, 2) EBR_K(8, 2)
    EBR_K(1, 4) EBR_K(2, 4) EBR_K(4, 4) EBR_K(8, 4)
#undef EBR_K
    return nullptr;
}

struct SmallLayout {
    size_t off_err, off_hist, off_count, off_scores, off_cand, total;
};

SmallLayout small_layout(const ebr_index* idx, int B) {
    SmallLayout L;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t o = 0;
    L.off_err = o;    o = al(o + 16 + 16 * 8);   // error word + 16 phase stamps
    L.off_hist = o;   o = al(o + (size_t)B * kHistBins * 4);
    L.off_count = o;  o = al(o + (size_t)B * 4);
    L.off_scores = o; o = al(o + (size_t)B * idx->n_pad * 4);
    L.off_cand = o;   o = al(o + (size_t)B * idx->n_pad * 8);
    L.total = o;
    return L;
}

}  // namespace

size_t small_workspace_bytes(const ebr_index* idx, int32_t slots, int32_t k) {
    (void)slots; (void)k;
    return small_layout(idx, kSmallMaxB).total;
}

// Runs users [0, B) (B <= kSmallMaxB) of one launch.
ebr_status run_small(const QueryArgs& q, int b0, int B) {
    const ebr_index* idx = q.idx;
    SmallLayout L = small_layout(idx, B);
    char* ws = static_cast<char*>(q.workspace);
    const int esz = idx->dtype == EBR_BF16 ? 2 : 4;
    const int row_bytes = idx->d_pad * esz;
    int lpr, vpl;
    if (row_bytes <= 512) { lpr = row_bytes / 16; vpl = 1; }
    else { lpr = 32; vpl = row_bytes / 512; }
    int nb = 1;
    while (nb < B) nb <<= 1;
    kern_t k = idx->dtype == EBR_BF16 ? pick_kernel<__nv_bfloat16>(nb, vpl) : pick_kernel<float>(nb, vpl);
    if (!k) return set_error(EBR_EUNSUPPORTED, "embedding row of %d bytes is not supported", row_bytes);

    const int items_cap = B * idx->n_fields * q.slots;
    const size_t item_bytes = (size_t)items_cap * (sizeof(Item) + 12) + 16;
    const size_t hist_bytes = (size_t)B * kHistBins * 4;
    const size_t sel_bytes = (size_t)pow2ceil_i(q.k) * 8 + 256 * 4 + 64;
    const size_t smem_cap = 220 * 1024;
    if (item_bytes + hist_bytes + 8 * 1024 > smem_cap)
        return set_error(EBR_EUNSUPPORTED, "too many user slots for the latency path (%d)", items_cap);
    // range size: one range per CTA if it fits, else as large as shared memory allows
    const int sms = idx->sm_count;
    int64_t R = (idx->n_ads + sms - 1) / sms;
    const int64_t R_fit = (int64_t)((smem_cap - item_bytes - hist_bytes) / (8 * (size_t)B));
    R = std::min<int64_t>(R, R_fit);
    R = std::max<int64_t>(32, R & ~(int64_t)31);
    const size_t p1_bytes = (size_t)8 * B * R + hist_bytes + item_bytes;
    const size_t smem = std::max(p1_bytes, sel_bytes);
    if (smem > 227 * 1024) return set_error(EBR_EUNSUPPORTED, "k=%d needs too much shared memory", q.k);

    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(small)");
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem);
    if (e != cudaSuccess || occ < 1) return cuda_check(e == cudaSuccess ? cudaErrorInvalidConfiguration : e, "occupancy(small)");

    SmallParams p;
    p.A = idx->A; p.d = idx->d; p.d_pad = idx->d_pad; p.lpr = lpr;
    p.n_ads = idx->n_ads; p.n_pad = idx->n_pad; p.ad_begin = (uint32_t)idx->ad_begin;
    p.key_chunk_off = idx->key_chunk_off; p.key_word_off = idx->key_word_off;
    p.hdr = idx->chunk_hdr; p.payload = idx->payload; p.cross_w = idx->cross_w;
    p.field_card = idx->field_card; p.field_base = idx->field_base; p.n_fields = idx->n_fields;
    p.U = static_cast<const char*>(q.user_emb) + (size_t)b0 * idx->d * esz;
    p.B = B; p.slots = q.slots; p.K = q.k;
    p.user_feat = q.user_feat + (size_t)b0 * idx->n_fields * q.slots;
    p.user_x = q.user_x + (size_t)b0 * idx->n_fields * q.slots;
    p.err = reinterpret_cast<uint32_t*>(ws + L.off_err);
    static const bool timers_on = getenv("EBR_PHASE_TIMERS") && getenv("EBR_PHASE_TIMERS")[0] == '1';
    p.timers = timers_on ? reinterpret_cast<unsigned long long*>(ws + L.off_err + 16) : nullptr;
    p.ghist = reinterpret_cast<uint32_t*>(ws + L.off_hist);
    p.cand_count = reinterpret_cast<uint32_t*>(ws + L.off_count);
    p.scores = reinterpret_cast<float*>(ws + L.off_scores);
    p.cand = reinterpret_cast<uint64_t*>(ws + L.off_cand);
    p.out_ids = q.out_ids ? q.out_ids + (size_t)b0 * q.k : nullptr;
    p.out_scores = q.out_scores ? q.out_scores + (size_t)b0 * q.k : nullptr;
    p.out_keys = q.out_keys ? q.out_keys + (size_t)b0 * q.k : nullptr;
    p.R = (int32_t)R;
    p.n_ranges = (int32_t)((idx->n_ads + R - 1) / R);
    p.items_cap = items_cap;

    // zero the per-call counters (histograms + candidate counts are contiguous)
    // the first launch of a call also clears the device error word (flags of the last call)
    const size_t z0 = (b0 == 0) ? L.off_err : L.off_hist;
    e = cudaMemsetAsync(ws + z0, 0, L.off_scores - z0, q.stream);
    if (e != cudaSuccess) return cuda_check(e, "memset(small)");
    const int grid = std::max(1, std::min<int>(p.n_ranges, occ * sms));
    void* args[] = {&p};
    e = cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kThreads), args, smem, q.stream);
    if (e != cudaSuccess) return cuda_check(e, "launch(small)");
    return EBR_OK;
}

}  // namespace ebr
