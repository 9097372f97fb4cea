// ebr_batch.cu -- the batched path (bf16 embeddings, user batch >= 16): every (user, ad) score of
// a pass of up to 512 users is produced tile by tile inside ONE persistent tcgen05 kernel and
// filtered against a per-user threshold on chip; no per-(user, ad) buffer ever reaches HBM.
//
//   s(u,a) = <h~_u, h~_a>                      deep, Eq. 1 / Eq. 8
//          + sum_{hot keys i} w~_ui L_ai       wide, the longest posting lists as one-hot columns
//          + sum_{cold keys i} w~_ui L_ai      wide, the compressed inverted lists (Alg. 2)
//
// A pass of P users is split into G = ceil(P/128) groups; the G CTAs of a thread-block cluster
// (one per group, one CTA per SM) walk the same ad tiles in lockstep and receive each 128-ad tile
// of A by ONE multicast TMA load, so A is read from HBM once per pass (not once per group).  Per
// CTA and tile (128 ads x 128 users, fp32 accumulator in TMEM, 4 stages):
//   * wide warps (8): expand the ads' hot-key bit masks into an fp16 one-hot K block (A side of
//     the hot MMA), scatter the cold keys' w~ into a shared-memory int32 fixed-point tile
//     [ads x users] (Alg. 2 l.358's AtomicAdd, exact and order-free), convert it once to fp32 and
//     store it into the TMEM accumulator stage with tcgen05.st;
//   * one thread issues tcgen05.mma: deep (bf16 A x bf16 U) and hot (fp16 one-hot x fp16 w~
//     pieces) accumulate ON TOP of the stored cold wide term: D = cold + deep + hot;
//   * epilogue warps (8): tcgen05.ld, A5 kappa, A6 sample store / threshold filter.
// The cold postings reach the tile as an "entry stream": the batch's distinct cold keys are
// decoded ONCE per pass (not once per user: the SpMM view of L w~) by range kernels into
// per-tile lists of (ad row, the key's user-pair list), read by every CTA of the cluster.
//
// Launches per pass (all on the caller's stream, no host synchronisation -- graph-capturable):
//   plan_a / plan_b / plan_c   A1: slots -> keys, w~ = fl32(w x), hot pieces, cold key
//                              union (hash) with user pairs, fixed-point scales, user tiles
//   span / entry_count / range_scan / entry_write    A2: the entry stream
//   score<0>  on every 16th tile: scores of the sample (A3-A5)
//   theta     A6a: theta_u = the r-th largest sampled key (r < K)
//   score<1>  on every tile: keys >= theta_u appended to per-user candidate lists (A3-A6b)
//   final     A6c: exact top-K of the candidates; a user with < K candidates is flagged
//   theta / score<1> / final again, gated on device flags: the flagged users with r = K, which
//             guarantees >= K candidates (the sample is a subset of the inventory) -- exact.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "ebr_tc.cuh"

namespace ebr {

namespace batch {

constexpr int kGroup = 128;          // users per CTA (UMMA N)
constexpr int kMaxCluster = 4;       // CTAs (user groups) per cluster
constexpr int kTileM = 128;          // ads per tile (UMMA M)
constexpr int kBlockK = 64;          // 16-bit elements per 128-byte swizzle row
constexpr int kBlockBytes = kTileM * 128;   // one ring stage: 128 rows x 128 B
constexpr int kSampleStride = 16;    // every 16th tile is sampled for theta
constexpr int kAccStages = 4;        // TMEM: 4 x 128 columns
constexpr int kAccPitch = kGroup + 4;   // int32 words per fixed-point row (16-B row reads conflict-free)
constexpr int kWideWarp0 = 4, kWideWarps = 8, kWideThreads = 32 * kWideWarps;
constexpr int kEpiWarp0 = kWideWarp0 + kWideWarps, kEpiWarps = 8;
constexpr int kGemmThreads = 32 * (kEpiWarp0 + kEpiWarps);   // 640: TMA, MMA, TMEM alloc, spare, 8 wide, 8 epilogue
constexpr int kMaxHotBlocks = 2;     // hot K blocks of 64 keys (the index keeps up to 128 hot keys)
constexpr int kPairWBits = 23;       // cold pair = pass user (9 bits) << 23 | w~ 2^S (23-bit two's complement)
constexpr int kPairWMax = 22;        // |w~ 2^S| < 2^22
constexpr int kEntryPsBits = 15;     // entry = row << 24 | (pair count - 1) << 15 | first pair
constexpr int kMaxPassPairs = 1 << kEntryPsBits;
constexpr int kRangeMaxTiles = 256;  // entry-stream range: <= 32768 ads (per-ad u32 counters in smem)
constexpr int kPlanThreads = 1024;
constexpr uint32_t kFlagShort = 1u, kFlagOverflow = 2u, kFlagRaise = 4u;   // uflags; overflow users carry their dense slot << 8
constexpr uint32_t kFlagAny = kFlagShort | kFlagOverflow | kFlagRaise;
constexpr int kMaxFallback = 2;      // overflowed users per pass recomputed exactly (dense scores)

// ------------------------------------------------------------------------------------------
// workspace
// ------------------------------------------------------------------------------------------
struct Ws {
    uint32_t* header;     // [0] n_union [1] n_pairs [2] any user short of K [3] entries total [4] overflowed users
    uint32_t* hkey;       // [TS] key + 1 (0 = empty)
    uint32_t* hcnt;       // [TS] user pairs of the key (left zero by plan_c)
    uint32_t* hslot;      // [TS] union slot of the key
    uint32_t* hpair;      // [TS] first pair of the key
    int32_t* item_t;      // [P*F*S] hash position of a cold slot, -1 otherwise
    float* item_w;        // [P*F*S] w~ of the slot
    float* hotw;          // [P_pad][128] sum of w~ per (user, hot key) (left zero by plan_c)
    float* bound;         // [P] sum |w~| of the cold slots (left zero by plan_b)
    uint32_t* emax;       // [P] max |w~| bits (left zero by plan_b)
    int32_t* ushift;      // [P] fixed-point scale S_u
    float* uscale;        // [P] 2^-S_u
    uint32_t* ukey;       // [NU] union slot -> key
    uint32_t* uc0;        // [NU] first chunk of the key
    uint32_t* uc1;        // [NU] end chunk
    uint32_t* ukwb;       // [NU] payload word base
    uint32_t* uentry;     // [NU] (count - 1) << 15 | first pair
    uint32_t* pairs;      // [NU]
    uint16_t* U;          // [P_pad][u_cols] deep bf16 | hot fp16 pieces
    uint32_t* span;       // [NU][n_ranges + 1] first chunk of the key with last id >= j R
    uint32_t* adcnt;      // [n_pad / 4] per-ad entry counts (u8)
    uint32_t* rtotal;     // [n_ranges]
    uint32_t* rbase;      // [n_ranges + 1]
    uint32_t* tile_off;   // [n_tiles + 1]
    uint32_t* entries;    // [n_pad * F]
    float* samp;          // [P][n_samp]
    uint64_t* theta;      // [P]
    uint32_t* cand_count; // [P]
    uint64_t* cand;       // [P][cap]
    uint32_t* uflags;     // [P] kFlagShort | kFlagOverflow
    float* dense;         // [kMaxFallback][n_pad] every score of an overflowed user
};

struct Layout {
    size_t total;
    size_t off[32];
    int64_t TS, NU, P, n_samp, cap, n_ranges, range_ads, n_tiles, u_cols;
};

static int64_t pow2ceil64(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// users per pass: <= kGroup * kMaxCluster, and the pass's pairs must fit the entry encoding
int pass_users(const ebr_index* idx, int32_t slots) {
    const int64_t fs = (int64_t)idx->n_fields * slots;
    int64_t p = std::min<int64_t>(kGroup * kMaxCluster, kMaxPassPairs / std::max<int64_t>(fs, 1));
    return (int)(p / 32 * 32);
}

static int64_t cand_cap(int k) {
    return std::max<int64_t>(65536, 4 * ((int64_t)k + (int64_t)(100.0 * std::sqrt((double)k)) + 256));
}

static Layout layout(const ebr_index* idx, int32_t slots, int32_t k) {
    Layout L;
    const int P = pass_users(idx, slots);
    L.P = P;
    L.NU = (int64_t)P * idx->n_fields * slots;
    L.TS = pow2ceil64(2 * L.NU);
    L.n_tiles = idx->n_pad / kTileM;
    L.n_samp = ((L.n_tiles + kSampleStride - 1) / kSampleStride) * kTileM;
    L.cap = cand_cap(k);
    const int64_t tpr = std::min<int64_t>(kRangeMaxTiles, std::max<int64_t>(1, (L.n_tiles + 2 * idx->sm_count - 1) /
                                                                                 (2 * idx->sm_count)));
    L.range_ads = tpr * kTileM;
    L.n_ranges = (L.n_tiles + tpr - 1) / tpr;
    L.u_cols = idx->d_pad + (int64_t)kMaxHotBlocks * 64 * 2;
    const int64_t Ppad = (int64_t)((P + kGroup - 1) / kGroup) * kGroup;
    const size_t sizes[] = {
        64,                                         // 0 header
        (size_t)L.TS * 4, (size_t)L.TS * 4, (size_t)L.TS * 4, (size_t)L.TS * 4,   // 1-4 hash
        (size_t)L.NU * 4, (size_t)L.NU * 4,         // 5-6 items
        (size_t)Ppad * 128 * 4,                     // 7 hotw
        (size_t)P * 4, (size_t)P * 4, (size_t)P * 4, (size_t)P * 4,   // 8-11 per user
        (size_t)L.NU * 4, (size_t)L.NU * 4, (size_t)L.NU * 4, (size_t)L.NU * 4, (size_t)L.NU * 4,   // 12-16 union
        (size_t)L.NU * 4,                           // 17 pairs
        (size_t)Ppad * L.u_cols * 2,                // 18 U
        (size_t)L.NU * (L.n_ranges + 1) * 4,        // 19 span
        (size_t)idx->n_pad,                         // 20 adcnt
        (size_t)L.n_ranges * 4, (size_t)(L.n_ranges + 1) * 4,   // 21-22
        (size_t)(L.n_tiles + 1) * 4,                // 23 tile_off
        (size_t)idx->n_pad * idx->n_fields * 4,     // 24 entries
        (size_t)P * L.n_samp * 4,                   // 25 samp
        (size_t)P * 8, (size_t)P * 4,               // 26-27 theta, count
        (size_t)P * L.cap * 8,                      // 28 cand
        (size_t)P * 4,                              // 29 flags
        (size_t)kMaxFallback * idx->n_pad * 4,      // 30 dense
    };
    size_t o = 0;
    for (int i = 0; i < 31; ++i) {
        L.off[i] = o;
        o = (o + sizes[i] + 1023) & ~(size_t)1023;
    }
    L.total = o;
    return L;
}

static Ws carve(char* b, const Layout& L) {
    Ws w;
    auto at = [&](int i) { return b + L.off[i]; };
    w.header = (uint32_t*)at(0);
    w.hkey = (uint32_t*)at(1); w.hcnt = (uint32_t*)at(2); w.hslot = (uint32_t*)at(3); w.hpair = (uint32_t*)at(4);
    w.item_t = (int32_t*)at(5); w.item_w = (float*)at(6);
    w.hotw = (float*)at(7);
    w.bound = (float*)at(8); w.emax = (uint32_t*)at(9); w.ushift = (int32_t*)at(10); w.uscale = (float*)at(11);
    w.ukey = (uint32_t*)at(12); w.uc0 = (uint32_t*)at(13); w.uc1 = (uint32_t*)at(14); w.ukwb = (uint32_t*)at(15);
    w.uentry = (uint32_t*)at(16); w.pairs = (uint32_t*)at(17);
    w.U = (uint16_t*)at(18);
    w.span = (uint32_t*)at(19);
    w.adcnt = (uint32_t*)at(20);
    w.rtotal = (uint32_t*)at(21); w.rbase = (uint32_t*)at(22);
    w.tile_off = (uint32_t*)at(23);
    w.entries = (uint32_t*)at(24);
    w.samp = (float*)at(25);
    w.theta = (uint64_t*)at(26); w.cand_count = (uint32_t*)at(27);
    w.cand = (uint64_t*)at(28);
    w.uflags = (uint32_t*)at(29);
    w.dense = (float*)at(30);
    return w;
}

// ------------------------------------------------------------------------------------------
// A1 plan
// ------------------------------------------------------------------------------------------
struct PlanArgs {
    const int32_t* user_feat;   // [P][F][S] of this pass
    const float* user_x;
    const uint16_t* user_emb;   // [P][d]
    const uint32_t* key_chunk_off;
    const uint32_t* key_word_off;
    const float* cross_w;
    const int32_t* field_card;
    const int32_t* field_base;
    const int32_t* hot_slot;
    int F, S, P, d, d_pad, n_hot_used, pieces, u_cols;
    int64_t TS;
    uint32_t* err;
};

__device__ __forceinline__ uint32_t hash_key(uint32_t k) {
    k ^= k >> 16; k *= 0x7feb352dU; k ^= k >> 15; k *= 0x846ca68bU; k ^= k >> 16;
    return k;
}

// plan_a: every slot of the pass.  Hot slot -> its w~ is summed into hotw[u][h]; cold slot with
// postings -> the key is inserted into the pass's hash table (the batch's key union) and the
// user's fixed-point bounds are updated.  w~ = fl32(w x): one rounding, never an FMA (R10).
__global__ void __launch_bounds__(256) plan_a_kernel(PlanArgs a, Ws ws) {
    const int n = a.P * a.F * a.S;
    const uint32_t mask = (uint32_t)a.TS - 1u;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        ws.item_t[i] = -1;
        const int f = (i / a.S) % a.F;
        const int u = i / (a.F * a.S);
        const int32_t v = a.user_feat[i];
        if (v < -1 || v >= a.field_card[f]) { atomicOr(a.err, 1u); continue; }   // outside [-1, V_f)
        if (v < 0) continue;
        const uint32_t key = (uint32_t)(a.field_base[f] + v);
        const float w = __fmul_rn(__ldg(&a.cross_w[key]), a.user_x[i]);
        const int h = a.n_hot_used ? __ldg(&a.hot_slot[key]) : -1;
        if (h >= 0 && h < a.n_hot_used && fabsf(w) < 16384.f) {   // fp16 pieces need |w~| < 2^14
            atomicAdd(&ws.hotw[(size_t)u * 128 + h], w);
            continue;
        }
        if (__ldg(&a.key_chunk_off[key + 1]) <= __ldg(&a.key_chunk_off[key])) continue;   // empty list
        atomicAdd(&ws.bound[u], fabsf(w));
        atomicMax(&ws.emax[u], __float_as_uint(fabsf(w)));
        uint32_t t = hash_key(key) & mask;
        while (true) {
            const uint32_t prev = atomicCAS(&ws.hkey[t], 0u, key + 1u);
            if (prev == 0u || prev == key + 1u) break;
            t = (t + 1u) & mask;
        }
        atomicAdd(&ws.hcnt[t], 1u);
        ws.item_t[i] = (int32_t)t;
        ws.item_w[i] = w;
    }
}

// plan_b (one CTA): compacts the hash table into union slots (scan), assigns each key its pair
// range, resets the table for the next pass, and derives every user's fixed-point scale
//   S_u = min(22 - e_max, 30 - e_sum),  max|w~| < 2^e_max,  sum|w~| < 2^e_sum
// so each w~ 2^S fits the 23-bit pair field and every partial sum fits int32 (R23).
__global__ void __launch_bounds__(kPlanThreads) plan_b_kernel(PlanArgs a, Ws ws) {
    __shared__ uint32_t sScan[40];
    __shared__ uint32_t sBase[2];
    const int tid = threadIdx.x;
    if (tid == 0) { sBase[0] = 0; sBase[1] = 0; }
    __syncthreads();
    for (int64_t t0 = 0; t0 < a.TS; t0 += kPlanThreads) {
        const int64_t t = t0 + tid;
        uint32_t key1 = 0, cnt = 0;
        if (t < a.TS) { key1 = ws.hkey[t]; cnt = key1 ? ws.hcnt[t] : 0u; }
        uint32_t tot_s, tot_p;
        const uint32_t ps = block_exclusive_scan(key1 ? 1u : 0u, sScan, &tot_s);
        const uint32_t pp = block_exclusive_scan(cnt, sScan, &tot_p);
        if (key1) {
            const uint32_t s = sBase[0] + ps, p0 = sBase[1] + pp;
            const uint32_t key = key1 - 1u;
            ws.hslot[t] = s;
            ws.hpair[t] = p0;
            ws.ukey[s] = key;
            ws.uc0[s] = a.key_chunk_off[key];
            ws.uc1[s] = a.key_chunk_off[key + 1];
            ws.ukwb[s] = a.key_word_off[key];
            ws.uentry[s] = ((cnt - 1u) << kEntryPsBits) | p0;
            ws.hkey[t] = 0u;
        }
        __syncthreads();
        if (tid == 0) { sBase[0] += tot_s; sBase[1] += tot_p; }
        __syncthreads();
    }
    if (tid == 0) { ws.header[0] = sBase[0]; ws.header[1] = sBase[1]; ws.header[2] = 0; ws.header[4] = 0; }
    for (int u = tid; u < a.P; u += kPlanThreads) {
        const float b = ws.bound[u], m = __uint_as_float(ws.emax[u]);
        int S = 0;
        if (b > 0.f) {
            int es = 0, em = 0;
            frexpf(b * 1.0001f, &es);   // b < 2^es (the margin covers the rounding of the float sum)
            frexpf(m, &em);             // m < 2^em
            S = min(kPairWMax - em, 30 - es);
        }
        ws.ushift[u] = S;
        ws.uscale[u] = ldexpf(1.f, -S);
        ws.bound[u] = 0.f;
        ws.emax[u] = 0u;
    }
}

// plan_c: the user pairs of every cold key (its own slot order is irrelevant: the integer sums are
// order-free), and the pass's user tile: deep part bf16, hot part the exact fp16 pieces of w~.
__global__ void __launch_bounds__(256) plan_c_kernel(PlanArgs a, Ws ws) {
    const int n = a.P * a.F * a.S;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    for (int i = gt; i < n; i += gs) {
        const int32_t t = ws.item_t[i];
        if (t < 0) continue;
        const int u = i / (a.F * a.S);
        const uint32_t pos = ws.hpair[t] + atomicSub(&ws.hcnt[t], 1u) - 1u;
        const int S = ws.ushift[u];
        const int32_t wf = (int32_t)__float2int_rn(ldexpf(ws.item_w[i], S));   // |wf| < 2^22
        ws.pairs[pos] = ((uint32_t)u << kPairWBits) | ((uint32_t)wf & ((1u << kPairWBits) - 1u));
    }
    const int Ppad = (a.P + kGroup - 1) / kGroup * kGroup;
    // deep part of U (zero padded rows and columns)
    for (int i = gt; i < Ppad * a.d_pad; i += gs) {
        const int u = i / a.d_pad, j = i - u * a.d_pad;
        ws.U[(size_t)u * a.u_cols + j] = (u < a.P && j < a.d) ? a.user_emb[(size_t)u * a.d + j] : (uint16_t)0;
    }
    // hot part: hot key h of block hb = h / 64 -> columns d_pad + (hb * pieces + p) * 64 + h % 64
    for (int i = gt; i < Ppad * a.n_hot_used; i += gs) {
        const int u = i / a.n_hot_used, h = i - u * a.n_hot_used;
        float w = ws.hotw[(size_t)u * 128 + h];
        ws.hotw[(size_t)u * 128 + h] = 0.f;
        uint16_t* dst = ws.U + (size_t)u * a.u_cols + a.d_pad + (size_t)(h >> 6) * a.pieces * 64 + (h & 63);
        for (int p = 0; p < a.pieces; ++p) {
            const __half hv = __float2half_rn(w);
            dst[p * 64] = __half_as_ushort(hv);
            w -= __half2float(hv);       // exact: the residual of a round-to-nearest
        }
    }
}

// ------------------------------------------------------------------------------------------
// A2 the entry stream: the union's cold postings, decoded once per pass, as per-tile lists
// ------------------------------------------------------------------------------------------
struct EntryArgs {
    const uint2* hdr;
    const uint32_t* chunk_last;
    const uint32_t* payload;
    int64_t n_ads, n_pad, range_ads;
    int n_ranges, n_tiles;
    int64_t NU;
};

// span: one warp per union key; span[s][j] = first chunk whose last id >= j R (j = 0..n_ranges)
__global__ void __launch_bounds__(256) span_kernel(EntryArgs e, Ws ws) {
    const int lane = threadIdx.x & 31;
    const uint32_t s = blockIdx.x * 8 + (threadIdx.x >> 5);
    const uint32_t nu = __ldcg(&ws.header[0]);
    if (s >= nu) return;
    const uint32_t c0 = ws.uc0[s], c1 = ws.uc1[s];
    uint32_t* sp = ws.span + (size_t)s * (e.n_ranges + 1);
    const uint32_t R = (uint32_t)e.range_ads;
    int last_r = -1;
    for (uint32_t cb = c0; cb < c1; cb += 32) {
        const uint32_t c = cb + lane;
        int r = -1, rp = -1;
        if (c < c1) {
            r = (int)(__ldg(&e.chunk_last[c]) / R);
            rp = (c == c0) ? -1 : (int)(__ldg(&e.chunk_last[c - 1]) / R);
            for (int j = rp + 1; j <= r; ++j) sp[j] = c;
        }
        const int m = __reduce_max_sync(FULL, r);
        last_r = max(last_r, m);
    }
    for (int j = last_r + 1 + lane; j <= e.n_ranges; j += 32) sp[j] = c1;
}

// Calls f(local ad) for every posting of union key s inside range j, one warp.
template <typename Fn>
__device__ __forceinline__ void range_postings(const EntryArgs& e, const Ws& ws, uint32_t s, int j, int lane, Fn f) {
    const uint32_t* sp = ws.span + (size_t)s * (e.n_ranges + 1);
    const uint32_t lo = sp[j], c1 = ws.uc1[s];
    const uint32_t hi = min(sp[j + 1] + 1u, c1);   // the chunk straddling the range end
    const uint32_t kwb = ws.ukwb[s];
    const uint32_t a0 = (uint32_t)((int64_t)j * e.range_ads), a1 = a0 + (uint32_t)e.range_ads;
    for (uint32_t c = lo; c < hi; ++c) {
        uint32_t id;
        const bool ok = decode_chunk(e.hdr, e.payload, kwb, c, lane, id);
        if (ok && id >= a0 && id < a1) f(id - a0);
    }
}

// entry_count: CTA = range; counts the postings of every ad (u8 per ad) and the range total
__global__ void __launch_bounds__(512) entry_count_kernel(EntryArgs e, Ws ws) {
    extern __shared__ uint32_t cnt[];      // [range_ads]
    __shared__ uint32_t sRed[16];
    const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R = (int)e.range_ads;
    for (int i = tid; i < R; i += 512) cnt[i] = 0;
    __syncthreads();
    const uint32_t nu = __ldcg(&ws.header[0]);
    for (uint32_t s = warp; s < nu; s += 16)
        range_postings(e, ws, s, j, lane, [&](uint32_t a) { atomicAdd(&cnt[a], 1u); });
    __syncthreads();
    uint32_t tot = 0;
    const int64_t a0 = (int64_t)j * R;
    for (int i = tid; i < R / 4; i += 512) {
        const uint32_t c0 = cnt[4 * i], c1 = cnt[4 * i + 1], c2 = cnt[4 * i + 2], c3 = cnt[4 * i + 3];
        tot += c0 + c1 + c2 + c3;
        if (a0 + 4 * i < e.n_pad) ws.adcnt[a0 / 4 + i] = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);   // <= F <= 255 each
    }
    tot = __reduce_add_sync(FULL, tot);
    if (lane == 0) sRed[warp] = tot;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < 16; ++w) t += sRed[w];
        ws.rtotal[j] = t;
    }
}

__global__ void __launch_bounds__(1024) range_scan_kernel(EntryArgs e, Ws ws) {
    __shared__ uint32_t sScan[40];
    __shared__ uint32_t sBase;
    if (threadIdx.x == 0) sBase = 0;
    __syncthreads();
    for (int j0 = 0; j0 < e.n_ranges; j0 += 1024) {
        const int j = j0 + threadIdx.x;
        const uint32_t v = j < e.n_ranges ? ws.rtotal[j] : 0u;
        uint32_t tot;
        const uint32_t pre = block_exclusive_scan(v, sScan, &tot);
        if (j < e.n_ranges) ws.rbase[j] = sBase + pre;
        __syncthreads();
        if (threadIdx.x == 0) sBase += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ws.rbase[e.n_ranges] = sBase;
        ws.tile_off[e.n_tiles] = sBase;
        ws.header[3] = sBase;
    }
}

// entry_write: CTA = range; per-ad offsets (scan of the counts), the tile offsets, then every
// posting written as an entry row << 24 | uentry[s] at its ad's next slot
__global__ void __launch_bounds__(512) entry_write_kernel(EntryArgs e, Ws ws) {
    extern __shared__ uint32_t cur[];      // [range_ads] running position of each ad's entries
    __shared__ uint32_t sScan[40];
    const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R = (int)e.range_ads;
    const int64_t a0 = (int64_t)j * R;
    const uint32_t base = ws.rbase[j];
    const uint8_t* cnt8 = reinterpret_cast<const uint8_t*>(ws.adcnt);
    // thread tid owns the ads [tid*pp, tid*pp + pp) of the range
    const int pp = (R + 511) / 512;
    const int i0 = tid * pp;
    uint32_t local = 0;
    for (int q = 0; q < pp; ++q) {
        const int i = i0 + q;
        if (i < R && a0 + i < e.n_pad) local += cnt8[a0 + i];
    }
    uint32_t tot;
    uint32_t pre = block_exclusive_scan(local, sScan, &tot);
    for (int q = 0; q < pp; ++q) {
        const int i = i0 + q;
        if (i >= R) break;
        cur[i] = pre;
        if ((i & (kTileM - 1)) == 0 && a0 + i < e.n_pad) ws.tile_off[(a0 + i) / kTileM] = base + pre;
        if (a0 + i < e.n_pad) pre += cnt8[a0 + i];
    }
    __syncthreads();
    const uint32_t nu = __ldcg(&ws.header[0]);
    for (uint32_t s = warp; s < nu; s += 16) {
        const uint32_t ent = ws.uentry[s];
        range_postings(e, ws, s, j, lane, [&](uint32_t a) {
            const uint32_t pos = atomicAdd(&cur[a], 1u);
            ws.entries[base + pos] = ((a & (kTileM - 1)) << 24) | ent;
        });
    }
}

// ------------------------------------------------------------------------------------------
// A3-A6b: the fused tensor-core kernel
// ------------------------------------------------------------------------------------------
struct GemmParams {
    int64_t n_ads, n_pad;
    uint32_t ad_begin;
    int n_kb, n_hb, pieces, u_blocks;
    int P;                  // users in this pass
    int n_tiles, tile_stride;
    int n_samp;
    int stages;
    int64_t cap;
    int rerun;              // filter rerun: only flagged users; gated on header[2] | header[4]
    int dense;              // sample-mode variant: every score of the overflowed users (gated on header[4])
    const uint4* hot_mask;
    Ws ws;
    uint32_t* err;
};

__device__ __forceinline__ int32_t pair_w(uint32_t pr) {
    return (int32_t)(pr << (32 - kPairWBits)) >> (32 - kPairWBits);   // sign-extend the 23-bit field
}

template <int MODE>   // 0: sample (store s; dense: all scores of overflowed users), 1: filter (append keys >= theta)
__global__ void __launch_bounds__(kGemmThreads, 1)
score_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmU, const GemmParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // gated launches (uniform over the grid): nothing to redo
    if (MODE == 1 && p.rerun && (*(volatile uint32_t*)&p.ws.header[2] | *(volatile uint32_t*)&p.ws.header[4]) == 0u)
        return;
    if (MODE == 0 && p.dense && *(volatile uint32_t*)&p.ws.header[4] == 0u) return;
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = tc::cluster_ctarank();
    uint32_t csize;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    const uint32_t cid = tc::cluster_id_x(), ncl = tc::cluster_count_x();
    const uint16_t mc_mask = (uint16_t)((1u << csize) - 1u);
    const int g = (int)rank;                         // this CTA's user group
    const int nu = min(kGroup, p.P - g * kGroup);    // valid users
    const int nu_pad = (nu + 31) & ~31;
    const int nkt = p.n_kb + p.n_hb;

    unsigned char* sU = smem;                                               // [u_blocks][128 x 128 B]
    unsigned char* sRing = sU + (size_t)p.u_blocks * kBlockBytes;          // [stages][128 x 128 B]
    int32_t* acc = reinterpret_cast<int32_t*>(sRing + (size_t)p.stages * kBlockBytes);   // [128][kAccPitch]
    uint64_t* bars = reinterpret_cast<uint64_t*>(acc + kTileM * kAccPitch);
    uint64_t* full = bars;
    uint64_t* empty = full + p.stages;
    uint64_t* tfull = empty + p.stages;
    uint64_t* tempty = tfull + kAccStages;
    uint64_t* wready = tempty + kAccStages;
    uint64_t* ufull = wready + kAccStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ufull + 1);
    uint64_t* sTheta = reinterpret_cast<uint64_t*>(tmem_slot + 2);          // [kGroup]
    float* sThetaS = reinterpret_cast<float*>(sTheta + kGroup);             // [kGroup]
    float* sScale = sThetaS + kGroup;                                       // [kGroup]
    int* sDense = reinterpret_cast<int*>(sScale + kGroup);                  // [kGroup] dense slot or -1

    if (tid == 0) {
        for (int s = 0; s < p.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], csize); }
        for (int s = 0; s < kAccStages; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kEpiWarps);
            mbar_init(&wready[s], 1);
        }
        mbar_init(ufull, 1);
        fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc(tmem_slot, kAccStages * 128);
    for (int i = tid; i < kTileM * kAccPitch / 4; i += kGemmThreads)
        reinterpret_cast<int4*>(acc)[i] = make_int4(0, 0, 0, 0);
    for (int i = tid; i < kGroup; i += kGemmThreads) {
        const int u = g * kGroup + i;
        const bool ok = i < nu;
        sScale[i] = ok ? p.ws.uscale[u] : 0.f;
        const uint32_t fl = ok ? __ldcg(&p.ws.uflags[u]) : 0u;
        if (MODE == 0) sDense[i] = (p.dense && (fl & kFlagOverflow)) ? (int)(fl >> 8) : -1;
        if (MODE == 1) {
            bool take = ok;
            if (p.rerun) take = ok && (fl & kFlagAny);
            sTheta[i] = take ? __ldcg(&p.ws.theta[u]) : ~0ull;
            sThetaS[i] = take ? score_of(sTheta[i]) : __int_as_float(0x7F800000);
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::cluster_sync_all();          // every CTA's barriers initialised before any multicast / remote commit
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer: U once, then the deep K blocks of every tile ----------------
            tc::tma_prefetch(&tmA);
            tc::tma_prefetch(&tmU);
            mbar_arrive_expect_tx(ufull, (uint32_t)(p.u_blocks * kBlockBytes));
            for (int kb = 0; kb < p.u_blocks; ++kb)
                tc::tma_load_2d(sU + (size_t)kb * kBlockBytes, &tmU, kb * kBlockK, g * kGroup, ufull);
            const uint64_t pol = tc::policy_evict_first();   // A is streamed once per pass
            uint32_t gb = 0;
            for (int t = (int)cid; t < p.n_tiles; t += (int)ncl) {
                const int row0 = t * p.tile_stride * kTileM;
                for (int kb = 0; kb < nkt; ++kb, ++gb) {
                    if (kb >= p.n_kb) continue;             // hot block: expanded by the wide warps
                    const uint32_t slot = gb % p.stages, round = gb / p.stages;
                    if (round > 0) mbar_wait_sleep(&empty[slot], (round - 1) & 1);
                    mbar_arrive_expect_tx(&full[slot], (uint32_t)kBlockBytes);
                    if (csize == 1)
                        tc::tma_load_2d_hint(sRing + (size_t)slot * kBlockBytes, &tmA, kb * kBlockK, row0, &full[slot], pol);
                    else if (rank == 0)
                        tc::tma_load_2d_mc(sRing + (size_t)slot * kBlockBytes, &tmA, kb * kBlockK, row0, &full[slot],
                                           mc_mask, pol);
                }
            }
            // every remote arrival into this CTA's ring barriers has landed before it exits
            for (uint32_t k = 0; k < (uint32_t)p.stages && k < gb; ++k) {
                const uint32_t q = gb - 1 - k;
                mbar_wait_sleep(&empty[q % p.stages], (q / p.stages) & 1);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            // The accumulator stage already holds the tile's cold wide term (stored by the wide
            // warps), so every MMA accumulates: D = cold + A U_deep^T + H (hi, lo)^T.
            const uint32_t idb = tc::idesc_bf16_m128(nu_pad), idh = tc::idesc_f16_m128(nu_pad);
            mbar_wait_sleep(ufull, 0);
            tc::fence_after();
            int it = 0;
            uint32_t gb = 0;
            for (int t = (int)cid; t < p.n_tiles; t += (int)ncl, ++it) {
                const int st = it % kAccStages;
                mbar_wait_sleep(&wready[st], (it / kAccStages) & 1);
                tc::fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(st * 128);
                for (int kb = 0; kb < nkt; ++kb, ++gb) {
                    const uint32_t slot = gb % p.stages;
                    mbar_wait_sleep(&full[slot], (gb / p.stages) & 1);
                    tc::fence_after();
                    const uint64_t da0 = tc::sdesc_sw128(sRing + (size_t)slot * kBlockBytes);
                    if (kb < p.n_kb) {
                        const uint64_t db0 = tc::sdesc_sw128(sU + (size_t)kb * kBlockBytes);
#pragma unroll
                        for (int k = 0; k < kBlockK / 16; ++k)
                            tc::umma_f16(d_tmem, da0 + (uint64_t)(k * 2), db0 + (uint64_t)(k * 2), idb, 1u);
                    } else {
                        const int h = kb - p.n_kb;
                        for (int pc = 0; pc < p.pieces; ++pc) {
                            const uint64_t db0 = tc::sdesc_sw128(sU + (size_t)(p.n_kb + h * p.pieces + pc) * kBlockBytes);
#pragma unroll
                            for (int k = 0; k < kBlockK / 16; ++k)
                                tc::umma_f16(d_tmem, da0 + (uint64_t)(k * 2), db0 + (uint64_t)(k * 2), idh, 1u);
                        }
                    }
                    if (csize == 1) tc::umma_commit(&empty[slot]);
                    else tc::umma_commit_mc(&empty[slot], mc_mask);
                }
                tc::umma_commit(&tfull[st]);
            }
        }
    } else if (warp >= kWideWarp0 && warp < kEpiWarp0) {
        // ---------------- wide warps: hot one-hot block, cold scatter, TMEM store ----------------
        const int wt = tid - kWideWarp0 * 32;
        const int q = warp & 3, half = (warp - kWideWarp0) >> 2;
        const int row = q * 32 + lane;
        const uint32_t* __restrict__ entries = p.ws.entries;
        const uint32_t* __restrict__ pairs = p.ws.pairs;
        int it = 0;
        uint32_t gb = 0;
        for (int t = (int)cid; t < p.n_tiles; t += (int)ncl, ++it) {
            const int st = it % kAccStages;
            const int64_t tw = (int64_t)t * p.tile_stride;
            // hot: the row's one-hot fp16 K block(s), written in the TMA 128B-swizzle layout
            if (p.n_hb) {
                const uint4 hm = __ldg(&p.hot_mask[tw * kTileM + row]);
                for (int h = 0; h < p.n_hb; ++h) {
                    const uint32_t pos = gb + p.n_kb + h;
                    const uint32_t slot = pos % p.stages, round = pos / p.stages;
                    if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
                    const uint64_t bits = h == 0 ? ((uint64_t)hm.y << 32 | hm.x) : ((uint64_t)hm.w << 32 | hm.z);
                    unsigned char* rowp = sRing + (size_t)slot * kBlockBytes + (size_t)row * 128;
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        const int c = half * 4 + cc;                 // 16-byte chunk: keys 8c .. 8c+7
                        const uint32_t byte = (uint32_t)(bits >> (8 * c)) & 0xFFu;
                        uint4 v;
                        v.x = ((byte & 1u) ? 0x3C00u : 0u) | ((byte & 2u) ? 0x3C000000u : 0u);
                        v.y = ((byte & 4u) ? 0x3C00u : 0u) | ((byte & 8u) ? 0x3C000000u : 0u);
                        v.z = ((byte & 16u) ? 0x3C00u : 0u) | ((byte & 32u) ? 0x3C000000u : 0u);
                        v.w = ((byte & 64u) ? 0x3C00u : 0u) | ((byte & 128u) ? 0x3C000000u : 0u);
                        *reinterpret_cast<uint4*>(rowp + ((c ^ (row & 7)) << 4)) = v;
                    }
                    tc::fence_proxy_async_smem();
                    tc::named_bar_sync(1, kWideThreads);
                    if (wt == 0) mbar_arrive(&full[slot]);
                }
            }
            gb += nkt;
            // cold: the tile's entries (row, the key's user pairs); this CTA takes its group's users
            const uint32_t e0 = __ldcg(&p.ws.tile_off[tw]), e1 = __ldcg(&p.ws.tile_off[tw + 1]);
            for (uint32_t e = e0 + wt; e < e1; e += kWideThreads) {
                const uint32_t ent = __ldcg(&entries[e]);
                const uint32_t r = ent >> 24;
                const uint32_t ps = ent & (kMaxPassPairs - 1);
                const uint32_t pe = ps + ((ent >> kEntryPsBits) & 511u) + 1u;
                int32_t* arow = acc + r * kAccPitch;
                for (uint32_t pi = ps; pi < pe; ++pi) {
                    const uint32_t pr = __ldcg(&pairs[pi]);
                    const uint32_t u = pr >> kPairWBits;
                    if ((int)(u >> 7) == g) atomicAdd(&arow[u & 127u], pair_w(pr));
                }
            }
            tc::named_bar_sync(1, kWideThreads);
            // the accumulator stage is free once the epilogue drained it (kAccStages tiles ago)
            if (it >= kAccStages) mbar_wait(&tempty[st], ((it / kAccStages) - 1) & 1);
            tc::fence_after();
#pragma unroll 1
            for (int ch = 0; ch < 2; ++ch) {
                const int c = half * 64 + ch * 32;
                if (c >= nu_pad) break;
                int4* src = reinterpret_cast<int4*>(acc + row * kAccPitch + c);
                uint32_t f[32];
#pragma unroll
                for (int v4 = 0; v4 < 8; ++v4) {
                    const int4 v = src[v4];
                    src[v4] = make_int4(0, 0, 0, 0);
                    f[4 * v4 + 0] = __float_as_uint((float)v.x * sScale[c + 4 * v4 + 0]);   // the one rounding
                    f[4 * v4 + 1] = __float_as_uint((float)v.y * sScale[c + 4 * v4 + 1]);
                    f[4 * v4 + 2] = __float_as_uint((float)v.z * sScale[c + 4 * v4 + 2]);
                    f[4 * v4 + 3] = __float_as_uint((float)v.w * sScale[c + 4 * v4 + 3]);
                }
                tc::tmem_st32_nowait(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(st * 128 + c), f);
            }
            tc::tmem_wait_st();
            tc::fence_before();
            tc::named_bar_sync(1, kWideThreads);
            if (wt == 0) mbar_arrive(&wready[st]);
        }
    } else if (warp >= kEpiWarp0) {
        // ---------------- epilogue: TMEM -> registers, kappa, sample store / filter ----------------
        const int e = warp - kEpiWarp0;
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int it = 0;
        for (int t = (int)cid; t < p.n_tiles; t += (int)ncl, ++it) {
            const int st = it % kAccStages;
            const int64_t a = (int64_t)t * p.tile_stride * kTileM + row;   // shard-local ad
            const bool valid = a < p.n_ads;
            mbar_wait_sleep(&tfull[st], (it / kAccStages) & 1);
            tc::fence_after();
#pragma unroll 1
            for (int ch = 0; ch < 2; ++ch) {
                const int c = (e >> 2) * 64 + ch * 32;
                if (c >= nu_pad) break;
                uint32_t r[32];
                tc::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(st * 128 + c), r);
                const int nuc = nu - c;
                const uint32_t umask = nuc >= 32 ? 0xFFFFFFFFu : (nuc > 0 ? (1u << nuc) - 1u : 0u);
                if (MODE == 0 && p.dense) {
                    for (int j = 0; j < 32; ++j) {
                        const int sl = sDense[c + j];
                        if (sl >= 0 && ((umask >> j) & 1u)) {
                            float s = __uint_as_float(r[j]);
                            if (s == 0.f) s = 0.f;
                            p.ws.dense[(size_t)sl * p.n_pad + a] = valid ? s : __int_as_float(0xFF800000);
                        }
                    }
                } else if (MODE == 0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        float s = __uint_as_float(r[j]);
                        if (s == 0.f) s = 0.f;                       // -0 -> +0 (R14)
                        if ((umask >> j) & 1u)
                            p.ws.samp[(size_t)(g * kGroup + c + j) * p.n_samp + (int64_t)t * kTileM + row] =
                                valid ? s : __int_as_float(0xFF800000);
                    }
                } else {
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
                    uint32_t cols = __reduce_or_sync(FULL, pass);
#pragma unroll 1
                    while (cols) {
                        const int j = __ffs(cols) - 1;
                        cols &= cols - 1u;
                        const int ul = c + j;                         // CTA-local user
                        const int u = g * kGroup + ul;                // pass user
                        const bool maybe = (pass >> j) & 1u;
                        float s = 0.f;
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) s = (jj == j) ? __uint_as_float(r[jj]) : s;
                        if (s == 0.f) s = 0.f;                       // -0 -> +0 (R14)
                        const uint64_t key = maybe ? kappa_of(s, p.ad_begin + (uint32_t)a) : 0ull;
                        const bool take = maybe && key >= sTheta[ul];
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
            tc::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[st]);
        }
    }
    __syncwarp();
    tc::fence_before();
    __syncthreads();
    tc::cluster_sync_all();
    if (warp == 2) tc::tmem_dealloc(tmem_base, kAccStages * 128);
}

// ------------------------------------------------------------------------------------------
// A6a theta: the r-th largest key of each user's sampled ads
// ------------------------------------------------------------------------------------------
// Two histogram passes over ord(score) (11 + 11 bits; private per-warp-group histograms) narrow
// the r-th largest down to a 22-bit prefix; the sampled keys at or above it are compacted into
// shared memory (or, past its capacity, selected from global memory) and the exact r-th is taken.
constexpr int kThetaThreads = 1024;
constexpr int kThetaCopies = 8;

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

// rerun = 1: only the users flagged by final_kernel, their lists reset: short users at rank K
// of the sample; overflowed users at rank K of ALL their scores (dense), an exact threshold
__global__ void __launch_bounds__(kThetaThreads, 1) theta_kernel(Ws ws, int n_samp, int rank, uint32_t ad_begin,
                                                                int P, int scap, int rerun, int64_t n_pad) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t sScalar[8];
    const int u = blockIdx.x;
    if (u >= P) return;
    const uint32_t fl = __ldcg(&ws.uflags[u]);
    if (rerun && !(fl & (kFlagShort | kFlagOverflow))) return;   // (kFlagRaise users: theta already set)
    const bool dense = rerun && (fl & kFlagOverflow);
    const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5;
    const int Pk = pow2ceil_i(rank);
    uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);                 // [Pk]
    uint32_t* hist = reinterpret_cast<uint32_t*>(sbuf + Pk);            // [kThetaCopies][2048]
    uint64_t* scand = reinterpret_cast<uint64_t*>(hist + kThetaCopies * 2048);   // [scap]
    uint32_t* myh = hist + (warp % kThetaCopies) * 2048;
    if (dense) n_samp = (int)n_pad;
    const float* sp = dense ? ws.dense + (size_t)(fl >> 8) * n_pad : ws.samp + (size_t)u * n_samp;
    const float4* sp4 = reinterpret_cast<const float4*>(sp);
    const int n4 = n_samp / 4;
    const int64_t stride = dense ? 1 : kSampleStride;
    auto ad_of = [stride](int64_t i) { return (i / kTileM) * stride * kTileM + (i % kTileM); };
    uint32_t prefix = 0, need = (uint32_t)rank;
    for (int pass = 0; pass < 2; ++pass) {
        const int shift = pass == 0 ? 21 : 10;
        for (int i = tid; i < kThetaCopies * 2048; i += nt) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < n4; i += nt) {
            const float4 v = __ldcg(&sp4[i]);
            const float f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t o = ord_of(f[r]);
                if (pass == 0 || (o >> 21) == (prefix >> 21)) atomicAdd(&myh[(o >> shift) & 2047u], 1u);
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
        const bool done = pass == 0 && (uint64_t)sScalar[1] + hist[sScalar[0]] <= (uint64_t)scap;
        __syncthreads();
        if (done) break;
    }
    if (tid == 0) sScalar[2] = 0;
    __syncthreads();
    for (int i = tid; i < n_samp; i += nt) {
        const float s = __ldcg(&sp[i]);
        if (ord_of(s) >= prefix) {
            const uint32_t pos = atomicAdd(&sScalar[2], 1u);
            if ((int)pos < scap) scand[pos] = kappa_of(s, ad_begin + (uint32_t)ad_of(i));
        }
    }
    __syncthreads();
    const int64_t cnt = sScalar[2];
    __syncthreads();
    int nsel;
    if (cnt <= scap) {
        nsel = cta_select_topk([scand](int64_t i) { return scand[i]; }, cnt, rank, sbuf, nullptr, 0, hist, sScalar);
    } else {
        auto get = [sp, ad_begin, ad_of](int64_t i) { return kappa_of(__ldcg(&sp[i]), ad_begin + (uint32_t)ad_of(i)); };
        // (the dense row's padding ads beyond n_ads hold -inf: they never reach rank K <= n_ads)
        nsel = cta_select_topk(get, n_samp, rank, sbuf, nullptr, 0, hist, sScalar);
    }
    if (tid == 0) {
        ws.theta[u] = (nsel >= rank) ? sbuf[rank - 1] : 0ull;
        ws.cand_count[u] = 0;
    }
}

// ------------------------------------------------------------------------------------------
// A6c final: exact top-K of the candidates
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1) final_kernel(Ws ws, int64_t cap, int K, int P, int32_t* out_ids,
                                                       float* out_scores, uint64_t* out_keys, int64_t scap,
                                                       int rerun, int rank, uint32_t* err) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t sScalar[8];
    const int u = blockIdx.x;
    if (u >= P) return;
    if (rerun) {
        const uint32_t f = __ldcg(&ws.uflags[u]);
        if (!(f & kFlagAny)) return;
    }
    const int64_t n = __ldcg(&ws.cand_count[u]);
    const int Pk = pow2ceil_i(K);
    uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);
    uint32_t* shist = reinterpret_cast<uint32_t*>(sbuf + Pk);
    uint64_t* scand = reinterpret_cast<uint64_t*>(shist + kSelBins);
    const uint64_t* cb = ws.cand + (size_t)u * cap;
    if (n > cap) {
        // candidate overflow (more than `cap` ads at or above theta: massive score ties, or an
        // inventory whose sampled tiles misrepresent the rest).  The first kMaxFallback such users
        // of a pass get their scores recomputed densely and an exact rank-K threshold; the others
        // a raised threshold, the K-th largest of the stored subset (a valid lower bound of the
        // K-th largest overall, since the subset's keys are all candidates).  Both are refiltered.
        __shared__ uint32_t sSlot;
        if (threadIdx.x == 0) sSlot = rerun ? (uint32_t)kMaxFallback + 1u : atomicAdd(&ws.header[4], 1u);
        __syncthreads();
        const uint32_t slot = sSlot;
        if (slot < (uint32_t)kMaxFallback) {
            if (threadIdx.x == 0) ws.uflags[u] = kFlagOverflow | (slot << 8);
        } else if (!rerun) {
            const int nsel = cta_select_topk([cb](int64_t i) { return __ldcg(&cb[i]); }, cap, K, sbuf, scand, scap,
                                             shist, sScalar);
            if (threadIdx.x == 0) {
                ws.theta[u] = sbuf[min(nsel, K) - 1];
                ws.cand_count[u] = 0u;
                ws.uflags[u] = kFlagRaise;
                ws.header[2] = 1u;
            }
        } else if (threadIdx.x == 0) {
            ws.uflags[u] = 0u;
            atomicOr(err, 2u);             // still overflowing after the rerun: flagged, output incomplete
        }
        return;
    }
    // fewer than K keys reached theta (theta at a sample rank below K): the top-K is not
    // guaranteed inside the candidates -- the gated rerun takes theta at rank K
    if (n < K && !rerun && rank < K) {
        if (threadIdx.x == 0) { ws.uflags[u] = kFlagShort; ws.header[2] = 1u; }
        return;
    }
    if (threadIdx.x == 0) ws.uflags[u] = 0u;
    const int nsel = cta_select_topk([cb](int64_t i) { return __ldcg(&cb[i]); }, n, K, sbuf, scand, scap, shist,
                                     sScalar);
    cta_write_topk(sbuf, nsel, K, out_ids ? out_ids + (size_t)u * K : nullptr,
                   out_scores ? out_scores + (size_t)u * K : nullptr, out_keys ? out_keys + (size_t)u * K : nullptr);
}

// ------------------------------------------------------------------------------------------
// host
// ------------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult qres;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) == cudaSuccess &&
            qres == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

static bool encode_2d_16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
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

struct Tuning {
    int n_hb, pieces;
};

static Tuning tuning(const ebr_index* idx) {
    Tuning t;
    t.n_hb = std::min(1, idx->n_hot / 64);                  // 64 hot keys: 80 % of C3's hits
    t.pieces = 2;
    if (const char* e = getenv("EBR_HOT_BLOCKS")) t.n_hb = std::max(0, std::min(t.n_hb, atoi(e)));
    if (getenv("EBR_NO_HOT")) t.n_hb = 0;                 // every key through the compressed lists
    if (const char* e = getenv("EBR_HOT_PIECES")) t.pieces = std::max(1, std::min(2, atoi(e)));
    return t;
}

static size_t gemm_smem(int u_blocks, int stages) {
    return 1024 + (size_t)(u_blocks + stages) * kBlockBytes + (size_t)kTileM * kAccPitch * 4 +
           (size_t)(2 * stages + 3 * kAccStages + 1) * 8 + 16 + (size_t)kGroup * 20;
}

}  // namespace batch

using namespace batch;

bool batch_eligible(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k) {
    if (getenv("EBR_NO_BATCH_PATH")) return false;
    // small batches take the tensor-core path too on large inventories, where the latency path's
    // per-user wide scratch no longer fits L2 (C5 sweep: B=4 at 20 M ads 3.9 ms latency path)
    const bool big = idx->n_ads >= ((int64_t)1 << 21);
    return idx->dtype == EBR_BF16 && (batch >= 16 || (big && batch >= 4)) && idx->d_pad <= 256 &&
           idx->n_fields <= 255 && pass_users(idx, slots) >= 32 &&
           idx->n_ads >= (int64_t)4 * kSampleStride * std::max(k, kTileM) && get_encode() != nullptr;
}

size_t batch_workspace_bytes(const ebr_index* idx, int32_t slots, int32_t k) {
    return layout(idx, slots, k).total + 1024;
}

int32_t batch_launches(const ebr_index* idx, int32_t batch, int32_t slots) {
    const int P = pass_users(idx, slots);
    return ((batch + P - 1) / P) * 15;
}

// The workspace passed here is the batched region (after the latency path's region).
ebr_status run_batch(const QueryArgs& q, void* region, uint32_t* err_word) {
    const ebr_index* idx = q.idx;
    const Layout L = layout(idx, q.slots, q.k);
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(region) + 1023) & ~(uintptr_t)1023);
    Ws ws = carve(base, L);
    Tuning tu = tuning(idx);
    const int n_kb = idx->d_pad / kBlockK;
    const int n_tiles = (int)L.n_tiles;
    const int n_samp_tiles = (int)(L.n_samp / kTileM);
    const int u_cols = (int)L.u_cols;
    int max_smem = 0;
    cudaError_t e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, idx->device);
    if (e != cudaSuccess) return cuda_check(e, "attr(max smem)");
    // ring stages: >= one tile's K blocks (the hot block's writer waits on the ring, see
    // score_kernel) plus one of lookahead; hot blocks are dropped until that fits
    int stages = 0;
    for (; tu.n_hb >= 0; --tu.n_hb) {
        const int ub = n_kb + tu.n_hb * tu.pieces, nkt = n_kb + tu.n_hb;
        stages = 6;
        while (stages > nkt + 1 && gemm_smem(ub, stages) > (size_t)max_smem) --stages;
        if (gemm_smem(ub, stages) <= (size_t)max_smem) break;
    }
    if (tu.n_hb < 0) return set_error(EBR_EUNSUPPORTED, "batched path: d=%d does not fit shared memory", idx->d);
    const int u_blocks = n_kb + tu.n_hb * tu.pieces;
    const size_t smem = gemm_smem(u_blocks, stages);
    CUtensorMap tmA, tmU;
    if (!encode_2d_16(&tmA, idx->A, (uint64_t)idx->d_pad, (uint64_t)idx->n_pad, kBlockK, kTileM))
        return set_error(EBR_ECUDA, "cuTensorMapEncodeTiled(A) failed");
    const int Ppad_max = (int)((L.P + kGroup - 1) / kGroup * kGroup);
    if (!encode_2d_16(&tmU, ws.U, (uint64_t)u_cols, (uint64_t)Ppad_max, kBlockK, kGroup))
        return set_error(EBR_ECUDA, "cuTensorMapEncodeTiled(U) failed");
    // kernel attributes: set once per process (values fixed by the build)
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        auto set = [&](const void* f, int bytes) {
            cudaError_t x = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            if (x != cudaSuccess && attr_err == cudaSuccess) attr_err = x;
        };
        const int big = 227 * 1024;
        set((const void*)score_kernel<0>, big);
        set((const void*)score_kernel<1>, big);
        set((const void*)theta_kernel, 200 * 1024);
        set((const void*)final_kernel, 200 * 1024);
        set((const void*)entry_count_kernel, kRangeMaxTiles * kTileM * 4);
        set((const void*)entry_write_kernel, kRangeMaxTiles * kTileM * 4);
        for (const void* f : {(const void*)score_kernel<0>, (const void*)score_kernel<1>}) {
            cudaError_t x = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            (void)x;
        }
    });
    if (attr_err != cudaSuccess) return cuda_check(attr_err, "attr(batched kernels)");

    const size_t tsmem = 200 * 1024;
    const size_t fsmem = 200 * 1024;
    const int64_t fscap = (int64_t)(fsmem - (size_t)pow2ceil_i(q.k) * 8 - kSelBins * 4) / 8;
    const double ks = (double)q.k / kSampleStride;
    int rank = (int)std::ceil(ks + 5.0 * std::sqrt(ks) + 8.0);
    if (const char* r = getenv("EBR_THETA_RANK")) rank = atoi(r);   // test hook
    rank = std::max(1, std::min(rank, q.k));
    auto tscap_of = [&](int r) { return (int)((tsmem - (size_t)pow2ceil_i(r) * 8 - kThetaCopies * 2048 * 4) / 8); };
    int64_t cap = L.cap;
    if (const char* c = getenv("EBR_TEST_CAND_CAP")) cap = std::min<int64_t>(cap, std::max(1, atoi(c)));

    EntryArgs ea;
    ea.hdr = idx->chunk_hdr; ea.chunk_last = idx->chunk_last; ea.payload = idx->payload;
    ea.n_ads = idx->n_ads; ea.n_pad = idx->n_pad; ea.range_ads = L.range_ads;
    ea.n_ranges = (int)L.n_ranges; ea.n_tiles = n_tiles; ea.NU = L.NU;
    const size_t rsmem = (size_t)L.range_ads * 4;

    for (int b0 = 0; b0 < q.batch; b0 += (int)L.P) {
        const int P = std::min((int)L.P, q.batch - b0);
        const int G = (P + kGroup - 1) / kGroup;
        PlanArgs pa;
        pa.user_feat = q.user_feat + (size_t)b0 * idx->n_fields * q.slots;
        pa.user_x = q.user_x + (size_t)b0 * idx->n_fields * q.slots;
        pa.user_emb = reinterpret_cast<const uint16_t*>(q.user_emb) + (size_t)b0 * idx->d;
        pa.key_chunk_off = idx->key_chunk_off; pa.key_word_off = idx->key_word_off; pa.cross_w = idx->cross_w;
        pa.field_card = idx->field_card; pa.field_base = idx->field_base; pa.hot_slot = idx->hot_slot;
        pa.F = idx->n_fields; pa.S = q.slots; pa.P = P; pa.d = idx->d; pa.d_pad = idx->d_pad;
        pa.n_hot_used = tu.n_hb * 64; pa.pieces = tu.pieces; pa.u_cols = u_cols; pa.TS = L.TS; pa.err = err_word;
        const int nslot = P * idx->n_fields * q.slots;
        const int pgrid = std::max(1, std::min(4 * idx->sm_count, (nslot + 255) / 256));
        plan_a_kernel<<<pgrid, 256, 0, q.stream>>>(pa, ws);
        plan_b_kernel<<<1, kPlanThreads, 0, q.stream>>>(pa, ws);
        plan_c_kernel<<<std::max(pgrid, 2 * idx->sm_count), 256, 0, q.stream>>>(pa, ws);
        span_kernel<<<(unsigned)((nslot + 7) / 8), 256, 0, q.stream>>>(ea, ws);
        entry_count_kernel<<<(unsigned)L.n_ranges, 512, rsmem, q.stream>>>(ea, ws);
        range_scan_kernel<<<1, 1024, 0, q.stream>>>(ea, ws);
        entry_write_kernel<<<(unsigned)L.n_ranges, 512, rsmem, q.stream>>>(ea, ws);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_check(e, "launch(plan/entries)");

        GemmParams gp;
        gp.n_ads = idx->n_ads; gp.n_pad = idx->n_pad; gp.dense = 0; gp.ad_begin = (uint32_t)idx->ad_begin;
        gp.n_kb = n_kb; gp.n_hb = tu.n_hb; gp.pieces = tu.pieces; gp.u_blocks = u_blocks;
        gp.P = P; gp.n_samp = (int)L.n_samp; gp.stages = stages; gp.cap = cap; gp.rerun = 0;
        gp.hot_mask = reinterpret_cast<const uint4*>(idx->hot_mask); gp.ws = ws; gp.err = err_word;
        // the U tensor map covers the whole pass tile: each CTA loads its group's 128 rows
        auto launch_score = [&](int mode, int tiles, int stride, int rerun, int dense = 0) -> cudaError_t {
            gp.n_tiles = tiles; gp.tile_stride = stride; gp.rerun = rerun; gp.dense = dense;
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)G;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.blockDim = dim3(kGemmThreads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = q.stream;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int ncl = idx->sm_count / G;
            {
                static std::mutex mu;
                static int cached[2][kMaxCluster + 1] = {};
                std::lock_guard<std::mutex> lk(mu);
                int& c = cached[mode][G];
                if (!c) {
                    cfg.gridDim = dim3((unsigned)(G * ncl));
                    int n = 0;
                    cudaError_t x = cudaOccupancyMaxActiveClusters(
                        &n, mode ? (const void*)score_kernel<1> : (const void*)score_kernel<0>, &cfg);
                    c = (x == cudaSuccess && n > 0) ? n : ncl;
                }
                ncl = std::min(ncl, c);
            }
            ncl = std::max(1, std::min(ncl, tiles));
            cfg.gridDim = dim3((unsigned)(G * ncl));
            return mode ? cudaLaunchKernelEx(&cfg, score_kernel<1>, tmA, tmU, gp)
                        : cudaLaunchKernelEx(&cfg, score_kernel<0>, tmA, tmU, gp);
        };
        int32_t* oi = q.out_ids ? q.out_ids + (size_t)b0 * q.k : nullptr;
        float* os = q.out_scores ? q.out_scores + (size_t)b0 * q.k : nullptr;
        uint64_t* ok = q.out_keys ? q.out_keys + (size_t)b0 * q.k : nullptr;
        e = launch_score(0, n_samp_tiles, kSampleStride, 0);
        if (e != cudaSuccess) return cuda_check(e, "launch(score sample)");
        theta_kernel<<<P, kThetaThreads, tsmem, q.stream>>>(ws, (int)L.n_samp, rank, (uint32_t)idx->ad_begin, P,
                                                           tscap_of(rank), 0, idx->n_pad);
        e = launch_score(1, n_tiles, 1, 0);
        if (e != cudaSuccess) return cuda_check(e, "launch(score filter)");
        final_kernel<<<P, 512, fsmem, q.stream>>>(ws, cap, q.k, P, oi, os, ok, fscap, 0, rank, err_word);
        // gated reruns (exact either way): the overflowed users' scores densely, then theta at rank
        // K for the users short of K candidates (sample) or overflowed (dense), filter, select
        e = launch_score(0, n_tiles, 1, 0, 1);
        if (e != cudaSuccess) return cuda_check(e, "launch(score dense)");
        theta_kernel<<<P, kThetaThreads, tsmem, q.stream>>>(ws, (int)L.n_samp, q.k, (uint32_t)idx->ad_begin, P,
                                                           tscap_of(q.k), 1, idx->n_pad);
        e = launch_score(1, n_tiles, 1, 1);
        if (e != cudaSuccess) return cuda_check(e, "launch(score rerun)");
        final_kernel<<<P, 512, fsmem, q.stream>>>(ws, cap, q.k, P, oi, os, ok, fscap, 1, q.k, err_word);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_check(e, "launch(batch)");
    }
    return EBR_OK;
}

}  // namespace ebr
