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
//   entry_bin / entry_sort     A2: the entry stream (decode once, bucket by ad range, sort by ad)
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

constexpr int kGroup = 128;          // users per CTA (UMMA M: TMEM lanes)
constexpr int kMaxCluster = 2;       // CTAs (user groups) per cluster: <= 256 users per pass
constexpr int kTileM = 128;          // ads per tile (UMMA M)
constexpr int kBlockK = 64;          // 16-bit elements per 128-byte swizzle row
constexpr int kBlockBytes = kTileM * 128;   // one ring stage: 128 rows x 128 B
constexpr int kSampleStride = 16;    // every 16th tile (at least) is sampled for theta
constexpr int kSampleStrideMax = 64; // ... and every 64th on large inventories (sample_stride())
#ifndef EBR_WIDE_WARPS
#define EBR_WIDE_WARPS 16
#endif
constexpr int kWideWarp0 = 4, kWideWarps = EBR_WIDE_WARPS, kWideThreads = 32 * kWideWarps;
constexpr int kEpiWarp0 = kWideWarp0 + kWideWarps, kEpiWarps = 8;
constexpr int kGemmThreads = 32 * (kEpiWarp0 + kEpiWarps);   // TMA, MMA, 2 hot, wide, 8 epilogue
constexpr int kMaxHotBlocks = 2;     // hot K blocks of 64 keys (the index keeps up to 128 hot keys)
constexpr int kPairUBits = 7;        // cold pair = w~ 2^S (25-bit two's complement) << 7 | user in the group
constexpr int kPairWMax = 24;        // |w~ 2^S| < 2^24
constexpr int kMaxUnion = 1 << 14;   // union key slots per pass (14 bits in the level-1 bin entries)
#ifndef EBR_BIN_ADS
#define EBR_BIN_ADS 1024
#endif
constexpr int kBinAds = EBR_BIN_ADS;  // ads per entry bin (8 tiles at 1024)
#ifndef EBR_ORDER_STAGE
#define EBR_ORDER_STAGE 16384
#endif
constexpr int kOrderStage = EBR_ORDER_STAGE;   // bin entries staged in shared memory by entry_order
constexpr int kClasses = 4;          // pair-count classes of an entry (1, 2, 3-4, 5+ pairs): a tile's
                                     // entries are ordered by class so a warp's entries carry similar work
#ifndef EBR_ORDER_THREADS
#define EBR_ORDER_THREADS 1024
#endif
#ifndef EBR_BIN_GRID
#define EBR_BIN_GRID 8
#endif
constexpr int kOrderThreads = EBR_ORDER_THREADS;
constexpr int kPlanThreads = 1024;
constexpr uint32_t kFlagShort = 1u, kFlagOverflow = 2u, kFlagRaise = 4u;   // uflags; overflow users carry their dense slot << 8
constexpr uint32_t kFlagAny = kFlagShort | kFlagOverflow | kFlagRaise;
constexpr int kMaxFallback = 2;      // overflowed users per pass recomputed exactly (dense scores)

constexpr int kMaxAccStages = 3;
constexpr int kMaxStages = 12;       // deep A ring stages (16 KB, or 8 KB per CTA of a pair; as many as fit)
constexpr int kPrefetchTiles = 4;    // tiles of A prefetched into L2 ahead of the ring's TMA loads
constexpr int kHotStages = 2;        // ring of on-chip generated one-hot K blocks
// int32 words per fixed-point row of the cold tile [users][ads]: an even pitch of 2 mod 32 words
// keeps the store phase's 64-bit read-and-clear exchanges conflict-free (lane = user)
constexpr int kAccPitch = kGroup + 2;
constexpr int kEntBuf = 2048;        // entries of a tile staged in shared memory (bulk copy; the rest from L2)
constexpr int kEntHdr = 16;          // words of an entry buffer's header (quarter bounds, copied count)
// shared memory of the fused kernel next to the A ring and the pairs: the hot ring, the cold
// quarter buffers, 2 entry buffers, the byte -> one-hot table, the heavy list, barriers and
// per-user scalars
__host__ __device__ constexpr size_t score_smem_fixed() {
    return (size_t)kHotStages * kBlockBytes + (size_t)kGroup * kAccPitch * 4 + 2 * (size_t)(kEntBuf + kEntHdr) * 4 +
           256 * 16 +
           (size_t)(2 * kMaxStages + 2 * kHotStages + 3 * kMaxAccStages + 4 + 1) * 8 + 16 +
           (size_t)kGroup * 20;
}

// ------------------------------------------------------------------------------------------
// workspace
// ------------------------------------------------------------------------------------------
struct Ws {
    uint32_t* header;     // [0] n_union [1] n_pairs [2] any user short of K [3] entries total [4] overflowed users
    uint32_t* hkey;       // [TS] key + 1 (0 = empty)
    uint32_t* hcnt;       // [TS][kMaxCluster] user pairs of the key per group (left zero by plan_c)
    uint32_t* hslot;      // [TS] union slot of the key
    uint32_t* hpair;      // [TS][kMaxCluster] first pair of the key in its group's list
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
    uint32_t* pinfo;      // [kMaxCluster][NU] group g's pairs of union slot s: first pair << 8 | count (0: none)
    uint32_t* ucls;       // [NU] 3 bits per group g at 3g: 0 = no user of g, else 1 + pair-count class
    uint32_t* pairs;      // [kMaxCluster][kGroup * F * S] each group's pairs, by union slot
    uint16_t* U;          // [P_pad][u_cols] deep bf16 | hot fp16 pieces
    uint32_t* uchunk;     // [NU + 1] exclusive scan of the union keys' chunk counts
    uint32_t* bin_cnt;    // [n_bins] entries in each ad-range bin (left zero by entry_sort)
    uint32_t* tbeg;       // [kMaxCluster][n_tiles] first entry of each tile in group g's stream
    uint32_t* tend;       // [kMaxCluster][n_tiles]
    uint32_t* gentries;   // [pool] the groups' entry streams (bins claim their ranges):
                          //   ad row << 24 | first pair << 8 | pairs, ordered by (tile, pair-count class)
    uint32_t* entries;    // [n_bins][bin_cap] level-1 bins (bin_cap = bin_ads * max keys of an ad)
    float* samp;          // [P][n_samp]
    uint64_t* theta;      // [P]
    uint32_t* cand_count; // [P]
    uint64_t* cand;       // [P][cap]
    uint32_t* uflags;     // [P] kFlagShort | kFlagOverflow
    float* dense;         // [kMaxFallback][n_pad] every score of an overflowed user
    unsigned long long* prof;   // [32] cycle accounting of the fused kernel's roles (EBR_DIAG & 4)
};

struct Layout {
    size_t total;
    size_t off[32];
    int64_t TS, NU, P, n_samp, cap, n_bins, bin_ads, bin_cap, n_tiles, u_cols, gcap, pool, sstride;
};

static int64_t pow2ceil64(int64_t x) {
    int64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// users per pass: <= kGroup * kMaxCluster, the union slots must fit 14 bits and a group's pairs
// the 16-bit first-pair field of an entry
int pass_users(const ebr_index* idx, int32_t slots) {
    const int64_t fs = (int64_t)idx->n_fields * slots;
    int64_t p = std::min<int64_t>(kGroup * kMaxCluster, kMaxUnion / std::max<int64_t>(fs, 1));
    if ((int64_t)kGroup * fs > 65535) p = 0;
    // shared memory of the fused kernel: >= one tile's deep K blocks + 1 of the A ring, the fixed
    // part and a group's worst-case pairs (4 B x 128 F S)
    const int64_t n_kb = (idx->d_pad + kBlockK - 1) / kBlockK;
    if (1024 + (n_kb + 1) * kBlockBytes + (int64_t)score_smem_fixed() + 4 * (int64_t)kGroup * fs > 232448) p = 0;
    return (int)(p / 32 * 32);
}

// the sample covers every sstride-th tile: the largest power of two <= kSampleStrideMax that keeps
// >= 4 max(K, 128) sampled ads (batch_eligible guarantees it for kSampleStride) and stride x K
// <= 160 k (a rank-K rerun then yields ~stride x K candidates per user: the list capacity)
static int64_t sample_stride(const ebr_index* idx, int k) {
    int64_t st = kSampleStrideMax;
    while (st > kSampleStride && (idx->n_ads < 4 * st * std::max(k, kTileM) || st * k > 160000)) st >>= 1;
    return st;
}

// candidate list capacity per user: the rank-K rerun's ~stride x K candidates with a 1.5x margin
static int64_t cand_cap(const ebr_index* idx, int k) {
    const int64_t st = sample_stride(idx, k);
    return std::max<int64_t>(65536, (3 * st * (int64_t)k) / 2 + 4096);
}

static Layout layout(const ebr_index* idx, int32_t slots, int32_t k) {
    Layout L;
    const int P = pass_users(idx, slots);
    L.P = P;
    L.NU = (int64_t)P * idx->n_fields * slots;
    L.gcap = (int64_t)kGroup * idx->n_fields * slots;
    L.TS = pow2ceil64(2 * L.NU);
    L.n_tiles = idx->n_pad / kTileM;
    L.sstride = sample_stride(idx, k);
    L.n_samp = ((L.n_tiles + L.sstride - 1) / L.sstride) * kTileM;
    L.cap = cand_cap(idx, k);
    // entry bins of kBinAds ads; a bin's worst case is bin_ads * F entries (an ad has <= F keys)
    L.bin_ads = kBinAds;
    L.bin_cap = L.bin_ads * std::max<int64_t>(1, idx->max_ad_keys);
    L.n_bins = (idx->n_pad + L.bin_ads - 1) / L.bin_ads;
    // group streams: an (ad, key) entry appears once per group querying the key, so at most
    // min(groups, ...) x F entries per ad; sized for the pass's largest group count
    L.pool = (int64_t)std::min<int64_t>(kMaxCluster, (P + kGroup - 1) / kGroup) * idx->n_pad *
             std::max<int64_t>(1, idx->max_ad_keys);
    L.u_cols = idx->d_pad + (int64_t)kMaxHotBlocks * 64 * 2;
    const int64_t Ppad = (int64_t)((P + kGroup - 1) / kGroup) * kGroup;
    const size_t sizes[] = {
        64,                                         // 0 header
        (size_t)L.TS * 4, (size_t)L.TS * 4 * kMaxCluster, (size_t)L.TS * 4, (size_t)L.TS * 4 * kMaxCluster,   // 1-4 hash
        (size_t)L.NU * 4, (size_t)L.NU * 4,         // 5-6 items
        (size_t)Ppad * 128 * 4,                     // 7 hotw
        (size_t)P * 4, (size_t)P * 4, (size_t)P * 4, (size_t)P * 4,   // 8-11 per user
        (size_t)L.NU * 4, (size_t)L.NU * 4, (size_t)L.NU * 4, (size_t)L.NU * 4,   // 12-15 union
        (size_t)kMaxCluster * L.NU * 4 + (size_t)L.NU * 4 + 1024,   // 16 pinfo | ucls
        (size_t)kMaxCluster * L.gcap * 4,           // 17 pairs
        (size_t)Ppad * L.u_cols * 2,                // 18 U
        (size_t)(L.NU + 1) * 4,                     // 19 uchunk
        (size_t)L.n_bins * 4,                       // 20 bin_cnt
        (size_t)L.n_tiles * 4 * kMaxCluster, (size_t)L.n_tiles * 4 * kMaxCluster,   // 21-22 tbeg / tend
        (size_t)L.pool * 4,                         // 23 gentries
        (size_t)L.n_bins * L.bin_cap * 4,           // 24 entries
        (size_t)P * L.n_samp * 4,                   // 25 samp
        (size_t)P * 8, (size_t)P * 4,               // 26-27 theta, count
        (size_t)P * L.cap * 8,                      // 28 cand
        (size_t)P * 4,                              // 29 flags
        (size_t)kMaxFallback * idx->n_pad * 4,      // 30 dense
        32 * 8,                                     // 31 prof
    };
    size_t o = 0;
    for (int i = 0; i < 32; ++i) {
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
    w.pinfo = (uint32_t*)at(16); w.pairs = (uint32_t*)at(17);
    w.ucls = (uint32_t*)(at(16) + (((size_t)kMaxCluster * L.NU * 4 + 1023) & ~(size_t)1023));
    w.U = (uint16_t*)at(18);
    w.uchunk = (uint32_t*)at(19);
    w.bin_cnt = (uint32_t*)at(20);
    w.tbeg = (uint32_t*)at(21); w.tend = (uint32_t*)at(22);
    w.gentries = (uint32_t*)at(23);
    w.entries = (uint32_t*)at(24);
    w.samp = (float*)at(25);
    w.theta = (uint64_t*)at(26); w.cand_count = (uint32_t*)at(27);
    w.cand = (uint64_t*)at(28);
    w.uflags = (uint32_t*)at(29);
    w.dense = (float*)at(30);
    w.prof = (unsigned long long*)at(31);
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
    int64_t TS, NU, gcap;
    uint32_t* err;
};

__device__ __forceinline__ uint32_t hash_key(uint32_t k) {
    k ^= k >> 16; k *= 0x7feb352dU; k ^= k >> 15; k *= 0x846ca68bU; k ^= k >> 16;
    return k;
}

__device__ __forceinline__ uint32_t pair_class(uint32_t c) {   // c >= 1 pairs -> 0..kClasses-1
    return c <= 2u ? c - 1u : c <= 4u ? 2u : 3u;
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
        atomicAdd(&ws.hcnt[(size_t)t * kMaxCluster + u / kGroup], 1u);
        ws.item_t[i] = (int32_t)t;
        ws.item_w[i] = w;
    }
}

// plan_b (one CTA): compacts the hash table into union slots, gives each (slot, group) its range
// in the group's pair list, resets the table for the next pass, and derives every user's
// fixed-point scale
//   S_u = min(24 - e_max, 30 - e_sum),  max|w~| < 2^e_max,  sum|w~| < 2^e_sum
// so each w~ 2^S fits the 25-bit pair field and every partial sum fits int32 (R23).
// Each thread scans a run of table positions; one block scan combines the runs (6 sums at once).
constexpr int kPlanNV = 2 + kMaxCluster;   // slots, chunks, per-group pairs
__global__ void __launch_bounds__(kPlanThreads) plan_b_kernel(PlanArgs a, Ws ws) {
    __shared__ uint32_t sW[kPlanThreads / 32][kPlanNV];
    __shared__ uint32_t sTot[kPlanNV];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t per = (a.TS + kPlanThreads - 1) / kPlanThreads;
    const int64_t t0 = (int64_t)tid * per, t1 = min(a.TS, t0 + per);
    uint32_t v[kPlanNV] = {};
    // 8 table positions per round with every load of a round in flight at once (this CTA alone
    // walks the whole table: the latency of dependent loads is the cost)
    for (int64_t tb = t0; tb < t1; tb += 8) {
        uint32_t key1[8], c0[8], c1[8], hc[8][kMaxCluster];
#pragma unroll
        for (int j = 0; j < 8; ++j) key1[j] = tb + j < t1 ? ws.hkey[tb + j] : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c0[j] = key1[j] ? a.key_chunk_off[key1[j] - 1u] : 0u;
            c1[j] = key1[j] ? a.key_chunk_off[key1[j]] : 0u;
#pragma unroll
            for (int g = 0; g < kMaxCluster; ++g) hc[j][g] = key1[j] ? ws.hcnt[(tb + j) * kMaxCluster + g] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            v[0] += key1[j] ? 1u : 0u;
            v[1] += c1[j] - c0[j];
#pragma unroll
            for (int g = 0; g < kMaxCluster; ++g) v[2 + g] += hc[j][g];
        }
    }
    // block exclusive scan of v[] over threads
    uint32_t incl[kPlanNV];
#pragma unroll
    for (int i = 0; i < kPlanNV; ++i) {
        uint32_t x = v[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        incl[i] = x;
        if (lane == 31) sW[warp][i] = x;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < kPlanNV; ++i) {
            const uint32_t w = sW[lane][i];
            uint32_t x = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            sW[lane][i] = x - w;
            if (lane == 31) sTot[i] = x;
        }
    }
    __syncthreads();
    uint32_t base[kPlanNV];
#pragma unroll
    for (int i = 0; i < kPlanNV; ++i) base[i] = sW[warp][i] + incl[i] - v[i];
    // (8 positions per round, their loads in flight together, as in the counting pass)
    for (int64_t tb = t0; tb < t1; tb += 8) {
        uint32_t key1[8], c0[8], c1[8], kw[8], hc[8][kMaxCluster];
#pragma unroll
        for (int j = 0; j < 8; ++j) key1[j] = tb + j < t1 ? ws.hkey[tb + j] : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t key = key1[j] ? key1[j] - 1u : 0u;
            c0[j] = key1[j] ? a.key_chunk_off[key] : 0u;
            c1[j] = key1[j] ? a.key_chunk_off[key + 1] : 0u;
            kw[j] = key1[j] ? a.key_word_off[key] : 0u;
#pragma unroll
            for (int g = 0; g < kMaxCluster; ++g) hc[j][g] = key1[j] ? ws.hcnt[(tb + j) * kMaxCluster + g] : 0u;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (!key1[j]) continue;
            const int64_t t = tb + j;
            const uint32_t sl = base[0];
            ws.hslot[t] = sl;
            ws.ukey[sl] = key1[j] - 1u;
            ws.uc0[sl] = c0[j];
            ws.uc1[sl] = c1[j];
            ws.ukwb[sl] = kw[j];
            ws.uchunk[sl] = base[1];
            uint32_t cls = 0;
#pragma unroll
            for (int g = 0; g < kMaxCluster; ++g) {
                const uint32_t c = hc[j][g];          // <= kGroup users
                ws.pinfo[(size_t)g * a.NU + sl] = c ? (base[2 + g] << 8) | c : 0u;
                ws.hpair[t * kMaxCluster + g] = base[2 + g];
                base[2 + g] += c;
                if (c) cls |= (1u + pair_class(c)) << (3 * g);
            }
            ws.ucls[sl] = cls;
            base[0] += 1u;
            base[1] += c1[j] - c0[j];
            ws.hkey[t] = 0u;
        }
    }
    __syncthreads();
    if (tid == 0) {
        const uint32_t nu = sTot[0];
        ws.header[0] = nu; ws.header[1] = 0; ws.header[2] = 0; ws.header[4] = 0; ws.header[6] = 0;
        ws.header[5] = sTot[1];                 // chunks of the union
        ws.uchunk[nu] = sTot[1];
        for (int g = 0; g < kMaxCluster; ++g) ws.header[8 + g] = sTot[2 + g];     // pairs of group g
    }
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
        const int u = i / (a.F * a.S), g = u / kGroup;
        const size_t hc = (size_t)t * kMaxCluster + g;
        const uint32_t pos = ws.hpair[hc] + atomicSub(&ws.hcnt[hc], 1u) - 1u;
        const int S = ws.ushift[u];
        const int32_t wf = (int32_t)__float2int_rn(ldexpf(ws.item_w[i], S));   // |wf| < 2^24
        ws.pairs[(size_t)g * a.gcap + pos] = ((uint32_t)wf << kPairUBits) | (uint32_t)(u % kGroup);
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
// A2 the entry stream: the union's cold postings, decoded ONCE per pass, as per-tile lists
// ------------------------------------------------------------------------------------------
// Level 1 (entry_bin): the union keys' chunks are decoded warp-cooperatively in key order (each
// chunk once; Alg. 2 l.355-357 with the chunk codec), every posting appended to the bin of its
// 1024-ad range; the lanes of a chunk that hit the same bin share one atomic (warp aggregation).
// Level 2 (entry_order): one CTA per bin orders the bin by (tile, pair-count class) with
// a shared-memory counting sort and expands it into the stream of every user group that queries
// the entry's key: entry = ad row << 24 | the group's first pair of the key << 8 | its pair count.
struct EntryArgs {
    const uint2* hdr;
    const uint32_t* payload;
    int64_t n_ads, n_pad;
    int bin_ads, n_bins, n_tiles;
    int64_t bin_cap;
    int G;                  // user groups of the pass
    int NU;                 // union slot capacity (pinfo row length)
};

// Work item = 16 consecutive chunks of the union (in slot order); each key's part is decoded by
// decode_unit16_warp (all headers, then all payload words in flight: two memory round trips per
// item); every posting is appended to its bin (lanes of a chunk hitting the same bin share one
// atomic).  (A two-pass variant with per-CTA bin segments measured 2.4x slower: its many small
// segments defeat write combining.)
// Bin entry = ad in bin << 20 | the slot's group class codes << 14 | union slot.
constexpr int kBinThreads = 256;
constexpr int kBinAdShift2 = 20, kBinClsShift = 14;
__global__ void __launch_bounds__(kBinThreads) entry_bin_kernel(EntryArgs e, Ws ws) {
    const int lane = threadIdx.x & 31;
    const uint32_t nu = __ldcg(&ws.header[0]), total = __ldcg(&ws.header[5]);
    const uint32_t n_items = (total + 15) / 16;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t R = (uint32_t)e.bin_ads;
    for (uint32_t item = gw; item < n_items; item += nw) {
        uint32_t g0 = item * 16;
        const uint32_t gend = min(total, g0 + 16);
        // the key holding chunk g0: last s with uchunk[s] <= g0 (warp 32-ary search)
        uint32_t lo = 0, hi = nu;
        while (hi - lo > 1) {
            const uint32_t step = (hi - lo + 31) / 32;
            const uint32_t pidx = lo + lane * step;
            const bool le = pidx < hi && __ldcg(&ws.uchunk[pidx]) <= g0;
            const uint32_t cntle = __popc(__ballot_sync(FULL, le));
            const uint32_t nlo = lo + (cntle - 1) * step;
            hi = min(hi, nlo + step);
            lo = nlo;
        }
        for (uint32_t s = lo; g0 < gend; ++s) {
            const uint32_t s_beg = __ldcg(&ws.uchunk[s]), s_end = __ldcg(&ws.uchunk[s + 1]);
            const uint32_t sub_end = min(gend, s_end);
            const uint32_t c0 = __ldcg(&ws.uc0[s]) + (g0 - s_beg);
            const uint32_t tag = (__ldcg(&ws.ucls[s]) << kBinClsShift) | s;
            decode_unit16_warp(e.hdr, e.payload, __ldcg(&ws.ukwb[s]), c0, c0 + (sub_end - g0), lane,
                               [&](uint32_t id, bool ok) {
                const uint32_t r = ok ? id / R : 0xFFFFFFFFu;
                const unsigned act = __ballot_sync(FULL, ok);
                if (ok) {
                    const unsigned peers = __match_any_sync(act, r);
                    const int leader = __ffs(peers) - 1;
                    uint32_t base = 0;
                    if (lane == leader) base = atomicAdd(&ws.bin_cnt[r], (uint32_t)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    const uint32_t pos = base + __popc(peers & ((1u << lane) - 1u));
                    ws.entries[(size_t)r * e.bin_cap + pos] = ((id - r * R) << kBinAdShift2) | tag;
                }
            });
            g0 = sub_end;
        }
    }
}

// Level 2: CTA = bin (8 tiles).  The bin is staged in shared memory when it fits (the common
// case), else read twice from L2: count per (group, tile, class), scan, claim the groups' ranges
// of the pool, scatter.
constexpr int kOrderCells = (kBinAds / kTileM) * kClasses;   // counters per group

__global__ void __launch_bounds__(kOrderThreads) entry_order_kernel(EntryArgs e, Ws ws) {
    extern __shared__ uint32_t smem_u[];
    __shared__ uint32_t cnt[kMaxCluster * kOrderCells];
    __shared__ uint32_t sN, sBase[kMaxCluster];
    uint32_t* buf = smem_u;                                 // [kOrderStage]
    const int r = blockIdx.x, tid = threadIdx.x, G = e.G;
    if (tid == 0) { sN = ws.bin_cnt[r]; ws.bin_cnt[r] = 0u; }   // left zero for the next pass
    for (int i = tid; i < kMaxCluster * kOrderCells; i += kOrderThreads) cnt[i] = 0;
    __syncthreads();
    const uint32_t n = sN;
    const bool staged = n <= (uint32_t)kOrderStage;
    const uint32_t* ent = ws.entries + (size_t)r * e.bin_cap;
    const uint32_t* pinfo = ws.pinfo;
    for (uint32_t i = tid; i < n; i += kOrderThreads) {
        const uint32_t v = __ldcs(&ent[i]);
        if (staged) buf[i] = v;
        const uint32_t a = v >> kBinAdShift2, cls = (v >> kBinClsShift) & 63u;
        for (int g = 0; g < G; ++g) {
            const uint32_t cc = (cls >> (3 * g)) & 7u;           // 0: no user of g, else 1 + class
            if (cc) atomicAdd(&cnt[g * kOrderCells + (a >> 7) * kClasses + cc - 1u], 1u);
        }
    }
    __syncthreads();
    // warp g: exclusive scan of group g's counters (lane = tile * kClasses + class), its range
    // claimed from the pool, the bounds of the bin's tiles
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int kCPL = kOrderCells / 32;                      // cells per lane
    static_assert(kOrderCells % 32 == 0, "whole cells per lane");
    if (warp < G) {
        uint32_t* c = cnt + warp * kOrderCells;
        uint32_t x[kCPL], run = 0;
#pragma unroll
        for (int k = 0; k < kCPL; ++k) { x[k] = c[lane * kCPL + k]; run += x[k]; }
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t tot = __shfl_sync(FULL, incl, 31);
        uint32_t acc = incl - run;
#pragma unroll
        for (int k = 0; k < kCPL; ++k) { c[lane * kCPL + k] = acc; acc += x[k]; }
        uint32_t base = 0;
        if (lane == 0) base = tot ? atomicAdd(&ws.header[6], tot) : 0u;
        base = __shfl_sync(FULL, base, 0);
        if (lane == 0) sBase[warp] = base;
        __syncwarp();
        constexpr int tpb = kBinAds / kTileM;                      // tiles per bin
        for (int tl = lane; tl < tpb; tl += 32) {
            const int64_t ti = (int64_t)r * tpb + tl;               // global tile
            if (ti >= (int64_t)e.n_tiles) break;
            const uint32_t tb = c[tl * kClasses];
            const uint32_t te = tl + 1 < tpb ? c[(tl + 1) * kClasses] : tot;
            ws.tbeg[(size_t)warp * e.n_tiles + ti] = base + tb;
            ws.tend[(size_t)warp * e.n_tiles + ti] = base + te;
        }
    }
    __syncthreads();
    for (uint32_t i = tid; i < n; i += kOrderThreads) {
        const uint32_t v = staged ? buf[i] : __ldcs(&ent[i]);
        const uint32_t a = v >> kBinAdShift2, cls = (v >> kBinClsShift) & 63u;
        const uint32_t sl = v & ((1u << kBinClsShift) - 1u);
        for (int g = 0; g < G; ++g) {
            const uint32_t cc = (cls >> (3 * g)) & 7u;
            if (cc) {
                const uint32_t pi = __ldg(&pinfo[(size_t)g * e.NU + sl]);
                const uint32_t pos = sBase[g] + atomicAdd(&cnt[g * kOrderCells + (a >> 7) * kClasses + cc - 1u], 1u);
                ws.gentries[pos] = ((a & (kTileM - 1)) << 24) | pi;
            }
        }
    }
}

// ------------------------------------------------------------------------------------------
// A3-A6b: the fused tensor-core kernel
// ------------------------------------------------------------------------------------------
// D[users x ads] = cold + U A^T (+ U_hot H^T), per CTA 128 users (TMEM lanes) x 128-ad tiles:
// the CTA's users are the MMA's A operand and stay resident in TMEM for the whole launch (loaded
// once), the ad tiles are B, streamed by TMA into a shared-memory ring (multicast to the cluster)
// and, for the hot keys, expanded from bit masks into fp16 one-hot blocks in the same ring.
struct GemmParams {
    int64_t n_ads, n_pad;
    uint32_t ad_begin;
    int n_kb, n_hb, pieces;
    int P;                  // users in this pass
    int n_tiles, tile_stride;
    int n_samp;
    int stages;             // max deep A ring stages (the kernel takes what the shared memory leaves)
    int smem_bytes;         // dynamic shared memory of the launch
    int acc_stages;         // TMEM accumulator stages (128 columns each)
    int u_cols;             // 16-bit columns of the pass's user tile U
    int64_t cap;
    int rerun;              // filter rerun: only flagged users; gated on header[2] | header[4]
    int dense;              // sample-mode variant: every score of the overflowed users (gated on header[4])
    const uint4* hot_mask;
    const void* A;          // the index's A [n_pad][d_pad] bf16 (L2 prefetch)
    Ws ws;
    uint32_t* err;
    int diag;               // A/B experiments (EBR_DIAG): 1 skip the cold scatter, 2 skip the epilogue work,
                            // 32 / 64 no TMEM load / store, 1024 no MMA issued, 2048 no one-hot writes,
                            // 32768 no A loads (results are wrong under any of these)
    int NU;                 // union slot capacity of the pass (toff row length - 1)
    int gcap;               // pair capacity of a group's list
    int n_tiles_all;        // tiles of the inventory (row length of the group streams' tile bounds)
    int deep_smem;          // the users' deep operand in shared memory (SS MMA), freeing TMEM for a third
                            // accumulator stage; else in TMEM with the hot pieces (TS MMA)
    int pair;               // 2-group pass as a CTA pair: tcgen05.mma.cta_group::2 (M = 256 users), each
                            // CTA staging half of every ad tile and one-hot block
};

// the producer's and the MMA issuer's waits: sleeping (default) or spinning (EBR_DIAG & 16)
__device__ __forceinline__ void crit_wait(uint64_t* bar, uint32_t parity, int diag) {
    if (diag & 256) mbar_wait_poll(bar, parity);
    else if (diag & 16) mbar_wait(bar, parity);
    else mbar_wait_sleep(bar, parity);
}

// role cycle accounting (EBR_DIAG & 4): prof[slot] += clock64 delta, from one thread per role
#define EBR_PROF_T0 const long long _pt0 = (p.diag & 4) ? clock64() : 0
#define EBR_PROF_ADD(slot) do { if ((p.diag & 4)) atomicAdd(&p.ws.prof[slot], (unsigned long long)(clock64() - _pt0)); } while (0)

template <int MODE, bool PAIR>   // MODE 0: sample (store s; dense: all scores of overflowed users), 1: filter
                                 // (append keys >= theta); PAIR: the 2-group CTA pair (cta_group::2)
__global__ void __launch_bounds__(kGemmThreads, 1)
score_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmA64, const GemmParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // gated launches (uniform over the grid): nothing to redo
    if (MODE == 1 && p.rerun && (*(volatile uint32_t*)&p.ws.header[2] | *(volatile uint32_t*)&p.ws.header[4]) == 0u)
        return;
    if (MODE == 0 && p.dense && *(volatile uint32_t*)&p.ws.header[4] == 0u) return;
    // 1024-byte alignment (SW128 tiles) by an integer offset into the shared array: the pointers
    // below stay in the shared state space (LDS/STS/ATOMS, not generic accesses)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long _pk0 = (p.diag & 4) ? clock64() : 0;
    const uint32_t rank = tc::cluster_ctarank();
    uint32_t csize;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    const uint32_t cid = tc::cluster_id_x(), ncl = tc::cluster_count_x();
    const uint16_t mc_mask = (uint16_t)((1u << csize) - 1u);
    const int g = (int)rank;                         // this CTA's user group
    const int nu = min(kGroup, p.P - g * kGroup);    // valid users
    // TMEM columns of the users' A operand: the hot pieces, and the deep part unless it is in smem
    const int a_cols = 32 * ((p.deep_smem ? 0 : p.n_kb) + p.n_hb * p.pieces);
    const int hot_col0 = p.deep_smem ? 0 : 32 * p.n_kb;     // TMEM column of the first hot piece
    const int nst = p.acc_stages;
    // deep A ring stages: what the shared memory leaves next to the fixed part and the largest
    // group's pairs of the pass (the same in every CTA of the cluster: the multicast writes the
    // ring stages at the same offsets)
    uint32_t n_gp_max = 0;
    for (uint32_t r = 0; r < csize; ++r) n_gp_max = max(n_gp_max, __ldcg(&p.ws.header[8 + r]));
    constexpr bool pair = PAIR;                     // CTA pair: this CTA stages ads 64 rank .. 64 rank + 63 of a tile
    const uint32_t sb = pair ? kBlockBytes / 2 : kBlockBytes;               // ring stage bytes of this CTA
    const size_t user_bytes = p.deep_smem ? (size_t)p.n_kb * kBlockBytes : 0;   // [n_kb][128 users x 128 B]
    // the group's pairs live in shared memory when they fit next to a minimal ring (one tile's deep
    // blocks + 1), else the scatter reads them from L2 (the same in both CTAs of a cluster)
    // (pair mode: the hot ring reservation's second half is free; a second fixed-point tile is
    // carved when it fits next to the pairs and a ring of >= 3 tiles' deep blocks)
    constexpr size_t kAccBytes = (size_t)kGroup * kAccPitch * 4;
    const size_t spare = pair ? (size_t)kHotStages * kBlockBytes / 2 : 0;
    size_t avail = (size_t)p.smem_bytes - 1024 - score_smem_fixed() - user_bytes + spare;
    const bool dbl = pair && !(p.diag & 512) &&
                     avail >= kAccBytes + (size_t)n_gp_max * 4 + (size_t)3 * p.n_kb * sb;
    if (dbl) avail -= kAccBytes;
    const bool pairs_smem = avail >= (size_t)(p.n_kb + 1) * sb + (size_t)n_gp_max * 4;
    const int nring = (int)min((size_t)kMaxStages, (avail - (pairs_smem ? (size_t)n_gp_max * 4 : 0)) / sb);

    unsigned char* sUser = smem;                                            // users' deep operand (deep_smem)
    unsigned char* sRing = smem + user_bytes;                                            // [nring][128 (pair: 64) ads x 128 B] deep blocks of A
    unsigned char* sHot = sRing + (size_t)nring * sb;                       // [kHotStages][128 (64) ads x 128 B] one-hot blocks
    int32_t* sAcc = reinterpret_cast<int32_t*>(sHot + (size_t)kHotStages * kBlockBytes - spare);   // [128 users][kAccPitch]
    uint32_t* sEnt = reinterpret_cast<uint32_t*>(sAcc + kGroup * kAccPitch);  // [2][kEntHdr + kEntBuf]
    uint4* sLut = reinterpret_cast<uint4*>(sEnt + 2 * (kEntHdr + kEntBuf));  // [256] byte -> 8 fp16 {0, 1}
    uint64_t* bars = reinterpret_cast<uint64_t*>(sLut + 256);
    uint64_t* full = bars;                          // [kMaxStages] A ring
    uint64_t* empty = full + kMaxStages;
    uint64_t* hfull = empty + kMaxStages;           // [kHotStages] hot ring
    uint64_t* hempty = hfull + kHotStages;
    uint64_t* tfull = hempty + kHotStages;          // [kMaxAccStages] TMEM accumulator stages
    uint64_t* tempty = tfull + kMaxAccStages;
    uint64_t* wready = tempty + kMaxAccStages;      // [kMaxAccStages] cold tile stored into the stage
    uint64_t* efull = wready + kMaxAccStages;       // [2] entry buffers
    uint64_t* eempty = efull + 2;
    uint64_t* aready = eempty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aready + 1);
    uint64_t* sTheta = reinterpret_cast<uint64_t*>(tmem_slot + 2);          // [kGroup]
    float* sThetaS = reinterpret_cast<float*>(sTheta + kGroup);             // [kGroup]
    float* sScale = sThetaS + kGroup;                                       // [kGroup]
    int* sDense = reinterpret_cast<int*>(sScale + kGroup);                  // [kGroup] dense slot or -1
    const uint32_t n_gp = __ldcg(&p.ws.header[8 + g]);
    unsigned char* after = reinterpret_cast<unsigned char*>(sDense + kGroup);
    after += (16u - (smem_u32(after) & 15u)) & 15u;
    int32_t* sAcc2 = dbl ? reinterpret_cast<int32_t*>(after) : nullptr;      // second fixed-point tile (dbl)
    uint32_t* sPairs = reinterpret_cast<uint32_t*>(after + (dbl ? kAccBytes : 0));   // [n_gp] the group's pairs

    if (tid == 0) {
        for (int s = 0; s < nring; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], (pair || (p.diag & 8)) ? 1u : csize); }
        for (int s = 0; s < 2; ++s) { mbar_init(&efull[s], 1); mbar_init(&eempty[s], 1); }
        for (int s = 0; s < kHotStages; ++s) { mbar_init(&hfull[s], pair ? 2u : 1u); mbar_init(&hempty[s], 1); }
        for (int s = 0; s < kMaxAccStages; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kEpiWarps);
        }
        for (int s = 0; s < kMaxAccStages; ++s) mbar_init(&wready[s], pair ? 2u : 1u);
        mbar_init(aready, pair ? 8u : 4u);
        fence_mbar_init();
    }
    if (warp == 2) {
        if (pair) tc::tmem_alloc2(tmem_slot, 512);
        else tc::tmem_alloc(tmem_slot, 512);
    }
    for (int i = tid; i < kGroup * kAccPitch / 4; i += kGemmThreads) {
        reinterpret_cast<int4*>(sAcc)[i] = make_int4(0, 0, 0, 0);
        if (dbl) reinterpret_cast<int4*>(sAcc2)[i] = make_int4(0, 0, 0, 0);
    }
    for (int b = tid; b < 256; b += kGemmThreads) {
        auto h2 = [b](int k) { return ((b >> k) & 1 ? 0x3C00u : 0u) | ((b >> (k + 1)) & 1 ? 0x3C000000u : 0u); };
        sLut[b] = make_uint4(h2(0), h2(2), h2(4), h2(6));
    }
    if (pairs_smem)
        for (uint32_t i = tid; i < n_gp; i += kGemmThreads) sPairs[i] = __ldcg(&p.ws.pairs[(size_t)g * p.gcap + i]);
    const uint32_t* __restrict__ gPairs = p.ws.pairs + (size_t)g * p.gcap;
    for (int i = tid; i < kGroup; i += kGemmThreads) {
        const int u = g * kGroup + i;
        const bool ok = i < nu;
        sScale[i] = ok ? p.ws.uscale[u] : 0.f;
        const uint32_t fl = ok ? __ldcg(&p.ws.uflags[u]) : 0u;
        sDense[i] = (MODE == 0 && p.dense && (fl & kFlagOverflow)) ? (int)(fl >> 8) : -1;
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
            // ---------------- TMA producer: the deep K blocks of every ad tile ----------------
            tc::tma_prefetch(&tmA);
            const uint64_t pol = tc::policy_evict_first();   // A is streamed once per pass
            uint32_t gb = 0;
            int it = 0;
            const size_t trow = (size_t)g * p.n_tiles_all;
            const uint32_t tile_bytes = (uint32_t)(kTileM * p.n_kb * 128);     // a tile's rows of A (contiguous)
            const unsigned char* Abase = reinterpret_cast<const unsigned char*>(p.A);
            // L2 prefetch kPrefetchTiles ahead of the TMA loads: the ring's loads then hit L2 (the
            // HBM latency of a multicast stage exceeds what the ring's depth covers)
            if (rank == 0)
                for (int k = 0; k < kPrefetchTiles; ++k) {
                    const int tp = (int)cid + k * (int)ncl;
                    if (tp < p.n_tiles) tc::bulk_prefetch_l2(Abase + (size_t)tp * p.tile_stride * tile_bytes, tile_bytes);
                }
            // tile bounds of the group stream, loaded two tiles ahead (never on the issue path)
            auto load_qb = [&](int tt, uint32_t (&qb)[2]) {
                if (tt < p.n_tiles) {
                    const size_t ti = trow + (size_t)tt * p.tile_stride;
                    qb[0] = __ldcg(&p.ws.tbeg[ti]);
                    qb[1] = __ldcg(&p.ws.tend[ti]);
                }
            };
            uint32_t qbA[2] = {}, qbB[2] = {};
            load_qb((int)cid, qbA);
            load_qb((int)cid + (int)ncl, qbB);
            for (int t = (int)cid; t < p.n_tiles; t += (int)ncl, ++it) {
                const int row0 = t * p.tile_stride * kTileM;
                uint32_t qb[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) { qb[q] = qbA[q]; qbA[q] = qbB[q]; }
                load_qb(t + 2 * (int)ncl, qbB);
                if (rank == 0) {
                    const int tp = t + kPrefetchTiles * (int)ncl;
                    if (tp < p.n_tiles) tc::bulk_prefetch_l2(Abase + (size_t)tp * p.tile_stride * tile_bytes, tile_bytes);
                }
                {
                    // this CTA's cold entries of the tile (contiguous in its group's stream) into
                    // entry buffer it % 2 by one bulk copy; header = quarter bounds relative to the
                    // copied base, and the number of entries copied
                    const int eb = it & 1;
                    if (it >= 2) crit_wait(&eempty[eb], ((it >> 1) - 1) & 1, p.diag);
                    uint32_t* hdr = sEnt + eb * (kEntHdr + kEntBuf);
                    if (p.diag & 1) qb[1] = qb[0];
                    const uint32_t base = qb[0] & ~3u;                          // 16-byte aligned source
                    const uint32_t ncopy = min((qb[1] - base + 3u) & ~3u, (uint32_t)kEntBuf);
                    hdr[0] = qb[0] - base;
                    hdr[1] = qb[1] - base;
                    hdr[2] = base;
                    hdr[3] = ncopy;
                    if (ncopy) {
                        mbar_arrive_expect_tx(&efull[eb], ncopy * 4);
                        bulk_g2s(hdr + kEntHdr, p.ws.gentries + base, ncopy * 4, &efull[eb]);
                    } else {
                        mbar_arrive(&efull[eb]);
                    }
                }
                for (int kb = 0; kb < p.n_kb; ++kb, ++gb) {
                    const uint32_t slot = gb % nring, round = gb / nring;
                    if (round > 0) { EBR_PROF_T0; crit_wait(&empty[slot], (round - 1) & 1, p.diag); EBR_PROF_ADD(0); }
                    if (pair) {
                        // each CTA its 64 rows; both halves' bytes complete on the leader's barrier
                        if (rank == 0) mbar_arrive_expect_tx(&full[slot], (uint32_t)kBlockBytes);
                        tc::tma_load_2d_pair(sRing + (size_t)slot * sb, &tmA64, kb * kBlockK, row0 + 64 * (int)rank,
                                             tc::cluster_addr(&full[slot], 0), pol);
                        continue;
                    }
                    if (p.diag & 32768) { mbar_arrive(&full[slot]); continue; }   // (A/B: no A loads)
                    mbar_arrive_expect_tx(&full[slot], (uint32_t)kBlockBytes);
                    if (csize == 1 || (p.diag & 8))
                        tc::tma_load_2d_hint(sRing + (size_t)slot * kBlockBytes, &tmA, kb * kBlockK, row0, &full[slot], pol);
                    else if (rank == 0)
                        tc::tma_load_2d_mc(sRing + (size_t)slot * kBlockBytes, &tmA, kb * kBlockK, row0, &full[slot],
                                           mc_mask, pol);
                }
            }
            // every remote arrival into this CTA's ring barriers has landed before it exits
            for (uint32_t k = 0; k < (uint32_t)nring && k < gb; ++k) {
                const uint32_t q = gb - 1 - k;
                crit_wait(&empty[q % nring], (q / nring) & 1, p.diag);
            }
        }
    } else if (warp == 1) {
        if (!pair || rank == 0) {   // (pair: the leader issues for both CTAs; the whole warp, one elected lane issues)
            // ---------------- MMA issuer ----------------
            // The accumulator stage already holds the tile's cold wide term (stored by the wide
            // warps), so every MMA accumulates: D = cold + U A^T + U_hot (one-hot)^T.
            const uint32_t idb = pair ? tc::idesc_bf16_m256(kTileM) : tc::idesc_bf16_m128(kTileM);
            const uint32_t idh = pair ? tc::idesc_f16_m256(kTileM) : tc::idesc_f16_m128(kTileM);
            // waits on barriers that receive the peer's arrivals take cluster-scope acquire
            auto pwait = [&](uint64_t* bar, uint32_t parity) {
                if (pair) tc::mbar_wait_cluster(bar, parity);
                else crit_wait(bar, parity, p.diag);
            };
            auto mma4 = [&](uint32_t d, uint32_t a, uint64_t b, uint32_t id) {   // one 64-wide K block
                if (pair) tc::umma2_f16_ts_x4_e(d, a, b, id, 1u);
                else tc::umma_f16_ts_x4_e(d, a, b, id, 1u);
            };
            auto commit_all = [&](uint64_t* bar) {       // the arrival every consumer of the stage waits for
                if (pair) tc::umma2_commit_mc_e(bar, (uint16_t)3);
                else tc::umma_commit_e(bar);
            };
            pwait(aready, 0);                               // users' A operand in TMEM (both CTAs)
            tc::fence_after();
            int it = 0;
            uint32_t gb = 0, hb = 0;
            for (int t = (int)cid; t < p.n_tiles; t += (int)ncl, ++it) {
                const int st = it % nst;
                { EBR_PROF_T0; pwait(&wready[st], (it / nst) & 1); if (lane == 0) EBR_PROF_ADD(1); }
                tc::fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(a_cols + st * kTileM);
                for (int kb = 0; kb < p.n_kb; ++kb, ++gb) {
                    const uint32_t slot = gb % nring;
                    if (!(p.diag & 128)) { EBR_PROF_T0; crit_wait(&full[slot], (gb / nring) & 1, p.diag); if (lane == 0) EBR_PROF_ADD(2); }
                    tc::fence_after();
                    const uint64_t db0 = tc::sdesc_sw128(sRing + (size_t)slot * sb);
                    if (p.deep_smem) {
                        const uint64_t da0 = tc::sdesc_sw128(sUser + (size_t)kb * kBlockBytes);
#pragma unroll
                        for (int k = 0; k < kBlockK / 16; ++k) {
                            if (pair) tc::umma2_f16_ss_e(d_tmem, da0 + (uint64_t)(k * 2), db0 + (uint64_t)(k * 2), idb, 1u);
                            else tc::umma_f16_e(d_tmem, da0 + (uint64_t)(k * 2), db0 + (uint64_t)(k * 2), idb, 1u);
                        }
                    } else if (!(p.diag & 1024)) {                // (A/B: no MMA issued)
                        static_assert(kBlockK == 64, "mma4 issues four K=16 steps");
                        mma4(d_tmem, tmem_base + (uint32_t)(kb * 32), db0, idb);
                    }
                    if (pair) tc::umma2_commit_mc_e(&empty[slot], (uint16_t)3);
                    else if (csize == 1 || (p.diag & 8)) tc::umma_commit_e(&empty[slot]);
                    else tc::umma_commit_mc_e(&empty[slot], mc_mask);
                }
                for (int h = 0; h < p.n_hb; ++h, ++hb) {
                    const uint32_t hs = hb % kHotStages;
                    { EBR_PROF_T0; pwait(&hfull[hs], (hb / kHotStages) & 1); if (lane == 0) EBR_PROF_ADD(2); }
                    tc::fence_after();
                    const uint64_t db0 = tc::sdesc_sw128(sHot + (size_t)hs * sb);
                    for (int pc = 0; pc < ((p.diag & 1024) ? 0 : p.pieces); ++pc) {
                        const uint32_t ac = (uint32_t)(hot_col0 + 32 * (h * p.pieces + pc));
                        mma4(d_tmem, tmem_base + ac, db0, idh);
                    }
                    commit_all(&hempty[hs]);
                }
                commit_all(&tfull[st]);
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ---------------- hot warps: the tile's hot-key one-hot fp16 K block(s) ----------------
        // Thread hw owns ad rows hw and hw + 64; each row's 64-key block is 8 chunks of 16 B written
        // in the TMA 128B-swizzle layout (chunk c of row r at (c ^ (r & 7)) * 16).  The masks of
        // the next tile are loaded while this one is written.
        if (p.n_hb) {
            // (pair: this CTA's 64 ad rows of the tile, rows 64 rank ..; thread hw owns row hw)
            const int hw = tid - 64;
            const int nrows = pair ? 1 : 2;
            const int rbase = pair ? 64 * (int)rank : 0;
            const uint32_t hfull_leader = pair ? tc::cluster_addr(&hfull[0], 0) : 0u;
            uint4 hm[2] = {}, hn[2] = {};
            auto load = [&](int tt, uint4 (&m)[2]) {
                if (tt < p.n_tiles) {
                    const int64_t tw = (int64_t)tt * p.tile_stride;
                    m[0] = __ldg(&p.hot_mask[tw * kTileM + rbase + hw]);
                    if (!pair) m[1] = __ldg(&p.hot_mask[tw * kTileM + hw + 64]);
                }
            };
            load((int)cid, hn);
            uint32_t hb = 0;
            for (int t = (int)cid; t < p.n_tiles; t += (int)ncl) {
                hm[0] = hn[0];
                hm[1] = hn[1];
                load(t + (int)ncl, hn);
                for (int h = 0; h < p.n_hb; ++h, ++hb) {
                    const uint32_t hs = hb % kHotStages, round = hb / kHotStages;
                    if (round > 0) { EBR_PROF_T0; crit_wait(&hempty[hs], (round - 1) & 1, p.diag); if (hw == 0) EBR_PROF_ADD(3); }
                    for (int rr = 0; rr < ((p.diag & 2048) ? 0 : nrows); ++rr) {   // (A/B: no one-hot writes)
                        const int row = hw + rr * 64;
                        const uint64_t bits = h == 0 ? ((uint64_t)hm[rr].y << 32 | hm[rr].x)
                                                     : ((uint64_t)hm[rr].w << 32 | hm[rr].z);
                        unsigned char* rowp = sHot + (size_t)hs * sb + (size_t)row * 128;
#pragma unroll
                        for (int c = 0; c < 8; ++c) {                  // 16-byte chunk: keys 8c .. 8c+7
                            const uint32_t byte = (uint32_t)(bits >> (8 * c)) & 0xFFu;
                            *reinterpret_cast<uint4*>(rowp + ((c ^ (row & 7)) << 4)) = sLut[byte];
                        }
                    }
                    tc::fence_proxy_async_smem();
                    tc::named_bar_sync(2, 64);
                    if (hw == 0) {
                        if (pair) tc::mbar_arrive_remote(hfull_leader + (uint32_t)(hs * 8));
                        else mbar_arrive(&hfull[hs]);
                    }
                }
            }
        }
    } else if (warp >= kWideWarp0 && warp < kEpiWarp0) {
        // ---------------- wide warps: users' A operand once, then the cold scatter ----------------
        const int wt = tid - kWideWarp0 * 32;
        if (warp < kWideWarp0 + 4) {
            // U row of this user -> TMEM A columns (two 16-bit K elements per 32-bit column)
            const int q = warp & 3;                      // TMEM lane quadrant = users 32q .. 32q + 31
            const int urow = q * 32 + lane;
            const uint32_t* urow_p = reinterpret_cast<const uint32_t*>(p.ws.U) +
                                     (size_t)(g * kGroup + urow) * (p.u_cols / 2);
            const int src0 = p.deep_smem ? 32 * p.n_kb : 0;   // U columns (32-bit) going to TMEM
            if (p.deep_smem) {
                // deep K blocks -> shared memory in the 128B-swizzle K-major layout (row urow, 16-byte
                // chunk c of a block at (c ^ (urow & 7)) * 16)
                for (int kb = 0; kb < p.n_kb; ++kb)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint4 v = *reinterpret_cast<const uint4*>(urow_p + kb * 32 + 4 * c);
                        *reinterpret_cast<uint4*>(sUser + (size_t)kb * kBlockBytes + (size_t)urow * 128 +
                                                  ((c ^ (urow & 7)) << 4)) = v;
                    }
                tc::fence_proxy_async_smem();
            }
            for (int c0 = 0; c0 < a_cols; c0 += 32) {
                uint32_t v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __ldcg(&urow_p[src0 + c0 + j]);
                tc::tmem_st32_nowait(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
            }
            tc::tmem_wait_st();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) {
                if (pair) tc::mbar_arrive_remote(tc::cluster_addr(aready, 0));
                else mbar_arrive(aready);
            }
        }
        // Per tile: its entries (ad row, the slot's first pair, pair count) of this CTA's group
        // stream (ordered by pair-count class), staged in shared memory by the producer's bulk
        // copy; each pair (user, w~ 2^S) is
        // added to the tile [128 users][128 ads] with a native 32-bit shared atomic (exact,
        // order-free; Alg. 2 l.358).  Then the tile is converted once to fp32 and stored into the
        // TMEM accumulator stage, which the tensor core accumulates onto.
        const uint32_t* __restrict__ entries = p.ws.gentries;
        const int q = warp & 3;                          // TMEM lane quadrant = users 32q .. 32q + 31
        const int cj = (warp - kWideWarp0) >> 2;         // this warp's 32-ad column chunk (store phase)
        const int urow = q * 32 + lane;
        const float uscale = sScale[urow];
        // scatter of tile `it`'s entries into the fixed-point tile `acc`
        auto scatter = [&](int it, int32_t* acc) {
            const int eb = it & 1;
            { EBR_PROF_T0; crit_wait(&efull[eb], (it >> 1) & 1, p.diag); if (wt == 0) EBR_PROF_ADD(11); }
            const long long _pc0 = (p.diag & 4) ? clock64() : 0;
            const uint32_t* hdr = sEnt + eb * (kEntHdr + kEntBuf);
            const uint32_t* ebuf = hdr + kEntHdr;
            const uint32_t ebase = hdr[2], ncopy = hdr[3];
            const uint32_t e0 = hdr[0], e1 = hdr[1];
            for (uint32_t ei = e0 + wt; ei < e1; ei += kWideThreads) {
                const uint32_t en = ei < ncopy ? ebuf[ei] : __ldcs(&entries[ebase + ei]);
                const uint32_t a = en >> 24, lo = (en >> 8) & 0xFFFFu, c = en & 0xFFu;
                // (a warp's entries share a pair-count class: little divergence in this loop)
#pragma unroll 2
                for (uint32_t qq = lo; qq < lo + c; ++qq) {
                    const uint32_t pr = pairs_smem ? sPairs[qq] : __ldg(&gPairs[qq]);
                    atomicAdd(&acc[(pr & (kGroup - 1)) * kAccPitch + a], (int32_t)pr >> kPairUBits);
                }
            }
            tc::named_bar_sync(1, kWideThreads);
            if (wt == 0) mbar_arrive(&eempty[eb]);      // entry buffer consumed
            if ((p.diag & 4) && wt == 0) atomicAdd(&p.ws.prof[4], (unsigned long long)(clock64() - _pc0));
        };
        // tile `it`'s cold term: read-and-clear `acc`, fp32, into the TMEM stage, MMA released
        auto store = [&](int it, int32_t* acc) {
            const int st = it % nst;
            // the accumulator stage is free once the epilogue drained it (nst tiles ago)
            if (it >= nst) { EBR_PROF_T0; crit_wait(&tempty[st], ((it / nst) - 1) & 1, p.diag); if (wt == 0) EBR_PROF_ADD(5); }
            const long long _ps0 = (p.diag & 4) ? clock64() : 0;
            tc::fence_after();
            {
                // this user's 32 ads of the tile: fixed point -> fp32 (the one rounding), zeroed;
                // read-and-clear in one shared-memory pass by 64-bit atomic exchanges (half the
                // traffic of a load + a zero store)
                unsigned long long* src = reinterpret_cast<unsigned long long*>(acc + urow * kAccPitch + cj * 32);
                uint32_t f[32];
#pragma unroll
                for (int v2 = 0; v2 < 16; ++v2) {
                    const unsigned long long v = atomicExch(&src[v2], 0ull);
                    f[2 * v2 + 0] = __float_as_uint((float)(int32_t)(uint32_t)v * uscale);
                    f[2 * v2 + 1] = __float_as_uint((float)(int32_t)(uint32_t)(v >> 32) * uscale);
                }
                if (!(p.diag & 64))                            // (A/B: no TMEM store)
                    tc::tmem_st32_nowait(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a_cols + st * kTileM + cj * 32), f);
            }
            tc::tmem_wait_st();
            tc::fence_before();
            tc::named_bar_sync(1, kWideThreads);
            if (wt == 0) {
                if (pair) tc::mbar_arrive_remote(tc::cluster_addr(&wready[st], 0));
                else mbar_arrive(&wready[st]);
            }
            if ((p.diag & 4) && wt == 0) atomicAdd(&p.ws.prof[6], (unsigned long long)(clock64() - _ps0));
        };
        const int n_my = (int)cid < p.n_tiles ? (p.n_tiles - (int)cid + (int)ncl - 1) / (int)ncl : 0;
        if (sAcc2) {
            // two fixed-point tiles: tile it + 1 is scattered while tile it waits for its TMEM stage
            if (n_my > 0) scatter(0, sAcc);
            for (int it = 0; it < n_my; ++it) {
                if (it + 1 < n_my) scatter(it + 1, (it & 1) ? sAcc : sAcc2);
                store(it, (it & 1) ? sAcc2 : sAcc);
            }
        } else {
            for (int it = 0; it < n_my; ++it) {
                scatter(it, sAcc);
                store(it, sAcc);
            }
        }
    } else if (warp >= kEpiWarp0) {
        // ---------------- epilogue: TMEM -> s, kappa, sample store / filter ----------------
        // thread = one user (TMEM lane) x half of the tile's ads (two 32-column chunks)
        const int e = warp - kEpiWarp0;
        const int q = warp & 3;
        const int ul = q * 32 + lane;                    // CTA-local user
        const int u = g * kGroup + ul;                   // pass user
        const bool uok = ul < nu;
        const int hf = e >> 2;
        float thS = 0.f;
        uint64_t th = 0;
        int dslot = -1;
        if (MODE == 1) { thS = sThetaS[ul]; th = sTheta[ul]; }
        else dslot = sDense[ul];
        int it = 0;
        for (int t = (int)cid; t < p.n_tiles; t += (int)ncl, ++it) {
            const int st = it % nst;
            const int64_t a0 = (int64_t)t * p.tile_stride * kTileM;   // shard-local first ad of the tile
            { EBR_PROF_T0; crit_wait(&tfull[st], (it / nst) & 1, p.diag); if (warp == kEpiWarp0 && lane == 0) EBR_PROF_ADD(7); }
            tc::fence_after();
            const long long _pe0 = (p.diag & 4) ? clock64() : 0;
#pragma unroll 1
            for (int ch = 0; ch < 2; ++ch) {
                const int qi = hf * 2 + ch;              // tile quarter = 32-column chunk
                const int c = qi * 32;
                uint32_t r[32];
                if (!(p.diag & 32))                            // (A/B: no TMEM read)
                    tc::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a_cols + st * kTileM + c), r);
                if (ch == 1) {
                    // the stage's last columns of this warp are in registers: hand the stage back
                    // now (the MMA of tile it + nst can start while this chunk is filtered)
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[st]);
                }
                if (p.diag & (2 | 32)) continue;
                const int64_t ac = a0 + c;
                const int nval = (int)min((int64_t)32, max((int64_t)0, p.n_ads - ac));   // valid ads in the chunk
                if (MODE == 0) {
                    if (p.dense) {
                        if (dslot >= 0) {
                            float* dst = p.ws.dense + (size_t)dslot * p.n_pad + ac;
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                float s = __uint_as_float(r[j]);
                                if (s == 0.f) s = 0.f;                       // -0 -> +0 (R14)
                                dst[j] = j < nval ? s : __int_as_float(0xFF800000);
                            }
                        }
                    } else if (uok) {
                        float4* dst = reinterpret_cast<float4*>(p.ws.samp + (size_t)u * p.n_samp + (int64_t)t * kTileM + c);
#pragma unroll
                        for (int j4 = 0; j4 < 8; ++j4) {
                            float o[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                float s = __uint_as_float(r[4 * j4 + k]);
                                if (s == 0.f) s = 0.f;                       // -0 -> +0 (R14)
                                o[k] = (4 * j4 + k) < nval ? s : __int_as_float(0xFF800000);
                            }
                            dst[j4] = make_float4(o[0], o[1], o[2], o[3]);
                        }
                    }
                } else {
                    // early out on the chunk's maximum (almost every chunk has no candidate)
                    float mx = __uint_as_float(r[0]);
#pragma unroll
                    for (int j = 1; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r[j]));
                    uint32_t pass = 0;
                    if (mx >= thS && uok) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) pass |= (__uint_as_float(r[j]) >= thS ? 1u : 0u) << j;
                        pass &= nval >= 32 ? 0xFFFFFFFFu : ((1u << nval) - 1u);
                    }
                    // exact key compare, then this user's appends (one atomic per thread and chunk)
                    uint32_t take = 0;
                    if (pass) {
#pragma unroll 1
                        for (uint32_t m = pass; m; m &= m - 1u) {
                            const int j = __ffs(m) - 1;
                            float s = 0.f;
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) s = (jj == j) ? __uint_as_float(r[jj]) : s;
                            if (s == 0.f) s = 0.f;                       // -0 -> +0 (R14)
                            if (kappa_of(s, p.ad_begin + (uint32_t)(ac + j)) >= th) take |= 1u << j;
                        }
                    }
                    if (take) {
                        uint32_t pos = atomicAdd(&p.ws.cand_count[u], (uint32_t)__popc(take));
                        for (uint32_t m = take; m; m &= m - 1u, ++pos) {
                            const int j = __ffs(m) - 1;
                            float s = 0.f;
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj) s = (jj == j) ? __uint_as_float(r[jj]) : s;
                            if (s == 0.f) s = 0.f;
                            if (pos < p.cap) p.ws.cand[(size_t)u * p.cap + pos] = kappa_of(s, p.ad_begin + (uint32_t)(ac + j));
                        }
                    }
                }
            }
            if ((p.diag & 4) && warp == kEpiWarp0 && lane == 0) atomicAdd(&p.ws.prof[8], (unsigned long long)(clock64() - _pe0));
        }
    }
    __syncwarp();
    tc::fence_before();
    __syncthreads();
    tc::cluster_sync_all();
    if ((p.diag & 4) && tid == 0) {
        atomicAdd(&p.ws.prof[9], 1ull);
        atomicAdd(&p.ws.prof[10], (unsigned long long)(clock64() - _pk0));
    }
    if (warp == 2) {
        if (pair) tc::tmem_dealloc2(tmem_base, 512);
        else tc::tmem_dealloc(tmem_base, 512);
    }
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
                                                                int P, int scap, int rerun, int64_t n_pad,
                                                                int64_t sstride) {
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
    const int64_t stride = dense ? 1 : sstride;
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

// EBR_TRACE=1: synchronise and report after every launch of the batched path (debugging only)
static void trace(cudaStream_t st, const char* what) {
    static const bool on = getenv("EBR_TRACE") != nullptr;
    if (!on) return;
    const cudaError_t e = cudaStreamSynchronize(st);
    fprintf(stderr, "[ebr] %s: %s\n", what, cudaGetErrorString(e));
}

struct Tuning {
    int n_hb, pieces;
};

static Tuning tuning(const ebr_index* idx) {
    Tuning t;
    t.n_hb = std::min(kMaxHotBlocks, idx->n_hot / 64);     // up to 128 hot keys: 89 % of C3's hits
    t.pieces = 2;
    if (const char* e = getenv("EBR_HOT_BLOCKS")) t.n_hb = std::max(0, std::min(t.n_hb, atoi(e)));
    if (getenv("EBR_NO_HOT")) t.n_hb = 0;                 // every key through the compressed lists
    if (const char* e = getenv("EBR_HOT_PIECES")) t.pieces = std::max(1, std::min(2, atoi(e)));
    return t;
}

static size_t gemm_smem(const Layout& L, int stages, int user_blocks = 0) {
    return 1024 + (size_t)(stages + user_blocks) * kBlockBytes + score_smem_fixed() + (size_t)L.gcap * 4;
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
    return ((batch + P - 1) / P) * 13;
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
    // score_kernel) plus one of lookahead; TMEM: the users' A operand (32 columns per 64 K) and
    // >= 2 accumulator stages of 128 columns; hot blocks are dropped until both fit
    int stages = 0, acc_stages = 0;
    // the users' deep operand in shared memory (SS MMA, a third TMEM accumulator stage): opt-in
    // (EBR_DEEP_SMEM=1, read per call so a test can exercise it); measured no faster (the ring loses
    // two stages), DESIGN.md §6.2
    const char* ds_env = getenv("EBR_DEEP_SMEM");
    const bool deep_smem = ds_env != nullptr && atoi(ds_env) != 0;
    for (; tu.n_hb >= 0; --tu.n_hb) {
        acc_stages = std::min(kMaxAccStages, (512 - 32 * ((deep_smem ? 0 : n_kb) + tu.n_hb * tu.pieces)) / kTileM);
        if (acc_stages < 2) continue;
        stages = n_kb + 1;          // the minimum with the worst-case pairs; the kernel takes more
        if (gemm_smem(L, stages, deep_smem ? n_kb : 0) - (size_t)L.gcap * 4 <= (size_t)max_smem) break;
    }
    if (tu.n_hb < 0) return set_error(EBR_EUNSUPPORTED, "batched path: d=%d does not fit shared memory / TMEM", idx->d);
    const size_t smem = (size_t)max_smem;
    CUtensorMap tmA, tmA64;
    if (!encode_2d_16(&tmA, idx->A, (uint64_t)idx->d_pad, (uint64_t)idx->n_pad, kBlockK, kTileM) ||
        !encode_2d_16(&tmA64, idx->A, (uint64_t)idx->d_pad, (uint64_t)idx->n_pad, kBlockK, kTileM / 2))
        return set_error(EBR_ECUDA, "cuTensorMapEncodeTiled(A) failed");
    // CTA-pair MMA for 2-group passes (3.00 vs 3.14 ms on C3); EBR_PAIR=0 selects the
    // single-CTA kernel (read per call, so a test can exercise both)
    const char* pair_env = getenv("EBR_PAIR");
    const bool use_pair = pair_env == nullptr || atoi(pair_env) != 0;
    // kernel attributes: set once per process (values fixed by the build)
    static std::once_flag attr_once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        auto set = [&](const void* f, int bytes) {
            cudaError_t x = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
            if (x != cudaSuccess && attr_err == cudaSuccess) attr_err = x;
        };
        const int big = 227 * 1024;
        for (const void* f : {(const void*)score_kernel<0, false>, (const void*)score_kernel<1, false>,
                              (const void*)score_kernel<0, true>, (const void*)score_kernel<1, true>})
            set(f, big);
        set((const void*)theta_kernel, 200 * 1024);
        set((const void*)final_kernel, 200 * 1024);
        set((const void*)entry_order_kernel, kOrderStage * 4);
        for (const void* f : {(const void*)score_kernel<0, false>, (const void*)score_kernel<1, false>,
                              (const void*)score_kernel<0, true>, (const void*)score_kernel<1, true>}) {
            cudaError_t x = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            (void)x;
        }
    });
    if (attr_err != cudaSuccess) return cuda_check(attr_err, "attr(batched kernels)");

    const size_t tsmem = 200 * 1024;
    const size_t fsmem = 200 * 1024;
    const int64_t fscap = (int64_t)(fsmem - (size_t)pow2ceil_i(q.k) * 8 - kSelBins * 4) / 8;
    const double ks = (double)q.k / (double)L.sstride;
    int rank = (int)std::ceil(ks + 5.0 * std::sqrt(ks) + 8.0);
    if (const char* r = getenv("EBR_THETA_RANK")) rank = atoi(r);   // test hook
    rank = std::max(1, std::min(rank, q.k));
    auto tscap_of = [&](int r) { return (int)((tsmem - (size_t)pow2ceil_i(r) * 8 - kThetaCopies * 2048 * 4) / 8); };
    int64_t cap = L.cap;
    if (const char* c = getenv("EBR_TEST_CAND_CAP")) cap = std::min<int64_t>(cap, std::max(1, atoi(c)));

    EntryArgs ea;
    ea.hdr = idx->chunk_hdr; ea.payload = idx->payload;
    ea.n_ads = idx->n_ads; ea.n_pad = idx->n_pad; ea.bin_ads = (int)L.bin_ads;
    ea.n_bins = (int)L.n_bins; ea.n_tiles = n_tiles; ea.bin_cap = L.bin_cap;
    ea.NU = (int)L.NU;

    for (int b0 = 0; b0 < q.batch; b0 += (int)L.P) {
        const int P = std::min((int)L.P, q.batch - b0);
        const int G = (P + kGroup - 1) / kGroup;
        ea.G = G;
        PlanArgs pa;
        pa.user_feat = q.user_feat + (size_t)b0 * idx->n_fields * q.slots;
        pa.user_x = q.user_x + (size_t)b0 * idx->n_fields * q.slots;
        pa.user_emb = reinterpret_cast<const uint16_t*>(q.user_emb) + (size_t)b0 * idx->d;
        pa.key_chunk_off = idx->key_chunk_off; pa.key_word_off = idx->key_word_off; pa.cross_w = idx->cross_w;
        pa.field_card = idx->field_card; pa.field_base = idx->field_base; pa.hot_slot = idx->hot_slot;
        pa.F = idx->n_fields; pa.S = q.slots; pa.P = P; pa.d = idx->d; pa.d_pad = idx->d_pad;
        pa.n_hot_used = tu.n_hb * 64; pa.pieces = tu.pieces; pa.u_cols = u_cols; pa.TS = L.TS; pa.NU = L.NU; pa.gcap = L.gcap; pa.err = err_word;
        const int nslot = P * idx->n_fields * q.slots;
        const int pgrid = std::max(1, std::min(4 * idx->sm_count, (nslot + 255) / 256));
        plan_a_kernel<<<pgrid, 256, 0, q.stream>>>(pa, ws);
        trace(q.stream, "plan_a");
        plan_b_kernel<<<1, kPlanThreads, 0, q.stream>>>(pa, ws);
        trace(q.stream, "plan_b");
        plan_c_kernel<<<std::max(pgrid, 2 * idx->sm_count), 256, 0, q.stream>>>(pa, ws);
        trace(q.stream, "plan_c");
        entry_bin_kernel<<<EBR_BIN_GRID * idx->sm_count, kBinThreads, 0, q.stream>>>(ea, ws);
        trace(q.stream, "entry_bin");
        entry_order_kernel<<<(unsigned)L.n_bins, kOrderThreads, kOrderStage * 4, q.stream>>>(ea, ws);
        trace(q.stream, "entry_order");
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_check(e, "launch(plan/entries)");

        GemmParams gp;
        gp.n_ads = idx->n_ads; gp.n_pad = idx->n_pad; gp.dense = 0; gp.ad_begin = (uint32_t)idx->ad_begin;
        gp.n_kb = n_kb; gp.n_hb = tu.n_hb; gp.pieces = tu.pieces; gp.acc_stages = acc_stages; gp.u_cols = u_cols;
        gp.P = P; gp.n_samp = (int)L.n_samp; gp.stages = stages; gp.smem_bytes = (int)smem; gp.cap = cap; gp.rerun = 0;
        gp.hot_mask = reinterpret_cast<const uint4*>(idx->hot_mask); gp.A = idx->A; gp.ws = ws; gp.err = err_word;
        static const int diag = getenv("EBR_DIAG") ? atoi(getenv("EBR_DIAG")) : 0;
        gp.diag = diag;
        gp.NU = (int)L.NU; gp.gcap = (int)L.gcap; gp.n_tiles_all = n_tiles;
        gp.pair = (G == 2 && use_pair) ? 1 : 0;
        gp.deep_smem = deep_smem ? 1 : 0;
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
                    const void* kf = gp.pair ? (mode ? (const void*)score_kernel<1, true> : (const void*)score_kernel<0, true>)
                                             : (mode ? (const void*)score_kernel<1, false> : (const void*)score_kernel<0, false>);
                    cudaError_t x = cudaOccupancyMaxActiveClusters(&n, kf, &cfg);
                    c = (x == cudaSuccess && n > 0) ? n : ncl;
                }
                ncl = std::min(ncl, c);
            }
            ncl = std::max(1, std::min(ncl, tiles));
            cfg.gridDim = dim3((unsigned)(G * ncl));
            if (gp.pair)
                return mode ? cudaLaunchKernelEx(&cfg, score_kernel<1, true>, tmA, tmA64, gp)
                            : cudaLaunchKernelEx(&cfg, score_kernel<0, true>, tmA, tmA64, gp);
            return mode ? cudaLaunchKernelEx(&cfg, score_kernel<1, false>, tmA, tmA64, gp)
                        : cudaLaunchKernelEx(&cfg, score_kernel<0, false>, tmA, tmA64, gp);
        };
        int32_t* oi = q.out_ids ? q.out_ids + (size_t)b0 * q.k : nullptr;
        float* os = q.out_scores ? q.out_scores + (size_t)b0 * q.k : nullptr;
        uint64_t* ok = q.out_keys ? q.out_keys + (size_t)b0 * q.k : nullptr;
        e = launch_score(0, n_samp_tiles, (int)L.sstride, 0);
        if (e != cudaSuccess) return cuda_check(e, "launch(score sample)");
        trace(q.stream, "score sample");
        theta_kernel<<<P, kThetaThreads, tsmem, q.stream>>>(ws, (int)L.n_samp, rank, (uint32_t)idx->ad_begin, P,
                                                           tscap_of(rank), 0, idx->n_pad, L.sstride);
        trace(q.stream, "theta");
        {
            KernelTimer kt(q.stream, "score_kernel<1> (fused tcgen05 deep + hot + cold wide + kappa + theta filter)");
            e = launch_score(1, n_tiles, 1, 0);
        }
        if (e != cudaSuccess) return cuda_check(e, "launch(score filter)");
        trace(q.stream, "score filter");
        if (diag & 4) {
            unsigned long long h[32];
            cudaMemcpyAsync(h, ws.prof, sizeof h, cudaMemcpyDeviceToHost, q.stream);
            cudaStreamSynchronize(q.stream);
            const double c = h[9] ? (double)h[9] : 1.0;
            fprintf(stderr, "[ebr prof] per CTA Mcycles (sample+filter): total %.2f tma_wait_empty %.2f mma_wait_wready %.2f "
                            "mma_wait_full %.2f hot_wait_empty %.2f wide_cold %.2f wide_wait_tempty %.2f wide_store %.2f "
                            "epi_wait_tfull %.2f epi_work %.2f wide_wait_efull %.2f (CTAs %llu)\n",
                    h[10] / c / 1e6, h[0] / c / 1e6, h[1] / c / 1e6, h[2] / c / 1e6, h[3] / c / 1e6, h[4] / c / 1e6,
                    h[5] / c / 1e6, h[6] / c / 1e6, h[7] / c / 1e6, h[8] / c / 1e6, h[11] / c / 1e6, h[9]);
            cudaMemsetAsync(ws.prof, 0, sizeof h, q.stream);
        }
        final_kernel<<<P, 512, fsmem, q.stream>>>(ws, cap, q.k, P, oi, os, ok, fscap, 0, rank, err_word);
        trace(q.stream, "final");
        // gated reruns (exact either way): the overflowed users' scores densely, then theta at rank
        // K for the users short of K candidates (sample) or overflowed (dense), filter, select
        e = launch_score(0, n_tiles, 1, 0, 1);
        if (e != cudaSuccess) return cuda_check(e, "launch(score dense)");
        trace(q.stream, "score dense");
        theta_kernel<<<P, kThetaThreads, tsmem, q.stream>>>(ws, (int)L.n_samp, q.k, (uint32_t)idx->ad_begin, P,
                                                           tscap_of(q.k), 1, idx->n_pad, L.sstride);
        trace(q.stream, "theta rerun");
        e = launch_score(1, n_tiles, 1, 1);
        if (e != cudaSuccess) return cuda_check(e, "launch(score rerun)");
        trace(q.stream, "score rerun");
        final_kernel<<<P, 512, fsmem, q.stream>>>(ws, cap, q.k, P, oi, os, ok, fscap, 1, q.k, err_word);
        trace(q.stream, "final rerun");
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_check(e, "launch(batch)");
    }
    return EBR_OK;
}

}  // namespace ebr
