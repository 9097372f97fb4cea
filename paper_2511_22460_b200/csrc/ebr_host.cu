// ebr_host.cu -- the C-ABI (include/ebr.h): index build (host encode + upload), query dispatch,
// cross-shard merge, debug decode, stats and error reporting.
//
// A0 index build follows the paper's Alg. 1 in purpose -- turn the binary matrix L
// into an inverted list keyed by feature index with ad indices as values, compressed
// and stored as a struct of arrays with per-key offsets -- with a different layout
// (DESIGN.md "Posting-chunk wire format"): each key's ascending list is cut into chunks of 32
// postings, delta-coded (gap-1) and bit-packed at the chunk's own width b (PforDelta-style,
// P:176).  Chunks play the role of the paper's uniform-size blocks: every chunk but
// a key's last holds exactly 32 postings, so a warp decodes any chunk in the same time.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ebr_device.cuh"

namespace ebr {

static thread_local std::string g_last_error;

ebr_status set_error(ebr_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

ebr_status cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return EBR_OK;
    return set_error(EBR_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------------------------------------
// dominant-kernel timer
// ------------------------------------------------------------------------------------------
struct TimerState {
    std::mutex mu;
    std::atomic<bool> on{false};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    std::string name;
};
static TimerState& timer_state() {
    static TimerState t;
    return t;
}

KernelTimer::KernelTimer(cudaStream_t stream, const char* name) {
    TimerState& t = timer_state();
    if (!t.on.load(std::memory_order_relaxed)) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    if (cudaEventCreate(&a) != cudaSuccess) { a = nullptr; return; }
    s = stream;
    cudaEventRecord(a, s);
    std::lock_guard<std::mutex> lk(t.mu);
    t.name = name;
}

KernelTimer::~KernelTimer() {
    if (!a) return;
    cudaEvent_t b = nullptr;
    if (cudaEventCreate(&b) != cudaSuccess) { cudaEventDestroy(a); return; }
    cudaEventRecord(b, s);
    TimerState& t = timer_state();
    std::lock_guard<std::mutex> lk(t.mu);
    t.ev.emplace_back(a, b);
}

#define EBR_CUDA(call)                                              \
    do {                                                            \
        cudaError_t e__ = (call);                                   \
        if (e__ != cudaSuccess) return cuda_check(e__, #call);      \
    } while (0)

ebr_status run_small(const QueryArgs& q, int b0, int B);
ebr_status device_encode(ebr_index* idx, const int32_t* d_feat, const int32_t* d_card, const int32_t* d_base,
                         cudaStream_t st, std::vector<int64_t>& key_count, const int64_t* d_off = nullptr,
                         const int32_t* d_keys = nullptr, int64_t nnz = 0);
uint32_t workspace_magic(const ebr_index* idx);
bool batch_eligible(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k);
int32_t batch_launches(const ebr_index* idx, int32_t batch, int32_t slots);
size_t batch_workspace_bytes(const ebr_index* idx, int32_t slots, int32_t k);
ebr_status run_batch(const QueryArgs& q, void* region, uint32_t* err_word);
size_t small_workspace_bytes(const ebr_index* idx, int32_t slots, int32_t k);

// ------------------------------------------------------------------------------------------
// host encoder
// ------------------------------------------------------------------------------------------
struct Encoded {
    std::vector<uint32_t> key_chunk_off, key_word_off, hdr, payload, last;
    std::vector<int64_t> key_count;   // postings per key
    int64_t nnz = 0;
};

static inline uint32_t bit_width(uint32_t v) { return v ? 32u - (uint32_t)__builtin_clz(v) : 0u; }

static ebr_status validate_inventory(const int32_t* ad_feat, int64_t n_ads, int32_t F,
                                     const int32_t* card, int64_t n_keys) {
    if (F < 0) return set_error(EBR_EINVAL, "n_fields < 0");
    int64_t m = 0;
    for (int f = 0; f < F; ++f) {
        if (card[f] < 1) return set_error(EBR_EINVAL, "field_card[%d] = %d < 1", f, card[f]);
        m += card[f];
    }
    if (m != n_keys) return set_error(EBR_EINVAL, "n_keys %lld != sum(field_card) %lld", (long long)n_keys, (long long)m);
    if (n_keys >= (int64_t)1 << 31) return set_error(EBR_EINVAL, "n_keys >= 2^31");
    for (int64_t a = 0; a < n_ads; ++a)
        for (int f = 0; f < F; ++f) {
            const int32_t v = ad_feat[a * F + f];
            if (v < -1 || v >= card[f])
                return set_error(EBR_EINVAL, "ad_feat[%lld][%d] = %d outside [-1, %d)", (long long)a, f, v, card[f]);
        }
    return EBR_OK;
}

// Encodes all posting lists of the shard; fields are independent (disjoint key ranges) and are
// encoded in parallel.
static ebr_status encode(const int32_t* ad_feat, int64_t n_ads, int32_t F, const int32_t* card,
                         int64_t n_keys, Encoded& out) {
    std::vector<int64_t> base(F + 1, 0);
    for (int f = 0; f < F; ++f) base[f + 1] = base[f] + card[f];
    std::vector<uint32_t> nchunks(n_keys, 0), nwords(n_keys, 0);
    out.key_count.assign(n_keys, 0);
    std::vector<std::vector<int32_t>> lists(F);
    std::vector<std::vector<int64_t>> loff(F);
    const int T = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
    std::atomic<int> next{0};
    std::atomic<bool> too_far{false};
    // pass 1: counting sort per field, chunk and word counts per key
    auto pass1 = [&]() {
        for (int f; (f = next.fetch_add(1)) < F;) {
            const int V = card[f];
            std::vector<int64_t>& off = loff[f];
            off.assign(V + 1, 0);
            for (int64_t a = 0; a < n_ads; ++a) {
                const int32_t v = ad_feat[a * F + f];
                if (v >= 0) off[v + 1]++;
            }
            for (int v = 0; v < V; ++v) off[v + 1] += off[v];
            std::vector<int32_t>& L = lists[f];
            L.resize(off[V]);
            std::vector<int64_t> fill(off.begin(), off.end() - 1);
            for (int64_t a = 0; a < n_ads; ++a) {
                const int32_t v = ad_feat[a * F + f];
                if (v >= 0) L[fill[v]++] = (int32_t)a;      // ascending a => ascending lists
            }
            for (int v = 0; v < V; ++v) {
                const int64_t n = off[v + 1] - off[v];
                const int64_t key = base[f] + v;
                out.key_count[key] = n;
                nchunks[key] = (uint32_t)((n + 31) / 32);
                uint64_t words = 0;
                for (int64_t c0 = off[v]; c0 < off[v + 1]; c0 += 32) {
                    const int64_t c1 = std::min<int64_t>(c0 + 32, off[v + 1]);
                    uint32_t mx = 0;
                    for (int64_t j = c0 + 1; j < c1; ++j) mx = std::max<uint32_t>(mx, (uint32_t)(L[j] - L[j - 1] - 1));
                    const uint32_t b = bit_width(mx);
                    words += ((uint64_t)(c1 - c0 - 1) * b + 31) / 32;
                }
                if (words >= (1u << 22)) too_far = true;   // relative word offset field is 22 bits
                nwords[key] = (uint32_t)words;
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 1; t < T; ++t) th.emplace_back(pass1);
        pass1();
        for (auto& t : th) t.join();
    }
    if (too_far) return set_error(EBR_EUNSUPPORTED, "a posting list exceeds 2^22 payload words");
    out.key_chunk_off.assign(n_keys + 1, 0);
    out.key_word_off.assign(n_keys, 0);
    uint64_t cacc = 0, wacc = 0;
    for (int64_t k = 0; k < n_keys; ++k) {
        out.key_chunk_off[k] = (uint32_t)cacc;
        out.key_word_off[k] = (uint32_t)wacc;
        cacc += nchunks[k];
        wacc += nwords[k];
        if (cacc >= 0xFFFFFFFFull || wacc >= 0xFFFFFFF0ull)
            return set_error(EBR_EUNSUPPORTED, "index exceeds 2^32 chunks/words");
    }
    out.key_chunk_off[n_keys] = (uint32_t)cacc;
    out.hdr.assign(2 * cacc, 0);
    out.last.assign(cacc, 0);
    out.payload.assign(wacc + 2, 0);   // two guard words: the decoder reads word w+1
    int64_t nnz = 0;
    for (int f = 0; f < F; ++f) nnz += (int64_t)lists[f].size();
    out.nnz = nnz;
    // pass 2: headers + payload
    next = 0;
    auto pass2 = [&]() {
        for (int f; (f = next.fetch_add(1)) < F;) {
            const int V = card[f];
            const std::vector<int32_t>& L = lists[f];
            const std::vector<int64_t>& off = loff[f];
            for (int v = 0; v < V; ++v) {
                const int64_t key = base[f] + v;
                uint32_t c = out.key_chunk_off[key];
                uint32_t rel = 0;
                uint32_t* pw = out.payload.data() + out.key_word_off[key];
                for (int64_t c0 = off[v]; c0 < off[v + 1]; c0 += 32, ++c) {
                    const int64_t c1 = std::min<int64_t>(c0 + 32, off[v + 1]);
                    uint32_t mx = 0;
                    for (int64_t j = c0 + 1; j < c1; ++j) mx = std::max<uint32_t>(mx, (uint32_t)(L[j] - L[j - 1] - 1));
                    const uint32_t b = bit_width(mx);
                    const uint32_t n = (uint32_t)(c1 - c0);
                    out.hdr[2 * (size_t)c] = (uint32_t)L[c0];
                    out.last[c] = (uint32_t)L[c1 - 1];
                    out.hdr[2 * (size_t)c + 1] = (n - 1u) | (b << 5) | (rel << 10);
                    if (b) {
                        for (int64_t j = c0 + 1; j < c1; ++j) {
                            const uint32_t val = (uint32_t)(L[j] - L[j - 1] - 1);
                            const uint64_t pos = (uint64_t)(j - c0 - 1) * b;
                            uint32_t* w = pw + rel + (pos >> 5);
                            const uint32_t sh = (uint32_t)(pos & 31);
                            w[0] |= val << sh;
                            if (sh + b > 32) w[1] |= val >> (32 - sh);
                        }
                    }
                    rel += (uint32_t)(((uint64_t)(n - 1) * b + 31) / 32);
                }
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 1; t < T; ++t) th.emplace_back(pass2);
        pass2();
        for (auto& t : th) t.join();
    }
    return EBR_OK;
}

// Padded kernel row width: row bytes a power of two in [64, 512] (>= 128 B for bf16, the TMA
// 128B-swizzle atom), or 1 KB / 2 KB.  Zero padding leaves every dot product exact.
static int32_t padded_width(int32_t d, int esz) {
    int64_t bytes = (int64_t)d * esz;
    int64_t p = (esz == 2) ? 128 : 64;
    while (p < bytes && p < 512) p <<= 1;
    if (bytes > 512) p = bytes <= 1024 ? 1024 : 2048;   // wider rows are rejected at build
    return (int32_t)(p / esz);
}

// ------------------------------------------------------------------------------------------
// Hot keys (bf16 indexes): the kMaxHot keys with the longest posting lists -- and at least
// max(64, n/512) postings -- also get a column of L stored as one bit of a 128-bit mask per ad
// (16 B/ad); the batched path expands a tile's masks into an fp16 one-hot block on chip and
// contracts it on the tensor cores.  The posting lists stay complete (the
// latency path and the batched path's cold keys read them).  EBR_HOT_KEYS=<n> caps the count.
// ------------------------------------------------------------------------------------------
__global__ void hot_mask_kernel(const int32_t* __restrict__ feat, int64_t n, int F,
                                const int32_t* __restrict__ field_base, const int32_t* __restrict__ hot_slot,
                                uint4* __restrict__ mask) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    uint32_t m[4] = {0u, 0u, 0u, 0u};
    for (int f = 0; f < F; ++f) {
        const int32_t v = feat[a * F + f];
        if (v < 0) continue;
        const int32_t h = hot_slot[field_base[f] + v];
        if (h >= 0) m[h >> 5] |= 1u << (h & 31);
    }
    mask[a] = make_uint4(m[0], m[1], m[2], m[3]);
}

__global__ void hot_mask_lists_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ keys, int64_t n,
                                      const int32_t* __restrict__ hot_slot, uint4* __restrict__ mask) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    uint32_t m[4] = {0u, 0u, 0u, 0u};
    for (int64_t q = off[a]; q < off[a + 1]; ++q) {
        const int32_t h = hot_slot[keys[q]];
        if (h >= 0) m[h >> 5] |= 1u << (h & 31);
    }
    mask[a] = make_uint4(m[0], m[1], m[2], m[3]);
}

static ebr_status build_hot(ebr_index* idx, const std::vector<int64_t>& key_count, const int32_t* ad_feat,
                            const int32_t* d_feat_all, cudaStream_t stream, const int64_t* d_off = nullptr,
                            const int32_t* d_keys = nullptr) {
    int cap = kMaxHot;
    if (const char* e = getenv("EBR_HOT_KEYS")) cap = std::max(0, std::min(kMaxHot, atoi(e)));
    const int64_t M = idx->n_keys, n = idx->n_ads;
    const int64_t min_count = std::max<int64_t>(64, n / 512);
    std::vector<int32_t> cand;
    for (int64_t k = 0; k < M; ++k)
        if (key_count[k] >= min_count) cand.push_back((int32_t)k);
    std::sort(cand.begin(), cand.end(), [&](int32_t x, int32_t y) {
        return key_count[x] != key_count[y] ? key_count[x] > key_count[y] : x < y;
    });
    if ((int64_t)cand.size() > cap) cand.resize(cap);
    const int n_hot = (int)((cand.size() + 63) / 64 * 64);
    idx->n_hot = n_hot;
    if (n_hot == 0) return EBR_OK;
    std::vector<int32_t> slot(M, -1), key(n_hot, -1);
    for (size_t h = 0; h < cand.size(); ++h) {
        slot[cand[h]] = (int32_t)h;
        key[h] = cand[h];
        idx->hot_nnz += key_count[cand[h]];
    }
    EBR_CUDA(cudaMalloc(&idx->hot_slot, (size_t)M * 4));
    EBR_CUDA(cudaMemcpyAsync(idx->hot_slot, slot.data(), (size_t)M * 4, cudaMemcpyHostToDevice, stream));
    EBR_CUDA(cudaMalloc(&idx->hot_key, (size_t)n_hot * 4));
    EBR_CUDA(cudaMemcpyAsync(idx->hot_key, key.data(), (size_t)n_hot * 4, cudaMemcpyHostToDevice, stream));
    const size_t mbytes = (size_t)idx->n_pad * 16;
    EBR_CUDA(cudaMalloc(&idx->hot_mask, mbytes));
    EBR_CUDA(cudaMemsetAsync(idx->hot_mask, 0, mbytes, stream));
    const int F = idx->n_fields;
    if (d_off) {                // device build from per-ad key lists
        hot_mask_lists_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_off, d_keys, n, idx->hot_slot,
                                                                              static_cast<uint4*>(idx->hot_mask));
        return cuda_check(cudaGetLastError(), "hot masks");
    }
    if (d_feat_all) {           // device build: the values are already on the device
        hot_mask_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_feat_all, n, F, idx->field_base, idx->hot_slot,
                                                                        static_cast<uint4*>(idx->hot_mask));
        return cuda_check(cudaGetLastError(), "hot masks");
    }
    const int64_t chunk = std::max<int64_t>(1, (int64_t)(256 << 20) / (4 * std::max(F, 1)));   // 256 MB of values
    int32_t* dfeat = nullptr;
    EBR_CUDA(cudaMalloc(&dfeat, (size_t)std::min(chunk, n) * F * 4));
    for (int64_t a0 = 0; a0 < n; a0 += chunk) {
        const int64_t m = std::min(chunk, n - a0);
        cudaError_t e = cudaMemcpyAsync(dfeat, ad_feat + a0 * F, (size_t)m * F * 4, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess) {
            hot_mask_kernel<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(
                dfeat, m, F, idx->field_base, idx->hot_slot, static_cast<uint4*>(idx->hot_mask) + a0);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);   // dfeat is reused
        if (e != cudaSuccess) { cudaFree(dfeat); return cuda_check(e, "hot masks"); }
    }
    cudaFree(dfeat);
    return EBR_OK;
}

// ------------------------------------------------------------------------------------------
// kernels owned by the host file: merge (A7) and debug decode
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) merge_kernel(const uint64_t* __restrict__ gathered, int G,
                                                         int B, int K, int32_t* out_ids,
                                                         float* out_scores, int64_t scand_cap) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t sScalar[8];
    const int P = pow2ceil_i(K);
    uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);
    uint32_t* shist = reinterpret_cast<uint32_t*>(sbuf + P);
    uint64_t* scand = reinterpret_cast<uint64_t*>(shist + kSelBins);
    const int b = blockIdx.x;
    const int64_t n = (int64_t)G * K;
    // The radix select needs unique keys: a shard's padding entries (key 0) become the distinct
    // sentinels i + 1 < 2^32, below every real kappa (ord(s) >= 1 for finite s), so they sort last
    // and are written out as padding when the shards together hold fewer than K ads.
    auto get = [=](int64_t i) {
        const int64_t g = i / K, q = i - g * K;
        const uint64_t x = __ldg(&gathered[(g * B + b) * (int64_t)K + q]);
        return x ? x : (uint64_t)(i + 1);
    };
    const int nsel = cta_select_topk(get, n, K, sbuf, scand_cap > 0 ? scand : nullptr, scand_cap, shist, sScalar);
    cta_write_topk(sbuf, nsel, K, out_ids + (size_t)b * K, out_scores + (size_t)b * K, nullptr);
}

// Threshold exchange (reading R24): with G shards, theta_u = min over ranks of
// each rank's ceil(K/G)-th local key is a lower bound of the global K-th key (every rank holds
// >= ceil(K/G) keys >= theta_u, so >= K keys overall), and every global top-K key is >= theta_u and
// inside its rank's local top K -- each rank only needs to send its local keys >= theta_u.
__global__ void kth_key_kernel(const uint64_t* __restrict__ keys, int B, int K, int kk, uint64_t* out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) out[b] = keys[(size_t)b * K + (kk - 1)];
}

// one CTA: theta_u, the count of local keys >= theta_u (keys are descending, padding 0), the
// exclusive scan of the counts (out_off[B] = total) and the packed keys
__global__ void __launch_bounds__(1024) exchange_pack_kernel(const uint64_t* __restrict__ keys, int B, int K,
                                                             const uint64_t* __restrict__ kq, int G,
                                                             uint32_t* out_count, uint32_t* out_off,
                                                             uint64_t* out_packed) {
    __shared__ uint32_t scratch[40];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int b0 = 0; b0 < B; b0 += blockDim.x) {
        const int b = b0 + threadIdx.x;
        uint32_t c = 0;
        if (b < B) {
            uint64_t th = ~0ull;
            for (int r = 0; r < G; ++r) th = min(th, kq[(size_t)r * B + b]);
            const uint64_t* kb = keys + (size_t)b * K;
            // first index with key < theta (or key == 0): binary search on the descending list
            int lo = 0, hi = K;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                const uint64_t x = kb[mid];
                if (x != 0 && x >= th) lo = mid + 1;
                else hi = mid;
            }
            c = (uint32_t)lo;
            out_count[b] = c;
        }
        uint32_t tot;
        const uint32_t pre = block_exclusive_scan(c, scratch, &tot) + carry;
        if (b < B) out_off[b] = pre;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) out_off[B] = carry;
    __syncthreads();
    // pack: user b's first count[b] keys to out_packed[off[b] ...] (one warp per user)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int b = warp; b < B; b += nw) {
        const uint32_t c = out_count[b], o = out_off[b];
        for (uint32_t j = lane; j < c; j += 32) out_packed[o + j] = keys[(size_t)b * K + j];
    }
}

// merge of packed per-rank lists: user b's candidates are, for every rank r, packed[r][off_r(b) ..
// off_r(b) + count_r(b)) with off_r the exclusive scan of count_r (counts [G][B])
__global__ void __launch_bounds__(kThreads) merge_packed_kernel(const uint64_t* __restrict__ packed, int64_t stride,
                                                                const uint32_t* __restrict__ counts, int G, int B,
                                                                int K, int32_t* out_ids, float* out_scores) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t sScalar[8];
    __shared__ int64_t sOff[16], sBeg[17];
    const int P = pow2ceil_i(K);
    uint64_t* sbuf = reinterpret_cast<uint64_t*>(smem);
    uint32_t* shist = reinterpret_cast<uint32_t*>(sbuf + P);
    const int b = blockIdx.x;
    // offsets of user b in every rank's packed list (warp r sums count_r[0..b))
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < G) {
        uint64_t s = 0;
        for (int u = lane; u < b; u += 32) s += counts[(size_t)warp * B + u];
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        if (lane == 0) sOff[warp] = (int64_t)s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int r = 0; r < G; ++r) { sBeg[r] = t; t += counts[(size_t)r * B + b]; }
        sBeg[G] = t;
    }
    __syncthreads();
    const int64_t n = sBeg[G];
    auto get = [=](int64_t i) {
        int r = 0;
        while (i >= sBeg[r + 1]) ++r;
        return __ldg(&packed[(size_t)r * stride + sOff[r] + (i - sBeg[r])]);
    };
    const int nsel = cta_select_topk(get, n, K, sbuf, nullptr, 0, shist, sScalar);
    cta_write_topk(sbuf, nsel, K, out_ids + (size_t)b * K, out_scores + (size_t)b * K, nullptr);
}

__global__ void decode_key_kernel(const uint2* __restrict__ hdr, const uint32_t* __restrict__ payload,
                                  uint32_t c0, uint32_t c1, uint32_t kwb, int32_t* out, int64_t cap) {
    const int lane = threadIdx.x & 31;
    const uint32_t c = c0 + blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (c >= c1) return;   // warp-uniform
    uint32_t id;
    const bool ok = decode_chunk(hdr, payload, kwb, c, lane, id);
    const int64_t pos = (int64_t)(c - c0) * 32 + lane;   // every chunk but the last is full
    if (ok && pos < cap) out[pos] = (int32_t)id;
}

ebr_status run_merge(const uint64_t* gathered, int32_t G, int32_t batch, int32_t k,
                     int32_t* out_ids, float* out_scores, cudaStream_t stream) {
    const size_t base = (size_t)pow2ceil_i(k) * 8 + kSelBins * 4;
    const size_t cap_bytes = 200 * 1024 > base ? 200 * 1024 - base : 0;
    int64_t scand_cap = std::min<int64_t>((int64_t)G * k, (int64_t)(cap_bytes / 8));
    if (scand_cap < (int64_t)G * k) scand_cap = 0;   // too many: select straight from global
    const size_t smem = base + (size_t)scand_cap * 8 + 64;
    EBR_CUDA(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    merge_kernel<<<batch, kThreads, smem, stream>>>(gathered, G, batch, k, out_ids, out_scores, scand_cap);
    return cuda_check(cudaGetLastError(), "launch(merge)");
}

ebr_status run_debug_decode(const ebr_index* idx, int64_t key, int32_t* dev_out, int64_t cap,
                            cudaStream_t stream) {
    uint32_t c[2], kwb;
    EBR_CUDA(cudaMemcpy(c, idx->key_chunk_off + key, 8, cudaMemcpyDeviceToHost));
    EBR_CUDA(cudaMemcpy(&kwb, idx->key_word_off + key, 4, cudaMemcpyDeviceToHost));
    if (c[1] > c[0]) {
        const uint32_t nch = c[1] - c[0];
        decode_key_kernel<<<(nch + 3) / 4, 128, 0, stream>>>(idx->chunk_hdr, idx->payload, c[0], c[1], kwb, dev_out, cap);
        EBR_CUDA(cudaGetLastError());
    }
    return EBR_OK;
}

static size_t small_region(const ebr_index* idx, int32_t slots, int32_t k) {
    return (small_workspace_bytes(idx, slots, k) + 1023) & ~(size_t)1023;
}

size_t workspace_bytes(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k) {
    size_t n = small_region(idx, slots, k);
    if (batch_eligible(idx, batch, slots, k)) n += batch_workspace_bytes(idx, slots, k);
    return n;
}

ebr_status run_query(const QueryArgs& q) {
    if (batch_eligible(q.idx, q.batch, q.slots, q.k)) {
        char* ws = static_cast<char*>(q.workspace);
        return run_batch(q, ws + small_region(q.idx, q.slots, q.k), reinterpret_cast<uint32_t*>(ws) + 1);
    }
    for (int b0 = 0; b0 < q.batch; b0 += kSmallMaxB) {
        const int B = std::min(kSmallMaxB, q.batch - b0);
        ebr_status st = run_small(q, b0, B);
        if (st != EBR_OK) return st;
    }
    return EBR_OK;
}

}  // namespace ebr

using namespace ebr;

// ------------------------------------------------------------------------------------------
// C-ABI
// ------------------------------------------------------------------------------------------
extern "C" {

const char* ebr_last_error(void) { return g_last_error.c_str(); }

ebr_status ebr_kernel_timer(int32_t enable) {
    timer_state().on.store(enable != 0);
    return EBR_OK;
}

ebr_status ebr_kernel_timer_read(double* total_ms, int64_t* launches, char* name, int32_t name_cap) {
    if (!total_ms || !launches) return set_error(EBR_EINVAL, "ebr_kernel_timer_read: null output");
    TimerState& t = timer_state();
    std::lock_guard<std::mutex> lk(t.mu);
    double tot = 0.0;
    ebr_status st = EBR_OK;
    for (auto& p : t.ev) {
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(p.second);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, p.first, p.second);
        if (e != cudaSuccess && st == EBR_OK) st = cuda_check(e, "kernel timer");
        tot += ms;
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    *total_ms = tot;
    *launches = (int64_t)t.ev.size();
    t.ev.clear();
    if (name && name_cap > 0) {
        strncpy(name, t.name.c_str(), (size_t)name_cap - 1);
        name[name_cap - 1] = 0;
    }
    return st;
}

int32_t ebr_query_launches(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k) {
    if (!idx || batch < 1 || slots < 1 || k < 1) return 0;
    if (batch_eligible(idx, batch, slots, k)) return batch_launches(idx, batch, slots);
    return (batch + kSmallMaxB - 1) / kSmallMaxB;
}

const char* ebr_version(void) {
#ifndef EBR_GIT
#define EBR_GIT "dev"
#endif
    return "ebr " EBR_GIT " sm_100a";
}

ebr_status ebr_encode_host(const int32_t* ad_feat, int64_t n_ads, int32_t n_fields,
                           const int32_t* field_card, int64_t n_keys, uint32_t* key_chunk_off,
                           uint32_t* key_word_off, uint32_t* chunk_hdr, int64_t hdr_cap,
                           uint32_t* payload, int64_t payload_cap, int64_t* n_chunks,
                           int64_t* n_words) {
    if (n_chunks) *n_chunks = -1;
    if (n_words) *n_words = -1;
    try {
        if (n_ads < 0 || (n_ads > 0 && !ad_feat) || !field_card)
            return set_error(EBR_EINVAL, "bad arguments");
        ebr_status st = validate_inventory(ad_feat, n_ads, n_fields, field_card, n_keys);
        if (st) return st;
        Encoded enc;
        st = encode(ad_feat, n_ads, n_fields, field_card, n_keys, enc);
        if (st) return st;
        const int64_t C = (int64_t)enc.hdr.size() / 2, W = (int64_t)enc.payload.size() - 2;
        if (n_chunks) *n_chunks = C;
        if (n_words) *n_words = W;
        if (C > hdr_cap || W > payload_cap) return set_error(EBR_EINVAL, "capacity too small");
        memcpy(key_chunk_off, enc.key_chunk_off.data(), sizeof(uint32_t) * (n_keys + 1));
        memcpy(key_word_off, enc.key_word_off.data(), sizeof(uint32_t) * n_keys);
        memcpy(chunk_hdr, enc.hdr.data(), sizeof(uint32_t) * 2 * C);
        memcpy(payload, enc.payload.data(), sizeof(uint32_t) * W);
        return EBR_OK;
    } catch (const std::bad_alloc&) {
        return set_error(EBR_ENOMEM, "host allocation failed");
    } catch (...) {
        return set_error(EBR_EINVAL, "unexpected exception");
    }
}

void ebr_free_index(ebr_index* idx) {
    if (!idx) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(idx->device);
    void* ptrs[] = {idx->A, idx->key_chunk_off, idx->key_word_off, idx->chunk_hdr, idx->chunk_last, idx->payload,
                    idx->cross_w, idx->field_card, idx->field_base, idx->hot_slot, idx->hot_key, idx->hot_mask};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    free(idx->tmap_A);
    if (prev >= 0) cudaSetDevice(prev);
    delete idx;
}

ebr_status ebr_build_index(const void* ad_emb, ebr_dtype dtype, int64_t ad_begin, int64_t ad_end,
                           int32_t d, const int32_t* ad_feat, int32_t n_fields,
                           const int32_t* field_card, const float* cross_w, int64_t n_keys,
                           int device, void* stream_v, ebr_index** out) {
    auto t0 = std::chrono::steady_clock::now();
    if (!out) return set_error(EBR_EINVAL, "out is null");
    *out = nullptr;
    if (d < 1) return set_error(EBR_EINVAL, "d < 1");
    if ((int64_t)d * (dtype == EBR_BF16 ? 2 : 4) > 2048)
        return set_error(EBR_EUNSUPPORTED, "embedding rows above 2 KB (d=%d) are not supported", d);
    if (dtype != EBR_F32 && dtype != EBR_BF16) return set_error(EBR_EINVAL, "bad dtype");
    if (ad_begin < 0 || ad_begin >= ad_end) return set_error(EBR_EINVAL, "need 0 <= ad_begin < ad_end");
    if (ad_end > 0x7FFFFFFFll) return set_error(EBR_EINVAL, "ad_end > 2^31-1");
    if (!ad_emb || !ad_feat || !field_card || (!cross_w && n_keys > 0))
        return set_error(EBR_EINVAL, "null input");
    const int64_t n = ad_end - ad_begin;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
    try {
        ebr_status st = validate_inventory(ad_feat, n, n_fields, field_card, n_keys);
        if (st) return st;
        int prev = -1;
        cudaGetDevice(&prev);
        EBR_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        EBR_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) {
            if (prev >= 0) cudaSetDevice(prev);
            return set_error(EBR_EUNSUPPORTED, "device %d is sm_%d%d, this library is built for sm_100a",
                             device, prop.major, prop.minor);
        }
        Encoded enc;
        const auto te0 = std::chrono::steady_clock::now();
        st = encode(ad_feat, n, n_fields, field_card, n_keys, enc);
        if (st) return st;
        const double enc_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te0).count();
        ebr_index* idx = new ebr_index();
        memset(idx, 0, sizeof(*idx));
        idx->device = device;
        idx->dtype = dtype;
        idx->d = d;
        const int esz = dtype == EBR_BF16 ? 2 : 4;
        idx->d_pad = padded_width(d, esz);
        idx->n_ads = n;
        idx->n_pad = (n + 127) / 128 * 128;
        idx->ad_begin = ad_begin;
        idx->n_fields = n_fields;
        idx->n_keys = n_keys;
        idx->nnz = enc.nnz;
        idx->n_chunks = (int64_t)enc.hdr.size() / 2;
        idx->n_words = (int64_t)enc.payload.size() - 2;
        idx->sm_count = prop.multiProcessorCount;
        idx->max_ad_keys = n_fields;
        idx->encode_ms = enc_ms;
        auto fail = [&](ebr_status s) { ebr_free_index(idx); if (prev >= 0) cudaSetDevice(prev); return s; };
#define EBR_TRY(call) do { cudaError_t e__ = (call); if (e__ != cudaSuccess) return fail(cuda_check(e__, #call)); } while (0)
        const size_t abytes = (size_t)idx->n_pad * idx->d_pad * esz;
        EBR_TRY(cudaMalloc(&idx->A, abytes));
        EBR_TRY(cudaMemsetAsync(idx->A, 0, abytes, stream));
        EBR_TRY(cudaMemcpy2DAsync(idx->A, (size_t)idx->d_pad * esz, ad_emb, (size_t)d * esz, (size_t)d * esz, n,
                                  cudaMemcpyHostToDevice, stream));
        auto upload = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
            cudaError_t e = cudaMalloc(dst, bytes ? bytes : 4);
            if (e != cudaSuccess || !bytes) return e;
            return cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, stream);
        };
        EBR_TRY(upload((void**)&idx->key_chunk_off, enc.key_chunk_off.data(), enc.key_chunk_off.size() * 4));
        EBR_TRY(upload((void**)&idx->key_word_off, enc.key_word_off.data(), enc.key_word_off.size() * 4));
        EBR_TRY(upload((void**)&idx->chunk_hdr, enc.hdr.data(), enc.hdr.size() * 4));
        EBR_TRY(upload((void**)&idx->chunk_last, enc.last.data(), enc.last.size() * 4));
        EBR_TRY(upload((void**)&idx->payload, enc.payload.data(), enc.payload.size() * 4));
        EBR_TRY(upload((void**)&idx->cross_w, cross_w, (size_t)n_keys * 4));
        std::vector<int32_t> fb(n_fields);
        int64_t acc = 0;
        for (int f = 0; f < n_fields; ++f) { fb[f] = (int32_t)acc; acc += field_card[f]; }
        EBR_TRY(upload((void**)&idx->field_card, field_card, (size_t)n_fields * 4));
        EBR_TRY(upload((void**)&idx->field_base, fb.data(), (size_t)n_fields * 4));
        if (dtype == EBR_BF16) {
            st = build_hot(idx, enc.key_count, ad_feat, nullptr, stream);
            if (st) return fail(st);
        }
        EBR_TRY(cudaStreamSynchronize(stream));
#undef EBR_TRY
        idx->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (prev >= 0) cudaSetDevice(prev);
        *out = idx;
        return EBR_OK;
    } catch (const std::bad_alloc&) {
        return set_error(EBR_ENOMEM, "host allocation failed");
    }
}

// device build from ad_feat (one value per field) or from per-ad key lists (ad_key_off/ad_keys)
static ebr_status build_device(const void* ad_emb, ebr_dtype dtype, int64_t ad_begin, int64_t ad_end, int32_t d,
                               const int32_t* ad_feat, const int64_t* ad_key_off, const int32_t* ad_keys,
                               int32_t n_fields, const int32_t* field_card, const float* cross_w, int64_t n_keys,
                               int device, void* stream_v, ebr_index** out) {
    auto t0 = std::chrono::steady_clock::now();
    if (!out) return set_error(EBR_EINVAL, "out is null");
    *out = nullptr;
    if (d < 1) return set_error(EBR_EINVAL, "d < 1");
    if ((int64_t)d * (dtype == EBR_BF16 ? 2 : 4) > 2048)
        return set_error(EBR_EUNSUPPORTED, "embedding rows above 2 KB (d=%d) are not supported", d);
    if (dtype != EBR_F32 && dtype != EBR_BF16) return set_error(EBR_EINVAL, "bad dtype");
    if (ad_begin < 0 || ad_begin >= ad_end) return set_error(EBR_EINVAL, "need 0 <= ad_begin < ad_end");
    if (ad_end > 0x7FFFFFFFll) return set_error(EBR_EINVAL, "ad_end > 2^31-1");
    const bool lists = ad_feat == nullptr;
    if (!ad_emb || (!ad_feat && (!ad_key_off || !ad_keys)) || !field_card || (!cross_w && n_keys > 0))
        return set_error(EBR_EINVAL, "null input");
    if (n_fields < 0) return set_error(EBR_EINVAL, "n_fields < 0");
    int64_t m = 0;
    for (int f = 0; f < n_fields; ++f) {
        if (field_card[f] < 1) return set_error(EBR_EINVAL, "field_card[%d] = %d < 1", f, field_card[f]);
        m += field_card[f];
    }
    if (m != n_keys) return set_error(EBR_EINVAL, "n_keys %lld != sum(field_card) %lld", (long long)n_keys, (long long)m);
    if (n_keys >= (int64_t)1 << 31) return set_error(EBR_EINVAL, "n_keys >= 2^31");
    const int64_t n = ad_end - ad_begin;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
    try {
        int prev = -1;
        cudaGetDevice(&prev);
        EBR_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        EBR_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) {
            if (prev >= 0) cudaSetDevice(prev);
            return set_error(EBR_EUNSUPPORTED, "device %d is sm_%d%d, this library is built for sm_100a",
                             device, prop.major, prop.minor);
        }
        ebr_index* idx = new ebr_index();
        memset(idx, 0, sizeof(*idx));
        idx->device = device;
        idx->dtype = dtype;
        idx->d = d;
        const int esz = dtype == EBR_BF16 ? 2 : 4;
        idx->d_pad = padded_width(d, esz);
        idx->n_ads = n;
        idx->n_pad = (n + 127) / 128 * 128;
        idx->ad_begin = ad_begin;
        idx->n_fields = n_fields;
        idx->n_keys = n_keys;
        idx->sm_count = prop.multiProcessorCount;
        idx->max_ad_keys = n_fields;
        int64_t nnz = 0;
        if (lists) {
            if (ad_key_off[0] != 0) return set_error(EBR_EINVAL, "ad_key_off[0] != 0");
            int64_t mx = 0;
            for (int64_t a = 0; a < n; ++a) {
                const int64_t c = ad_key_off[a + 1] - ad_key_off[a];
                if (c < 0) return set_error(EBR_EINVAL, "ad_key_off not ascending");
                mx = std::max(mx, c);
            }
            if (mx > 1024) return set_error(EBR_EUNSUPPORTED, "an ad with more than 1024 keys");
            nnz = ad_key_off[n];
            idx->max_ad_keys = (int32_t)std::max<int64_t>(mx, 1);
        }
        int32_t* d_feat = nullptr;
        int64_t* d_off = nullptr;
        int32_t* d_keys = nullptr;
        auto fail = [&](ebr_status s) {
            if (d_feat) cudaFree(d_feat);
            if (d_off) cudaFree(d_off);
            if (d_keys) cudaFree(d_keys);
            ebr_free_index(idx);
            if (prev >= 0) cudaSetDevice(prev);
            return s;
        };
#define EBR_TRY(call) do { cudaError_t e__ = (call); if (e__ != cudaSuccess) return fail(cuda_check(e__, #call)); } while (0)
        const size_t abytes = (size_t)idx->n_pad * idx->d_pad * esz;
        EBR_TRY(cudaMalloc(&idx->A, abytes));
        EBR_TRY(cudaMemsetAsync(idx->A, 0, abytes, stream));
        EBR_TRY(cudaMemcpy2DAsync(idx->A, (size_t)idx->d_pad * esz, ad_emb, (size_t)d * esz, (size_t)d * esz, n,
                                  cudaMemcpyHostToDevice, stream));
        auto upload = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
            cudaError_t e = cudaMalloc(dst, bytes ? bytes : 4);
            if (e != cudaSuccess || !bytes) return e;
            return cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, stream);
        };
        EBR_TRY(cudaStreamSynchronize(stream));        // (A's upload is not part of encode_ms)
        const auto te0 = std::chrono::steady_clock::now();
        if (lists) {
            EBR_TRY(upload((void**)&d_off, ad_key_off, (size_t)(n + 1) * 8));
            EBR_TRY(upload((void**)&d_keys, ad_keys, (size_t)std::max<int64_t>(nnz, 1) * 4));
        } else {
            EBR_TRY(upload((void**)&d_feat, ad_feat, (size_t)n * n_fields * 4));
        }
        EBR_TRY(upload((void**)&idx->cross_w, cross_w, (size_t)n_keys * 4));
        std::vector<int32_t> fb(n_fields);
        int64_t acc = 0;
        for (int f = 0; f < n_fields; ++f) { fb[f] = (int32_t)acc; acc += field_card[f]; }
        EBR_TRY(upload((void**)&idx->field_card, field_card, (size_t)n_fields * 4));
        EBR_TRY(upload((void**)&idx->field_base, fb.data(), (size_t)n_fields * 4));
        std::vector<int64_t> key_count;
        ebr_status st = device_encode(idx, d_feat, idx->field_card, idx->field_base, stream, key_count, d_off, d_keys,
                                      nnz);
        if (st) return fail(st);
        if (dtype == EBR_BF16) {
            st = build_hot(idx, key_count, ad_feat, d_feat, stream, d_off, d_keys);
            if (st) return fail(st);
        }
        EBR_TRY(cudaStreamSynchronize(stream));
        idx->encode_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te0).count();
        cudaFree(d_feat);
        cudaFree(d_off);
        cudaFree(d_keys);
        d_feat = nullptr;
        d_off = nullptr;
        d_keys = nullptr;
#undef EBR_TRY
        idx->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (prev >= 0) cudaSetDevice(prev);
        *out = idx;
        return EBR_OK;
    } catch (const std::bad_alloc&) {
        return set_error(EBR_ENOMEM, "host allocation failed");
    }
}

ebr_status ebr_build_index_device(const void* ad_emb, ebr_dtype dtype, int64_t ad_begin, int64_t ad_end,
                                  int32_t d, const int32_t* ad_feat, int32_t n_fields,
                                  const int32_t* field_card, const float* cross_w, int64_t n_keys,
                                  int device, void* stream_v, ebr_index** out) {
    if (!ad_feat) return set_error(EBR_EINVAL, "null input");
    return build_device(ad_emb, dtype, ad_begin, ad_end, d, ad_feat, nullptr, nullptr, n_fields, field_card, cross_w,
                        n_keys, device, stream_v, out);
}

ebr_status ebr_build_index_lists(const void* ad_emb, ebr_dtype dtype, int64_t ad_begin, int64_t ad_end, int32_t d,
                                 const int64_t* ad_key_off, const int32_t* ad_keys, int32_t n_fields,
                                 const int32_t* field_card, const float* cross_w, int64_t n_keys, int device,
                                 void* stream_v, ebr_index** out) {
    if (!ad_key_off || !ad_keys) return set_error(EBR_EINVAL, "null input");
    return build_device(ad_emb, dtype, ad_begin, ad_end, d, nullptr, ad_key_off, ad_keys, n_fields, field_card,
                        cross_w, n_keys, device, stream_v, out);
}

ebr_status ebr_index_export(const ebr_index* idx, int32_t which, void* out_host, int64_t cap_bytes, int64_t* bytes) {
    if (!idx || !bytes) return set_error(EBR_EINVAL, "null argument");
    const void* src = nullptr;
    int64_t nb = 0;
    switch (which) {
        case 0: src = idx->key_chunk_off; nb = (idx->n_keys + 1) * 4; break;
        case 1: src = idx->key_word_off; nb = idx->n_keys * 4; break;
        case 2: src = idx->chunk_hdr; nb = idx->n_chunks * 8; break;
        case 3: src = idx->chunk_last; nb = idx->n_chunks * 4; break;
        case 4: src = idx->payload; nb = (idx->n_words + 2) * 4; break;
        case 5: src = idx->hot_mask; nb = idx->hot_mask ? idx->n_pad * 16 : 0; break;
        default: return set_error(EBR_EINVAL, "which must be 0..5");
    }
    *bytes = nb;
    if (!out_host || cap_bytes < nb) return out_host ? set_error(EBR_EINVAL, "capacity %lld < %lld", (long long)cap_bytes, (long long)nb) : EBR_OK;
    if (nb) {
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != idx->device) cudaSetDevice(idx->device);
        cudaError_t e = cudaMemcpy(out_host, src, (size_t)nb, cudaMemcpyDeviceToHost);
        if (prev >= 0 && prev != idx->device) cudaSetDevice(prev);
        if (e != cudaSuccess) return cuda_check(e, "export");
    }
    return EBR_OK;
}

size_t ebr_workspace_bytes(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k) {
    if (!idx || batch < 1 || slots < 1 || slots > 64 || k < 1 || k > EBR_MAX_K) return 0;
    return workspace_bytes(idx, batch, slots, k);
}

static ebr_status query_common(const ebr_index* idx, const void* user_emb, int32_t batch,
                               const int32_t* user_feat, const float* user_x, int32_t slots,
                               int32_t k, int32_t* out_ids, float* out_scores, uint64_t* out_keys,
                               void* workspace, size_t workspace_bytes_, void* stream) {
    if (!idx) return set_error(EBR_EINVAL, "null index");
    if (batch < 1) return set_error(EBR_EINVAL, "batch < 1");
    if (slots < 1 || slots > 64) return set_error(EBR_EINVAL, "slots must be in [1, 64]");
    if (k < 1 || k > EBR_MAX_K) return set_error(EBR_EINVAL, "k must be in [1, %d]", EBR_MAX_K);
    if (!user_emb || !user_feat || !user_x || !workspace) return set_error(EBR_EINVAL, "null pointer");
    if (!out_keys && (!out_ids || !out_scores)) return set_error(EBR_EINVAL, "null output");
    const size_t need = workspace_bytes(idx, batch, slots, k);
    if (workspace_bytes_ < need)
        return set_error(EBR_EINVAL, "workspace %zu bytes < required %zu", workspace_bytes_, need);
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return set_error(EBR_EINVAL, "workspace not 256-byte aligned");
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != idx->device) cudaSetDevice(idx->device);
    QueryArgs q{idx, user_emb, batch, user_feat, user_x, slots, k, out_ids, out_scores, out_keys,
                workspace, workspace_bytes_, static_cast<cudaStream_t>(stream)};
    ebr_status st = run_query(q);
    if (prev >= 0 && prev != idx->device) cudaSetDevice(prev);
    return st;
}

ebr_status ebr_score_topk(const ebr_index* idx, const void* user_emb, int32_t batch,
                          const int32_t* user_feat, const float* user_x, int32_t slots, int32_t k,
                          int32_t* out_ids, float* out_scores, void* workspace,
                          size_t workspace_bytes_, void* stream) {
    return query_common(idx, user_emb, batch, user_feat, user_x, slots, k, out_ids, out_scores,
                        nullptr, workspace, workspace_bytes_, stream);
}

ebr_status ebr_score_topk_keys(const ebr_index* idx, const void* user_emb, int32_t batch,
                               const int32_t* user_feat, const float* user_x, int32_t slots,
                               int32_t k, uint64_t* out_keys, void* workspace,
                               size_t workspace_bytes_, void* stream) {
    if (!out_keys) return set_error(EBR_EINVAL, "null out_keys");
    return query_common(idx, user_emb, batch, user_feat, user_x, slots, k, nullptr, nullptr,
                        out_keys, workspace, workspace_bytes_, stream);
}

ebr_status ebr_workspace_init(const ebr_index* idx, void* workspace, size_t bytes, void* stream) {
    if (!idx || !workspace) return set_error(EBR_EINVAL, "null argument");
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return set_error(EBR_EINVAL, "workspace not 256-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != idx->device) cudaSetDevice(idx->device);
    EBR_CUDA(cudaMemsetAsync(workspace, 0, bytes, s));
    const uint32_t magic = workspace_magic(idx);
    EBR_CUDA(cudaMemcpyAsync(workspace, &magic, 4, cudaMemcpyHostToDevice, s));
    EBR_CUDA(cudaStreamSynchronize(s));   // `magic` lives on this stack frame
    if (prev >= 0 && prev != idx->device) cudaSetDevice(prev);
    return EBR_OK;
}

ebr_status ebr_query_error(void* workspace, void* stream, uint32_t* flags) {
    if (!workspace) return set_error(EBR_EINVAL, "null workspace");
    uint32_t f = 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // workspace header: word 0 = state magic, word 1 = validation flags
    uint32_t* flag_word = static_cast<uint32_t*>(workspace) + 1;
    EBR_CUDA(cudaMemcpyAsync(&f, flag_word, 4, cudaMemcpyDeviceToHost, s));
    EBR_CUDA(cudaMemsetAsync(flag_word, 0, 4, s));
    EBR_CUDA(cudaStreamSynchronize(s));
    if (flags) *flags = f;
    return f ? set_error(EBR_EDEVICE, "device validation flags 0x%x", f) : EBR_OK;
}

// e2e: inputs staged after the query workspace
static size_t host_stage_bytes(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k) {
    const int esz = idx->dtype == EBR_BF16 ? 2 : 4;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t nfs = (size_t)batch * idx->n_fields * slots;
    return al((size_t)batch * idx->d * esz) + al(nfs * 4) + al(nfs * 4) + al((size_t)batch * k * 4) * 2;
}

size_t ebr_workspace_bytes_host(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k) {
    const size_t w = ebr_workspace_bytes(idx, batch, slots, k);
    if (!w) return 0;
    return ((w + 255) & ~(size_t)255) + host_stage_bytes(idx, batch, slots, k);
}

ebr_status ebr_score_topk_host(const ebr_index* idx, const void* user_emb_host, int32_t batch,
                               const int32_t* user_feat_host, const float* user_x_host,
                               int32_t slots, int32_t k, int32_t* out_ids_host,
                               float* out_scores_host, void* workspace, size_t workspace_bytes_,
                               void* stream_v) {
    if (!idx) return set_error(EBR_EINVAL, "null index");
    const size_t w = ebr_workspace_bytes(idx, batch, slots, k);
    if (!w) return set_error(EBR_EINVAL, "bad batch/slots/k");
    if (workspace_bytes_ < ebr_workspace_bytes_host(idx, batch, slots, k))
        return set_error(EBR_EINVAL, "workspace too small for the host variant");
    if (!user_emb_host || !user_feat_host || !user_x_host || !out_ids_host || !out_scores_host)
        return set_error(EBR_EINVAL, "null host pointer");
    cudaStream_t s = static_cast<cudaStream_t>(stream_v);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const int esz = idx->dtype == EBR_BF16 ? 2 : 4;
    const size_t nfs = (size_t)batch * idx->n_fields * slots;
    char* st = static_cast<char*>(workspace) + al(w);
    char* d_emb = st;            st += al((size_t)batch * idx->d * esz);
    int32_t* d_feat = (int32_t*)st; st += al(nfs * 4);
    float* d_x = (float*)st;     st += al(nfs * 4);
    int32_t* d_ids = (int32_t*)st; st += al((size_t)batch * k * 4);
    float* d_sc = (float*)st;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != idx->device) cudaSetDevice(idx->device);
    const size_t in_bytes = (size_t)(reinterpret_cast<char*>(d_ids) - d_emb);       // emb | feat | x
    const size_t out_bytes = (size_t)(reinterpret_cast<char*>(d_sc) - reinterpret_cast<char*>(d_ids)) +
                             (size_t)batch * k * 4;                                  // ids | scores
    // small requests (latency path): one H2D and one D2H through a pinned staging buffer (the
    // per-copy latency, not the bytes, dominates); large ones copy each array directly
    thread_local char* pin = nullptr;
    thread_local size_t pin_bytes = 0;
    const size_t need = std::max(in_bytes, out_bytes);
    const bool staged = need <= ((size_t)1 << 20);
    if (staged && pin_bytes < need) {
        if (pin) cudaFreeHost(pin);
        pin = nullptr;
        pin_bytes = 0;
        if (cudaMallocHost(&pin, need) == cudaSuccess) pin_bytes = need;
    }
    if (staged && pin) {
        memcpy(pin, user_emb_host, (size_t)batch * idx->d * esz);
        memcpy(pin + (reinterpret_cast<char*>(d_feat) - d_emb), user_feat_host, nfs * 4);
        memcpy(pin + (reinterpret_cast<char*>(d_x) - d_emb), user_x_host, nfs * 4);
        EBR_CUDA(cudaMemcpyAsync(d_emb, pin, in_bytes, cudaMemcpyHostToDevice, s));
    } else {
        EBR_CUDA(cudaMemcpyAsync(d_emb, user_emb_host, (size_t)batch * idx->d * esz, cudaMemcpyHostToDevice, s));
        EBR_CUDA(cudaMemcpyAsync(d_feat, user_feat_host, nfs * 4, cudaMemcpyHostToDevice, s));
        EBR_CUDA(cudaMemcpyAsync(d_x, user_x_host, nfs * 4, cudaMemcpyHostToDevice, s));
    }
    ebr_status r = ebr_score_topk(idx, d_emb, batch, d_feat, d_x, slots, k, d_ids, d_sc, workspace, w, stream_v);
    if (r != EBR_OK) return r;
    if (staged && pin) {
        // the H2D above read `pin`; this D2H is stream-ordered after it, so reusing it is safe
        EBR_CUDA(cudaMemcpyAsync(pin, d_ids, out_bytes, cudaMemcpyDeviceToHost, s));
        EBR_CUDA(cudaStreamSynchronize(s));
        memcpy(out_ids_host, pin, (size_t)batch * k * 4);
        memcpy(out_scores_host, pin + (reinterpret_cast<char*>(d_sc) - reinterpret_cast<char*>(d_ids)),
               (size_t)batch * k * 4);
    } else {
        EBR_CUDA(cudaMemcpyAsync(out_ids_host, d_ids, (size_t)batch * k * 4, cudaMemcpyDeviceToHost, s));
        EBR_CUDA(cudaMemcpyAsync(out_scores_host, d_sc, (size_t)batch * k * 4, cudaMemcpyDeviceToHost, s));
        EBR_CUDA(cudaStreamSynchronize(s));
    }
    if (prev >= 0 && prev != idx->device) cudaSetDevice(prev);
    return EBR_OK;
}

ebr_status ebr_exchange_kth(const uint64_t* local_keys, int32_t batch, int32_t k, int32_t G, uint64_t* out_kq,
                            void* stream) {
    if (!local_keys || !out_kq) return set_error(EBR_EINVAL, "null pointer");
    if (G < 1 || G > 16 || batch < 1 || k < 1 || k > EBR_MAX_K) return set_error(EBR_EINVAL, "bad G/batch/k");
    const int kk = (k + G - 1) / G;
    kth_key_kernel<<<(batch + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(local_keys, batch, k, kk, out_kq);
    return cuda_check(cudaGetLastError(), "launch(kth)");
}

ebr_status ebr_exchange_pack(const uint64_t* local_keys, int32_t batch, int32_t k, const uint64_t* kq_gathered,
                             int32_t G, uint32_t* out_count, uint32_t* out_off, uint64_t* out_packed, void* stream) {
    if (!local_keys || !kq_gathered || !out_count || !out_off || !out_packed)
        return set_error(EBR_EINVAL, "null pointer");
    if (G < 1 || G > 16 || batch < 1 || k < 1 || k > EBR_MAX_K) return set_error(EBR_EINVAL, "bad G/batch/k");
    exchange_pack_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(local_keys, batch, k, kq_gathered, G,
                                                                          out_count, out_off, out_packed);
    return cuda_check(cudaGetLastError(), "launch(exchange pack)");
}

ebr_status ebr_merge_topk_packed(const uint64_t* packed, int64_t stride, const uint32_t* counts, int32_t G,
                                 int32_t batch, int32_t k, int32_t* out_ids, float* out_scores, void* stream) {
    if (!packed || !counts || !out_ids || !out_scores) return set_error(EBR_EINVAL, "null pointer");
    if (G < 1 || G > 16 || batch < 1 || k < 1 || k > EBR_MAX_K || stride < 0)
        return set_error(EBR_EINVAL, "bad G/batch/k/stride");
    const size_t smem = (size_t)pow2ceil_i(k) * 8 + kSelBins * 4 + 64;
    EBR_CUDA(cudaFuncSetAttribute(merge_packed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    merge_packed_kernel<<<batch, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(packed, stride, counts, G,
                                                                                     batch, k, out_ids, out_scores);
    return cuda_check(cudaGetLastError(), "launch(merge packed)");
}

size_t ebr_merge_workspace_bytes(int32_t G, int32_t batch, int32_t k) {
    if (G < 1 || batch < 1 || k < 1 || k > EBR_MAX_K) return 0;
    return 256;
}

ebr_status ebr_merge_topk(const uint64_t* gathered, int32_t G, int32_t batch, int32_t k,
                          int32_t* out_ids, float* out_scores, void* workspace,
                          size_t workspace_bytes_, void* stream) {
    (void)workspace; (void)workspace_bytes_;
    if (!gathered || !out_ids || !out_scores) return set_error(EBR_EINVAL, "null pointer");
    if (G < 1 || batch < 1 || k < 1 || k > EBR_MAX_K) return set_error(EBR_EINVAL, "bad G/batch/k");
    return run_merge(gathered, G, batch, k, out_ids, out_scores, static_cast<cudaStream_t>(stream));
}

ebr_status ebr_debug_decode(const ebr_index* idx, int64_t key, int32_t* out_ads, int64_t cap,
                            int64_t* n) {
    if (!idx || !n) return set_error(EBR_EINVAL, "null argument");
    if (key < 0 || key >= idx->n_keys) return set_error(EBR_EINVAL, "key out of range");
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != idx->device) cudaSetDevice(idx->device);
    uint32_t c[2];
    EBR_CUDA(cudaMemcpy(c, idx->key_chunk_off + key, 8, cudaMemcpyDeviceToHost));
    int64_t len = 0;
    if (c[1] > c[0]) {
        uint32_t last_hdr[2];
        EBR_CUDA(cudaMemcpy(last_hdr, idx->chunk_hdr + (c[1] - 1), 8, cudaMemcpyDeviceToHost));
        len = (int64_t)(c[1] - c[0] - 1) * 32 + (last_hdr[1] & 31u) + 1;
    }
    *n = len;
    if (len > cap) return set_error(EBR_EINVAL, "list of %lld ids exceeds cap", (long long)len);
    if (len == 0) return EBR_OK;
    int32_t* dev = nullptr;
    EBR_CUDA(cudaMalloc(&dev, (size_t)len * 4));
    ebr_status st = run_debug_decode(idx, key, dev, len, nullptr);
    if (st == EBR_OK) {
        cudaError_t e = cudaMemcpy(out_ads, dev, (size_t)len * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) st = cuda_check(e, "cudaMemcpy(decode)");
    }
    cudaFree(dev);
    if (prev >= 0 && prev != idx->device) cudaSetDevice(prev);
    return st;
}

ebr_status ebr_index_stats(const ebr_index* idx, ebr_stats* o) {
    if (!idx || !o) return set_error(EBR_EINVAL, "null argument");
    const int esz = idx->dtype == EBR_BF16 ? 2 : 4;
    o->n_ads = idx->n_ads;
    o->ad_begin = idx->ad_begin;
    o->d = idx->d;
    o->d_pad = idx->d_pad;
    o->dtype = idx->dtype;
    o->n_fields = idx->n_fields;
    o->n_keys = idx->n_keys;
    o->nnz = idx->nnz;
    o->chunks = idx->n_chunks;
    o->payload_words = idx->n_words;
    o->index_bytes = (idx->n_keys * 2 + 1) * 4 + idx->n_chunks * 12 + (idx->n_words + 2) * 4 + idx->n_keys * 4 +
                     (idx->hot_mask ? (int64_t)idx->n_pad * 16 + idx->n_keys * 4 : 0);
    o->emb_bytes = idx->n_pad * idx->d_pad * esz;
    o->build_ms = idx->build_ms;
    o->n_hot = idx->n_hot;
    o->hot_nnz = idx->hot_nnz;
    o->hot_bytes = idx->hot_mask ? (int64_t)idx->n_pad * 16 : 0;
    o->encode_ms = idx->encode_ms;
    return EBR_OK;
}

}  // extern "C"
