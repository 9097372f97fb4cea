// ebr_paper.cu -- SURVEY.md §8(f) NEXT-3: the paper's own GPU inverted list, built and queried on
// B200 as an ablation of this library's chunk codec (never a dispatch path of the hot path).
//
// Index (Alg. 1; "Block Grouping / Logarithmic Categorization / Block
// Compression / Storage Layout", l.291-295): every key's ascending ad list is split into blocks of
// ads sharing the high 24 bits h = ad >> 8; a block of n ads goes to group g = ceil(log2 n)
// (n = 1 -> 0) and is padded to 2^g one-byte residuals l = ad & 255; per group, a struct of
// arrays: key offsets [M+1] (reading R6: the garbled keys loop is a CSR of each key's blocks),
// headers (h << 8 | (n - 1): the count in the header word neutralises the "pad with 0" of Alg. 1,
// reading R5 / S:204), values (2^g bytes per block).
//
// Query (Alg. 2, l.346-364): for one user's (key, w~) items, for every group in parallel: the
// items' block counts, their exclusive scan, a load-balanced assignment of (block, lane) work to
// threads (the merge-based balance of l.302-304 realised as a flat index space searched per
// thread), and AtomicAdd(scores[h 2^8 + l], w~) (l.358) into a global fp32 score array.
//
// The chunk-codec counterpart (ebr_chunk_hitmatch) runs the same algorithm -- flat chunk space,
// warp-cooperative decode, fp32 AtomicAdd into global scores -- on this library's index, so the
// two layouts are compared on equal terms.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "ebr_device.cuh"

struct ebr_paper_index {
    int device;
    int64_t n_ads, n_keys;
    int64_t blocks[9];          // blocks per group
    uint32_t* key_off[9];       // [M+1] per group
    uint32_t* header[9];        // [blocks] h << 8 | (n - 1)
    uint8_t* values[9];         // [blocks << g]
    int64_t bytes;              // device bytes of the index
    double build_ms;
};

namespace ebr {
using PaperIndex = ::ebr_paper_index;

namespace paper {

constexpr int kMaxItems = 1024;     // query items per call (64 at C2: 32 fields x 2 slots)

// one kernel for all 9 groups: blockIdx.y = group; threads walk the group's flat (block, lane)
// space; a lane covers residual positions lane, lane + span, ... of its block
__global__ void __launch_bounds__(256) hitmatch_kernel(PaperIndex pi, const int32_t* __restrict__ keys,
                                                       const float* __restrict__ w, int n_items,
                                                       float* __restrict__ scores) {
    const int g = blockIdx.y;
    if (pi.blocks[g] == 0) return;
    __shared__ uint32_t seg[kMaxItems + 1];      // exclusive scan of the items' block counts
    __shared__ uint32_t beg[kMaxItems];
    const uint32_t* ko = pi.key_off[g];
    // k_length, k_seg (Alg. 2 l.352-353): block-wide scan in shared memory (items <= 1024)
    for (int i = threadIdx.x; i < n_items; i += blockDim.x) {
        const int32_t k = keys[i];
        const uint32_t b = (k >= 0 && k < pi.n_keys) ? __ldg(&ko[k]) : 0u;
        const uint32_t e = (k >= 0 && k < pi.n_keys) ? __ldg(&ko[k + 1]) : 0u;
        beg[i] = b;
        seg[i + 1] = e - b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        seg[0] = 0;
        for (int i = 0; i < n_items; ++i) seg[i + 1] += seg[i];
    }
    __syncthreads();
    const uint32_t total = seg[n_items];
    const int len = 1 << g;                          // padded block length
    const int span = min(len, 32);                   // lanes per block
    const uint64_t work = (uint64_t)total * span;
    const uint32_t* hdr = pi.header[g];
    const uint8_t* val = pi.values[g];
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < work; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(t / span), lane = (uint32_t)(t % span);
        // LoadBalance (l.354): the item owning flat block j (upper bound in seg)
        int lo = 0, hi = n_items;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (seg[mid] <= j) lo = mid;
            else hi = mid;
        }
        const uint32_t blk = beg[lo] + (j - seg[lo]);
        const uint32_t h = __ldg(&hdr[blk]);
        const uint32_t n = (h & 0xFFu) + 1u;         // valid residuals (padding lanes skipped)
        const float wk = __ldg(&w[lo]);
        const uint32_t base = (h >> 8) << 8;
        for (uint32_t q = lane; q < n; q += span)
            atomicAdd(&scores[base + __ldg(&val[((size_t)blk << g) + q])], wk);   // Alg. 2 l.358
    }
}

}  // namespace paper

// the same algorithm on the chunk codec: flat chunk space over the items, warp per chunk
__global__ void __launch_bounds__(256) chunk_hitmatch_kernel(const uint32_t* __restrict__ key_chunk_off,
                                                             const uint32_t* __restrict__ key_word_off,
                                                             const uint2* __restrict__ hdr,
                                                             const uint32_t* __restrict__ payload, int64_t n_keys,
                                                             const int32_t* __restrict__ keys,
                                                             const float* __restrict__ w, int n_items,
                                                             float* __restrict__ scores) {
    __shared__ uint32_t seg[paper::kMaxItems + 1];
    __shared__ uint32_t beg[paper::kMaxItems], kwb[paper::kMaxItems];
    for (int i = threadIdx.x; i < n_items; i += blockDim.x) {
        const int32_t k = keys[i];
        const bool ok = k >= 0 && k < n_keys;
        const uint32_t b = ok ? __ldg(&key_chunk_off[k]) : 0u, e = ok ? __ldg(&key_chunk_off[k + 1]) : 0u;
        beg[i] = b;
        kwb[i] = ok ? __ldg(&key_word_off[k]) : 0u;
        seg[i + 1] = e - b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        seg[0] = 0;
        for (int i = 0; i < n_items; ++i) seg[i + 1] += seg[i];
    }
    __syncthreads();
    const uint32_t total = seg[n_items];
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < total; j += nw) {
        int lo = 0, hi = n_items;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (seg[mid] <= j) lo = mid;
            else hi = mid;
        }
        const uint32_t c = beg[lo] + (j - seg[lo]);
        uint32_t id;
        if (decode_chunk(hdr, payload, kwb[lo], c, lane, id)) atomicAdd(&scores[id], __ldg(&w[lo]));
    }
}

}  // namespace ebr

using namespace ebr;

extern "C" {

ebr_status ebr_paper_index_build(const int32_t* ad_feat, int64_t n_ads, int32_t n_fields,
                                 const int32_t* field_card, int64_t n_keys, int device, void* stream_v,
                                 PaperIndex** out) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!out || !ad_feat || !field_card || n_ads < 1 || n_fields < 1) return set_error(EBR_EINVAL, "bad arguments");
    *out = nullptr;
    std::vector<int64_t> base(n_fields + 1, 0);
    for (int f = 0; f < n_fields; ++f) base[f + 1] = base[f] + field_card[f];
    if (base[n_fields] != n_keys) return set_error(EBR_EINVAL, "n_keys != sum(field_card)");
    for (int64_t i = 0; i < n_ads * n_fields; ++i) {
        const int f = (int)(i % n_fields);
        if (ad_feat[i] < -1 || ad_feat[i] >= field_card[f]) return set_error(EBR_EINVAL, "ad_feat out of range");
    }
    // Alg. 1 step 1: (key, ad) lists ascending (counting sort by key)
    std::vector<int64_t> koff(n_keys + 1, 0);
    for (int64_t a = 0; a < n_ads; ++a)
        for (int f = 0; f < n_fields; ++f) {
            const int32_t v = ad_feat[a * n_fields + f];
            if (v >= 0) koff[base[f] + v + 1]++;
        }
    for (int64_t k = 0; k < n_keys; ++k) koff[k + 1] += koff[k];
    std::vector<int32_t> ads(koff[n_keys]);
    {
        std::vector<int64_t> fill(koff.begin(), koff.end() - 1);
        for (int64_t a = 0; a < n_ads; ++a)
            for (int f = 0; f < n_fields; ++f) {
                const int32_t v = ad_feat[a * n_fields + f];
                if (v >= 0) ads[fill[base[f] + v]++] = (int32_t)a;
            }
    }
    // steps 2-3: blocks by h, groups by ceil(log2 n), per-group SoA (blocks ordered by key, then h)
    std::vector<std::vector<uint32_t>> goff(9, std::vector<uint32_t>(n_keys + 1, 0));
    std::vector<std::vector<uint32_t>> ghdr(9);
    std::vector<std::vector<uint8_t>> gval(9);
    for (int64_t k = 0; k < n_keys; ++k) {
        for (int g = 0; g < 9; ++g) goff[g][k] = (uint32_t)ghdr[g].size();
        for (int64_t i = koff[k]; i < koff[k + 1];) {
            const int32_t h = ads[i] >> 8;
            int64_t e = i;
            while (e < koff[k + 1] && (ads[e] >> 8) == h) ++e;
            const int n = (int)(e - i);
            int g = 0;
            while ((1 << g) < n) ++g;
            ghdr[g].push_back(((uint32_t)h << 8) | (uint32_t)(n - 1));
            for (int q = 0; q < (1 << g); ++q) gval[g].push_back(q < n ? (uint8_t)(ads[i + q] & 255) : (uint8_t)0);
            i = e;
        }
    }
    for (int g = 0; g < 9; ++g) goff[g][n_keys] = (uint32_t)ghdr[g].size();
    PaperIndex* pi = new PaperIndex();
    memset(pi, 0, sizeof(*pi));
    pi->device = device;
    pi->n_ads = n_ads;
    pi->n_keys = n_keys;
    cudaStream_t st = static_cast<cudaStream_t>(stream_v);
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaError_t e = cudaSuccess;
    for (int g = 0; g < 9 && e == cudaSuccess; ++g) {
        pi->blocks[g] = (int64_t)ghdr[g].size();
        e = cudaMalloc(&pi->key_off[g], (size_t)(n_keys + 1) * 4);
        if (e == cudaSuccess) e = cudaMemcpyAsync(pi->key_off[g], goff[g].data(), (size_t)(n_keys + 1) * 4, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMalloc(&pi->header[g], std::max<size_t>(4, ghdr[g].size() * 4));
        if (e == cudaSuccess && !ghdr[g].empty())
            e = cudaMemcpyAsync(pi->header[g], ghdr[g].data(), ghdr[g].size() * 4, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMalloc(&pi->values[g], std::max<size_t>(4, gval[g].size()));
        if (e == cudaSuccess && !gval[g].empty())
            e = cudaMemcpyAsync(pi->values[g], gval[g].data(), gval[g].size(), cudaMemcpyHostToDevice, st);
        pi->bytes += (int64_t)(n_keys + 1) * 4 + (int64_t)ghdr[g].size() * 4 + (int64_t)gval[g].size();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (prev >= 0) cudaSetDevice(prev);
    if (e != cudaSuccess) {
        for (int g = 0; g < 9; ++g) { cudaFree(pi->key_off[g]); cudaFree(pi->header[g]); cudaFree(pi->values[g]); }
        delete pi;
        return cuda_check(e, "paper index upload");
    }
    pi->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *out = pi;
    return EBR_OK;
}

void ebr_paper_index_free(PaperIndex* pi) {
    if (!pi) return;
    for (int g = 0; g < 9; ++g) { cudaFree(pi->key_off[g]); cudaFree(pi->header[g]); cudaFree(pi->values[g]); }
    delete pi;
}

ebr_status ebr_paper_index_info(const PaperIndex* pi, int64_t* blocks9, int64_t* bytes, double* build_ms) {
    if (!pi) return set_error(EBR_EINVAL, "null index");
    if (blocks9) for (int g = 0; g < 9; ++g) blocks9[g] = pi->blocks[g];
    if (bytes) *bytes = pi->bytes;
    if (build_ms) *build_ms = pi->build_ms;
    return EBR_OK;
}

ebr_status ebr_paper_hitmatch(const PaperIndex* pi, const int32_t* keys, const float* w, int32_t n_items,
                              float* scores, void* stream_v) {
    if (!pi || !keys || !w || !scores) return set_error(EBR_EINVAL, "null pointer");
    if (n_items < 0 || n_items > paper::kMaxItems) return set_error(EBR_EINVAL, "n_items must be in [0, 1024]");
    cudaStream_t st = static_cast<cudaStream_t>(stream_v);
    cudaError_t e = cudaMemsetAsync(scores, 0, (size_t)pi->n_ads * 4, st);    // Alg. 2 l.350
    if (e != cudaSuccess) return cuda_check(e, "memset(scores)");
    if (n_items == 0) return EBR_OK;
    paper::hitmatch_kernel<<<dim3(148, 9), 256, 0, st>>>(*pi, keys, w, n_items, scores);
    return cuda_check(cudaGetLastError(), "launch(paper hitmatch)");
}

ebr_status ebr_chunk_hitmatch(const ebr_index* idx, const int32_t* keys, const float* w, int32_t n_items,
                              float* scores, void* stream_v) {
    if (!idx || !keys || !w || !scores) return set_error(EBR_EINVAL, "null pointer");
    if (n_items < 0 || n_items > paper::kMaxItems) return set_error(EBR_EINVAL, "n_items must be in [0, 1024]");
    cudaStream_t st = static_cast<cudaStream_t>(stream_v);
    cudaError_t e = cudaMemsetAsync(scores, 0, (size_t)idx->n_ads * 4, st);
    if (e != cudaSuccess) return cuda_check(e, "memset(scores)");
    if (n_items == 0) return EBR_OK;
    chunk_hitmatch_kernel<<<4 * idx->sm_count, 256, 0, st>>>(idx->key_chunk_off, idx->key_word_off, idx->chunk_hdr,
                                                           idx->payload, idx->n_keys, keys, w, n_items, scores);
    return cuda_check(cudaGetLastError(), "launch(chunk hitmatch)");
}

}  // extern "C"

// ------------------------------------------------------------------------------------------
// NEXT-4: the IPNN extension of a tower output (Eq. 7-8): h~ = [h, W u] per row, the
// W u part accumulated in fp32 and rounded once to the index dtype.  Rows = users (per query,
// before ebr_score_topk) or ads (before ebr_build_index).
// ------------------------------------------------------------------------------------------
namespace ebr {
template <typename T>
__global__ void __launch_bounds__(256) ipnn_kernel(const T* __restrict__ h, const float* __restrict__ u,
                                                   const float* __restrict__ W, int64_t rows, int d0, int n, int d1,
                                                   T* __restrict__ out) {
    extern __shared__ float su[];                    // [n] this row's u
    for (int64_t b = blockIdx.x; b < rows; b += gridDim.x) {
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) su[i] = u[b * n + i];
        __syncthreads();
        T* o = out + b * (int64_t)(d0 + d1);
        for (int j = threadIdx.x; j < d0; j += blockDim.x) o[j] = h[b * d0 + j];
        for (int j = threadIdx.x; j < d1; j += blockDim.x) {
            const float* wr = W + (int64_t)j * n;
            float s = 0.f;
            for (int i = 0; i < n; ++i) s = fmaf(__ldg(&wr[i]), su[i], s);
            if constexpr (sizeof(T) == 2) o[d0 + j] = __float2bfloat16_rn(s);
            else o[d0 + j] = s;
        }
    }
}
}  // namespace ebr

extern "C" ebr_status ebr_ipnn_extend(const void* h, const float* u, const float* W, int64_t rows, int32_t d0,
                                      int32_t n, int32_t d1, ebr_dtype dtype, void* out, void* stream_v) {
    if (!out || (d0 > 0 && !h) || (n > 0 && (!u || !W))) return set_error(EBR_EINVAL, "null pointer");
    if (rows < 0 || d0 < 0 || n < 0 || d1 < 0 || n > 12 * 1024) return set_error(EBR_EINVAL, "bad sizes");
    if (dtype != EBR_F32 && dtype != EBR_BF16) return set_error(EBR_EINVAL, "bad dtype");
    if (rows == 0) return EBR_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream_v);
    const unsigned grid = (unsigned)std::min<int64_t>(rows, 148 * 16);
    if (dtype == EBR_BF16)
        ipnn_kernel<__nv_bfloat16><<<grid, 256, (size_t)n * 4, st>>>(static_cast<const __nv_bfloat16*>(h), u, W, rows,
                                                                    d0, n, d1, static_cast<__nv_bfloat16*>(out));
    else
        ipnn_kernel<float><<<grid, 256, (size_t)n * 4, st>>>(static_cast<const float*>(h), u, W, rows, d0, n, d1,
                                                            static_cast<float*>(out));
    return cuda_check(cudaGetLastError(), "launch(ipnn)");
}
