// ebr_build_dev.cu -- A0 on the device: the compressed inverted list of
// L built by GPU kernels instead of the host encoder, bit-identical to it (the same chunk codec,
// DESIGN.md §4.2), so that an inventory refresh ("every few minutes") costs tens
// of milliseconds next to the queries instead of seconds of host time.
//
// Alg. 1 builds, for every key, the ascending list of ads holding it, cuts it into
// blocks and compresses them; every loop of it is data-parallel ("in parallel").  Here:
//   1. pairs (key, ad) for every (ad, field) slot, key = base_f + v (empty slots -> key M, sorted
//      last); values outside [-1, V_f) raise a device flag (EBR_EINVAL);
//   2. a stable radix sort by key (cub::DeviceRadixSort, LSD: the ads of a key stay ascending);
//   3. postings per key (warp-aggregated counts over the sorted keys), exclusive scans -> the
//      postings / chunk offsets of every key;
//   4. one warp per 32-posting chunk: first id, last id, gaps - 1, bit width b; scan of the chunk
//      payload word counts -> each key's word base and each chunk's relative offset; the payload
//      bits are OR-ed into place (lanes whose fields straddle a word write two words).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "ebr_device.cuh"

namespace ebr {
namespace build {

__global__ void pairs_kernel(const int32_t* __restrict__ feat, int64_t n, int F, const int32_t* __restrict__ card,
                             const int32_t* __restrict__ base, uint32_t M, uint32_t* __restrict__ keys,
                             int32_t* __restrict__ ads, uint32_t* err) {
    const int64_t N = n * F;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = i / F;
        const int f = (int)(i - a * F);
        const int32_t v = feat[i];
        uint32_t k = M;
        if (v < -1 || v >= __ldg(&card[f])) atomicOr(err, 1u);
        else if (v >= 0) k = (uint32_t)(__ldg(&base[f]) + v);
        keys[i] = k;
        ads[i] = (int32_t)a;
    }
}

// pairs given ad by ad (multi-valued fields): thread = ad, its keys in order (ads ascending in the
// pair order, so the stable key sort keeps each list ascending); keys outside [0, M) flagged
__global__ void pairs_from_lists_kernel(const int64_t* __restrict__ off, const int32_t* __restrict__ ad_keys,
                                        int64_t n, uint32_t M, uint32_t* __restrict__ keys, int32_t* __restrict__ ads,
                                        uint32_t* err) {
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
        for (int64_t q = off[a]; q < off[a + 1]; ++q) {
            const int32_t k = ad_keys[q];
            const bool ok = k >= 0 && (uint32_t)k < M;
            if (!ok) atomicOr(err, 1u);
            keys[q] = ok ? (uint32_t)k : M;
            ads[q] = (int32_t)a;
        }
}

// after the sort: a (key, ad) pair listed twice for one ad is an error (L is binary)
__global__ void duplicate_check_kernel(const uint32_t* __restrict__ keys, const int32_t* __restrict__ ads, int64_t N,
                                       uint32_t M, uint32_t* err) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < N; i += (int64_t)gridDim.x * blockDim.x)
        if (keys[i] < M && keys[i] == keys[i - 1] && ads[i] == ads[i - 1]) atomicOr(err, 4u);
}

// postings per key over the sorted keys (equal keys are adjacent: one atomic per run per warp)
__global__ void count_kernel(const uint32_t* __restrict__ keys, int64_t N, uint32_t M, uint32_t* __restrict__ count) {
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; i0 < N;
         i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + lane;
        const uint32_t k = i < N ? keys[i] : M;
        const unsigned peers = __match_any_sync(FULL, k);
        if (k < M && lane == __ffs(peers) - 1) atomicAdd(&count[k], (uint32_t)__popc(peers));
    }
}

__global__ void chunks_per_key_kernel(const uint32_t* __restrict__ count, uint32_t M, uint32_t* __restrict__ nch) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < M) nch[k] = (count[k] + 31u) / 32u;
}

// chunk -> key: the first chunk of every key holds the key, a max-scan fills the rest
__global__ void chunk_key_seed_kernel(const uint32_t* __restrict__ key_chunk_off, uint32_t M, uint32_t* __restrict__ ck) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < M && key_chunk_off[k + 1] > key_chunk_off[k]) ck[key_chunk_off[k]] = k;
}

// one warp per chunk: first / last id, bit width, payload words (pass A); pass B writes the header
// with the relative word offset and OR-s the b-bit fields into the payload
template <int PASS>
__global__ void chunk_kernel(const uint32_t* __restrict__ ck, const uint32_t* __restrict__ key_chunk_off,
                             const uint32_t* __restrict__ post_off, const uint32_t* __restrict__ count,
                             const int32_t* __restrict__ ads, uint64_t C, uint32_t* __restrict__ words,
                             const uint32_t* __restrict__ word_start, uint32_t* __restrict__ key_word_off,
                             uint32_t* __restrict__ hdr, uint32_t* __restrict__ last, uint32_t* __restrict__ payload,
                             uint32_t* err) {
    const int lane = threadIdx.x & 31;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < C; c += nw) {
        const uint32_t k = ck[c];
        const uint32_t lc = (uint32_t)c - key_chunk_off[k];
        const uint32_t n = min(32u, count[k] - 32u * lc);
        const uint32_t p = post_off[k] + 32u * lc + (uint32_t)lane;
        const uint32_t id = (uint32_t)lane < n ? (uint32_t)ads[p] : 0u;
        const uint32_t prev = __shfl_up_sync(FULL, id, 1);
        const uint32_t g = (lane >= 1 && (uint32_t)lane < n) ? id - prev - 1u : 0u;
        uint32_t mx = g;
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
        const uint32_t b = mx ? 32u - (uint32_t)__clz(mx) : 0u;
        if (PASS == 0) {
            if (lane == 0) words[c] = (uint32_t)(((uint64_t)(n - 1) * b + 31) / 32);
        } else {
            const uint32_t kwo = word_start[key_chunk_off[k]];
            const uint32_t rel = word_start[c] - kwo;
            if (lane == 0) {
                if (rel >= (1u << 22)) atomicOr(err, 2u);     // relative word offset field is 22 bits
                if (lc == 0) key_word_off[k] = kwo;
                hdr[2 * c] = id;
                hdr[2 * c + 1] = (n - 1u) | (b << 5) | (rel << 10);
            }
            if ((uint32_t)lane == n - 1u) last[c] = id;
            if (b && lane >= 1 && (uint32_t)lane < n) {
                const uint64_t pos = (uint64_t)(lane - 1) * b;
                uint32_t* w = payload + kwo + rel + (pos >> 5);
                const uint32_t sh = (uint32_t)(pos & 31);
                atomicOr(&w[0], g << sh);
                if (sh + b > 32) atomicOr(&w[1], g >> (32 - sh));
            }
        }
    }
}

// keys without postings: their word base is the running total at their position
__global__ void empty_key_word_off_kernel(const uint32_t* __restrict__ key_chunk_off, const uint32_t* __restrict__ word_start,
                                          uint32_t M, uint32_t* __restrict__ key_word_off) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < M && key_chunk_off[k + 1] == key_chunk_off[k]) key_word_off[k] = word_start[key_chunk_off[k]];
}

struct Max {
    __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

}  // namespace build

// Device encoder: d_feat [n][F] on the device; fills idx's posting arrays (and n_chunks, n_words,
// nnz) and returns the postings per key on the host (hot-key selection).  Host-synchronous.
ebr_status device_encode(ebr_index* idx, const int32_t* d_feat, const int32_t* d_card, const int32_t* d_base,
                         cudaStream_t st, std::vector<int64_t>& key_count, const int64_t* d_off,
                         const int32_t* d_keys, int64_t nnz) {
    using namespace build;
    const int64_t n = idx->n_ads;
    const int F = idx->n_fields;
    const uint32_t M = (uint32_t)idx->n_keys;
    const bool lists = d_off != nullptr;                 // (ad, key) pairs given ad by ad
    const int64_t N = lists ? nnz : n * F;
    std::vector<void*> tmp;
    auto dalloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return nullptr;
        tmp.push_back(p);
        return p;
    };
    auto release = [&]() { for (void* p : tmp) cudaFree(p); tmp.clear(); };
#define EBR_DTRY(call) do { cudaError_t e__ = (call); if (e__ != cudaSuccess) { release(); return cuda_check(e__, #call); } } while (0)
#define EBR_DALLOC(var, type, count) type* var = static_cast<type*>(dalloc((size_t)(count) * sizeof(type))); \
    if (!var) { release(); return set_error(EBR_ENOMEM, "device build: cudaMalloc failed"); }
    EBR_DALLOC(err, uint32_t, 4);
    EBR_DTRY(cudaMemsetAsync(err, 0, 16, st));
    EBR_DALLOC(keys, uint32_t, N);
    EBR_DALLOC(ads, int32_t, N);
    EBR_DALLOC(keys2, uint32_t, N);
    EBR_DALLOC(ads2, int32_t, N);
    const int grid = 4 * idx->sm_count;
    if (lists) pairs_from_lists_kernel<<<grid, 256, 0, st>>>(d_off, d_keys, n, M, keys, ads, err);
    else pairs_kernel<<<grid, 256, 0, st>>>(d_feat, n, F, d_card, d_base, M, keys, ads, err);
    EBR_DTRY(cudaGetLastError());
    int bits = 1;
    while (bits < 32 && ((uint64_t)1 << bits) <= (uint64_t)M) ++bits;     // key M (empty) included
    cub::DoubleBuffer<uint32_t> kb(keys, keys2);
    cub::DoubleBuffer<int32_t> vb(ads, ads2);
    size_t tbytes = 0;
    EBR_DTRY(cub::DeviceRadixSort::SortPairs(nullptr, tbytes, kb, vb, N, 0, bits, st));
    void* tsort = dalloc(tbytes);
    if (!tsort) { release(); return set_error(EBR_ENOMEM, "device build: sort workspace"); }
    EBR_DTRY(cub::DeviceRadixSort::SortPairs(tsort, tbytes, kb, vb, N, 0, bits, st));
    const uint32_t* skeys = kb.Current();
    const int32_t* sads = vb.Current();
    if (lists) duplicate_check_kernel<<<grid, 256, 0, st>>>(skeys, sads, N, M, err);
    EBR_DALLOC(count, uint32_t, M + 1);
    EBR_DTRY(cudaMemsetAsync(count, 0, (size_t)(M + 1) * 4, st));
    count_kernel<<<grid, 256, 0, st>>>(skeys, N, M, count);
    EBR_DTRY(cudaGetLastError());
    EBR_DALLOC(post_off, uint32_t, M + 1);
    EBR_DALLOC(nch, uint32_t, M + 1);
    size_t sb = 0;
    EBR_DTRY(cub::DeviceScan::ExclusiveSum(nullptr, sb, count, post_off, M + 1, st));
    void* tscan = dalloc(std::max<size_t>(sb, 1 << 20) * 2);
    if (!tscan) { release(); return set_error(EBR_ENOMEM, "device build: scan workspace"); }
    size_t tscan_bytes = std::max<size_t>(sb, 1 << 20) * 2;
    EBR_DTRY(cub::DeviceScan::ExclusiveSum(tscan, sb, count, post_off, M + 1, st));
    chunks_per_key_kernel<<<(M + 255) / 256, 256, 0, st>>>(count, M, nch);
    EBR_DTRY(cudaMemsetAsync(nch + M, 0, 4, st));
    EBR_DTRY(cudaMalloc(&idx->key_chunk_off, (size_t)(M + 1) * 4));
    sb = 0;
    EBR_DTRY(cub::DeviceScan::ExclusiveSum(nullptr, sb, nch, idx->key_chunk_off, M + 1, st));
    if (sb > tscan_bytes) { release(); return set_error(EBR_ENOMEM, "device build: scan workspace"); }
    EBR_DTRY(cub::DeviceScan::ExclusiveSum(tscan, sb, nch, idx->key_chunk_off, M + 1, st));
    uint32_t totals[2] = {0, 0};
    EBR_DTRY(cudaMemcpyAsync(&totals[0], idx->key_chunk_off + M, 4, cudaMemcpyDeviceToHost, st));
    EBR_DTRY(cudaMemcpyAsync(&totals[1], post_off + M, 4, cudaMemcpyDeviceToHost, st));
    key_count.assign(M, 0);
    std::vector<uint32_t> hc(M);
    if (M) EBR_DTRY(cudaMemcpyAsync(hc.data(), count, (size_t)M * 4, cudaMemcpyDeviceToHost, st));
    EBR_DTRY(cudaStreamSynchronize(st));
    for (uint32_t k = 0; k < M; ++k) key_count[k] = hc[k];
    const uint64_t C = totals[0];
    idx->nnz = totals[1];
    idx->n_chunks = (int64_t)C;
    EBR_DALLOC(ck0, uint32_t, C + 1);
    EBR_DALLOC(ck, uint32_t, C + 1);
    EBR_DTRY(cudaMemsetAsync(ck0, 0, (size_t)(C + 1) * 4, st));
    chunk_key_seed_kernel<<<(M + 255) / 256, 256, 0, st>>>(idx->key_chunk_off, M, ck0);
    sb = 0;
    EBR_DTRY(cub::DeviceScan::InclusiveScan(nullptr, sb, ck0, ck, Max(), C ? C : 1, st));
    if (sb > tscan_bytes) { release(); return set_error(EBR_ENOMEM, "device build: scan workspace"); }
    if (C) EBR_DTRY(cub::DeviceScan::InclusiveScan(tscan, sb, ck0, ck, Max(), C, st));
    EBR_DALLOC(words, uint32_t, C + 1);
    EBR_DALLOC(word_start, uint32_t, C + 1);
    EBR_DTRY(cudaMemsetAsync(words, 0, (size_t)(C + 1) * 4, st));
    const int cgrid = (int)std::min<uint64_t>((C + 7) / 8 + 1, (uint64_t)64 * idx->sm_count);
    if (C) chunk_kernel<0><<<cgrid, 256, 0, st>>>(ck, idx->key_chunk_off, post_off, count, sads, C, words, nullptr,
                                                  nullptr, nullptr, nullptr, nullptr, err);
    EBR_DTRY(cudaGetLastError());
    sb = 0;
    EBR_DTRY(cub::DeviceScan::ExclusiveSum(nullptr, sb, words, word_start, C + 1, st));
    if (sb > tscan_bytes) { release(); return set_error(EBR_ENOMEM, "device build: scan workspace"); }
    EBR_DTRY(cub::DeviceScan::ExclusiveSum(tscan, sb, words, word_start, C + 1, st));
    uint32_t W = 0;
    EBR_DTRY(cudaMemcpyAsync(&W, word_start + C, 4, cudaMemcpyDeviceToHost, st));
    EBR_DTRY(cudaStreamSynchronize(st));
    idx->n_words = W;
    EBR_DTRY(cudaMalloc(&idx->key_word_off, (size_t)std::max<uint32_t>(M, 1) * 4));
    EBR_DTRY(cudaMalloc(&idx->chunk_hdr, (size_t)std::max<uint64_t>(C, 1) * 8));
    EBR_DTRY(cudaMalloc(&idx->chunk_last, (size_t)std::max<uint64_t>(C, 1) * 4));
    EBR_DTRY(cudaMalloc(&idx->payload, (size_t)(W + 2) * 4));
    EBR_DTRY(cudaMemsetAsync(idx->payload, 0, (size_t)(W + 2) * 4, st));
    if (M) empty_key_word_off_kernel<<<(M + 255) / 256, 256, 0, st>>>(idx->key_chunk_off, word_start, M, idx->key_word_off);
    if (C) chunk_kernel<1><<<cgrid, 256, 0, st>>>(ck, idx->key_chunk_off, post_off, count, sads, C, words, word_start,
                                                  idx->key_word_off, reinterpret_cast<uint32_t*>(idx->chunk_hdr),
                                                  idx->chunk_last, idx->payload, err);
    EBR_DTRY(cudaGetLastError());
    uint32_t herr = 0;
    EBR_DTRY(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
    EBR_DTRY(cudaStreamSynchronize(st));
    release();
#undef EBR_DTRY
#undef EBR_DALLOC
    if (herr & 1u) return set_error(EBR_EINVAL, lists ? "ad key outside [0, n_keys)" : "ad_feat value outside [-1, V_f)");
    if (herr & 4u) return set_error(EBR_EINVAL, "a key listed twice for one ad (L is binary)");
    if (herr & 2u) return set_error(EBR_EUNSUPPORTED, "a posting list exceeds 2^22 payload words");
    return EBR_OK;
}

}  // namespace ebr
