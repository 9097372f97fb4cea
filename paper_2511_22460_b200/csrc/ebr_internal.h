// ebr_internal.h -- library-internal types shared by the host code and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ebr.h"

// Device-resident, immutable index of one inventory shard.
struct ebr_index {
    int device;
    int dtype;              // ebr_dtype
    int32_t d, d_pad;       // embedding width, padded kernel width (zeros; exact)
    int64_t n_ads;          // shard size
    int64_t n_pad;          // rows of A (multiple of 128; padded rows are zero)
    int64_t ad_begin;       // global id of local ad 0
    int32_t n_fields;
    int64_t n_keys;         // M
    int64_t nnz, n_chunks, n_words;
    // device arrays
    void* A;                        // [n_pad][d_pad] fp32 or bf16
    uint32_t* key_chunk_off;        // [M+1]
    uint32_t* key_word_off;         // [M]
    uint2* chunk_hdr;               // [C]  {first local id, meta}
    uint32_t* chunk_last;           // [C]  last local id of each chunk (exact chunk spans per ad range)
    uint32_t* payload;              // [W + 2] (2 guard words)
    float* cross_w;                 // [M]
    int32_t* field_card;            // [F]
    int32_t* field_base;            // [F]
    // The hottest keys' columns of L (bf16 indexes only; DESIGN.md §6.2 "hot keys"): bit h of
    // hot_mask[a] is set iff ad a has hot key hot_key[h].  The batched path expands the bits of a
    // tile into an fp16 one-hot block on chip and contracts it on the tensor cores; those keys'
    // posting lists are then skipped.  Slots are ordered by posting count, descending.
    int32_t n_hot;                  // multiple of 64, <= kMaxHot (0: none)
    int32_t* hot_slot;              // [M] slot of key i, or -1
    int32_t* hot_key;               // [n_hot] key of each slot (-1 for unused padding slots)
    void* hot_mask;                 // [n_pad] uint4: 128 bits per ad
    int64_t hot_nnz;                // postings covered by the hot columns
    double build_ms;
    double encode_ms;               // the inverted-list part of build_ms (ebr_stats)
    int sm_count;
    int32_t max_ad_keys;            // most keys of one ad (= n_fields for ad_feat builds; key lists: the max)
    void* tmap_A;                   // CUtensorMap (host copy) for the tcgen05 path, or null
};

namespace ebr {

// Fixed design constants.
constexpr int kHistBits = 11;               // first-level radix histogram of ord(score)
constexpr int kHistBins = 1 << kHistBits;
constexpr int kSmallMaxB = 4;               // users per launch of the latency-path kernel
constexpr int kThreads = 512;               // CTA size of the small-batch / select kernels
constexpr int kMaxHot = 128;                // hot-key columns per index (bf16 indexes; one 128-bit mask per ad)

struct QueryArgs {
    const ebr_index* idx;
    const void* user_emb;
    int32_t batch;
    const int32_t* user_feat;
    const float* user_x;
    int32_t slots;
    int32_t k;
    int32_t* out_ids;
    float* out_scores;
    uint64_t* out_keys;
    void* workspace;
    size_t workspace_bytes;
    cudaStream_t stream;
};

size_t workspace_bytes(const ebr_index* idx, int32_t batch, int32_t slots, int32_t k);
ebr_status run_query(const QueryArgs& q);
ebr_status run_merge(const uint64_t* gathered, int32_t G, int32_t batch, int32_t k,
                     int32_t* out_ids, float* out_scores, cudaStream_t stream);
ebr_status run_debug_decode(const ebr_index* idx, int64_t key, int32_t* dev_out, int64_t cap,
                            cudaStream_t stream);
ebr_status set_error(ebr_status st, const char* fmt, ...);

// Dominant-kernel timer (ebr_kernel_timer*, measurement support): while enabled, a KernelTimer
// scope records a CUDA event pair on `stream` around the launch it encloses (skipped while the
// stream is being captured into a graph).
struct KernelTimer {
    cudaEvent_t a = nullptr;
    cudaStream_t s = nullptr;
    KernelTimer(cudaStream_t stream, const char* name);
    ~KernelTimer();
};
ebr_status cuda_check(cudaError_t e, const char* what);

}  // namespace ebr
