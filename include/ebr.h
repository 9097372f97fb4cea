/*
 * ebr.h -- C-ABI of the B200-native Wide & Deep ad-retrieval scorer (arXiv 2511.22460).
 *
 * One hot path: score every ad of an inventory shard for a batch of users as
 *     s(u,a) = <h~_u, h~_a> + sum_i w_i x_i L_{a,i}          (Eq. 9, l.253-257)
 * -- the dual-tower inner product ("deep", Eq. 1 l.188 / Eq. 8 l.243) plus the HitMatch cross
 * features ("wide", l.251-252), the latter read through a compressed inverted list of L
 * (l.280-296, Alg. 1 l.309-344, Alg. 2 l.346-364) -- and return each user's top-K ads
 * ("retrieve top k relevant ads", l.157), ties broken by ascending ad id.
 *
 * Citations "P:n" are /root/reference/PAPER.md lines.  Readings of the paper where it is silent
 * or ambiguous are numbered R1..R21 in DESIGN.md.
 *
 * Conventions for every call
 *   - No exception crosses the ABI.  Every call returns an ebr_status; on failure a thread-local
 *     message is available from ebr_last_error().
 *   - Pointers documented "host" are CPU memory; "device" pointers are CUDA device memory on the
 *     index's device (e.g. torch tensor storage).  All device memory passed in is caller-owned;
 *     memory behind an ebr_index is library-owned and released by ebr_free_index().
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls marked
 *     "async" only enqueue work on it; their device outputs are valid after the stream syncs.
 *     Kernel faults surface at the caller's next synchronisation.
 *   - There is no CPU fallback: with no usable sm_100 device every compute call fails with
 *     EBR_ECUDA / EBR_EUNSUPPORTED.
 */
#ifndef EBR_H_
#define EBR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ebr_index ebr_index; /* opaque; immutable after build, shareable across streams */

typedef enum {
    EBR_OK = 0,
    EBR_EINVAL = 1,         /* bad argument (bounds, sizes, undersized workspace)            */
    EBR_ENOMEM = 2,         /* host or device allocation failed                               */
    EBR_ECUDA = 3,          /* CUDA runtime error (message in ebr_last_error)                 */
    EBR_EUNSUPPORTED = 4,   /* device is not sm_100 / feature outside the supported envelope */
    EBR_EDEVICE = 5         /* a device-side validation flag was raised (see ebr_query_error) */
} ebr_status;

typedef enum { EBR_F32 = 0, EBR_BF16 = 1 } ebr_dtype;

/* Largest K one call returns (one CTA sorts the K results in shared memory). */
#define EBR_MAX_K 16384

/* ------------------------------------------------------------------------------------------ */
/* A0  Index build  (Alg. 1 l.309-344, "Storage Layout" l.295; refresh l.307)          */
/* ------------------------------------------------------------------------------------------ */
/*
 * Builds this rank's shard: global ads [ad_begin, ad_end).  Host inputs are copied; the caller
 * may free them on return.  Synchronous w.r.t. the host (uploads run on `stream`, which is
 * synchronised before return).
 *
 *  ad_emb     host, [n][d] row-major, n = ad_end - ad_begin; fp32 (EBR_F32) or raw bf16 bit
 *             patterns (EBR_BF16, uint16).  This is h~_a (Eq. 8: tower output + IPNN extension,
 *             already concatenated; reading R19).  Rows are zero-padded on the device to the
 *             kernel width (exact).
 *  ad_feat    host, [n][n_fields] int32, the ad's value v in field f, -1 = empty (L_{a,i}=0).
 *             Defines L: L[a, base_f + v] = 1 (reading R1).  Must be in [-1, V_f).
 *  field_card host, [n_fields] int32 V_f >= 1; key i = base_f + v with base_f = sum_{g<f} V_g.
 *  cross_w    host, [n_keys] fp32, the learned weight w_i of every key (Eq. 9).
 *  n_keys     must equal sum V_f and be < 2^31.
 *  device     CUDA ordinal; the index lives there.
 *  out        receives the handle.
 * Errors: EBR_EINVAL for d < 1, ad_begin >= ad_end, ad_end > 2^31-1, ad_feat out of range,
 *         n_keys != sum V_f; EBR_ENOMEM / EBR_ECUDA; EBR_EUNSUPPORTED on a non-sm_100 device.
 *
 * Device layout: ad embeddings A[n_pad][d_pad]; the posting lists of
 * every key as 32-posting chunks, delta-coded and bit-packed (DESIGN.md "Posting-chunk wire
 * format"), with an SoA directory key_chunk_off[M+1], key_word_off[M], chunk_hdr[C] (u32 pairs)
 * and payload words; w[M].  bf16 indexes also keep the up to 256 longest posting lists (>= max(64,
 * n/512) postings) as dense one-hot columns H[n_pad][n_hot] of L in bf16 for the batched
 * tensor-core path (R22; EBR_HOT_KEYS=<n> caps n_hot, 0 disables); the compressed lists
 * stay complete.  Device memory: A + H + the encoded lists (ebr_index_stats reports the sizes).
 */
ebr_status ebr_build_index(const void *ad_emb, ebr_dtype dtype, int64_t ad_begin, int64_t ad_end,
                           int32_t d, const int32_t *ad_feat, int32_t n_fields,
                           const int32_t *field_card, const float *cross_w, int64_t n_keys,
                           int device, void *stream, ebr_index **out);

/*
 * Same contract and result as ebr_build_index, with the inverted list built on the DEVICE
 * (Alg. 1, whose loops are data-parallel): ad_feat is uploaded,
 * (key, ad) pairs are radix-sorted by key on the GPU (stable: lists stay ascending), chunked,
 * delta-coded and bit-packed by GPU kernels -- the arrays are bit-identical to the host encoder's
 * (ebr_index_export).  Bounds errors in ad_feat are detected on the device (EBR_EINVAL).  Needs
 * ~20 B of temporary device memory per (ad, field) slot during the build.  Host-synchronous;
 * queries on other streams with other indexes keep running meanwhile (double-buffered refresh:
 * build the new index, swap the handle, free the old one once its queries completed).
 */
ebr_status ebr_build_index_device(const void *ad_emb, ebr_dtype dtype, int64_t ad_begin,
                                  int64_t ad_end, int32_t d, const int32_t *ad_feat,
                                  int32_t n_fields, const int32_t *field_card,
                                  const float *cross_w, int64_t n_keys, int device, void *stream,
                                  ebr_index **out);

/*
 * NEXT-4, multi-valued ad fields (tags): the same index (device build) from L given ad by
 * ad as key lists -- ad a (shard-local) holds the global keys ad_keys[ad_key_off[a] ..
 * ad_key_off[a+1]), any number per field (key = base_f + v as for ad_feat; <= 1024 keys per ad).
 * L is binary: a key listed twice for one ad is EBR_EINVAL; keys outside [0, n_keys) are EBR_EINVAL.
 *  ad_key_off host [n + 1] int64 (ad_key_off[0] = 0, ascending), ad_keys host [ad_key_off[n]] int32.
 * Every other argument and the result as ebr_build_index_device.  The query calls are unchanged.
 */
ebr_status ebr_build_index_lists(const void *ad_emb, ebr_dtype dtype, int64_t ad_begin,
                                 int64_t ad_end, int32_t d, const int64_t *ad_key_off,
                                 const int32_t *ad_keys, int32_t n_fields, const int32_t *field_card,
                                 const float *cross_w, int64_t n_keys, int device, void *stream,
                                 ebr_index **out);

void ebr_free_index(ebr_index *idx);

/* ------------------------------------------------------------------------------------------ */
/* A1-A6  Query: plan, posting decode, wide accumulate, deep score, fuse, top-K                 */
/* ------------------------------------------------------------------------------------------ */
/*
 * Device workspace size for ebr_score_topk / ebr_score_topk_keys with this batch, slot count
 * and k.  Returns 0 for invalid arguments.
 */
size_t ebr_workspace_bytes(const ebr_index *idx, int32_t batch, int32_t slots, int32_t k);

/*
 * async.  For each user b in [0, batch):
 *   A1 plan: for every slot (f,s) with v = user_feat[b][f][s] >= 0: key i = base_f + v,
 *      w~ = fl32(w_i * user_x[b][f][s])  (one rounding, never fused into an FMA, R10);
 *   A2/A3 decode each such key's posting chunks and add w~ to the wide score of every listed ad
 *      (Alg. 2 l.355-358);
 *   A4 deep score <user_emb[b], A[a]> with fp32 accumulation (Eq. 1);
 *   A5 s = deep + wide (Eq. 9), -0 canonicalised to +0, key kappa = (ord(s) << 32) | ~id;
 *   A6 the k largest kappa, i.e. score descending, ties by ascending global ad id.
 *
 *  user_emb   device, [batch][d] in the index dtype (fp32 or bf16 bits).
 *  user_feat  device, [batch][n_fields][slots] int32, -1 = empty slot.  A value outside
 *             [-1, V_f) is skipped and raises the device error flag (see ebr_query_error).
 *  user_x     device, [batch][n_fields][slots] fp32, the user's statistic x_i for that slot.
 *  slots      1 <= slots <= 64.
 *  k          1 <= k <= EBR_MAX_K.  k may exceed the shard size: missing entries are returned
 *             as (id -1, score -inf) (reading R15).
 *  out_ids    device, [batch][k] int32 global ad ids (ad_begin + local), best first.
 *  out_scores device, [batch][k] fp32 s(u,a) of those ads.
 *  workspace  device, >= ebr_workspace_bytes(idx, batch, slots, k) bytes, 256-byte aligned,
 *             caller-owned; one in-flight call per workspace.  Initialise a new buffer once with
 *             ebr_workspace_init(); every call then leaves it ready for the next, so each query
 *             is a single kernel launch.  Do not modify it between calls.
 * Errors: EBR_EINVAL for batch < 1, slots out of range, k out of range, undersized workspace;
 *         EBR_ECUDA on a launch failure.  Duplicate (f,v) slots of one user add (reading R3).
 */
ebr_status ebr_score_topk(const ebr_index *idx, const void *user_emb, int32_t batch,
                          const int32_t *user_feat, const float *user_x, int32_t slots, int32_t k,
                          int32_t *out_ids, float *out_scores, void *workspace,
                          size_t workspace_bytes, void *stream);

/*
 * async.  Same as ebr_score_topk but emits the packed keys
 *   kappa = (ord(score) << 32) | (0xFFFFFFFF - global_id),  [batch][k] uint64, descending,
 * padding entries = 0 -- the all-gather payload of the multi-GPU path (A7).
 */
ebr_status ebr_score_topk_keys(const ebr_index *idx, const void *user_emb, int32_t batch,
                               const int32_t *user_feat, const float *user_x, int32_t slots,
                               int32_t k, uint64_t *out_keys, void *workspace,
                               size_t workspace_bytes, void *stream);

/*
 * Reads (and clears) the device-side validation flag of `workspace` written by the last
 * ebr_score_topk* call on it (each call clears it when it starts).  Host-synchronous on `stream`.  *flags bit 0 = a user_feat value
 * was outside [-1, V_f).  Returns EBR_EDEVICE if any bit was set, EBR_OK otherwise.
 */
ebr_status ebr_query_error(void *workspace, void *stream, uint32_t *flags);

/*
 * async.  Prepares a freshly allocated workspace (zero fill + state word) for use with `idx`.
 * Required once per buffer before its first ebr_score_topk* / ebr_score_topk_host call (and
 * again if the buffer was written by anything else).  bytes = the buffer size.
 */
ebr_status ebr_workspace_init(const ebr_index *idx, void *workspace, size_t bytes, void *stream);

/*
 * End-to-end variant with HOST buffers (the e2e measurement): copies user_emb, user_feat and
 * user_x host->device, runs ebr_score_topk, copies ids and scores device->host and synchronises
 * `stream` before returning.  Requests whose inputs and outputs each fit 1 MB are staged through
 * a library-owned, thread-local pinned buffer (one H2D and one D2H copy: per-copy latency
 * dominates at these sizes); larger ones copy each array directly, so their host buffers should
 * be pinned for full speed.  Not reentrant within one thread across streams.
 * workspace: device, >= ebr_workspace_bytes_host(idx, batch, slots, k).
 */
size_t ebr_workspace_bytes_host(const ebr_index *idx, int32_t batch, int32_t slots, int32_t k);
ebr_status ebr_score_topk_host(const ebr_index *idx, const void *user_emb_host, int32_t batch,
                               const int32_t *user_feat_host, const float *user_x_host,
                               int32_t slots, int32_t k, int32_t *out_ids_host,
                               float *out_scores_host, void *workspace, size_t workspace_bytes,
                               void *stream);

/* ------------------------------------------------------------------------------------------ */
/* A7  Cross-GPU merge (not in the paper: the inventory is sharded over the GPUs of one box)    */
/* ------------------------------------------------------------------------------------------ */
/*
 * async.  gathered: device, [G][batch][k] uint64 kappa lists (each descending, padding 0) from
 * G shards.  Writes the global top k per user: out_ids [batch][k] int32, out_scores fp32.
 * Because kappa is unique per ad, the result equals the single-GPU answer exactly.
 * workspace: device, >= ebr_merge_workspace_bytes(G, batch, k).
 */
size_t ebr_merge_workspace_bytes(int32_t G, int32_t batch, int32_t k);
ebr_status ebr_merge_topk(const uint64_t *gathered, int32_t G, int32_t batch, int32_t k,
                          int32_t *out_ids, float *out_scores, void *workspace,
                          size_t workspace_bytes, void *stream);

/*
 * Threshold exchange for large batch x k (reading R24), three async
 * calls around two small collectives that replace the all-gather of G*batch*k keys:
 *   1. ebr_exchange_kth: out_kq[b] = local_keys[b][ceil(k/G) - 1] (device, [batch] uint64) -- this
 *      rank's ceil(k/G)-th key; all-gather it into kq_gathered [G][batch].
 *   2. ebr_exchange_pack: theta_b = min_r kq_gathered[r][b] is a lower bound of user b's global
 *      k-th key (every rank holds >= ceil(k/G) keys >= theta_b), and every global top-k key is
 *      >= theta_b and in its rank's local top k.  Writes out_count[b] = #{local keys >= theta_b}
 *      (device, [batch] uint32), out_off[0..batch] = their exclusive scan (out_off[batch] = total)
 *      and the packed keys out_packed[out_off[b] + j] = local_keys[b][j] (device, >= batch*k).
 *      All-gather the counts ([G][batch]) and the packed lists, each padded to the largest total.
 *   3. ebr_merge_topk_packed: packed [G][stride] (rank r's list at r*stride), counts [G][batch]:
 *      the global top k per user, exactly the single-GPU answer (kappa is unique).
 * local_keys: device, [batch][k] descending kappa, padding 0 (ebr_score_topk_keys).  G in 1..16.
 */
ebr_status ebr_exchange_kth(const uint64_t *local_keys, int32_t batch, int32_t k, int32_t G,
                            uint64_t *out_kq, void *stream);
ebr_status ebr_exchange_pack(const uint64_t *local_keys, int32_t batch, int32_t k,
                             const uint64_t *kq_gathered, int32_t G, uint32_t *out_count,
                             uint32_t *out_off, uint64_t *out_packed, void *stream);
ebr_status ebr_merge_topk_packed(const uint64_t *packed, int64_t stride, const uint32_t *counts,
                                 int32_t G, int32_t batch, int32_t k, int32_t *out_ids,
                                 float *out_scores, void *stream);

/* ------------------------------------------------------------------------------------------ */
/* Parity / introspection                                                                       */
/* ------------------------------------------------------------------------------------------ */
/*
 * Host-synchronous.  Decodes key `key`'s posting list ON THE DEVICE with the same warp decoder
 * the query path uses and copies the shard-local ad ids (ascending) to out_ads (host, cap
 * entries).  *n receives the list length (also when it exceeds cap, then EBR_EINVAL).
 */
ebr_status ebr_debug_decode(const ebr_index *idx, int64_t key, int32_t *out_ads, int64_t cap,
                            int64_t *n);

typedef struct {
    int64_t n_ads;        /* shard size                                        */
    int64_t ad_begin;     /* first global id of the shard                      */
    int32_t d, d_pad;     /* embedding width and padded kernel width           */
    int32_t dtype;        /* ebr_dtype                                         */
    int32_t n_fields;
    int64_t n_keys;       /* M                                                 */
    int64_t nnz;          /* postings (entries of L in the shard)              */
    int64_t chunks;       /* 32-posting chunks                                 */
    int64_t payload_words;
    int64_t index_bytes;  /* directory + headers + payload + w                 */
    int64_t emb_bytes;    /* device bytes of A                                 */
    double build_ms;      /* host encode + upload wall time                    */
    int32_t n_hot;        /* dense hot-key columns of L (bf16 indexes; 0 = none) */
    int32_t pad0;
    int64_t hot_nnz;      /* postings covered by the hot columns               */
    int64_t hot_bytes;    /* device bytes of the hot-key bit masks             */
    double encode_ms;     /* the inverted-list part of build_ms: host encode, or (device build)
                             ad_feat upload + GPU sort/encode + hot masks; excludes A's upload */
} ebr_stats;
ebr_status ebr_index_stats(const ebr_index *idx, ebr_stats *out);

/*
 * Host-synchronous copy of one device array of the index to out_host (cap_bytes); *bytes
 * receives its size (out_host = NULL: size only).  which: 0 key_chunk_off [M+1] u32, 1
 * key_word_off [M] u32, 2 chunk_hdr [C] u32x2, 3 chunk_last [C] u32, 4 payload [W+2] u32,
 * 5 hot_mask [n_pad] u32x4 (0 bytes without hot columns).  Parity support (host vs device build).
 */
ebr_status ebr_index_export(const ebr_index *idx, int32_t which, void *out_host, int64_t cap_bytes,
                            int64_t *bytes);

/*
 * Host-only encoder (no device needed; used to pin the wire format on CPU).  Encodes the
 * posting lists of ad_feat (shard-local ids 0..n_ads-1) exactly as ebr_build_index does.
 * Output capacities: key_chunk_off [n_keys+1], key_word_off [n_keys], chunk_hdr [2*hdr_cap],
 * payload [payload_cap].  *n_chunks / *n_words receive the sizes; EBR_EINVAL if a capacity is
 * too small (sizes still written) or the inputs are invalid.
 */
ebr_status ebr_encode_host(const int32_t *ad_feat, int64_t n_ads, int32_t n_fields,
                           const int32_t *field_card, int64_t n_keys, uint32_t *key_chunk_off,
                           uint32_t *key_word_off, uint32_t *chunk_hdr, int64_t hdr_cap,
                           uint32_t *payload, int64_t payload_cap, int64_t *n_chunks,
                           int64_t *n_words);

/* ------------------------------------------------------------------------------------------ */
/* NEXT-3 ablation: the paper's own inverted list (Alg. 1-2) on the same B200          */
/* ------------------------------------------------------------------------------------------ */
/*
 * Not a path of ebr_score_topk: an ablation that builds the paper's index -- blocks of the ads
 * sharing the high 24 bits of their id, grouped by ceil(log2 n) and padded to 2^g one-byte
 * residuals, per-group SoA with per-key offsets (Alg. 1; readings R5-R7 of DESIGN.md:
 * the valid count rides in the header word, keys are a CSR) -- and runs Alg. 2 for one
 * user: scores[a] = sum over the query items (key, w) of w * L[a, key], by fp32 AtomicAdd into a
 * global score array (zeroed first, Alg. 2 l.350).  ebr_chunk_hitmatch runs the same algorithm on
 * this library's chunk codec, for an equal-terms comparison of the two layouts.
 *
 *  ad_feat etc.   host, as ebr_build_index (shard-local ids 0..n_ads-1); host-synchronous build.
 *  keys, w        device, [n_items] int32 keys (out-of-range keys ignored) and fp32 weights w~.
 *  scores         device, [n_ads] fp32, overwritten.  n_items <= 1024.  Async on `stream`.
 * Errors: EBR_EINVAL (bad arguments / values), EBR_ECUDA.
 */
typedef struct ebr_paper_index ebr_paper_index;
ebr_status ebr_paper_index_build(const int32_t *ad_feat, int64_t n_ads, int32_t n_fields,
                                 const int32_t *field_card, int64_t n_keys, int device,
                                 void *stream, ebr_paper_index **out);
void ebr_paper_index_free(ebr_paper_index *pidx);
/* blocks per group (host, [9]), device bytes and host build time of the paper index */
ebr_status ebr_paper_index_info(const ebr_paper_index *pidx, int64_t *blocks9, int64_t *bytes,
                                double *build_ms);
ebr_status ebr_paper_hitmatch(const ebr_paper_index *pidx, const int32_t *keys, const float *w,
                              int32_t n_items, float *scores, void *stream);
ebr_status ebr_chunk_hitmatch(const ebr_index *idx, const int32_t *keys, const float *w,
                              int32_t n_items, float *scores, void *stream);

/*
 * NEXT-4, in-query IPNN (Eq. 7-8): async.  For rows b in [0, rows):
 *   out[b] = [h[b], W u[b]]  (length d0 + d1), the W u part accumulated in fp32 (fma over i in
 *   order) and rounded once to `dtype` (bf16: round-to-nearest-even).
 * h: device [rows][d0] in `dtype` (the dual tower's output h_u or h_a); u: device [rows][n] fp32
 * (the pooled user / ad features); W: device [d1][n] fp32 row-major (W^(u) or W^(v)); out: device
 * [rows][d0 + d1] in `dtype` -- the h~ that ebr_build_index (ads) and ebr_score_topk (users) take.
 * Errors: EBR_EINVAL (null pointers, negative sizes, n > 12288, bad dtype), EBR_ECUDA.
 */
ebr_status ebr_ipnn_extend(const void *h, const float *u, const float *W, int64_t rows, int32_t d0,
                           int32_t n, int32_t d1, ebr_dtype dtype, void *out, void *stream);

/* Number of CUDA kernels (and memsets) one ebr_score_topk* call with these arguments enqueues on
 * its stream (the latency path: one cooperative launch per 4 users; the batched tensor-core path:
 * 1 memset plus 7 launches per group of 128 users).  Excludes the rare overflow fallback. */
int32_t ebr_query_launches(const ebr_index *idx, int32_t batch, int32_t slots, int32_t k);

/*
 * Dominant-kernel timer (measurement support for bench.py's roofline; off by default).  While
 * enabled, every query records a CUDA event pair on its stream around its dominant kernel: the
 * batched path's full filter pass of the fused tensor-core kernel (score_kernel<1>), the latency
 * path's fused cooperative kernel.  Calls on a stream that is being captured into a CUDA graph
 * record nothing.  ebr_kernel_timer_read() synchronises on the recorded events, returns their
 * summed elapsed milliseconds and the number of timed launches, copies the kernel's name into
 * `name` (host, name_cap bytes, may be NULL) and clears the record.  Host-synchronous.
 */
ebr_status ebr_kernel_timer(int32_t enable);
ebr_status ebr_kernel_timer_read(double *total_ms, int64_t *launches, char *name, int32_t name_cap);

/* Thread-local message describing the last failure of any ebr_* call on this thread. */
const char *ebr_last_error(void);

/* Library build identifier ("ebr <git-describe> sm_100a"). */
const char *ebr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EBR_H_ */
