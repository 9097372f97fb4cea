// ebr_small.cu -- host side of the latency path (see ebr_small_kernel.cuh for the kernel).
#include <mutex>
#include <vector>

#include "ebr_small_kernel.cuh"

namespace ebr {
namespace small {

// --------------------------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------------------------
// lanes per row x 16-byte vectors per lane: rows of 64..512 B (one warp pass) or 1-2 KB
template <typename T>
kern_t pick_kernel(int nb, int lpr, int vpl) {
    if (vpl == 1) {
        switch (lpr) {
            case 4: return pick_nb<T, 4, 1>(nb);
            case 8: return pick_nb<T, 8, 1>(nb);
            case 16: return pick_nb<T, 16, 1>(nb);
            case 32: return pick_nb<T, 32, 1>(nb);
        }
        return nullptr;
    }
    if (lpr != 32) return nullptr;
    if (vpl == 2) return pick_nb<T, 32, 2>(nb);
    if (vpl == 4) return pick_nb<T, 32, 4>(nb);
    return nullptr;
}

struct SmallLayout {
    size_t off_header, off_hist, off_count, off_scores, off_cand, off_timers, total;
};

SmallLayout small_layout(const ebr_index* idx, int B) {
    SmallLayout L;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t o = 0;
    L.off_header = o; o = al(o + 16 + 16 * 8);   // magic, error word, 16 phase stamps
    L.off_hist = o;   o = al(o + (size_t)B * kHistBins * 4);
    L.off_count = o;  o = al(o + (size_t)B * (idx->sm_count + 1) * 4);   // [B][n_ranges]
    L.off_scores = o; o = al(o + (size_t)B * idx->n_pad * 4);
    L.off_cand = o;   o = al(o + (size_t)B * idx->n_pad * 8);
    L.off_timers = o; o = al(o + (size_t)(idx->sm_count + 1) * 16 * 8);   // per-CTA phase stamps
    L.total = o;
    return L;
}

}  // namespace small

using namespace small;

uint32_t workspace_magic(const ebr_index* idx) {
    return kMagic ^ (uint32_t)((uint64_t)idx->n_pad * 2654435761ull);
}

size_t small_workspace_bytes(const ebr_index* idx, int32_t slots, int32_t k) {
    (void)slots; (void)k;
    return small_layout(idx, kSmallMaxB).total;
}

// Runs users [b0, b0 + B) (B <= kSmallMaxB) in one launch.
ebr_status run_small(const QueryArgs& q, int b0, int B) {
    const ebr_index* idx = q.idx;
    SmallLayout L = small_layout(idx, kSmallMaxB);   // fixed layout: any B shares one workspace
    char* ws = static_cast<char*>(q.workspace);
    const int esz = idx->dtype == EBR_BF16 ? 2 : 4;
    const int row_bytes = idx->d_pad * esz;
    int lpr, vpl;
    if (row_bytes <= 512) { lpr = row_bytes / 16; vpl = 1; }
    else { lpr = 32; vpl = row_bytes / 512; }
    int nb = 1;
    while (nb < B) nb <<= 1;      // 1, 2 or 4 (kSmallMaxB)
    kern_t k = idx->dtype == EBR_BF16 ? pick_kernel<__nv_bfloat16>(nb, lpr, vpl) : pick_kernel<float>(nb, lpr, vpl);
    if (!k) return set_error(EBR_EUNSUPPORTED, "embedding row of %d bytes is not supported", row_bytes);

    const int items_cap = B * idx->n_fields * q.slots;
    const int sms = idx->sm_count;
    int64_t R = (idx->n_ads + sms - 1) / sms;
    R = std::max<int64_t>(32, (R + 31) & ~(int64_t)31);
    const int n_ranges = (int)((idx->n_ads + R - 1) / R);
    // per item: the Item + span lo/hi + unit offset + fixed-point parts
    const size_t plan_bytes = (size_t)kHistCopies * B * kHistBins * 4 + (size_t)items_cap * (sizeof(Item) + 20) + 64;
    // phase E: candidate staging (>= 16k keys) and the rare single-CTA fallback select
    const size_t sel_min = std::max((size_t)(n_ranges + 2) * 4 + 128 * 1024,
                                    (size_t)(n_ranges + 2) * 4 + (size_t)pow2ceil_i(q.k) * 8 + kSelBins * 4 + 64);
    const size_t cap = 227 * 1024;
    if (plan_bytes + 8 * 1024 + (size_t)B * 32 * 12 > cap)
        return set_error(EBR_EUNSUPPORTED, "latency path: %d user slots need too much shared memory", items_cap);
    // tile: as many ads as fit (deep fp32 + two 32-bit accumulator words per user and ad)
    int64_t T = (int64_t)((cap - 8 * 1024 - plan_bytes) / ((size_t)B * 12));
    T = std::min<int64_t>(T, 16384) & ~(int64_t)31;
    const bool resident = T >= R;
    if (resident) T = R;
    const size_t p1 = plan_bytes + (size_t)B * T * 12;
    const size_t smem = std::max(p1, sel_min);
    if (smem > cap)
        return set_error(EBR_EUNSUPPORTED, "latency path: %d user slots / k=%d need %zu B of shared memory",
                         items_cap, q.k, smem);

    // the attribute and the occupancy of a (kernel, smem, device) are fixed: computed once (the
    // per-call host work is part of the end-to-end latency of a query)
    // (the max-dynamic-smem attribute is per kernel and shapes its occupancy, so it is re-set
    // whenever this call's size differs from the last one set for the kernel on this device)
    struct OccKey { kern_t k; size_t smem; int dev; int occ; };
    struct AttrKey { kern_t k; int dev; size_t smem; };
    static std::mutex occ_mu;
    static std::vector<OccKey> occ_cache;
    static std::vector<AttrKey> attr_set;
    int occ = 0;
    cudaError_t e = cudaSuccess;
    // held until the launch is enqueued: another thread re-setting the kernel's attribute between
    // this call's set and its launch would make the cooperative launch fail
    std::unique_lock<std::mutex> lk(occ_mu);
    {
        AttrKey* cur = nullptr;
        for (AttrKey& a : attr_set)
            if (a.k == k && a.dev == idx->device) cur = &a;
        if (!cur || cur->smem != smem) {
            e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(small)");
            if (cur) cur->smem = smem;
            else attr_set.push_back({k, idx->device, smem});
        }
        for (const OccKey& o : occ_cache)
            if (o.k == k && o.smem == smem && o.dev == idx->device) { occ = o.occ; break; }
        if (!occ) {
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem);
            if (e != cudaSuccess || occ < 1)
                return cuda_check(e == cudaSuccess ? cudaErrorInvalidConfiguration : e, "occupancy(small)");
            occ_cache.push_back({k, smem, idx->device, occ});
        }
    }

    SmallParams p;
    p.A = idx->A; p.d = idx->d; p.d_pad = idx->d_pad;
    p.row_bytes = row_bytes;
    p.n_ads = idx->n_ads; p.n_pad = idx->n_pad; p.ad_begin = (uint32_t)idx->ad_begin;
    p.key_chunk_off = idx->key_chunk_off; p.key_word_off = idx->key_word_off;
    p.hdr = idx->chunk_hdr; p.payload = idx->payload; p.cross_w = idx->cross_w;
    p.field_card = idx->field_card; p.field_base = idx->field_base; p.n_fields = idx->n_fields;
    p.U = static_cast<const char*>(q.user_emb) + (size_t)b0 * idx->d * esz;
    p.B = B; p.slots = q.slots; p.K = q.k;
    p.user_feat = q.user_feat + (size_t)b0 * idx->n_fields * q.slots;
    p.user_x = q.user_x + (size_t)b0 * idx->n_fields * q.slots;
    p.header = reinterpret_cast<uint32_t*>(ws + L.off_header);
    static const bool timers_on = getenv("EBR_PHASE_TIMERS") && getenv("EBR_PHASE_TIMERS")[0] == '1';
    static const int diag = getenv("EBR_DIAG") ? atoi(getenv("EBR_DIAG")) : 0;
    p.diag = diag;
    p.timers = timers_on ? reinterpret_cast<unsigned long long*>(ws + L.off_timers) : nullptr;
    // the magic ties the workspace's zeroed state to this index geometry
    p.magic = workspace_magic(idx);
    p.ghist = reinterpret_cast<uint32_t*>(ws + L.off_hist);
    p.cand_count = reinterpret_cast<uint32_t*>(ws + L.off_count);
    p.scores = reinterpret_cast<float*>(ws + L.off_scores);
    p.cand = reinterpret_cast<uint64_t*>(ws + L.off_cand);
    p.out_ids = q.out_ids ? q.out_ids + (size_t)b0 * q.k : nullptr;
    p.out_scores = q.out_scores ? q.out_scores + (size_t)b0 * q.k : nullptr;
    p.out_keys = q.out_keys ? q.out_keys + (size_t)b0 * q.k : nullptr;
    p.R = (int32_t)R;
    p.n_ranges = n_ranges;
    p.resident = resident ? 1 : 0;
    p.T = (int32_t)T;
    p.chunk_last = idx->chunk_last;
    p.items_cap = items_cap;
    p.smem_bytes = (int32_t)smem;

    if (timers_on) {
        e = cudaMemsetAsync(ws + L.off_timers, 0, (size_t)(sms + 1) * 16 * 8, q.stream);
        if (e != cudaSuccess) return cuda_check(e, "memset(timers)");
    }
    const int grid = std::max(1, std::min<int>(std::max(p.n_ranges, B), occ * sms));
    void* args[] = {&p};
    {
        KernelTimer kt(q.stream, "small_kernel (fused plan + decode + wide + GEMV + fuse + top-K)");
        e = cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(kThreads), args, smem, q.stream);
    }
    if (e != cudaSuccess) return cuda_check(e, "launch(small)");
    return EBR_OK;
}

}  // namespace ebr
