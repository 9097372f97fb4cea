/*
 * ebr_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU oracle for the
 * Wide & Deep retrieval hot path of arXiv 2511.22460.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA library (paper_2511_22460_b200/csrc) and neither side
 * includes or links the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n.
 *
 *  - oracle_scores_user  (scorer A, the plain definition of the scored quantity, Eq. 9,
 *    P:253-257):   s(u,a) = <h~_u, h~_a> + sum_i w_i x_i L_{a,i}
 *      * deep term: Eq. 1 / Eq. 8, accumulated in fp64 over the exact input values
 *        (bf16 inputs are widened exactly).
 *      * wide term through an uncompressed per-user cross-weight table T_u[M] (fp64):
 *        T_u[i] = sum over the user's slots carrying key i of w_i * x_i  (w~_i = w_i x_i),
 *        and wide(u,a) = sum_f T_u[key(a,f)], i.e. sum_i T_u[i] L_{a,i} (L_{a,i}=1 iff ad a has
 *        value v in field f with i = base_f + v; "keys are the feature indices,
 *        values are the ad indices"; reading R1 in DESIGN.md).
 *      * also returns sigma(a) = sum_j |h_u[j] h_a[j]| + sum_hits |w~|, the summation-error scale
 *        the tolerances are stated against (reading R12).
 *  - oracle_wide_pairs_user (scorer B): the wide term by explicit feature-pair enumeration --
 *        sum over fields f and user slots s of [user value == ad value] * w_{key} * x_{u,f,s}
 *        ("the ad component in the side information feature looks up the matched feature values
 *        from the user sequences. It then performs a weighted sum").
 *  - oracle_topk: scorer A for every ad, then a brute-force full sort by (score desc, ad id asc)
 *        and the first K ("retrieve top k relevant ads"; tie-break reading R13), padded
 *        with (id -1, -inf) when K > N (reading R15).
 *  - oracle_postings: the inverted list of L straight from the raw ad feature values: one
 *        ascending list of ad ids per key ("each list represents a column in L").
 *  - oracle_decode_chunks: an independent decoder of the library's documented wire format
 *        (DESIGN.md "Posting-chunk wire format"), written from that text bit by bit, used only to
 *        pin the host encoder before any kernel exists.
 *
 * Build: gcc -O2 -fno-fast-math -shared -fPIC -pthread (no -ffast-math: fp64 as written).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- input helpers */

static double emb_at(const void *emb, int is_bf16, int64_t row, int d, int j) {
    if (is_bf16) {
        uint16_t b = ((const uint16_t *)emb)[row * (int64_t)d + j];
        uint32_t u = ((uint32_t)b) << 16; /* bf16 is the top half of an fp32: exact widening */
        float f;
        memcpy(&f, &u, sizeof f);
        return (double)f;
    }
    return (double)((const float *)emb)[row * (int64_t)d + j];
}

static int64_t key_base(const int32_t *field_card, int f) {
    int64_t b = 0;
    for (int g = 0; g < f; ++g) b += field_card[g];
    return b;
}

/* ---------------------------------------------------------------- scorer A */

typedef struct {
    int64_t n_ads;
    int d, emb_is_bf16, n_fields, slots;
    const void *ad_emb;
    const int32_t *ad_feat, *field_card;
    const float *cross_w;
    int64_t n_keys;
} inventory_t;

/* Fills T[M] (zeroed by the caller) from one user's slots; returns 0, or -1 on a bad value. */
static int fill_table(const inventory_t *iv, const int32_t *ufeat, const float *ux, double *T) {
    for (int f = 0; f < iv->n_fields; ++f) {
        int64_t base = key_base(iv->field_card, f);
        for (int s = 0; s < iv->slots; ++s) {
            int32_t v = ufeat[f * iv->slots + s];
            if (v < 0) continue;                     /* empty slot: x_i absent from the query */
            if (v >= iv->field_card[f]) return -1;
            int64_t i = base + v;
            T[i] += (double)iv->cross_w[i] * (double)ux[f * iv->slots + s]; /* w~_i = w_i x_i */
        }
    }
    return 0;
}

static void score_all(const inventory_t *iv, const void *uemb, const double *T, int64_t *bases,
                      double *r, double *sigma) {
    for (int64_t a = 0; a < iv->n_ads; ++a) {
        double deep = 0.0, sg = 0.0;
        for (int j = 0; j < iv->d; ++j) {
            double p = emb_at(uemb, iv->emb_is_bf16, 0, iv->d, j) *
                       emb_at(iv->ad_emb, iv->emb_is_bf16, a, iv->d, j);
            deep += p;
            sg += fabs(p);
        }
        double wide = 0.0;
        for (int f = 0; f < iv->n_fields; ++f) {
            int32_t v = iv->ad_feat[a * iv->n_fields + f];
            if (v < 0) continue;                     /* L_{a,i} = 0 for an empty ad field */
            double t = T[bases[f] + v];
            wide += t;
            sg += fabs(t);
        }
        r[a] = deep + wide;
        if (sigma) sigma[a] = sg;
    }
}

static int check_inventory(const inventory_t *iv) {
    int64_t m = 0;
    for (int f = 0; f < iv->n_fields; ++f) {
        if (iv->field_card[f] < 1) return -1;
        m += iv->field_card[f];
    }
    if (m != iv->n_keys) return -1;
    for (int64_t a = 0; a < iv->n_ads; ++a)
        for (int f = 0; f < iv->n_fields; ++f) {
            int32_t v = iv->ad_feat[a * iv->n_fields + f];
            if (v < -1 || v >= iv->field_card[f]) return -1;
        }
    return 0;
}

int oracle_scores_user(int64_t n_ads, int d, int emb_is_bf16, const void *ad_emb, int n_fields,
                       const int32_t *ad_feat, const int32_t *field_card, const float *cross_w,
                       int64_t n_keys, const void *user_emb, int slots, const int32_t *user_feat,
                       const float *user_x, double *r_out, double *sigma_out) {
    inventory_t iv = {n_ads, d, emb_is_bf16, n_fields, slots, ad_emb, ad_feat, field_card,
                      cross_w, n_keys};
    if (check_inventory(&iv)) return -1;
    double *T = calloc((size_t)(n_keys > 0 ? n_keys : 1), sizeof(double));
    int64_t *bases = malloc(sizeof(int64_t) * (size_t)(n_fields > 0 ? n_fields : 1));
    if (!T || !bases) { free(T); free(bases); return -2; }
    for (int f = 0; f < n_fields; ++f) bases[f] = key_base(field_card, f);
    int rc = fill_table(&iv, user_feat, user_x, T);
    if (rc == 0) score_all(&iv, user_emb, T, bases, r_out, sigma_out);
    free(T);
    free(bases);
    return rc;
}

/* ---------------------------------------------------------------- scorer B */

int oracle_wide_pairs_user(int64_t n_ads, int n_fields, const int32_t *ad_feat,
                           const int32_t *field_card, const float *cross_w, int slots,
                           const int32_t *user_feat, const float *user_x, double *wide_out) {
    for (int64_t a = 0; a < n_ads; ++a) {
        double wide = 0.0;
        for (int f = 0; f < n_fields; ++f) {
            int32_t av = ad_feat[a * n_fields + f];
            for (int s = 0; s < slots; ++s) {
                int32_t uv = user_feat[f * slots + s];
                if (uv < 0 || av < 0) continue;
                if (uv == av) {
                    int64_t i = key_base(field_card, f) + uv;
                    wide += (double)cross_w[i] * (double)user_x[f * slots + s];
                }
            }
        }
        wide_out[a] = wide;
    }
    return 0;
}

/* ---------------------------------------------------------------- top-K by brute-force sort */

typedef struct { double r; int64_t id; double sigma; } item_t;

static int cmp_item(const void *pa, const void *pb) {
    const item_t *a = pa, *b = pb;
    if (a->r > b->r) return -1;                      /* score descending */
    if (a->r < b->r) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id);   /* ties: ad id ascending */
}

typedef struct {
    const inventory_t *iv;
    const void *user_emb;
    const int32_t *user_feat;
    const float *user_x;
    int k;
    int64_t id_base;
    int32_t *out_ids;
    double *out_r, *out_sigma;
    int b_begin, b_end, rc;
} job_t;

static void *topk_job(void *arg) {
    job_t *jb = arg;
    const inventory_t *iv = jb->iv;
    int64_t N = iv->n_ads;
    size_t esz = iv->emb_is_bf16 ? 2 : 4;
    double *T = calloc((size_t)(iv->n_keys > 0 ? iv->n_keys : 1), sizeof(double));
    double *r = malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    double *sg = malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    item_t *it = malloc(sizeof(item_t) * (size_t)(N > 0 ? N : 1));
    int64_t *bases = malloc(sizeof(int64_t) * (size_t)(iv->n_fields > 0 ? iv->n_fields : 1));
    if (!T || !r || !sg || !it || !bases) { jb->rc = -2; goto out; }
    for (int f = 0; f < iv->n_fields; ++f) bases[f] = key_base(iv->field_card, f);
    for (int b = jb->b_begin; b < jb->b_end; ++b) {
        memset(T, 0, sizeof(double) * (size_t)(iv->n_keys > 0 ? iv->n_keys : 1));
        const int32_t *uf = jb->user_feat + (int64_t)b * iv->n_fields * iv->slots;
        const float *ux = jb->user_x + (int64_t)b * iv->n_fields * iv->slots;
        if (fill_table(iv, uf, ux, T)) { jb->rc = -1; goto out; }
        const void *ue = (const char *)jb->user_emb + (size_t)b * iv->d * esz;
        score_all(iv, ue, T, bases, r, sg);
        for (int64_t a = 0; a < N; ++a) {
            it[a].r = r[a];
            it[a].id = a + jb->id_base;
            it[a].sigma = sg[a];
        }
        qsort(it, (size_t)N, sizeof(item_t), cmp_item);
        for (int q = 0; q < jb->k; ++q) {
            int64_t o = (int64_t)b * jb->k + q;
            if (q < N) {
                jb->out_ids[o] = (int32_t)it[q].id;
                jb->out_r[o] = it[q].r;
                if (jb->out_sigma) jb->out_sigma[o] = it[q].sigma;
            } else {                                  /* K > N: pad (reading R15) */
                jb->out_ids[o] = -1;
                jb->out_r[o] = -INFINITY;
                if (jb->out_sigma) jb->out_sigma[o] = 0.0;
            }
        }
    }
out:
    free(T); free(r); free(sg); free(it); free(bases);
    return NULL;
}

int oracle_topk(int64_t n_ads, int d, int emb_is_bf16, const void *ad_emb, int n_fields,
                const int32_t *ad_feat, const int32_t *field_card, const float *cross_w,
                int64_t n_keys, int batch, const void *user_emb, int slots,
                const int32_t *user_feat, const float *user_x, int k, int64_t id_base,
                int threads, int32_t *out_ids, double *out_r, double *out_sigma) {
    inventory_t iv = {n_ads, d, emb_is_bf16, n_fields, slots, ad_emb, ad_feat, field_card,
                      cross_w, n_keys};
    if (k < 1 || batch < 0 || check_inventory(&iv)) return -1;
    if (threads < 1) threads = 1;
    if (threads > batch) threads = batch > 0 ? batch : 1;
    job_t *jobs = calloc((size_t)threads, sizeof(job_t));
    pthread_t *th = calloc((size_t)threads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return -2; }
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (job_t){&iv, user_emb, user_feat, user_x, k, id_base, out_ids, out_r, out_sigma,
                          (int)((int64_t)batch * t / threads),
                          (int)((int64_t)batch * (t + 1) / threads), 0};
    }
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, topk_job, &jobs[t]);
    topk_job(&jobs[0]);
    int rc = jobs[0].rc;
    for (int t = 1; t < threads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    free(jobs);
    free(th);
    return rc;
}

/* ---------------------------------------------------------------- posting lists */

/* offsets[M+1] (int64) and ads[nnz] (int32): list[i] = ascending ads a with ad_feat[a][f] == v,
   i = base_f + v.  Call with ads == NULL to get offsets only (nnz = offsets[M]). */
int oracle_postings(int64_t n_ads, int n_fields, const int32_t *ad_feat, const int32_t *field_card,
                    int64_t n_keys, int64_t *offsets, int32_t *ads) {
    memset(offsets, 0, sizeof(int64_t) * (size_t)(n_keys + 1));
    for (int64_t a = 0; a < n_ads; ++a)
        for (int f = 0; f < n_fields; ++f) {
            int32_t v = ad_feat[a * n_fields + f];
            if (v < 0) continue;
            if (v >= field_card[f]) return -1;
            offsets[key_base(field_card, f) + v + 1] += 1;
        }
    for (int64_t i = 0; i < n_keys; ++i) offsets[i + 1] += offsets[i];
    if (!ads) return 0;
    int64_t *fill = malloc(sizeof(int64_t) * (size_t)(n_keys > 0 ? n_keys : 1));
    if (!fill) return -2;
    memcpy(fill, offsets, sizeof(int64_t) * (size_t)n_keys);
    for (int64_t a = 0; a < n_ads; ++a)          /* ascending a => each list is ascending */
        for (int f = 0; f < n_fields; ++f) {
            int32_t v = ad_feat[a * n_fields + f];
            if (v < 0) continue;
            int64_t i = key_base(field_card, f) + v;
            ads[fill[i]++] = (int32_t)a;
        }
    free(fill);
    return 0;
}

/* ---------------------------------------------------------------- wire-format decoder */

/* Decodes every key's chunks:
 *   key_chunk_off[M+1] u32 : key i owns chunks [key_chunk_off[i], key_chunk_off[i+1])
 *   key_word_off[M]    u32 : payload word base of key i
 *   chunk_hdr[2*C]     u32 : per chunk {first, meta}; meta bits 0..4 = n-1, bits 5..9 = b,
 *                            bits 10..31 = payload word offset relative to key_word_off[i]
 *   payload[W]         u32 : values gap_j - 1 (j = 1..n-1), b bits each, LSB-first
 * Writes offsets[M+1] (int64) and ads[] like oracle_postings.  Returns 0, or -1 on a structural
 * error (ids not strictly increasing, reads past the payload). */
int oracle_decode_chunks(int64_t n_keys, const uint32_t *key_chunk_off,
                         const uint32_t *key_word_off, const uint32_t *chunk_hdr,
                         const uint32_t *payload, int64_t n_words, int64_t *offsets,
                         int32_t *ads, int64_t cap) {
    int64_t n = 0;
    offsets[0] = 0;
    for (int64_t i = 0; i < n_keys; ++i) {
        for (uint32_t c = key_chunk_off[i]; c < key_chunk_off[i + 1]; ++c) {
            uint32_t first = chunk_hdr[2 * (int64_t)c];
            uint32_t meta = chunk_hdr[2 * (int64_t)c + 1];
            uint32_t cnt = (meta & 31u) + 1u;
            uint32_t b = (meta >> 5) & 31u;
            int64_t word0 = (int64_t)key_word_off[i] + (int64_t)(meta >> 10);
            int64_t id = first;
            if (n >= cap) return -1;
            ads[n++] = (int32_t)id;
            for (uint32_t j = 1; j < cnt; ++j) {
                uint64_t val = 0;
                for (uint32_t t = 0; t < b; ++t) {     /* one bit at a time, LSB-first */
                    int64_t bit = (int64_t)(j - 1) * b + t;
                    int64_t w = word0 + bit / 32;
                    if (w >= n_words) return -1;
                    val |= (uint64_t)((payload[w] >> (bit % 32)) & 1u) << t;
                }
                int64_t nid = id + (int64_t)val + 1;  /* gap = value + 1 */
                if (nid <= id) return -1;
                if (n >= cap) return -1;
                ads[n++] = (int32_t)nid;
                id = nid;
            }
        }
        offsets[i + 1] = n;
    }
    return 0;
}

/*
 * oracle_ipnn_extend (NEXT-4, Eq. 7-8): the IPNN extension of a tower output,
 *   h~ = [h, W u],  W in R^{d1 x n} row-major, u in R^n,
 * written out in fp64 (W u accumulated over i in order); out is fp64 [rows][d0 + d1].  h is read as
 * fp32 or bf16 bits (widened exactly).
 */
int oracle_ipnn_extend(int64_t rows, int d0, int n, int d1, int h_is_bf16, const void *h, const float *u,
                       const float *W, double *out) {
    if (rows < 0 || d0 < 0 || n < 0 || d1 < 0) return 1;
    for (int64_t b = 0; b < rows; ++b) {
        double *o = out + b * (int64_t)(d0 + d1);
        for (int j = 0; j < d0; ++j) o[j] = emb_at(h, h_is_bf16, b, d0, j);
        for (int j = 0; j < d1; ++j) {
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += (double)W[(int64_t)j * n + i] * (double)u[b * (int64_t)n + i];
            o[d0 + j] = s;
        }
    }
    return 0;
}

/*
 * oracle_scores_user_pairs (NEXT-4, multi-valued ad fields -- tags): scorer A with L given
 * as its nonzeros, ad by ad: ad a holds the keys ad_keys[ad_key_off[a] .. ad_key_off[a+1]); L is
 * binary (L_{a,i} in {0,1}), so a key listed twice for one ad counts once.  Otherwise the
 * same definition as oracle_scores_user: r(a) = <h_u, h_a> + sum_{i: L_{a,i}=1} T_u[i], with
 * T_u[i] = sum over the user's slots carrying key i of w_i x_i (Eq. 9).
 */
int oracle_scores_user_pairs(int64_t n_ads, int d, int emb_is_bf16, const void *ad_emb,
                             const int64_t *ad_key_off, const int32_t *ad_keys, int n_fields,
                             const int32_t *field_card, const float *cross_w, int64_t n_keys,
                             const void *user_emb, int slots, const int32_t *user_feat,
                             const float *user_x, double *r, double *sigma) {
    inventory_t iv = {n_ads, d, emb_is_bf16, n_fields, slots, ad_emb, NULL, field_card, cross_w, n_keys};
    int64_t m = 0;
    for (int f = 0; f < n_fields; ++f) m += field_card[f];
    if (m != n_keys) return 1;
    double *T = (double *)calloc((size_t)(n_keys > 0 ? n_keys : 1), sizeof(double));
    if (!T) return 3;
    if (fill_table(&iv, user_feat, user_x, T)) { free(T); return 2; }
    for (int64_t a = 0; a < n_ads; ++a) {
        double deep = 0.0, sg = 0.0;
        for (int j = 0; j < d; ++j) {
            double p = emb_at(user_emb, emb_is_bf16, 0, d, j) * emb_at(ad_emb, emb_is_bf16, a, d, j);
            deep += p;
            sg += fabs(p);
        }
        double wide = 0.0;
        for (int64_t q = ad_key_off[a]; q < ad_key_off[a + 1]; ++q) {
            int32_t k = ad_keys[q];
            if (k < 0 || k >= n_keys) { free(T); return 1; }
            int seen = 0;                            /* L is binary: each key of the ad once */
            for (int64_t q2 = ad_key_off[a]; q2 < q; ++q2) seen |= ad_keys[q2] == k;
            if (seen) continue;
            wide += T[k];
            sg += fabs(T[k]);
        }
        r[a] = deep + wide;
        if (sigma) sigma[a] = sg;
    }
    free(T);
    return 0;
}
