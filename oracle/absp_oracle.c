/* TEST INFRASTRUCTURE ONLY — see absp_oracle.h. Plain-C restatement of the
 * reference path; compiled with -ffp-contract=off so every fp32 multiply and add
 * rounds separately, exactly as the reference build does. */
#include "absp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

static float bf16_to_f32(uint16_t x) {
    uint32_t u = (uint32_t)x << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

/* PagedKVCache::key_row, kv_cache.cpp:94-100: token -> page_table[token / P], row token % P. */
static const uint16_t* pool_row(const uint16_t* pool, size_t pool_pages, const uint32_t* page_table,
                                size_t h, size_t token, size_t d, size_t P) {
    const size_t page = page_table[token / P];
    return pool + (((h * pool_pages + page) * P) + token % P) * d;
}

void absp_oracle_offsets(size_t n, const uint32_t* block_sizes, size_t H, uint64_t* offsets) {
    offsets[0] = 0;
    for (size_t h = 0; h < H; ++h) offsets[h + 1] = offsets[h] + ceil_div(n, block_sizes[h]);
}

int absp_oracle_centroids(const uint16_t* k_pool, size_t pool_pages, const uint32_t* page_table,
                          size_t n, size_t H, size_t d, size_t P, const uint32_t* block_sizes,
                          int method, float* values, float* values_min) {
    if (n == 0) return 1; /* centroids.cpp:89-91 */
    uint64_t* offsets = malloc((H + 1) * sizeof *offsets);
    absp_oracle_offsets(n, block_sizes, H, offsets);
    long hh;
#pragma omp parallel for schedule(dynamic)
    for (hh = 0; hh < (long)H; ++hh) {
        const size_t h = (size_t)hh;
        const size_t B = block_sizes[h];
        const size_t nb = offsets[h + 1] - offsets[h];
        double* acc = malloc(d * sizeof *acc);
        for (size_t b = 0; b < nb; ++b) {
            float* out = values + (offsets[h] + b) * d;
            const size_t begin = b * B;
            const size_t end = begin + B < n ? begin + B : n;
            if (method == 0) {
                /* centroids.cpp:25-31: fp64 sum over rows in order, then *(1/cnt), cast */
                for (size_t c = 0; c < d; ++c) acc[c] = 0.0;
                for (size_t t = begin; t < end; ++t) {
                    const uint16_t* row = pool_row(k_pool, pool_pages, page_table, h, t, d, P);
                    for (size_t c = 0; c < d; ++c) acc[c] += (double)bf16_to_f32(row[c]);
                }
                const double inv = 1.0 / (double)(end - begin);
                for (size_t c = 0; c < d; ++c) out[c] = (float)(acc[c] * inv);
            } else {
                /* centroids.cpp:33-41: std::max/std::min seeded with -inf/+inf */
                float* lo = values_min + (offsets[h] + b) * d;
                for (size_t c = 0; c < d; ++c) {
                    out[c] = -INFINITY;
                    lo[c] = INFINITY;
                }
                for (size_t t = begin; t < end; ++t) {
                    const uint16_t* row = pool_row(k_pool, pool_pages, page_table, h, t, d, P);
                    for (size_t c = 0; c < d; ++c) {
                        const float v = bf16_to_f32(row[c]);
                        out[c] = (out[c] < v) ? v : out[c]; /* std::max(a,b) = a<b ? b : a */
                        lo[c] = (v < lo[c]) ? v : lo[c];    /* std::min(a,b) = b<a ? b : a */
                    }
                }
            }
        }
        free(acc);
    }
    free(offsets);
    return 0;
}

/* quantizer.cpp:16-59 for one head's segment. */
static void quantize_segment(const float* src, size_t nc, size_t d, int bits, int mode,
                             float* scales, float* zps, uint8_t* codes) {
    const int levels_i = (1 << bits) - 1;
    const float levels = (float)levels_i;
    const int mid = (1 << (bits - 1)) - 1;
    const float floor_ = 1e-8f; /* kRangeFloor, quantizer.cpp:11 */
    for (size_t c = 0; c < d; ++c) {
        float scale, zp;
        if (mode == 1) {
            float lo = src[c], hi = src[c];
            for (size_t i = 1; i < nc; ++i) {
                const float v = src[i * d + c];
                lo = (v < lo) ? v : lo;
                hi = (hi < v) ? v : hi;
            }
            const float range = hi - lo;
            scale = ((range < floor_) ? floor_ : range) / levels;
            zp = lo;
        } else {
            float absmax = 0.0f;
            for (size_t i = 0; i < nc; ++i) {
                const float a = fabsf(src[i * d + c]);
                absmax = (absmax < a) ? a : absmax;
            }
            scale = ((absmax < floor_) ? floor_ : absmax) / (float)mid;
            zp = 0.0f;
        }
        scales[c] = scale;
        zps[c] = zp;
    }
    for (size_t i = 0; i < nc; ++i) {
        for (size_t c = 0; c < d; ++c) {
            const float v = src[i * d + c];
            int q;
            if (mode == 1) {
                q = (int)roundf((v - zps[c]) / scales[c]); /* std::round: half away from 0 */
                q = q < 0 ? 0 : (q > levels_i ? levels_i : q);
            } else {
                q = (int)roundf(v / scales[c]);
                q = (q < -mid ? -mid : (q > mid ? mid : q)) + mid;
            }
            codes[i * d + c] = (uint8_t)q;
        }
    }
}

int absp_oracle_quantize(const float* values, const uint64_t* offsets, size_t H, size_t d,
                         int bits, int mode, uint8_t* codes, float* scales, float* zps) {
    if (bits != 2 && bits != 4 && bits != 8) return 1; /* config.cpp:8-12 */
    if (offsets[H] == 0) return 1;                     /* quantizer.cpp:86-88 */
    long hh;
#pragma omp parallel for schedule(dynamic)
    for (hh = 0; hh < (long)H; ++hh) {
        const size_t h = (size_t)hh;
        const size_t nc = offsets[h + 1] - offsets[h];
        if (nc == 0) continue; /* quantizer.cpp:65 */
        quantize_segment(values + offsets[h] * d, nc, d, bits, mode, scales + h * d, zps + h * d,
                         codes + offsets[h] * d);
    }
    return 0;
}

/* engine.cpp:34-40 */
static float dequant(uint8_t code, float scale, float zp, int mode, int mid) {
    if (mode == 1) return zp + (float)code * scale;
    return (float)((int)code - mid) * scale;
}

void absp_oracle_scores_quant(const float* q, const uint8_t* codes, const uint8_t* codes_min,
                              const float* scales, const float* zps, const float* scales_min,
                              const float* zps_min, const uint64_t* offsets, size_t H, size_t d,
                              int bits, int mode, int method, float* scores) {
    const int mid = (1 << (bits - 1)) - 1;
    const long total = (long)offsets[H];
    long i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < total; ++i) {
        size_t h = 0; /* head_of_flat_index, engine.cpp:16-19 */
        while (offsets[h + 1] <= (uint64_t)i) ++h;
        const float* qh = q + h * d;
        const uint8_t* hi = codes + (size_t)i * d;
        const float* sc = scales + h * d;
        const float* zp = zps + h * d;
        float acc = 0.0f;
        if (method == 0) {
            for (size_t c = 0; c < d; ++c) acc += qh[c] * dequant(hi[c], sc[c], zp[c], mode, mid);
        } else {
            const uint8_t* lo = codes_min + (size_t)i * d;
            const float* scm = scales_min + h * d;
            const float* zpm = zps_min + h * d;
            for (size_t c = 0; c < d; ++c) {
                const float a = qh[c] * dequant(hi[c], sc[c], zp[c], mode, mid);
                const float b = qh[c] * dequant(lo[c], scm[c], zpm[c], mode, mid);
                acc += (a < b) ? b : a;
            }
        }
        scores[i] = acc;
    }
}

void absp_oracle_scores_f32(const float* q, const float* values, const float* values_min,
                            const uint64_t* offsets, size_t H, size_t d, int method,
                            float* scores) {
    const long total = (long)offsets[H];
    long i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < total; ++i) {
        size_t h = 0;
        while (offsets[h + 1] <= (uint64_t)i) ++h;
        const float* qh = q + h * d;
        const float* hi = values + (size_t)i * d;
        float acc = 0.0f;
        if (method == 0) {
            for (size_t c = 0; c < d; ++c) acc += qh[c] * hi[c];
        } else {
            const float* lo = values_min + (size_t)i * d;
            for (size_t c = 0; c < d; ++c) {
                const float a = qh[c] * hi[c], b = qh[c] * lo[c];
                acc += (a < b) ? b : a;
            }
        }
        scores[i] = acc;
    }
}

/* Comparator of select_head, engine.cpp:123-128: score desc, then index asc.
 * `!=` makes -0.0 and +0.0 a tie. */
typedef struct {
    float s;
    uint32_t i;
} Pair;

static int better_cmp(const void* pa, const void* pb) {
    const Pair* a = pa;
    const Pair* b = pb;
    if (a->s != b->s) return a->s > b->s ? -1 : 1;
    return a->i < b->i ? -1 : (a->i > b->i ? 1 : 0);
}

int absp_oracle_select(const float* scores, const uint64_t* offsets, const uint32_t* block_sizes,
                       size_t H, size_t n, size_t token_budget, uint32_t* blocks, size_t max_k,
                       uint32_t* counts, uint32_t* budgets) {
    if (token_budget == 0) return 1; /* engine.cpp:161-163 */
    uint64_t* check = malloc((H + 1) * sizeof *check);
    absp_oracle_offsets(n, block_sizes, H, check);
    const int ok = memcmp(check, offsets, (H + 1) * sizeof *check) == 0; /* engine.cpp:158 */
    free(check);
    if (!ok) return 1;
    for (size_t h = 0; h < H; ++h) {
        const size_t nb = offsets[h + 1] - offsets[h];
        const size_t k = ceil_div(token_budget, block_sizes[h]); /* engine.cpp:174 */
        if (budgets) budgets[h] = (uint32_t)k;
        Pair* p = malloc((nb ? nb : 1) * sizeof *p);
        for (size_t j = 0; j < nb; ++j) {
            p[j].s = scores[offsets[h] + j];
            p[j].i = (uint32_t)j;
        }
        /* engine.cpp:131-147: all sorted if nb <= k; else the top k, with the
         * trailing block displacing the weakest pick, re-sorted. A full sort
         * followed by the same adjustment is the reference's own naive twin
         * (TopKMode::kFullSort, engine.cpp:138-139). */
        qsort(p, nb, sizeof *p, better_cmp);
        size_t take = nb;
        if (nb > k) {
            take = k;
            int has_trailing = 0;
            for (size_t j = 0; j < k; ++j) has_trailing |= (p[j].i == nb - 1);
            if (!has_trailing) {
                p[k - 1].s = scores[offsets[h] + nb - 1];
                p[k - 1].i = (uint32_t)(nb - 1);
                qsort(p, k, sizeof *p, better_cmp);
            }
        }
        if (take > max_k) {
            free(p);
            return 1;
        }
        counts[h] = (uint32_t)take;
        for (size_t j = 0; j < take; ++j) blocks[h * max_k + j] = p[j].i;
        free(p);
    }
    return 0;
}

int absp_oracle_attend(const float* q, const uint16_t* k_pool, const uint16_t* v_pool,
                       size_t pool_pages, const uint32_t* page_table, size_t n, size_t H, size_t d,
                       size_t P, const uint32_t* block_sizes, const uint32_t* blocks, size_t max_k,
                       const uint32_t* counts, float* out) {
    if (n == 0) return 1;
    for (size_t h = 0; h < H; ++h)
        if (counts[h] == 0) return 1; /* engine.cpp:223-227 */
    const float inv_sqrt_d = 1.0f / sqrtf((float)d); /* engine.cpp:290 */
    long hh;
    int bad = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
    for (hh = 0; hh < (long)H; ++hh) {
        const size_t h = (size_t)hh;
        const size_t B = block_sizes[h];
        const size_t nb = ceil_div(n, B);
        /* RowRef list, engine.cpp:299-320, via block_to_pages (kv_cache.cpp:118-138) */
        size_t rows = 0;
        for (size_t j = 0; j < counts[h]; ++j) {
            const size_t b = blocks[h * max_k + j];
            if (b >= nb) bad = 1;
            else rows += (B < n - b * B) ? B : n - b * B;
        }
        if (bad) continue;
        const uint16_t** kr = malloc(rows * sizeof *kr);
        const uint16_t** vr = malloc(rows * sizeof *vr);
        size_t r = 0;
        for (size_t j = 0; j < counts[h]; ++j) {
            const size_t b = blocks[h * max_k + j];
            const size_t begin = b * B;
            const size_t valid = (B < n - begin) ? B : n - begin;
            for (size_t t = begin; t < begin + valid; ++t, ++r) {
                kr[r] = pool_row(k_pool, pool_pages, page_table, h, t, d, P);
                vr[r] = pool_row(v_pool, pool_pages, page_table, h, t, d, P);
            }
        }
        /* attend_rows, engine.cpp:189-210 */
        const float* qh = q + h * d;
        float* w = malloc(rows * sizeof *w);
        float max_logit = -INFINITY;
        for (r = 0; r < rows; ++r) {
            float acc = 0.0f; /* dot_f32, engine.cpp:180-184 */
            for (size_t c = 0; c < d; ++c) acc += qh[c] * bf16_to_f32(kr[r][c]);
            const float z = acc * inv_sqrt_d;
            w[r] = z;
            max_logit = (max_logit < z) ? z : max_logit;
        }
        float denom = 0.0f;
        for (r = 0; r < rows; ++r) {
            w[r] = expf(w[r] - max_logit);
            denom += w[r];
        }
        float* o = out + h * d;
        for (size_t c = 0; c < d; ++c) o[c] = 0.0f;
        for (r = 0; r < rows; ++r) {
            const float a = w[r] / denom;
            for (size_t c = 0; c < d; ++c) o[c] += a * bf16_to_f32(vr[r][c]);
        }
        free(w);
        free(kr);
        free(vr);
    }
    return bad ? 2 : 0;
}

int absp_oracle_full_attention(const float* q, const uint16_t* k_pool, const uint16_t* v_pool,
                               size_t pool_pages, const uint32_t* page_table, size_t n, size_t H,
                               size_t d, size_t P, float* out) {
    if (n == 0) return 1; /* engine.cpp:358-360 */
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    long hh;
#pragma omp parallel for schedule(dynamic)
    for (hh = 0; hh < (long)H; ++hh) {
        const size_t h = (size_t)hh;
        const float* qh = q + h * d;
        double* w = malloc(n * sizeof *w);
        double* acc = calloc(d, sizeof *acc);
        double max_logit = -INFINITY;
        for (size_t t = 0; t < n; ++t) {
            const uint16_t* k = pool_row(k_pool, pool_pages, page_table, h, t, d, P);
            double z = 0.0;
            for (size_t c = 0; c < d; ++c) z += (double)qh[c] * (double)bf16_to_f32(k[c]);
            z *= inv_sqrt_d;
            w[t] = z;
            max_logit = (max_logit < z) ? z : max_logit;
        }
        double denom = 0.0;
        for (size_t t = 0; t < n; ++t) {
            w[t] = exp(w[t] - max_logit);
            denom += w[t];
        }
        for (size_t t = 0; t < n; ++t) {
            w[t] /= denom;
            const uint16_t* v = pool_row(v_pool, pool_pages, page_table, h, t, d, P);
            for (size_t c = 0; c < d; ++c) acc[c] += w[t] * (double)bf16_to_f32(v[c]);
        }
        for (size_t c = 0; c < d; ++c) out[h * d + c] = (float)acc[c];
        free(w);
        free(acc);
    }
    return 0;
}
