// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C shim over the *unmodified* reference C++ core (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests, the golden-fixture generator and bench.py's reference arm call
// the reference functions on flat arrays:
//
//   compute_block_centroids   centroids.hpp:56-57
//   quantize_store            quantizer.hpp:43
//   estimate_scores           engine.hpp:47-49
//   select_topk               engine.hpp:61-64
//   populate_page_spans       engine.hpp:71
//   sparse_attention          engine.hpp:79-80
//   full_attention_oracle     engine.hpp:86
//   DecodeEngine              engine.hpp:99-129
//   save_trace / load_trace   workload.hpp:70-71
//   profile_sensitivity, transfer_check, assign_block_sizes   calibrator.hpp:52-76
//
// One handle = one sequence (the reference has no batch dimension,
// kv_cache.hpp:26-67). Batch and GQA are layered on top in Python exactly as
// SURVEY.md Appendix A prescribes.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "absparse/calibrator.hpp"
#include "absparse/centroids.hpp"
#include "absparse/config.hpp"
#include "absparse/engine.hpp"
#include "absparse/kv_cache.hpp"
#include "absparse/quantizer.hpp"
#include "absparse/workload.hpp"

using namespace absparse;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 out_of_range, 3 runtime_error, 4 logic_error, 9 other
int code_of(const std::exception& e) {
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
    if (dynamic_cast<const std::runtime_error*>(&e)) return 3;
    if (dynamic_cast<const std::logic_error*>(&e)) return 4;
    return 9;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

struct Seq {
    std::unique_ptr<PagedKVCache> cache;
    BlockAssignment assignment;
    CentroidStore store;
    std::optional<QuantizedCentroidStore> qstore;
    SelectionResult sel;
};

struct Engine {
    std::unique_ptr<DecodeEngine> engine;
    StepResult last;
};

std::optional<QuantSpec> make_spec(int bits, int mode) {
    if (bits == 0) return std::nullopt;
    QuantSpec s;
    s.bits = bits;
    s.mode = mode == 0 ? QuantMode::kSymmetric : QuantMode::kAsymmetric;
    return s;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// keys/values: [H][n][d] fp32 (head-major, as DecodeEngine::prefill takes them).
// method: 0 mean, 1 maxmin. bits: 0 (no quant), 2, 4, 8. mode: 0 sym, 1 asym.
int ref_seq_create(size_t H, size_t d, size_t P, size_t n, size_t capacity, const float* keys,
                   const float* values, const size_t* block_sizes, int method, int bits, int mode,
                   void** out) {
    return guard([&] {
        auto s = std::make_unique<Seq>();
        s->cache = std::make_unique<PagedKVCache>(H, d, P, std::max(capacity, n));
        std::vector<float> k(H * d), v(H * d);
        for (size_t t = 0; t < n; ++t) {
            for (size_t h = 0; h < H; ++h) {
                std::memcpy(k.data() + h * d, keys + (h * n + t) * d, d * sizeof(float));
                std::memcpy(v.data() + h * d, values + (h * n + t) * d, d * sizeof(float));
            }
            s->cache->append(k, v);
        }
        s->assignment.block_sizes.assign(block_sizes, block_sizes + H);
        s->store = compute_block_centroids(*s->cache, s->assignment,
                                           method == 0 ? CentroidMethod::kMean
                                                       : CentroidMethod::kMaxMin);
        if (auto spec = make_spec(bits, mode)) s->qstore = quantize_store(s->store, *spec);
        *out = s.release();
    });
}

void ref_seq_destroy(void* h) { delete static_cast<Seq*>(h); }

size_t ref_seq_total_centroids(void* h) { return static_cast<Seq*>(h)->store.total_centroids(); }

// offsets: H+1 entries.
void ref_seq_offsets(void* h, uint64_t* offsets) {
    const auto& o = static_cast<Seq*>(h)->store.offsets;
    for (size_t i = 0; i < o.size(); ++i) offsets[i] = o[i];
}

// Any output pointer may be null. values/_min: [total][d] fp32; codes/_min: [total][d] u8;
// scales/zps(/_min): [H][d].
int ref_seq_store(void* h, float* values, float* values_min, uint8_t* codes, uint8_t* codes_min,
                  float* scales, float* zps, float* scales_min, float* zps_min) {
    return guard([&] {
        const Seq* s = static_cast<Seq*>(h);
        auto cp = [](auto* dst, const auto& src) {
            if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
        };
        cp(values, s->store.values);
        cp(values_min, s->store.values_min);
        if (s->qstore) {
            cp(codes, s->qstore->codes);
            cp(codes_min, s->qstore->codes_min);
            cp(scales, s->qstore->scales);
            cp(zps, s->qstore->zero_points);
            cp(scales_min, s->qstore->scales_min);
            cp(zps_min, s->qstore->zero_points_min);
        }
    });
}

// query: [H][d]; scores: [total]. Uses the quantized store when present
// (engine.cpp:451-452 picks the same way).
int ref_seq_estimate(void* h, const float* query, float* scores) {
    return guard([&] {
        const Seq* s = static_cast<Seq*>(h);
        const size_t qn = s->store.num_heads * s->store.head_dim;
        std::span<const float> q(query, qn);
        std::vector<float> r = s->qstore ? estimate_scores(q, *s->qstore) : estimate_scores(q, s->store);
        std::memcpy(scores, r.data(), r.size() * sizeof(float));
    });
}

int ref_seq_estimate_naive(void* h, const float* query, float* scores) {
    return guard([&] {
        const Seq* s = static_cast<Seq*>(h);
        const size_t qn = s->store.num_heads * s->store.head_dim;
        std::span<const float> q(query, qn);
        std::vector<float> r =
            s->qstore ? estimate_scores_naive(q, *s->qstore) : estimate_scores_naive(q, s->store);
        std::memcpy(scores, r.data(), r.size() * sizeof(float));
    });
}

// Runs select_topk on caller scores; stores the selection (with page spans) in
// the handle. blocks: [H][max_k] (row stride max_k), counts: [H], budgets: [H].
int ref_seq_select(void* h, const float* scores, size_t token_budget, uint32_t* blocks,
                   size_t max_k, uint32_t* counts, uint32_t* budgets) {
    return guard([&] {
        Seq* s = static_cast<Seq*>(h);
        std::vector<float> sc(scores, scores + s->store.total_centroids());
        s->sel = select_topk(sc, s->store.offsets, s->assignment, s->cache->seq_len(), token_budget);
        populate_page_spans(s->sel, *s->cache);
        for (size_t hh = 0; hh < s->sel.num_heads; ++hh) {
            const auto& b = s->sel.blocks[hh];
            if (b.size() > max_k) throw std::invalid_argument("ref_seq_select: max_k too small");
            counts[hh] = static_cast<uint32_t>(b.size());
            budgets[hh] = static_cast<uint32_t>(s->sel.budget_blocks[hh]);
            for (size_t j = 0; j < b.size(); ++j) blocks[hh * max_k + j] = static_cast<uint32_t>(b[j]);
        }
    });
}

int ref_seq_select_naive(void* h, const float* scores, size_t token_budget, uint32_t* blocks,
                         size_t max_k, uint32_t* counts) {
    return guard([&] {
        Seq* s = static_cast<Seq*>(h);
        std::vector<float> sc(scores, scores + s->store.total_centroids());
        SelectionResult r = select_topk_naive(sc, s->store.offsets, s->assignment,
                                              s->cache->seq_len(), token_budget);
        for (size_t hh = 0; hh < r.num_heads; ++hh) {
            counts[hh] = static_cast<uint32_t>(r.blocks[hh].size());
            for (size_t j = 0; j < r.blocks[hh].size(); ++j)
                blocks[hh * max_k + j] = static_cast<uint32_t>(r.blocks[hh][j]);
        }
    });
}

// sparse_attention over the selection stored by ref_seq_select. query/out: [H][d].
int ref_seq_attend(void* h, const float* query, float* out) {
    return guard([&] {
        const Seq* s = static_cast<Seq*>(h);
        const size_t qn = s->store.num_heads * s->store.head_dim;
        AttentionOutput o = sparse_attention(std::span<const float>(query, qn), *s->cache, s->sel);
        std::memcpy(out, o.output.data(), qn * sizeof(float));
    });
}

int ref_seq_full_attention(void* h, const float* query, float* out) {
    return guard([&] {
        const Seq* s = static_cast<Seq*>(h);
        const size_t qn = s->store.num_heads * s->store.head_dim;
        AttentionOutput o = full_attention_oracle(std::span<const float>(query, qn), *s->cache);
        std::memcpy(out, o.output.data(), qn * sizeof(float));
    });
}

// full_attention_oracle with its weights. query/out: [H][d]; weights: [H][n] fp64.
int ref_seq_full_attention_w(void* h, const float* query, float* out, double* weights) {
    return guard([&] {
        const Seq* s = static_cast<Seq*>(h);
        const size_t qn = s->store.num_heads * s->store.head_dim;
        AttentionOutput o = full_attention_oracle(std::span<const float>(query, qn), *s->cache);
        std::memcpy(out, o.output.data(), qn * sizeof(float));
        std::memcpy(weights, o.weights.data(), o.weights.size() * sizeof(double));
    });
}

// One GQA decode step per SURVEY.md Appendix A: q_group is [Hkv*G][d]
// (q head hq = h*G + g). The KV-head query used for scoring is the left-to-right
// fp32 group sum; attention runs once per group member. out: [Hkv*G][d].
// scores/blocks/counts may be null.
int ref_seq_decode_gqa(void* h, const float* q_group, size_t G, size_t token_budget, float* out) {
    return guard([&] {
        Seq* s = static_cast<Seq*>(h);
        const size_t H = s->store.num_heads, d = s->store.head_dim;
        std::vector<float> qsum(H * d);
        for (size_t hh = 0; hh < H; ++hh)
            for (size_t c = 0; c < d; ++c) {
                float acc = q_group[(hh * G) * d + c];
                for (size_t g = 1; g < G; ++g) acc += q_group[(hh * G + g) * d + c];
                qsum[hh * d + c] = acc;
            }
        std::vector<float> sc = s->qstore ? estimate_scores(qsum, *s->qstore)
                                          : estimate_scores(qsum, s->store);
        s->sel = select_topk(sc, s->store.offsets, s->assignment, s->cache->seq_len(), token_budget);
        populate_page_spans(s->sel, *s->cache);
        std::vector<float> qg(H * d);
        for (size_t g = 0; g < G; ++g) {
            for (size_t hh = 0; hh < H; ++hh)
                std::memcpy(qg.data() + hh * d, q_group + (hh * G + g) * d, d * sizeof(float));
            AttentionOutput o = sparse_attention(qg, *s->cache, s->sel);
            for (size_t hh = 0; hh < H; ++hh)
                std::memcpy(out + (hh * G + g) * d, o.output.data() + hh * d, d * sizeof(float));
        }
    });
}

// ---- DecodeEngine (engine.hpp:99-129) ------------------------------------
int ref_engine_create(size_t H, size_t d, size_t P, const size_t* cands, size_t n_cands,
                      size_t token_budget, int method, int bits, int mode,
                      const size_t* block_sizes, size_t capacity, void** out) {
    return guard([&] {
        EngineConfig cfg;
        cfg.num_heads = H;
        cfg.head_dim = d;
        cfg.page_size = P;
        cfg.candidate_block_sizes.assign(cands, cands + n_cands);
        cfg.token_budget = token_budget;
        cfg.centroid_method = method == 0 ? CentroidMethod::kMean : CentroidMethod::kMaxMin;
        cfg.quant = make_spec(bits, mode);
        BlockAssignment a;
        a.block_sizes.assign(block_sizes, block_sizes + H);
        auto e = std::make_unique<Engine>();
        e->engine = std::make_unique<DecodeEngine>(cfg, a, capacity);
        *out = e.release();
    });
}

void ref_engine_destroy(void* h) { delete static_cast<Engine*>(h); }

int ref_engine_prefill(void* h, const float* keys, const float* values, size_t n, size_t per_head) {
    return guard([&] {
        Engine* e = static_cast<Engine*>(h);
        const size_t H = e->engine->config().num_heads;
        const size_t d = e->engine->config().head_dim;
        e->engine->prefill(std::span<const float>(keys, H * per_head * d),
                           std::span<const float>(values, H * per_head * d), n);
    });
}

// k/v/q: [H][d]. out: [H][d]. blocks: [H][max_k]; counts: [H]. fallback: 0/1.
int ref_engine_step(void* h, const float* k, const float* v, const float* q, float* out,
                    uint32_t* blocks, size_t max_k, uint32_t* counts, int* fallback) {
    return guard([&] {
        Engine* e = static_cast<Engine*>(h);
        const size_t H = e->engine->config().num_heads;
        const size_t d = e->engine->config().head_dim;
        e->last = e->engine->step(std::span<const float>(k, H * d), std::span<const float>(v, H * d),
                                  std::span<const float>(q, H * d));
        std::memcpy(out, e->last.output.output.data(), H * d * sizeof(float));
        if (fallback) *fallback = e->last.full_attention_fallback ? 1 : 0;
        if (blocks && counts) {
            for (size_t hh = 0; hh < H; ++hh) {
                const auto& b = e->last.selection.blocks[hh];
                if (b.size() > max_k) throw std::invalid_argument("ref_engine_step: max_k too small");
                counts[hh] = static_cast<uint32_t>(b.size());
                for (size_t j = 0; j < b.size(); ++j) blocks[hh * max_k + j] = static_cast<uint32_t>(b[j]);
            }
        }
    });
}

// Quantized-store snapshot of the engine (after prefill/step) for parity checks.
int ref_engine_store(void* h, uint64_t* offsets, float* values, uint8_t* codes, float* scales,
                     float* zps, size_t* total) {
    return guard([&] {
        const Engine* e = static_cast<Engine*>(h);
        const CentroidStore& st = e->engine->centroids();
        if (total) *total = st.total_centroids();
        if (offsets)
            for (size_t i = 0; i < st.offsets.size(); ++i) offsets[i] = st.offsets[i];
        if (values) std::memcpy(values, st.values.data(), st.values.size() * sizeof(float));
        const QuantizedCentroidStore* q = e->engine->quantized();
        if (q) {
            if (codes) std::memcpy(codes, q->codes.data(), q->codes.size());
            if (scales) std::memcpy(scales, q->scales.data(), q->scales.size() * sizeof(float));
            if (zps) std::memcpy(zps, q->zero_points.data(), q->zero_points.size() * sizeof(float));
        }
    });
}

// ---- config validation (config.cpp:48-78) and assignment validation -------
int ref_config_validate(size_t H, size_t d, size_t P, const size_t* cands, size_t n_cands,
                        size_t token_budget, int bits) {
    return guard([&] {
        EngineConfig cfg;
        cfg.num_heads = H;
        cfg.head_dim = d;
        cfg.page_size = P;
        cfg.candidate_block_sizes.assign(cands, cands + n_cands);
        cfg.token_budget = token_budget;
        if (bits) cfg.quant = QuantSpec{bits, QuantMode::kAsymmetric};
        cfg.validate();
    });
}

// ---- workload generator (test-data source only; workload.cpp:192-249) ----
// kinds: 0 uniform, 1 clustered(a=count, b=width), 2 scattered(a=hot tokens).
int ref_generate_synthetic(size_t n, size_t H, size_t d, const int* kinds, const size_t* a,
                           const size_t* b, double signal, uint64_t seed, size_t scatter_gap,
                           float* keys, float* values, float* queries) {
    return guard([&] {
        WorkloadSpec spec;
        spec.seq_len = n;
        spec.num_heads = H;
        spec.head_dim = d;
        spec.signal_strength = signal;
        spec.seed = seed;
        spec.scatter_gap = scatter_gap;
        for (size_t h = 0; h < H; ++h) {
            if (kinds[h] == 1) spec.head_profiles.push_back(HeadProfile::clustered(a[h], b[h]));
            else if (kinds[h] == 2) spec.head_profiles.push_back(HeadProfile::scattered(a[h]));
            else spec.head_profiles.push_back(HeadProfile::uniform());
        }
        Trace t = generate_synthetic(spec);
        std::memcpy(keys, t.keys.data(), t.keys.size() * sizeof(float));
        std::memcpy(values, t.values.data(), t.values.size() * sizeof(float));
        std::memcpy(queries, t.queries.data(), t.queries.size() * sizeof(float));
    });
}

// ---- trace I/O and calibration (workload.cpp:260-309, calibrator.cpp) ----------
int ref_save_trace(const char* path, size_t H, size_t d, size_t n, uint64_t seed, const float* keys,
                   const float* values, const float* queries) {
    return guard([&] {
        Trace t;
        t.num_heads = H;
        t.head_dim = d;
        t.seq_len = n;
        t.seed = seed;
        t.keys.assign(keys, keys + H * n * d);
        t.values.assign(values, values + H * n * d);
        t.queries.assign(queries, queries + H * d);
        save_trace(t, path);
    });
}

// dims: H, d, n, seed (as u64 x4); arrays sized by the caller after a first call with
// keys == nullptr (dims only).
int ref_load_trace(const char* path, uint64_t* dims, float* keys, float* values, float* queries) {
    return guard([&] {
        const Trace t = load_trace(path);
        dims[0] = t.num_heads;
        dims[1] = t.head_dim;
        dims[2] = t.seq_len;
        dims[3] = t.seed;
        if (!keys) return;
        std::memcpy(keys, t.keys.data(), t.keys.size() * 4);
        std::memcpy(values, t.values.data(), t.values.size() * 4);
        std::memcpy(queries, t.queries.data(), t.queries.size() * 4);
    });
}

namespace {
EngineConfig calib_config(size_t H, size_t d, size_t P, const size_t* cands, size_t nc, size_t T, int method,
                          int bits, int mode) {
    EngineConfig c;
    c.num_heads = H;
    c.head_dim = d;
    c.page_size = P;
    c.candidate_block_sizes.assign(cands, cands + nc);
    c.token_budget = T;
    c.centroid_method = method == 0 ? CentroidMethod::kMean : CentroidMethod::kMaxMin;
    c.quant = make_spec(bits, mode);
    return c;
}
// samples back to back: keys/values [S][H][n][d], queries [S][H][d]
TraceProvider calib_provider(size_t H, size_t d, size_t n, const float* keys, const float* values,
                             const float* queries) {
    return [=](size_t i) {
        Trace t;
        t.num_heads = H;
        t.head_dim = d;
        t.seq_len = n;
        t.seed = i;
        const size_t per = H * n * d;
        t.keys.assign(keys + i * per, keys + (i + 1) * per);
        t.values.assign(values + i * per, values + (i + 1) * per);
        t.queries.assign(queries + i * H * d, queries + (i + 1) * H * d);
        return t;
    };
}
}  // namespace

// recalls: [H][nc]
int ref_profile_sensitivity(size_t H, size_t d, size_t P, const size_t* cands, size_t nc, size_t T, int method,
                            int bits, int mode, size_t samples, size_t n, const float* keys, const float* values,
                            const float* queries, double* recalls) {
    return guard([&] {
        const EngineConfig c = calib_config(H, d, P, cands, nc, T, method, bits, mode);
        const RecallTable t = profile_sensitivity(calib_provider(H, d, n, keys, values, queries), samples, c);
        std::memcpy(recalls, t.recalls.data(), t.recalls.size() * sizeof(double));
    });
}

// out: adaptive_recall, delta, avg_block_size, matched_candidate, uniform_recalls[nc]
int ref_transfer_check(size_t H, size_t d, size_t P, const size_t* cands, size_t nc, size_t T, int method,
                       int bits, int mode, const size_t* block_sizes, size_t samples, size_t n, const float* keys,
                       const float* values, const float* queries, double* out) {
    return guard([&] {
        const EngineConfig c = calib_config(H, d, P, cands, nc, T, method, bits, mode);
        BlockAssignment a;
        a.block_sizes.assign(block_sizes, block_sizes + H);
        const TransferReport r = transfer_check(a, calib_provider(H, d, n, keys, values, queries), samples, c);
        out[0] = r.adaptive_recall;
        out[1] = r.delta;
        out[2] = r.avg_block_size;
        out[3] = double(r.matched_candidate);
        for (size_t i = 0; i < nc; ++i) out[4 + i] = r.uniform_recalls[i];
    });
}

int ref_write_recall_csv(const char* path, size_t H, const size_t* cands, size_t nc, const double* recalls,
                         const char* tag) {
    return guard([&] {
        RecallTable t;
        t.num_heads = H;
        t.candidates.assign(cands, cands + nc);
        t.recalls.assign(recalls, recalls + H * nc);
        write_recall_csv(path, t, tag);
    });
}

int ref_write_min_block_csv(const char* path, const size_t* sizes, size_t H, const char* tag) {
    return guard([&] { write_min_block_csv(path, std::vector<std::size_t>(sizes, sizes + H), tag); });
}

int ref_assign_block_sizes(size_t H, const size_t* cands, size_t nc, const double* recalls, double tau,
                           size_t* out) {
    return guard([&] {
        RecallTable t;
        t.num_heads = H;
        t.candidates.assign(cands, cands + nc);
        t.recalls.assign(recalls, recalls + H * nc);
        const BlockAssignment a = assign_block_sizes(t, tau);
        for (size_t h = 0; h < H; ++h) out[h] = a.block_sizes[h];
    });
}

}  // extern "C"
