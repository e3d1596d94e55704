// absp::DecodeEngine (include/absp.hpp over the absp_engine_* C ABI: no PyTorch, the
// engine owns its device cache, store and stream) against the reference's own
// DecodeEngine (engine.hpp:99-129, engine.cpp:405-463; the unmodified reference core in
// oracle/_ref, reached through the test shim's C functions — the checker, never the
// product).
//
//   prefill, then >= 100 decode steps (append + refresh_tail_centroids +
//   requantize_heads + estimate -> select -> attend), crossing the token budget (the
//   reference's full-attention fallback) and many block boundaries:
//     store (offsets, centroids, codes, scales, zero points) after every step : bit-exact
//     ordered selection per head                                              : equal
//     output                                              : |got-want| <= 1e-3 + 1e-2|want|
//   plus the reference's exception classes for misuse.
// Prints "OK engine" and exits 0 on success.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "absp.hpp"

extern "C" {  // oracle/ref_shim.cpp (oracle/_ref/libabsparse_ref.so)
int ref_engine_create(size_t H, size_t d, size_t P, const size_t* cands, size_t n_cands, size_t token_budget,
                      int method, int bits, int mode, const size_t* block_sizes, size_t capacity, void** out);
void ref_engine_destroy(void* h);
int ref_engine_prefill(void* h, const float* keys, const float* values, size_t n, size_t per_head);
int ref_engine_step(void* h, const float* k, const float* v, const float* q, float* out, uint32_t* blocks,
                    size_t max_k, uint32_t* counts, int* fallback);
int ref_engine_store(void* h, uint64_t* offsets, float* values, uint8_t* codes, float* scales, float* zps,
                     size_t* total);
const char* ref_last_error();
}

namespace {

int g_fail = 0;
#define EXPECT(cond)                                                                       \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #cond); \
            if (++g_fail > 20) std::exit(1);                                               \
        }                                                                                  \
    } while (0)

void ref_ok(int rc) {
    if (rc != 0) {
        std::fprintf(stderr, "reference error %d: %s\n", rc, ref_last_error());
        std::exit(1);
    }
}

template <typename E, typename F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// N(0,1) values rounded to bf16 (the engine stores bf16; bf16-representable inputs make
// the reference's fp32 cache hold exactly the same numbers)
std::vector<float> bf16_normals(std::mt19937_64& rng, size_t n) {
    std::normal_distribution<float> nd(0.0f, 1.0f);
    std::vector<float> x(n);
    for (float& v : x) {
        uint32_t u;
        float f = nd(rng);
        std::memcpy(&u, &f, 4);
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
        std::memcpy(&v, &u, 4);
    }
    return x;
}

bool same_bits(const void* a, const void* b, size_t bytes) { return std::memcmp(a, b, bytes) == 0; }

}  // namespace

int main() {
    const size_t H = 4, d = 128, P = 16, T = 256, n0 = 200, steps = 130;
    const std::vector<size_t> cands = {16, 32, 64};
    const std::vector<size_t> bs = {16, 32, 64, 16};
    const size_t cap = n0 + steps + 5;

    absp::EngineConfig cfg;
    cfg.num_heads = H;
    cfg.head_dim = d;
    cfg.page_size = P;
    cfg.candidate_block_sizes = cands;
    cfg.token_budget = T;
    cfg.quant = absp::QuantSpec{4, absp::QuantMode::kAsymmetric};
    absp::BlockAssignment assignment{bs};

    // misuse first: the reference's exception classes
    {
        absp::BlockAssignment bad{{16, 48, 64, 16}};
        EXPECT(throws<std::invalid_argument>([&] { absp::DecodeEngine e(cfg, bad, cap); }));
        EXPECT(throws<std::invalid_argument>([&] { absp::DecodeEngine e(cfg, assignment, 0); }));
        absp::DecodeEngine e(cfg, assignment, 40);
        std::vector<float> z(H * d, 0.0f);
        EXPECT(throws<std::logic_error>([&] { e.step(z, z, z); }));  // engine.cpp:444
        std::vector<float> small(H * 10 * d, 1.0f);
        EXPECT(throws<std::invalid_argument>([&] { e.prefill(small, small, 11); }));  // engine.cpp:420-423
        std::vector<float> big(H * 41 * d, 1.0f);
        EXPECT(throws<std::runtime_error>([&] { e.prefill(big, big, 41); }));  // capacity
        std::vector<float> ok(H * 38 * d, 1.0f);
        e.prefill(ok, ok, 38);
        EXPECT(throws<std::logic_error>([&] { e.prefill(ok, ok, 38); }));  // engine.cpp:416
        std::vector<float> wrong(H * d + 1, 0.0f);
        EXPECT(throws<std::invalid_argument>([&] { e.step(wrong, z, z); }));  // kv_cache.cpp:45-47
        EXPECT(throws<std::invalid_argument>([&] { e.step(z, z, wrong); }));  // engine.cpp:74-76
        e.step(z, z, z);
        e.step(z, z, z);
        EXPECT(e.seq_len() == 40);
        EXPECT(throws<std::runtime_error>([&] { e.step(z, z, z); }));  // kv_cache.cpp:48-50
    }

    absp::DecodeEngine eng(cfg, assignment, cap);
    void* ref = nullptr;
    ref_ok(ref_engine_create(H, d, P, cands.data(), cands.size(), T, 0, 4, 1, bs.data(), cap, &ref));

    std::mt19937_64 rng(2024);
    const std::vector<float> keys = bf16_normals(rng, H * n0 * d), vals = bf16_normals(rng, H * n0 * d);
    eng.prefill(keys, vals, n0);
    ref_ok(ref_engine_prefill(ref, keys.data(), vals.data(), n0, n0));

    const size_t max_k = T / 16 + 1;
    std::vector<float> want(H * d);
    std::vector<uint32_t> wb(H * max_k), wc(H);
    size_t fallbacks = 0;
    double max_err = 0.0;
    for (size_t s = 0; s < steps; ++s) {
        const std::vector<float> k = bf16_normals(rng, H * d), v = bf16_normals(rng, H * d),
                                 q = bf16_normals(rng, H * d);
        const absp::StepResult got = eng.step(k, v, q);
        int fb = 0;
        ref_ok(ref_engine_step(ref, k.data(), v.data(), q.data(), want.data(), wb.data(), max_k, wc.data(), &fb));
        EXPECT(got.full_attention_fallback == (fb != 0));
        fallbacks += fb;
        for (size_t h = 0; h < H; ++h) {
            EXPECT(got.blocks[h].size() == wc[h]);
            for (size_t j = 0; j < got.blocks[h].size() && j < wc[h]; ++j) EXPECT(got.blocks[h][j] == wb[h * max_k + j]);
        }
        for (size_t i = 0; i < H * d; ++i) {
            const double e = std::fabs(double(got.output[i]) - double(want[i]));
            max_err = std::max(max_err, e);
            EXPECT(e <= 1e-3 + 1e-2 * std::fabs(double(want[i])));
        }
        // store after every step (incremental maintenance vs requantize-everything)
        size_t total = 0;
        ref_ok(ref_engine_store(ref, nullptr, nullptr, nullptr, nullptr, nullptr, &total));
        std::vector<uint64_t> off(H + 1);
        std::vector<float> rv(total * d), rs(H * d), rz(H * d);
        std::vector<uint8_t> rcodes(total * d);
        ref_ok(ref_engine_store(ref, off.data(), rv.data(), rcodes.data(), rs.data(), rz.data(), nullptr));
        const absp::StoreSnapshot st = *eng.quantized();
        EXPECT(st.offsets.size() == H + 1);
        for (size_t h = 0; h <= H; ++h) EXPECT(st.offsets[h] == off[h]);
        EXPECT(st.values.size() == rv.size() && same_bits(st.values.data(), rv.data(), rv.size() * 4));
        EXPECT(st.codes == rcodes);
        EXPECT(same_bits(st.scales.data(), rs.data(), rs.size() * 4));
        EXPECT(same_bits(st.zero_points.data(), rz.data(), rz.size() * 4));
        if (g_fail) {
            std::fprintf(stderr, "first failure at step %zu\n", s);
            break;
        }
    }
    ref_engine_destroy(ref);
    EXPECT(eng.seq_len() == n0 + steps);
    EXPECT(fallbacks == T - n0);  // seq_len n0+1 .. T take the fallback
    if (g_fail) {
        std::fprintf(stderr, "%d failure(s)\n", g_fail);
        return 1;
    }
    std::printf("OK engine: %zu steps (%zu with the full-attention fallback), store bit-exact every step, "
                "max |err| %.3g\n", steps, fallbacks, max_err);
    return 0;
}
