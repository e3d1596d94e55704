// C++ host-side test of the drop-in boundary: a reference-style call site written
// against include/absp.hpp (namespace absp, std:: exceptions) over libabsp.so.
//
//   test_host_cpp cpu  : no GPU needed — config / assignment validation with the
//                        reference's exception classes (config.cpp:48-78,
//                        centroids.cpp:59-76), build_offsets KAT
//                        (test_centroids.cpp:65-82), assignment file round trip
//                        (calibrator.cpp:277-311), and no CPU fallback.
//   test_host_cpp gpu  : one decode step on cuda:0 through DecodeAttention,
//                        checked against the C oracle (oracle/absp_oracle.c, the
//                        checker only): store + scores bit-exact, ordered
//                        selections equal, output within 1e-3 + 1e-2|want|.
// Prints "OK <mode>" and exits 0 on success; any failure exits 1 with a message.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "absp.hpp"
#include "../../oracle/absp_oracle.h"

namespace {

int g_fail = 0;
#define EXPECT(cond)                                                         \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #cond); \
            ++g_fail;                                                        \
        }                                                                    \
    } while (0)

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

absp::EngineConfig base_config() {
    absp::EngineConfig c;
    c.num_heads = 8;
    c.head_dim = 128;
    c.page_size = 16;
    c.candidate_block_sizes = {16, 32, 64};
    c.token_budget = 512;
    c.quant = absp::QuantSpec{4, absp::QuantMode::kAsymmetric};
    c.num_q_heads = 32;
    c.max_batch = 2;
    c.max_seq_len = 4096;
    return c;
}

void cpu_tests(const char* tmpdir) {
    // EngineConfig::validate semantics (config.cpp:48-78).
    absp::EngineConfig c = base_config();
    c.validate();
    { auto b = c; b.page_size = 0; EXPECT(throws<std::invalid_argument>([&] { b.validate(); })); }
    { auto b = c; b.candidate_block_sizes = {16, 24}; EXPECT(throws<std::invalid_argument>([&] { b.validate(); })); }
    { auto b = c; b.candidate_block_sizes = {32, 16}; EXPECT(throws<std::invalid_argument>([&] { b.validate(); })); }
    { auto b = c; b.candidate_block_sizes = {16, 16}; EXPECT(throws<std::invalid_argument>([&] { b.validate(); })); }
    { auto b = c; b.token_budget = 32; EXPECT(throws<std::invalid_argument>([&] { b.validate(); })); }
    { auto b = c; b.recall_threshold = 0.0; EXPECT(throws<std::invalid_argument>([&] { b.validate(); })); }
    { auto b = c; b.quant = absp::QuantSpec{3}; EXPECT(throws<std::invalid_argument>([&] { b.validate(); })); }
    EXPECT(absp::quant_spec_name(absp::parse_quant_spec("int8xsym")) == "int8xsym");
    EXPECT(throws<std::invalid_argument>([] { absp::parse_quant_spec("int5xasym"); }));

    // BlockAssignment::validate (centroids.cpp:59-76).
    absp::BlockAssignment a = absp::BlockAssignment::cycled(8, {16, 32, 64});
    a.validate(c);
    { auto b = a; b.block_sizes[3] = 48; EXPECT(throws<std::invalid_argument>([&] { b.validate(c); })); }
    { auto b = a; b.block_sizes.pop_back(); EXPECT(throws<std::invalid_argument>([&] { b.validate(c); })); }

    // build_offsets KAT, test_centroids.cpp:65-82: {32,64,16} @ 128 -> [0,4,6,14].
    const auto off = absp::build_offsets(128, absp::BlockAssignment{{32, 64, 16}});
    EXPECT((off == std::vector<std::size_t>{0, 4, 6, 14}));

    // Assignment file round trip + malformed input (calibrator.cpp:277-311).
    const std::string path = std::string(tmpdir) + "/assignment.txt";
    absp::BlockAssignment{{16, 64, 32}}.save(path);
    EXPECT((absp::BlockAssignment::load(path).block_sizes == std::vector<std::size_t>{16, 64, 32}));
    {
        FILE* f = std::fopen(path.c_str(), "w");
        std::fputs("0 16\n2 32\n", f);
        std::fclose(f);
        EXPECT(throws<std::runtime_error>([&] { absp::BlockAssignment::load(path); }));
    }

    // No CPU fallback: without a usable B200 the context cannot be created.
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        EXPECT(throws<absp::cuda_error>([&] { absp::DecodeAttention da(c); }));
    }
}

float bf16f(uint16_t x) {
    uint32_t u = uint32_t(x) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
        std::exit(1);
    }
}

void gpu_tests() {
    const absp::EngineConfig cfg = base_config();
    const std::size_t H = cfg.num_heads, G = cfg.group_size(), d = cfg.head_dim, P = cfg.page_size;
    const std::vector<uint32_t> lens = {3000, 1777};
    const uint32_t batch = uint32_t(lens.size());
    const uint32_t max_pages = uint32_t((cfg.max_seq_len + P - 1) / P);
    std::size_t used = 0;
    for (uint32_t n : lens) used += (n + P - 1) / P;
    const uint64_t pool_pages = used + 5;

    absp::DecodeAttention da(cfg);
    const absp::BlockAssignment asg = absp::BlockAssignment::cycled(H, cfg.candidate_block_sizes);
    da.set_assignment(0, asg);

    // Reference-style misuse surfaces as the reference's exception classes.
    EXPECT(throws<std::out_of_range>([&] { da.set_assignment(7, asg); }));
    EXPECT(throws<std::logic_error>([&] { da.build_store(0); }));

    // caller-owned device cache: pools, page table (scattered pages), queries
    const std::size_t pool_elems = H * pool_pages * P * d, q_elems = batch * H * G * d;
    uint16_t *k = nullptr, *v = nullptr, *q = nullptr;
    uint32_t* pt = nullptr;
    float* out = nullptr;
    cuda_ok(cudaMalloc(&k, pool_elems * 2), "malloc k");
    cuda_ok(cudaMalloc(&v, pool_elems * 2), "malloc v");
    cuda_ok(cudaMalloc(&q, q_elems * 2), "malloc q");
    cuda_ok(cudaMalloc(&pt, batch * max_pages * 4), "malloc pt");
    cuda_ok(cudaMalloc(&out, q_elems * 4), "malloc out");
    absp::check(absp_fill_synthetic_bf16(k, pool_elems, 7, 0, nullptr));
    absp::check(absp_fill_synthetic_bf16(v, pool_elems, 7, 1, nullptr));
    absp::check(absp_fill_synthetic_bf16(q, q_elems, 7, 2, nullptr));
    std::vector<uint32_t> table(batch * max_pages, 0);
    std::vector<uint32_t> perm(pool_pages);
    for (uint64_t i = 0; i < pool_pages; ++i) perm[i] = uint32_t((i * 13 + 5) % pool_pages);
    std::size_t o = 0;
    for (uint32_t b = 0; b < batch; ++b)
        for (uint32_t p = 0; p < (lens[b] + P - 1) / P; ++p) table[b * max_pages + p] = perm[o++];
    cuda_ok(cudaMemcpy(pt, table.data(), table.size() * 4, cudaMemcpyHostToDevice), "copy pt");

    {  // capacity: a sequence longer than max_seq_len (kv_cache.cpp:48-50)
        std::vector<uint32_t> too_long = {uint32_t(cfg.max_seq_len + 1)};
        EXPECT(throws<std::runtime_error>([&] { da.bind(0, k, v, pool_pages, pt, max_pages, too_long); }));
    }
    da.bind(0, k, v, pool_pages, pt, max_pages, lens);
    EXPECT(throws<std::logic_error>([&] { da.decode_step(0, q, out); }));  // store not built
    da.build_store(0);
    // absp_select fills the reference's full estimate_scores output (checked below);
    // absp_decode_step selects through its own path and must pick the same blocks
    const absp_layer_info info = da.layer_info(0);
    uint32_t *sblocks = nullptr, *scounts = nullptr;
    cuda_ok(cudaMalloc(&sblocks, batch * H * info.max_select * 4), "malloc sblocks");
    cuda_ok(cudaMalloc(&scounts, batch * H * 4), "malloc scounts");
    da.select(0, q, sblocks, info.max_select, scounts);
    cuda_ok(cudaDeviceSynchronize(), "select");
    std::vector<std::vector<float>> exact_scores;
    for (uint32_t b = 0; b < batch; ++b) exact_scores.push_back(da.download_scores(0, b));
    da.decode_step(0, q, out);
    cuda_ok(cudaDeviceSynchronize(), "decode_step");

    std::vector<uint16_t> hk(pool_elems), hv(pool_elems), hq(q_elems);
    std::vector<float> got(q_elems);
    cuda_ok(cudaMemcpy(hk.data(), k, pool_elems * 2, cudaMemcpyDeviceToHost), "k");
    cuda_ok(cudaMemcpy(hv.data(), v, pool_elems * 2, cudaMemcpyDeviceToHost), "v");
    cuda_ok(cudaMemcpy(hq.data(), q, q_elems * 2, cudaMemcpyDeviceToHost), "q");
    cuda_ok(cudaMemcpy(got.data(), out, q_elems * 4, cudaMemcpyDeviceToHost), "out");
    const uint32_t *sel_blocks = nullptr, *sel_counts = nullptr;
    uint32_t stride = 0;
    absp::check(absp_last_selection(da.handle(), 0, &sel_blocks, &stride, &sel_counts));
    std::vector<uint32_t> dblocks(batch * H * stride), dcounts(batch * H);
    cuda_ok(cudaMemcpy(dblocks.data(), sel_blocks, dblocks.size() * 4, cudaMemcpyDeviceToHost), "blocks");
    cuda_ok(cudaMemcpy(dcounts.data(), sel_counts, dcounts.size() * 4, cudaMemcpyDeviceToHost), "counts");

    std::vector<uint32_t> bs(asg.block_sizes.begin(), asg.block_sizes.end());
    double max_err = 0.0;
    for (uint32_t b = 0; b < batch; ++b) {
        const std::size_t n = lens[b];
        const uint32_t* ptb = table.data() + b * max_pages;
        std::vector<uint64_t> offs(H + 1);
        absp_oracle_offsets(n, bs.data(), H, offs.data());
        const std::size_t total = offs[H];
        std::vector<float> vals(total * d), scales(H * d), zps(H * d), scores(total);
        std::vector<uint8_t> codes(total * d);
        EXPECT(absp_oracle_centroids(hk.data(), pool_pages, ptb, n, H, d, P, bs.data(), 0, vals.data(), nullptr) == 0);
        EXPECT(absp_oracle_quantize(vals.data(), offs.data(), H, d, 4, 1, codes.data(), scales.data(), zps.data()) == 0);
        // selection query: fp32 left-to-right group sum
        std::vector<float> qs(H * d), qg(H * d);
        for (std::size_t h = 0; h < H; ++h)
            for (std::size_t c = 0; c < d; ++c) {
                float acc = bf16f(hq[((b * H + h) * G) * d + c]);
                for (std::size_t g = 1; g < G; ++g) {
                    volatile float t = acc + bf16f(hq[((b * H + h) * G + g) * d + c]);
                    acc = t;
                }
                qs[h * d + c] = acc;
            }
        absp_oracle_scores_quant(qs.data(), codes.data(), nullptr, scales.data(), zps.data(), nullptr, nullptr,
                                 offs.data(), H, d, 4, 1, 0, scores.data());
        const std::size_t max_k = stride;
        std::vector<uint32_t> wblocks(H * max_k), wcounts(H);
        EXPECT(absp_oracle_select(scores.data(), offs.data(), bs.data(), H, n, cfg.token_budget, wblocks.data(),
                                  max_k, wcounts.data(), nullptr) == 0);

        const absp::StoreSnapshot st = da.download_store(0, b);
        EXPECT(st.offsets == std::vector<std::size_t>(offs.begin(), offs.end()));
        EXPECT(std::memcmp(st.values.data(), vals.data(), vals.size() * 4) == 0);
        EXPECT(st.codes == codes);
        EXPECT(std::memcmp(st.scales.data(), scales.data(), scales.size() * 4) == 0);
        EXPECT(std::memcmp(st.zero_points.data(), zps.data(), zps.size() * 4) == 0);
        const std::vector<float>& dsc = exact_scores[b];
        EXPECT(dsc.size() == scores.size() && std::memcmp(dsc.data(), scores.data(), scores.size() * 4) == 0);
        for (std::size_t h = 0; h < H; ++h) {
            EXPECT(dcounts[b * H + h] == wcounts[h]);
            EXPECT(std::memcmp(dblocks.data() + (b * H + h) * stride, wblocks.data() + h * max_k,
                               wcounts[h] * 4) == 0);
        }
        // attention per group member g over its KV head's selection
        for (std::size_t g = 0; g < G; ++g) {
            std::vector<float> qm(H * d), want(H * d);
            for (std::size_t h = 0; h < H; ++h)
                for (std::size_t c = 0; c < d; ++c) qm[h * d + c] = bf16f(hq[((b * H + h) * G + g) * d + c]);
            EXPECT(absp_oracle_attend(qm.data(), hk.data(), hv.data(), pool_pages, ptb, n, H, d, P, bs.data(),
                                      wblocks.data(), max_k, wcounts.data(), want.data()) == 0);
            for (std::size_t h = 0; h < H; ++h)
                for (std::size_t c = 0; c < d; ++c) {
                    const double w = want[h * d + c], x = got[((b * H + h) * G + g) * d + c];
                    const double err = std::fabs(x - w);
                    max_err = err > max_err ? err : max_err;
                    EXPECT(err <= 1e-3 + 1e-2 * std::fabs(w));
                }
        }
    }
    std::printf("max attention error %.3g, %llu kernel launches\n", max_err,
                (unsigned long long)da.launch_count());
    cudaFree(sblocks);
    cudaFree(scounts);
    cudaFree(k);
    cudaFree(v);
    cudaFree(q);
    cudaFree(pt);
    cudaFree(out);
}

}  // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    try {
        if (mode == "cpu") cpu_tests(argc > 2 ? argv[2] : "/tmp");
        else gpu_tests();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "unexpected exception: %s\n", e.what());
        return 1;
    }
    if (g_fail) {
        std::fprintf(stderr, "%d expectation(s) failed\n", g_fail);
        return 1;
    }
    std::printf("OK %s\n", mode.c_str());
    return 0;
}
