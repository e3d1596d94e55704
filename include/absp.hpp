/*
 * absp.hpp — header-only C++ host layer over the C ABI (absp.h), in the shape of
 * the reference's namespace absparse (/root/reference/proj/include/absparse):
 *
 *   absp::QuantSpec, CentroidMethod, QuantMode   <- config.hpp:11-26
 *   absp::EngineConfig (+ GQA/batch/capacity)     <- config.hpp:36-52
 *   absp::BlockAssignment, build_offsets          <- centroids.hpp:12-26
 *   absp::StoreSnapshot (one sequence's device     <- CentroidStore + QuantizedCentroidStore
 *     store read back in the reference layouts)      centroids.hpp:31-52, quantizer.hpp:18-38
 *   BlockAssignment::load / save                   <- read/write_assignment_file
 *                                                     calibrator.cpp:277-311
 *   absp::DecodeEngine / StepResult               <- DecodeEngine (engine.hpp:84-129): owns its
 *                                                    device cache, store and stream (absp_engine_*)
 *   absp::DecodeAttention                         <- the device replacement of
 *     build_store   = compute_block_centroids + quantize_store (centroids.hpp:56-57,
 *                                                              quantizer.hpp:43)
 *     select        = estimate_scores + select_topk             (engine.hpp:47-68)
 *     attend        = populate_page_spans + sparse_attention     (engine.hpp:71-82)
 *     append        = DecodeEngine::step's append + refresh + requantize (engine.cpp:443-449)
 *     decode_step   = DecodeEngine::step's estimate->select->attend (engine.cpp:450-461)
 *
 * Errors are rethrown as the reference's exception classes:
 *   ABSP_EINVAL -> std::invalid_argument, ABSP_ERANGE -> std::out_of_range,
 *   ABSP_ECAPACITY -> std::runtime_error, ABSP_ESTATE -> std::logic_error,
 *   ABSP_ECUDA / ABSP_ENOMEM -> absp::cuda_error (a std::runtime_error).
 *
 * No CUDA headers are needed: device buffers are plain pointers owned by the
 * caller (streams are cudaStream_t passed as void*). Link with -labsp.
 */
#ifndef ABSP_HPP
#define ABSP_HPP

#include <cstddef>
#include <cstdint>
#include <fstream>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "absp.h"

namespace absp {

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Maps a status onto the reference's exception classes.
inline void check(absp_status st) {
    if (st == ABSP_OK) return;
    const std::string msg = absp_last_error();
    switch (st) {
        case ABSP_EINVAL: throw std::invalid_argument(msg);
        case ABSP_ERANGE: throw std::out_of_range(msg);
        case ABSP_ECAPACITY: throw std::runtime_error(msg);
        case ABSP_ESTATE: throw std::logic_error(msg);
        default: throw cuda_error(msg);
    }
}

enum class CentroidMethod { kMean = ABSP_CENTROID_MEAN, kMaxMin = ABSP_CENTROID_MAXMIN };
enum class QuantMode { kSymmetric = ABSP_QUANT_SYM, kAsymmetric = ABSP_QUANT_ASYM };

// QuantSpec (config.hpp:17-26).
struct QuantSpec {
    int bits = 4;
    QuantMode mode = QuantMode::kAsymmetric;
    int levels() const { return (1 << bits) - 1; }
    int sym_mid() const { return (1 << (bits - 1)) - 1; }
    bool operator==(const QuantSpec& o) const { return bits == o.bits && mode == o.mode; }
    void validate() const {  // config.cpp:8-12
        if (bits != 2 && bits != 4 && bits != 8)
            throw std::invalid_argument("quant bits must be one of {2, 4, 8}");
    }
};

// quant_spec_name / parse_quant_spec (config.cpp:14-28).
inline std::string quant_spec_name(const QuantSpec& s) {
    return "int" + std::to_string(s.bits) + (s.mode == QuantMode::kSymmetric ? "xsym" : "xasym");
}
inline QuantSpec parse_quant_spec(const std::string& name) {
    for (int bits : {2, 4, 8})
        for (QuantMode m : {QuantMode::kSymmetric, QuantMode::kAsymmetric}) {
            QuantSpec s{bits, m};
            if (quant_spec_name(s) == name) return s;
        }
    throw std::invalid_argument("unknown quant spec '" + name + "'");
}

// EngineConfig (config.hpp:36-52) plus the batch / GQA / capacity extensions.
struct EngineConfig {
    std::size_t num_heads = 8;  // KV heads
    std::size_t head_dim = 64;
    std::size_t page_size = 16;
    std::vector<std::size_t> candidate_block_sizes = {16, 32, 64};
    std::size_t token_budget = 4096;
    double recall_threshold = 0.98;
    CentroidMethod centroid_method = CentroidMethod::kMean;
    std::optional<QuantSpec> quant;
    // extensions
    std::size_t num_q_heads = 0;  // 0 = num_heads (MHA)
    std::size_t max_batch = 1;
    std::size_t max_seq_len = 131072;
    std::size_t num_layers = 1;

    std::size_t min_candidate() const {
        std::size_t m = candidate_block_sizes.empty() ? 0 : candidate_block_sizes.front();
        for (std::size_t b : candidate_block_sizes) m = b < m ? b : m;
        return m;
    }
    std::size_t max_candidate() const {
        std::size_t m = 0;
        for (std::size_t b : candidate_block_sizes) m = b > m ? b : m;
        return m;
    }
    std::size_t group_size() const { return (num_q_heads ? num_q_heads : num_heads) / num_heads; }

    absp_config to_abi() const {
        if (candidate_block_sizes.size() > ABSP_MAX_CANDIDATES)
            throw std::invalid_argument("too many candidate block sizes");
        absp_config c{};
        c.num_kv_heads = uint32_t(num_heads);
        c.num_q_heads = uint32_t(num_q_heads ? num_q_heads : num_heads);
        c.head_dim = uint32_t(head_dim);
        c.page_size = uint32_t(page_size);
        c.num_candidates = uint32_t(candidate_block_sizes.size());
        for (std::size_t i = 0; i < candidate_block_sizes.size(); ++i)
            c.candidate_block_sizes[i] = uint32_t(candidate_block_sizes[i]);
        c.token_budget = uint32_t(token_budget);
        c.centroid_method = uint32_t(centroid_method);
        c.quant_bits = quant ? uint32_t(quant->bits) : 0u;
        c.quant_mode = uint32_t(quant ? quant->mode : QuantMode::kAsymmetric);
        c.max_batch = uint32_t(max_batch);
        c.max_seq_len = uint32_t(max_seq_len);
        c.num_layers = uint32_t(num_layers);
        return c;
    }
    // EngineConfig::validate (config.cpp:48-78) + this build's limits.
    void validate() const {
        if (recall_threshold <= 0.0) throw std::invalid_argument("recall_threshold must be positive");
        if (quant) quant->validate();
        const absp_config c = to_abi();
        check(absp_config_validate(&c));
    }
};

// BlockAssignment (centroids.hpp:12-23).
struct BlockAssignment {
    std::vector<std::size_t> block_sizes;

    static BlockAssignment uniform(std::size_t num_heads, std::size_t block_size) {
        return BlockAssignment{std::vector<std::size_t>(num_heads, block_size)};
    }
    // Heads cycle through the candidates (cmd_bench, cli_commands.cpp:445-451).
    static BlockAssignment cycled(std::size_t num_heads, const std::vector<std::size_t>& cands) {
        BlockAssignment a;
        for (std::size_t h = 0; h < num_heads; ++h) a.block_sizes.push_back(cands[h % cands.size()]);
        return a;
    }
    // read_assignment_file (calibrator.cpp:285-311): "head block_size" per line,
    // consecutive heads from 0, empty lines skipped; std::runtime_error otherwise.
    static BlockAssignment load(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw std::runtime_error("read_assignment_file: cannot open " + path);
        BlockAssignment a;
        std::string line;
        std::size_t expected = 0;
        while (std::getline(in, line)) {
            if (line.empty()) continue;
            std::istringstream row(line);
            std::size_t head = 0, block = 0;
            if (!(row >> head >> block) || head != expected)
                throw std::runtime_error("read_assignment_file: malformed line '" + line +
                                         "' (expected 'head block_size' with consecutive heads)");
            std::string extra;
            if (row >> extra)
                throw std::runtime_error("read_assignment_file: trailing tokens on line '" + line + "'");
            a.block_sizes.push_back(block);
            ++expected;
        }
        if (a.block_sizes.empty()) throw std::runtime_error("read_assignment_file: empty file " + path);
        return a;
    }
    // write_assignment_file (calibrator.cpp:277-283).
    void save(const std::string& path) const {
        std::ofstream out(path, std::ios::trunc);
        if (!out) throw std::runtime_error("write_assignment_file: cannot open " + path);
        for (std::size_t h = 0; h < block_sizes.size(); ++h) out << h << ' ' << block_sizes[h] << '\n';
    }
    std::size_t num_heads() const { return block_sizes.size(); }
    double average_block_size() const {
        if (block_sizes.empty()) return 0.0;
        double s = 0.0;
        for (std::size_t b : block_sizes) s += double(b);
        return s / double(block_sizes.size());
    }
    // BlockAssignment::validate (centroids.cpp:59-76).
    void validate(const EngineConfig& config) const {
        if (block_sizes.size() != config.num_heads)
            throw std::invalid_argument("assignment covers " + std::to_string(block_sizes.size()) +
                                        " heads, config has " + std::to_string(config.num_heads));
        for (std::size_t h = 0; h < block_sizes.size(); ++h) {
            const std::size_t b = block_sizes[h];
            bool cand = false;
            for (std::size_t c : config.candidate_block_sizes) cand |= c == b;
            if (!cand)
                throw std::invalid_argument("head " + std::to_string(h) + ": block size " +
                                            std::to_string(b) + " is not a candidate");
            if (b % config.page_size != 0)
                throw std::invalid_argument("head " + std::to_string(h) + ": block size " +
                                            std::to_string(b) + " is not a multiple of page_size");
        }
    }
};

// build_offsets (centroids.cpp:78-84).
inline std::vector<std::size_t> build_offsets(std::size_t seq_len, const BlockAssignment& a) {
    std::vector<std::size_t> off(a.num_heads() + 1, 0);
    for (std::size_t h = 0; h < a.num_heads(); ++h)
        off[h + 1] = off[h] + (seq_len + a.block_sizes[h] - 1) / a.block_sizes[h];
    return off;
}

// One sequence's device store read back in the reference layouts
// (CentroidStore + QuantizedCentroidStore fields, centroids.hpp:31-52,
// quantizer.hpp:18-38; codes one per byte).
struct StoreSnapshot {
    std::vector<std::size_t> offsets;
    std::vector<float> values, values_min;
    std::vector<uint8_t> codes, codes_min;
    std::vector<float> scales, zero_points, scales_min, zero_points_min;
    std::size_t total_centroids() const { return offsets.empty() ? 0 : offsets.back(); }
};

// Ordered per-(sequence, KV head) selection read back from the device
// (SelectionResult::blocks, engine.hpp:19-26).
struct Selection {
    std::size_t batch = 0, num_heads = 0;
    std::vector<std::vector<std::size_t>> blocks;  // [b * num_heads + h], score-descending
};

// Device-resident decode attention over caller-owned paged KV caches; one
// instance per device per host thread. Every call is
// stream-ordered; only the download_* and *_host calls synchronise.
class DecodeAttention {
  public:
    DecodeAttention(const EngineConfig& config, int device = 0) : config_(config) {
        config_.validate();
        const absp_config c = config_.to_abi();
        check(absp_ctx_create(device, &c, &ctx_));
    }
    ~DecodeAttention() { absp_ctx_destroy(ctx_); }
    DecodeAttention(const DecodeAttention&) = delete;
    DecodeAttention& operator=(const DecodeAttention&) = delete;
    DecodeAttention(DecodeAttention&& o) noexcept : config_(std::move(o.config_)), ctx_(o.ctx_) {
        o.ctx_ = nullptr;
    }

    const EngineConfig& config() const { return config_; }
    absp_ctx* handle() const { return ctx_; }

    void set_assignment(uint32_t layer, const BlockAssignment& a) {
        a.validate(config_);
        std::vector<uint32_t> b(a.block_sizes.begin(), a.block_sizes.end());
        check(absp_set_assignment(ctx_, layer, b.data()));
    }
    // k_pool/v_pool: bf16 [H][pool_pages][P][d] (device); page_table: u32
    // [batch][max_pages] (device); seq_lens: host.
    void bind(uint32_t layer, const void* k_pool, const void* v_pool, uint64_t pool_pages,
              const uint32_t* page_table, uint32_t max_pages, const std::vector<uint32_t>& seq_lens) {
        check(absp_kv_bind(ctx_, layer, k_pool, v_pool, pool_pages, page_table, max_pages,
                           seq_lens.data(), uint32_t(seq_lens.size())));
    }
    void build_store(uint32_t layer, void* stream = nullptr) { check(absp_build_store(ctx_, layer, stream)); }
    // One token per sequence (bf16 [batch][H][d], device) + refresh_tail_centroids +
    // requantize_heads: the maintenance half of DecodeEngine::step (engine.cpp:443-449).
    void append(uint32_t layer, const void* k_new, const void* v_new, void* stream = nullptr) {
        check(absp_append(ctx_, layer, k_new, v_new, stream));
    }
    void select(uint32_t layer, const void* q, uint32_t* blocks, uint32_t stride, uint32_t* counts,
                void* stream = nullptr) {
        check(absp_select(ctx_, layer, q, blocks, stride, counts, stream));
    }
    // validate = true: the reference's check_selection semantics (synchronises the
    // stream; std::invalid_argument / std::out_of_range on a bad selection).
    void attend(uint32_t layer, const void* q, const uint32_t* blocks, uint32_t stride,
                const uint32_t* counts, float* out, void* stream = nullptr, bool validate = true) {
        check(absp_attend(ctx_, layer, q, blocks, stride, counts, out, stream));
        if (validate) check(absp_attend_validate(ctx_, layer, stream));
    }
    uint64_t layout_version(uint32_t layer) const { return absp_layout_version(ctx_, layer); }
    void decode_step(uint32_t layer, const void* q, float* out, void* stream = nullptr) {
        check(absp_decode_step(ctx_, layer, q, out, stream));
    }
    void decode_step_host(uint32_t layer, const uint16_t* q_host, float* out_host, void* stream = nullptr) {
        check(absp_decode_step_host(ctx_, layer, q_host, out_host, stream));
    }
    absp_layer_info layer_info(uint32_t layer) const {
        absp_layer_info i{};
        check(absp_get_layer_info(ctx_, layer, &i));
        return i;
    }
    uint64_t launch_count() const { return absp_launch_count(ctx_); }

    StoreSnapshot download_store(uint32_t layer, uint32_t seq) const {
        const std::size_t H = config_.num_heads, d = config_.head_dim;
        std::vector<uint64_t> off(H + 1);
        check(absp_download_store(ctx_, layer, seq, off.data(), nullptr, nullptr, nullptr, nullptr,
                                  nullptr, nullptr, nullptr, nullptr));
        StoreSnapshot s;
        s.offsets.assign(off.begin(), off.end());
        const std::size_t n = s.total_centroids();
        const bool mm = config_.centroid_method == CentroidMethod::kMaxMin;
        s.values.resize(n * d);
        if (mm) s.values_min.resize(n * d);
        if (config_.quant) {
            s.codes.resize(n * d);
            s.scales.resize(H * d);
            s.zero_points.resize(H * d);
            if (mm) {
                s.codes_min.resize(n * d);
                s.scales_min.resize(H * d);
                s.zero_points_min.resize(H * d);
            }
        }
        auto p = [](auto& v) { return v.empty() ? nullptr : v.data(); };
        check(absp_download_store(ctx_, layer, seq, nullptr, p(s.values), p(s.values_min), p(s.codes),
                                  p(s.codes_min), p(s.scales), p(s.zero_points), p(s.scales_min),
                                  p(s.zero_points_min)));
        return s;
    }
    // The layer's last selection (decode_step / select) per (sequence, KV head).
    Selection download_selection(uint32_t layer) const {
        const uint32_t* b = nullptr;
        const uint32_t* c = nullptr;
        uint32_t stride = 0;
        check(absp_last_selection(ctx_, layer, &b, &stride, &c));
        const absp_layer_info info = layer_info(layer);
        const std::size_t H = config_.num_heads, units = std::size_t(info.batch) * H;
        std::vector<uint32_t> blocks(units * stride), counts(units);
        check(absp_download_selection(ctx_, layer, blocks.data(), counts.data()));
        Selection s;
        s.batch = info.batch;
        s.num_heads = H;
        for (std::size_t u = 0; u < units; ++u)
            s.blocks.emplace_back(blocks.begin() + u * stride, blocks.begin() + u * stride + counts[u]);
        return s;
    }
    // estimate_scores' flattened output for one sequence (engine.hpp:47-49).
    std::vector<float> download_scores(uint32_t layer, uint32_t seq) const {
        std::vector<uint64_t> off(config_.num_heads + 1);
        check(absp_download_store(ctx_, layer, seq, off.data(), nullptr, nullptr, nullptr, nullptr,
                                  nullptr, nullptr, nullptr, nullptr));
        std::vector<float> sc(off.back());
        check(absp_download_scores(ctx_, layer, seq, sc.data()));
        return sc;
    }

  private:
    EngineConfig config_;
    absp_ctx* ctx_ = nullptr;
};

// StepResult (engine.hpp:84-88): the attention output [Hq][d], the ordered selection
// per KV head (SelectionResult::blocks) and whether the reference would have used its
// full-attention fallback (seq_len <= token_budget; every block is then selected).
struct StepResult {
    std::vector<float> output;
    std::vector<std::vector<std::size_t>> blocks;
    bool full_attention_fallback = false;
};

// DecodeEngine (engine.hpp:90-129, engine.cpp:405-463) for one sequence on one GPU:
// owns its paged bf16 KV cache, quantized centroid store and stream (absp_engine_*),
// with the reference's constructor, prefill and step signatures (spans as pointer +
// length) and exceptions. centroids() / quantized() return host snapshots of the device
// store in the reference layouts (CentroidStore / QuantizedCentroidStore).
class DecodeEngine {
  public:
    DecodeEngine(const EngineConfig& config, const BlockAssignment& assignment, std::size_t capacity_tokens,
                 int device = 0)
        : config_(config), assignment_(assignment) {
        config_.validate();
        assignment_.validate(config_);
        const absp_config c = config_.to_abi();
        std::vector<uint32_t> b(assignment_.block_sizes.begin(), assignment_.block_sizes.end());
        check(absp_engine_create(device, &c, b.data(), capacity_tokens, &eng_));
        absp_ctx* ctx = nullptr;
        check(absp_engine_info(eng_, nullptr, &stride_, &ctx));
    }
    ~DecodeEngine() { absp_engine_destroy(eng_); }
    DecodeEngine(const DecodeEngine&) = delete;
    DecodeEngine& operator=(const DecodeEngine&) = delete;

    // keys / values head-major [head][token][channel] (engine.hpp:102-105)
    void prefill(const float* keys, std::size_t keys_len, const float* values, std::size_t values_len,
                 std::size_t num_tokens) {
        check(absp_engine_prefill(eng_, keys, keys_len, values, values_len, num_tokens));
    }
    void prefill(const std::vector<float>& keys, const std::vector<float>& values, std::size_t num_tokens) {
        prefill(keys.data(), keys.size(), values.data(), values.size(), num_tokens);
    }
    // keys / values: num_heads * head_dim floats; query: num_q_heads * head_dim floats
    StepResult step(const float* keys, std::size_t keys_len, const float* values, std::size_t values_len,
                    const float* query, std::size_t query_len) {
        const std::size_t H = config_.num_heads;
        const std::size_t Hq = config_.num_q_heads ? config_.num_q_heads : H;
        StepResult r;
        r.output.resize(Hq * config_.head_dim);
        std::vector<uint32_t> blocks(H * stride_), counts(H);
        int fb = 0;
        check(absp_engine_step(eng_, keys, keys_len, values, values_len, query, query_len, r.output.data(),
                               blocks.data(), stride_, counts.data(), &fb));
        r.blocks.resize(H);
        for (std::size_t h = 0; h < H; ++h)
            r.blocks[h].assign(blocks.begin() + h * stride_, blocks.begin() + h * stride_ + counts[h]);
        r.full_attention_fallback = fb != 0;
        return r;
    }
    StepResult step(const std::vector<float>& keys, const std::vector<float>& values,
                    const std::vector<float>& query) {
        return step(keys.data(), keys.size(), values.data(), values.size(), query.data(), query.size());
    }

    const EngineConfig& config() const { return config_; }
    const BlockAssignment& assignment() const { return assignment_; }
    std::size_t seq_len() const {
        uint64_t n = 0;
        check(absp_engine_info(eng_, &n, nullptr, nullptr));
        return std::size_t(n);
    }
    // CentroidStore (+ QuantizedCentroidStore when quantized) of the sequence.
    StoreSnapshot centroids() const { return snapshot(); }
    std::optional<StoreSnapshot> quantized() const {
        if (!config_.quant) return std::nullopt;
        return snapshot();
    }
    absp_engine* handle() const { return eng_; }

  private:
    StoreSnapshot snapshot() const {
        absp_ctx* ctx = nullptr;
        check(absp_engine_info(eng_, nullptr, nullptr, &ctx));
        const std::size_t H = config_.num_heads, d = config_.head_dim;
        std::vector<uint64_t> off(H + 1);
        check(absp_download_store(ctx, 0, 0, off.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                  nullptr, nullptr));
        StoreSnapshot s;
        s.offsets.assign(off.begin(), off.end());
        const std::size_t n = s.total_centroids();
        const bool mm = config_.centroid_method == CentroidMethod::kMaxMin;
        s.values.resize(n * d);
        if (mm) s.values_min.resize(n * d);
        if (config_.quant) {
            s.codes.resize(n * d);
            s.scales.resize(H * d);
            s.zero_points.resize(H * d);
            if (mm) {
                s.codes_min.resize(n * d);
                s.scales_min.resize(H * d);
                s.zero_points_min.resize(H * d);
            }
        }
        auto p = [](auto& v) { return v.empty() ? nullptr : v.data(); };
        check(absp_download_store(ctx, 0, 0, nullptr, p(s.values), p(s.values_min), p(s.codes), p(s.codes_min),
                                  p(s.scales), p(s.zero_points), p(s.scales_min), p(s.zero_points_min)));
        return s;
    }

    EngineConfig config_;
    BlockAssignment assignment_;
    absp_engine* eng_ = nullptr;
    uint32_t stride_ = 0;
};

}  // namespace absp

#endif  // ABSP_HPP
