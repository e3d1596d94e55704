/*
 * absp_calib.hpp — header-only C++ host layer for trace replay and calibration over the
 * C ABI (absp.h), in the shape of the reference's calibrator.hpp / workload.hpp:
 *
 *   absp::Trace, save_trace, load_trace          <- workload.hpp:36-75, workload.cpp:260-309
 *                                                   (binary "ABSP" format, bit-exact)
 *   absp::RecallTable, CalibrationReport,        <- calibrator.hpp:15-44
 *     TransferReport, TraceProvider
 *   absp::profile_sensitivity                    <- calibrator.cpp:73-114 (per sample on the GPU:
 *                                                   absp_profile_sample)
 *   absp::assign_block_sizes, normalized_recall, <- calibrator.cpp:116-157
 *     make_report
 *   absp::transfer_check                         <- calibrator.cpp:159-224 (per sample on the GPU)
 *   absp::topk_page_recall(_per_head)            <- calibrator.cpp:226-249
 *   absp::write_recall_csv, write_min_block_csv  <- calibrator.cpp:253-275
 *
 * The loops over samples and the Eq.-2 assignment rule are host code, as in the
 * reference; each sample's dense fp64 oracle, stores, selections and recall sums run
 * in libabsp.so. Errors follow the reference's exception classes.
 */
#ifndef ABSP_CALIB_HPP
#define ABSP_CALIB_HPP

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <set>

#include "absp.hpp"

namespace absp {

// ---------------------------------------------------------------------------
// Trace I/O
// ---------------------------------------------------------------------------
struct Trace {
    std::uint32_t version = 1;
    std::size_t num_heads = 0;
    std::size_t head_dim = 0;
    std::size_t seq_len = 0;
    std::uint64_t seed = 0;
    std::vector<float> keys;     // num_heads * seq_len * head_dim
    std::vector<float> values;   // num_heads * seq_len * head_dim
    std::vector<float> queries;  // num_heads * head_dim
};

namespace detail {
inline void put_le(std::ofstream& out, std::uint64_t v, int bytes) {
    unsigned char b[8];
    for (int i = 0; i < bytes; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    out.write(reinterpret_cast<const char*>(b), bytes);
}
inline std::uint64_t get_le(std::ifstream& in, int bytes, const char* section) {
    unsigned char b[8];
    in.read(reinterpret_cast<char*>(b), bytes);
    if (in.gcount() != bytes)
        throw std::runtime_error(std::string("load_trace: truncated file in section '") + section + "'");
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= std::uint64_t(b[i]) << (8 * i);
    return v;
}
inline void put_f32s(std::ofstream& out, const std::vector<float>& a) {
    for (float f : a) {
        std::uint32_t u;
        std::memcpy(&u, &f, 4);
        put_le(out, u, 4);
    }
}
inline void get_f32s(std::ifstream& in, std::vector<float>& a, std::size_t n, const char* section) {
    a.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        const std::uint32_t u = std::uint32_t(get_le(in, 4, section));
        std::memcpy(&a[i], &u, 4);
    }
}
}  // namespace detail

// magic "ABSP" | u32 version | u32 num_heads | u32 head_dim | u64 seq_len | u64 seed |
// keys | values | queries, little-endian
inline void save_trace(const Trace& t, const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("save_trace: cannot open " + path);
    out.write("ABSP", 4);
    detail::put_le(out, t.version, 4);
    detail::put_le(out, t.num_heads, 4);
    detail::put_le(out, t.head_dim, 4);
    detail::put_le(out, t.seq_len, 8);
    detail::put_le(out, t.seed, 8);
    detail::put_f32s(out, t.keys);
    detail::put_f32s(out, t.values);
    detail::put_f32s(out, t.queries);
    if (!out) throw std::runtime_error("save_trace: write failed for " + path);
}

inline Trace load_trace(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("load_trace: cannot open " + path);
    char magic[4];
    in.read(magic, 4);
    if (in.gcount() != 4) throw std::runtime_error("load_trace: truncated file in section 'header'");
    if (std::memcmp(magic, "ABSP", 4) != 0) throw std::runtime_error("load_trace: format error, bad magic bytes");
    Trace t;
    t.version = std::uint32_t(detail::get_le(in, 4, "header"));
    if (t.version != 1)
        throw std::runtime_error("load_trace: version mismatch (file " + std::to_string(t.version) +
                                 ", expected 1)");
    t.num_heads = detail::get_le(in, 4, "header");
    t.head_dim = detail::get_le(in, 4, "header");
    t.seq_len = detail::get_le(in, 8, "header");
    t.seed = detail::get_le(in, 8, "header");
    if (t.num_heads == 0 || t.head_dim == 0 || t.seq_len == 0)
        throw std::runtime_error("load_trace: dimension inconsistency in header");
    const std::size_t per = t.num_heads * t.seq_len * t.head_dim;
    detail::get_f32s(in, t.keys, per, "keys");
    detail::get_f32s(in, t.values, per, "values");
    detail::get_f32s(in, t.queries, t.num_heads * t.head_dim, "queries");
    in.peek();
    if (!in.eof()) throw std::runtime_error("load_trace: trailing bytes after queries section");
    return t;
}

// ---------------------------------------------------------------------------
// Calibration
// ---------------------------------------------------------------------------
struct RecallTable {
    std::size_t num_heads = 0;
    std::vector<std::size_t> candidates;
    std::vector<double> recalls;  // num_heads x candidates, row-major
    std::size_t sample_count = 0;
    double at(std::size_t h, std::size_t ci) const { return recalls[h * candidates.size() + ci]; }
    double& at(std::size_t h, std::size_t ci) { return recalls[h * candidates.size() + ci]; }
};

struct CalibrationReport {
    BlockAssignment assignment;
    RecallTable normalized_recalls;
    std::vector<std::size_t> min_block_sizes;
    double avg_block_size = 0.0;
};

struct TransferReport {
    double adaptive_recall = 0.0;
    std::vector<std::size_t> candidates;
    std::vector<double> uniform_recalls;
    double avg_block_size = 0.0;
    std::size_t matched_candidate = 0;
    double delta = 0.0;
};

using TraceProvider = std::function<Trace(std::size_t)>;

namespace detail {
inline void check_trace_dims(const Trace& t, const EngineConfig& c, std::size_t i) {
    if (t.num_heads != c.num_heads || t.head_dim != c.head_dim)
        throw std::invalid_argument("calibration sample " + std::to_string(i) +
                                    ": trace dimensions do not match the config");
}
// One sample on the GPU: recalls [H][candidates] (+ the assignment's per-head recall).
inline void profile_sample(const Trace& t, const EngineConfig& config, const BlockAssignment* a, int device,
                           std::vector<double>& rec, std::vector<double>* arec) {
    absp_config c = config.to_abi();
    c.num_q_heads = uint32_t(t.num_heads);
    if (t.keys.size() != t.num_heads * t.seq_len * t.head_dim || t.values.size() != t.keys.size() ||
        t.queries.size() != t.num_heads * t.head_dim)
        throw std::invalid_argument("profile_sample: trace tensor sizes do not match its header");
    rec.assign(t.num_heads * config.candidate_block_sizes.size(), 0.0);
    std::vector<uint32_t> bs;
    if (a) {
        for (std::size_t b : a->block_sizes) bs.push_back(uint32_t(b));
        arec->assign(t.num_heads, 0.0);
    }
    check(absp_profile_sample(device, &c, t.keys.data(), t.values.data(), t.queries.data(), t.seq_len,
                              a ? bs.data() : nullptr, rec.data(), a ? arec->data() : nullptr));
}
}  // namespace detail

inline RecallTable profile_sensitivity(const TraceProvider& provider, std::size_t sample_count,
                                       const EngineConfig& config, int device = 0) {
    config.validate();
    if (sample_count == 0) throw std::invalid_argument("profile_sensitivity: need at least one calibration sample");
    RecallTable table;
    table.num_heads = config.num_heads;
    table.candidates = config.candidate_block_sizes;
    table.recalls.assign(config.num_heads * table.candidates.size(), 0.0);
    std::size_t used = 0;
    std::vector<double> rec;
    for (std::size_t i = 0; i < sample_count; ++i) {
        const Trace t = provider(i);
        detail::check_trace_dims(t, config, i);
        if (t.seq_len <= config.token_budget) {
            std::cerr << "profile_sensitivity: skipping sample " << i << " (seq_len " << t.seq_len
                      << " <= budget " << config.token_budget << ", recall is trivially 1)\n";
            continue;
        }
        detail::profile_sample(t, config, nullptr, device, rec, nullptr);
        for (std::size_t k = 0; k < rec.size(); ++k) table.recalls[k] += rec[k];
        ++used;
    }
    if (used == 0)
        throw std::runtime_error("profile_sensitivity: no usable samples (every seq_len <= token_budget)");
    for (double& r : table.recalls) r /= double(used);
    table.sample_count = used;
    return table;
}

inline BlockAssignment assign_block_sizes(const RecallTable& table, double tau) {
    if (table.candidates.empty() || table.num_heads == 0)
        throw std::invalid_argument("assign_block_sizes: empty recall table");
    if (!std::is_sorted(table.candidates.begin(), table.candidates.end()))
        throw std::invalid_argument("assign_block_sizes: candidates must be ascending");
    BlockAssignment a;
    for (std::size_t h = 0; h < table.num_heads; ++h) {
        const double peak = table.at(h, 0);
        if (peak <= 0.0)
            throw std::invalid_argument("assign_block_sizes: head " + std::to_string(h) +
                                        " has zero recall at the minimum block size");
        std::size_t best = table.candidates[0];
        for (std::size_t ci = 0; ci < table.candidates.size(); ++ci)
            if (table.at(h, ci) >= tau * peak) best = std::max(best, table.candidates[ci]);
        a.block_sizes.push_back(best);
    }
    return a;
}

inline RecallTable normalized_recall(const RecallTable& table) {
    RecallTable out = table;
    for (std::size_t h = 0; h < table.num_heads; ++h) {
        const double peak = table.at(h, 0);
        if (peak <= 0.0) throw std::invalid_argument("normalized_recall: zero recall at the minimum block size");
        for (std::size_t ci = 0; ci < table.candidates.size(); ++ci) out.at(h, ci) = table.at(h, ci) / peak;
    }
    return out;
}

inline CalibrationReport make_report(const RecallTable& table, double tau) {
    CalibrationReport r;
    r.assignment = assign_block_sizes(table, tau);
    r.normalized_recalls = normalized_recall(table);
    r.min_block_sizes = r.assignment.block_sizes;
    r.avg_block_size = r.assignment.average_block_size();
    return r;
}

inline TransferReport transfer_check(const BlockAssignment& assignment, const TraceProvider& holdout,
                                     std::size_t sample_count, const EngineConfig& config, int device = 0) {
    config.validate();
    assignment.validate(config);
    TransferReport r;
    r.candidates = config.candidate_block_sizes;
    r.uniform_recalls.assign(r.candidates.size(), 0.0);
    r.avg_block_size = assignment.average_block_size();
    const std::size_t H = config.num_heads, nc = r.candidates.size();
    std::size_t used = 0;
    std::vector<double> rec, arec;
    for (std::size_t i = 0; i < sample_count; ++i) {
        const Trace t = holdout(i);
        detail::check_trace_dims(t, config, i);
        if (t.seq_len <= config.token_budget) {
            std::cerr << "transfer_check: skipping sample " << i << " (seq_len <= budget)\n";
            continue;
        }
        detail::profile_sample(t, config, &assignment, device, rec, &arec);
        for (double x : arec) r.adaptive_recall += x / double(H);
        for (std::size_t ci = 0; ci < nc; ++ci)
            for (std::size_t h = 0; h < H; ++h) r.uniform_recalls[ci] += rec[h * nc + ci] / double(H);
        ++used;
    }
    if (used == 0) throw std::runtime_error("transfer_check: no usable holdout samples");
    r.adaptive_recall /= double(used);
    for (double& x : r.uniform_recalls) x /= double(used);
    std::size_t best = 0;
    double gap = std::abs(double(r.candidates[0]) - r.avg_block_size);
    for (std::size_t ci = 1; ci < nc; ++ci) {
        const double g = std::abs(double(r.candidates[ci]) - r.avg_block_size);
        if (g <= gap) {  // ties go coarser
            gap = g;
            best = ci;
        }
    }
    r.matched_candidate = r.candidates[best];
    r.delta = r.adaptive_recall - r.uniform_recalls[best];
    return r;
}

inline std::vector<double> topk_page_recall_per_head(const std::vector<std::vector<std::size_t>>& selected,
                                                     const std::vector<std::vector<std::size_t>>& reference) {
    if (selected.size() != reference.size()) throw std::invalid_argument("topk_page_recall: head count mismatch");
    std::vector<double> out;
    for (std::size_t h = 0; h < selected.size(); ++h) {
        const std::set<std::size_t> ref(reference[h].begin(), reference[h].end());
        if (ref.empty()) throw std::invalid_argument("topk_page_recall: empty reference selection");
        std::size_t hit = 0;
        for (std::size_t b : selected[h]) hit += ref.count(b);
        out.push_back(double(hit) / double(ref.size()));
    }
    return out;
}

inline double topk_page_recall(const std::vector<std::vector<std::size_t>>& selected,
                               const std::vector<std::vector<std::size_t>>& reference) {
    const std::vector<double> per = topk_page_recall_per_head(selected, reference);
    double acc = 0.0;
    for (double r : per) acc += r;
    return acc / double(per.size());
}

// CSV reports (calibrator.cpp:253-275): numbers as printf("%.10g").
inline void write_recall_csv(const std::string& path, const RecallTable& table, const std::string& layer_tag) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw std::runtime_error("write_recall_csv: cannot open " + path);
    out << "head,layer,block_size,recall\n";
    char buf[64];
    for (std::size_t h = 0; h < table.num_heads; ++h)
        for (std::size_t ci = 0; ci < table.candidates.size(); ++ci) {
            std::snprintf(buf, sizeof(buf), "%.10g", table.at(h, ci));
            out << h << ',' << layer_tag << ',' << table.candidates[ci] << ',' << buf << '\n';
        }
}

inline void write_min_block_csv(const std::string& path, const std::vector<std::size_t>& min_block_sizes,
                                const std::string& layer_tag) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw std::runtime_error("write_min_block_csv: cannot open " + path);
    out << "head,layer,min_block_size\n";
    for (std::size_t h = 0; h < min_block_sizes.size(); ++h) out << h << ',' << layer_tag << ',' << min_block_sizes[h] << '\n';
}

}  // namespace absp

#endif  // ABSP_CALIB_HPP
