// Reference-style call site of the C++ calibration / trace host layer (include/absp_calib.hpp),
// driven by tests/test_cpp_host.py:
//   roundtrip <in> <out>   load_trace(in) -> save_trace(out)              (CPU)
//   load <file>            load_trace; prints the exception message       (CPU)
//   calib <dir> S H d P T tau c1 [c2 ...]                                 (GPU)
//       profile_sensitivity over <dir>/s<i>.absp, then assign_block_sizes(tau) and
//       transfer_check of that assignment; prints every number with 17 digits.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "absp_calib.hpp"

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string mode = argv[1];
    try {
        if (mode == "roundtrip" && argc == 4) {
            absp::save_trace(absp::load_trace(argv[2]), argv[3]);
            std::printf("OK roundtrip\n");
            return 0;
        }
        if (mode == "load" && argc == 3) {
            const absp::Trace t = absp::load_trace(argv[2]);
            std::printf("loaded %zu %zu %zu\n", t.num_heads, t.head_dim, t.seq_len);
            return 0;
        }
        if (mode == "calib" && argc >= 10) {
            const std::string dir = argv[2];
            const std::size_t S = std::strtoul(argv[3], nullptr, 10);
            absp::EngineConfig c;
            c.num_heads = std::strtoul(argv[4], nullptr, 10);
            c.head_dim = std::strtoul(argv[5], nullptr, 10);
            c.page_size = std::strtoul(argv[6], nullptr, 10);
            c.token_budget = std::strtoul(argv[7], nullptr, 10);
            const double tau = std::strtod(argv[8], nullptr);
            c.candidate_block_sizes.clear();
            for (int i = 9; i < argc; ++i) c.candidate_block_sizes.push_back(std::strtoul(argv[i], nullptr, 10));
            c.quant = absp::QuantSpec{};
            auto provider = [&](std::size_t i) { return absp::load_trace(dir + "/s" + std::to_string(i) + ".absp"); };
            const absp::RecallTable t = absp::profile_sensitivity(provider, S, c);
            std::printf("recalls");
            for (double r : t.recalls) std::printf(" %.17g", r);
            std::printf("\n");
            const absp::BlockAssignment a = absp::assign_block_sizes(t, tau);
            std::printf("assignment");
            for (std::size_t b : a.block_sizes) std::printf(" %zu", b);
            std::printf("\n");
            const absp::TransferReport r = absp::transfer_check(a, provider, S, c);
            std::printf("transfer %.17g %.17g %.17g %zu", r.adaptive_recall, r.delta, r.avg_block_size,
                        r.matched_candidate);
            for (double u : r.uniform_recalls) std::printf(" %.17g", u);
            std::printf("\nOK calib\n");
            return 0;
        }
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 0;
    }
    return 2;
}
