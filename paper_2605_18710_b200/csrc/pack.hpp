// pack.hpp — device packing of candidate-option tables (pack.cu).
#pragma once
#include <vector>

namespace mg {

constexpr int PACK_MAXD = 16;  // d grid values per surface
constexpr int PACK_MAXA = 64;  // a grid values per surface

struct PackInput {  // one module's surface grid, axes ascending, grid[di * na + ai]
    std::vector<double> dv, av, lat, bw, mem;
    double membase = 0.0;
};

struct PackedRow {  // CandidateOption (stage_eval.hpp:58-63)
    int d, u;
    double base, B, fp;
};

// candidate_options for every module, computed by k_pack_options.  range_err[m] = 1 when
// module m's surface cannot answer the d = 1 lookup (the reference's SurfaceRangeError).
std::vector<std::vector<PackedRow>> pack_options_device(const std::vector<PackInput>& mods, int G,
                                                        int L, double cap, int device,
                                                        long long* h2d_bytes,
                                                        std::vector<int>* range_err);

}  // namespace mg
