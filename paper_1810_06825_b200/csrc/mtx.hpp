// Matrix Market coordinate I/O (mtx.cpp), plain C++ shared by the CUDA units.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace fb {

struct MtxData {
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> r, c;  // 0-based, symmetric storage expanded, file order
    std::vector<double> v;
};
// load_matrix_market's parse (matrix_market.hpp:27-93), up to from_triplets
void mtx_read(const std::string& path, MtxData& out);
// write_matrix_market (matrix_market.hpp:95-116)
void mtx_write(const std::string& path, int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci,
               const double* v);

}  // namespace fb
