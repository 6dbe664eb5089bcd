// lyndon.h -- host-side Lyndon tables for the logsignature bases (see lyndon.cpp).
#pragma once
#include <cstdint>
#include <functional>
#include <vector>

namespace sigb200 {

struct LyndonTables {
    int C = 0, N = 0;
    std::vector<int64_t> flat_index;  // [w] offset of each Lyndon word in the flat S layout
    std::vector<int> level;           // [w] its length
    std::vector<int> level_begin;     // [N+2] first Lyndon word of each length (1-based)
    // exact integer inverse of psi o phi (block diagonal by degree), CSR over all w rows
    std::vector<int> minv_rowptr, minv_col;
    std::vector<double> minv_val;
    std::vector<int> minvT_rowptr, minvT_col;  // its transpose
    std::vector<double> minvT_val;
};

LyndonTables build_lyndon_tables(int C, int N, bool need_brackets);
int64_t witt_dimension(int64_t C, int N);

}  // namespace sigb200
