// Host 1D numerics shared by the C ABI (see tables.cpp for reference citations).
#pragma once
#include <vector>

namespace sphp {
void make_rule(int q, int ptype, std::vector<double>& z, std::vector<double>& w);
void diff_matrix(const std::vector<double>& z, std::vector<double>& D);
void basis_table(int btype, int m, const std::vector<double>& z, std::vector<double>& B,
                 std::vector<double>& Bd);
void modified_b_table(int Pa, int Pb, const std::vector<double>& z, std::vector<double>& B,
                      std::vector<double>& Bd, std::vector<int>& pidx, std::vector<int>& bstart);
}  // namespace sphp
