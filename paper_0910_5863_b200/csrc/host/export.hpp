// Host exports of the reference's auxiliary operators (export.cpp).
#pragma once

#include <string>
#include <tuple>
#include <vector>

#include "host.hpp"

namespace b200 {

struct CsrMatrix {  // general CSR, int64 indices
  i64 rows = 0, cols = 0;
  std::vector<i64> ptr, idx;
  std::vector<double> val;
};

/// K = sum_s R^cT T_s^T A_s T_s R^c, full symmetric (bddc_operator.cpp:7-23).
CsrMatrix transformed_operator(const Model& m, const ChangeOfVariables& cov);
/// Pi K Pi + t (I - Pi), symmetrized and pruned (bddc_operator.cpp:25-36);
/// t <= 0 uses max diag K, written to *t_used.
CsrMatrix stabilized_operator(const Model& m, const ChangeOfVariables& cov, double t, double* t_used);
/// The t the reference's BddcPreconditioner would use (stabilization_t()).
double stabilization_t(const Model& m, const ChangeOfVariables& cov, double t);
/// D^c: one row (e_anchor - e_member) per non-anchor group member (transform.cpp:151-164).
CsrMatrix transformed_constraint_matrix(const ChangeOfVariables& cov, i64 wc_dim);
/// matrix_market.cpp:12-38 (symmetric: lower triangle, column-major order).
void write_matrix_market(const std::string& path, const CsrMatrix& a, bool symmetric);

}  // namespace b200
