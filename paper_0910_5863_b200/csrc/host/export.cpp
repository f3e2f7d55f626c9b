// Host-side exports of the reference's auxiliary operators (debugging dumps
// and the BddcPreconditioner accessors), not on the device path:
//   assemble_transformed_operator  bddc_operator.cpp:7-23
//   stabilize                      bddc_operator.cpp:25-36
//   transformed_constraint_matrix  transform.cpp:151-164
//   write_matrix_market[_symmetric] matrix_market.cpp:12-38
// The device path never forms these matrices: it factors the exact primal
// reformulation, so they exist for the reference's
// `stabilized()` accessor and its `export_directory` dumps (experiment.cpp:172-178).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <tuple>

#include "export.hpp"

namespace b200 {

namespace {
// B_s = cov.basis[s] (transform.cpp:94-149) as sparse columns: identity except the
// dense glob blocks t (B(local[a], local[b]) = t[a][b]).
struct SparseCols {
  std::vector<std::vector<std::pair<int, double>>> col;  // col[j] = {(row, value)}
};

SparseCols basis_of(const Model& m, const ChangeOfVariables& cov, int s) {
  const int dim = m.subs[s].dim();
  SparseCols b;
  b.col.resize(dim);
  std::vector<char> covered(dim, 0);
  for (const GlobTransform& gt : cov.transforms) {
    const Glob& g = m.globs[gt.glob];
    if (!std::binary_search(g.subdomains.begin(), g.subdomains.end(), s)) continue;
    const auto& dofs = m.glob_dofs[gt.glob];
    const int n = gt.n;
    std::vector<int> local(n);
    for (int a = 0; a < n; ++a) local[a] = m.maps.local_of(dofs[a], s);
    const std::vector<double> t = gt.dense_t();
    for (int bcol = 0; bcol < n; ++bcol) {
      covered[local[bcol]] = 1;
      for (int a = 0; a < n; ++a)
        if (t[std::size_t(a) * n + bcol] != 0.0) b.col[local[bcol]].emplace_back(local[a], t[std::size_t(a) * n + bcol]);
    }
  }
  for (int j = 0; j < dim; ++j)
    if (!covered[j]) b.col[j].emplace_back(j, 1.0);
  return b;
}

CsrMatrix from_triplets(i64 rows, i64 cols, std::vector<std::tuple<i64, i64, double>>& trip) {
  std::sort(trip.begin(), trip.end(), [](const auto& x, const auto& y) {
    return std::get<0>(x) != std::get<0>(y) ? std::get<0>(x) < std::get<0>(y) : std::get<1>(x) < std::get<1>(y);
  });
  CsrMatrix a;
  a.rows = rows;
  a.cols = cols;
  a.ptr.assign(rows + 1, 0);
  for (std::size_t k = 0; k < trip.size();) {
    const i64 r = std::get<0>(trip[k]), c = std::get<1>(trip[k]);
    double v = 0.0;
    for (; k < trip.size() && std::get<0>(trip[k]) == r && std::get<1>(trip[k]) == c; ++k) v += std::get<2>(trip[k]);
    a.idx.push_back(c);
    a.val.push_back(v);
    a.ptr[r + 1]++;
  }
  for (i64 r = 0; r < rows; ++r) a.ptr[r + 1] += a.ptr[r];
  return a;
}
}  // namespace

CsrMatrix transformed_operator(const Model& m, const ChangeOfVariables& cov) {
  // upper triangle summed over substructures, then mirrored (SparseSymMatrix)
  std::vector<std::tuple<i64, i64, double>> trip;
  for (int s = 0; s < static_cast<int>(m.subs.size()); ++s) {
    const CSR& A = m.matrix(s);
    const SparseCols B = basis_of(m, cov, s);
    const int dim = A.n;
    const auto& to_wc = m.maps.local_to_wc[s];
    // C = A B column by column, then K_s = B^T C through the rows of B
    std::vector<std::vector<std::pair<int, double>>> brow(dim);
    for (int l = 0; l < dim; ++l)
      for (const auto& [i, bil] : B.col[l]) brow[i].emplace_back(l, bil);
    std::vector<double> acc(dim, 0.0), out(dim, 0.0);
    std::vector<char> mark(dim, 0), omark(dim, 0);
    std::vector<int> touched, otouched;
    for (int j = 0; j < dim; ++j) {
      touched.clear();
      otouched.clear();
      for (const auto& [k, bkj] : B.col[j])
        for (int e = A.ptr[k]; e < A.ptr[k + 1]; ++e) {
          const int i = A.idx[e];
          if (!mark[i]) {
            mark[i] = 1;
            touched.push_back(i);
          }
          acc[i] += A.val[e] * bkj;
        }
      std::sort(touched.begin(), touched.end());
      for (int i : touched)
        for (const auto& [l, bil] : brow[i]) {
          if (!omark[l]) {
            omark[l] = 1;
            otouched.push_back(l);
          }
          out[l] += bil * acc[i];
        }
      for (int l : otouched) {
        const i64 r = to_wc[l], c = to_wc[j];
        if (r <= c) trip.emplace_back(r, c, out[l]);
        out[l] = 0.0;
        omark[l] = 0;
      }
      for (int i : touched) {
        acc[i] = 0.0;
        mark[i] = 0;
      }
    }
  }
  CsrMatrix upper = from_triplets(m.maps.wc_dim, m.maps.wc_dim, trip);
  std::vector<std::tuple<i64, i64, double>> full;
  full.reserve(2 * upper.val.size());
  for (i64 r = 0; r < upper.rows; ++r)
    for (i64 e = upper.ptr[r]; e < upper.ptr[r + 1]; ++e) {
      full.emplace_back(r, upper.idx[e], upper.val[e]);
      if (upper.idx[e] != r) full.emplace_back(upper.idx[e], r, upper.val[e]);
    }
  return from_triplets(upper.rows, upper.cols, full);
}

CsrMatrix stabilized_operator(const Model& m, const ChangeOfVariables& cov, double t, double* t_used) {
  const CsrMatrix k = transformed_operator(m, cov);
  const i64 n = k.rows;
  if (t <= 0) {
    t = 0.0;
    bool first = true;
    for (i64 r = 0; r < n; ++r)
      for (i64 e = k.ptr[r]; e < k.ptr[r + 1]; ++e)
        if (k.idx[e] == r && (first || k.val[e] > t)) {
          t = k.val[e];
          first = false;
        }
  }
  if (t_used) *t_used = t;
  // Pi: group members -> group mean (GroupProjector, transform.cpp:12-46)
  std::vector<int> grp(n, -1);
  for (std::size_t g = 0; g < cov.groups.size(); ++g)
    for (i64 w : cov.groups[g]) grp[w] = static_cast<int>(g);
  auto members = [&](i64 i, auto f) {
    if (grp[i] < 0) return f(i, 1.0);
    const auto& G = cov.groups[grp[i]];
    for (i64 w : G) f(w, 1.0 / G.size());
  };
  std::vector<std::tuple<i64, i64, double>> trip;
  for (i64 kr = 0; kr < n; ++kr)
    for (i64 e = k.ptr[kr]; e < k.ptr[kr + 1]; ++e) {
      const i64 kc = k.idx[e];
      const double v = k.val[e];
      members(kr, [&](i64 i, double pik) {
        members(kc, [&](i64 j, double plj) { trip.emplace_back(i, j, pik * v * plj); });
      });
    }
  for (const auto& G : cov.groups)  // t (I - Pi) on each group block
    for (i64 a : G)
      for (i64 b : G) trip.emplace_back(a, b, t * ((a == b ? 1.0 : 0.0) - 1.0 / G.size()));
  for (i64 i = 0; i < n; ++i)
    if (grp[i] < 0) trip.emplace_back(i, i, 0.0);  // t (I - Pi) is zero off the groups
  CsrMatrix mat = from_triplets(n, n, trip);
  // symmetrize 0.5 (M^T + M), then prune |v| <= 1e-12 max|v| (sparse.cpp:98-108)
  std::vector<std::tuple<i64, i64, double>> sym;
  sym.reserve(2 * mat.val.size());
  for (i64 r = 0; r < n; ++r)
    for (i64 e = mat.ptr[r]; e < mat.ptr[r + 1]; ++e) {
      sym.emplace_back(r, mat.idx[e], 0.5 * mat.val[e]);
      sym.emplace_back(mat.idx[e], r, 0.5 * mat.val[e]);
    }
  CsrMatrix s = from_triplets(n, n, sym);
  double amax = 0.0;
  for (double v : s.val) amax = std::max(amax, std::fabs(v));
  const double cut = 1e-12 * (amax > 0 ? amax : 1.0);
  CsrMatrix out;
  out.rows = out.cols = n;
  out.ptr.assign(n + 1, 0);
  for (i64 r = 0; r < n; ++r) {
    for (i64 e = s.ptr[r]; e < s.ptr[r + 1]; ++e)
      if (std::fabs(s.val[e]) > cut) {
        out.idx.push_back(s.idx[e]);
        out.val.push_back(s.val[e]);
      }
    out.ptr[r + 1] = static_cast<i64>(out.idx.size());
  }
  return out;
}

double stabilization_t(const Model& m, const ChangeOfVariables& cov, double t) {
  if (t > 0) return t;
  // max diagonal of K: (B^T A B)_{ll} summed over the copies of each W^c id
  std::vector<double> diag(m.maps.wc_dim, 0.0);
  for (int s = 0; s < static_cast<int>(m.subs.size()); ++s) {
    const CSR& A = m.matrix(s);
    const SparseCols B = basis_of(m, cov, s);
    for (int l = 0; l < A.n; ++l) {
      double v = 0.0;
      for (const auto& [i, bil] : B.col[l])
        for (const auto& [k, bkl] : B.col[l]) {
          double aik = 0.0;
          for (int e = A.ptr[i]; e < A.ptr[i + 1]; ++e)
            if (A.idx[e] == k) aik = A.val[e];
          v += bil * aik * bkl;
        }
      diag[m.maps.local_to_wc[s][l]] += v;
    }
  }
  return diag.empty() ? 0.0 : *std::max_element(diag.begin(), diag.end());
}

CsrMatrix transformed_constraint_matrix(const ChangeOfVariables& cov, i64 wc_dim) {
  std::vector<std::tuple<i64, i64, double>> trip;
  i64 row = 0;
  for (const auto& g : cov.groups)
    for (std::size_t i = 1; i < g.size(); ++i) {
      trip.emplace_back(row, g.front(), 1.0);
      trip.emplace_back(row, g[i], -1.0);
      ++row;
    }
  return from_triplets(row, wc_dim, trip);
}

void write_matrix_market(const std::string& path, const CsrMatrix& a, bool symmetric) {
  FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw Error(kError, "cannot open " + path);
  // Eigen iterates column-major; for the symmetric (lower) dump the entries of
  // column c are the rows r >= c, i.e. row c's upper part of the symmetric CSR.
  i64 nnz = 0;
  if (symmetric) {
    for (i64 r = 0; r < a.rows; ++r)
      for (i64 e = a.ptr[r]; e < a.ptr[r + 1]; ++e)
        if (a.idx[e] >= r) ++nnz;
  } else {
    nnz = static_cast<i64>(a.val.size());
  }
  std::fprintf(f, "%%%%MatrixMarket matrix coordinate real %s\n", symmetric ? "symmetric" : "general");
  std::fprintf(f, "%lld %lld %lld\n", (long long)a.rows, (long long)a.cols, (long long)nnz);
  if (symmetric) {
    for (i64 c = 0; c < a.rows; ++c)  // column c of the lower triangle = row c, columns >= c
      for (i64 e = a.ptr[c]; e < a.ptr[c + 1]; ++e)
        if (a.idx[e] >= c) std::fprintf(f, "%lld %lld %.17g\n", (long long)a.idx[e] + 1, (long long)c + 1, a.val[e]);
  } else {
    // column-major order like Eigen's default storage
    std::vector<std::vector<std::pair<i64, double>>> cols(a.cols);
    for (i64 r = 0; r < a.rows; ++r)
      for (i64 e = a.ptr[r]; e < a.ptr[r + 1]; ++e) cols[a.idx[e]].emplace_back(r, a.val[e]);
    for (i64 c = 0; c < a.cols; ++c)
      for (const auto& [r, v] : cols[c]) std::fprintf(f, "%lld %lld %.17g\n", (long long)r + 1, (long long)c + 1, v);
  }
  std::fclose(f);
}

}  // namespace b200
