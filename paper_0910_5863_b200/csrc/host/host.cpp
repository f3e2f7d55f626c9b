// Host-side substructuring: mesh, Q1 assembly, globs, embeddings, constraints,
// change of variables, pair index spaces.  See host.hpp for the contract.
#include "host.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <deque>
#include <limits>
#include <iterator>
#include <numeric>
#include <unordered_set>

namespace b200 {

// ============================================================================
// Seeded coefficient fields; must match
// oracle/experiment.py bit for bit.
// ============================================================================
namespace {
struct SplitMix64 {
  std::uint64_t state;
  explicit SplitMix64(std::uint64_t s) : state(s) {}
  std::uint64_t next() {
    state += 0x9E3779B97F4A7C15ULL;
    std::uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
  double normal() {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2);
  }
};
}  // namespace

std::vector<double> element_scale_for(int config, const int ne[3], std::uint64_t seed) {
  const int nx = ne[0], ny = ne[1], nz = ne[2];
  const std::size_t n = std::size_t(nx) * ny * nz;
  std::vector<double> out;
  if (config == 1) return out;
  SplitMix64 rng(seed);
  out.assign(n, 1.0);
  if (config == 2) {
    std::vector<char> col(std::size_t(nx) * ny);
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) col[std::size_t(j) * nx + i] = rng.uniform() < 0.1;
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
          out[(std::size_t(k) * ny + j) * nx + i] = col[std::size_t(j) * nx + i] ? 1e6 : 1.0;
  } else if (config == 3) {
    for (std::size_t e = 0; e < n; ++e) out[e] = std::exp(2.0 * rng.normal());
  } else if (config == 4) {
    double sph[20][4];
    for (auto& s : sph) {
      s[0] = rng.uniform();
      s[1] = rng.uniform();
      s[2] = rng.uniform();
      s[3] = 0.05 + 0.05 * rng.uniform();
    }
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          const double x = (i + 0.5) / nx, y = (j + 0.5) / ny, z = (k + 0.5) / nz;
          bool inside = false;
          for (auto& s : sph) {
            const double dx = x - s[0], dy = y - s[1], dz = z - s[2];
            if (dx * dx + dy * dy + dz * dz < s[3] * s[3]) inside = true;
          }
          out[(std::size_t(k) * ny + j) * nx + i] = inside ? 1e4 : 1.0;
        }
  } else if (config == 5) {
    for (int k = 0; k < nz; ++k) {
      const double v = ((k / 3) % 2 == 1) ? 1e5 : 1.0;
      for (std::size_t t = 0; t < std::size_t(nx) * ny; ++t) out[std::size_t(k) * nx * ny + t] = v;
    }
  } else {
    throw Error(kBadProblemSpec, "unknown config");
  }
  return out;
}

Problem baseline_problem(int config, std::uint64_t seed, const int* sub_override,
                         int epe_override) {
  Problem p;
  static const int subs[6][3] = {{0, 0, 0}, {3, 3, 3}, {3, 3, 3}, {8, 8, 8}, {6, 6, 6}, {12, 12, 12}};
  static const int epes[6] = {0, 8, 8, 10, 8, 8};
  if (config < 1 || config > 5) throw Error(kBadProblemSpec, "config must be 1..5");
  for (int a = 0; a < 3; ++a) p.subdomains[a] = sub_override ? sub_override[a] : subs[config][a];
  p.elements_per_edge = epe_override > 0 ? epe_override : epes[config];
  p.physics = config >= 4 ? kElasticity : kScalar;
  DirichletSpec d;
  d.face = kXMin;
  p.dirichlet.push_back(d);
  if (p.physics == kScalar) {
    p.source = 1.0;
  } else {
    p.materials[0] = Material{1.0, 1.0, 0.3};
    p.body_force[2] = -1.0;
  }
  int ne[3];
  for (int a = 0; a < 3; ++a) ne[a] = p.subdomains[a] * p.elements_per_edge;
  p.element_scale = element_scale_for(config, ne, seed);
  return p;
}

// ============================================================================
// Mesh (mesh.cpp:9-82)
// ============================================================================
void Mesh::sharers(int node, std::vector<int>& out) const {
  out.clear();
  const int g[3] = {node % np[0], (node / np[0]) % np[1], node / (np[0] * np[1])};
  int cand[3][2], nc[3];
  for (int a = 0; a < 3; ++a) {
    nc[a] = 0;
    // subdomain index s owns element range [s*epe, (s+1)*epe) -> nodes [s*epe, (s+1)*epe]
    if (g[a] % epe == 0 && g[a] > 0) cand[a][nc[a]++] = g[a] / epe - 1;
    if (g[a] / epe < sub[a]) cand[a][nc[a]++] = g[a] / epe;
  }
  for (int k = 0; k < nc[2]; ++k)
    for (int j = 0; j < nc[1]; ++j)
      for (int i = 0; i < nc[0]; ++i)
        out.push_back((cand[2][k] * sub[1] + cand[1][j]) * sub[0] + cand[0][i]);
  std::sort(out.begin(), out.end());
}

double CSR::diag(int r) const {
  for (int t = ptr[r]; t < ptr[r + 1]; ++t)
    if (idx[t] == r) return val[t];
  return 0.0;
}

// ============================================================================
// Element stiffness (assemble.cpp:11-99)
// ============================================================================
namespace {
const int kXi[8] = {-1, 1, 1, -1, -1, 1, 1, -1};
const int kEta[8] = {-1, -1, 1, 1, -1, -1, 1, 1};
const int kZeta[8] = {-1, -1, -1, -1, 1, 1, 1, 1};

std::vector<double> element_stiffness(double h, const Material& m, int physics) {
  const int nc = components(physics);
  const int nd = 8 * nc;
  std::vector<double> ke(std::size_t(nd) * nd, 0.0);
  double corners[8][3];
  for (int i = 0; i < 8; ++i) {
    corners[i][0] = (kXi[i] > 0) * h;
    corners[i][1] = (kEta[i] > 0) * h;
    corners[i][2] = (kZeta[i] > 0) * h;
  }
  const double lambda = m.youngs * m.poisson / ((1 + m.poisson) * (1 - 2 * m.poisson));
  const double mu = m.youngs / (2 * (1 + m.poisson));
  double ct[6][6] = {};
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) ct[a][b] = lambda;
    ct[a][a] = lambda + 2 * mu;
    ct[3 + a][3 + a] = mu;
  }
  const double g = 1.0 / std::sqrt(3.0);
  for (int ia : {-1, 1})
    for (int ib : {-1, 1})
      for (int ic : {-1, 1}) {
        const double xi = ia * g, eta = ib * g, zeta = ic * g, w = 1.0;
        double d[8][3];
        for (int i = 0; i < 8; ++i) {
          d[i][0] = 0.125 * kXi[i] * (1 + eta * kEta[i]) * (1 + zeta * kZeta[i]);
          d[i][1] = 0.125 * (1 + xi * kXi[i]) * kEta[i] * (1 + zeta * kZeta[i]);
          d[i][2] = 0.125 * (1 + xi * kXi[i]) * (1 + eta * kEta[i]) * kZeta[i];
        }
        double J[3][3] = {};
        for (int i = 0; i < 8; ++i)
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) J[a][b] += corners[i][a] * d[i][b];
        const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        if (det <= 0) throw Error(kDegenerateElement, "element with nonpositive Jacobian");
        double inv[3][3];
        inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
        inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
        inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
        inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
        inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
        inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
        inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
        inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
        inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
        double grad[8][3];  // dref * J^{-1}
        for (int i = 0; i < 8; ++i)
          for (int b = 0; b < 3; ++b) {
            grad[i][b] = 0;
            for (int a = 0; a < 3; ++a) grad[i][b] += d[i][a] * inv[a][b];
          }
        if (physics == kScalar) {
          for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) {
              const double gg = grad[i][0] * grad[j][0] + grad[i][1] * grad[j][1] +
                                grad[i][2] * grad[j][2];
              ke[i * 8 + j] += m.conductivity * w * det * gg;
            }
        } else {
          double B[6][24] = {};
          for (int i = 0; i < 8; ++i) {
            const double dx = grad[i][0], dy = grad[i][1], dz = grad[i][2];
            B[0][3 * i] = dx;
            B[1][3 * i + 1] = dy;
            B[2][3 * i + 2] = dz;
            B[3][3 * i] = dy;
            B[3][3 * i + 1] = dx;
            B[4][3 * i + 1] = dz;
            B[4][3 * i + 2] = dy;
            B[5][3 * i] = dz;
            B[5][3 * i + 2] = dx;
          }
          double CB[6][24];
          for (int a = 0; a < 6; ++a)
            for (int c = 0; c < 24; ++c) {
              double s = 0;
              for (int b = 0; b < 6; ++b) s += ct[a][b] * B[b][c];
              CB[a][c] = s;
            }
          for (int r = 0; r < 24; ++r)
            for (int c = 0; c < 24; ++c) {
              double s = 0;
              for (int a = 0; a < 6; ++a) s += B[a][r] * CB[a][c];
              ke[r * 24 + c] += w * det * s;
            }
        }
      }
  return ke;
}

bool node_on_face(const Mesh& m, int node, int f) {
  const int i = node % m.np[0], j = (node / m.np[0]) % m.np[1], k = node / (m.np[0] * m.np[1]);
  switch (f) {
    case kXMin: return i == 0;
    case kXMax: return i == m.np[0] - 1;
    case kYMin: return j == 0;
    case kYMax: return j == m.np[1] - 1;
    case kZMin: return k == 0;
    case kZMax: return k == m.np[2] - 1;
  }
  return false;
}

bool element_on_face(const Mesh& m, int i, int j, int k, int f) {
  switch (f) {
    case kXMin: return i == 0;
    case kXMax: return i == m.ne[0] - 1;
    case kYMin: return j == 0;
    case kYMax: return j == m.ne[1] - 1;
    case kZMin: return k == 0;
    case kZMax: return k == m.ne[2] - 1;
  }
  return false;
}

const int kFaceLocalNodes[6][4] = {{0, 3, 7, 4}, {1, 2, 6, 5}, {0, 1, 5, 4},
                                   {3, 2, 6, 7}, {0, 1, 2, 3}, {4, 5, 6, 7}};

std::vector<int> grid_neighbors(const Mesh& m, int node) {  // globs.cpp:21-34
  const int nx = m.np[0], ny = m.np[1], nz = m.np[2];
  const int i = node % nx, j = (node / nx) % ny, k = node / (nx * ny);
  std::vector<int> out;
  out.reserve(6);
  if (i > 0) out.push_back(node - 1);
  if (i + 1 < nx) out.push_back(node + 1);
  if (j > 0) out.push_back(node - nx);
  if (j + 1 < ny) out.push_back(node + nx);
  if (k > 0) out.push_back(node - nx * ny);
  if (k + 1 < nz) out.push_back(node + nx * ny);
  return out;
}

void sort_canonical(std::vector<Glob>& globs) {  // globs.cpp:38-44
  std::sort(globs.begin(), globs.end(), [](const Glob& a, const Glob& b) {
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.nodes.front() < b.nodes.front();
  });
}

bool strict_superset(const std::vector<int>& big, const std::vector<int>& small) {
  return big.size() > small.size() &&
         std::includes(big.begin(), big.end(), small.begin(), small.end());
}
}  // namespace

int Maps::local_of(i64 g, int s) const {
  for (i64 t = copy_ptr[g]; t < copy_ptr[g + 1]; ++t)
    if (copy_sub[t] == s) return copy_local[t];
  return -1;
}

// ============================================================================
// Model::build = build_cube_mesh + decompose_cube + apply_dirichlet +
// assemble_subdomains + classify_globs + select_corners + build_embeddings
// (experiment.cpp:116-128)
// ============================================================================
namespace {

// VTK vertex order of the Q1 element: local grid offsets, and the inverse map
const int kVertexOff[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                              {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

// assemble_subdomains, structural part (assemble.cpp:202-269): local numbering,
// loads and the stiffness diagonal.  Values are summed element by element in
// the element loop order (k, j, i), which the device assembly and
// assemble_values reproduce entry by entry.
void assemble(Model& md) {
  const Mesh& m = md.mesh;
  const Problem& p = md.spec;
  const int nc = m.ncomp, epe = m.epe, ed = 8 * nc;
  std::map<int, int> mat_index;  // assemble.cpp:145-169
  md.ke_ref.clear();
  md.element_ke.resize(m.element_material.size());
  for (std::size_t e = 0; e < m.element_material.size(); ++e) {
    const int mat = m.element_material[e];
    auto f = mat_index.find(mat);
    if (f == mat_index.end()) {
      auto it = p.materials.find(mat);
      if (it == p.materials.end()) throw Error(kBadProblemSpec, "element references unknown material");
      f = mat_index.emplace(mat, static_cast<int>(md.ke_ref.size())).first;
      md.ke_ref.push_back(element_stiffness(m.h, it->second, m.physics));
    }
    md.element_ke[e] = f->second;
  }
  const int nsub = m.sub[0] * m.sub[1] * m.sub[2];
  md.subs.assign(nsub, Subdomain{});
  const int ln = epe + 1;  // local node grid per axis
#pragma omp parallel for schedule(dynamic, 4) if (nsub >= 64)
  for (int s = 0; s < nsub; ++s) {
    Subdomain& S = md.subs[s];
    S.id = s;
    const int si = s % m.sub[0], sj = (s / m.sub[0]) % m.sub[1], sk = s / (m.sub[0] * m.sub[1]);
    const int i0 = si * epe, j0 = sj * epe, k0 = sk * epe;
    S.origin[0] = i0;
    S.origin[1] = j0;
    S.origin[2] = k0;
    // nodes ascending by global id == (lk, lj, li) lexicographic
    S.lnode.assign(std::size_t(ln) * ln * ln * nc, -1);
    for (int lk = 0; lk < ln; ++lk)
      for (int lj = 0; lj < ln; ++lj)
        for (int li = 0; li < ln; ++li) {
          const int node = m.node_id(i0 + li, j0 + lj, k0 + lk);
          S.nodes.push_back(node);
          for (int c = 0; c < nc; ++c) {
            const i64 g = md.dof[i64(node) * nc + c];
            if (g < 0) continue;
            S.lnode[((std::size_t(lk) * ln + lj) * ln + li) * nc + c] = S.dim();
            S.global_dof.push_back(g);
          }
        }
    const int n = S.dim();
    S.load.assign(n, 0.0);
    S.diag.assign(n, 0.0);
    const double cell = m.h * m.h * m.h / 8.0;
    for (int lk = 0; lk < epe; ++lk)
      for (int lj = 0; lj < epe; ++lj)
        for (int li = 0; li < epe; ++li) {
          const int gi = i0 + li, gj = j0 + lj, gk = k0 + lk;
          const int e = (gk * m.ne[1] + gj) * m.ne[0] + gi;
          const std::vector<double>& ke = md.ke_ref[md.element_ke[e]];
          const double sc = m.element_scale.empty() ? 1.0 : m.element_scale[e];
          int local[24];
          for (int a = 0; a < 8; ++a)
            for (int c = 0; c < nc; ++c)
              local[a * nc + c] = S.lnode[((std::size_t(lk + kVertexOff[a][2]) * ln + lj + kVertexOff[a][1]) * ln +
                                           li + kVertexOff[a][0]) * nc + c];
          for (int a = 0; a < ed; ++a)
            if (local[a] >= 0) S.diag[local[a]] += sc == 1.0 ? ke[a * ed + a] : sc * ke[a * ed + a];
          for (int a = 0; a < 8; ++a)  // assemble.cpp:260-269
            for (int c = 0; c < nc; ++c) {
              const int l = local[a * nc + c];
              if (l < 0) continue;
              const double dens = m.physics == kScalar ? p.source : p.body_force[c];
              S.load[l] += dens * cell;
            }
          for (const auto& ls : p.loads) {  // assemble.cpp:271-283
            if (!element_on_face(m, gi, gj, gk, ls.face)) continue;
            const double qa = m.h * m.h / 4.0;
            for (int fn : kFaceLocalNodes[ls.face])
              for (int c = 0; c < nc; ++c) {
                const int l = local[fn * nc + c];
                if (l < 0) continue;
                const double t = m.physics == kScalar ? ls.flux : ls.traction[c];
                S.load[l] += t * qa;
              }
          }
        }
  }
}

// assemble_subdomains, values (assemble.cpp:202-258): upper entries accumulated
// per element in loop order, the full symmetric CSR mirrored from them.
void assemble_values(const Model& md, const Subdomain& S, CSR& A) {
  const Mesh& m = md.mesh;
  const int nc = m.ncomp, epe = m.epe, ed = 8 * nc, ln = epe + 1, slots = 27 * nc;
  const int n = S.dim();
  const int i0 = S.origin[0], j0 = S.origin[1], k0 = S.origin[2];
  std::vector<double> acc(std::size_t(n) * slots, 0.0);
  for (int lk = 0; lk < epe; ++lk)
    for (int lj = 0; lj < epe; ++lj)
      for (int li = 0; li < epe; ++li) {
        const int e = ((k0 + lk) * m.ne[1] + j0 + lj) * m.ne[0] + i0 + li;
        const std::vector<double>& ke = md.ke_ref[md.element_ke[e]];
        const double sc = m.element_scale.empty() ? 1.0 : m.element_scale[e];
        int local[24];
        for (int a = 0; a < 8; ++a)
          for (int c = 0; c < nc; ++c)
            local[a * nc + c] = S.lnode[((std::size_t(lk + kVertexOff[a][2]) * ln + lj + kVertexOff[a][1]) * ln + li +
                                         kVertexOff[a][0]) * nc + c];
        for (int a = 0; a < ed; ++a) {
          if (local[a] < 0) continue;
          const int na = a / nc;
          for (int b = 0; b < ed; ++b) {
            if (local[b] < 0 || local[b] < local[a]) continue;
            const int nb = b / nc, cb = b % nc;
            const int slot = ((kVertexOff[nb][2] - kVertexOff[na][2] + 1) * 3 + (kVertexOff[nb][1] - kVertexOff[na][1] + 1)) * 3 +
                             (kVertexOff[nb][0] - kVertexOff[na][0] + 1);
            const double v = sc == 1.0 ? ke[a * ed + b] : sc * ke[a * ed + b];
            acc[std::size_t(local[a]) * slots + slot * nc + cb] += v;
          }
        }
      }
  // CSR of the full symmetric matrix: columns ascending = slot order.
  A.n = n;
  A.ptr.assign(n + 1, 0);
  A.idx.clear();
  A.val.clear();
  std::vector<int> row_node(n), row_comp(n);
  for (int lk = 0; lk < ln; ++lk)
    for (int lj = 0; lj < ln; ++lj)
      for (int li = 0; li < ln; ++li)
        for (int c = 0; c < nc; ++c) {
          const int l = S.lnode[((std::size_t(lk) * ln + lj) * ln + li) * nc + c];
          if (l >= 0) {
            row_node[l] = (lk * ln + lj) * ln + li;
            row_comp[l] = c;
          }
        }
  for (int r = 0; r < n; ++r) {
    const int rn = row_node[r];
    const int rl = rn % ln, rm = (rn / ln) % ln, rk = rn / (ln * ln);
    const int ra = row_comp[r];
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int ci = rl + dx, cj = rm + dy, ck = rk + dz;
          if (ci < 0 || cj < 0 || ck < 0 || ci >= ln || cj >= ln || ck >= ln) continue;
          for (int c = 0; c < nc; ++c) {
            const int col = S.lnode[((std::size_t(ck) * ln + cj) * ln + ci) * nc + c];
            if (col < 0) continue;
            // upper entries were accumulated at (min, max)
            double v;
            if (col >= r) {
              const int slot = ((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1);
              v = acc[std::size_t(r) * slots + slot * nc + c];
            } else {
              const int slot = ((-dz + 1) * 3 + (-dy + 1)) * 3 + (-dx + 1);
              v = acc[std::size_t(col) * slots + slot * nc + ra];
            }
            A.idx.push_back(col);
            A.val.push_back(v);
          }
        }
    A.ptr[r + 1] = static_cast<int>(A.idx.size());
  }
}

void classify_and_select(Model& md) {
  const Mesh& m = md.mesh;
  // classify_globs (globs.cpp:61-99)
  std::map<std::vector<int>, std::vector<int>> groups;
  std::vector<int> sh;
  std::vector<std::vector<int>> node_subs(m.node_count());
  for (int n = 0; n < m.node_count(); ++n) {
    m.sharers(n, sh);
    node_subs[n] = sh;
    if (sh.size() >= 2) groups[sh].push_back(n);
  }
  std::vector<Glob>& out = md.globs;
  out.clear();
  for (const auto& [sharers, nodes] : groups) {
    std::unordered_set<int> pending(nodes.begin(), nodes.end());
    for (int seed : nodes) {
      if (!pending.count(seed)) continue;
      Glob g;
      g.subdomains = sharers;
      std::deque<int> frontier{seed};
      pending.erase(seed);
      while (!frontier.empty()) {
        const int n = frontier.front();
        frontier.pop_front();
        g.nodes.push_back(n);
        for (int nb : grid_neighbors(m, n))
          if (pending.count(nb)) {
            pending.erase(nb);
            frontier.push_back(nb);
          }
      }
      std::sort(g.nodes.begin(), g.nodes.end());
      g.kind = sharers.size() == 2 ? kFace : (g.nodes.size() == 1 ? kCorner : kEdge);
      out.push_back(std::move(g));
    }
  }
  md.classification_corners = static_cast<int>(md.count(kCorner));
  sort_canonical(out);

  // select_corners (globs.cpp:103-254)
  std::vector<int> corners;
  for (const auto& g : out)
    if (g.kind == kCorner) corners.push_back(g.nodes.front());
  auto promote = [&](std::size_t source, int node) {
    auto& nodes = out[source].nodes;
    nodes.erase(std::find(nodes.begin(), nodes.end(), node));
    Glob c;
    c.kind = kCorner;
    c.nodes = {node};
    c.subdomains = node_subs[node];
    out.push_back(std::move(c));
    corners.push_back(node);
  };
  auto in_glob_neighbors = [&](const std::unordered_set<int>& members, int node) {
    int cnt = 0;
    for (int nb : grid_neighbors(m, node)) cnt += members.count(nb) ? 1 : 0;
    return cnt;
  };
  // promote_edge_endpoints
  const std::size_t n_globs = out.size();
  for (std::size_t gi = 0; gi < n_globs; ++gi) {
    if (out[gi].kind != kEdge) continue;
    const std::unordered_set<int> members(out[gi].nodes.begin(), out[gi].nodes.end());
    std::vector<int> promoted;
    for (int node : out[gi].nodes) {
      if (in_glob_neighbors(members, node) > 1) continue;
      bool bigger = false;
      for (int nb : grid_neighbors(m, node))
        if (strict_superset(node_subs[nb], out[gi].subdomains)) {
          bigger = true;
          break;
        }
      if (!bigger) promoted.push_back(node);
    }
    for (int node : promoted) promote(gi, node);
  }
  auto shared_corners = [&](const std::vector<int>& pair) {
    std::vector<int> r;
    for (int c : corners)
      if (std::includes(node_subs[c].begin(), node_subs[c].end(), pair.begin(), pair.end()))
        r.push_back(c);
    return r;
  };
  auto pinned = [&](const std::vector<int>& shared) {
    if (m.physics == kScalar) return !shared.empty();
    if (shared.size() < 3) return false;
    double p0[3];
    m.coords(shared[0], p0);
    for (std::size_t a = 1; a < shared.size(); ++a) {
      double p1[3];
      m.coords(shared[a], p1);
      const double u[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
      for (std::size_t b = a + 1; b < shared.size(); ++b) {
        double p2[3];
        m.coords(shared[b], p2);
        const double v[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
        const double cx = u[1] * v[2] - u[2] * v[1];
        const double cy = u[2] * v[0] - u[0] * v[2];
        const double cz = u[0] * v[1] - u[1] * v[0];
        if (cx * cx + cy * cy + cz * cz > 1e-16) return true;
      }
    }
    return false;
  };
  auto promote_candidates = [&](std::size_t glob, std::vector<int> candidates,
                                const std::vector<int>& pair) {
    while (!candidates.empty()) {
      const auto shared = shared_corners(pair);
      if (pinned(shared)) return;
      std::vector<std::pair<double, int>> ranked;
      for (int node : candidates) {
        double dmin = std::numeric_limits<double>::infinity();
        double pn[3];
        m.coords(node, pn);
        for (int c : shared) {
          double pc[3];
          m.coords(c, pc);
          const double dx = pn[0] - pc[0], dy = pn[1] - pc[1], dz = pn[2] - pc[2];
          dmin = std::min(dmin, dx * dx + dy * dy + dz * dz);
        }
        ranked.emplace_back(dmin, node);
      }
      std::sort(ranked.begin(), ranked.end(), [](const auto& a, const auto& b) {
        if (a.first != b.first) return a.first > b.first;
        return a.second < b.second;
      });
      const double top = ranked.front().first;
      std::vector<int> group;
      for (const auto& [d, node] : ranked)
        if (d == top || std::abs(d - top) <= 1e-9 * std::max(1.0, top)) group.push_back(node);
      for (int node : group) {
        promote(glob, node);
        candidates.erase(std::find(candidates.begin(), candidates.end(), node));
      }
    }
  };
  // repair_pairs
  std::vector<std::size_t> faces;
  for (std::size_t gi = 0; gi < out.size(); ++gi)
    if (out[gi].kind == kFace) faces.push_back(gi);
  std::sort(faces.begin(), faces.end(), [&](std::size_t a, std::size_t b) {
    if (out[a].subdomains != out[b].subdomains) return out[a].subdomains < out[b].subdomains;
    return out[a].nodes.front() < out[b].nodes.front();
  });
  for (std::size_t gi : faces) {
    const std::vector<int> pair = out[gi].subdomains;
    if (pinned(shared_corners(pair))) continue;
    const auto nodes = out[gi].nodes;
    const std::unordered_set<int> members(nodes.begin(), nodes.end());
    std::vector<int> rim;
    for (int node : nodes)
      if (in_glob_neighbors(members, node) <= 2) rim.push_back(node);
    promote_candidates(gi, rim, pair);
    if (!pinned(shared_corners(pair))) promote_candidates(gi, out[gi].nodes, pair);
    if (!pinned(shared_corners(pair)))
      throw Error(kCornerSelectionFailed, "cannot pin substructure pair " +
                                              std::to_string(pair[0]) + "," + std::to_string(pair[1]));
  }
  out.erase(std::remove_if(out.begin(), out.end(), [](const Glob& g) { return g.nodes.empty(); }),
            out.end());
  sort_canonical(out);
}

void embeddings(Model& md) {  // spaces.cpp:9-56
  Maps& mp = md.maps;
  const int nsub = static_cast<int>(md.subs.size());
  mp.w_offset.assign(nsub, 0);
  mp.w_dim = 0;
  for (int s = 0; s < nsub; ++s) {
    mp.w_offset[s] = mp.w_dim;
    mp.w_dim += md.subs[s].dim();
  }
  std::vector<i64> cnt(md.free_count + 1, 0);
  for (const auto& S : md.subs)
    for (i64 g : S.global_dof) ++cnt[g + 1];
  mp.copy_ptr.assign(md.free_count + 1, 0);
  for (i64 g = 0; g < md.free_count; ++g) mp.copy_ptr[g + 1] = mp.copy_ptr[g] + cnt[g + 1];
  mp.copy_sub.assign(mp.copy_ptr.back(), 0);
  mp.copy_local.assign(mp.copy_ptr.back(), 0);
  std::vector<i64> fill(mp.copy_ptr.begin(), mp.copy_ptr.end() - 1);
  for (int s = 0; s < nsub; ++s)
    for (int l = 0; l < md.subs[s].dim(); ++l) {
      const i64 g = md.subs[s].global_dof[l];
      mp.copy_sub[fill[g]] = s;
      mp.copy_local[fill[g]] = l;
      ++fill[g];
    }
  mp.interface_dofs.clear();
  mp.global_to_interface.assign(md.free_count, -1);
  for (i64 g = 0; g < md.free_count; ++g)
    if (mp.copy_ptr[g + 1] - mp.copy_ptr[g] >= 2) {
      mp.global_to_interface[g] = static_cast<i64>(mp.interface_dofs.size());
      mp.interface_dofs.push_back(g);
    }
  mp.corner_dof_of_global.assign(md.free_count, -1);
  mp.corner_dof_count = 0;
  for (int node : md.corner_nodes())
    for (int c = 0; c < md.mesh.ncomp; ++c) {
      const i64 g = md.dof[i64(node) * md.mesh.ncomp + c];
      if (g < 0) continue;
      mp.corner_dof_of_global[g] = mp.corner_dof_count++;
    }
  mp.wc_dim = mp.corner_dof_count;
  mp.local_to_wc.assign(nsub, {});
  for (int s = 0; s < nsub; ++s) {
    auto& S = md.subs[s];
    mp.local_to_wc[s].resize(S.dim());
    S.interior.clear();
    S.boundary.clear();
    for (int l = 0; l < S.dim(); ++l) {
      const i64 g = S.global_dof[l];
      const i64 corner = mp.corner_dof_of_global[g];
      mp.local_to_wc[s][l] = corner >= 0 ? corner : mp.wc_dim++;
      if (mp.copy_ptr[g + 1] - mp.copy_ptr[g] >= 2)
        S.boundary.push_back(l);
      else
        S.interior.push_back(l);
    }
  }
}

}  // namespace

namespace {
// BDDC_B200_PROFILE=1: host phase times of Model::build on stderr
struct BuildTimer {
  using clk = std::chrono::steady_clock;
  bool on;
  clk::time_point t = clk::now();
  std::string line;
  BuildTimer() {
    const char* e = std::getenv("BDDC_B200_PROFILE");
    on = e && *e && *e != '0';
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = clk::now();
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s=%.3fms", what, std::chrono::duration<double, std::milli>(now - t).count());
    line += buf;
    t = now;
  }
  ~BuildTimer() {
    if (on) std::fprintf(stderr, "[profile] model build:%s\n", line.c_str());
  }
};
}  // namespace

void Model::build(const Problem& p) {
  BuildTimer bt;
  spec = p;
  if (p.elements_per_edge < 1) throw Error(kBadProblemSpec, "elements per subdomain edge must be >= 1");
  for (int a = 0; a < 3; ++a)
    if (p.subdomains[a] < 1) throw Error(kBadProblemSpec, "subdomain counts must be >= 1");
  mesh = Mesh{};
  mesh.physics = p.physics;
  mesh.ncomp = components(p.physics);
  mesh.epe = p.elements_per_edge;
  mesh.h = 1.0 / p.elements_per_edge;
  for (int a = 0; a < 3; ++a) {
    mesh.sub[a] = p.subdomains[a];
    mesh.ne[a] = p.subdomains[a] * p.elements_per_edge;
    mesh.np[a] = mesh.ne[a] + 1;
  }
  mesh.element_material.assign(mesh.element_count(), 0);
  for (int k = 0; k < mesh.ne[2]; ++k)
    for (int j = 0; j < mesh.ne[1]; ++j)
      for (int i = 0; i < mesh.ne[0]; ++i) {
        int mat = 0;
        for (const auto& r : p.regions)
          if (i >= r.lo[0] && i < r.hi[0] && j >= r.lo[1] && j < r.hi[1] && k >= r.lo[2] &&
              k < r.hi[2])
            mat = r.material;
        mesh.element_material[(k * mesh.ne[1] + j) * mesh.ne[0] + i] = mat;
      }
  if (!p.element_scale.empty()) {
    if (static_cast<int>(p.element_scale.size()) != mesh.element_count())
      throw Error(kBadProblemSpec, "element_scale length does not match the mesh");
    mesh.element_scale = p.element_scale;
  }
  // apply_dirichlet (assemble.cpp:101-141)
  const int nc = mesh.ncomp;
  dof.assign(i64(mesh.node_count()) * nc, 0);
  for (int n = 0; n < mesh.node_count(); ++n)
    for (const auto& d : p.dirichlet)
      if (node_on_face(mesh, n, d.face))
        for (int c = 0; c < nc; ++c)
          if (d.constrained[c]) dof[i64(n) * nc + c] = -1;
  free_count = 0;
  for (auto& d : dof)
    if (d == 0) d = free_count++;
  bt.mark("mesh+dirichlet");
  assemble(*this);
  bt.mark("assemble");
  classify_and_select(*this);
  bt.mark("globs");
  embeddings(*this);
  bt.mark("embeddings");
  // per-glob free dofs, per-subdomain glob lists and Dirichlet flags (pair index support)
  glob_dofs.resize(globs.size());
  sub_globs.assign(subs.size(), {});
  for (std::size_t gi = 0; gi < globs.size(); ++gi) {
    glob_dofs[gi] = glob_free_dofs(static_cast<int>(gi));
    for (int s : globs[gi].subdomains) sub_globs[s].push_back(static_cast<int>(gi));
  }
  sub_constrained.assign(subs.size(), 0);
  for (std::size_t s = 0; s < subs.size(); ++s)
    for (int node : subs[s].nodes)
      for (int c = 0; c < nc; ++c) sub_constrained[s] |= dof[i64(node) * nc + c] < 0;
  bt.mark("glob_lists");
}

const CSR& Model::matrix(int s) const {
  const Subdomain& S = subs.at(s);
  if (!S.have_A) {
    assemble_values(*this, S, S.A);
    S.have_A = true;
  }
  return S.A;
}

std::vector<i64> Model::glob_free_dofs(int gi) const {
  std::vector<i64> out;
  for (int node : globs[gi].nodes)
    for (int c = 0; c < mesh.ncomp; ++c) {
      const i64 g = dof[i64(node) * mesh.ncomp + c];
      if (g >= 0) out.push_back(g);
    }
  return out;
}

std::vector<int> Model::corner_nodes() const {
  std::vector<int> out;
  for (const auto& g : globs)
    if (g.kind == kCorner) out.push_back(g.nodes.front());
  return out;
}

i64 Model::count(int kind) const {
  i64 n = 0;
  for (const auto& g : globs) n += g.kind == kind;
  return n;
}

// ============================================================================
// Dense QR (dense_eig.cpp:17-75), row-major storage
// ============================================================================
PivotedQr pivoted_qr(const std::vector<double>& a, int m, int n, double rel_drop_tol, bool want_q) {
  PivotedQr o;
  o.m = m;
  o.n = n;
  o.r = a;
  if (want_q) {
    o.q.assign(std::size_t(m) * m, 0.0);
    for (int i = 0; i < m; ++i) o.q[std::size_t(i) * m + i] = 1.0;
  }
  o.perm.resize(n);
  std::iota(o.perm.begin(), o.perm.end(), 0);
  auto R = [&](int i, int j) -> double& { return o.r[std::size_t(i) * n + j]; };
  auto Q = [&](int i, int j) -> double& { return o.q[std::size_t(i) * m + j]; };
  const int steps = std::min(m, n);
  std::vector<double> v(m), tmp(std::max(m, n));
  for (int k = 0; k < steps; ++k) {
    auto colnorm = [&](int j) {
      double s = 0;
      for (int i = k; i < m; ++i) s += R(i, j) * R(i, j);
      return std::sqrt(s);
    };
    int best = k;
    double best_norm = colnorm(k);
    for (int j = k + 1; j < n; ++j) {
      const double nj = colnorm(j);
      if (nj > best_norm) {
        best = j;
        best_norm = nj;
      }
    }
    if (best != k) {
      for (int i = 0; i < m; ++i) std::swap(R(i, k), R(i, best));
      std::swap(o.perm[k], o.perm[best]);
    }
    if (best_norm == 0.0) break;
    double xn = 0;
    for (int i = k; i < m; ++i) xn += R(i, k) * R(i, k);
    xn = std::sqrt(xn);
    const double alpha = (R(k, k) >= 0 ? -1.0 : 1.0) * xn;
    for (int i = k; i < m; ++i) v[i] = R(i, k);
    v[k] -= alpha;
    double vsq = 0;
    for (int i = k; i < m; ++i) vsq += v[i] * v[i];
    if (vsq > 0) {
      const double f = 2.0 / vsq;
      for (int j = k; j < n; ++j) {  // block -= f v (v^T block)
        double s = 0;
        for (int i = k; i < m; ++i) s += v[i] * R(i, j);
        for (int i = k; i < m; ++i) R(i, j) -= f * v[i] * s;
      }
      for (int i = 0; want_q && i < m; ++i) {  // qblock -= (qblock v)(f v)^T
        double s = 0;
        for (int j = k; j < m; ++j) s += Q(i, j) * v[j];
        for (int j = k; j < m; ++j) Q(i, j) -= s * f * v[j];
      }
    }
    R(k, k) = alpha;
    for (int i = k + 1; i < m; ++i) R(i, k) = 0.0;
    if (R(k, k) < 0) {
      for (int j = k; j < n; ++j) R(k, j) = -R(k, j);
      for (int i = 0; want_q && i < m; ++i) Q(i, k) = -Q(i, k);
    }
  }
  const double d0 = (m && n) ? std::abs(R(0, 0)) : 0.0;
  o.rank = 0;
  for (int k = 0; k < steps; ++k) {
    if (std::abs(R(k, k)) > rel_drop_tol * d0 && d0 > 0)
      ++o.rank;
    else
      break;
  }
  return o;
}

// ============================================================================
// Constraints (constraints.cpp) and transforms (transform.cpp)
// ============================================================================
i64 ConstraintSet::row_count(const Model& m) const {
  i64 rows = 0;
  for (const auto& a : averages) rows += static_cast<i64>(m.globs[a.glob].subdomains.size()) - 1;
  return rows;
}

std::vector<std::vector<int>> ConstraintSet::by_glob(std::size_t n) const {
  std::vector<std::vector<int>> out(n);
  for (std::size_t a = 0; a < averages.size(); ++a) out[averages[a].glob].push_back(int(a));
  return out;
}

ConstraintSet arithmetic_constraints(const Model& md, bool edges, bool faces) {
  ConstraintSet cs;
  const int nc = md.mesh.ncomp;
  for (std::size_t gi = 0; gi < md.globs.size(); ++gi) {
    const Glob& g = md.globs[gi];
    if (g.kind == kCorner) continue;
    if (g.kind == kEdge && !edges) continue;
    if (g.kind == kFace && !faces) continue;
    std::vector<int> comp;
    for (int node : g.nodes)
      for (int c = 0; c < nc; ++c)
        if (md.dof[i64(node) * nc + c] >= 0) comp.push_back(c);
    if (comp.empty()) continue;
    for (int c = 0; c < nc; ++c) {
      Average a;
      a.glob = static_cast<int>(gi);
      a.weights.assign(comp.size(), 0.0);
      bool any = false;
      for (std::size_t t = 0; t < comp.size(); ++t)
        if (comp[t] == c) {
          a.weights[t] = 1.0;
          any = true;
        }
      if (any) cs.averages.push_back(std::move(a));
    }
  }
  return cs;
}

bool average_admissible(const std::vector<const std::vector<double>*>& existing, const std::vector<double>& w) {
  bool nz = false;
  for (double x : w) nz |= (x != 0.0);
  if (!nz) return false;
  if (!existing.empty()) {
    const int m = static_cast<int>(w.size());
    const int n = static_cast<int>(existing.size()) + 1;
    std::vector<double> stack(std::size_t(m) * n);
    for (int i = 0; i < m; ++i) {
      for (int c = 0; c + 1 < n; ++c) stack[std::size_t(i) * n + c] = (*existing[c])[i];
      stack[std::size_t(i) * n + n - 1] = w[i];
    }
    if (pivoted_qr(stack, m, n, 1e-8, false).rank <= n - 1) return false;
  }
  return true;
}

bool add_average(ConstraintSet& cs, Average avg) {
  std::vector<const std::vector<double>*> existing;
  for (const auto& a : cs.averages)
    if (a.glob == avg.glob) existing.push_back(&a.weights);
  if (!average_admissible(existing, avg.weights)) return false;
  cs.averages.push_back(std::move(avg));
  return true;
}

namespace {
// Upper-triangular solve U X = B (U r x r row-major, B r x c row-major), in place.
void upper_solve(const std::vector<double>& U, int r, std::vector<double>& B, int c) {
  for (int col = 0; col < c; ++col)
    for (int i = r - 1; i >= 0; --i) {
      double s = B[std::size_t(i) * c + col];
      for (int k = i + 1; k < r; ++k) s -= U[std::size_t(i) * r + k] * B[std::size_t(k) * c + col];
      B[std::size_t(i) * c + col] = s / U[std::size_t(i) * r + i];
    }
}
}  // namespace

GlobTransform build_glob_transform(int glob, const std::vector<double>& rows, int r_in, int n) {
  const PivotedQr qr = pivoted_qr(rows, r_in, n, 1e-8, false);
  if (qr.rank < r_in) throw Error(kSingularGram, "dependent averages slipped past the rank filter");
  const int r = qr.rank;
  std::vector<double> u(std::size_t(r) * r), v(std::size_t(r) * (n - r));
  for (int i = 0; i < r; ++i) {
    for (int j = 0; j < r; ++j) u[std::size_t(i) * r + j] = qr.r[std::size_t(i) * n + j];
    for (int j = r; j < n; ++j) v[std::size_t(i) * (n - r) + j - r] = qr.r[std::size_t(i) * n + j];
  }
  std::vector<double> uinv(std::size_t(r) * r, 0.0);
  for (int i = 0; i < r; ++i) uinv[std::size_t(i) * r + i] = 1.0;
  upper_solve(u, r, uinv, r);
  // Compact form: t.row(perm[i]) = t_perm.row(i) with t_perm rows i >= r equal
  // to unit rows, so t is the permutation plus the r dense rows
  // D = [U^{-1} | -U^{-1} V] (transform.cpp:51-90).
  GlobTransform gt;
  gt.glob = glob;
  gt.rank = r;
  gt.n = n;
  gt.perm = qr.perm;
  gt.D.assign(std::size_t(r) * n, 0.0);
  for (int i = 0; i < r; ++i) {
    for (int j = 0; j < r; ++j) gt.D[std::size_t(i) * n + j] = uinv[std::size_t(i) * r + j];
    for (int j = r; j < n; ++j) {
      double acc = 0;
      for (int k = 0; k < r; ++k) acc += uinv[std::size_t(i) * r + k] * v[std::size_t(k) * (n - r) + j - r];
      gt.D[std::size_t(i) * n + j] = -acc;
    }
  }
  return gt;
}

std::vector<double> glob_kernel(const std::vector<double>* rows, int r_in, int n, int* cols) {
  if (!rows) {
    std::vector<double> k(std::size_t(n) * n, 0.0);
    for (int i = 0; i < n; ++i) k[std::size_t(i) * n + i] = 1.0;
    *cols = n;
    return k;
  }
  const PivotedQr qr = pivoted_qr(*rows, r_in, n);
  const int r = qr.rank;
  *cols = n - r;
  std::vector<double> k(std::size_t(n) * (n - r), 0.0);
  if (n > r) {
    std::vector<double> u(std::size_t(r) * r), top(std::size_t(r) * (n - r));
    for (int i = 0; i < r; ++i) {
      for (int j = 0; j < r; ++j) u[std::size_t(i) * r + j] = qr.r[std::size_t(i) * n + j];
      for (int j = r; j < n; ++j) top[std::size_t(i) * (n - r) + j - r] = qr.r[std::size_t(i) * n + j];
    }
    upper_solve(u, r, top, n - r);
    for (int a = 0; a < r; ++a)
      for (int c = 0; c < n - r; ++c) k[std::size_t(qr.perm[a]) * (n - r) + c] = -top[std::size_t(a) * (n - r) + c];
    for (int a = r; a < n; ++a) k[std::size_t(qr.perm[a]) * (n - r) + a - r] = 1.0;
  }
  return k;
}

std::vector<double> GlobTransform::dense_t() const {
  std::vector<double> t(std::size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      t[std::size_t(perm[i]) * n + j] = i < rank ? D[std::size_t(i) * n + j] : (i == j ? 1.0 : 0.0);
  return t;
}

KernelCompact glob_kernel_compact(const std::vector<double>* rows, int r_in, int n) {
  KernelCompact kc;
  kc.n = n;
  if (!rows) {
    kc.r = 0;
    kc.perm.resize(n);
    std::iota(kc.perm.begin(), kc.perm.end(), 0);
    return kc;
  }
  const PivotedQr qr = pivoted_qr(*rows, r_in, n, 1e-8, false);
  const int r = qr.rank;
  kc.r = r;
  kc.perm = qr.perm;
  kc.neg_top.assign(std::size_t(r) * (n - r), 0.0);
  if (n > r && r > 0) {
    std::vector<double> u(std::size_t(r) * r), top(std::size_t(r) * (n - r));
    for (int i = 0; i < r; ++i) {
      for (int j = 0; j < r; ++j) u[std::size_t(i) * r + j] = qr.r[std::size_t(i) * n + j];
      for (int j = r; j < n; ++j) top[std::size_t(i) * (n - r) + j - r] = qr.r[std::size_t(i) * n + j];
    }
    upper_solve(u, r, top, n - r);
    for (std::size_t t = 0; t < top.size(); ++t) kc.neg_top[t] = -top[t];
  }
  return kc;
}

ChangeOfVariables change_of_variables(const ConstraintSet& cs, const Model& md) {
  ChangeOfVariables cov;
  const auto bg = cs.by_glob(md.globs.size());
  std::vector<int> constrained;
  for (std::size_t gi = 0; gi < md.globs.size(); ++gi)
    if (!bg[gi].empty()) constrained.push_back(static_cast<int>(gi));
  // the per-glob QRs are independent; groups keep glob order
  cov.transforms.resize(constrained.size());
#pragma omp parallel for schedule(dynamic, 16) if (constrained.size() >= 512)
  for (int q = 0; q < static_cast<int>(constrained.size()); ++q) {
    const int gi = constrained[q];
    const int n = static_cast<int>(md.glob_dofs[gi].size());
    const int r_in = static_cast<int>(bg[gi].size());
    std::vector<double> rows(std::size_t(r_in) * n);
    for (int a = 0; a < r_in; ++a)
      for (int t = 0; t < n; ++t) rows[std::size_t(a) * n + t] = cs.averages[bg[gi][a]].weights[t];
    cov.transforms[q] = build_glob_transform(gi, rows, r_in, n);
  }
  // one group per explicit dof, in glob order (offsets first, then the fill in parallel)
  std::vector<std::size_t> goff(constrained.size() + 1, 0);
  for (std::size_t q = 0; q < constrained.size(); ++q) goff[q + 1] = goff[q] + cov.transforms[q].rank;
  cov.groups.resize(goff.back());
  cov.group_subs.resize(goff.back());
  cov.group_local.resize(goff.back());
#pragma omp parallel for schedule(dynamic, 16) if (constrained.size() >= 512)
  for (int q = 0; q < static_cast<int>(constrained.size()); ++q) {
    const int gi = constrained[q];
    const Glob& g = md.globs[gi];
    const auto& dofs = md.glob_dofs[gi];
    const GlobTransform& gt = cov.transforms[q];
    for (int k = 0; k < gt.rank; ++k) {  // explicit_slots[k] == k
      const i64 gdof = dofs[k];
      std::vector<i64>& grp = cov.groups[goff[q] + k];
      std::vector<int>& gs = cov.group_subs[goff[q] + k];
      std::vector<int>& gl = cov.group_local[goff[q] + k];
      grp.reserve(g.subdomains.size());
      gs.reserve(g.subdomains.size());
      gl.reserve(g.subdomains.size());
      for (int s : g.subdomains) {
        const int l = md.maps.local_of(gdof, s);
        grp.push_back(md.maps.local_to_wc[s][l]);
        gs.push_back(s);
        gl.push_back(l);
      }
    }
  }
  return cov;
}

std::vector<CoarseLeaf> primal_leaves(const Model& md, const ChangeOfVariables& cov, CoarseBounds* bounds) {
  const int ns = static_cast<int>(md.subs.size());
  const i64 ncd = md.maps.corner_dof_count;
  const std::size_t n_primal = static_cast<std::size_t>(ncd) + cov.groups.size();
  std::vector<CoarseLeaf> leaves(ns);
  for (int s = 0; s < ns; ++s)
    for (int a = 0; a < 3; ++a) leaves[s].coord[a] = md.subs[s].origin[a] / md.mesh.epe;
  if (bounds) {
    bounds->lo.assign(3 * n_primal, 1 << 30);
    bounds->hi.assign(3 * n_primal, -1);
  }
  auto hold = [&](std::size_t k, int s) {
    leaves[s].coarse.push_back(static_cast<int>(k));
    if (!bounds) return;
    for (int a = 0; a < 3; ++a) {
      bounds->lo[3 * k + a] = std::min(bounds->lo[3 * k + a], leaves[s].coord[a]);
      bounds->hi[3 * k + a] = std::max(bounds->hi[3 * k + a], leaves[s].coord[a] + 1);
    }
  };
  for (std::size_t g = 0; g < md.globs.size(); ++g)
    for (i64 dof : md.glob_dofs[g]) {
      const i64 cid = md.maps.corner_dof_of_global[dof];
      if (cid < 0) continue;
      for (int s : md.globs[g].subdomains) hold(static_cast<std::size_t>(cid), s);
    }
  for (std::size_t g = 0; g < cov.groups.size(); ++g)
    for (int s : cov.group_subs[g]) hold(static_cast<std::size_t>(ncd) + g, s);
  return leaves;
}

// ============================================================================
// Pairs (pair.cpp:67-146, adaptive.cpp:12-20)
// ============================================================================
std::vector<std::pair<int, int>> face_pairs(const Model& md) {
  std::vector<std::pair<int, int>> pairs;
  for (const auto& g : md.globs)
    if (g.kind == kFace) pairs.emplace_back(g.subdomains[0], g.subdomains[1]);
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  return pairs;
}

PairIndex build_pair_index(const Model& md, int si, int sj) {
  PairIndex p;
  p.si = si;
  p.sj = sj;
  // globs touching either side, ascending (the reference scans all globs in
  // order, pair.cpp:80-108; only these can contribute)
  const auto& gi_list = md.sub_globs[si];
  const auto& gj_list = md.sub_globs[sj];
  std::vector<int> touched;
  std::merge(gi_list.begin(), gi_list.end(), gj_list.begin(), gj_list.end(), std::back_inserter(touched));
  touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
  for (int gi : touched) {
    const Glob& g = md.globs[gi];
    const bool hi = std::binary_search(g.subdomains.begin(), g.subdomains.end(), si);
    const bool hj = std::binary_search(g.subdomains.begin(), g.subdomains.end(), sj);
    const auto& dofs = md.glob_dofs[gi];
    if (hi && hj) {
      if (g.kind == kCorner) {
        p.corner_globals.insert(p.corner_globals.end(), dofs.begin(), dofs.end());
      } else {
        p.shared_globs.push_back(static_cast<int>(gi));
        p.glob_offset.push_back(static_cast<int>(p.noncorner_globals.size()));
        p.glob_size.push_back(static_cast<int>(dofs.size()));
        p.noncorner_globals.insert(p.noncorner_globals.end(), dofs.begin(), dofs.end());
      }
    } else if (hi) {
      p.outer_i.insert(p.outer_i.end(), dofs.begin(), dofs.end());
    } else if (hj) {
      p.outer_j.insert(p.outer_j.end(), dofs.begin(), dofs.end());
    }
  }
  if (p.corner_globals.empty() && p.noncorner_globals.empty())
    throw Error(kNotAdjacent, "substructures share no interface dofs");
  const auto& Ai = md.subs[si].diag;
  const auto& Aj = md.subs[sj].diag;
  for (i64 g : p.noncorner_globals) {
    const double di = Ai[md.maps.local_of(g, si)];
    const double dj = Aj[md.maps.local_of(g, sj)];
    p.rho_i.push_back(di / (di + dj));
  }
  // floating: neither side holds a Dirichlet-eliminated node-component
  p.floating = !md.sub_constrained[si] && !md.sub_constrained[sj];
  return p;
}

std::vector<double> rigid_modes(const Model& md, const std::vector<i64>& dofs, int* nmodes) {
  // free dof -> (node, comp): invert md.dof once per call (small lists)
  const int nc = md.mesh.ncomp;
  const int nm = nc == 1 ? 1 : 6;
  *nmodes = nm;
  const std::size_t n = dofs.size();
  std::vector<double> z(nm * n, 0.0);
  static thread_local const Model* cached = nullptr;
  static thread_local std::vector<i64> inv;
  if (cached != &md || inv.size() != std::size_t(md.free_count)) {
    inv.assign(md.free_count, -1);
    for (std::size_t t = 0; t < md.dof.size(); ++t)
      if (md.dof[t] >= 0) inv[md.dof[t]] = static_cast<i64>(t);
    cached = &md;
  }
  double cen[3] = {0, 0, 0};
  for (std::size_t t = 0; t < n; ++t) {
    double x[3];
    md.mesh.coords(static_cast<int>(inv[dofs[t]] / nc), x);
    for (int a = 0; a < 3; ++a) cen[a] += x[a] / double(n);
  }
  for (std::size_t t = 0; t < n; ++t) {
    const i64 nccomp = inv[dofs[t]];
    const int node = static_cast<int>(nccomp / nc), c = static_cast<int>(nccomp % nc);
    if (nc == 1) {
      z[t] = 1.0;
      continue;
    }
    double x[3];
    md.mesh.coords(node, x);
    for (int a = 0; a < 3; ++a) x[a] -= cen[a];
    z[std::size_t(c) * n + t] = 1.0;  // translations
    // rotations: about z (-y, x, 0), about x (0, -z, y), about y (z, 0, -x)
    const double rz[3] = {-x[1], x[0], 0}, rx[3] = {0, -x[2], x[1]}, ry[3] = {x[2], 0, -x[0]};
    z[3 * n + t] = rz[c];
    z[4 * n + t] = rx[c];
    z[5 * n + t] = ry[c];
  }
  // modified Gram-Schmidt (twice)
  for (int pass = 0; pass < 2; ++pass)
    for (int a = 0; a < nm; ++a) {
      for (int b = 0; b < a; ++b) {
        double d = 0;
        for (std::size_t t = 0; t < n; ++t) d += z[a * n + t] * z[b * n + t];
        for (std::size_t t = 0; t < n; ++t) z[a * n + t] -= d * z[b * n + t];
      }
      double nn = 0;
      for (std::size_t t = 0; t < n; ++t) nn += z[a * n + t] * z[a * n + t];
      nn = std::sqrt(nn);
      for (std::size_t t = 0; t < n; ++t) z[a * n + t] /= nn;
    }
  return z;
}

// ============================================================================
// Lanczos condition estimate (pcg.cpp:11-26): eigenvalues of the symmetric
// tridiagonal by implicit QL (host; tiny).
// ============================================================================
double lanczos_condition_estimate(const std::vector<double>& alphas,
                                  const std::vector<double>& betas) {
  const int n = static_cast<int>(alphas.size());
  if (n == 0) return 1.0;
  std::vector<double> d(n), e(n, 0.0);
  d[0] = 1.0 / alphas[0];
  for (int j = 1; j < n; ++j) {
    d[j] = 1.0 / alphas[j] + betas[j - 1] / alphas[j - 1];
    e[j - 1] = std::sqrt(betas[j - 1]) / alphas[j - 1];
  }
  // tqli (eigenvalues only)
  for (int l = 0; l < n; ++l) {
    int iter = 0, m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
        if (std::abs(e[m]) <= std::numeric_limits<double>::epsilon() * dd) break;
      }
      if (m != l) {
        if (++iter > 60) break;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + (g >= 0 ? std::abs(r) : -std::abs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i], b = c * e[i];
          e[i + 1] = (r = std::hypot(f, g));
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          d[i + 1] = g + (p = s * r);
          g = c * r - b;
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  const double lo = *std::min_element(d.begin(), d.end());
  const double hi = *std::max_element(d.begin(), d.end());
  return lo > 0 ? hi / lo : std::numeric_limits<double>::infinity();
}

HaloPlan halo_plan(const Model& m, const std::vector<int>& owner, int me, int world) {
  HaloPlan H;
  const i64 n = static_cast<i64>(m.maps.interface_dofs.size());
  std::vector<std::vector<int>> ranks(n);
  for (i64 i = 0; i < n; ++i) {
    const i64 g = m.maps.interface_dofs[i];
    for (i64 t = m.maps.copy_ptr[g]; t < m.maps.copy_ptr[g + 1]; ++t) ranks[i].push_back(owner.at(m.maps.copy_sub[t]));
    std::sort(ranks[i].begin(), ranks[i].end());
    ranks[i].erase(std::unique(ranks[i].begin(), ranks[i].end()), ranks[i].end());
  }
  H.touched.assign(n, 0);
  H.owned.assign(n, 0);
  std::vector<std::vector<int>> per_peer(world);
  for (i64 i = 0; i < n; ++i) {
    if (!std::binary_search(ranks[i].begin(), ranks[i].end(), me)) continue;
    H.touched[i] = 1;
    H.owned[i] = ranks[i].front() == me;
    for (int r : ranks[i])
      if (r != me) per_peer.at(r).push_back(static_cast<int>(i));
  }
  H.peer_off.assign(1, 0);
  std::vector<int> slot(world, -1);
  for (int r = 0; r < world; ++r)
    if (!per_peer[r].empty()) {
      slot[r] = static_cast<int>(H.peers.size());
      H.peers.push_back(r);
      H.shared.insert(H.shared.end(), per_peer[r].begin(), per_peer[r].end());
      H.peer_off.push_back(static_cast<int>(H.shared.size()));
    }
  H.sum_ptr.assign(1, 0);
  for (i64 i = 0; i < n; ++i) {
    if (!H.touched[i] || ranks[i].size() < 2) continue;
    H.sum_dof.push_back(static_cast<int>(i));
    for (int r : ranks[i]) {
      if (r == me) {
        H.sum_src.push_back(-1);
        continue;
      }
      const auto b = H.shared.begin() + H.peer_off[slot[r]], e = H.shared.begin() + H.peer_off[slot[r] + 1];
      H.sum_src.push_back(static_cast<int>(std::lower_bound(b, e, static_cast<int>(i)) - H.shared.begin()));
    }
    H.sum_ptr.push_back(static_cast<int>(H.sum_src.size()));
  }
  return H;
}

}  // namespace b200
