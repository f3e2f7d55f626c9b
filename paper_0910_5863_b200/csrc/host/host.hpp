// Host-side substructuring for the B200 adaptive-BDDC path.
//
// This is the product's C++ host layer: it keeps the reference library's
// solver interface (mesh and substructuring input, constraint selection,
// change of variables) with flat, device-uploadable arrays instead of Eigen
// objects.  Each routine cites the reference file:line whose semantics it
// keeps (paths relative to /root/reference/proj/).  Index maps and glob
// ordering are bit-identical to the reference (checked against the oracle by
// tests/test_host_parity.py).
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "coarse_tree.hpp"

namespace b200 {

using i64 = std::int64_t;

// --- error taxonomy (core/include/bddc/types.hpp:21-63) ---------------------
enum Status : int {
  kOk = 0,
  kError = 1,
  kNotPositiveDefinite = 2,
  kDegenerateElement = 3,
  kCornerSelectionFailed = 4,
  kNullspaceInclusionViolated = 5,
  kSingularGram = 6,
  kNotAdjacent = 7,
  kBadProblemSpec = 8,
  kMaxIterations = 9,
  kCudaError = 10,
  kUnsupported = 11,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

enum Physics : int { kScalar = 0, kElasticity = 1 };
inline int components(int physics) { return physics == kScalar ? 1 : 3; }

enum Face : int { kXMin = 0, kXMax, kYMin, kYMax, kZMin, kZMax };

struct Material {  // mesh.hpp:17-21
  double conductivity = 1.0, youngs = 1.0, poisson = 0.3;
};
struct Region {  // mesh.hpp:25-30 (half-open element box)
  int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  int material = 0;
};
struct DirichletSpec {  // problem.hpp:23-26
  int face = kXMin;
  bool constrained[3] = {true, true, true};
};
struct LoadSpec {  // problem.hpp:28-32
  int face = kXMax;
  double traction[3] = {0, 0, 0};
  double flux = 0;
};

struct Problem {  // problem.hpp:43-53 + per-element coefficient extension
  int subdomains[3] = {1, 1, 1};
  int elements_per_edge = 1;
  int physics = kScalar;
  std::map<int, Material> materials{{0, Material{}}};
  std::vector<Region> regions;
  std::vector<DirichletSpec> dirichlet;
  std::vector<LoadSpec> loads;
  double body_force[3] = {0, 0, 0};
  double source = 0;
  double tolerance = 1e-8;
  int max_iterations = 500;
  std::vector<double> element_scale;  // empty = 1 everywhere
};

/// Seeded coefficient fields of BASELINE.json configs 2-5.
std::vector<double> element_scale_for(int config, const int ne[3], std::uint64_t seed);
/// BASELINE.json configs[config-1]; subdomains/epe override for shrunken parity cases.
Problem baseline_problem(int config, std::uint64_t seed, const int* subdomains_override,
                         int epe_override);

// --- mesh / decomposition (mesh.cpp:9-82) ------------------------------------
struct Mesh {
  int physics = kScalar;
  int ncomp = 1;
  int ne[3] = {0, 0, 0}, np[3] = {0, 0, 0};
  int sub[3] = {1, 1, 1};
  int epe = 1;
  double h = 1.0;
  std::vector<int> element_material;
  std::vector<double> element_scale;
  int node_count() const { return np[0] * np[1] * np[2]; }
  int element_count() const { return ne[0] * ne[1] * ne[2]; }
  int node_id(int i, int j, int k) const { return (k * np[1] + j) * np[0] + i; }
  void coords(int node, double* x) const {
    x[0] = (node % np[0]) * h;
    x[1] = ((node / np[0]) % np[1]) * h;
    x[2] = (node / (np[0] * np[1])) * h;
  }
  /// Sorted sharing set of a node (decompose_cube, mesh.cpp:70-80).
  void sharers(int node, std::vector<int>& out) const;
};

struct CSR {
  int n = 0;
  std::vector<int> ptr, idx;
  std::vector<double> val;
  double diag(int r) const;
};

struct Subdomain {  // assemble.hpp:41-51
  int id = 0;
  std::vector<int> nodes;        // ascending global node ids
  std::vector<i64> global_dof;   // local dof -> global free dof
  int origin[3] = {0, 0, 0};     // first element (i, j, k) of the subdomain block
  std::vector<int> lnode;        // local node grid (x fastest) * ncomp + c -> local dof, -1 if eliminated
  std::vector<double> diag;      // diagonal of the local stiffness (same summation order as A)
  mutable CSR A;                 // full symmetric local stiffness, built on demand (Model::matrix)
  mutable bool have_A = false;
  std::vector<double> load;
  std::vector<int> interior, boundary;  // spaces.cpp:119-125 (local ids, ascending)
  int dim() const { return static_cast<int>(global_dof.size()); }
};

// --- globs (globs.hpp:15-44) --------------------------------------------------
enum GlobKind : int { kCorner = 0, kEdge = 1, kFace = 2 };
struct Glob {
  int kind = kFace;
  std::vector<int> nodes;       // ascending
  std::vector<int> subdomains;  // ascending sharing set
};

struct Maps {  // spaces.hpp:23-43 (flat CSR forms)
  std::vector<i64> w_offset;
  i64 w_dim = 0;
  std::vector<i64> copy_ptr;            // global dof -> [copy_ptr[g], copy_ptr[g+1])
  std::vector<int> copy_sub;            // copy subdomain (ascending per dof)
  std::vector<int> copy_local;          // copy local dof
  std::vector<i64> interface_dofs;
  std::vector<i64> global_to_interface;
  i64 corner_dof_count = 0, wc_dim = 0;
  std::vector<std::vector<i64>> local_to_wc;
  std::vector<i64> corner_dof_of_global;
  int local_of(i64 g, int s) const;     // local copy of dof g in s, or -1
};

struct Average {  // constraints.hpp:23-27
  int glob = 0;
  std::vector<double> weights;
  int adaptive = 0;
};

struct GlobTransform {  // transform.hpp:20-27, compact form
  int glob = 0;
  int rank = 0;
  int n = 0;
  std::vector<int> perm;   // QR column pivots: t.row(perm[i]) = t_perm.row(i)
  std::vector<double> D;   // rank x n row-major: the dense rows t_perm[0:rank, :]
  /// Full basis change t (n x n row-major), for checks: unit rows t[perm[i]][i], i >= rank.
  std::vector<double> dense_t() const;
};

struct PivotedQr {  // dense_eig.hpp:20-29 (row-major m x n r, m x m q)
  int m = 0, n = 0, rank = 0;
  std::vector<double> q, r;
  std::vector<int> perm;
};
PivotedQr pivoted_qr(const std::vector<double>& a_rowmajor, int m, int n,
                     double rel_drop_tol = 1e-8, bool want_q = true);

/// Everything the host knows about one problem instance.
struct Model {
  Problem spec;
  Mesh mesh;
  std::vector<i64> dof;  // node*ncomp+c -> free dof or -1 (assemble.cpp:101-141)
  i64 free_count = 0;
  std::vector<Subdomain> subs;
  std::vector<Glob> globs;
  int classification_corners = 0;
  Maps maps;
  std::vector<std::vector<i64>> glob_dofs;   // glob_free_dofs per glob (cached)
  std::vector<std::vector<int>> sub_globs;   // globs containing each subdomain, ascending
  std::vector<char> sub_constrained;         // subdomain holds a Dirichlet dof
  // reference element matrices (one per material, ed x ed row-major, ed = 8 ncomp)
  // and the per-element index into them (assemble.cpp:145-169: congruent elements)
  std::vector<std::vector<double>> ke_ref;
  std::vector<int> element_ke;

  void build(const Problem& p);  // experiment.cpp:116-128
  /// Local stiffness of substructure s (assemble.cpp:202-292); the device path
  /// assembles the dense fronts itself, the CSR is built only when asked for.
  const CSR& matrix(int s) const;
  std::vector<i64> glob_free_dofs(int gi) const;  // constraints.cpp:25-32
  std::vector<int> corner_nodes() const;
  i64 count(int kind) const;
};

// --- constraints (constraints.cpp, transform.cpp) ----------------------------
struct ConstraintSet {
  std::vector<Average> averages;
  i64 row_count(const Model& m) const;                       // constraints.cpp:11-16
  std::vector<std::vector<int>> by_glob(std::size_t n) const;  // :18-23
};
ConstraintSet arithmetic_constraints(const Model& m, bool edges, bool faces);  // :34-59
bool add_average(ConstraintSet& cs, Average avg);                              // :61-76
/// The rank test of add_average: `w` is nonzero and independent of `existing`
/// (same glob); pivoted QR, tolerance 1e-8 (constraints.cpp:61-76).
bool average_admissible(const std::vector<const std::vector<double>*>& existing, const std::vector<double>& w);
GlobTransform build_glob_transform(int glob, const std::vector<double>& rows, int r_in,
                                   int n);  // transform.cpp:51-90
/// Kernel basis of a glob's averages, n x (n-rank) row-major (pair.cpp:167-188).
std::vector<double> glob_kernel(const std::vector<double>* rows, int r_in, int n, int* cols);
/// The same basis in compact form: column c has a unit entry at row perm[r+c]
/// and the values neg_top[a*(n-r)+c] at rows perm[a], a < r.
struct KernelCompact {
  int n = 0, r = 0;
  std::vector<int> perm;
  std::vector<double> neg_top;
};
KernelCompact glob_kernel_compact(const std::vector<double>* rows, int r_in, int n);

/// Change of variables restricted to the interface: per subdomain the
/// constrained glob blocks (local boundary positions + t), and per
/// (glob, explicit dof) the W^c group (transform.cpp:94-149).
struct ChangeOfVariables {
  std::vector<GlobTransform> transforms;
  std::vector<std::vector<i64>> groups;       // W^c ids, anchor first
  std::vector<std::vector<int>> group_subs;   // member subdomains
  std::vector<std::vector<int>> group_local;  // member local dofs
};
ChangeOfVariables change_of_variables(const ConstraintSet& cs, const Model& m);

/// Leaves of the primal tree over ALL substructures (coarse_tree.hpp): the
/// primal unknowns each substructure holds (corner dofs by corner id, then one
/// unknown per explicit-dof group of `cov`, numbered corner_dof_count + group)
/// and its lattice position; `bounds` receives every unknown's bounding box.
/// Global host data: every rank of a sharded engine computes the same lists.
std::vector<CoarseLeaf> primal_leaves(const Model& md, const ChangeOfVariables& cov, CoarseBounds* bounds);

// --- pairs (pair.cpp:67-209) ---------------------------------------------------
struct PairIndex {
  int si = 0, sj = 0;
  std::vector<int> shared_globs;
  std::vector<i64> corner_globals, noncorner_globals, outer_i, outer_j;
  std::vector<double> rho_i;
  std::vector<int> glob_offset;   // per shared glob: slot offset
  std::vector<int> glob_size;
  bool floating = false;          // no Dirichlet dof in either side
};
std::vector<std::pair<int, int>> face_pairs(const Model& m);  // adaptive.cpp:12-20
PairIndex build_pair_index(const Model& m, int si, int sj);

/// Rigid-body (null) modes of a floating pair restricted to the listed dofs:
/// returns nmodes x ndofs row-major, orthonormalized.
std::vector<double> rigid_modes(const Model& m, const std::vector<i64>& dofs, int* nmodes);

/// Interface halo of one rank of a sharded run: the interface
/// dofs it touches (a copy in one of its substructures), the ones it owns
/// (lowest rank holding a copy), per peer the shared dofs in ascending
/// interface order, and per shared dof the contributions in ascending rank
/// order (sum_src < 0: this rank's own partial; else a position in the
/// per-peer concatenated receive buffer).  shard.py HaloPlan is the same plan.
struct HaloPlan {
  std::vector<int> peers, peer_off, shared;
  std::vector<char> touched, owned;
  std::vector<int> sum_dof, sum_ptr, sum_src;
};
HaloPlan halo_plan(const Model& m, const std::vector<int>& owner, int rank, int world);

double lanczos_condition_estimate(const std::vector<double>& alphas,
                                  const std::vector<double>& betas);  // pcg.cpp:11-26

}  // namespace b200
