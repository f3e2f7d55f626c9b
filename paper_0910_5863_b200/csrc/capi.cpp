// C ABI (include/bddc_b200.h) over the host model and the device engine.
#include "../../include/bddc_b200.h"

#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>

#include "cuda/engine.hpp"
#include "host/export.hpp"
#include "host/host.hpp"

using namespace b200;

struct bddc_b200 {
  Model model;
  ConstraintSet cs;
  std::unique_ptr<Engine> engine;
  EnrichOutcome last_enrich;
  bool analysed = false;
  double t = -1.0;          // stabilization parameter of the last setup (bddc_operator.hpp:32-35)
  CsrMatrix stabilized;     // cached by bddc_b200_stabilized (query, then fill)
  bool have_stabilized = false;
};

namespace {
thread_local std::string g_last_error;

template <class F>
int guarded(F f) {
  try {
    f();
    return BDDC_B200_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BDDC_B200_ERROR;
  }
}

Engine& engine(bddc_b200_t* h) {
  if (!h->engine) h->engine.reset(new Engine(h->model));
  return *h->engine;
}

void ensure_analysis(bddc_b200_t* h) {
  if (!h->analysed) {
    engine(h).analysis();
    h->analysed = true;
  }
}
}  // namespace

extern "C" {

const char* bddc_b200_last_error(void) { return g_last_error.c_str(); }

int bddc_b200_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int bddc_b200_set_device(int device) {
  return guarded([&] {
    const cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) throw Error(kCudaError, cudaGetErrorString(e));
  });
}

int bddc_b200_nccl_unique_id(unsigned char* id128) {
  return guarded([&] { nccl_unique_id(id128); });
}

int bddc_b200_shard_nccl(bddc_b200_t* h, const unsigned char* id128, int rank, int world, const int* owner) {
  return guarded([&] {
    std::vector<int> own(owner, owner + h->model.subs.size());
    engine(h).set_shard(make_nccl_comm(id128, rank, world), own);
  });
}

int bddc_b200_shard_loopback(bddc_b200_t* h, int group, int rank, int world, const int* owner) {
  return guarded([&] {
    std::vector<int> own(owner, owner + h->model.subs.size());
    engine(h).set_shard(make_loopback_comm(group, rank, world), own);
  });
}

int bddc_b200_subdomain_lattice(const bddc_b200_t* h, int64_t* dims3) {
  return guarded([&] {
    for (int a = 0; a < 3; ++a) dims3[a] = h->model.mesh.sub[a];
  });
}

int bddc_b200_create(const bddc_b200_problem* p, bddc_b200_t** out) {
  return guarded([&] {
    Problem pr;
    for (int a = 0; a < 3; ++a) pr.subdomains[a] = p->subdomains[a];
    pr.elements_per_edge = p->elements_per_edge;
    pr.physics = p->physics;
    pr.materials.clear();
    pr.materials[0] = Material{};
    for (int i = 0; i < p->n_materials; ++i)
      pr.materials[p->material_id[i]] = Material{p->conductivity[i], p->youngs[i], p->poisson[i]};
    for (const auto& [id, mat] : pr.materials) {  // problem.cpp:176-187
      if (pr.physics == kScalar && mat.conductivity <= 0) throw Error(kBadProblemSpec, "conductivity must be positive");
      if (pr.physics == kElasticity && (mat.youngs <= 0 || mat.poisson <= 0 || mat.poisson >= 0.5))
        throw Error(kBadProblemSpec, "bad elasticity material");
    }
    for (int i = 0; i < p->n_regions; ++i) {
      Region r;
      const int* b = p->region_box + 6 * i;
      r.lo[0] = b[0]; r.hi[0] = b[1]; r.lo[1] = b[2]; r.hi[1] = b[3]; r.lo[2] = b[4]; r.hi[2] = b[5];
      r.material = p->region_material[i];
      pr.regions.push_back(r);
    }
    for (int i = 0; i < p->n_dirichlet; ++i) {
      DirichletSpec d;
      d.face = p->dirichlet_face[i];
      for (int c = 0; c < 3; ++c) d.constrained[c] = p->dirichlet_components[3 * i + c] != 0;
      pr.dirichlet.push_back(d);
    }
    for (int i = 0; i < p->n_loads; ++i) {
      LoadSpec l;
      l.face = p->load_face[i];
      for (int c = 0; c < 3; ++c) l.traction[c] = p->load_traction[3 * i + c];
      l.flux = p->load_flux[i];
      pr.loads.push_back(l);
    }
    for (int c = 0; c < 3; ++c) pr.body_force[c] = p->body_force[c];
    pr.source = p->source;
    pr.tolerance = p->tolerance > 0 ? p->tolerance : 1e-8;
    pr.max_iterations = p->max_iterations > 0 ? p->max_iterations : 500;
    if (p->element_scale) {
      const std::size_t ne = std::size_t(p->subdomains[0]) * p->subdomains[1] * p->subdomains[2] *
                             p->elements_per_edge * p->elements_per_edge * p->elements_per_edge;
      pr.element_scale.assign(p->element_scale, p->element_scale + ne);
    }
    auto h = std::make_unique<bddc_b200>();
    h->model.build(pr);
    *out = h.release();
  });
}

int bddc_b200_create_config(int config, uint64_t seed, const int* sub, int epe, bddc_b200_t** out) {
  return guarded([&] {
    auto h = std::make_unique<bddc_b200>();
    h->model.build(baseline_problem(config, seed, sub, epe));
    *out = h.release();
  });
}

void bddc_b200_destroy(bddc_b200_t* h) { delete h; }

int bddc_b200_structure_get(const bddc_b200_t* h, bddc_b200_structure* o) {
  return guarded([&] {
    const Model& m = h->model;
    o->dofs = i64(m.mesh.node_count()) * m.mesh.ncomp;
    o->free_dofs = m.free_count;
    o->interface_dofs = static_cast<i64>(m.maps.interface_dofs.size());
    o->corners = m.count(kCorner);
    o->classification_corners = m.classification_corners;
    o->edges = m.count(kEdge);
    o->faces = m.count(kFace);
    o->coarse_space_dim = m.maps.wc_dim;
    o->subdomains = static_cast<i64>(m.subs.size());
    o->w_dim = m.maps.w_dim;
    o->elements = m.mesh.element_count();
  });
}

int bddc_b200_interface_dofs(const bddc_b200_t* h, int64_t* out) {
  return guarded([&] {
    const auto& v = h->model.maps.interface_dofs;
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  });
}

int bddc_b200_subdomain_dim(const bddc_b200_t* h, int s, int64_t* dim) {
  return guarded([&] { *dim = h->model.subs.at(s).dim(); });
}

int bddc_b200_local_to_wc(const bddc_b200_t* h, int s, int64_t* out) {
  return guarded([&] {
    const auto& v = h->model.maps.local_to_wc.at(s);
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  });
}

int bddc_b200_global_dof(const bddc_b200_t* h, int s, int64_t* out) {
  return guarded([&] {
    const auto& v = h->model.subs.at(s).global_dof;
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  });
}

int bddc_b200_element_scale(const bddc_b200_t* h, double* out) {
  return guarded([&] {
    const Mesh& m = h->model.mesh;
    for (int e = 0; e < m.element_count(); ++e) out[e] = m.element_scale.empty() ? 1.0 : m.element_scale[e];
  });
}

int bddc_b200_subdomain_matrix(const bddc_b200_t* h, int s, int64_t* nnz, int64_t* ptr, int64_t* idx, double* val,
                               double* load) {
  return guarded([&] {
    const Subdomain& S = h->model.subs.at(s);
    const CSR& A = h->model.matrix(s);
    *nnz = static_cast<int64_t>(A.idx.size());
    if (!ptr) return;
    for (int r = 0; r <= A.n; ++r) ptr[r] = A.ptr[r];
    for (std::size_t t = 0; t < A.idx.size(); ++t) {
      idx[t] = A.idx[t];
      val[t] = A.val[t];
    }
    for (int l = 0; l < S.dim(); ++l) load[l] = S.load[l];
  });
}

int bddc_b200_leaf_front(bddc_b200_t* h, int s, int64_t* ld, double* front, int64_t* pos) {
  return guarded([&] {
    if (s < 0 || s >= static_cast<int>(h->model.subs.size())) throw Error(kError, "substructure out of range");
    std::vector<double> f;
    std::vector<int> p;
    int n = 0;
    engine(h).leaf_front(s, front ? &f : nullptr, &p, &n);
    *ld = n;
    if (!front) return;
    std::memcpy(front, f.data(), f.size() * sizeof(double));
    for (std::size_t i = 0; i < p.size(); ++i) pos[i] = p[i];
  });
}

int bddc_b200_glob_count(const bddc_b200_t* h, int64_t* n) {
  return guarded([&] { *n = static_cast<int64_t>(h->model.globs.size()); });
}

int bddc_b200_glob_info(const bddc_b200_t* h, int g, int* kind, int64_t* nn, int64_t* nsub) {
  return guarded([&] {
    const Glob& gl = h->model.globs.at(g);
    *kind = gl.kind;
    *nn = static_cast<int64_t>(gl.nodes.size());
    *nsub = static_cast<int64_t>(gl.subdomains.size());
  });
}

int bddc_b200_glob_nodes(const bddc_b200_t* h, int g, int64_t* nodes, int64_t* subs) {
  return guarded([&] {
    const Glob& gl = h->model.globs.at(g);
    for (std::size_t i = 0; i < gl.nodes.size(); ++i) nodes[i] = gl.nodes[i];
    for (std::size_t i = 0; i < gl.subdomains.size(); ++i) subs[i] = gl.subdomains[i];
  });
}

int bddc_b200_constraints_arithmetic(bddc_b200_t* h, int edges, int faces) {
  return guarded([&] { h->cs = arithmetic_constraints(h->model, edges != 0, faces != 0); });
}

int bddc_b200_constraints_clear(bddc_b200_t* h) {
  return guarded([&] { h->cs = ConstraintSet{}; });
}

int bddc_b200_constraint_add(bddc_b200_t* h, int glob, const double* weights, int64_t n, int adaptive,
                             int* kept) {
  return guarded([&] {
    if (glob < 0 || glob >= static_cast<int>(h->model.globs.size()))
      throw Error(kBadProblemSpec, "constraint_add: glob index out of range");
    const std::size_t nd = h->model.glob_dofs[glob].size();
    if (static_cast<std::size_t>(n) != nd)
      throw Error(kBadProblemSpec, "constraint_add: weights length " + std::to_string(n) +
                                       " != free dofs of the glob " + std::to_string(nd));
    Average a;
    a.glob = glob;
    a.weights.assign(weights, weights + n);
    a.adaptive = adaptive;
    const bool k = add_average(h->cs, std::move(a));
    if (kept) *kept = k ? 1 : 0;
  });
}

int bddc_b200_constraint_rows(const bddc_b200_t* h, int64_t* rows) {
  return guarded([&] { *rows = h->cs.row_count(h->model); });
}

int bddc_b200_constraint_count(const bddc_b200_t* h, int64_t* n) {
  return guarded([&] { *n = static_cast<int64_t>(h->cs.averages.size()); });
}

int bddc_b200_constraint_get(const bddc_b200_t* h, int a, int* glob, int64_t* nw, double* w) {
  return guarded([&] {
    const Average& av = h->cs.averages.at(a);
    *glob = av.glob;
    *nw = static_cast<int64_t>(av.weights.size());
    if (w) std::memcpy(w, av.weights.data(), av.weights.size() * sizeof(double));
  });
}

int bddc_b200_analysis(bddc_b200_t* h) {
  return guarded([&] {
    h->analysed = false;
    ensure_analysis(h);
  });
}

int bddc_b200_enrich(bddc_b200_t* h, double tau, int max_vectors, int keep_edge, int fixed_count,
                     int indicator_only, double* omega_tilde) {
  return guarded([&] {
    ensure_analysis(h);
    EnrichOptions o;
    o.tau = tau;
    o.max_vectors = max_vectors;
    o.keep_edge_constraints = keep_edge != 0;
    o.fixed_count = fixed_count;
    o.indicator_only = indicator_only != 0;
    h->last_enrich = engine(h).enrich(h->cs, o);
    if (omega_tilde) *omega_tilde = h->last_enrich.omega_tilde;
  });
}

int bddc_b200_pair_count(const bddc_b200_t* h, int64_t* n) {
  return guarded([&] { *n = static_cast<int64_t>(h->last_enrich.pairs.size()); });
}

int bddc_b200_pair_report(const bddc_b200_t* h, int k, int* si, int* sj, int* enforced, double* omega_next,
                          int* saturated, int64_t* n_eig, double* eig) {
  return guarded([&] {
    const PairReport& r = h->last_enrich.pairs.at(k);
    *si = r.si;
    *sj = r.sj;
    *enforced = r.enforced;
    *omega_next = r.omega_next;
    *saturated = r.saturated ? 1 : 0;
    *n_eig = static_cast<int64_t>(r.eigenvalues.size());
    if (eig) std::memcpy(eig, r.eigenvalues.data(), r.eigenvalues.size() * sizeof(double));
  });
}

int bddc_b200_setup_preconditioner(bddc_b200_t* h) { return bddc_b200_setup_preconditioner_t(h, -1.0); }

int bddc_b200_setup_preconditioner_t(bddc_b200_t* h, double t) {
  return guarded([&] {
    ensure_analysis(h);
    engine(h).set_constraints(h->cs);
    h->t = t;
    h->have_stabilized = false;
  });
}

int bddc_b200_stabilization_t(bddc_b200_t* h, double* t) {
  return guarded([&] { *t = stabilization_t(h->model, change_of_variables(h->cs, h->model), h->t); });
}

int bddc_b200_stabilized(bddc_b200_t* h, int64_t* n, int64_t* nnz, int64_t* ptr, int64_t* idx, double* val) {
  return guarded([&] {
    if (!h->have_stabilized) {
      h->stabilized = stabilized_operator(h->model, change_of_variables(h->cs, h->model), h->t, nullptr);
      h->have_stabilized = true;
    }
    const CsrMatrix& a = h->stabilized;
    *n = a.rows;
    *nnz = static_cast<int64_t>(a.val.size());
    if (ptr) {
      std::memcpy(ptr, a.ptr.data(), a.ptr.size() * sizeof(int64_t));
      std::memcpy(idx, a.idx.data(), a.idx.size() * sizeof(int64_t));
      std::memcpy(val, a.val.data(), a.val.size() * sizeof(double));
      h->stabilized = CsrMatrix{};  // filled: release the cache
      h->have_stabilized = false;
    }
  });
}

int bddc_b200_glob_transform(bddc_b200_t* h, int glob, int* rank, int64_t* n, double* t) {
  return guarded([&] {
    const ChangeOfVariables cov = change_of_variables(h->cs, h->model);
    for (const GlobTransform& gt : cov.transforms)
      if (gt.glob == glob) {
        *rank = gt.rank;
        *n = gt.n;
        if (t) {
          const std::vector<double> d = gt.dense_t();
          std::memcpy(t, d.data(), d.size() * sizeof(double));
        }
        return;
      }
    *rank = 0;
    *n = static_cast<int64_t>(h->model.glob_dofs.at(glob).size());
    if (t)
      for (int64_t i = 0; i < *n * *n; ++i) t[i] = (i % (*n + 1)) == 0 ? 1.0 : 0.0;
  });
}

int bddc_b200_halo_plan(const bddc_b200_t* h, const int* owner, int rank, int world, int64_t* n_peers,
                        int64_t* n_shared, int* peers, int* peer_off, int* shared, int* touched, int* owned) {
  return guarded([&] {
    const std::vector<int> own(owner, owner + h->model.subs.size());
    const HaloPlan p = halo_plan(h->model, own, rank, world);
    *n_peers = static_cast<int64_t>(p.peers.size());
    *n_shared = static_cast<int64_t>(p.shared.size());
    if (!peers) return;
    std::copy(p.peers.begin(), p.peers.end(), peers);
    std::copy(p.peer_off.begin(), p.peer_off.end(), peer_off);
    std::copy(p.shared.begin(), p.shared.end(), shared);
    for (std::size_t i = 0; i < p.touched.size(); ++i) {
      touched[i] = p.touched[i];
      owned[i] = p.owned[i];
    }
  });
}

int bddc_b200_primal_tree_plan(const bddc_b200_t* h, const int* owner, int rank, int world, int depth,
                               int64_t* depth_used, int64_t* n_top, int64_t* n_fronts, int64_t* n_own, int* top,
                               int* front_level, int* front_ptr, int* front_own) {
  return guarded([&] {
    const Model& m = h->model;
    const std::vector<int> own(owner, owner + m.subs.size());
    const ChangeOfVariables cov = change_of_variables(h->cs, m);
    CoarseBounds bounds;
    const std::vector<CoarseLeaf> all = primal_leaves(m, cov, &bounds);
    const int n_primal = static_cast<int>(m.maps.corner_dof_count + cov.groups.size());
    int maxd = coarse_tree_max_depth(m.mesh.sub);
    if (world > 1) maxd = coarse_tree_shard_depth(m.mesh.sub, own, maxd);
    const int d = std::max(0, std::min(depth, maxd));
    std::vector<CoarseLeaf> mine;
    for (std::size_t s = 0; s < all.size(); ++s)
      if (world <= 1 || own[s] == rank) mine.push_back(all[s]);
    const CoarseTree t = plan_coarse_tree(mine, m.mesh.sub, n_primal, d, 12288, true, world > 1 ? &bounds : nullptr);
    *depth_used = d;
    *n_top = static_cast<int64_t>(t.top.size());
    int64_t nf = 0, no = 0;
    for (const auto& L : t.levels)
      for (const auto& f : L.fronts) {
        ++nf;
        no += static_cast<int64_t>(f.own.size());
      }
    *n_fronts = nf;
    *n_own = no;
    if (!top) return;
    std::copy(t.top.begin(), t.top.end(), top);
    int64_t fi = 0, at = 0;
    front_ptr[0] = 0;
    for (std::size_t l = 0; l < t.levels.size(); ++l)
      for (const auto& f : t.levels[l].fronts) {
        front_level[fi] = static_cast<int>(l);
        std::copy(f.own.begin(), f.own.end(), front_own + at);
        at += static_cast<int64_t>(f.own.size());
        front_ptr[++fi] = static_cast<int>(at);
      }
  });
}

int bddc_b200_export_matrix_market(bddc_b200_t* h, const char* stem) {
  return guarded([&] {
    const ChangeOfVariables cov = change_of_variables(h->cs, h->model);
    write_matrix_market(std::string(stem) + "_stabilized.mtx", stabilized_operator(h->model, cov, h->t, nullptr),
                        true);
    write_matrix_market(std::string(stem) + "_constraints.mtx",
                        transformed_constraint_matrix(cov, h->model.maps.wc_dim), false);
  });
}

int bddc_b200_interface_size(const bddc_b200_t* h, int64_t* n) {
  return guarded([&] { *n = static_cast<int64_t>(h->model.maps.interface_dofs.size()); });
}

int bddc_b200_schur_apply(bddc_b200_t* h, const double* x, double* y) {
  return guarded([&] {
    ensure_analysis(h);
    engine(h).schur_apply(x, y);
  });
}

int bddc_b200_precond_apply(bddc_b200_t* h, const double* r, double* z) {
  return guarded([&] { engine(h).precond_apply(r, z); });
}

int bddc_b200_restrict_residual(bddc_b200_t* h, const double* r, double* wc) {
  return guarded([&] { engine(h).restrict_residual(r, wc); });
}

int bddc_b200_coarse_solve(bddc_b200_t* h, const double* wc_residual, double* wc_out) {
  return guarded([&] { engine(h).coarse_solve(wc_residual, wc_out); });
}

int bddc_b200_prolong(bddc_b200_t* h, const double* wc, double* z) {
  return guarded([&] { engine(h).prolong(wc, z); });
}

int bddc_b200_operator_times(bddc_b200_t* h, int reps, double out[13]) {
  return guarded([&] {
    Engine& e = engine(h);
    const Engine::OpTimes t = e.time_operators(reps);
    const double v[13] = {t.schur,    t.precond,  t.restrict_,  t.leaf_fwd,         t.tree_fwd,
                          t.root,     t.tree_bwd, t.leaf_bwd,   t.prolong,          t.sum_copies,
                          e.schur_bytes(), e.pcg_bytes_per_iteration() - e.schur_bytes(), t.leaf_sweep_bytes};
    std::memcpy(out, v, sizeof(v));
  });
}

int bddc_b200_rhs(bddc_b200_t* h, double* out) {
  return guarded([&] {
    ensure_analysis(h);
    engine(h).rhs(out);
  });
}

int bddc_b200_recover(bddc_b200_t* h, const double* u, double* out) {
  return guarded([&] {
    ensure_analysis(h);
    engine(h).recover(u, out);
  });
}

int bddc_b200_pcg(bddc_b200_t* h, const double* b, double* x, double tol, int max_it, int prec_res,
                  bddc_b200_pcg_result* res, double* alphas, double* betas) {
  int capped = 0;
  const int rc = guarded([&] {
    const PcgOut o = engine(h).pcg(b, x, tol, max_it, prec_res != 0);
    res->iterations = o.iterations;
    res->relative_residual = o.relative_residual;
    res->condition_estimate = o.condition_estimate;
    res->converged = o.converged ? 1 : 0;
    if (alphas) std::memcpy(alphas, o.alphas.data(), o.alphas.size() * sizeof(double));
    if (betas) std::memcpy(betas, o.betas.data(), o.betas.size() * sizeof(double));
    capped = !o.converged;
  });
  if (rc == BDDC_B200_OK && capped) {
    g_last_error = "conjugate gradients did not reach the tolerance";
    return BDDC_B200_MAX_ITERATIONS;
  }
  return rc;
}

int bddc_b200_run_item(bddc_b200_t* h, const char* mode_c, double tau, int max_vectors, int keep_edge,
                       int base_faces, bddc_b200_row* row) {
  return guarded([&] {
    const std::string mode(mode_c);
    if (mode != "c" && mode != "c+e" && mode != "c+e+f" && mode != "c+e+f-3eigv" && mode != "adaptive")
      throw Error(kBadProblemSpec, "unknown constraint mode '" + mode + "'");
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    ensure_analysis(h);
    Engine& e = engine(h);
    const double t_an = e.times().analysis;
    const auto t1 = clk::now();
    // experiment.cpp:148-170
    const bool edges = mode != "c";
    const bool faces = mode == "c+e+f" || ((mode == "adaptive" || mode == "c+e+f-3eigv") && base_faces);
    h->cs = arithmetic_constraints(h->model, edges, faces);
    row->omega_tilde = std::numeric_limits<double>::quiet_NaN();
    double t_eig = 0;
    if (mode == "adaptive" || mode == "c+e+f-3eigv") {
      EnrichOptions o;
      o.keep_edge_constraints = keep_edge != 0;
      if (mode == "c+e+f-3eigv") {
        o.fixed_count = 3;
      } else {
        o.tau = tau;
        o.max_vectors = max_vectors;
      }
      h->last_enrich = e.enrich(h->cs, o);
      row->omega_tilde = h->last_enrich.omega_tilde;
      t_eig = e.times().eigen;
    }
    row->constraint_rows = h->cs.row_count(h->model);
    e.set_constraints(h->cs);
    const auto t2 = clk::now();
    const PcgOut o = e.pcg(nullptr, nullptr, h->model.spec.tolerance, h->model.spec.max_iterations, false);
    const auto t3 = clk::now();
    row->kappa = o.condition_estimate;
    row->iterations = o.iterations;
    row->converged = o.converged ? 1 : 0;
    row->seconds_analysis = t_an;
    row->seconds_factorization = std::chrono::duration<double>(t2 - t1).count();
    row->seconds_iterations = std::chrono::duration<double>(t3 - t2).count();
    row->seconds_total = row->seconds_analysis + row->seconds_factorization + row->seconds_iterations;
    row->seconds_eigen = t_eig;
    row->seconds_preconditioner = e.times().preconditioner;
    row->root_size = e.root_size();
    (void)t0;
  });
}

int bddc_b200_step(bddc_b200_t* h, const char* mode_c, double tau, int max_vectors, int keep_edge,
                   int base_faces, int e2e, double* u_free, bddc_b200_step_out* out) {
  return guarded([&] {
    const std::string mode(mode_c);
    if (mode != "c" && mode != "c+e" && mode != "c+e+f" && mode != "c+e+f-3eigv" && mode != "adaptive")
      throw Error(kBadProblemSpec, "unknown constraint mode '" + mode + "'");
    if (e2e && !u_free) throw Error(kBadProblemSpec, "e2e step needs a u_free buffer");
    StepSpec sp;
    sp.edges = mode != "c";
    sp.faces = mode == "c+e+f" || ((mode == "adaptive" || mode == "c+e+f-3eigv") && base_faces);
    sp.adaptive = mode == "adaptive";
    sp.fixed_count = mode == "c+e+f-3eigv" ? 3 : -1;
    sp.tau = tau;
    sp.max_vectors = max_vectors;
    sp.keep_edge = keep_edge != 0;
    sp.tol = h->model.spec.tolerance;
    sp.max_it = h->model.spec.max_iterations;
    sp.e2e = e2e != 0;
    Engine& e = engine(h);
    const StepOut o = e.step(sp, h->cs, u_free);
    h->analysed = true;
    out->seconds = o.seconds;
    out->setup_seconds = o.setup_seconds;
    out->solve_seconds = o.solve_seconds;
    out->h2d_bytes = o.h2d_bytes;
    out->d2h_bytes = o.d2h_bytes;
    out->launches = o.launches;
    out->constraint_rows = o.constraint_rows;
    out->omega_tilde = o.omega_tilde;
    out->iterations = o.pcg.iterations;
    out->kappa = o.pcg.condition_estimate;
    out->converged = o.pcg.converged ? 1 : 0;
    out->leaf_factor_seconds = e.times().leaf_factor;
    out->leaf_flops = e.times().flops_leaf;
  });
}

int64_t bddc_b200_launch_count(void) { return launch_count(); }

int bddc_b200_lanczos(const double* alphas, const double* betas, int64_t n, double* kappa) {
  return guarded([&] {
    std::vector<double> a(alphas, alphas + n), b(betas, betas + n);
    *kappa = lanczos_condition_estimate(a, b);
  });
}

int bddc_b200_times(const bddc_b200_t* h, double out[11]) {
  return guarded([&] {
    if (!h->engine) throw Error(kError, "no engine yet");
    const PhaseTimes& t = h->engine->times();
    out[0] = t.analysis;
    out[1] = t.eigen;
    out[2] = t.preconditioner;
    out[3] = t.pcg;
    out[4] = t.flops_leaf;
    out[5] = h->engine->leaf_front_bytes();
    out[6] = h->engine->schur_bytes();
    out[7] = h->engine->root_size();
    out[8] = t.leaf_factor;
    out[9] = t.pcg_iterations;
    out[10] = h->engine->pcg_bytes_per_iteration();
  });
}

}  // extern "C"
