/*
 * bddc_b200.h -- C ABI of the B200-native adaptive-BDDC hot path.
 *
 * The reference (/root/reference/proj) is a C++ class library with no FFI; its
 * two drop-in seams are the LinearOperator pair handed to pcg
 * (core/include/bddc/pcg.hpp:18,49-50) and the Factorization pImpl
 * (core/include/bddc/sparse.hpp:55-66).  Each entry point below names the
 * reference interface it replaces.  Plain pointers and sizes only; host
 * buffers are borrowed for the duration of a call; the handle owns all device
 * memory.  Every call returns a status code (BDDC_B200_*) mirroring the
 * reference's exception taxonomy (core/include/bddc/types.hpp:21-63);
 * bddc_b200_last_error() returns the message of the last failure.
 */
#ifndef BDDC_B200_H
#define BDDC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (types.hpp:21-63, pcg.hpp:40-45) */
#define BDDC_B200_OK 0
#define BDDC_B200_ERROR 1
#define BDDC_B200_NOT_POSITIVE_DEFINITE 2
#define BDDC_B200_DEGENERATE_ELEMENT 3
#define BDDC_B200_CORNER_SELECTION_FAILED 4
#define BDDC_B200_NULLSPACE_INCLUSION_VIOLATED 5
#define BDDC_B200_SINGULAR_GRAM 6
#define BDDC_B200_NOT_ADJACENT 7
#define BDDC_B200_BAD_PROBLEM_SPEC 8
#define BDDC_B200_MAX_ITERATIONS 9
#define BDDC_B200_CUDA_ERROR 10
#define BDDC_B200_UNSUPPORTED 11

typedef struct bddc_b200 bddc_b200_t;

/* Problem description: ProblemSpec (core/include/bddc/problem.hpp:43-53) plus
 * an optional per-element coefficient multiplier (element_scale, length =
 * element count, x-fastest element order; NULL = 1). */
typedef struct bddc_b200_problem {
  int subdomains[3];
  int elements_per_edge;
  int physics; /* 0 scalar, 1 elasticity (types.hpp:13) */
  int n_materials;
  const int* material_id;
  const double* conductivity;
  const double* youngs;
  const double* poisson;
  int n_regions;
  const int* region_box;      /* 6 per region: x0 x1 y0 y1 z0 z1 (half-open, problem.cpp:123-126) */
  const int* region_material;
  int n_dirichlet;
  const int* dirichlet_face;  /* 0 xmin 1 xmax 2 ymin 3 ymax 4 zmin 5 zmax */
  const int* dirichlet_components; /* 3 flags per entry */
  int n_loads;
  const int* load_face;
  const double* load_traction; /* 3 per load */
  const double* load_flux;
  double body_force[3];
  double source;
  double tolerance;
  int max_iterations;
  const double* element_scale;
} bddc_b200_problem;

/* StructureSummary (core/include/bddc/experiment.hpp:48-57) */
typedef struct bddc_b200_structure {
  int64_t dofs, free_dofs, interface_dofs;
  int64_t corners, classification_corners, edges, faces;
  int64_t coarse_space_dim; /* W^c dimension */
  int64_t subdomains, w_dim;
  int64_t elements;
} bddc_b200_structure;

/* PcgResult (core/include/bddc/pcg.hpp:28-34) */
typedef struct bddc_b200_pcg_result {
  int64_t iterations;
  double relative_residual;
  double condition_estimate;
  int converged;
} bddc_b200_pcg_result;

/* ResultRow (core/include/bddc/experiment.hpp:37-46) with device-timed phases */
typedef struct bddc_b200_row {
  double omega_tilde; /* NaN for non-eigenvalue modes */
  int64_t constraint_rows;
  double kappa;
  int64_t iterations;
  int converged;
  double seconds_analysis, seconds_factorization, seconds_iterations, seconds_total;
  double seconds_eigen, seconds_preconditioner; /* factorization = eigen + host constraints + preconditioner */
  int64_t root_size;
} bddc_b200_row;

const char* bddc_b200_last_error(void);
int bddc_b200_device_count(void);
/* Select the CUDA device used by handles created afterwards on this thread
 * (one process per GPU). */
int bddc_b200_set_device(int device);

/* Sharding over GPUs (one process or host thread per shard).
 * Call after create and before any device work.  owner[s] = rank owning
 * substructure s (one entry per substructure, e.g. shard.partition); face
 * pairs belong to the owner of their lower substructure.  Every rank then
 * returns the complete interface vectors, constraint set, root and solution.
 * NCCL: rank 0 makes the 128-byte id with bddc_b200_nccl_unique_id and shares
 * it; loopback: ranks are host threads of this process (tests), `group`
 * names the set of handles that exchange with each other. */
int bddc_b200_nccl_unique_id(unsigned char* id128);
int bddc_b200_shard_nccl(bddc_b200_t* h, const unsigned char* id128, int rank, int world, const int* owner);
int bddc_b200_shard_loopback(bddc_b200_t* h, int group, int rank, int world, const int* owner);
/* Interface halo plan of `rank` for the partition `owner` (host only; the
 * sharded engine's exchange): peers (ascending), per peer the shared interface
 * dofs (ascending, concatenated; peer_off has n_peers + 1 entries), and per
 * interface dof whether this rank touches / owns it.  Query the counts with
 * peers == NULL. */
int bddc_b200_halo_plan(const bddc_b200_t* h, const int* owner, int rank, int world, int64_t* n_peers,
                        int64_t* n_shared, int* peers, int* peer_off, int* shared, int* touched, int* owned);
/* Primal-tree plan of `rank` for the partition `owner` and the current
 * constraint set (host only; DESIGN.md sections 3.7 and 9): the nested
 * dissection of the primal unknowns that replaces the reference's single sparse
 * factorization of the auxiliary operator (bddc_operator.cpp:38-50).  top = the
 * unknowns of the top front (the same list on every rank; the only front that
 * is summed over the ranks); the fronts of the boxes inside this rank's block,
 * deepest level first, with the unknowns each eliminates (front_ptr has
 * n_fronts + 1 entries).  depth is clamped to what the lattice and the
 * partition allow (depth_used); world == 1 gives the single-GPU plan.  Query
 * the counts with top == NULL. */
int bddc_b200_primal_tree_plan(const bddc_b200_t* h, const int* owner, int rank, int world, int depth,
                               int64_t* depth_used, int64_t* n_top, int64_t* n_fronts, int64_t* n_own, int* top,
                               int* front_level, int* front_ptr, int* front_own);
/* Substructure lattice (nx, ny, nz), substructure ids x-fastest (mesh.cpp:68-70). */
int bddc_b200_subdomain_lattice(const bddc_b200_t* h, int64_t* dims3);

/* Build mesh, decomposition, Dirichlet map, substructure matrices, globs,
 * corners and embeddings (experiment.cpp:116-128; support.hpp:89-100). */
int bddc_b200_create(const bddc_b200_problem* problem, bddc_b200_t** out);
/* The same from BASELINE.json config 1..5 with its seeded coefficient field;
 * subdomains_override (3 ints) / epe_override (>0) shrink it for parity runs. */
int bddc_b200_create_config(int config, uint64_t seed, const int* subdomains_override,
                            int epe_override, bddc_b200_t** out);
void bddc_b200_destroy(bddc_b200_t* h);

int bddc_b200_structure_get(const bddc_b200_t* h, bddc_b200_structure* out);
/* Index maps (spaces.hpp:23-43), for parity checks. */
int bddc_b200_interface_dofs(const bddc_b200_t* h, int64_t* out);
int bddc_b200_subdomain_dim(const bddc_b200_t* h, int s, int64_t* dim);
int bddc_b200_local_to_wc(const bddc_b200_t* h, int s, int64_t* out);
int bddc_b200_global_dof(const bddc_b200_t* h, int s, int64_t* out);
/* Per-element coefficient multipliers (element count entries; 1 when unset). */
int bddc_b200_element_scale(const bddc_b200_t* h, double* out);
/* Substructure stiffness (assemble.cpp:202-292) as CSR (full symmetric) and
 * its load: query nnz with ptr == NULL, then fill ptr (dim+1), idx, val (nnz), load (dim). */
int bddc_b200_subdomain_matrix(const bddc_b200_t* h, int s, int64_t* nnz, int64_t* ptr, int64_t* idx,
                               double* val, double* load);
/* Dense leaf front of substructure s as assembled on the device (assemble.cpp:
 * 202-258 evaluated per entry from the reference element matrices), column-major
 * ld x ld in [interior | boundary] order: query ld with front == NULL, then fill
 * front (ld*ld) and pos (dim: local dof -> front position).  Does not disturb an
 * analysis (the next analysis re-assembles). */
int bddc_b200_leaf_front(bddc_b200_t* h, int s, int64_t* ld, double* front, int64_t* pos);
/* Globs (globs.hpp:18-44): count, then per glob kind / node count / sharer count. */
int bddc_b200_glob_count(const bddc_b200_t* h, int64_t* n);
int bddc_b200_glob_info(const bddc_b200_t* h, int g, int* kind, int64_t* n_nodes, int64_t* n_subs);
int bddc_b200_glob_nodes(const bddc_b200_t* h, int g, int64_t* nodes, int64_t* subs);

/* Constraint set held by the handle (constraints.cpp:34-76). */
int bddc_b200_constraints_arithmetic(bddc_b200_t* h, int edge_globs, int face_globs);
int bddc_b200_constraint_rows(const bddc_b200_t* h, int64_t* rows);
int bddc_b200_constraint_count(const bddc_b200_t* h, int64_t* n);
int bddc_b200_constraint_get(const bddc_b200_t* h, int a, int* glob, int64_t* n_weights, double* weights);
/* A caller-built ConstraintSet (tests/test_constraints.cpp:83-100): clear the
 * handle's set, then add_average (constraints.cpp:61-76) one average at a
 * time -- `weights` has one entry per free dof of the glob (glob_free_dofs,
 * constraints.cpp:25-32); the pivoted-QR rank filter (tolerance 1e-8) decides
 * whether it is kept (*kept = 1) or dropped as dependent / zero (*kept = 0). */
int bddc_b200_constraints_clear(bddc_b200_t* h);
int bddc_b200_constraint_add(bddc_b200_t* h, int glob, const double* weights, int64_t n, int adaptive, int* kept);

/* HarmonicExtension ctor (spaces.cpp:108-147): device A_II factorization and
 * dense interface Schur complements. */
int bddc_b200_analysis(bddc_b200_t* h);
/* enrich_constraints / pair_indicator (adaptive.cpp:129-144).  fixed_count < 0
 * uses tau; indicator_only != 0 adds no rows.  omega_tilde out. */
int bddc_b200_enrich(bddc_b200_t* h, double tau, int max_vectors, int keep_edge, int fixed_count,
                     int indicator_only, double* omega_tilde);
/* Pair report k of the last enrich call (adaptive.hpp:14-22). */
int bddc_b200_pair_count(const bddc_b200_t* h, int64_t* n);
int bddc_b200_pair_report(const bddc_b200_t* h, int k, int* si, int* sj, int* enforced,
                          double* omega_next, int* saturated, int64_t* n_eig, double* eigenvalues);
/* change_of_variables + BddcPreconditioner ctor (bddc_operator.cpp:38-50). */
int bddc_b200_setup_preconditioner(bddc_b200_t* h);
/* The same with the stabilization parameter t of the reference ctor
 * (bddc_operator.hpp:32-35; t <= 0 means max diag K).  The device path factors
 * the exact primal reformulation, on which t does not act, so
 * t only sets what the accessors below report. */
int bddc_b200_setup_preconditioner_t(bddc_b200_t* h, double t);
/* BddcPreconditioner::stabilization_t() (bddc_operator.hpp:52): the t used. */
int bddc_b200_stabilization_t(bddc_b200_t* h, double* t);
/* BddcPreconditioner::stabilized() (bddc_operator.hpp:51), formed on the host
 * (bddc_operator.cpp:7-36: Pi K Pi + t (I - Pi), symmetrized, pruned at 1e-12
 * max|entry|) as full symmetric CSR: query n and nnz with ptr == NULL, then
 * fill ptr (n+1), idx, val (nnz). */
int bddc_b200_stabilized(bddc_b200_t* h, int64_t* n, int64_t* nnz, int64_t* ptr, int64_t* idx, double* val);
/* GlobTransform of one glob under the handle's constraint set
 * (transform.cpp:51-90, transform.hpp:20-27): rank and the dense n x n basis
 * block t (row-major; the identity for an unconstrained glob). */
int bddc_b200_glob_transform(bddc_b200_t* h, int glob, int* rank, int64_t* n, double* t);
/* run_items' export_directory dumps (experiment.cpp:172-178, matrix_market.cpp:
 * 12-38): <stem>_stabilized.mtx (symmetric, lower triangle) and
 * <stem>_constraints.mtx (the transformed constraint matrix D^c). */
int bddc_b200_export_matrix_market(bddc_b200_t* h, const char* stem);

/* LinearOperator seam (pcg.hpp:18): InterfaceProblem::apply (schur.cpp:12-36)
 * and BddcPreconditioner::apply (bddc_operator.cpp:101-103); interface vectors. */
int bddc_b200_interface_size(const bddc_b200_t* h, int64_t* n);
int bddc_b200_schur_apply(bddc_b200_t* h, const double* x, double* y);
int bddc_b200_precond_apply(bddc_b200_t* h, const double* r, double* z);
/* BddcPreconditioner::restrict_residual / coarse_solve / prolong
 * (bddc_operator.hpp:40-48, bddc_operator.cpp:52-99) on W^c vectors (length
 * structure.coarse_space_dim, indexed by bddc_b200_local_to_wc; transformed
 * variables, explicit dof k = glob slot k as transform.cpp:94-149):
 *   restrict_residual: interface r -> Pi T^T E^T r;
 *   coarse_solve: any W^c residual (interior entries included) -> the
 *     constrained-minimization solution Pi A~^{-1} Pi r with the refinement
 *     pass, i.e. the saddle-point solve of acceptance criterion 11
 *     (acceptance_main.cpp:376-420), exact on the device's primal
 *     reformulation for every stabilization t;
 *   prolong: W^c -> interface (T, then the weighted average E).
 * precond_apply == prolong(coarse_solve(restrict_residual(r))).  The stages
 * run on the device as inside precond_apply; the W^c <-> device layout maps
 * are applied on the host (these are not the PCG's path).  Single GPU.
 * generalized_eig_sym (dense_eig.hpp:47-53) has one call site on the path,
 * solve_pair (adaptive.cpp:30-47): bddc_b200_enrich + bddc_b200_pair_report
 * return its eigenvalue list per pair (zeros beyond rank(lhs) included). */
int bddc_b200_restrict_residual(bddc_b200_t* h, const double* r_interface, double* wc);
int bddc_b200_coarse_solve(bddc_b200_t* h, const double* wc_residual, double* wc_out);
int bddc_b200_prolong(bddc_b200_t* h, const double* wc, double* z_interface);
/* Device-timed applications for rooflines (no reference counterpart; the
 * reference times phases only, experiment.cpp:114-203): mean seconds over
 * `reps` applications with device-resident vectors, CUDA events on the handle's
 * stream.  out[13] = [schur, precond, restrict, leaf_fwd, tree_fwd, root,
 * tree_bwd, leaf_bwd, prolong, sum_copies (seconds), schur_bytes,
 * precond_bytes, leaf_sweep_bytes (algorithmic bytes per application)]. */
int bddc_b200_operator_times(bddc_b200_t* h, int reps, double out[13]);
/* InterfaceProblem::rhs / recover (schur.cpp:38-75). */
int bddc_b200_rhs(bddc_b200_t* h, double* out);
int bddc_b200_recover(bddc_b200_t* h, const double* u_interface, double* u_free);
/* pcg + lanczos_condition_estimate (pcg.cpp:11-77).  b == NULL uses the
 * condensed rhs; alphas/betas (length max_iterations) may be NULL.  Returns
 * BDDC_B200_MAX_ITERATIONS with the partial result filled when capped. */
int bddc_b200_pcg(bddc_b200_t* h, const double* b, double* x, double tolerance, int max_iterations,
                  int preconditioned_residual, bddc_b200_pcg_result* res, double* alphas,
                  double* betas);

/* One work item of run_items (experiment.cpp:143-205): mode "c", "c+e",
 * "c+e+f", "c+e+f-3eigv" or "adaptive"; base_faces != 0 starts the adaptive
 * enrichment from c+e+f (BASELINE config 4).  Runs analysis if needed. */
int bddc_b200_run_item(bddc_b200_t* h, const char* mode, double tau, int max_vectors, int keep_edge,
                       int base_faces, bddc_b200_row* row);

/* One pass of the hot path, timed on the device with CUDA events (bench
 * "step"): analysis + constraints (+ enrichment) + preconditioner + PCG.
 * e2e != 0 adds the host->device copies of the inputs (subdomain CSR, loads,
 * maps) and the device->host copy of the recovered solution (u_free, length
 * free_dofs) inside the timed region. */
typedef struct bddc_b200_step_out {
  double seconds, setup_seconds, solve_seconds;
  double h2d_bytes, d2h_bytes;
  int64_t launches;
  int64_t constraint_rows;
  double omega_tilde;
  int64_t iterations;
  double kappa;
  int converged;
  double leaf_factor_seconds, leaf_flops;
} bddc_b200_step_out;
int bddc_b200_step(bddc_b200_t* h, const char* mode, double tau, int max_vectors, int keep_edge,
                   int base_faces, int e2e, double* u_free, bddc_b200_step_out* out);
int64_t bddc_b200_launch_count(void);
/* lanczos_condition_estimate (pcg.cpp:11-26) on given CG coefficients (host). */
int bddc_b200_lanczos(const double* alphas, const double* betas, int64_t n, double* kappa);

/* Device-timed phase seconds and work of the last calls:
 * [analysis, eigen, preconditioner, pcg, leaf_flops, leaf_front_bytes, schur_bytes, root_size,
 *  leaf_factor, pcg_iterations, pcg_bytes_per_iteration] */
int bddc_b200_times(const bddc_b200_t* h, double out[11]);

#ifdef __cplusplus
}
#endif
#endif /* BDDC_B200_H */
