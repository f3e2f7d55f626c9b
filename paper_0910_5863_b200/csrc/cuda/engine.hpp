// Device engine of the B200 adaptive-BDDC path.
//
// Owns all device state of one problem instance (one GPU, one stream) and
// implements the hot path of SURVEY.md section 8(a):
//   analysis()          HarmonicExtension ctor (spaces.cpp:108-147) + dense
//                       interface Schur complements S_s (pair.cpp:32-63)
//   set_constraints()   change_of_variables + BddcPreconditioner ctor
//                       (transform.cpp:94-149, bddc_operator.cpp:38-50)
//   schur_apply()       InterfaceProblem::apply (schur.cpp:12-36)
//   precond_apply()     BddcPreconditioner::apply (bddc_operator.cpp:52-103)
//   pcg()               pcg + lanczos_condition_estimate (pcg.cpp:11-77)
//   rhs(), recover()    InterfaceProblem::rhs / recover (schur.cpp:38-75)
//   enrich()            enrich_constraints / pair_indicator (adaptive.cpp:66-144)
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "../host/host.hpp"
#include "comm.hpp"
#include "dense.cuh"

namespace b200 {

struct PcgOut {
  int iterations = 0;
  double relative_residual = 0;
  bool converged = true;
  std::vector<double> alphas, betas;
  double condition_estimate = 1.0;
};

struct EnrichOptions {  // adaptive.hpp:24-29
  double tau = 10.0;
  int max_vectors = 15;
  bool keep_edge_constraints = false;
  int fixed_count = -1;
  bool indicator_only = false;  // pair_indicator (no rows added)
};

struct PairReport {  // adaptive.hpp:14-22
  int si = 0, sj = 0;
  std::vector<double> eigenvalues;
  int enforced = 0;
  double omega_next = 0;
  bool saturated = false;
  int kept = 0, dropped = 0;
};

struct EnrichOutcome {
  std::vector<PairReport> pairs;
  double omega_tilde = 0;
  i64 kept = 0, dropped = 0;
};

struct PhaseTimes {  // device-timed seconds (CUDA events) of the last calls
  double analysis = 0, eigen = 0, preconditioner = 0, pcg = 0;
  double leaf_factor = 0;  // the batched partial Cholesky of the substructure leaves
  double flops_leaf = 0;   // algorithmic FP64 flops of the last leaf factorization
  int pcg_iterations = 0;  // of the last pcg()
};

/// One pass of the hot path (bench "step"): analysis + constraint selection
/// (+ adaptive enrichment) + transformed preconditioner + PCG [+ recovery].
struct StepSpec {
  bool edges = true, faces = false, adaptive = false;
  int fixed_count = -1;
  double tau = 10.0;
  int max_vectors = 15;
  bool keep_edge = false;
  double tol = 1e-8;
  int max_it = 500;
  bool e2e = false;          // host->device inputs and device->host solution inside the step
};
struct StepOut {
  double seconds = 0, setup_seconds = 0, solve_seconds = 0;
  double h2d_bytes = 0, d2h_bytes = 0;
  long long launches = 0;
  i64 constraint_rows = 0;
  double omega_tilde = 0;
  PcgOut pcg;
};

struct DeviceState;

class Engine {
 public:
  explicit Engine(const Model& m);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  /// Shard this engine (before any device work): `owner[s]` is the rank that
  /// owns substructure s; this rank assembles and factors its substructures
  /// plus the neighbours its face pairs need (ghosts), runs its pairs, and
  /// exchanges through `comm` (interface sums, root, selected constraints).
  void set_shard(std::shared_ptr<Comm> comm, const std::vector<int>& owner);
  bool sharded() const;
  void prepare();              // host staging + device allocation + first upload
  double upload_inputs(bool on_copy_stream = false);  // host->device copies of the inputs; returns bytes
  void analysis();
  void analysis_launch();  // enqueue only
  void analysis_finish();  // wait + pivot checks
  void set_constraints(const ConstraintSet& cs);
  StepOut step(const StepSpec& spec, ConstraintSet& cs, double* u_free_host);
  void recover_device(const double* d_uiface, double* d_ufree);
  EnrichOutcome enrich(ConstraintSet& cs, const EnrichOptions& o);

  void schur_apply(const double* x, double* y);      // host vectors, interface size
  /// Device-assembled dense front of substructure s (before factorization);
  /// out == nullptr returns only ld and the position map.
  void leaf_front(int s, std::vector<double>* out, std::vector<int>* pos, int* ld);
  void precond_apply(const double* r, double* z);
  /// BddcPreconditioner::{restrict_residual, coarse_solve, prolong}
  /// (bddc_operator.cpp:52-99): interface <-> W^c (maps.wc_dim) host vectors.
  void restrict_residual(const double* r_interface, double* wc);
  void coarse_solve(const double* wc_residual, double* wc_out);
  void prolong(const double* wc, double* z_interface);
  void rhs(double* out);
  void recover(const double* u_interface, double* u_free);
  /// b == nullptr: use the condensed rhs on the device.  x may be nullptr.
  PcgOut pcg(const double* b, double* x, double tol, int max_it, bool precond_residual = false);

  i64 interface_size() const;
  int root_size() const;
  const PhaseTimes& times() const { return times_; }
  double leaf_front_bytes() const;   // bytes of the preconditioner's leaf factors (+root)
  double schur_bytes() const;        // bytes of the dense S_s read per Schur apply
  /// Algorithmic bytes of one PCG iteration: the dense S_s of the Schur apply,
  /// the leaf operators of both preconditioner sweeps and the root apply.
  double pcg_bytes_per_iteration() const;
  /// Device-timed operator applications (bench rooflines): mean seconds of
  /// the Schur apply and of the preconditioner apply (device-resident vectors,
  /// CUDA events on the engine stream) and of the preconditioner's stages.
  struct OpTimes {
    double schur = 0, precond = 0;
    double restrict_ = 0, leaf_fwd = 0, tree_fwd = 0, root = 0, tree_bwd = 0, leaf_bwd = 0, prolong = 0,
           sum_copies = 0;
    double leaf_sweep_bytes = 0;  // algorithmic bytes of one leaf sweep
  };
  OpTimes time_operators(int reps);
  cudaStream_t stream() const;
  /// The pair stage reuses the preconditioner's memory (large runs): the next
  /// set_constraints rebuilds it.
  void invalidate_preconditioner();

 private:
  const Model& m_;
  std::unique_ptr<DeviceState> d_;
  PhaseTimes times_;
};

}  // namespace b200
