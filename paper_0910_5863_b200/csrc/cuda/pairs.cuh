// Adaptive face eigenproblems on the device (see pairs.cu).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <vector>

#include "../host/host.hpp"
#include "comm.hpp"

namespace b200 {

struct EnrichOptions;
struct EnrichOutcome;

struct PairBuffers;
struct PairPrep;

class PairEngine {
 public:
  PairEngine();
  ~PairEngine();
  /// Pairs are owned by the rank of their lower substructure; the selected
  /// constraints are exchanged so that every rank ends with the same set.
  void set_shard(std::shared_ptr<Comm> comm, const std::vector<int>& owner);
  /// Frees the pair-stage arenas (large runs: the memory goes to the
  /// preconditioner's fronts and root; the next enrich reallocates).
  void release_buffers();
  /// Provider of the pair stage's device region (the engine's stage arena).
  void set_region(std::function<double*(std::size_t)> f) { region_ = std::move(f); }
  void attach(const Model& m, const double* S, const std::vector<long long>& s_off,
              const std::vector<int>& PB, const std::vector<int>& nB, cudaStream_t st);
  /// Host-side preparation (pair index spaces, kernel bases, rigid modes); no
  /// device work, so it can run while the device is busy.
  std::shared_ptr<PairPrep> prepare(const ConstraintSet& cs, const EnrichOptions& o) const;
  /// Reserves the arenas and enqueues the hub stage on the stream (it follows
  /// the leaf factorization in stream order); enrich calls it if nobody did.
  void start(const std::shared_ptr<PairPrep>& prep);
  EnrichOutcome enrich(ConstraintSet& cs, const EnrichOptions& o, std::shared_ptr<PairPrep> prep = nullptr);

 private:
  const Model* m_ = nullptr;
  const double* S_ = nullptr;
  std::vector<long long> s_off_;
  std::vector<int> PB_, nB_;
  cudaStream_t st_ = nullptr;
  std::unique_ptr<PairBuffers> bufs_;
  std::function<double*(std::size_t)> region_;
  std::shared_ptr<Comm> comm_;
  std::vector<int> owner_;
};

}  // namespace b200
