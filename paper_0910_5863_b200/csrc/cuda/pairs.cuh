// Adaptive face eigenproblems on the device (see pairs.cu).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "../host/host.hpp"

namespace b200 {

struct EnrichOptions;
struct EnrichOutcome;

struct PairBuffers;

class PairEngine {
 public:
  PairEngine();
  ~PairEngine();
  void attach(const Model& m, const double* S, const std::vector<long long>& s_off,
              const std::vector<int>& PB, const std::vector<int>& nB, cudaStream_t st);
  EnrichOutcome enrich(ConstraintSet& cs, const EnrichOptions& o);

 private:
  const Model* m_ = nullptr;
  const double* S_ = nullptr;
  std::vector<long long> s_off_;
  std::vector<int> PB_, nB_;
  cudaStream_t st_ = nullptr;
  std::unique_ptr<PairBuffers> bufs_;
};

}  // namespace b200
