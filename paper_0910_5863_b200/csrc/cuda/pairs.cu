// Adaptive face eigenproblems on the device.
#include "pairs.cuh"

#include "engine.hpp"

namespace b200 {

void PairEngine::attach(const Model& m, const double* S, const std::vector<long long>& s_off,
                        const std::vector<int>& PB, const std::vector<int>& nB, cudaStream_t st) {
  m_ = &m;
  S_ = S;
  s_off_ = s_off;
  PB_ = PB;
  nB_ = nB;
  st_ = st;
}

EnrichOutcome PairEngine::enrich(ConstraintSet&, const EnrichOptions&) {
  throw Error(kUnsupported, "adaptive enrichment not built yet");
}

}  // namespace b200
