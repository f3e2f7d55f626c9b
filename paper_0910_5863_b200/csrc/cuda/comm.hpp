// Exchange layer of the sharded engine (BASELINE.json
// north_star: "NCCL over NVLink is used only for the interface neighbour
// exchange, the PCG dot-product allreduce and the gather of the root front").
//
// One process (or host thread) per GPU shard.  The engine needs two
// operations, both with results identical on every rank:
//   allreduce  in-place sum of a device array (interface vectors after the
//              per-shard copy sums, the root right-hand side, the root front);
//   allgather  host byte blobs in rank order (selected face constraints and
//              pair reports, so every rank applies the same rank filter);
//   exchange   point-to-point device messages with the neighbour ranks (the
//              interface halo of every operator apply, the Schur complements
//              of the ghost substructures a rank's face pairs need).
// Backends: NCCL (libnccl loaded at run time, one communicator per handle) and
// a loopback group of host threads in one process (tests: ranks exchange only
// through the host after synchronizing their own streams, so no kernel ever
// waits on another rank).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <vector>

namespace b200 {

/// One message of a neighbour exchange: n doubles at device address ptr,
/// to (send) or from (recv) rank `peer`.
struct Segment {
  int peer;
  double* ptr;
  std::size_t n;
};

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  /// In-place sum over ranks of n doubles on the device, ordered on `st`.
  virtual void allreduce(double* d, std::size_t n, cudaStream_t st) = 0;
  /// Point-to-point neighbour exchange (NCCL send/recv in one group): the
  /// k-th send to a peer matches that peer's k-th receive from this rank.
  /// Ordered on `st`.
  virtual void exchange(const std::vector<Segment>& sends, const std::vector<Segment>& recvs, cudaStream_t st) = 0;
  /// Blobs of every rank, in rank order (host memory; synchronizing).
  virtual std::vector<std::vector<char>> allgather(const std::vector<char>& mine) = 0;
  /// Max of a host double over ranks (synchronizing).
  double max_all(double v);
};

/// Loopback group `group` of `world` ranks inside this process (one host
/// thread per rank).  Sums are taken in rank order, so they are deterministic.
std::shared_ptr<Comm> make_loopback_comm(int group, int rank, int world);

/// NCCL communicator from a 128-byte ncclUniqueId made by nccl_unique_id().
std::shared_ptr<Comm> make_nccl_comm(const unsigned char* id, int rank, int world);
void nccl_unique_id(unsigned char* id);  // 128 bytes

}  // namespace b200
