// Batched dense FP64 kernels for the adaptive-BDDC fronts (sm_100a).
//
// A "front" is a dense symmetric matrix, column-major, padded to a multiple of
// 64, whose first p columns are eliminated by Cholesky (partial factorization):
//
//      [ A_ee  .   ]      [ L_ee   .  ]  [ L_ee^T  L_ce^T ]
//      [ A_ce A_cc ]  ->  [ L_ce   I  ]  [   0     S_cc   ]
//
// leaving the Schur complement S_cc = A_cc - L_ce L_ce^T in the trailing block
// (lower tiles; diagonal tiles full).  The same kernels factor the substructure
// leaves (A_II eliminated -> interface Schur S_s), the transformed leaf fronts of
// the preconditioner, the root front, and the pair reductions of the adaptive
// eigenproblems.  Tile updates run on FP64 tensor cores (DMMA,
// mma.sync.m16n8k16.f64); see DESIGN.md "Kernels".
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b200 {

constexpr int kTile = 64;

struct FrontDesc {
  double* a;      // n x n column-major (ld = n)
  double* dinv;   // (p/64) inverses of the diagonal L tiles, 64x64 column-major each
  int n;          // padded dimension (multiple of 64)
  int p;          // eliminated columns (multiple of 64, <= n)
  int* info;      // 0, or 1 + first failing pivot column
  // 0, or the first row (multiple of 64, >= p) of an identity-augmented block:
  // rows aug + q hold e_q in the eliminated columns (fronts [[A, .], [I, 0]]).
  // Their factor rows are L^{-T} (upper triangular), so augmented tile (a, k)
  // is zero for a > k and the updates skip those tiles and K ranges.
  int aug;
  // True (unpadded) extents of a plain front (aug == 0): rows/columns [ne, p)
  // and [p + nc, n) are padding (unit diagonal, zeros elsewhere), which
  // contributes nothing to any product.  The dataflow schedule then trims the K
  // ranges to ne (rounded up to 16) and skips the 16-row / 8-column DMMA
  // blocks that lie in padding.  0 = unknown (every tile computed in full).
  int ne = 0, nc = 0;
};

struct SolveDesc {
  const double* a;
  const double* dinv;
  double* x;      // length n
  int n;
  int p;
  const int* cmap;      // optional (backward): x[p+c] = cmap[c] >= 0 ? croot[cmap[c]] : 0
  const double* croot;
  // True (unpadded) extents: rows/columns [ne, p) of the eliminated block and
  // rows [p + nc, n) of the trailing block are padding (unit diagonal, zero
  // vector entries).  The dataflow sweeps never load them, so a sweep moves the
  // factor's own bytes rather than whole 64x64 tiles.  0 = unknown (use p, n - p).
  int ne = 0, nc = 0;
};

/// Streaming multiprocessors of the current device.
int sm_count();

/// One-time per-device state: function attributes (dynamic shared memory),
/// occupancy and SM counts belong to a device, and bddc_b200_set_device lets a
/// process use several.  Returns the value cached for (current device, key),
/// computing it with `make` the first time (thread-safe: loopback ranks are
/// host threads).
int per_device(const void* key, int (*make)());

/// Allocate (once per stream, outside any graph capture) the counters of the
/// dataflow front sweeps.
void ensure_sweep_workspace(cudaStream_t stream);

/// Kernel-launch accounting (bench "gpu_launches").
void count_launch(long long n);
long long launch_count();

/// Timestamps (ns) of front 0's diagonal tasks in the dataflow schedule:
/// out[2j] accumulation done, out[2j+1] Dinv_j published; out[128..143] phase
/// stamps of the first panel factorization (tools/chol_bench).
void chol_trace(bool on, unsigned long long* out);

/// Partial Cholesky of a batch of fronts (device descriptor array).
/// max_n/max_p bound the descriptors' n/p.  Launches on `stream`.
/// max_m bounds the trailing dimension n - p.
void partial_cholesky(const FrontDesc* d_descs, int batch, int max_n, int max_p, int max_m,
                      cudaStream_t stream);

/// Several engines share this device and launch concurrently (the loopback
/// ranks of the tests: host threads of one process on one GPU).  The dataflow
/// Cholesky's chunked mode (diagonal workers and two task queues) needs its
/// whole grid resident at once, which concurrent launches of other engines can
/// deny; while the count is non-zero small batches take the plain queue, whose
/// tasks wait only for tasks already held by running CTAs (deadlock-free for
/// any residency).  One process per GPU never sets it.
void shared_device_users(int delta);

/// Forward sweep x <- [L_ee^{-1} x_e ; x_c - L_ce L_ee^{-1} x_e] per front.
void front_forward(const SolveDesc* d_descs, int batch, int max_n, cudaStream_t stream,
                   const int* done = nullptr);
/// Backward sweep x_e <- L_ee^{-T} (x_e - L_ce^T x_c) per front (x_c given).
void front_backward(const SolveDesc* d_descs, int batch, int max_n, cudaStream_t stream,
                    const int* done = nullptr);

/// Symmetric copy of each front's trailing block into a dense full matrix.
struct TrailDesc {
  const double* a;  // front (ld = n)
  double* s;        // output m x m, ld = m, where m = n - p
  int n;
  int p;
};
void copy_trailing_full(const TrailDesc* d_descs, int batch, int max_m, cudaStream_t stream);

}  // namespace b200
