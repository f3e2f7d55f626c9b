// Batched FP64 partial Cholesky and front solves on sm_100a (see dense.cuh).
//
// Algorithm: left-looking tiled Cholesky over 64x64 tiles.
//   for each eliminated tile column j:
//     k_syrk_column : C_ij -= L_i,[0:j) L_j,[0:j)^T  for all i >= j  (DMMA GEMM, K = 64 j)
//     k_panel       : L_jj = chol(C_jj);  L_ij = C_ij L_jj^{-T};  Dinv_j = L_jj^{-1}
//   k_syrk_trailing : S_ab -= L_a,[0:p) L_b,[0:p)^T for trailing tiles a >= b  (K = p)
// The GEMM tiles stream 64x32 operand panels through a two-stage cp.async
// pipeline into padded shared memory (ld 68 doubles: conflict-free fragment
// loads) and issue mma.sync.aligned.m16n8k16.f64 (FP64 tensor cores).
#include "dense.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstdio>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

namespace b200 {

namespace {

constexpr int LDS = 68;          // padded smem leading dimension (doubles)
constexpr int KC = 32;           // K chunk per pipeline stage
constexpr int GEMM_THREADS = 128;

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Warp-level 32x32 slice of a 64x64 tile product over `kdim` (multiple of 16):
// acc[m][n] += sum_k As[k*LDS + m] * Bs[k*LDS + n].  Only the first vm rows and
// vn columns of the tile are needed (the rest is padding whose product is
// zero): a warp whose 32x32 quadrant lies in padding skips its DMMAs.
__device__ __forceinline__ bool warp_active(int vm, int vn) {
  const int warp = (threadIdx.x >> 5) & 3;
  return vm > (warp & 1) * 32 && vn > (warp >> 1) * 32;
}
// The 32x32 quadrant at (m0, n0) over the K steps [k0, k1) (multiples of 16).
__device__ __forceinline__ void warp_mma_at(const double* As, const double* Bs, int k0, int k1,
                                            double (&acc)[2][4][4], int m0, int n0) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t0 = lane & 3;
#pragma unroll 2
  for (int kk = k0; kk < k1; kk += 16) {
    double a[2][8], b[4][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        a[mi][v] = As[(kk + t0 + 4 * (v >> 1)) * LDS + m0 + mi * 16 + g + 8 * (v & 1)];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v) b[ni][v] = Bs[(kk + t0 + 4 * v) * LDS + n0 + ni * 8 + g];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
  }
}
__device__ __forceinline__ void warp_mma(const double* As, const double* Bs, int kdim,
                                         double (&acc)[2][4][4], bool active = true) {
  const int warp = (threadIdx.x >> 5) & 3;
  if (!active) return;
  warp_mma_at(As, Bs, 0, kdim, acc, (warp & 1) * 32, (warp >> 1) * 32);
}

// Visit the accumulator elements with their tile coordinates.
template <class F>
__device__ __forceinline__ void for_acc(double (&acc)[2][4][4], F f) {
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 3;
  const int g = lane >> 2, t0 = lane & 3;
  const int m0 = (warp & 1) * 32, n0 = (warp >> 1) * 32;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v)
        f(m0 + mi * 16 + g + 8 * (v >> 1), n0 + ni * 8 + 2 * t0 + (v & 1), acc[mi][ni][v]);
}

// C[i0:i0+64, j0:j0+64] -= A[i0:i0+64, 0:K] * A[j0:j0+64, 0:K]^T  (A column-major, ld)
// out == nullptr: C[i0:,j0:] -= A[i0:, kb:ke] A[j0:, kb:ke]^T in place;
// otherwise the product over [kb, ke) is stored to out (64x64, ld 64).
__device__ void tile_update_range(double* a, int ld, int i0, int j0, int kb, int ke, double* out);

__device__ void tile_update_range(double* a, int ld, int i0, int j0, int kb, int ke, double* out) {
  const int K = ke - kb;
  a += (size_t)kb * ld;  // column offset of the K range
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                       // [2][KC*LDS]
  double* Bs = smem + 2 * KC * LDS;        // [2][KC*LDS]
  double acc[2][4][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[mi][ni][v] = 0.0;
  const int nchunks = K / KC;
  auto load = [&](int c, int buf) {
    const int k0 = c * KC;
    for (int q = threadIdx.x; q < KC * 32; q += GEMM_THREADS) {
      const int col = q >> 5, part = q & 31;
      const double* srcA = a + (size_t)(k0 + col) * ld + i0 + part * 2;
      const double* srcB = a + (size_t)(k0 + col) * ld + j0 + part * 2;
      cp_async16(As + buf * KC * LDS + col * LDS + part * 2, srcA);
      cp_async16(Bs + buf * KC * LDS + col * LDS + part * 2, srcB);
    }
    cp_async_commit();
  };
  if (nchunks > 0) load(0, 0);
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      load(c + 1, (c + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    warp_mma(As + (c & 1) * KC * LDS, Bs + (c & 1) * KC * LDS, KC, acc);
    __syncthreads();
  }
  if (out) {
    for_acc(acc, [&](int m, int n, double v) { out[n * 64 + m] = v; });
  } else {
    a -= (size_t)kb * ld;
    for_acc(acc, [&](int m, int n, double v) { a[(size_t)(j0 + n) * ld + i0 + m] -= v; });
  }
}

// First K column with a nonzero factor entry in tile row i0 (see FrontDesc::aug).
__device__ __forceinline__ int aug_k0(const FrontDesc& d, int i0) { return d.aug && i0 >= d.aug ? i0 - d.aug : 0; }

// Split-K column update for fronts with little tile parallelism (single large
// root): CTA (t, b, s) forms the partial product of tile (j + t, j) over the
// K slice s into a workspace; k_splitk_reduce subtracts the slices in a fixed
// order (deterministic).
__global__ void __launch_bounds__(GEMM_THREADS) k_syrk_column_splitk(const FrontDesc* ds, int j, int nsplit,
                                                                    int tiles, double* work) {
  const FrontDesc d = ds[blockIdx.y];
  const int i = j + blockIdx.x;
  if (j * kTile >= d.p || i * kTile >= d.n) return;
  const int K0 = aug_k0(d, i * kTile), K1 = j * kTile;  // K0 > K1: zero tile
  const int K = max(K1 - K0, 0);
  const int chunk = ((K / nsplit + KC - 1) / KC) * KC;
  const int kb = K0 + blockIdx.z * chunk, ke = min(K1, kb + chunk);
  double* out = work + (((size_t)blockIdx.y * tiles + blockIdx.x) * nsplit + blockIdx.z) * 64 * 64;
  if (kb >= ke) {
    for (int e = threadIdx.x; e < 64 * 64; e += GEMM_THREADS) out[e] = 0.0;
    return;
  }
  tile_update_range(d.a, d.n, i * kTile, j * kTile, kb, ke, out);
}

__global__ void k_splitk_reduce(const FrontDesc* ds, int j, int nsplit, int tiles, const double* work) {
  const FrontDesc d = ds[blockIdx.y];
  const int i = j + blockIdx.x;
  if (j * kTile >= d.p || i * kTile >= d.n) return;
  const double* w = work + ((size_t)blockIdx.y * tiles + blockIdx.x) * nsplit * 64 * 64;
  double* c = d.a + (size_t)(j * kTile) * d.n + i * kTile;
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += w[(size_t)q * 64 * 64 + e];
    c[(size_t)(e >> 6) * d.n + (e & 63)] -= s;
  }
}

__global__ void __launch_bounds__(GEMM_THREADS) k_syrk_column(const FrontDesc* ds, int j) {
  const FrontDesc d = ds[blockIdx.y];
  const int i = j + blockIdx.x;
  if (j * kTile >= d.p || i * kTile >= d.n) return;
  const int k0 = aug_k0(d, i * kTile);
  if (k0 > j * kTile) return;  // zero tile of the augmented block
  tile_update_range(d.a, d.n, i * kTile, j * kTile, k0, j * kTile, nullptr);
}

__global__ void __launch_bounds__(GEMM_THREADS) k_syrk_trailing(const FrontDesc* ds) {
  const FrontDesc d = ds[blockIdx.y];
  const int pt = d.p / kTile, m = d.n / kTile - pt;
  const long t = blockIdx.x;
  if (d.p == 0 || t >= (long)m * (m + 1) / 2) return;
  int ii = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((long)ii * (ii + 1) / 2 > t) --ii;
  while ((long)(ii + 1) * (ii + 2) / 2 <= t) ++ii;
  const int jj = static_cast<int>(t - (long)ii * (ii + 1) / 2);
  tile_update_range(d.a, d.n, (pt + ii) * kTile, (pt + jj) * kTile, min(aug_k0(d, (pt + ii) * kTile), d.p), d.p,
                    nullptr);
}

// Panel step (one CTA per front): L_jj = chol(C_jj) and Dinv_j = L_jj^{-1}.
//   POTRF: 16-wide blocked.  Warp 0 factors each 16x16 diagonal block in
//          registers (lane r holds row r; pivots and column entries move by
//          shuffles), the panel rows below are solved row-parallel and the
//          trailing block updated by the whole CTA.
//   L^{-1}: 16x16 diagonal-block inverses (one warp each), off-diagonal blocks by
//          block diagonals: Linv_ij = -Linv_ii sum_k L_ik Linv_kj.
// k_trsm then forms X = C L^{-T} = C Linv^T as one 64x64x64 DMMA tile product.
// Cholesky of the 16x16 diagonal block at Lo (ld LDS, lower triangle) by one
// warp: lane r holds row r in registers; column entries move by shuffles.  The
// pivot chain is kept short: lane k+1 updates its own next pivot with its own
// L[k+1][k] (no shuffle), so one step is shuffle -> rsqrt -> mul -> fma.
// Kept out of line so the unrolled row stays in registers.
// Writes 1/L_kk to rd[k].  Returns 1 + the first non-positive pivot, or 0.
__device__ __noinline__ int chol16(double* Lo, double* rd, int lane) {
  __shared__ __align__(16) double cb[2][16];  // column k of L, double-buffered (warp broadcast)
  const int r = lane & 15;
  double a[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) a[c] = Lo[c * LDS + r];
  int bad = 0;
  double dk = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double inv = dk > 0.0 ? rsqrt(dk) : 1.0;
    if (!(dk > 0.0) && !bad) bad = k + 1;
    if (lane == k) rd[k] = inv;
    const double l = (r == k) ? (dk > 0.0 ? dk * inv : 1.0) : (r > k ? a[k] * inv : a[k]);
    a[k] = l;
    if (k + 1 < 16) {
      // next pivot first: lane k+1 owns L[k+1][k] = l
      const double own = a[k + 1] - l * l;
      const double dn = __shfl_sync(0xffffffffu, own, k + 1);
      if (lane < 16) cb[k & 1][r] = l;
      __syncwarp();
      const double2* col = reinterpret_cast<const double2*>(cb[k & 1]);
#pragma unroll
      for (int q = (k + 1) / 2; q < 8; ++q) {
        const double2 v = col[q];  // L[2q][k], L[2q+1][k]
        if (2 * q > k) a[2 * q] = (r >= 2 * q) ? a[2 * q] - l * v.x : a[2 * q];
        a[2 * q + 1] = (r >= 2 * q + 1) ? a[2 * q + 1] - l * v.y : a[2 * q + 1];
      }
      dk = dn;
    }
  }
  if (lane < 16) {
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (c <= r) Lo[c * LDS + r] = a[c];
  }
  return bad;
}

// 16x16 block product on one warp (DMMA m16n8k16): acc += op(A) B with
// A(m, k) = A[m * ars + k * acs], B(k, n) = B[k * brs + n * bcs], K a multiple
// of 16; op negates A when NEG.  acc[ni][v] is C(g + 8 (v >> 1), 8 ni + 2 t0 + (v & 1)).
template <bool NEG>
__device__ __forceinline__ void mma16(double (&acc)[2][4], const double* A, int ars, int acs, const double* B,
                                      int brs, int bcs, int K) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t0 = lane & 3;
  for (int kk = 0; kk < K; kk += 16) {
    double a[8], b[2][4];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const double x = A[(g + 8 * (v & 1)) * ars + (kk + t0 + 4 * (v >> 1)) * acs];
      a[v] = NEG ? -x : x;
    }
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v) b[ni][v] = B[(kk + t0 + 4 * v) * brs + (ni * 8 + g) * bcs];
    dmma(acc[0], a, b[0]);
    dmma(acc[1], a, b[1]);
  }
}

template <class F>
__device__ __forceinline__ void for_acc16(double (&acc)[2][4], F f) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t0 = lane & 3;
#pragma unroll
  for (int ni = 0; ni < 2; ++ni)
#pragma unroll
    for (int v = 0; v < 4; ++v) f(g + 8 * (v >> 1), ni * 8 + 2 * t0 + (v & 1), acc[ni][v]);
}

constexpr int PANEL_THREADS = 256;

// Timestamps of front 0's diagonal tasks (tools/chol_bench): [2j] accumulation
// done, [2j+1] Dinv_j published.
__device__ unsigned long long g_dag_trace[2 * 64];
__device__ int g_dag_trace_on;
__device__ unsigned long long g_pf_trace[16];
__device__ __forceinline__ void pf_mark(int slot) {
#ifndef DENSE_TRACE
  return;
#endif
  if (g_dag_trace_on && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_pf_trace[slot] = t;
  }
}
__device__ __forceinline__ void dag_mark(int b, int slot) {
#ifndef DENSE_TRACE
  return;
#endif
  if (g_dag_trace_on && b == 0 && threadIdx.x == 0 && slot < 128) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_dag_trace[slot] = t;
  }
}


// POTRF of the 64x64 tile in L (shared, ld LDS, lower triangle) and its
// inverse into V, by NT threads.  Returns 1 + the first non-positive pivot
// (uniform over the CTA), or 0.  On success dinv_out (64x64, column-major)
// receives L^{-1} with zeros above the block diagonal.
// Trailing block (bi, bj) of the tile minus X_bi X_bj^T, X = block column o
// (one warp, DMMA).
__device__ __forceinline__ void panel_trailing_block(double* L, int o, int bi, int bj) {
  double acc[2][4];
  double* Cb = L + (16 * bj) * LDS + 16 * bi;
  for_acc16(acc, [&](int m, int n, double& v) { v = Cb[n * LDS + m]; });
  mma16<true>(acc, L + o * LDS + 16 * bi, 1, LDS, L + o * LDS + 16 * bj, LDS, 1, 16);
  for_acc16(acc, [&](int m, int n, double& v) { Cb[n * LDS + m] = v; });
}

// Off-diagonal block (i, j), j < i, of W = L^{-1} (one warp, DMMA):
// T = sum_{k=j}^{i-1} L_ik W_kj;  W_ij = -W_ii T.  T in the strictly upper block
// (0, ts) of the tile, which the factorization leaves unused.
__device__ __forceinline__ void panel_inverse_block(double* L, double* V, int i, int j, int ts) {
  double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  mma16<false>(acc, L + (16 * j) * LDS + 16 * i, 1, LDS, V + (16 * j) * LDS + 16 * j, 1, LDS, 16 * (i - j));
  double* T = L + (16 * ts) * LDS;
  for_acc16(acc, [&](int m, int n, double& v) { T[n * LDS + m] = v; });
  __syncwarp();
  double acc2[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  mma16<true>(acc2, V + (16 * i) * LDS + 16 * i, 1, LDS, T, 1, LDS, 16);
  for_acc16(acc2, [&](int m, int n, double& v) { V[(16 * j + n) * LDS + 16 * i + m] = v; });
  __syncwarp();
}

template <int NT>
__device__ int panel_factor(double* L, double* V, double* dinv_out) {
  static_assert(NT >= 128, "four warps");
  __shared__ double rd[64];  // reciprocal diagonal of L_jj
  __shared__ int bad_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bad_s = 0;
  __syncthreads();
  pf_mark(0);
  // ---- blocked POTRF, 16-wide, with lookahead.  Step kb:
  //   phase 1: warp 0 factors diagonal block kb (its update by column block
  //            kb-1 was applied by warp 0 at the end of step kb-1); warps 1-3
  //            apply column block kb-1 to the other trailing blocks and form
  //            row kb-1 of L^{-1} (blocks left of the diagonal);
  //   phase 2: warp 0 inverts the diagonal block (W_kk, into V) while warps
  //            1-2 solve the rows below (thread per row, right-looking);
  //   phase 3: warp 0 applies column block kb to diagonal block kb+1.
  for (int kb = 0; kb < 4; ++kb) {
    const int o = kb * 16;
    if (warp == 0) {
      const int bad = chol16(L + o * LDS + o, rd + o, lane);
      if (lane == 0 && bad && !bad_s) bad_s = o + bad;
    } else if (warp < 4 && kb > 0) {
      // column block kb-1 applied to blocks (bi, bj), kb <= bj <= bi < 4, except (kb, kb)
      int q = 0;
      for (int bi = kb; bi < 4; ++bi)
        for (int bj = kb; bj <= bi; ++bj) {
          if (bi == kb && bj == kb) continue;
          if (q++ % 3 == warp - 1) panel_trailing_block(L, o - 16, bi, bj);
        }
      // row kb-1 of L^{-1}: blocks (kb-1, j), j < kb-1
      for (int j = warp - 1; j < kb - 1; j += 3) panel_inverse_block(L, V, kb - 1, j, warp);
    }
    __syncthreads();
    pf_mark(1 + 3 * kb);
    if (warp == 0) {
      if (lane < 16) {  // column c of W_kk = L_kk^{-1}, right-looking (short dependency chains)
        const int c = lane;
        double x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = (r == c) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          x[k] = (k >= c) ? x[k] * rd[o + k] : 0.0;
#pragma unroll
          for (int r = k + 1; r < 16; ++r) x[r] -= L[(o + k) * LDS + o + r] * x[k];
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) V[(o + c) * LDS + o + r] = x[r];
      }
    } else if (tid - 32 < 48 - o) {  // panel rows below: x L_kk^T = a, right-looking
      const int r = o + 16 + (tid - 32);
      double x[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) x[c] = L[(o + c) * LDS + r];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        x[c] *= rd[o + c];
#pragma unroll
        for (int c2 = c + 1; c2 < 16; ++c2) x[c2] -= x[c] * L[(o + c) * LDS + o + c2];
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) L[(o + c) * LDS + r] = x[c];
    }
    __syncthreads();
    pf_mark(2 + 3 * kb);
    if (warp == 0 && kb < 3) {
      panel_trailing_block(L, o, kb + 1, kb + 1);
      __syncwarp();  // chol16 reads the block with another lane mapping
    }
  }
  // row 3 of L^{-1}
  if (warp < 3) panel_inverse_block(L, V, 3, warp, warp + 1);
  __syncthreads();
  const int bad = bad_s;
  if (bad) return bad;
  pf_mark(14);
  // Dinv = L^{-1} (zero above the block diagonal).
  double2* dv = reinterpret_cast<double2*>(dinv_out);
  for (int q = tid; q < 64 * 32; q += NT) {
    const int c = q >> 5, r = (q & 31) * 2;
    double2 v;
    v.x = (r >> 4) >= (c >> 4) ? V[c * LDS + r] : 0.0;
    v.y = (r >> 4) >= (c >> 4) ? V[c * LDS + r + 1] : 0.0;
    dv[q] = v;
    V[c * LDS + r] = v.x;  // the dataflow worker multiplies by V directly
    V[c * LDS + r + 1] = v.y;
  }
  pf_mark(15);
  return 0;
}

__global__ void __launch_bounds__(PANEL_THREADS) k_panel(const FrontDesc* ds, int j) {
  const FrontDesc d = ds[blockIdx.y];
  if (j * kTile >= d.p) return;
  extern __shared__ __align__(16) double smem[];
  double* L = smem;             // 64 x LDS, column-major: L[c*LDS + r]
  double* V = smem + 64 * LDS;  // L^{-1} (lower block triangle only)
  const int tid = threadIdx.x;
  const size_t ld = d.n;
  const double* diag = d.a + (size_t)(j * kTile) * ld + j * kTile;
  for (int q = tid; q < 64 * 32; q += PANEL_THREADS) {
    const int col = q >> 5, part = q & 31;
    cp_async16(L + col * LDS + part * 2, diag + (size_t)col * ld + part * 2);
  }
  cp_async_commit();
  cp_async_wait<0>();
  // The diagonal tile itself is never read again (solves and later updates
  // touch only off-diagonal tiles), so it is not written back.
  const int bad = panel_factor<PANEL_THREADS>(L, V, d.dinv + (size_t)j * 64 * 64);
  if (bad && tid == 0) atomicCAS(d.info, 0, j * kTile + bad);
}

// Off-diagonal tiles of column j: X = C_ij L_jj^{-T} = C_ij Dinv_j^T as one
// 64x64x64 DMMA tile product (Dinv_j written by k_panel).
__global__ void __launch_bounds__(GEMM_THREADS) k_trsm(const FrontDesc* ds, int j) {
  const FrontDesc d = ds[blockIdx.y];
  const int i = j + 1 + blockIdx.x;
  if (j * kTile >= d.p || i * kTile >= d.n) return;
  if (aug_k0(d, i * kTile) > j * kTile) return;  // zero tile of the augmented block
  extern __shared__ __align__(16) double smem[];
  double* V = smem;
  double* C = smem + 64 * LDS;
  const size_t ld = d.n;
  const double* dv = d.dinv + (size_t)j * 64 * 64;
  const double* ct = d.a + (size_t)(j * kTile) * ld + i * kTile;
  for (int q = threadIdx.x; q < 64 * 32; q += GEMM_THREADS) {
    const int col = q >> 5, part = q & 31;
    cp_async16(V + col * LDS + part * 2, dv + (size_t)col * 64 + part * 2);
    cp_async16(C + col * LDS + part * 2, ct + (size_t)col * ld + part * 2);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  double acc[2][4][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[mi][ni][v] = 0.0;
  warp_mma(C, V, 64, acc);
  double* out = d.a + (size_t)(j * kTile) * ld + i * kTile;
  for_acc(acc, [&](int m, int n, double v) { out[(size_t)n * ld + m] = v; });
}

// ---------------------------------------------------------------------------
// Dataflow partial Cholesky for latency-bound batches: one persistent launch
// instead of ~3 launches per tile column.  Task (b, i, j) is tile (i, j) of
// front b; an atomic counter hands the tasks out in a fixed topological order
// (column j major; within a column the diagonal tiles of every front first,
// then the off-diagonal rows in increasing i):
//   j <  p_b/64 : C_ij -= sum_{k<j} L_ik L_jk^T, accumulated as the columns k
//                 become final; then i == j: L_jj = chol(C_jj), Dinv_j = L_jj^{-1}
//                 (panel_factor), i > j: L_ij = C_ij Dinv_j^T (one DMMA tile product)
//   j >= p_b/64 : trailing tile S_ij -= sum_{k<p} L_ik L_jk^T
// prog[b][i] = 1 + the last column k whose tile (i, k) is final; it is stored
// with release semantics after the tile (monotone: tile (i, k) is written only
// after its task has read (i, k-1)).  A task waits only for tasks with smaller
// indices, which were handed to CTAs that are already running, so the schedule
// cannot deadlock for any grid size.  The arithmetic is the tiled path's
// (same K order of the DMMA accumulation, same panel and trsm).
// ---------------------------------------------------------------------------
constexpr int DAG_THREADS = 128;
constexpr int DAG_CTL = 288;  // ints before the progress counters: [0] tasks, [1] roles, [32..288) SM flags

// Polls read the flags relaxed (an acquire load invalidates L1 on every
// iteration); one acquire fence follows the successful poll.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// acc = sum over K in [kb, ke) of A[i0:i0+64, K] A[j0:j0+64, K]^T, waiting for
// column block k of rows i0/64 and j0/64 (prog pointers pi, pj) before reading it.
// vm / vn: valid rows of tile rows i0/64 and j0/64; kv: valid end of the K
// range (columns >= kv are padding, FrontDesc::ne): the range is cut at kv
// rounded up to 16.
__device__ void dag_accumulate(const double* a, int ld, int i0, int j0, int kb, int ke, const int* pi,
                               const int* pj, double (&acc)[2][4][4], double* smem, int* s_ready, int vm = 64,
                               int vn = 64, int kv = 1 << 30) {
  double* As = smem;                 // [2][KC*LDS]
  double* Bs = smem + 2 * KC * LDS;  // [2][KC*LDS]
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[mi][ni][v] = 0.0;
  ke = min(ke, (kv + 15) & ~15);
  const int nch = (ke - kb + KC - 1) / KC;
  if (nch <= 0 || vm <= 0 || vn <= 0) return;
  // Warp roles.  Inside a front warp w owns quadrant (w & 1, w >> 1).  In an
  // edge tile whose lower (right) half is padding the two warps of that half
  // would idle while the other two set the tile's time: they take the second
  // half of every K chunk of their neighbour's quadrant instead, and the two
  // partial sums are added through shared memory at the end (fixed order).
  const int warp = (threadIdx.x >> 5) & 3;
  int wm = warp & 1, wn = warp >> 1, khalf = 0;
  bool split = false, active = true;
  if (vm <= 32 && vn > 32) {
    split = true;
    khalf = wm;
    wm = 0;
  } else if (vn <= 32 && vm > 32) {
    split = true;
    khalf = wn;
    wn = 0;
  } else {
    active = warp_active(vm, vn);
  }
  int ready = 0;  // column blocks [0, ready) final for both rows (uniform over the CTA)
  auto blk = [&](int c) { return (kb + c * KC) >> 6; };
  auto poll = [&](int need, bool block) {
    __syncthreads();  // every thread has read the previous s_ready
    if (threadIdx.x == 0) {
      int v;
      do {
        v = min(ld_relaxed(pi), ld_relaxed(pj));
      } while (block && v <= need);
      fence_acquire();
      *s_ready = v;
    }
    __syncthreads();
    ready = *s_ready;
  };
  auto load = [&](int c, int buf) {
    const int k0 = kb + c * KC;
    for (int q = threadIdx.x; q < KC * 32; q += DAG_THREADS) {
      const int col = q >> 5, part = q & 31;
      const double* srcA = a + (size_t)(k0 + col) * ld + i0 + part * 2;
      const double* srcB = a + (size_t)(k0 + col) * ld + j0 + part * 2;
      cp_async16(As + buf * KC * LDS + col * LDS + part * 2, srcA);
      cp_async16(Bs + buf * KC * LDS + col * LDS + part * 2, srcB);
    }
    cp_async_commit();
  };
  if (blk(0) >= ready) poll(blk(0), true);
  load(0, 0);
  for (int c = 0; c < nch; ++c) {
    bool pf = false;
    if (c + 1 < nch) {
      if (blk(c + 1) >= ready) poll(blk(c + 1), false);
      pf = blk(c + 1) < ready;
    }
    if (pf) {
      load(c + 1, (c + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    {
      const int kdim = min(KC, ke - kb - c * KC);
      const double* Ac = As + (c & 1) * KC * LDS;
      const double* Bc = Bs + (c & 1) * KC * LDS;
      if (split)
        warp_mma_at(Ac, Bc, khalf ? 16 : 0, khalf ? kdim : min(kdim, 16), acc, wm * 32, wn * 32);
      else if (active)
        warp_mma_at(Ac, Bc, 0, kdim, acc, wm * 32, wn * 32);
    }
    __syncthreads();
    if (c + 1 < nch && !pf) {
      poll(blk(c + 1), true);
      load(c + 1, (c + 1) & 1);
    }
  }
  if (split) {  // helpers hand their partial sums to the quadrant's owner and clear their own (padding) quadrant
    const int lane = threadIdx.x & 31;
    double* xch = smem + ((vm <= 32 ? wn : wm) * 32 + lane);  // [32 values][2 owners x 32 lanes]
    if (khalf) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            xch[((mi * 4 + ni) * 4 + v) * 64] = acc[mi][ni][v];
            acc[mi][ni][v] = 0.0;
          }
    }
    __syncthreads();
    if (!khalf) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[mi][ni][v] += xch[((mi * 4 + ni) * 4 + v) * 64];
    }
    __syncthreads();  // the operand buffers are free for the caller again
  }
}

// Valid (unpadded) rows of tile row i of a plain front, and the valid end of
// its eliminated columns (FrontDesc::ne / nc; 64 and p when unknown).
__device__ __forceinline__ int front_valid(const FrontDesc& d, int i) {
  if (d.ne <= 0 || d.aug) return kTile;
  const int pt = d.p / kTile;
  return max(0, min(kTile, i < pt ? d.ne - i * kTile : d.nc - (i - pt) * kTile));
}
__device__ __forceinline__ int front_kvalid(const FrontDesc& d) { return d.ne > 0 && !d.aug ? d.ne : d.p; }

// Diagonal tile j of front b: C_jj -= sum_k L_jk L_jk^T (waiting for the
// columns), L_jj = chol(C_jj), Dinv_j; publishes prog[j] = j + 1.
__device__ void dag_diagonal(const FrontDesc& d, int b, int j, int* prog, double* smem, int* s_ready) {
  const int tid = threadIdx.x, j0 = j * kTile;
  const size_t ld = d.n;
  double acc[2][4][4];
  dag_accumulate(d.a, d.n, j0, j0, 0, j0, prog + j, prog + j, acc, smem, s_ready, front_valid(d, j),
                 front_valid(d, j), front_kvalid(d));
  dag_mark(b, 2 * j);
  double* tile = d.a + (size_t)j0 * ld + j0;
  double* C = smem;
  double* V = smem + 64 * LDS;
  for (int q = tid; q < 64 * 32; q += DAG_THREADS) {
    const int col = q >> 5, part = q & 31;
    cp_async16(C + col * LDS + part * 2, tile + (size_t)col * ld + part * 2);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for_acc(acc, [&](int m, int n, double v) { C[n * LDS + m] -= v; });
  __syncthreads();
  // keep the updated (unfactored) diagonal tile in the front, as the tiled path does
  for (int q = tid; q < 64 * 32; q += DAG_THREADS) {
    const int col = q >> 5, part = q & 31;
    *reinterpret_cast<double2*>(tile + (size_t)col * ld + part * 2) =
        *reinterpret_cast<const double2*>(C + col * LDS + part * 2);
  }
  const int bad = panel_factor<DAG_THREADS>(C, V, d.dinv + (size_t)j * 64 * 64);
  if (bad && tid == 0) atomicCAS(d.info, 0, j0 + bad);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(prog + j, j + 1);
  }
  dag_mark(b, 2 * j + 1);
}

// ctl: [0] task counter, [1] role counter, [DAG_CTL ...] prog[b][i].
// The first `workers` CTAs to start (they are resident) own the eliminated
// diagonal tiles of fronts b = role, role + workers, ... column by column,
// accumulating each tile while its columns arrive; the others take the
// remaining tasks from the queue.  workers == 0: every task from the queue.
// Off-diagonal tile (i, j), j < p/64: L_ij = (C_ij - sum_{k<j} L_ik L_jk^T) Dinv_j^T;
// publishes prog[i] = j + 1.
__device__ void dag_offdiag(const FrontDesc& d, int i, int j, int* prog, double* smem, int* s_ready) {
  const int tid = threadIdx.x, i0 = i * kTile, j0 = j * kTile;
  const size_t ld = d.n;
  const int kb = aug_k0(d, i0);
  if (kb > j0) return;  // zero tile of the augmented block
  double acc[2][4][4];
  const int vi = front_valid(d, i), vj = front_valid(d, j);
  dag_accumulate(d.a, d.n, i0, j0, kb, j0, prog + i, prog + j, acc, smem, s_ready, vi, vj, front_kvalid(d));
  double* tile = d.a + (size_t)j0 * ld + i0;
  double* C = smem;
  double* V = smem + 64 * LDS;
  for (int q = tid; q < 64 * 32; q += DAG_THREADS) {
    const int col = q >> 5, part = q & 31;
    cp_async16(C + col * LDS + part * 2, tile + (size_t)col * ld + part * 2);
  }
  cp_async_commit();
  __syncthreads();
  if (tid == 0)
    while (ld_relaxed(prog + j) <= j) {
    }
  if (tid == 0) fence_acquire();
  __syncthreads();
  const double* dv = d.dinv + (size_t)j * 64 * 64;
  for (int q = tid; q < 64 * 32; q += DAG_THREADS) {
    const int col = q >> 5, part = q & 31;
    cp_async16(V + col * LDS + part * 2, dv + (size_t)col * 64 + part * 2);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for_acc(acc, [&](int m, int n, double v) { C[n * LDS + m] -= v; });
  __syncthreads();
  double x[2][4][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int v = 0; v < 4; ++v) x[mi][ni][v] = 0.0;
  warp_mma(C, V, min(64, (vj + 15) & ~15), x, warp_active(vi, vj));  // padding rows / columns of L_ij stay zero
  for_acc(x, [&](int m, int n, double v) { tile[(size_t)n * ld + m] = v; });
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(prog + i, j + 1);
  }
}

// tile (64x64 at t, ld) -= acc, staged through shared memory so that the
// global read-modify-write is coalesced (16-byte accesses along columns).
// Call after dag_accumulate (its trailing barrier frees the operand buffers).
__device__ __forceinline__ void tile_sub_acc(double* t, size_t ld, double (&acc)[2][4][4], double* smem) {
  for_acc(acc, [&](int m, int n, double v) { smem[n * LDS + m] = v; });
  __syncthreads();
  for (int q = threadIdx.x; q < 64 * 32; q += DAG_THREADS) {
    const int col = q >> 5, part = q & 31;
    double2* g = reinterpret_cast<double2*>(t + (size_t)col * ld + part * 2);
    const double2 a = *reinterpret_cast<const double2*>(smem + col * LDS + part * 2);
    double2 v = *g;
    v.x -= a.x;
    v.y -= a.y;
    *g = v;
  }
}

// Trailing tile (i, j), i >= j >= p/64: S_ij -= sum over K in [kb, ke) of L_iK L_jK^T.
__device__ void dag_trailing(const FrontDesc& d, int i, int j, int kb, int ke, int* prog, double* smem,
                             int* s_ready) {
  const int i0 = i * kTile, j0 = j * kTile;
  double acc[2][4][4];
  dag_accumulate(d.a, d.n, i0, j0, kb, ke, prog + i, prog + j, acc, smem, s_ready, front_valid(d, i),
                 front_valid(d, j), front_kvalid(d));
  tile_sub_acc(d.a + (size_t)j0 * d.n + i0, d.n, acc, smem);
}

__device__ __forceinline__ void wait_flag(const int* f, int v) {
  __syncthreads();
  if (threadIdx.x == 0)
    while (ld_relaxed(f) < v) {
    }
  if (threadIdx.x == 0) fence_acquire();
  __syncthreads();
}

__device__ __forceinline__ void load_tile(double* dst, const double* src, size_t ld) {
  for (int q = threadIdx.x; q < 64 * 32; q += DAG_THREADS) {
    const int col = q >> 5, part = q & 31;
    cp_async16(dst + col * LDS + part * 2, src + (size_t)col * ld + part * 2);
  }
  cp_async_commit();
}

// Diagonal worker of one front (chunked mode).  Iteration j, with
// C = C_jj - sum_{k<j} L_jk L_jk^T already in shared memory:
//   L_jj = chol(C), Dinv_j (panel_factor; V keeps L_jj^{-1})      -> prog[j] = j+1
//   L_{j+1,j} = C'_{j+1,j} Dinv_j^T (C' prepared by a queue task)    -> prog[j+1] = j+1
//   C = C'_{j+1,j+1} - L_{j+1,j} L_{j+1,j}^T                        (next pivot tile)
// so the pivot chain never leaves the SM: the queue prepares the tiles
// (every column but the last), the worker applies the last one.
__device__ void dag_worker(const FrontDesc& d, int b, int* prog, const int* presub, const int* prediag,
                           double* smem) {
  const int tid = threadIdx.x, pt = d.p / kTile, nt = d.n / kTile;
  const size_t ld = d.n;
  double* C = smem;
  double* V = smem + 64 * LDS;
  if (pt == 0) return;
  load_tile(C, d.a, ld);
  cp_async_wait<0>();
  __syncthreads();
  for (int j = 0; j < pt; ++j) {
    const int j0 = j * kTile;
    double* tile = d.a + (size_t)j0 * ld + j0;
    dag_mark(b, 2 * j);
    // keep the updated (unfactored) diagonal tile in the front, as the tiled path does
    for (int q = tid; q < 64 * 32; q += DAG_THREADS) {
      const int col = q >> 5, part = q & 31;
      *reinterpret_cast<double2*>(tile + (size_t)col * ld + part * 2) =
          *reinterpret_cast<const double2*>(C + col * LDS + part * 2);
    }
    const int bad = panel_factor<DAG_THREADS>(C, V, d.dinv + (size_t)j * 64 * 64);
    if (bad && tid == 0) atomicCAS(d.info, 0, j0 + bad);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(prog + j, j + 1);
    }
    dag_mark(b, 2 * j + 1);
    const int i = j + 1, i0 = i * kTile;
    if (i >= nt || aug_k0(d, i0) > j0) continue;  // no sub-diagonal tile (or a zero one)
    double* sub = d.a + (size_t)j0 * ld + i0;
    if (j > 0) wait_flag(presub + j, 1);
    load_tile(C, sub, ld);
    cp_async_wait<0>();
    __syncthreads();
    double x[2][4][4];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[mi][ni][v] = 0.0;
    warp_mma(C, V, 64, x);
    __syncthreads();  // C and V are read by every warp
    for_acc(x, [&](int m, int n, double v) {
      sub[(size_t)n * ld + m] = v;
      C[n * LDS + m] = v;
    });
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(prog + i, j + 1);
    }
    if (i >= pt) continue;
    // next pivot tile: C'_{i,i} (prepared through column j-1) minus L_ij L_ij^T
    if (i >= 2) wait_flag(prediag + i, 1);
    double* diag = d.a + (size_t)i0 * ld + i0;
    load_tile(V, diag, ld);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int v = 0; v < 4; ++v) x[mi][ni][v] = 0.0;
    warp_mma(C, C, 64, x);
    cp_async_wait<0>();
    __syncthreads();
    for_acc(x, [&](int m, int n, double v) { C[n * LDS + m] = V[n * LDS + m] - v; });
    __syncthreads();
  }
}

// Queue task preparing tile (i, j) for the worker: C_ij -= sum over K in
// [kb, ke) of L_iK L_jK^T, stored in place; then flag = 1.
__device__ void dag_prepare(const FrontDesc& d, int i, int j, int kb, int ke, int* prog, int* flag, double* smem,
                            int* s_ready) {
  if (ke > kb) {
    const int i0 = i * kTile, j0 = j * kTile;
    double acc[2][4][4];
    dag_accumulate(d.a, d.n, i0, j0, kb, ke, prog + i, prog + j, acc, smem, s_ready, front_valid(d, i),
                   front_valid(d, j), front_kvalid(d));
    tile_sub_acc(d.a + (size_t)j0 * d.n + i0, d.n, acc, smem);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(flag, 1);
  }
}

// ctl: [0] task counter (A), [1] role counter, [2] queue CTAs that left, [3] queue roles,
// [4] task counter (B), [32, 288) per-SM worker flags,
// [DAG_CTL ...] prog[b][i] (batch x nt); chunked mode adds tflag[b][ii * mt + jj]
// (batch x mt x mt), presub[b][j] and prediag[b][j] (batch x nt each).
//
// Plain mode (chunked == 0): the queue holds every tile, column j major
// (diagonals of every front, then the off-diagonal rows); trailing tiles are
// single tasks over the whole K range.
// Chunked mode (small batches): the first `batch` CTAs to start are the
// fronts' diagonal workers (dag_worker); queue CTAs that land on a worker's SM
// leave, so the pivot chain runs on an otherwise idle SM.  Two queues:
//   A = E_0, E_1, ..., E_{pt-1}   and   B = R_0, R_1, ..., R_{pt-1}
// E_c = [L_{c+2,c}] [prepare (c+2, c+1) through column c] [prepare (c+2, c+2)
// through column c] [L_{i,c}, i >= c+3]  (every front each), R_k = the updates
// of every trailing tile by the columns [k cw, (k+1) cw) (chunk k of a tile waits for chunk
// k-1 of the same tile).  Half of the queue CTAs take B only; the others take A
// and then B.  A waits only on A and the workers, B on A and B: no cycle.
__global__ void __launch_bounds__(DAG_THREADS, 3) k_chol_dag(const FrontDesc* ds, int batch, int nt, int pt_max,
                                                          int mt, int* ctl, int total, int chunked, int cw, int bq) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_task, s_ready;
  const int tid = threadIdx.x;
  int* tflag = ctl + DAG_CTL + (size_t)batch * nt;
  int* presub = tflag + (size_t)batch * mt * mt;
  int* prediag = presub + (size_t)batch * nt;
  if (chunked) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (tid == 0) s_task = atomicAdd(ctl + 1, 1);
    __syncthreads();
    const int role = s_task;
    __syncthreads();
    if (role < batch) {
      if (tid == 0) atomicExch(ctl + 32 + (smid & 255), 1);
      const FrontDesc d = ds[role];
      dag_worker(d, role, ctl + DAG_CTL + (size_t)role * nt, presub + (size_t)role * nt,
                 prediag + (size_t)role * nt, smem);
      return;
    }
    // share no SM with a worker, but keep at least half of the queue CTAs
    if (tid == 0) s_task = atomicAdd(ctl + 32 + (smid & 255), 0) && atomicAdd(ctl + 2, 1) < (gridDim.x - batch) / 2;
    __syncthreads();
    if (s_task) return;
  }
  const int rsize = batch * (mt * (mt + 1) / 2);
  // chunked mode: queue A = E_0 .. E_{pt-1} (elimination), queue B = R_0 .. R_{pt-1}
  // (trailing updates).  Every other queue CTA works on B only, so the trailing
  // updates never hold back the elimination; A CTAs move on to B when A is empty.
  int etotal = 0;
  if (chunked)
    for (int c = 0; c < pt_max; ++c) etotal += batch * (max(nt - c - 2, 0) + 2);
  bool on_b = false;
  if (chunked) {
    if (tid == 0) s_task = atomicAdd(ctl + 3, 1);
    __syncthreads();
    on_b = (s_task % 12) < bq;  // bq twelfths of the queue CTAs serve B only
  }
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      int t = total;
      if (!chunked || !on_b) {
        t = atomicAdd(ctl, 1);
        if (chunked && t >= etotal) on_b = true;
      }
      if (chunked && on_b) t = etotal + atomicAdd(ctl + 4, 1);
      s_task = t;
    }
    __syncthreads();
    const int t = s_task;
    if (t >= total) return;
    if (chunked && t >= etotal) on_b = true;
    if (!chunked) {
      int b, i, j = 0, r = t;
      const int telim = batch * (pt_max * nt - pt_max * (pt_max - 1) / 2);  // tasks of the columns j < pt_max
      if (t < telim) {
        while (r >= batch * (nt - j)) {
          r -= batch * (nt - j);
          ++j;
        }
        // within a column: every front's diagonal tile, then the rows front by
        // front (consecutive tasks share the front's row-j panel in L2)
        if (r < batch) {
          b = r;
          i = j;
        } else {
          r -= batch;
          b = r / (nt - j - 1);
          i = j + 1 + r % (nt - j - 1);
        }
      } else {
        // columns past every front's eliminated part: the trailing tiles front by
        // front, so the tiles in flight share their few fronts' row panels
        // L(i, 0:p) in L2 (mt panels for mt (mt + 1) / 2 tiles) instead of every
        // tile streaming its own pair of panels from DRAM
        const int mtm = nt - pt_max, per = mtm * (mtm + 1) / 2;
        r = t - telim;
        b = r / per;
        const int q = r - b * per;
        int ii = static_cast<int>((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
        while (ii * (ii + 1) / 2 > q) --ii;
        while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
        i = pt_max + ii;
        j = pt_max + q - ii * (ii + 1) / 2;
      }
      const FrontDesc d = ds[b];
      if (i * kTile >= d.n) continue;
      int* prog = ctl + DAG_CTL + (size_t)b * nt;
      const int pt = d.p / kTile;
      if (j < pt) {
        if (i == j) dag_diagonal(d, b, j, prog, smem, &s_ready);
        else dag_offdiag(d, i, j, prog, smem, &s_ready);
      } else if (d.p > 0) {
        dag_trailing(d, i, j, min(aug_k0(d, i * kTile), d.p), d.p, prog, smem, &s_ready);
      }
      continue;
    }
    int r = t, kind = 0, col = 0;  // kind 0: E_col, 1: R_col
    if (t < etotal) {
      for (col = 0;; ++col) {
        const int es = batch * (max(nt - col - 2, 0) + 2);
        if (r < es) break;
        r -= es;
      }
    } else {
      kind = 1;
      r = t - etotal;
      col = r / rsize;
      r -= col * rsize;
    }
    if (kind == 0) {
      const int b = r % batch, slot = r / batch;
      const FrontDesc d = ds[b];
      const int pt = d.p / kTile, ntb = d.n / kTile;
      if (col >= pt) continue;
      int* prog = ctl + DAG_CTL + (size_t)b * nt;
      if (slot == 1 || slot == 2) {
        // slot 1: tile (c+2, c+1) for the worker's sub-diagonal solve of column c+1;
        // slot 2: tile (c+2, c+2), the worker's next pivot tile but one
        const int i = col + 2, j = slot == 1 ? col + 1 : col + 2;
        if (i >= ntb || j >= pt) continue;
        const int kb = aug_k0(d, i * kTile);
        if (kb > (col + 1) * kTile) continue;  // zero tile: the worker skips it too
        dag_prepare(d, i, j, kb, (col + 1) * kTile, prog,
                    (slot == 1 ? presub : prediag) + (size_t)b * nt + j, smem, &s_ready);
      } else {
        const int i = slot == 0 ? col + 2 : col + slot;
        if (i >= ntb) continue;
        dag_offdiag(d, i, col, prog, smem, &s_ready);
      }
    } else {
      const int b = r % batch, q = r / batch;
      int ii = static_cast<int>((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
      while (ii * (ii + 1) / 2 > q) --ii;
      while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
      const int jj = q - ii * (ii + 1) / 2;
      const FrontDesc d = ds[b];
      const int pt = d.p / kTile, i = pt + ii, j = pt + jj;
      if (i * kTile >= d.n) continue;
      // chunk col: columns [col * cw, (col + 1) * cw) of the K range, which starts
      // at the first nonzero column of row i (augmented rows)
      const int kz = min(aug_k0(d, i * kTile), d.p);
      const int kb = max(col * cw * kTile, kz), ke = min((col + 1) * cw * kTile, d.p);
      if (kb >= ke) continue;
      const int c0 = kz / (cw * kTile);  // first chunk with work
      int* flag = tflag + ((size_t)b * mt + ii) * mt + jj;
      wait_flag(flag, col - c0);
      dag_trailing(d, i, j, kb, ke, ctl + DAG_CTL + (size_t)b * nt, smem, &s_ready);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        st_release(flag, col - c0 + 1);
      }
    }
  }
}

// Forward sweep, one CTA per front (fronts that fill the GPU on their own):
// measured faster than the cluster kernel with CL = 1.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_front_forward(const SolveDesc* ds, const int* done) {
  if (done && *done) return;
  const SolveDesc d = ds[blockIdx.x];
  extern __shared__ double xs[];
  double* z = xs + d.n;  // 64 scratch
  const int tid = threadIdx.x;
  for (int r = tid; r < d.n; r += THREADS) xs[r] = d.x[r];
  __syncthreads();
  const size_t ld = d.n;
  for (int kb = 0; kb < d.p / kTile; ++kb) {
    const int k0 = kb * kTile;
    // z = Dinv_kb * x[k0:k0+64]: 4 threads per output row
    if (tid < 256) {
      const int row = tid >> 2, part = tid & 3;
      const double* dv = d.dinv + (size_t)kb * 64 * 64;
      double s = 0.0;
      for (int c = part; c < 64; c += 4) s += dv[(size_t)c * 64 + row] * xs[k0 + c];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (part == 0) z[row] = s;
    }
    __syncthreads();
    if (tid < 64) xs[k0 + tid] = z[tid];
    // x[r] -= sum_c L[r, k0+c] z[c] for rows below the block
    for (int r = k0 + kTile + tid; r < d.n; r += THREADS) {
      const double* col = d.a + (size_t)k0 * ld + r;
      double s[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) s[q] = 0.0;
#pragma unroll 2
      for (int c = 0; c < 64; c += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] += col[(size_t)(c + q) * ld] * z[c + q];
      }
      xs[r] -= ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    }
    __syncthreads();
  }
  for (int r = tid; r < d.n; r += THREADS) d.x[r] = xs[r];
}

// ---------------------------------------------------------------------------
// Front solves: one CTA, or a thread-block cluster of CL CTAs, per front (few fronts:
// more SMs and more loads in flight per front).  Row tile t (64 rows) belongs
// to CTA t % CL.  Forward: the owner of block kb forms z = Dinv_kb x_kb and
// the others read it through distributed shared memory; every CTA updates its
// own rows.  Backward: every CTA forms the partial sums of its rows; the owner
// adds them in rank order and solves the block.  One cluster barrier per block.
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;

template <int CL>
__global__ void __launch_bounds__(256) k_front_forward_cl(const SolveDesc* ds, const int* done) {
  if (done && *done) return;
  cg::cluster_group cl = cg::this_cluster();
  const int me = static_cast<int>(cl.block_rank());
  const SolveDesc d = ds[blockIdx.x / CL];
  extern __shared__ double xs[];
  double* zb = xs + d.n;      // [2][64] double-buffered block solution (read remotely)
  double* zl = zb + 128;      // local copy of a remote z
  const int tid = threadIdx.x;
  const int nt = d.n / kTile;
  for (int r = tid; r < d.n; r += 256)
    if ((r >> 6) % CL == me) xs[r] = d.x[r];
  __syncthreads();
  const size_t ld = d.n;
  for (int kb = 0; kb < d.p / kTile; ++kb) {
    const int k0 = kb * kTile, owner = kb % CL;
    double* zc = zb + (kb & 1) * 64;
    if (me == owner) {
      const int row = tid >> 2, part = tid & 3;
      const double* dv = d.dinv + (size_t)kb * 64 * 64;
      double sum = 0.0;
      for (int c = part; c < 64; c += 4) sum += dv[(size_t)c * 64 + row] * xs[k0 + c];
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (part == 0) zc[row] = sum;
      __syncthreads();
      if (tid < 64) xs[k0 + tid] = zc[tid];
    }
    cl.sync();
    const double* z = zc;
    if (me != owner) {
      const double* rz = cl.map_shared_rank(zc, owner);
      if (tid < 64) zl[tid] = rz[tid];
      __syncthreads();
      z = zl;
    }
    // own row tiles below the block: t = first, first + CL, ...
    int first = kb + 1 + ((me - (kb + 1) % CL) + CL) % CL;
    const int ntiles = first < nt ? (nt - 1 - first) / CL + 1 : 0;
    for (int i = tid; i < 64 * ntiles; i += 256) {
      const int r = (first + (i >> 6) * CL) * 64 + (i & 63);
      const double* col = d.a + (size_t)k0 * ld + r;
      double sq[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) sq[q] = 0.0;
#pragma unroll 2
      for (int c = 0; c < 64; c += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) sq[q] += col[(size_t)(c + q) * ld] * z[c + q];
      }
      xs[r] -= ((sq[0] + sq[1]) + (sq[2] + sq[3])) + ((sq[4] + sq[5]) + (sq[6] + sq[7]));
    }
    __syncthreads();
  }
  for (int r = tid; r < d.n; r += 256)
    if ((r >> 6) % CL == me) d.x[r] = xs[r];
  cl.sync();  // no CTA leaves while its shared memory may still be read
}

template <int CL>
__global__ void __launch_bounds__(256) k_front_backward_cl(const SolveDesc* ds, const int* done) {
  if (done && *done) return;
  cg::cluster_group cl = cg::this_cluster();
  const int me = static_cast<int>(cl.block_rank());
  const SolveDesc d = ds[blockIdx.x / CL];
  extern __shared__ __align__(16) double xs_[];
  double* dvs = xs_;                 // 64 x LDS: Dinv of this CTA's next block (cp.async prefetch)
  double* pb = xs_ + 64 * LDS;       // [2][CL][64] partial sums, written by every rank into the owner
  double* t = pb + 2 * CL * 64;      // 64
  double* xs = t + 64;               // the vector (own row tiles)
  __shared__ double part[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = d.n / kTile, nb = d.p / kTile;
  auto prefetch = [&](int kb) {
    const double* dv = d.dinv + (size_t)kb * 64 * 64;
    for (int q = tid; q < 64 * 32; q += 256) cp_async16(dvs + (q >> 5) * LDS + (q & 31) * 2, dv + (q >> 5) * 64 + (q & 31) * 2);
    cp_async_commit();
  };
  {
    // the last block this CTA owns comes first in the backward order
    int kl = nb - 1 - ((nb - 1 - me) % CL + CL) % CL;
    if (kl >= 0 && kl % CL == me) prefetch(kl);
  }
  for (int r = tid; r < d.n; r += 256) {
    if ((r >> 6) % CL != me) continue;
    double v = d.x[r];
    if (d.cmap && r >= d.p) {
      const int k = d.cmap[r - d.p];
      v = k >= 0 ? d.croot[k] : 0.0;
    }
    xs[r] = v;
  }
  __syncthreads();
  const size_t ld = d.n;
  for (int kb = d.p / kTile - 1; kb >= 0; --kb) {
    const int k0 = kb * kTile, owner = kb % CL;
    // partial t over this CTA's row tiles below the block: warp w owns columns
    // w, w+8, ..., w+56; a lane reads a row pair (16-byte loads)
    {
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
      const double* base = d.a + (size_t)(k0 + warp) * ld;
      const int first = kb + 1 + ((me - (kb + 1) % CL) + CL) % CL;
      for (int tt = first; tt < nt; tt += CL) {
        const int r = tt * 64 + 2 * lane;
        const double x0 = xs[r], x1 = xs[r + 1];
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldg(reinterpret_cast<const double2*>(base + (size_t)(8 * q) * ld + r));
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] += v[q].x * x0 + v[q].y * x1;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double sum = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) part[warp + 8 * q] = sum;
      }
    }
    __syncthreads();
    double* slot = pb + (kb & 1) * CL * 64 + me * 64;
    if (tid < 64) {
      double* dst = me == owner ? slot : cl.map_shared_rank(slot, owner);
      dst[tid] = part[tid];
    }
    cl.sync();
    if (me == owner) {
      cp_async_wait<0>();
      if (tid < 64) {
        const double* ps = pb + (kb & 1) * CL * 64;
        double sum = 0.0;
#pragma unroll
        for (int q = 0; q < CL; ++q) sum += ps[q * 64 + tid];
        t[tid] = xs[k0 + tid] - sum;
      }
      __syncthreads();
      // x[k0:k0+64] = Dinv^T t  (column `row` of Dinv)
      const int row = tid >> 2, prt = tid & 3;
      double sum = 0.0;
      for (int c = prt; c < 64; c += 4) sum += dvs[row * LDS + c] * t[c];
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      __syncthreads();
      if (prt == 0) xs[k0 + row] = sum;
      if (kb - CL >= 0) prefetch(kb - CL);  // overlaps the partial sums of the next CL blocks
    }
    __syncthreads();
  }
  for (int r = tid; r < d.n; r += 256)
    if ((r >> 6) % CL == me) d.x[r] = xs[r];
  cl.sync();
}

// ---------------------------------------------------------------------------
// Dataflow front sweeps (k_sweep_fwd_dag / k_sweep_bwd_dag): a batch of fronts
// as a pool of row-tile tasks over a persistent grid instead of one CTA (or
// cluster) per front.  Forward task (front f, row tile i) is left-looking: it
// streams the tiles L(i, k), k < min(i, nb) -- each factor tile is read by
// exactly one task, once -- and adds L(i, k) z_k as soon as block k is solved
// (per-front progress counter: release store by the solver, relaxed polls +
// one acquire fence by the readers).  The L loads are issued before the wait,
// so they are in flight while the pivot chain advances.  A block-row task then
// solves z_i = Dinv_i (x_i - acc) (Dinv_i prefetched into shared memory with
// cp.async at task start) and publishes it; coarse-row tasks (i >= nb) only
// subtract.  The backward sweep is the mirror image: task (f, kb) streams the
// tiles L(r, kb) of rows r > kb, last rows first, and solves x_kb = Dinv_kb^T
// (x_kb - sum_r L(r,kb)^T x_r).  Tasks are handed out level-major by an atomic
// ticket (row tile i of every front before row tile i + 1), so a task only waits
// for tasks with smaller tickets, which run on CTAs that already hold them: the
// schedule cannot deadlock for any grid.  Every sum is formed in a fixed order
// (deterministic).
// ---------------------------------------------------------------------------
constexpr int SW_LDS = 68;  // shared-memory ld of the Dinv tile (16-byte rows, few bank conflicts)

// cp.async of 16 bytes, or 16 bytes of zeros without touching global memory
__device__ __forceinline__ void cp_async16_or_zero(void* smem, const void* gmem, bool read) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = read ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// Dinv tile (lower triangular, 64x64 column-major) into shared memory: only
// the lower triangle of the `valid` leading rows/columns is read (row pairs
// reaching the diagonal); everything else is zero-filled.
__device__ __forceinline__ void sweep_prefetch_dinv(double* dvs, const double* dv, int valid) {
  for (int q = threadIdx.x; q < 64 * 32; q += 256) {
    const int c = q >> 5, r = (q & 31) * 2;
    cp_async16_or_zero(dvs + c * SW_LDS + r, dv + c * 64 + r, r + 1 >= c && r < valid && c < valid);
  }
  cp_async_commit();
}

// Valid (unpadded) rows of row tile i of a front.
__device__ __forceinline__ int sweep_valid_rows(const SolveDesc& d, int i) {
  const int nb = d.p / kTile;
  const int ne = d.ne > 0 ? d.ne : d.p, nc = d.ne > 0 ? d.nc : d.n - d.p;
  const int v = i < nb ? ne - i * kTile : nc - (i - nb) * kTile;
  return max(0, min(kTile, v));
}

// The last CTA to leave zeroes the counters for the next launch (no memset
// node per sweep; the buffer is zeroed once when allocated).
__device__ __forceinline__ void sweep_exit(int* ctl, int batch) {
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(ctl + 1, 1) == static_cast<int>(gridDim.x) - 1;
  }
  __syncthreads();
  if (s_last) {
    for (int q = threadIdx.x; q < batch + 2; q += blockDim.x) ctl[q] = 0;
    __threadfence();
  }
}

// Lane 0 of each warp polls (relaxed) and takes the acquire fence; __syncwarp
// orders the other lanes' reads of the published block after it.
__device__ __forceinline__ void sweep_wait(const int* prog, int need, int& ready) {
  if (ready >= need) return;
  if ((threadIdx.x & 31) == 0) {
    int v;
    while ((v = ld_relaxed(prog)) < need) {
    }
    fence_acquire();
    ready = v;
  }
  ready = __shfl_sync(0xffffffffu, ready, 0);
  __syncwarp();
}

__global__ void __launch_bounds__(256, 4) k_sweep_fwd_dag(const SolveDesc* ds, int batch, int levels, int* ctl,
                                                           const int* done) {
  if (done && *done) return;
  __shared__ __align__(16) double dvs[64 * SW_LDS];
  __shared__ double red[8][64];
  __shared__ double v[64];
  __shared__ int s_task;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* prog = ctl + 2;
  const long total = (long)levels * batch;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(ctl, 1);
    __syncthreads();
    const long t = s_task;
    if (t >= total) {
      sweep_exit(ctl, batch);
      return;
    }
    const int i = static_cast<int>(t / batch), f = static_cast<int>(t % batch);
    const SolveDesc d = ds[f];
    const int nt = d.n / kTile, nb = d.p / kTile;
    if (i < nt) {
      const bool solve = i < nb;
      const int vrows = sweep_valid_rows(d, i);
      if (solve) sweep_prefetch_dinv(dvs, d.dinv + (size_t)i * 64 * 64, vrows);
      const size_t ld = d.n;
      const int K = min(i, nb);
      const int ne = d.ne > 0 ? d.ne : d.p;
      double a0 = 0.0, a1 = 0.0;
      int ready = 0;
      const double* lrow = d.a + (size_t)(8 * warp) * ld + i * kTile + 2 * lane;
      const bool row_ok = 2 * lane < vrows;  // padding rows are never loaded
      for (int k = 0; k < K; ++k) {
        const double* base = lrow + (size_t)k * kTile * ld;
        const int cols = ne - (k * kTile + 8 * warp);  // valid columns of this warp's eight
        double2 L[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          L[q] = row_ok && q < cols ? __ldcs(reinterpret_cast<const double2*>(base + (size_t)q * ld))
                                    : make_double2(0.0, 0.0);
        sweep_wait(prog + f, k + 1, ready);
        const double* z = d.x + k * kTile + 8 * warp;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double zq = __ldcg(z + q);
          a0 += L[q].x * zq;
          a1 += L[q].y * zq;
        }
      }
      red[warp][2 * lane] = a0;
      red[warp][2 * lane + 1] = a1;
      __syncthreads();
      if (tid < 64) {
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) acc += red[w][tid];
        const double val = __ldcg(d.x + i * kTile + tid) - acc;
        if (solve) v[tid] = val;
        else d.x[i * kTile + tid] = val;
      }
      if (solve) {
        cp_async_wait<0>();
        __syncthreads();
        const int row = tid >> 2, part = tid & 3;
        double sum = 0.0;
        for (int c = part; c < 64; c += 4) sum += dvs[c * SW_LDS + row] * v[c];
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (part == 0) d.x[i * kTile + row] = sum;
        __syncthreads();
        if (tid == 0) st_release(prog + f, i + 1);  // fence.acq_rel + store: covers the CTA's writes (bar.sync)
      }
    }
    __syncthreads();  // s_task and the shared buffers are reused by the next task
  }
}

__device__ __forceinline__ double sweep_xin(const double* x, int p, const int* cmap, const double* croot, int r) {
  if (cmap && r >= p) {
    const int k = cmap[r - p];
    return k >= 0 ? croot[k] : 0.0;
  }
  return __ldcg(x + r);
}

__global__ void __launch_bounds__(256, 3) k_sweep_bwd_dag(const SolveDesc* ds, int batch, int levels, int* ctl,
                                                           const int* done) {
  if (done && *done) return;
  __shared__ __align__(16) double dvs[64 * SW_LDS];
  __shared__ double v[64];
  __shared__ int s_task;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* prog = ctl + 2;
  const long total = (long)levels * batch;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(ctl, 1);
    __syncthreads();
    const long t = s_task;
    if (t >= total) {
      sweep_exit(ctl, batch);
      return;
    }
    const int l = static_cast<int>(t / batch), f = static_cast<int>(t % batch);
    const SolveDesc d = ds[f];
    const int nt = d.n / kTile, nb = d.p / kTile;
    const int kb = nb - 1 - l;
    if (l == 0 && d.cmap)  // the first task of a front writes its coarse rows (others read croot)
      for (int r = d.p + tid; r < d.n; r += 256) d.x[r] = sweep_xin(d.x, d.p, d.cmap, d.croot, r);
    if (kb >= 0) {
      sweep_prefetch_dinv(dvs, d.dinv + (size_t)kb * 64 * 64, sweep_valid_rows(d, kb));
      const size_t ld = d.n;
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
      int ready = 0;
      const double* lcol = d.a + (size_t)(kb * kTile + 8 * warp) * ld + 2 * lane;
      const int cols = (d.ne > 0 ? d.ne : d.p) - (kb * kTile + 8 * warp);  // valid columns of this warp's eight
      for (int r = nt - 1; r > kb; --r) {
        const double* base = lcol + r * kTile;
        const bool row_ok = 2 * lane < sweep_valid_rows(d, r);  // padding rows are never loaded
        double2 L[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          L[q] = row_ok && q < cols ? __ldcs(reinterpret_cast<const double2*>(base + (size_t)q * ld))
                                    : make_double2(0.0, 0.0);
        if (r < nb) sweep_wait(prog + f, nb - r, ready);
        const int row = r * kTile + 2 * lane;
        const double x0 = sweep_xin(d.x, d.p, d.cmap, d.croot, row), x1 = sweep_xin(d.x, d.p, d.cmap, d.croot, row + 1);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] += L[q].x * x0 + L[q].y * x1;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double sum = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) v[8 * warp + q] = __ldcg(d.x + kb * kTile + 8 * warp + q) - sum;
      }
      cp_async_wait<0>();
      __syncthreads();
      const int row = tid >> 2, part = tid & 3;
      double sum = 0.0;
      for (int c = part; c < 64; c += 4) sum += dvs[row * SW_LDS + c] * v[c];
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (part == 0) d.x[kb * kTile + row] = sum;
      __syncthreads();
      if (tid == 0) st_release(prog + f, l + 1);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// One large front (the root when R^{-1} is not formed) over the whole GPU:
// a cooperative grid of G CTAs, row tile t owned by CTA t % G, the CTA's own
// rows kept in shared memory.  Forward: at block kb every CTA updates its rows
// below with z_kb; the owner of tile kb+1 then forms z_{kb+1} (its rows are
// final) -- one grid barrier per block.  Backward: every CTA writes the
// partial sums of its rows, and after the barrier the owner of tile kb adds
// them in CTA order and solves the block (deterministic).
// ---------------------------------------------------------------------------
// out = Dinv_kb * xb (64 values); the owner's copy of the block := out
__device__ __forceinline__ void big_z(const SolveDesc& d, int kb, double* xb, double* out) {
  const int tid = threadIdx.x, row = tid >> 2, part = tid & 3;
  const double* dv = d.dinv + (size_t)kb * 64 * 64;
  double sum = 0.0;
  for (int c = part; c < 64; c += 4) sum += dv[(size_t)c * 64 + row] * xb[c];
  sum += __shfl_xor_sync(0xffffffffu, sum, 1);
  sum += __shfl_xor_sync(0xffffffffu, sum, 2);
  __syncthreads();
  if (part == 0) {
    out[row] = sum;
    xb[row] = sum;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_big_forward(const SolveDesc* ds, double* zbuf, const int* done) {
  if (done && *done) return;
  cg::grid_group grid = cg::this_grid();
  const SolveDesc d = ds[0];
  const int G = gridDim.x, me = blockIdx.x, tid = threadIdx.x;
  const int nt = d.n / kTile, nb = d.p / kTile;
  extern __shared__ double xs[];  // own tiles: tile t at (t / G) * 64
  __shared__ double zs[64];
  for (int t = me; t < nt; t += G)
    for (int r = tid; r < 64; r += 256) xs[(t / G) * 64 + r] = d.x[(size_t)t * 64 + r];
  __syncthreads();
  const size_t ld = d.n;
  if (nb > 0 && me == 0) big_z(d, 0, xs, zbuf);
  grid.sync();
  for (int kb = 0; kb < nb; ++kb) {
    if (tid < 64) zs[tid] = zbuf[(kb & 1) * 64 + tid];
    __syncthreads();
    const int k0 = kb * kTile;
    const int first = kb + 1 + ((me - (kb + 1) % G) % G + G) % G;  // own tiles below the block
    const int ntl = first < nt ? (nt - 1 - first) / G + 1 : 0;
    for (int i = tid; i < 64 * ntl; i += 256) {
      const int t = first + (i >> 6) * G, r = t * 64 + (i & 63);
      const double* col = d.a + (size_t)k0 * ld + r;
      double sq[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) sq[q] = 0.0;
#pragma unroll 2
      for (int c = 0; c < 64; c += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) sq[q] += col[(size_t)(c + q) * ld] * zs[c + q];
      }
      xs[(t / G) * 64 + (i & 63)] -= ((sq[0] + sq[1]) + (sq[2] + sq[3])) + ((sq[4] + sq[5]) + (sq[6] + sq[7]));
    }
    __syncthreads();
    if (kb + 1 < nb && (kb + 1) % G == me) big_z(d, kb + 1, xs + ((kb + 1) / G) * 64, zbuf + ((kb + 1) & 1) * 64);
    grid.sync();
  }
  for (int t = me; t < nt; t += G)
    for (int r = tid; r < 64; r += 256) d.x[(size_t)t * 64 + r] = xs[(t / G) * 64 + r];
}

__global__ void __launch_bounds__(256) k_big_backward(const SolveDesc* ds, double* pbuf, const int* done) {
  if (done && *done) return;
  cg::grid_group grid = cg::this_grid();
  const SolveDesc d = ds[0];
  const int G = gridDim.x, me = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nt = d.n / kTile, nb = d.p / kTile;
  extern __shared__ double xs[];
  __shared__ double part[64], tv[64], red4[4][64];
  for (int t = me; t < nt; t += G)
    for (int r = tid; r < 64; r += 256) {
      const int row = t * 64 + r;
      double v = d.x[row];
      if (d.cmap && row >= d.p) {
        const int k = d.cmap[row - d.p];
        v = k >= 0 ? d.croot[k] : 0.0;
      }
      xs[(t / G) * 64 + r] = v;
    }
  __syncthreads();
  const size_t ld = d.n;
  for (int kb = nb - 1; kb >= 0; --kb) {
    const int k0 = kb * kTile;
    {
      double acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.0;
      const double* base = d.a + (size_t)(k0 + warp) * ld;
      const int first = kb + 1 + ((me - (kb + 1) % G) % G + G) % G;
      for (int t = first; t < nt; t += G) {
        const int r = t * 64 + 2 * lane;
        const double x0 = xs[(t / G) * 64 + 2 * lane], x1 = xs[(t / G) * 64 + 2 * lane + 1];
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldg(reinterpret_cast<const double2*>(base + (size_t)(8 * q) * ld + r));
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] += v[q].x * x0 + v[q].y * x1;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        double sum = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) part[warp + 8 * q] = sum;
      }
    }
    __syncthreads();
    if (tid < 64) pbuf[((size_t)(kb & 1) * G + me) * 64 + tid] = part[tid];
    grid.sync();
    if (kb % G == me) {
      double* xb = xs + (kb / G) * 64;
      {
        // sum of the CTAs' partials: four fixed-order strands, then combined
        const int c = tid & 63, q = tid >> 6;
        const double* ps = pbuf + (size_t)(kb & 1) * G * 64 + c;
        double s0 = 0.0, s1 = 0.0;
        int g = q;
        for (; g + 4 < G; g += 8) {
          s0 += ps[(size_t)g * 64];
          s1 += ps[(size_t)(g + 4) * 64];
        }
        if (g < G) s0 += ps[(size_t)g * 64];
        red4[q][c] = s0 + s1;
      }
      __syncthreads();
      if (tid < 64) tv[tid] = xb[tid] - ((red4[0][tid] + red4[1][tid]) + (red4[2][tid] + red4[3][tid]));
      __syncthreads();
      const int row = tid >> 2, prt = tid & 3;
      const double* dv = d.dinv + (size_t)kb * 64 * 64 + (size_t)row * 64;
      double sum = 0.0;
      for (int c = prt; c < 64; c += 4) sum += dv[c] * tv[c];
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      __syncthreads();
      if (prt == 0) xb[row] = sum;
    }
    __syncthreads();
  }
  for (int t = me; t < nt; t += G)
    for (int r = tid; r < 64; r += 256) d.x[(size_t)t * 64 + r] = xs[(t / G) * 64 + r];
}

// 32x32 tiles of the lower triangle: each is read once down its columns
// (coalesced), written in place and, transposed through shared memory, into the
// mirrored tile -- both stores run down columns too.
__global__ void __launch_bounds__(256) k_copy_trailing(const TrailDesc* ds) {
  const TrailDesc d = ds[blockIdx.y];
  const int m = d.n - d.p, nt = (m + 31) / 32;
  const long tiles = (long)nt * (nt + 1) / 2;
  __shared__ double t[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (long q = blockIdx.x; q < tiles; q += gridDim.x) {
    int ti = static_cast<int>((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
    while ((long)ti * (ti + 1) / 2 > q) --ti;
    while ((long)(ti + 1) * (ti + 2) / 2 <= q) ++ti;
    const int tj = static_cast<int>(q - (long)ti * (ti + 1) / 2);  // tj <= ti
    const int r = ti * 32 + tx;
    for (int cc = ty; cc < 32; cc += 8) {
      const int c = tj * 32 + cc;
      double v = 0.0;
      if (r < m && c < m) {
        // diagonal tiles: the strictly upper entries come from their mirror images
        v = r >= c ? d.a[(size_t)(d.p + c) * d.n + d.p + r] : d.a[(size_t)(d.p + r) * d.n + d.p + c];
        d.s[(size_t)c * m + r] = v;
      }
      t[cc][tx] = v;
    }
    __syncthreads();
    if (ti != tj) {
      const int r2 = tj * 32 + tx;  // row of the mirrored tile
      for (int cc = ty; cc < 32; cc += 8) {
        const int c2 = ti * 32 + cc;
        if (r2 < m && c2 < m) d.s[(size_t)c2 * m + r2] = t[tx][cc];
      }
    }
    __syncthreads();
  }
}

int configure_device() {
  const int gemm_smem = 4 * KC * LDS * sizeof(double);
  cudaFuncSetAttribute(k_syrk_column, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem);
  cudaFuncSetAttribute(k_syrk_trailing, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem);
  cudaFuncSetAttribute(k_syrk_column_splitk, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm_smem);
  cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * LDS * (int)sizeof(double));
  cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * LDS * (int)sizeof(double));
  cudaFuncSetAttribute(k_front_forward<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_backward_cl<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_big_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_big_backward, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_forward_cl<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_forward_cl<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_backward_cl<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_backward_cl<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_forward_cl<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_backward_cl<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_forward_cl<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_backward_cl<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_front_forward_cl<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_front_backward_cl<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return 1;
}

std::atomic<long long> g_launches{0};

// Grow-only split-K workspace, one per stream: work on one stream is ordered,
// and engines (one stream each, possibly driven by different host threads of
// one process) never share a workspace.
double* stream_workspace(int slot, size_t doubles, cudaStream_t stream) {
  struct Ws {
    double* p = nullptr;
    size_t cap = 0;
  };
  static std::mutex mu;
  static std::map<std::pair<cudaStream_t, int>, Ws> ws;
  std::lock_guard<std::mutex> lk(mu);
  Ws& w = ws[{stream, slot}];
  if (doubles > w.cap) {
    if (w.p) {
      cudaStreamSynchronize(stream);  // the old buffer may still be in use on this stream
      cudaFree(w.p);
    }
    w.p = nullptr;
    if (cudaMalloc(&w.p, doubles * sizeof(double)) != cudaSuccess) {
      w.cap = 0;
      return nullptr;
    }
    w.cap = doubles;
  }
  return w.p;
}
// Counters of the dataflow sweeps: zeroed once when (re)allocated, then kept
// zero by the kernels themselves (sweep_exit).  Fixed minimum size so captured
// graphs keep a valid pointer.
int* sweep_counters(size_t ints, cudaStream_t stream) {
  struct Ws {
    int* p = nullptr;
    size_t cap = 0;
  };
  static std::mutex mu;
  static std::map<cudaStream_t, Ws> ws;
  std::lock_guard<std::mutex> lk(mu);
  Ws& w = ws[stream];
  if (ints > w.cap) {
    if (w.p) {
      cudaStreamSynchronize(stream);
      cudaFree(w.p);
    }
    const size_t cap = std::max<size_t>(16384, ints);
    if (cudaMalloc(&w.p, cap * sizeof(int)) != cudaSuccess) throw std::runtime_error("sweep counters");
    cudaMemsetAsync(w.p, 0, cap * sizeof(int), stream);
    w.cap = cap;
  }
  return w.p;
}

// slot 0: split-K partial tiles; slot 1: the large-front sweeps (small, never
// reallocated once sized, so captured PCG graphs keep a valid pointer)
double* splitk_workspace(size_t doubles, cudaStream_t stream) { return stream_workspace(0, doubles, stream); }

}  // namespace

void ensure_sweep_workspace(cudaStream_t stream) { sweep_counters(16384, stream); }

int per_device(const void* key, int (*make)()) {
  static std::mutex m;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(m);
    auto it = cache.find({dev, key});
    if (it != cache.end()) return it->second;
  }
  const int v = make();  // outside the lock: may launch CUDA API calls
  std::lock_guard<std::mutex> g(m);
  return cache.emplace(std::make_pair(dev, key), v).first->second;
}

namespace {
int query_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}
}  // namespace

int sm_count() { return per_device(reinterpret_cast<const void*>(&query_sm_count), query_sm_count); }

void count_launch(long long n) { g_launches += n; }
long long launch_count() { return g_launches.load(); }

void chol_trace(bool on, unsigned long long* out) {
  const int v = on ? 1 : 0;
  cudaMemcpyToSymbol(g_dag_trace_on, &v, sizeof(int));
  if (out) {
    cudaMemcpyFromSymbol(out, g_dag_trace, sizeof(unsigned long long) * 128);
    cudaMemcpyFromSymbol(out + 128, g_pf_trace, sizeof(unsigned long long) * 16);
  }
}

namespace {
// Dataflow schedule (k_chol_dag; measured faster than the tiled launches on
// every front kind of configs 1-5) or one launch per tile-column step (tiled).
// BDDC_B200_CHOL=dag|tiled overrides.
bool use_dag(int batch, int nt, int pt) {
  if (const char* env = std::getenv("BDDC_B200_CHOL"); env && *env) {
    if (std::string(env) == "dag") return true;
    if (std::string(env) == "tiled") return false;
  }
  (void)batch;
  (void)nt;
  (void)pt;
  return true;
}

std::atomic<int> g_shared_device{0};

void partial_cholesky_dag(const FrontDesc* d_descs, int batch, int nt, int pt, int mt, cudaStream_t stream) {
  const int smem = 4 * KC * LDS * sizeof(double);
  const int per_sm = per_device(reinterpret_cast<const void*>(&k_chol_dag), [] {
    const int smem = 4 * KC * LDS * sizeof(double);
    int n = 0;
    cudaFuncSetAttribute(k_chol_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_chol_dag, DAG_THREADS, smem);
    return n > 0 ? n : 1;
  });
  const long resident = (long)per_sm * sm_count();
  // chunked mode (dedicated diagonal workers, trailing updates per column) when
  // the fronts leave most of the grid to the queue; BDDC_B200_DAGW=0|1 overrides
  bool chunked = 2L * batch <= sm_count() && resident >= 2L * sm_count();
  if (g_shared_device.load(std::memory_order_relaxed) > 0) chunked = false;  // see shared_device_users
  if (const char* e = std::getenv("BDDC_B200_DAGW"); e && *e) chunked = *e == '1' && 3L * batch <= resident;
  long total;
  int cw = 1, bq = 6;
  size_t ints = DAG_CTL + (size_t)batch * nt;
  if (chunked) {
    cw = std::max(1, (pt + 2) / 3);  // about three trailing chunks per tile
    const int nchunk = (pt + cw - 1) / cw;
    total = (long)nchunk * batch * mt * (mt + 1) / 2;
    for (int c = 0; c < pt; ++c) total += (long)batch * (std::max(nt - c - 2, 0) + 2);
    ints += (size_t)batch * mt * mt + 2 * (size_t)batch * nt;
  } else {
    total = (long)batch * nt * (nt + 1) / 2;
  }
  int* ctl = reinterpret_cast<int*>(stream_workspace(2, (ints + 1) / 2, stream));
  if (!ctl) throw std::runtime_error("partial_cholesky: workspace allocation failed");
  cudaMemsetAsync(ctl, 0, ints * sizeof(int), stream);
  const int grid = static_cast<int>(std::min<long>(total + (chunked ? batch : 0), resident));
  k_chol_dag<<<grid, DAG_THREADS, smem, stream>>>(d_descs, batch, nt, pt, mt, ctl, static_cast<int>(total),
                                                 chunked ? 1 : 0, cw, bq);
  count_launch(1);
}
}  // namespace

void shared_device_users(int delta) { g_shared_device.fetch_add(delta, std::memory_order_relaxed); }

void partial_cholesky(const FrontDesc* d_descs, int batch, int max_n, int max_p, int max_m,
                      cudaStream_t stream) {
  if (batch == 0) return;
  per_device(reinterpret_cast<const void*>(&configure_device), configure_device);
  if (max_p > 0 && use_dag(batch, max_n / kTile, max_p / kTile)) {
    partial_cholesky_dag(d_descs, batch, max_n / kTile, max_p / kTile, max_m / kTile, stream);
    return;
  }
  const int gemm_smem = 4 * KC * LDS * sizeof(double);
  const int panel_smem = 2 * 64 * LDS * sizeof(double);
  const int nt = max_n / kTile, pt = max_p / kTile;
  for (int j = 0; j < pt; ++j) {
    if (j > 0) {
      const int tiles = nt - j;
      const long ctas = (long)tiles * batch;
      const int K = j * kTile;
      int nsplit = 1;
      if (ctas < 2L * sm_count() && K >= 8 * KC)
        nsplit = static_cast<int>(std::min<long>({16L, K / (4 * KC), (2L * sm_count() + ctas - 1) / ctas}));
      double* work = nsplit > 1 ? splitk_workspace((size_t)ctas * nsplit * 64 * 64, stream) : nullptr;
      if (nsplit > 1 && work) {
        k_syrk_column_splitk<<<dim3(tiles, batch, nsplit), GEMM_THREADS, gemm_smem, stream>>>(d_descs, j, nsplit,
                                                                                             tiles, work);
        k_splitk_reduce<<<dim3(tiles, batch), 256, 0, stream>>>(d_descs, j, nsplit, tiles, work);
        count_launch(2);
      } else {
        k_syrk_column<<<dim3(tiles, batch), GEMM_THREADS, gemm_smem, stream>>>(d_descs, j);
        count_launch(1);
      }
    }
    k_panel<<<dim3(1, batch), PANEL_THREADS, panel_smem, stream>>>(d_descs, j);
    count_launch(1);
    if (nt - j - 1 > 0) {
      k_trsm<<<dim3(nt - j - 1, batch), GEMM_THREADS, 2 * 64 * LDS * (int)sizeof(double), stream>>>(d_descs, j);
      count_launch(1);
    }
  }
  // trailing tiles: worst case over the batch is bounded by the largest trailing block
  const long mt = max_m / kTile;
  const long max_tr = mt * (mt + 1) / 2;
  if (max_p > 0 && max_tr > 0) {
    k_syrk_trailing<<<dim3(static_cast<unsigned>(max_tr), batch), GEMM_THREADS, gemm_smem, stream>>>(d_descs);
    count_launch(1);
  }
}

namespace {
// CTAs per front: a cluster of 16, 8, 4 or 2 when the fronts alone cannot fill
// the GPU (about three CTAs per SM), else one.
int sweep_cluster(int batch, int max_cl) {
  const long cap = 3L * sm_count();
  if (max_cl >= 16 && (long)batch * 16 <= cap) return 16;
  if (max_cl >= 8 && (long)batch * 8 <= cap) return 8;
  if ((long)batch * 4 <= cap) return 4;
  if ((long)batch * 2 <= cap) return 2;
  return 1;
}

template <class K>
void launch_cluster(K kern, int cl, int batch, size_t smem, cudaStream_t stream, const SolveDesc* d, const int* done) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(batch * cl);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, d, done) != cudaSuccess) {
    // the device could not place a cluster this wide (large clusters are not
    // portable): clear the error; the caller retries narrower
    (void)cudaGetLastError();
    throw std::runtime_error("cluster launch");
  }
}
}  // namespace

namespace {
// one front spread over the GPU when it is large (BDDC_B200_BIGSWEEP=0|1 overrides)
bool big_sweep(int batch, int max_n) {
  if (batch != 1) return false;
  if (const char* env = std::getenv("BDDC_B200_BIGSWEEP")) {
    if (*env == '0') return false;
    if (*env == '1') return true;
  }
  return max_n >= 8192;
}

template <class K>
void launch_big(K kern, int max_n, size_t ws_per_cta, cudaStream_t stream, const SolveDesc* d, const int* done) {
  const int G = sm_count();
  const int tiles = (max_n / kTile + G - 1) / G;
  const size_t smem = (size_t)tiles * 64 * sizeof(double);
  double* buf = stream_workspace(1, std::max<size_t>(ws_per_cta, 2 * 64) * G, stream);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, d, buf, done);
}
}  // namespace

namespace {
// Dataflow sweeps for batches of two or more fronts (BDDC_B200_SWEEP=dag|cluster
// overrides; the cluster kernels are the round-1 path).
bool dag_sweep(int batch) {
  if (const char* e = std::getenv("BDDC_B200_SWEEP"); e && *e) return std::string(e) == "dag";
  return batch >= 2;
}

using SweepKernel = void (*)(const SolveDesc*, int, int, int*, const int*);
void launch_sweep_dag(SweepKernel kern, const SolveDesc* d_descs, int batch, int levels, cudaStream_t stream,
                      const int* done) {
  // ctl[0] = ticket counter, ctl[1 + f] = progress of front f; fixed minimum
  // size so captured graphs keep a valid pointer
  int* ctl = sweep_counters(batch + 2, stream);
  const int occ = kern == k_sweep_fwd_dag
                      ? per_device(reinterpret_cast<const void*>(&k_sweep_fwd_dag), [] {
                          int o = 0;
                          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_sweep_fwd_dag, 256, 0);
                          return o;
                        })
                      : per_device(reinterpret_cast<const void*>(&k_sweep_bwd_dag), [] {
                          int o = 0;
                          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_sweep_bwd_dag, 256, 0);
                          return o;
                        });
  const long tasks = (long)levels * batch;
  // a front's chain keeps little more than one task streaming at a time: CTAs
  // beyond ~2 per front only spin on the progress counters (measured on cfg4,
  // 216 fronts: 432 CTAs beat 297 and the resident 592 / 444)
  const long want = std::min<long>((long)std::max(occ, 1) * sm_count(), std::max<long>(sm_count(), 2L * batch));
  const int grid = static_cast<int>(std::max<long>(1, std::min<long>(tasks, want)));
  kern<<<grid, 256, 0, stream>>>(d_descs, batch, levels, ctl, done);
  count_launch(1);
}
}  // namespace

void front_forward(const SolveDesc* d_descs, int batch, int max_n, cudaStream_t stream, const int* done) {
  if (batch == 0) return;
  per_device(reinterpret_cast<const void*>(&configure_device), configure_device);
  if (big_sweep(batch, max_n)) {
    launch_big(k_big_forward, max_n, 2, stream, d_descs, done);  // z double buffer (2 x 64 <= 2 G)
    count_launch(1);
    return;
  }
  if (dag_sweep(batch)) {
    launch_sweep_dag(k_sweep_fwd_dag, d_descs, batch, std::max(1, max_n / kTile), stream, done);
    return;
  }
  const int cl = sweep_cluster(batch, 4);  // measured: wider forward clusters are slower
  const size_t smem = (max_n + 64 * 3) * sizeof(double);
  if (cl == 16) launch_cluster(k_front_forward_cl<16>, 16, batch, smem, stream, d_descs, done);
  else if (cl == 8) launch_cluster(k_front_forward_cl<8>, 8, batch, smem, stream, d_descs, done);
  else if (cl == 4) launch_cluster(k_front_forward_cl<4>, 4, batch, smem, stream, d_descs, done);
  else if (cl == 2) launch_cluster(k_front_forward_cl<2>, 2, batch, smem, stream, d_descs, done);
  else k_front_forward<256><<<batch, 256, (max_n + 64) * sizeof(double), stream>>>(d_descs, done);
  count_launch(1);
}

void front_backward(const SolveDesc* d_descs, int batch, int max_n, cudaStream_t stream, const int* done) {
  if (batch == 0) return;
  per_device(reinterpret_cast<const void*>(&configure_device), configure_device);
  if (big_sweep(batch, max_n)) {
    launch_big(k_big_backward, max_n, 2 * 64, stream, d_descs, done);  // partials: 2 x G x 64
    count_launch(1);
    return;
  }
  if (dag_sweep(batch)) {
    launch_sweep_dag(k_sweep_bwd_dag, d_descs, batch, std::max(1, max_n / kTile), stream, done);
    return;
  }
  static int max_cl = 16;  // lowered once if the device refuses a cluster width
  int cl = sweep_cluster(batch, max_cl);
  const size_t smem = (64 * LDS + max_n + 64 + 2 * 16 * 64) * sizeof(double);
  while (cl >= 8) {
    try {
      if (cl == 16) launch_cluster(k_front_backward_cl<16>, 16, batch, smem, stream, d_descs, done);
      else launch_cluster(k_front_backward_cl<8>, 8, batch, smem, stream, d_descs, done);
      count_launch(1);
      return;
    } catch (const std::runtime_error&) {
      max_cl = cl / 2;
      cl = sweep_cluster(batch, max_cl);
    }
  }
  if (cl == 4) launch_cluster(k_front_backward_cl<4>, 4, batch, smem, stream, d_descs, done);
  else if (cl == 2) launch_cluster(k_front_backward_cl<2>, 2, batch, smem, stream, d_descs, done);
  else k_front_backward_cl<1><<<batch, 256, smem, stream>>>(d_descs, done);
  count_launch(1);
}

void copy_trailing_full(const TrailDesc* d_descs, int batch, int max_m, cudaStream_t stream) {
  if (batch == 0) return;
  const long nt = (max_m + 31) / 32;
  const int blocks = static_cast<int>(std::min<long>(nt * (nt + 1) / 2, 1024));
  k_copy_trailing<<<dim3(blocks, batch), 256, 0, stream>>>(d_descs);
  count_launch(1);
}

}  // namespace b200
