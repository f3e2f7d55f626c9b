// Adaptive face eigenproblems on the device (adaptive.cpp:30-125, pair.cpp:32-209).
//
// The reference forms, per face pair, the dense pencil (J^T S J, Z^T S Z) of
// dimension ~2 n_B and eigendecomposes it twice on the host (dense_eig.cpp:77-126).
// Here the same pencil is reduced exactly before any eigensolve:
//   * lhs = J^T S J only involves the jump coordinates alpha of the shared globs
//     (J = Z - avg Z vanishes on corner, continuous and outer columns), and
//     lhs = K^T M K with M = 4 (D_{1-rho} S_i,ff D_{1-rho} + D_rho S_j,ff D_rho);
//   * the Rayleigh quotient is maximized over the other coordinates, so rhs is
//     replaced by its Schur complement B onto alpha: outer dofs of each side are
//     eliminated from S_i, S_j (batched DMMA partial Cholesky), the two sides are
//     glued in [corner | continuous | alpha] coordinates (Q), and corner +
//     continuous are eliminated (partial Cholesky); the rigid-body null space of
//     floating pairs is deflated exactly by a rank-nm shift sigma N N^T;
//   * C = L^{-1} lhs L^{-T} (B = L L^T) is formed by two augmented partial
//     factorizations and diagonalized by a parallel cyclic Jacobi sweep per pair;
//   * eigenvectors map back by alpha = L^{-T} y, and the jump functional
//     a = (1 - rho) d_i - rho d_j (adaptive.cpp:51-58) equals 1/2 M K alpha.
// Eigenvalues, their count and the functionals match generalized_eig_sym
// (modulo null(rhs)) in exact arithmetic; the host then runs the reference's
// selection, splitting, normalization and rank filter unchanged.
#include "pairs.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include "dense.cuh"
#include "devbuf.cuh"
#include "engine.hpp"

namespace b200 {

namespace {

inline int rup(int v, int m) { return (v + m - 1) / m * m; }

struct PairDev {
  // sides
  const double* S[2];   // interface Schur of each side (PB x PB)
  int PB[2];
  const int* pos[2];    // kept slots [corner | shared] -> boundary position in S_s
  double* G[2];         // side fronts
  int NG[2], PO[2], no[2];
  int nc, nf, nj, nm, PQ, PJ, k;
  double* Q;            // NQ = PQ + PJ
  double* F3;           // 2 PJ
  double* F4;           // 2 PJ
  double* M;            // nf x nf
  // kernel basis K (nf x nj), compact: column b = e_{unit} + sum_a kvals[vals+a] e_{krows[rows+a]}
  const int4* kc;       // per column: (unit row, r, rows offset, vals offset)
  const int* krows;
  const double* kvals;
  double* H;            // nf x nj scratch
  const double* N;      // nm x (nc + nf) row-major, orthonormal
  const double* rho;    // nf
  double* A;            // eigensolver workspace (packed matrix + scratch when not in shared memory)
  int* need;            // eigenvectors formed by k_syevx (the enforced count): the rest are zeros
  double* evals;        // k
  double* vecs;         // 2PJ x k (solve vectors, column m at m*2PJ)
  double* func;         // nf x k
};

// sum_u f(u) K[u][b] for the compact kernel basis
template <class F>
__device__ __forceinline__ double kdot(const PairDev& d, int b, F f) {
  const int4 c = d.kc[b];
  double s = f(c.x);
  for (int a = 0; a < c.y; ++a) s += d.kvals[c.w + a] * f(d.krows[c.z + a]);
  return s;
}

}  // namespace

// Grow-only arenas of the pair reductions, reused across enrich() calls.
// Gather of a front [outer | kept] from a symmetric source (lower triangle
// read), identity on the padding: the hub fronts from S_s and the side fronts
// from the hubs' Schur complements.
struct GatherDesc {
  const double* src;
  const int* pos;  // front index (outer, then kept) -> source index
  double* dst;
  int ld, N, PO, no, m1;
  int full;  // src holds both triangles (the substructure's S): every read runs down a column (coalesced)
};

struct PairBuffers {
  DBuf<double> G, Q, F, Dv, M, KV, H, N, R, A, E, W, Fu, Hub, DvH;
  DBuf<int> Pv, info, KR, Gpos, Hpos, hinfo;
  HBuf<double> h_ev, h_fu;  // page-locked result copies
  HBuf<int> h_inf;
  DBuf<GatherDesc> ghub, gside;
  DBuf<FrontDesc> dHub;
  DBuf<int4> KC;
  DBuf<PairDev> dpd;
  DBuf<FrontDesc> dG, dQ, d3, d4;
  DBuf<SolveDesc> dsv;
  DBuf<int> svoff, need;  // first descriptor of each pair in dsv; eigenvectors formed per pair
  UploadBatch up_index, up_desc;  // per chunk: index arrays, then descriptors (one copy each)
};

PairEngine::PairEngine() : bufs_(new PairBuffers) {}
PairEngine::~PairEngine() = default;

namespace {

__global__ void k_gather_front(const GatherDesc* gd) {
  const GatherDesc d = gd[blockIdx.y];
  const int col = blockIdx.x;
  if (col >= d.N) return;
  auto valid = [&](int a) { return a < d.no || (a >= d.PO && a < d.PO + d.m1); };
  auto bidx = [&](int a) { return a < d.no ? a : d.no + (a - d.PO); };
  const bool vc = valid(col);
  const int pc = vc ? d.pos[bidx(col)] : 0;
  double* out = d.dst + (size_t)col * d.N;
  for (int r = threadIdx.x; r < d.N; r += blockDim.x) {
    double v;
    if (vc && valid(r)) {
      const int pr = d.pos[bidx(r)];
      const int hi = pr >= pc ? pr : pc, lo = pr >= pc ? pc : pr;
      v = d.full ? d.src[(size_t)pc * d.ld + pr] : d.src[(size_t)lo * d.ld + hi];
    } else {
      v = (r == col) ? 1.0 : 0.0;
    }
    out[r] = v;
  }
}

__device__ __forceinline__ double hat(const PairDev& d, int side, int a, int b) {
  // condensed side matrix (lower triangle of the trailing block)
  const int hi = a >= b ? a : b, lo = a >= b ? b : a;
  const int PO = d.PO[side], NG = d.NG[side];
  return d.G[side][(size_t)(PO + lo) * NG + PO + hi];
}

// (c) M = 4 (D_{1-rho} C_i D_{1-rho} + D_rho C_j D_rho), C = original S on shared slots
__global__ void k_build_M(const PairDev* pd) {
  const PairDev d = pd[blockIdx.y];
  const int nf = d.nf;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nf * nf; e += gridDim.x * blockDim.x) {
    const int t = e % nf, u = e / nf;
    const int base_i = d.nc, base_j = d.nc;  // pos points at the kept slots [corner | shared]
    const double ci = d.S[0][(size_t)d.pos[0][base_i + u] * d.PB[0] + d.pos[0][base_i + t]];
    const double cj = d.S[1][(size_t)d.pos[1][base_j + u] * d.PB[1] + d.pos[1][base_j + t]];
    const double rt = d.rho[t], ru = d.rho[u];
    d.M[(size_t)u * nf + t] = 4.0 * ((1.0 - rt) * (1.0 - ru) * ci + rt * ru * cj);
  }
}

// (d1) H = (hat_i + hat_j)_ff K   (nf x nj)
__global__ void k_build_H(const PairDev* pd) {
  const PairDev d = pd[blockIdx.y];
  const int nf = d.nf, nj = d.nj, nc = d.nc;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nf * nj; e += gridDim.x * blockDim.x) {
    const int t = e % nf, b = e / nf;
    d.H[(size_t)b * nf + t] =
        kdot(d, b, [&](int u) { return hat(d, 0, nc + t, nc + u) + hat(d, 1, nc + t, nc + u); });
  }
}

// (d2) Q in [corner | continuous | pad | alpha | pad] coordinates (lower part + pads)
__global__ void k_assemble_Q(const PairDev* pd) {
  const PairDev d = pd[blockIdx.y];
  const int nc = d.nc, nf = d.nf, nj = d.nj, m1 = nc + nf, PQ = d.PQ, NQ = d.PQ + d.PJ;
  __shared__ double sig;
  if (threadIdx.x == 0) sig = 0.0;
  __syncthreads();
  if (d.nm > 0) {  // sigma = max diagonal of the glued corner/continuous block
    double mx = 0.0;
    for (int a = threadIdx.x; a < m1; a += blockDim.x) mx = fmax(mx, hat(d, 0, a, a) + hat(d, 1, a, a));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    __shared__ double wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
      sig = m;
    }
    __syncthreads();
  }
  const long total = (long)NQ * NQ;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e % NQ), c = static_cast<int>(e / NQ);
    if (r < c) continue;
    double v = 0.0;
    if (r < m1 && c < m1) {
      v = hat(d, 0, r, c) + hat(d, 1, r, c);
      for (int k = 0; k < d.nm; ++k) v += sig * d.N[(size_t)k * m1 + r] * d.N[(size_t)k * m1 + c];
    } else if (r >= PQ && r < PQ + nj && c < m1) {
      const int al = r - PQ;
      v = kdot(d, al, [&](int t) { return hat(d, 0, nc + t, c) - hat(d, 1, nc + t, c); });
    } else if (r >= PQ && r < PQ + nj && c >= PQ && c < PQ + nj) {
      const int al = r - PQ, be = c - PQ;
      const double* hcol = d.H + (size_t)be * nf;
      v = kdot(d, al, [&](int t) { return hcol[t]; });
    } else if (r == c) {
      v = 1.0;  // pads
    }
    d.Q[(size_t)c * NQ + r] = v;
  }
}

// (f) F3 = [[B, .], [lhs, 0]]  with lhs = K^T M K
__global__ void k_build_F3(const PairDev* pd) {
  const PairDev d = pd[blockIdx.y];
  const int nj = d.nj, nf = d.nf, PJ = d.PJ, N2 = 2 * PJ, PQ = d.PQ, NQ = d.PQ + d.PJ;
  const long total = (long)N2 * N2;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e % N2), c = static_cast<int>(e / N2);
    double v = 0.0;
    if (r < PJ && c < PJ) {
      if (r < nj && c < nj) {
        const int hi = r >= c ? r : c, lo = r >= c ? c : r;
        v = d.Q[(size_t)(PQ + lo) * NQ + PQ + hi];
      } else {
        v = r == c ? 1.0 : 0.0;
      }
    } else if (r >= PJ && c < PJ) {
      const int al = r - PJ;
      if (al < nj && c < nj) {  // (K^T M K)[al][c] = sum_t K[t][al] (M K)[t][c]; H holds M K here
        const double* hcol = d.H + (size_t)c * nf;
        v = kdot(d, al, [&](int t) { return hcol[t]; });
      }
    }
    d.F3[(size_t)c * N2 + r] = v;
  }
}

// H = M K (reuses the scratch after Q is assembled)
__global__ void k_build_MK(const PairDev* pd) {
  const PairDev d = pd[blockIdx.y];
  const int nf = d.nf, nj = d.nj;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nf * nj; e += gridDim.x * blockDim.x) {
    const int t = e % nf, b = e / nf;
    d.H[(size_t)b * nf + t] = kdot(d, b, [&](int u) { return d.M[(size_t)u * nf + t]; });
  }
}

// (h) F4 = [[B, .], [W^T, 0]],  W = lhs L^{-T} from F3's factor
__global__ void k_build_F4(const PairDev* pd) {
  const PairDev d = pd[blockIdx.y];
  const int nj = d.nj, PJ = d.PJ, N2 = 2 * PJ, PQ = d.PQ, NQ = d.PQ + d.PJ;
  const long total = (long)N2 * N2;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(e % N2), c = static_cast<int>(e / N2);
    double v = 0.0;
    if (r < PJ && c < PJ) {
      if (r < nj && c < nj) {
        const int hi = r >= c ? r : c, lo = r >= c ? c : r;
        v = d.Q[(size_t)(PQ + lo) * NQ + PQ + hi];
      } else {
        v = r == c ? 1.0 : 0.0;
      }
    } else if (r >= PJ && c < PJ) {
      const int al = r - PJ;
      if (al < nj && c < nj) v = d.F3[(size_t)al * N2 + PJ + c];  // W^T[al][c] = W[c][al]
    }
    d.F4[(size_t)c * N2 + r] = v;
  }
}

// (j) Top-k symmetric eigensolver.  One CTA per pair:
//   1. Householder tridiagonalization of C, packed lower storage in shared
//      memory (global memory beyond 236 rows), reflectors kept in place;
//   2. the k largest eigenvalues of the tridiagonal by 16-way multisection on
//      Sturm counts (16 threads per eigenvalue);
//   3. eigenvectors of the tridiagonal by inverse iteration (one thread per
//      vector, partial-pivoting LU of T - lambda I, distinct start vectors),
//      modified Gram-Schmidt inside clusters;
//   4. back-transformation y = H_0 ... H_{n-3} z (one warp per vector).
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__device__ __forceinline__ size_t pk(int r, int c) { return (size_t)r * (r + 1) / 2 + c; }  // c <= r

// 1/q: hardware approximation refined by two Newton steps (full double
// precision; only the sign of the Sturm recurrence matters downstream).
__device__ __forceinline__ double fast_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = fma(r, fma(-q, r, 1.0), r);
  return fma(r, fma(-q, r, 1.0), r);
}

// Sturm count with the squared off-diagonal precomputed (e2[j] = e[j]^2)
__device__ int sturm_count_sq(const double* d, const double* e2, int n, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (q < 0) ++cnt;
  for (int j = 1; j < n; ++j) {
    if (fabs(q) < pivmin) q = -pivmin;
    q = (d[j] - x) - e2[j - 1] * fast_rcp(q);
    if (q < 0) ++cnt;
  }
  return cnt;
}

// stage timestamps of block 0 (BDDC_B200_PROFILE=1): load, tridiagonalization,
// multisection, inverse iteration, orthogonalization, back-transformation
__device__ unsigned long long g_syevx_trace[8];
__device__ int g_syevx_trace_on;
__device__ __forceinline__ void syevx_mark(int i) {
  if (g_syevx_trace_on && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_syevx_trace[i] = t;
  }
}

// Eigenvectors are formed only for the eigenvalues the selection enforces
// (adaptive.cpp:60-88: the leading ones above tau, at most max_vectors; or
// fixed_count; none for pair_indicator): `need` below, counted on the very
// eigenvalues the host reads back, so both take the same decision.  The other
// vector slots are written as zeros.
constexpr int kSyevxVec = 16;     // work vectors of length n per CTA
constexpr int kSyevxFusedMax = 288;  // one-pass tridiagonalization up to this order (nine 32-column groups per lane)

struct EigSelect {
  double tau;
  int max_vectors, fixed_count, indicator_only;
};

__global__ void __launch_bounds__(256) k_syevx(const PairDev* pd, int smem_cap, EigSelect sel) {
  const PairDev dd = pd[blockIdx.x];
  const int n = dd.nj, k = dd.k, N2 = 2 * dd.PJ, PJ = dd.PJ;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ double sm[];
  const size_t np = (size_t)n * (n + 1) / 2;
  // shared-memory placement, most to least: packed L, the 16n work vectors,
  // the inverse-iteration scratch (6n per vector) and the vectors Z (n per vector)
  const long wk = 7L * n * (k > 0 ? k : 1);
  const bool in_smem = (long)np + kSyevxVec * n + wk <= smem_cap;
  const bool work_smem = in_smem || (long)kSyevxVec * n + wk <= smem_cap;
  double* L = in_smem ? sm : dd.A;  // packed lower
  double* vec = in_smem ? sm + np : sm;  // v, p, d, e, tau, lam, vp, wp, colpart[8] (16n)
  double* wbase = work_smem ? vec + kSyevxVec * n : dd.A + (in_smem ? 0 : np);
  double* Z = wbase + (size_t)6 * n * k;  // k x n eigenvectors of T, then of C
  double* v = vec;
  double* p = vec + n;
  double* dg = vec + 2 * n;
  double* eg = vec + 3 * n;
  double* tau = vec + 4 * n;
  double* lam = vec + 5 * n;
  __shared__ double red[32];
  __shared__ double pg[256];  // column-group partials of A22 v
  if (n == 0 || k == 0) return;
  syevx_mark(0);
  for (int r = 0; r < n; ++r)
    for (int c = tid; c <= r; c += blockDim.x) L[pk(r, c)] = dd.F4[(size_t)c * N2 + PJ + r];
  __syncthreads();
  syevx_mark(1);
  // 1. tridiagonalization (dsytd2, lower).  One pass over the trailing matrix
  // per Householder step: the rank-2 update of step kk-1 is applied while the
  // product A v of step kk is formed from the updated entries (each element is
  // read and written once per step; the two-pass form below reads it three
  // times and writes it once).  Row r is owned by warp r mod 8, lanes over the
  // columns: the row sums come from a warp reduction, the column sums (the
  // symmetric half of the product) are kept per lane for its columns and the
  // eight warps' parts are added in a fixed order.
  if (n <= kSyevxFusedMax) {
    double* vp = vec + 6 * n;   // pending update: A -= vp wp^T + wp vp^T on rows/cols >= kk
    double* wp = vec + 7 * n;
    double* colpart = vec + 8 * n;  // [8][n]
    bool pending = false;
    for (int kk = 0; kk + 2 < n; ++kk) {
      const int m0 = kk + 1;
      // (a) column kk with the pending update, its norm, the reflector
      const double vpk = pending ? vp[kk] : 0.0, wpk = pending ? wp[kk] : 0.0;
      double part = 0.0;
      for (int i = kk + tid; i < n; i += blockDim.x) {
        double a = L[pk(i, kk)];
        if (pending) a -= vp[i] * wpk + wp[i] * vpk;
        v[i] = a;  // v[kk] = the diagonal entry, v[m0..] = x
        if (i >= m0) part += a * a;
      }
      const double ss = block_sum(part, red);  // barriers: v is complete afterwards
      const double x0 = v[m0];
      const double alpha = (x0 >= 0 ? -1.0 : 1.0) * sqrt(ss);
      const double v0 = x0 - alpha;
      const double vtv = ss - x0 * x0 + v0 * v0;
      const double t = (ss > 0.0 && vtv > 0.0) ? 2.0 / vtv : 0.0;
      __syncthreads();  // every thread has read v[m0]
      if (tid == 0) {
        dg[kk] = v[kk];
        eg[kk] = t != 0.0 ? alpha : x0;
        tau[kk] = t;
        v[m0] = t != 0.0 ? v0 : 0.0;
      }
      if (t == 0.0)  // no reflector: v = 0, the pass below only applies the pending update
        for (int i = m0 + 1 + tid; i < n; i += blockDim.x) v[i] = 0.0;
      __syncthreads();
      // (b) one pass: update, store, row and column sums of A v
      {
        double cacc[kSyevxFusedMax / 32];
#pragma unroll
        for (int q = 0; q < kSyevxFusedMax / 32; ++q) cacc[q] = 0.0;
        for (int r = m0 + warp; r < n; r += 8) {
          double* row = L + pk(r, 0);
          const double vr = v[r], vpr = pending ? vp[r] : 0.0, wpr = pending ? wp[r] : 0.0;
          double racc = 0.0;
#pragma unroll
          for (int q = 0; q < kSyevxFusedMax / 32; ++q) {
            const int c = m0 + lane + 32 * q;
            if (c <= r) {
              double a = row[c];
              if (pending) {
                a -= vpr * wp[c] + wpr * vp[c];
                row[c] = a;
              }
              racc += a * v[c];
              if (c < r) cacc[q] += a * vr;
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, o);
          if (lane == 0) p[r] = racc;
        }
#pragma unroll
        for (int q = 0; q < kSyevxFusedMax / 32; ++q) {
          const int c = m0 + lane + 32 * q;
          if (c < n) colpart[warp * n + c] = cacc[q];
        }
      }
      __syncthreads();
      double pv = 0.0;
      for (int i = m0 + tid; i < n; i += blockDim.x) {
        double sacc = p[i];
#pragma unroll
        for (int w = 0; w < 8; ++w) sacc += colpart[w * n + i];
        sacc *= t;
        p[i] = sacc;
        pv += sacc * v[i];
      }
      const double K = 0.5 * t * block_sum(pv, red);
      // (c) w = p - K v becomes the pending update; the reflector replaces the column
      for (int i = m0 + tid; i < n; i += blockDim.x) {
        const double vi = v[i];
        wp[i] = p[i] - K * vi;
        vp[i] = vi;
        if (t != 0.0) L[pk(i, kk)] = vi;
      }
      pending = true;
      __syncthreads();
    }
    if (tid == 0) {  // the last 2x2 block (1x1 when n == 1) with the pending update
      const int a0 = n >= 2 ? n - 2 : 0;
      for (int i = a0; i < n; ++i) {
        double d = L[pk(i, i)];
        if (pending) d -= 2.0 * vp[i] * wp[i];
        dg[i] = d;
        tau[i] = 0.0;
      }
      if (n >= 2) {
        double e = L[pk(n - 1, n - 2)];
        if (pending) e -= vp[n - 1] * wp[n - 2] + wp[n - 1] * vp[n - 2];
        eg[n - 2] = e;
      }
    }
  } else {
    // 1. tridiagonalization (dsytd2, lower)
    for (int kk = 0; kk + 2 < n; ++kk) {
      const int m0 = kk + 1;
      double part = 0.0;
      for (int i = m0 + tid; i < n; i += blockDim.x) {
        const double x = L[pk(i, kk)];
        part += x * x;
      }
      const double ss = block_sum(part, red);
      const double x0 = L[pk(m0, kk)];
      const double alpha = (x0 >= 0 ? -1.0 : 1.0) * sqrt(ss);
      const double v0 = x0 - alpha;
      const double vtv = ss - x0 * x0 + v0 * v0;
      const double t = (ss > 0.0 && vtv > 0.0) ? 2.0 / vtv : 0.0;
      for (int i = m0 + tid; i < n; i += blockDim.x) v[i] = (i == m0) ? v0 : L[pk(i, kk)];
      if (tid == 0) {
        dg[kk] = L[pk(kk, kk)];
        eg[kk] = t != 0.0 ? alpha : x0;
        tau[kk] = t;
      }
      __syncthreads();
      if (t == 0.0) continue;
      // p = t * A22 v.  Packed L in global memory: thread per row (sequential
      // row reads stay in L1 lines).  In shared memory: thread (row, column
      // group), four column groups reduced in a fixed order.
      if (!in_smem) {
        for (int r = m0 + tid; r < n; r += blockDim.x) {
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          const double* row = L + pk(r, 0);
          int c = m0;
          for (; c + 3 <= r; c += 4) {
            s0 += row[c] * v[c];
            s1 += row[c + 1] * v[c + 1];
            s2 += row[c + 2] * v[c + 2];
            s3 += row[c + 3] * v[c + 3];
          }
          for (; c <= r; ++c) s0 += row[c] * v[c];
          // column r below the diagonal: the warp walks the rows c2 together, so
          // its 32 lanes read 32 consecutive entries of packed row c2 (coalesced)
          const int base = r - (tid & 31);
          int c2 = base + 1;
          for (; c2 + 3 < n; c2 += 4) {
            const double* q = L + pk(c2, 0);
            const double a0 = c2 > r ? q[r] : 0.0;
            const double a1 = c2 + 1 > r ? q[c2 + 1 + r] : 0.0;
            const double a2 = c2 + 2 > r ? q[2 * c2 + 3 + r] : 0.0;
            const double a3 = c2 + 3 > r ? q[3 * c2 + 6 + r] : 0.0;
            s1 += a0 * v[c2];
            s2 += a1 * v[c2 + 1];
            s3 += a2 * v[c2 + 2];
            s0 += a3 * v[c2 + 3];
          }
          for (; c2 < n; ++c2)
            if (c2 > r) s1 += L[pk(c2, r)] * v[c2];
          p[r] = t * ((s0 + s1) + (s2 + s3));
        }
        __syncthreads();
      } else {
        const int g = tid >> 6;
        for (int r0 = m0; r0 < n; r0 += 64) {
          const int r = r0 + (tid & 63);
          double s0 = 0.0, s1 = 0.0;
          if (r < n) {
            int c = m0 + g;
            for (; c + 4 < n; c += 8) {
              s0 += L[c <= r ? pk(r, c) : pk(c, r)] * v[c];
              s1 += L[c + 4 <= r ? pk(r, c + 4) : pk(c + 4, r)] * v[c + 4];
            }
            if (c < n) s0 += L[c <= r ? pk(r, c) : pk(c, r)] * v[c];
          }
          pg[g * 64 + (tid & 63)] = s0 + s1;
          __syncthreads();
          if (tid < 64 && r < n) p[r] = t * ((pg[tid] + pg[64 + tid]) + (pg[128 + tid] + pg[192 + tid]));
          __syncthreads();
        }
      }
      double pv = 0.0;
      for (int i = m0 + tid; i < n; i += blockDim.x) pv += p[i] * v[i];
      const double K = 0.5 * t * block_sum(pv, red);
      for (int i = m0 + tid; i < n; i += blockDim.x) p[i] -= K * v[i];  // p becomes w
      __syncthreads();
      // rank-2 update of the trailing lower triangle: warp per row, lanes over columns
      for (int r = m0 + warp; r < n; r += 8) {
        double* row = L + pk(r, 0);
        const double vr = v[r], wr = p[r];
        for (int c = m0 + lane; c <= r; c += 128) {  // four independent elements in flight
          double x[4];
  #pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c + 32 * q <= r) x[q] = row[c + 32 * q];
  #pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int cc = c + 32 * q;
            if (cc <= r) row[cc] = x[q] - (vr * p[cc] + wr * v[cc]);
          }
        }
      }
      __syncthreads();
      // keep the reflector in the eliminated column (for the back-transformation)
      for (int i = m0 + tid; i < n; i += blockDim.x) L[pk(i, kk)] = v[i];
      __syncthreads();
    }
    if (tid == 0) {
      if (n >= 2) {
        dg[n - 2] = L[pk(n - 2, n - 2)];
        eg[n - 2] = L[pk(n - 1, n - 2)];
        tau[n - 2] = 0.0;
      }
      dg[n - 1] = L[pk(n - 1, n - 1)];
      tau[n - 1] = 0.0;
    }
  }
  __syncthreads();
  syevx_mark(2);
  // 2. top-k eigenvalues by multisection (16 threads per eigenvalue)
  double tnorm = 0.0, emax2 = 0.0, glo = 1e300, ghi = -1e300;
  for (int i = 0; i < n; ++i) {
    const double a = i > 0 ? fabs(eg[i - 1]) : 0.0, b = i + 1 < n ? fabs(eg[i]) : 0.0;
    glo = fmin(glo, dg[i] - a - b);
    ghi = fmax(ghi, dg[i] + a + b);
    tnorm = fmax(tnorm, fabs(dg[i]) + a + b);
    if (i + 1 < n) emax2 = fmax(emax2, eg[i] * eg[i]);
  }
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax2);
  double* e2g = v;  // the reflector scratch is free after the tridiagonalization
  for (int i = tid; i + 1 < n; i += blockDim.x) e2g[i] = eg[i] * eg[i];
  __syncthreads();
  glo -= 2.2e-16 * tnorm + 2 * pivmin;
  ghi += 2.2e-16 * tnorm + 2 * pivmin;
  const int G = 16;
  for (int base = 0; base < k; base += (int)blockDim.x / G) {
    const int m = base + tid / G, j = tid % G;
    const bool active = m < k;
    const int target = n - 1 - (active ? m : 0);  // ascending index
    double lo = glo, hi = ghi;
    for (int it = 0; it < 30; ++it) {
      const double x = lo + (hi - lo) * (j + 1) / (G + 1);
      const int ok = active ? (sturm_count_sq(dg, e2g, n, x, pivmin) <= target) : 1;
      // lo = largest x with count <= target; hi = smallest x with count > target
      const unsigned mask = __ballot_sync(0xffffffffu, ok);
      const unsigned sub = (mask >> ((lane / G) * G)) & 0xffffu;
      const int nok = __popc(sub);  // points j < nok are <= target (count is monotone)
      const double nlo = nok > 0 ? lo + (hi - lo) * nok / (G + 1) : lo;
      const double nhi = nok < G ? lo + (hi - lo) * (nok + 1) / (G + 1) : hi;
      lo = nlo;
      hi = nhi;
      const bool conv = hi - lo <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + pivmin;
      if (__all_sync(0xffffffffu, conv)) break;  // both 16-lane groups of the warp
    }
    if (active && j == 0) lam[m] = 0.5 * (lo + hi);
  }
  __syncthreads();
  syevx_mark(3);
  int need = 0;
  if (!sel.indicator_only) {
    if (sel.fixed_count >= 0) {
      need = min(sel.fixed_count, k);
    } else {
      while (need < k && fmax(lam[need], 0.0) > sel.tau) ++need;
      need = min(need, sel.max_vectors);
    }
  }
  if (tid == 0) *dd.need = need;
  // 3. inverse iteration on T (thread m), scratch in global memory
  if (tid < need) {
    const int m = tid;
    double* work = wbase + (size_t)m * 6 * n;
    double* xd = work;           // U diagonal
    double* xu = work + n;       // U first superdiagonal
    double* xu2 = work + 2 * n;  // U second superdiagonal (row interchanges)
    double* fm = work + 3 * n;   // multipliers
    double* b = work + 4 * n;    // rhs / solution
    double* sw = work + 5 * n;   // 1.0 where rows i, i+1 were interchanged
    double* z = Z + (size_t)m * n;
    const double shift = lam[m] + 4.0 * 2.2e-16 * tnorm * ((m & 1) ? 1.0 : -1.0);
    const double tiny = 2.2e-16 * tnorm + pivmin;
    // LU of T - shift I with partial pivoting, factored once; the running row
    // is carried in registers so the recurrence never waits on memory
    double cd = dg[0] - shift, cu = n > 1 ? eg[0] : 0.0;
    for (int i = 0; i + 1 < n; ++i) {
      const double sub = eg[i];
      const double nd = dg[i + 1] - shift;
      const double nu = i + 2 < n ? eg[i + 1] : 0.0;
      if (fabs(cd) >= fabs(sub)) {
        if (cd == 0.0) cd = tiny;
        const double f = sub / cd;
        xd[i] = cd;
        xu[i] = cu;
        xu2[i] = 0.0;
        fm[i] = f;
        sw[i] = 0.0;
        cd = nd - f * cu;
        cu = nu;
      } else {  // interchange rows i and i+1
        const double f = cd / sub;
        xd[i] = sub;
        xu[i] = nd;
        xu2[i] = nu;
        fm[i] = f;
        sw[i] = 1.0;
        cd = cu - f * nd;
        cu = -f * nu;
      }
    }
    xd[n - 1] = cd == 0.0 ? tiny : cd;
    for (int i = 0; i < n; ++i) xd[i] = 1.0 / xd[i];  // reciprocals: the solves below multiply
    unsigned long long seed = 0x9E3779B97F4A7C15ULL * (m + 1);
    for (int i = 0; i < n; ++i) {
      seed ^= seed << 13; seed ^= seed >> 7; seed ^= seed << 17;
      z[i] = 0.5 + (double)(seed >> 11) * (1.0 / 9007199254740992.0);
    }
    for (int it = 0; it < 3; ++it) {
      double cb = z[0];
#pragma unroll 4
      for (int i = 0; i + 1 < n; ++i) {
        const double nb = z[i + 1];
        if (sw[i] == 0.0) {
          b[i] = cb;
          cb = nb - fm[i] * cb;
        } else {
          b[i] = nb;
          cb = cb - fm[i] * nb;
        }
      }
      b[n - 1] = cb;
      double x1 = b[n - 1] * xd[n - 1], x2 = 0.0;
      b[n - 1] = x1;
      double nn = x1 * x1;
#pragma unroll 4
      for (int i = n - 2; i >= 0; --i) {
        const double xi = (b[i] - xu[i] * x1 - xu2[i] * x2) * xd[i];
        b[i] = xi;
        nn += xi * xi;
        x2 = x1;
        x1 = xi;
      }
      nn = 1.0 / sqrt(nn);
      for (int i = 0; i < n; ++i) z[i] = b[i] * nn;
    }
  }
  __syncthreads();
  syevx_mark(4);
  // modified Gram-Schmidt inside clusters (eigenvalues closer than 1e-7 ||T||)
  if (warp == 0) {
    for (int m = 1; m < need; ++m) {
      int c0 = m;
      while (c0 > 0 && fabs(lam[c0 - 1] - lam[c0]) <= 1e-7 * tnorm) --c0;
      double* zm = Z + (size_t)m * n;
      for (int q = c0; q < m; ++q) {
        const double* zq = Z + (size_t)q * n;
        double s = 0.0;
        for (int i = lane; i < n; i += 32) s += zq[i] * zm[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        for (int i = lane; i < n; i += 32) zm[i] -= s * zq[i];
      }
      if (c0 < m) {
        double s = 0.0;
        for (int i = lane; i < n; i += 32) s += zm[i] * zm[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        s = 1.0 / sqrt(s);
        for (int i = lane; i < n; i += 32) zm[i] *= s;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  syevx_mark(5);
  // 4. back-transformation y = H_0 ... H_{n-3} z: warp w carries vectors w and
  // w + 8 through the reflectors together (their reductions interleave), then
  // the vectors are written out with the solve padding zeroed
  for (int m0 = warp; m0 < need; m0 += 16) {
    const int m1 = m0 + 8;
    const bool two = m1 < need;
    double* y0 = Z + (size_t)m0 * n;
    double* y1 = Z + (size_t)(two ? m1 : m0) * n;
    for (int kk = n - 3; kk >= 0; --kk) {
      const double t = tau[kk];
      if (t == 0.0) continue;
      double s0 = 0.0, s1 = 0.0;
      for (int i = kk + 1 + lane; i < n; i += 32) {
        const double h = L[pk(i, kk)];
        s0 += h * y0[i];
        s1 += h * y1[i];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      s0 *= t;
      s1 *= t;
      for (int i = kk + 1 + lane; i < n; i += 32) {
        const double h = L[pk(i, kk)];
        y0[i] -= s0 * h;
        if (two) y1[i] -= s1 * h;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < k * N2; e += blockDim.x) {
    const int m = e / N2, i = e % N2;
    dd.vecs[e] = (m < need && i < n) ? Z[(size_t)m * n + i] : 0.0;
  }
  for (int m = tid; m < k; m += blockDim.x) dd.evals[m] = fmax(lam[m], 0.0);
  syevx_mark(6);
}

// The back-substitution sweeps of the vectors k_syevx did not form (zeros) are
// switched off: their descriptors get n = p = 0, so their tasks are empty.
__global__ void k_trim_solves(const PairDev* pd, const int* __restrict__ svoff, SolveDesc* sv) {
  const PairDev& d = pd[blockIdx.x];
  for (int m = *d.need + threadIdx.x; m < d.k; m += blockDim.x) {
    sv[svoff[blockIdx.x] + m].n = 0;
    sv[svoff[blockIdx.x] + m].p = 0;
  }
}

// (l) functional a_m = 1/2 M K alpha_m (alpha = first nj entries of vecs after the back solve)
__global__ void k_functional(const PairDev* pd) {
  const PairDev d = pd[blockIdx.y];
  const int nf = d.nf, nj = d.nj, N2 = 2 * d.PJ;
  const int m = blockIdx.x;
  if (m >= d.k || m >= *d.need) return;  // zero vectors beyond the enforced count: never read
  const double* al = d.vecs + (size_t)m * N2;
  for (int t = threadIdx.x; t < nf; t += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nj; ++b) s += d.H[(size_t)b * nf + t] * al[b];  // H = M K
    d.func[(size_t)m * nf + t] = 0.5 * s;
  }
}

}  // namespace

void PairEngine::release_buffers() {
  if (st_) CK(cudaStreamSynchronize(st_));
  bufs_.reset(new PairBuffers);
}

void PairEngine::set_shard(std::shared_ptr<Comm> comm, const std::vector<int>& owner) {
  comm_ = std::move(comm);
  owner_ = owner;
}

void PairEngine::attach(const Model& m, const double* S, const std::vector<long long>& s_off,
                        const std::vector<int>& PB, const std::vector<int>& nB, cudaStream_t st) {
  m_ = &m;
  S_ = S;
  s_off_ = s_off;
  PB_ = PB;
  nB_ = nB;
  st_ = st;
}

namespace detail {
struct HostPair {
  PairIndex idx;
  std::vector<int> pos[2];   // [outer | corner | shared] boundary positions per side
  int hub[2] = {-1, -1};     // two-level side fronts: the hub of each side
  int nout[2] = {0, 0};      // hub slots eliminated in the side front (U \ K)
  std::vector<int> gpos[2];  // [U \ K | corner | shared] as indices into the hub's U
  std::vector<int4> kc;      // compact kernel columns (unit row, r, rows off, vals off), pair-local offsets
  std::vector<int> krows;
  std::vector<double> kvals;
  std::vector<double> N;     // nm x m1 row-major
  std::vector<int> glob_off, glob_n;  // shared glob slot offsets
  int nj = 0, nm = 0, r_total = 0;    // r_total = admissible columns - nullity
};

// Hub of the two-level side-front elimination: substructure s, side g (1: its
// faces towards higher neighbours, 0: towards lower), U = union of the pair
// faces' closures (kept), rest = its other boundary slots (eliminated first).
struct Hub {
  int s = 0, g = 0;
  std::vector<int> U, rest;  // boundary positions, ascending
};

struct Dims { int no[2], PO[2], NG[2], nc, nf, nj, PQ, PJ, k, nm; };
struct ChunkHost {
  int p0 = 0, p1 = 0;
  std::vector<Dims> dims;
  std::vector<int> posv, krv, gposv;
  std::vector<int4> kcv;
  std::vector<double> kvv, Nv, Rv;
  std::vector<long long> oGp;  // per side: offset into gposv
  std::vector<long long> oG, oQ, oF3, oF4, oM, oKC, oKR, oKV, oH, oN, oR, oA, oE, oW, oFu, oDG, oDQ, oD3, oD4, oP;
  long long nG = 0, nQ = 0, nF = 0, nM = 0, nH = 0, nA = 0, nE = 0, nW = 0, nFu = 0, nD = 0;
};
ChunkHost build_chunk(const std::vector<HostPair>& hp, int p0, int request);
}  // namespace detail
using detail::HostPair;
using detail::ChunkHost;
using detail::Dims;
using detail::Hub;

// Host preparation of the face-pair eigenproblems: depends on the model and the
// base constraint set only, so Engine::step runs it while the leaf
// factorization is on the device.
struct PairPrep {
  ConstraintSet base;
  std::vector<std::pair<int, int>> pairs;  // this rank's face pairs
  std::vector<int> gidx;                    // their positions in face_pairs(m)
  std::vector<HostPair> hp;
  std::vector<ChunkHost> chunks;
  std::vector<Hub> hubs;
  int request = 0;
  double prep_ms = 0.0;
  // hub stage (PairEngine::start): padded sizes and arena offsets of the hubs
  bool started = false;
  std::vector<int> hubNH, hubPH;
  std::vector<long long> hubOff;
};

namespace {
// flat byte records for the constraint exchange of the sharded engine
struct ByteWriter {
  std::vector<char> buf;
  template <class T>
  void put(const T& x) {
    const char* p = reinterpret_cast<const char*>(&x);
    buf.insert(buf.end(), p, p + sizeof(T));
  }
  void i(int x) { put(x); }
  void d(double x) { put(x); }
  void v(const std::vector<double>& x) {
    i(static_cast<int>(x.size()));
    const char* p = reinterpret_cast<const char*>(x.data());
    buf.insert(buf.end(), p, p + x.size() * sizeof(double));
  }
};
struct ByteReader {
  const std::vector<char>& buf;
  std::size_t at = 0;
  explicit ByteReader(const std::vector<char>& b) : buf(b) {}
  template <class T>
  T get() {
    T x;
    std::memcpy(&x, buf.data() + at, sizeof(T));
    at += sizeof(T);
    return x;
  }
  int i() { return get<int>(); }
  double d() { return get<double>(); }
  std::vector<double> v() {
    const int n = i();
    std::vector<double> x(n);
    std::memcpy(x.data(), buf.data() + at, n * sizeof(double));
    at += n * sizeof(double);
    return x;
  }
};

int count_above(const std::vector<double>& v, double tau) {
  int k = 0;
  while (k < static_cast<int>(v.size()) && v[k] > tau) ++k;
  return k;
}
}  // namespace

namespace detail {
// One chunk of pair problems (bounded by a device-memory budget): dimensions,
// arena offsets and the concatenated host inputs, built in PairEngine::prepare.
ChunkHost build_chunk(const std::vector<HostPair>& hp, int p0, int request) {
  const int np = static_cast<int>(hp.size());
  const double budget = 24e9;  // bytes of pair fronts per chunk
  ChunkHost ch;
  ch.p0 = p0;
  long long& nG = ch.nG; long long& nQ = ch.nQ; long long& nF = ch.nF; long long& nM = ch.nM;
  long long& nH = ch.nH; long long& nA = ch.nA; long long& nE = ch.nE; long long& nW = ch.nW;
  long long& nFu = ch.nFu; long long& nD = ch.nD;
  int p1 = p0;
  double bytes = 0;
  std::vector<Dims>& dims = ch.dims;
  while (p1 < np) {
    const HostPair& h = hp[p1];
    Dims dm{};
    dm.nc = static_cast<int>(h.idx.corner_globals.size());
    dm.nf = static_cast<int>(h.idx.noncorner_globals.size());
    dm.nj = h.nj;
    dm.nm = h.nm;
    const int m1 = dm.nc + dm.nf;
    for (int side = 0; side < 2; ++side) {
      dm.no[side] = h.nout[side];  // slots of the side's hub eliminated in its side front
      dm.PO[side] = rup(dm.no[side], kTile);
      dm.NG[side] = dm.PO[side] + rup(std::max(m1, 1), kTile);
    }
    dm.PQ = rup(std::max(m1, 1), kTile);
    dm.PJ = rup(std::max(dm.nj, 1), kTile);
    dm.k = std::min(request, std::min(h.nj, std::max(h.r_total, 0)));
    dm.k = std::min(dm.k, 64);
    const double b = 8.0 * (double(dm.NG[0]) * dm.NG[0] + double(dm.NG[1]) * dm.NG[1] +
                            double(dm.PQ + dm.PJ) * (dm.PQ + dm.PJ) + 8.0 * dm.PJ * dm.PJ);
    if (p1 > p0 && bytes + b > budget) break;
    bytes += b;
    dims.push_back(dm);
    ++p1;
  }
  ch.p1 = p1;
  const int nb = p1 - p0;
  auto& posv = ch.posv; auto& krv = ch.krv; auto& kcv = ch.kcv;
  auto& kvv = ch.kvv; auto& Nv = ch.Nv; auto& Rv = ch.Rv;
  auto sized = [](std::vector<long long>& v, int n) -> std::vector<long long>& { v.assign(n, 0); return v; };
  auto& oG = sized(ch.oG, 2 * nb); auto& oQ = sized(ch.oQ, nb); auto& oF3 = sized(ch.oF3, nb);
  auto& oF4 = sized(ch.oF4, nb); auto& oM = sized(ch.oM, nb); auto& oKC = sized(ch.oKC, nb);
  auto& oKR = sized(ch.oKR, nb); auto& oKV = sized(ch.oKV, nb); auto& oH = sized(ch.oH, nb);
  auto& oN = sized(ch.oN, nb); auto& oR = sized(ch.oR, nb); auto& oA = sized(ch.oA, nb);
  auto& oE = sized(ch.oE, nb); auto& oW = sized(ch.oW, nb); auto& oFu = sized(ch.oFu, nb);
  auto& oDG = sized(ch.oDG, 2 * nb); auto& oDQ = sized(ch.oDQ, nb); auto& oD3 = sized(ch.oD3, nb);
  auto& oD4 = sized(ch.oD4, nb); auto& oP = sized(ch.oP, 2 * nb);
  auto& oGp = sized(ch.oGp, 2 * nb);
  auto& gposv = ch.gposv;
  for (int b = 0; b < nb; ++b) {
    const Dims& dm = dims[b];
    const HostPair& h = hp[p0 + b];
    for (int side = 0; side < 2; ++side) {
      oG[2 * b + side] = nG;
      nG += (long long)dm.NG[side] * dm.NG[side];
      oDG[2 * b + side] = nD;
      nD += (long long)(dm.PO[side] / kTile) * kTile * kTile;
      oP[2 * b + side] = posv.size();
      posv.insert(posv.end(), h.pos[side].begin(), h.pos[side].end());
      oGp[2 * b + side] = gposv.size();
      gposv.insert(gposv.end(), h.gpos[side].begin(), h.gpos[side].end());
    }
    const int NQ = dm.PQ + dm.PJ, N2 = 2 * dm.PJ, n2 = dm.nj + (dm.nj & 1);
    oQ[b] = nQ;
    nQ += (long long)NQ * NQ;
    oDQ[b] = nD;
    nD += (long long)(dm.PQ / kTile) * kTile * kTile;
    oF3[b] = nF;
    nF += (long long)N2 * N2;
    oF4[b] = nF;
    nF += (long long)N2 * N2;
    oD3[b] = nD;
    nD += (long long)(dm.PJ / kTile) * kTile * kTile;
    oD4[b] = nD;
    nD += (long long)(dm.PJ / kTile) * kTile * kTile;
    oM[b] = nM;
    nM += (long long)dm.nf * dm.nf;
    oKC[b] = kcv.size();
    kcv.insert(kcv.end(), h.kc.begin(), h.kc.end());
    oKR[b] = krv.size();
    krv.insert(krv.end(), h.krows.begin(), h.krows.end());
    oKV[b] = kvv.size();
    kvv.insert(kvv.end(), h.kvals.begin(), h.kvals.end());
    oH[b] = nH;
    nH += (long long)dm.nf * std::max(dm.nj, 1);
    oN[b] = Nv.size();
    Nv.insert(Nv.end(), h.N.begin(), h.N.end());
    oR[b] = Rv.size();
    Rv.insert(Rv.end(), h.idx.rho_i.begin(), h.idx.rho_i.end());
    oA[b] = nA;
    // Jacobi: A and V (2 n2^2); tridiagonal path: packed C + 4 n k LU scratch
    nA += std::max(2LL * n2 * n2, (long long)dm.nj * (dm.nj + 1) / 2 + 7LL * dm.nj * std::max(dm.k, 1)) + 64;
    oE[b] = nE;
    nE += std::max(dm.k, 1);
    oW[b] = nW;
    nW += (long long)N2 * std::max(dm.k, 1);
    oFu[b] = nFu;
    nFu += (long long)dm.nf * std::max(dm.k, 1);
  }
  return ch;
}
}  // namespace detail

std::shared_ptr<PairPrep> PairEngine::prepare(const ConstraintSet& cs, const EnrichOptions& o) const {
  using clk = std::chrono::steady_clock;
  const auto h0 = clk::now();
  auto prep = std::make_shared<PairPrep>();
  const Model& m = *m_;
  prep->base = cs;  // adaptive.cpp:133: every pair sees the same base
  const ConstraintSet& base = prep->base;
  const auto bg = base.by_glob(m.globs.size());
  prep->request = o.indicator_only ? 1 : (o.fixed_count >= 0 ? o.fixed_count : o.max_vectors) + 1;
  {
    // a face pair belongs to the owner of its lower substructure (shard.py)
    const auto all = face_pairs(m);
    for (std::size_t g = 0; g < all.size(); ++g)
      if (!comm_ || owner_[std::min(all[g].first, all[g].second)] == comm_->rank()) {
        prep->pairs.push_back(all[g]);
        prep->gidx.push_back(static_cast<int>(g));
      }
  }
  const auto& pairs = prep->pairs;
  const int np = static_cast<int>(pairs.size());
  prep->hp.resize(np);
  std::vector<HostPair>& hp = prep->hp;
  // boundary position of each local dof, per subdomain
  std::vector<std::vector<int>> bpos(m.subs.size());
  for (std::size_t s = 0; s < m.subs.size(); ++s) {
    bpos[s].assign(m.subs[s].dim(), -1);
    for (std::size_t b = 0; b < m.subs[s].boundary.size(); ++b) bpos[s][m.subs[s].boundary[b]] = static_cast<int>(b);
  }
  // pass 1: pair index spaces (independent per pair)
#pragma omp parallel for schedule(dynamic, 8) if (np >= 256)
  for (int p = 0; p < np; ++p) hp[p].idx = build_pair_index(m, pairs[p].first, pairs[p].second);
  // pass 2: one kernel basis (QR) per shared glob
  std::vector<KernelCompact> kern(m.globs.size());
  std::vector<char> kern_need(m.globs.size(), 0);
  for (int p = 0; p < np; ++p)
    for (int g : hp[p].idx.shared_globs) kern_need[g] = 1;
  std::vector<int> kern_list;
  for (std::size_t g = 0; g < m.globs.size(); ++g)
    if (kern_need[g]) kern_list.push_back(static_cast<int>(g));
#pragma omp parallel for schedule(dynamic, 8) if (kern_list.size() >= 256)
  for (int q = 0; q < static_cast<int>(kern_list.size()); ++q) {
    const int g = kern_list[q];
    const int n = static_cast<int>(m.glob_dofs[g].size());
    if (bg[g].empty()) {
      kern[g] = glob_kernel_compact(nullptr, 0, n);
    } else {
      std::vector<double> rows(bg[g].size() * std::size_t(n));
      for (std::size_t a = 0; a < bg[g].size(); ++a)
        for (int t = 0; t < n; ++t) rows[a * n + t] = base.averages[bg[g][a]].weights[t];
      kern[g] = glob_kernel_compact(&rows, static_cast<int>(bg[g].size()), n);
    }
  }
  // pass 3: positions, compact kernel columns, rigid modes
#pragma omp parallel for schedule(dynamic, 8) if (np >= 256)
  for (int p = 0; p < np; ++p) {
    HostPair& h = hp[p];
    const PairIndex& x = h.idx;
    const int nf = static_cast<int>(x.noncorner_globals.size());
    for (int side = 0; side < 2; ++side) {
      const int s = side == 0 ? x.si : x.sj;
      const auto& outer = side == 0 ? x.outer_i : x.outer_j;
      auto& pos = h.pos[side];
      for (i64 g : outer) pos.push_back(bpos[s][m.maps.local_of(g, s)]);
      for (i64 g : x.corner_globals) pos.push_back(bpos[s][m.maps.local_of(g, s)]);
      for (i64 g : x.noncorner_globals) pos.push_back(bpos[s][m.maps.local_of(g, s)]);
    }
    // kernel blocks of the installed averages (pair.cpp:167-188)
    int nj = 0;
    for (std::size_t gi = 0; gi < x.shared_globs.size(); ++gi) {
      const int g = x.shared_globs[gi];
      const int n = x.glob_size[gi], off = x.glob_offset[gi];
      const KernelCompact& kc = kern[g];
      const int r = kc.r, cols = n - r;
      const int rows_off = static_cast<int>(h.krows.size());
      for (int a = 0; a < r; ++a) h.krows.push_back(off + kc.perm[a]);
      for (int c = 0; c < cols; ++c) {
        const int vals_off = static_cast<int>(h.kvals.size());
        for (int a = 0; a < r; ++a) h.kvals.push_back(kc.neg_top[std::size_t(a) * cols + c]);
        h.kc.push_back(make_int4(off + kc.perm[r + c], r, rows_off, vals_off));
      }
      nj += cols;
    }
    h.nj = nj;
    const int m1 = static_cast<int>(x.corner_globals.size()) + nf;
    if (x.floating) {
      std::vector<i64> dofs(x.corner_globals);
      dofs.insert(dofs.end(), x.noncorner_globals.begin(), x.noncorner_globals.end());
      h.N = rigid_modes(m, dofs, &h.nm);
    }
    const int n_adm = m1 + nj + static_cast<int>(x.outer_i.size() + x.outer_j.size());
    h.r_total = n_adm - h.nm;
    (void)m1;
  }
  // pass 4: hubs of the two-level side fronts.  Side 0 of a pair is its lower
  // substructure (the face is on that substructure's upper side, g = 1).  Used
  // when the pairs fill the GPU (the extra stage costs latency on small runs);
  // BDDC_B200_GTREE=0|1 overrides.
  bool two_level = np >= sm_count();
  if (const char* env = std::getenv("BDDC_B200_GTREE")) {
    if (*env == '0') two_level = false;
    if (*env == '1') two_level = true;
  }
  if (!two_level) {
    // single level: the side front [outer | corner | shared] straight from S_s
    for (int p = 0; p < np; ++p)
      for (int side = 0; side < 2; ++side) {
        HostPair& h = hp[p];
        h.hub[side] = -1;
        h.nout[side] = static_cast<int>((side == 0 ? h.idx.outer_i : h.idx.outer_j).size());
        h.gpos[side] = h.pos[side];
      }
  } else {
    std::map<std::pair<int, int>, int> hub_of;
    auto& hubs = prep->hubs;
    for (int p = 0; p < np; ++p)
      for (int side = 0; side < 2; ++side) {
        const int s = side == 0 ? hp[p].idx.si : hp[p].idx.sj, g = side == 0 ? 1 : 0;
        auto it = hub_of.find({s, g});
        if (it == hub_of.end()) {
          it = hub_of.emplace(std::make_pair(s, g), static_cast<int>(hubs.size())).first;
          Hub hb;
          hb.s = s;
          hb.g = g;
          hubs.push_back(hb);
        }
        hp[p].hub[side] = it->second;
      }
    // U = union of the kept slots (corner + shared) of the hub's pair sides
    std::vector<std::vector<char>> inU(hubs.size());
    for (std::size_t q = 0; q < hubs.size(); ++q) inU[q].assign(m.subs[hubs[q].s].boundary.size(), 0);
    for (int p = 0; p < np; ++p)
      for (int side = 0; side < 2; ++side) {
        const auto& pos = hp[p].pos[side];
        const int no = static_cast<int>((side == 0 ? hp[p].idx.outer_i : hp[p].idx.outer_j).size());
        for (std::size_t a = no; a < pos.size(); ++a) inU[hp[p].hub[side]][pos[a]] = 1;
      }
    std::vector<std::vector<int>> idxU(hubs.size());
    for (std::size_t q = 0; q < hubs.size(); ++q) {
      idxU[q].assign(inU[q].size(), -1);
      for (int b = 0; b < static_cast<int>(inU[q].size()); ++b) {
        if (inU[q][b]) {
          idxU[q][b] = static_cast<int>(hubs[q].U.size());
          hubs[q].U.push_back(b);
        } else {
          hubs[q].rest.push_back(b);
        }
      }
    }
    // side fronts from the hub: [U \ K | corner | shared] as indices into U
#pragma omp parallel for schedule(dynamic, 8) if (np >= 256)
    for (int p = 0; p < np; ++p)
      for (int side = 0; side < 2; ++side) {
        HostPair& h = hp[p];
        const int q = h.hub[side];
        const auto& pos = h.pos[side];
        const int no = static_cast<int>((side == 0 ? h.idx.outer_i : h.idx.outer_j).size());
        std::vector<char> inK(hubs[q].U.size(), 0);
        for (std::size_t a = no; a < pos.size(); ++a) inK[idxU[q][pos[a]]] = 1;
        auto& gp = h.gpos[side];
        gp.clear();
        for (int u = 0; u < static_cast<int>(hubs[q].U.size()); ++u)
          if (!inK[u]) gp.push_back(u);
        h.nout[side] = static_cast<int>(gp.size());
        for (std::size_t a = no; a < pos.size(); ++a) gp.push_back(idxU[q][pos[a]]);
      }
  }
  for (int p0 = 0; p0 < np;) {
    prep->chunks.push_back(detail::build_chunk(hp, p0, prep->request));
    p0 = prep->chunks.back().p1;
  }
  prep->prep_ms = std::chrono::duration<double, std::milli>(clk::now() - h0).count();
  return prep;
}

// Reserves the pair stage's arenas and enqueues the hub stage (gather +
// partial Cholesky of the hubs) on the engine's stream.  It needs only the
// preparation and the substructures' S_s, which the stream produces before it,
// so Engine::step calls it BEFORE waiting for the leaf factorization: the
// device goes from the analysis straight into the hubs while the host checks
// the pivots and builds the first chunk's descriptors.
void PairEngine::start(const std::shared_ptr<PairPrep>& prep) {
  if (prep->started) return;
  prep->started = true;
  // Arenas sized once for the largest chunk: views into the engine's stage
  // arena (no allocation between chunks or steps; see StageArena).
  {
    HostTimer hr("enrich reserve");
    PairBuffers& B_ = *bufs_;
    long long hH = 0, hD = 0;
    for (const auto& h : prep->hubs) {
      const long long PH = rup(static_cast<int>(h.rest.size()), kTile);
      const long long NH = PH + rup(std::max(static_cast<int>(h.U.size()), 1), kTile);
      hH += NH * NH;
      hD += (PH / kTile) * kTile * kTile;
    }
    long long mx[10] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    for (const ChunkHost& c : prep->chunks) {
      const long long v[10] = {c.nG, c.nQ, c.nF, c.nD, c.nM, c.nH, c.nA, c.nE, c.nW, c.nFu};
      for (int i = 0; i < 10; ++i) mx[i] = std::max(mx[i], v[i]);
    }
    DBuf<double>* bufs[12] = {&B_.G, &B_.Q, &B_.F, &B_.Dv, &B_.M, &B_.H, &B_.A, &B_.E, &B_.W, &B_.Fu, &B_.Hub, &B_.DvH};
    const long long want[12] = {mx[0], mx[1], mx[2], mx[3], mx[4], mx[5], mx[6], mx[7], mx[8], mx[9],
                                std::max(hH, 1LL), std::max(hD, 1LL)};
    RegionPlan rp;
    for (int i = 0; i < 12; ++i) rp.add(*bufs[i], want[i]);
    if (region_)
      rp.place(region_(rp.total()));
    else
      for (int i = 0; i < 12; ++i) bufs[i]->alloc(want[i]);
    hr.mark("alloc");
  }
  const auto& hubs = prep->hubs;
  const int nh = static_cast<int>(hubs.size());
  std::vector<int>& hubNH = prep->hubNH;
  std::vector<int>& hubPH = prep->hubPH;
  std::vector<long long>& hubOff = prep->hubOff;
  hubNH.assign(nh, 0);
  hubPH.assign(nh, 0);
  hubOff.assign(nh, 0);
  // hub stage of the two-level side fronts: [rest | U] gathered from S_s, the
  // rest eliminated once per hub (Schur complement onto U in the trailing block)
  {
    HostTimer hth("enrich hubs");
    PairBuffers& B_ = *bufs_;
    long long nH = 0, nDH = 0;
    int maxNH = 0, maxPH = 0, maxMH = 0;
    std::vector<int> hposv;
    std::vector<GatherDesc> gh(nh);
    std::vector<FrontDesc> fh(nh);
    std::vector<long long> hposOff(nh), hubDOff(nh);
    for (int q = 0; q < nh; ++q) {
      const int nR = static_cast<int>(hubs[q].rest.size()), nU = static_cast<int>(hubs[q].U.size());
      hubPH[q] = rup(nR, kTile);
      hubNH[q] = hubPH[q] + rup(std::max(nU, 1), kTile);
      hubOff[q] = nH;
      nH += (long long)hubNH[q] * hubNH[q];
      hubDOff[q] = nDH;
      nDH += (long long)(hubPH[q] / kTile) * kTile * kTile;
      hposOff[q] = hposv.size();
      hposv.insert(hposv.end(), hubs[q].rest.begin(), hubs[q].rest.end());
      hposv.insert(hposv.end(), hubs[q].U.begin(), hubs[q].U.end());
      maxNH = std::max(maxNH, hubNH[q]);
      maxPH = std::max(maxPH, hubPH[q]);
      maxMH = std::max(maxMH, hubNH[q] - hubPH[q]);
    }
    if (nh) {
      B_.Hub.alloc(nH);
      B_.DvH.alloc(std::max<long long>(nDH, 1));
      B_.Hpos.upload(hposv, st_);
      B_.hinfo.alloc(nh);
      CK(cudaMemsetAsync(B_.hinfo.p, 0, nh * sizeof(int), st_));
      for (int q = 0; q < nh; ++q) {
        const int sub = hubs[q].s;
        gh[q] = GatherDesc{S_ + s_off_[sub], B_.Hpos.p + hposOff[q], B_.Hub.p + hubOff[q], PB_[sub], hubNH[q],
                           hubPH[q], static_cast<int>(hubs[q].rest.size()), static_cast<int>(hubs[q].U.size()), 1};
        fh[q] = FrontDesc{B_.Hub.p + hubOff[q], B_.DvH.p + hubDOff[q], hubNH[q], hubPH[q], B_.hinfo.p + q, 0,
                          static_cast<int>(hubs[q].rest.size()), static_cast<int>(hubs[q].U.size())};
      }
      B_.ghub.upload(gh, st_);
      B_.dHub.upload(fh, st_);
      StageProfiler hprof("enrich", st_);
      k_gather_front<<<dim3(maxNH, nh), 128, 0, st_>>>(B_.ghub.p);
      count_launch(1);
      CK(cudaGetLastError());
      hprof.mark("gatherHub");
      partial_cholesky(B_.dHub.p, nh, maxNH, maxPH, maxMH, st_);
      CK(cudaGetLastError());
      hprof.mark("cholHub");
    }
  }
}

EnrichOutcome PairEngine::enrich(ConstraintSet& cs, const EnrichOptions& o, std::shared_ptr<PairPrep> prep) {
  NvtxRange nvtx("bddc:eigen");
  using clk = std::chrono::steady_clock;
  const bool overlapped = prep != nullptr;
  if (!prep) prep = prepare(cs, o);
  const auto h1 = clk::now();
  const Model& m = *m_;
  const std::vector<HostPair>& hp = prep->hp;
  const int np = static_cast<int>(hp.size());
  const int request = prep->request;
  // device buffers, processed in chunks bounded by a memory budget
  EnrichOutcome out;
  std::vector<std::vector<double>> all_evals(np), all_funcs(np);
  std::vector<int> all_k(np);
  start(prep);  // arenas and hub stage (a no-op when Engine::step started it already)
  const auto& hubs = prep->hubs;
  const int nh = static_cast<int>(hubs.size());
  const std::vector<int>& hubNH = prep->hubNH;
  const std::vector<int>& hubPH = prep->hubPH;
  const std::vector<long long>& hubOff = prep->hubOff;
  // The chunks are pipelined: chunk c's results are copied into their own part
  // of the page-locked buffers behind its kernels (an event marks the end), the
  // host goes on to build and enqueue chunk c + 1 (stream order protects the
  // arenas the chunks share) and reads chunk c's results while c + 1 runs.
  const std::size_t nchunks = prep->chunks.size();
  std::vector<std::size_t> hoE(nchunks + 1, 0), hoFu(nchunks + 1, 0), hoInf(nchunks + 1, 0);
  {
    int q0 = 0;
    for (std::size_t c = 0; c < nchunks; ++c) {
      const ChunkHost& ch = prep->chunks[c];
      hoE[c + 1] = hoE[c] + static_cast<std::size_t>(std::max<long long>(ch.nE, 1));
      hoFu[c + 1] = hoFu[c] + static_cast<std::size_t>(std::max<long long>(ch.nFu, 1));
      hoInf[c + 1] = hoInf[c] + 4 * static_cast<std::size_t>(ch.p1 - q0);
      q0 = ch.p1;
    }
    bufs_->h_ev.reserve(hoE[nchunks]);
    bufs_->h_fu.reserve(hoFu[nchunks]);
    bufs_->h_inf.reserve(hoInf[nchunks]);
  }
  std::vector<cudaEvent_t> chunk_done(nchunks, nullptr);
  struct EventGuard {
    std::vector<cudaEvent_t>& v;
    ~EventGuard() {
      for (cudaEvent_t e : v)
        if (e) cudaEventDestroy(e);
    }
  } event_guard{chunk_done};
  auto finish_chunk = [&](std::size_t c) {
    const ChunkHost& ch = prep->chunks[c];
    const int q0 = c == 0 ? 0 : prep->chunks[c - 1].p1, nb = ch.p1 - q0;
    CK(cudaEventSynchronize(chunk_done[c]));
    if (c == 0 && nh) {
      std::vector<int> hinf(nh);
      CK(cudaMemcpy(hinf.data(), bufs_->hinfo.p, nh * sizeof(int), cudaMemcpyDeviceToHost));
      for (int q = 0; q < nh; ++q)
        if (hinf[q])
          throw Error(kNotPositiveDefinite, "pair eigenproblem hub of substructure " + std::to_string(hubs[q].s) +
                                                ": reduction not positive definite");
    }
    const double* ev = bufs_->h_ev.p + hoE[c];
    const double* fu = bufs_->h_fu.p + hoFu[c];
    const int* inf = bufs_->h_inf.p + hoInf[c];
    for (int b = 0; b < nb; ++b)
      for (int q = 0; q < 4; ++q)
        if (inf[4 * b + q])
          throw Error(kNotPositiveDefinite, "pair eigenproblem " + std::to_string(hp[q0 + b].idx.si) + "," +
                                                std::to_string(hp[q0 + b].idx.sj) + ": reduction not positive definite");
#pragma omp parallel for schedule(static) if (nb >= 256)
    for (int b = 0; b < nb; ++b) {
      const Dims& dm = ch.dims[b];
      const HostPair& h = hp[q0 + b];
      // eigenvalue list of generalized_eig_sym: top min(request, r) with zeros beyond rank(lhs)
      const int take = std::min(request, std::max(h.r_total, 0));
      std::vector<double> lam(take, 0.0);
      for (int q = 0; q < std::min(dm.k, take); ++q) lam[q] = ev[ch.oE[b] + q];
      all_evals[q0 + b] = lam;
      all_funcs[q0 + b].assign(fu + ch.oFu[b], fu + ch.oFu[b] + (long long)dm.nf * dm.k);
      all_k[q0 + b] = dm.k;
    }
  };
  int p0 = 0;
  std::size_t chunk_id = 0;
  while (p0 < np) {
    const ChunkHost& ch = prep->chunks[chunk_id++];
    HostTimer ht("enrich chunk");
    const int p1 = ch.p1, nb = p1 - p0;
    const auto& dims = ch.dims;
    const auto& posv = ch.posv; const auto& krv = ch.krv; const auto& kcv = ch.kcv;
    const auto& kvv = ch.kvv; const auto& Nv = ch.Nv; const auto& Rv = ch.Rv;
    const auto& oG = ch.oG; const auto& oQ = ch.oQ; const auto& oF3 = ch.oF3; const auto& oF4 = ch.oF4;
    const auto& oM = ch.oM; const auto& oKC = ch.oKC; const auto& oKR = ch.oKR; const auto& oKV = ch.oKV;
    const auto& oH = ch.oH; const auto& oN = ch.oN; const auto& oR = ch.oR; const auto& oA = ch.oA;
    const auto& oE = ch.oE; const auto& oW = ch.oW; const auto& oFu = ch.oFu; const auto& oDG = ch.oDG;
    const auto& oDQ = ch.oDQ; const auto& oD3 = ch.oD3; const auto& oD4 = ch.oD4; const auto& oP = ch.oP;
    const long long nG = ch.nG, nQ = ch.nQ, nF = ch.nF, nM = ch.nM, nH = ch.nH, nA = ch.nA, nE = ch.nE, nW = ch.nW,
                    nFu = ch.nFu, nD = ch.nD;
    std::vector<PairDev> pd(nb);
    ht.mark("host_arrays");
    PairBuffers& B_ = *bufs_;
    auto& G = B_.G; auto& Q = B_.Q; auto& F = B_.F; auto& Dv = B_.Dv; auto& M = B_.M;
    auto& H = B_.H; auto& N = B_.N; auto& R = B_.R; auto& A = B_.A; auto& E = B_.E; auto& W = B_.W;
    auto& Fu = B_.Fu;
    auto& Pv = B_.Pv; auto& info = B_.info;
    G.alloc(nG);
    Q.alloc(nQ);
    F.alloc(nF);
    Dv.alloc(std::max<long long>(nD, 1));
    M.alloc(std::max<long long>(nM, 1));
    B_.up_index.add(B_.KC, kcv);
    B_.up_index.add(B_.KR, krv);
    B_.up_index.add(B_.KV, kvv);
    H.alloc(std::max<long long>(nH, 1));
    B_.up_index.add(N, Nv);
    B_.up_index.add(R, Rv);
    A.alloc(std::max<long long>(nA, 1));
    E.alloc(nE);
    W.alloc(nW);
    Fu.alloc(std::max<long long>(nFu, 1));
    B_.up_index.add(Pv, posv);
    B_.up_index.add(B_.Gpos, ch.gposv);
    B_.up_index.flush(st_);
    info.alloc(4 * nb);
    CK(cudaMemsetAsync(info.p, 0, 4 * nb * sizeof(int), st_));
    B_.need.alloc(nb);
    CK(cudaMemsetAsync(B_.need.p, 0, nb * sizeof(int), st_));
    ht.mark("alloc_upload");
    std::vector<FrontDesc> fG(2 * nb), fQ(nb), f3(nb), f4(nb);
    int maxNG = 0, maxPO = 0, maxM1 = 0, maxNQ = 0, maxPQ = 0, maxPJ = 0, maxk = 0, maxnf = 0, maxn2 = 0;
    for (int b = 0; b < nb; ++b) {
      const Dims& dm = dims[b];
      const HostPair& h = hp[p0 + b];
      PairDev& d = pd[b];
      for (int side = 0; side < 2; ++side) {
        const int s = side == 0 ? h.idx.si : h.idx.sj;
        d.S[side] = S_ + s_off_[s];
        d.PB[side] = PB_[s];
        d.pos[side] = Pv.p + oP[2 * b + side] + (side == 0 ? h.idx.outer_i : h.idx.outer_j).size();
        d.G[side] = G.p + oG[2 * b + side];
        d.NG[side] = dm.NG[side];
        d.PO[side] = dm.PO[side];
        d.no[side] = dm.no[side];
        fG[2 * b + side] = FrontDesc{d.G[side], Dv.p + oDG[2 * b + side], dm.NG[side], dm.PO[side], info.p + 4 * b + side, 0,
                                     dm.no[side], dm.nc + dm.nf};
        maxNG = std::max(maxNG, dm.NG[side]);
        maxPO = std::max(maxPO, dm.PO[side]);
        maxM1 = std::max(maxM1, dm.NG[side] - dm.PO[side]);
      }
      d.nc = dm.nc;
      d.nf = dm.nf;
      d.nj = dm.nj;
      d.nm = dm.nm;
      d.PQ = dm.PQ;
      d.PJ = dm.PJ;
      d.k = dm.k;
      d.Q = Q.p + oQ[b];
      d.F3 = F.p + oF3[b];
      d.F4 = F.p + oF4[b];
      d.M = M.p + oM[b];
      d.kc = B_.KC.p + oKC[b];
      d.krows = B_.KR.p + oKR[b];
      d.kvals = B_.KV.p + oKV[b];
      d.H = H.p + oH[b];
      d.N = N.p + oN[b];
      d.rho = R.p + oR[b];
      const int n2 = dm.nj + (dm.nj & 1);
      d.A = A.p + oA[b];
      d.need = B_.need.p + b;
      d.evals = E.p + oE[b];
      d.vecs = W.p + oW[b];
      d.func = Fu.p + oFu[b];
      const int NQ = dm.PQ + dm.PJ, N2 = 2 * dm.PJ;
      fQ[b] = FrontDesc{d.Q, Dv.p + oDQ[b], NQ, dm.PQ, info.p + 4 * b + 2, 0};
      f3[b] = FrontDesc{d.F3, Dv.p + oD3[b], N2, dm.PJ, info.p + 4 * b + 3, 0};
      f4[b] = FrontDesc{d.F4, Dv.p + oD4[b], N2, dm.PJ, info.p + 4 * b + 3, 0};
      maxNQ = std::max(maxNQ, NQ);
      maxPQ = std::max(maxPQ, dm.PQ);
      maxPJ = std::max(maxPJ, dm.PJ);
      maxk = std::max(maxk, dm.k);
      maxnf = std::max(maxnf, dm.nf);
      maxn2 = std::max(maxn2, n2);
    }
    auto& dpd = B_.dpd;
    auto& dG = B_.dG; auto& dQ = B_.dQ; auto& d3 = B_.d3; auto& d4 = B_.d4;
    B_.up_desc.add(dpd, pd);
    B_.up_desc.add(dG, fG);
    B_.up_desc.add(dQ, fQ);
    B_.up_desc.add(d3, f3);
    B_.up_desc.add(d4, f4);
    // side-front gathers and the back-substitution descriptors of (k)
    std::vector<GatherDesc> gs(2 * nb);
    for (int b = 0; b < nb; ++b)
      for (int side = 0; side < 2; ++side) {
        const HostPair& h = hp[p0 + b];
        const int q = h.hub[side];
        const int sub = side == 0 ? h.idx.si : h.idx.sj;
        const double* src = q >= 0 ? B_.Hub.p + hubOff[q] + (size_t)hubPH[q] * hubNH[q] + hubPH[q]
                                   : S_ + s_off_[sub];
        const int lds = q >= 0 ? hubNH[q] : PB_[sub];
        gs[2 * b + side] = GatherDesc{src, B_.Gpos.p + ch.oGp[2 * b + side], pd[b].G[side], lds,
                                      dims[b].NG[side], dims[b].PO[side], dims[b].no[side],
                                      dims[b].nc + dims[b].nf, q >= 0 ? 0 : 1};
      }
    B_.up_desc.add(B_.gside, gs);
    std::vector<SolveDesc> sv;
    std::vector<int> svoff(nb);
    for (int b = 0; b < nb; ++b) {
      svoff[b] = static_cast<int>(sv.size());
      for (int mm = 0; mm < dims[b].k; ++mm)
        sv.push_back(SolveDesc{pd[b].F3, Dv.p + oD3[b], pd[b].vecs + (size_t)mm * 2 * dims[b].PJ, 2 * dims[b].PJ,
                               dims[b].PJ, nullptr, nullptr});
    }
    B_.up_desc.add(B_.dsv, sv);
    B_.up_desc.add(B_.svoff, svoff);
    B_.up_desc.flush(st_);
    ht.mark("descriptors");
    StageProfiler prof("enrich", st_);
    // (a)-(b) side fronts, eliminate the outer skeleton
    {
      // side fronts [U \ K | corner | shared] from the hubs' Schur complements
      k_gather_front<<<dim3(maxNG, 2 * nb), 128, 0, st_>>>(B_.gside.p);
      count_launch(1);
    }
    CK(cudaGetLastError());
    prof.mark("gatherG");
    partial_cholesky(dG.p, 2 * nb, maxNG, maxPO, maxM1, st_);
    prof.mark("cholG");
    // (c) M from the original shared block
    k_build_M<<<dim3(16, nb), 256, 0, st_>>>(dpd.p);
    // (d) Q and its elimination onto alpha
    k_build_H<<<dim3(32, nb), 256, 0, st_>>>(dpd.p);
    k_assemble_Q<<<dim3(64, nb), 256, 0, st_>>>(dpd.p);
    CK(cudaGetLastError());
    prof.mark("buildQ");
    partial_cholesky(dQ.p, nb, maxNQ, maxPQ, maxPJ, st_);
    prof.mark("cholQ");
    // (f)-(i) C = L^{-1} lhs L^{-T}
    k_build_MK<<<dim3(32, nb), 256, 0, st_>>>(dpd.p);
    k_build_F3<<<dim3(64, nb), 256, 0, st_>>>(dpd.p);
    partial_cholesky(d3.p, nb, 2 * maxPJ, maxPJ, maxPJ, st_);
    k_build_F4<<<dim3(64, nb), 256, 0, st_>>>(dpd.p);
    partial_cholesky(d4.p, nb, 2 * maxPJ, maxPJ, maxPJ, st_);
    CK(cudaGetLastError());
    prof.mark("reduceC");
    // (j) top-k eigenpairs of C
    {
      const int maxn = maxn2;  // >= every nj
      const long need = (long)maxn * (maxn + 1) / 2 + (long)kSyevxVec * maxn + 7L * maxn * std::max(maxk, 1);
      const long cap = (220 * 1024) / 8;  // leaves room for the kernel's static arrays
      // shared memory holds one CTA per SM here; with more pairs than SMs the
      // global-memory placement (about four CTAs per SM) takes fewer waves
      bool smem_ok = need <= cap && nb <= sm_count();
      if (const char* e = std::getenv("BDDC_B200_SYEVX"); e && *e) smem_ok = *e == 'S' && need <= cap;
      // all in shared memory when it fits; otherwise only the 16n work vectors, so that
      // several CTAs share an SM and hide the L2 latency of the packed matrix
      const long dyn = smem_ok ? need : (long)kSyevxVec * maxn;
      CK(static_cast<cudaError_t>(per_device(reinterpret_cast<const void*>(&k_syevx), [] {
        return static_cast<int>(cudaFuncSetAttribute(k_syevx, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      224 * 1024));
      })));
      const char* pe = std::getenv("BDDC_B200_PROFILE");
      const int tr_on = pe && *pe && *pe != '0';
      CK(cudaMemcpyToSymbolAsync(g_syevx_trace_on, &tr_on, sizeof(int), 0, cudaMemcpyHostToDevice, st_));
      const EigSelect sel{o.tau, o.max_vectors, o.fixed_count, o.indicator_only ? 1 : 0};
      k_syevx<<<nb, 256, static_cast<int>(dyn * 8), st_>>>(dpd.p, static_cast<int>(dyn), sel);
      if (tr_on) {
        unsigned long long t[8];
        CK(cudaMemcpyFromSymbolAsync(t, g_syevx_trace, sizeof(t), 0, cudaMemcpyDeviceToHost, st_));
        CK(cudaStreamSynchronize(st_));
        std::fprintf(stderr, "[profile] syevx block 0 (n=%d k=%d): load=%.1fus tridiag=%.1fus multisection=%.1fus "
                     "inverse_iteration=%.1fus mgs=%.1fus back_transform=%.1fus\n", dims[0].nj, dims[0].k,
                     (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3,
                     (t[5] - t[4]) * 1e-3, (t[6] - t[5]) * 1e-3);
      }
      prof.mark(smem_ok ? "syevx_smem" : "syevx_gmem");
    }
    CK(cudaGetLastError());
    // (k) alpha = L^{-T} y via F3's factor; (l) functionals
    auto& dsv = B_.dsv;
    k_trim_solves<<<nb, 32, 0, st_>>>(dpd.p, B_.svoff.p, dsv.p);
    front_backward(dsv.p, static_cast<int>(sv.size()), 2 * maxPJ, st_);
    k_functional<<<dim3(std::max(maxk, 1), nb), 128, 0, st_>>>(dpd.p);
    count_launch(10);
    CK(cudaGetLastError());
    prof.mark("vectors");
    ht.mark("launch");
    // results into this chunk's part of the page-locked buffers: the copies
    // queue behind the kernels, the event behind the copies
    {
      const std::size_t c = chunk_id - 1;
      CK(cudaMemcpyAsync(B_.h_ev.p + hoE[c], E.p, static_cast<std::size_t>(std::max<long long>(nE, 1)) * sizeof(double),
                         cudaMemcpyDeviceToHost, st_));
      CK(cudaMemcpyAsync(B_.h_fu.p + hoFu[c], Fu.p,
                         static_cast<std::size_t>(std::max<long long>(nFu, 1)) * sizeof(double),
                         cudaMemcpyDeviceToHost, st_));
      CK(cudaMemcpyAsync(B_.h_inf.p + hoInf[c], info.p, 4 * nb * sizeof(int), cudaMemcpyDeviceToHost, st_));
      CK(cudaEventCreateWithFlags(&chunk_done[c], cudaEventDisableTiming));
      CK(cudaEventRecord(chunk_done[c], st_));
      if (c > 0) finish_chunk(c - 1);  // while this chunk runs
      ht.mark("previous_results");
    }
    p0 = p1;
  }
  if (nchunks) finish_chunk(nchunks - 1);
  const auto h2 = clk::now();
  // host selection, splitting and rank filter (adaptive.cpp:66-125).  The
  // candidate averages are enumerated in the sequential order; whether one is
  // kept depends only on the earlier ones of its glob, so the rank tests run per
  // glob in parallel and the kept averages are appended in the original order.
  struct Cand {
    int p, glob;
    std::vector<double> w;
    char ok;
  };
  std::vector<Cand> cands;
  std::vector<PairReport> reps(np);
  // per pair in parallel (independent), concatenated in pair order below
  std::vector<std::vector<Cand>> pair_cands(np);
#pragma omp parallel for schedule(dynamic, 8) if (np >= 256)
  for (int p = 0; p < np; ++p) {
    const HostPair& h = hp[p];
    PairReport& rep = reps[p];
    rep.si = h.idx.si;
    rep.sj = h.idx.sj;
    rep.eigenvalues = all_evals[p];
    const auto& lam = rep.eigenvalues;
    const int L = static_cast<int>(lam.size());
    if (!o.indicator_only) {
      if (o.fixed_count >= 0)
        rep.enforced = std::min(o.fixed_count, L);
      else
        rep.enforced = std::min(count_above(lam, o.tau), o.max_vectors);
      rep.omega_next = rep.enforced < L ? lam[rep.enforced] : 0.0;
      rep.saturated = rep.omega_next > o.tau && o.fixed_count < 0;
      const int nf = static_cast<int>(h.idx.noncorner_globals.size());
      for (int mm = 0; mm < rep.enforced; ++mm) {
        std::vector<double> func(nf, 0.0);
        if (mm < all_k[p])
          std::copy(all_funcs[p].begin() + (long long)mm * nf, all_funcs[p].begin() + (long long)(mm + 1) * nf, func.begin());
        double scale = 0;
        for (double v : func) scale += v * v;
        scale = std::sqrt(scale);
        for (std::size_t gi = 0; gi < h.idx.shared_globs.size(); ++gi) {
          const int g = h.idx.shared_globs[gi];
          const int off = h.idx.glob_offset[gi], n = h.idx.glob_size[gi];
          std::vector<double> piece(func.begin() + off, func.begin() + off + n);
          double pn = 0;
          for (double v : piece) pn += v * v;
          pn = std::sqrt(pn);
          if (pn <= 1e-12 * scale) continue;
          if (m.globs[g].kind == kEdge && !o.keep_edge_constraints) continue;
          int top = 0;
          for (int t = 1; t < n; ++t)
            if (std::abs(piece[t]) > std::abs(piece[top])) top = t;
          const double div = piece[top] < 0 ? -pn : pn;
          for (double& v : piece) v /= div;
          pair_cands[p].push_back(Cand{p, g, std::move(piece), 0});
        }
      }
    } else {
      rep.omega_next = L > 0 ? lam[0] : 0.0;
    }
  }
  for (int p = 0; p < np; ++p)
    for (Cand& c : pair_cands[p]) cands.push_back(std::move(c));
  if (comm_) {
    // every rank's reports and candidates, in the global pair order, so that all
    // ranks apply the same rank filter and end with the same constraint set
    ByteWriter w;
    w.i(static_cast<int>(reps.size()));
    for (int p = 0; p < static_cast<int>(reps.size()); ++p) {
      const PairReport& r = reps[p];
      w.i(prep->gidx[p]); w.i(r.si); w.i(r.sj); w.i(r.enforced); w.i(r.saturated ? 1 : 0);
      w.d(r.omega_next);
      w.v(r.eigenvalues);
    }
    w.i(static_cast<int>(cands.size()));
    for (const Cand& c : cands) {
      w.i(prep->gidx[c.p]); w.i(c.glob);
      w.v(c.w);
    }
    const auto all = comm_->allgather(w.buf);
    std::vector<std::pair<int, PairReport>> greps;
    std::vector<Cand> gc;
    for (const auto& blob : all) {
      ByteReader rd(blob);
      const int nr = rd.i();
      for (int t = 0; t < nr; ++t) {
        PairReport r;
        const int g = rd.i();
        r.si = rd.i(); r.sj = rd.i(); r.enforced = rd.i(); r.saturated = rd.i() != 0;
        r.omega_next = rd.d();
        r.eigenvalues = rd.v();
        greps.emplace_back(g, std::move(r));
      }
      const int nc = rd.i();
      for (int t = 0; t < nc; ++t) {
        Cand c;
        c.p = rd.i(); c.glob = rd.i(); c.w = rd.v(); c.ok = 0;
        gc.push_back(std::move(c));
      }
    }
    std::stable_sort(greps.begin(), greps.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    std::stable_sort(gc.begin(), gc.end(), [](const Cand& a, const Cand& b) { return a.p < b.p; });
    // reports indexed by global pair, candidates pointing at them
    reps.clear();
    std::vector<int> where(greps.empty() ? 0 : greps.back().first + 1, -1);
    for (auto& gr : greps) {
      where[gr.first] = static_cast<int>(reps.size());
      reps.push_back(std::move(gr.second));
    }
    for (Cand& c : gc) c.p = where[c.p];
    cands = std::move(gc);
  }
  {
    std::vector<std::vector<int>> by_g(m.globs.size());
    for (std::size_t c = 0; c < cands.size(); ++c) by_g[cands[c].glob].push_back(static_cast<int>(c));
    const auto existing_idx = cs.by_glob(m.globs.size());
    std::vector<int> glist;
    for (std::size_t g = 0; g < by_g.size(); ++g)
      if (!by_g[g].empty()) glist.push_back(static_cast<int>(g));
#pragma omp parallel for schedule(dynamic, 4) if (glist.size() >= 64)
    for (int q = 0; q < static_cast<int>(glist.size()); ++q) {
      const int g = glist[q];
      std::vector<const std::vector<double>*> ex;
      for (int a : existing_idx[g]) ex.push_back(&cs.averages[a].weights);
      for (int c : by_g[g]) {
        cands[c].ok = average_admissible(ex, cands[c].w) ? 1 : 0;
        if (cands[c].ok) ex.push_back(&cands[c].w);
      }
    }
  }
  for (Cand& c : cands) {
    if (c.ok) {
      Average av;
      av.glob = c.glob;
      av.weights = std::move(c.w);
      av.adaptive = 1;
      cs.averages.push_back(std::move(av));
      ++reps[c.p].kept;
    } else {
      ++reps[c.p].dropped;
    }
  }
  for (int p = 0; p < static_cast<int>(reps.size()); ++p) {
    out.omega_tilde = std::max(out.omega_tilde, reps[p].omega_next);
    out.kept += reps[p].kept;
    out.dropped += reps[p].dropped;
    out.pairs.push_back(std::move(reps[p]));
  }
  const char* prof_env = std::getenv("BDDC_B200_PROFILE");
  if (prof_env && *prof_env && *prof_env != '0') {
    const auto h3 = clk::now();
    std::fprintf(stderr, "[profile] enrich host: pairs=%d prep=%.3fms%s device+copy=%.3fms select=%.3fms\n", np,
                 prep->prep_ms, overlapped ? " (overlapped)" : "",
                 std::chrono::duration<double, std::milli>(h2 - h1).count(),
                 std::chrono::duration<double, std::milli>(h3 - h2).count());
  }
  return out;
}

}  // namespace b200
