// Device engine: analysis (leaf factorization + interface Schur), the
// transformed preconditioner (leaf fronts + dense root), and a device-resident
// PCG whose iteration is one captured CUDA graph.  See engine.hpp and
// DESIGN.md "Data layout" for the arenas used below.
#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include <cooperative_groups.h>

#include "devbuf.cuh"
#include "../host/coarse_tree.hpp"
#include "pairs.cuh"

namespace b200 {

void cuda_check(cudaError_t e, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(kCudaError, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + file + ":" +
                                std::to_string(line));
}

namespace {

constexpr int kRed = 256;  // blocks of the deterministic dot-product reductions
constexpr int kRootInverseMax = 12288;  // explicit root inverse up to this padded size (2.4 GB front)
constexpr int kTreeApplies = 40;      // preconditioner applies assumed when choosing the primal tree depth

inline int rup(int v, int m) { return (v + m - 1) / m * m; }

struct PcgState {
  double rz, pq, alpha, beta, bnorm, ref, relres, tol;
  int it, max_it, done, precond_residual;
  unsigned int arrive;  // CTAs of k_beta_update that finished this iteration
};

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// Device assembly of the dense leaf fronts (assemble.cpp:202-258; SURVEY
// 8(f) row 1).  Elements are congruent: K_e = scale_e * K_ref[material_e].
struct AsmDesc {
  double* a;         // dense front [interior | boundary], ld x ld
  const int* lnode;  // local node grid (x fastest) * nc + c -> local dof or -1
  const int* pos;    // local dof -> front position
  int ld, nI, PI, nB, i0, j0, k0;
  int* ipos;         // front position -> local dof, or -1 (padding)
  int* dofq;         // local dof -> node grid index * nc + component
  int lnode_n, dim;  // entries of lnode, local dofs
};
struct AsmMesh {
  const double* ke;      // reference element matrices, ed x ed row-major each
  const int* eke;        // element -> reference matrix
  const double* escale;  // element scale, or nullptr (all 1)
  int ne0, ne1, epe, nc;
};

// Inverse maps of the front layout (per substructure, blockIdx.y): position ->
// local dof (ipos, preset to -1) and local dof -> node grid slot (dofq).
__global__ void k_front_maps(const AsmDesc* ds) {
  const AsmDesc d = ds[blockIdx.y];
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < d.lnode_n + d.dim; t += gridDim.x * blockDim.x) {
    if (t < d.lnode_n) {
      const int l = d.lnode[t];
      if (l >= 0) d.dofq[l] = t;
    } else {
      const int l = t - d.lnode_n;
      d.ipos[d.pos[l]] = l;
    }
  }
}

// Dense leaf fronts (assemble.cpp:202-258) in two passes over the block-lower
// triangle (tiles (a, b), a >= b, the diagonal tiles in full) -- the only part
// of a leaf front the factorization and the sweeps read:
//   k_zero_fronts      streams zeros (16-byte stores; 1 on a padding diagonal),
//   k_assemble_sparse  writes the stiffness entries, one thread per (row dof,
//                      neighbour node, component): at most 27 nc per row.
// A stiffness entry is the sum over the elements holding both nodes in the
// host's element order (k, j, i) of the reference element matrix entry times
// the element scale, multiply and add rounded separately: the front equals the
// host CSR bitwise.  (One thread per dense entry, the round-1 kernel, spent its
// time deciding that 98% of the entries are zero: 2.35 ms on cfg3.)
__global__ void __launch_bounds__(256) k_zero_fronts(const AsmDesc* ds) {
  const AsmDesc d = ds[blockIdx.y];
  for (int col = blockIdx.x; col < d.ld; col += gridDim.x) {
    const int r0 = col & ~63;
    const bool pad = (col >= d.nI && col < d.PI) || col >= d.PI + d.nB;  // no dof at this position
    double2* out = reinterpret_cast<double2*>(d.a + (size_t)col * d.ld);
    for (int r = r0 + 2 * threadIdx.x; r < d.ld; r += 2 * blockDim.x)
      out[r >> 1] = make_double2(pad && r == col ? 1.0 : 0.0, pad && r + 1 == col ? 1.0 : 0.0);
  }
}

__global__ void __launch_bounds__(256) k_assemble_sparse(const AsmDesc* ds, AsmMesh mm) {
  const AsmDesc d = ds[blockIdx.y];
  const int nc = mm.nc, ln = mm.epe + 1, ed = 8 * nc;
  const int vtx[8] = {0, 1, 3, 2, 4, 5, 7, 6};  // (dx + 2 dy + 4 dz) -> VTK vertex
  const int per = 27 * nc;
  const long total = (long)d.dim * per;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
    const int dr = static_cast<int>(t / per), rest = static_cast<int>(t % per);
    const int nbr = rest / nc, cb = rest % nc;
    const int g = d.dofq[dr], q = g / nc;
    const int4 a = make_int4(q % ln, (q / ln) % ln, q / (ln * ln), g % nc);
    const int4 b = make_int4(a.x + nbr % 3 - 1, a.y + (nbr / 3) % 3 - 1, a.z + nbr / 9 - 1, cb);
    if (b.x < 0 || b.y < 0 || b.z < 0 || b.x >= ln || b.y >= ln || b.z >= ln) continue;
    const int dc = d.lnode[((b.z * ln + b.y) * ln + b.x) * nc + cb];
    if (dc < 0) continue;
    const int pr = d.pos[dr], pc = d.pos[dc];
    if ((pr >> 6) < (pc >> 6)) continue;  // strictly upper tile: never read
    const bool lo = dr <= dc;
    const int4 P = lo ? a : b, Q = lo ? b : a;
    double s = 0.0;
    for (int ek = max(max(P.z, Q.z) - 1, 0); ek <= min(min(P.z, Q.z), mm.epe - 1); ++ek)
      for (int ej = max(max(P.y, Q.y) - 1, 0); ej <= min(min(P.y, Q.y), mm.epe - 1); ++ej)
        for (int ei = max(max(P.x, Q.x) - 1, 0); ei <= min(min(P.x, Q.x), mm.epe - 1); ++ei) {
          const int el = ((d.k0 + ek) * mm.ne1 + d.j0 + ej) * mm.ne0 + d.i0 + ei;
          const int va = vtx[(P.x - ei) + 2 * (P.y - ej) + 4 * (P.z - ek)];
          const int vb = vtx[(Q.x - ei) + 2 * (Q.y - ej) + 4 * (Q.z - ek)];
          const double kv = mm.ke[(size_t)mm.eke[el] * ed * ed + (va * nc + P.w) * ed + vb * nc + Q.w];
          const double sc = mm.escale ? mm.escale[el] : 1.0;
          s = __dadd_rn(s, sc == 1.0 ? kv : __dmul_rn(sc, kv));
        }
    d.a[(size_t)pc * d.ld + pr] = s;
  }
}

// upper triangle := lower (leaf_front's full copy of one front for the tests)
__global__ void k_mirror_upper(double* a, int ld) {
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)ld * ld; t += (long)gridDim.x * blockDim.x) {
    const int r = static_cast<int>(t % ld), c = static_cast<int>(t / ld);
    if (r < c) a[t] = a[(size_t)r * ld + c];
  }
}

struct SubDesc {        // per-subdomain pointers used by the PCG kernels
  const double* S;      // PB x PB full interface Schur
  double* F;            // transformed leaf front
  double* FV;           // F-layout vector
  const int* biface;    // nB: interface index of each boundary dof
  const double* bw;     // nB: averaging weights
  const int* posF;      // nB: F position
  const int* bglob;     // nB: transform instance or -1
  const int* bslot;     // nB: slot within the glob
  double* WB;           // nB: boundary scratch
  int nB, PB, NF, PE;
  int ldF;              // leading dimension of F (NF, or NF + PE for the augmented front)
  int nE;               // non-coarse boundary dofs (F rows [0, nE) and [PE, PE + nB - nE) are used)
};

struct XformDesc {      // glob transforms, flat
  const int* inst_tr;
  const int* inst_pos;  // per instance: offset into tpos
  const int* tpos;      // glob slot -> boundary position
  const int* tr_n;
  const int* tr_r;
  const int* tr_off_perm;
  const int* tr_off_d;
  const int* perm;
  const int* iperm;
  const double* D;      // r x n row-major per transform (= t_perm rows 0..r-1)
  const int* cpos;      // per instance (offset inst_pos): cpos[i] = tpos[perm[i]]
  const int* item_ptr;  // per subdomain: [item_ptr[s], item_ptr[s+1]) constrained rows
  const int* item_inst; // instance of the item
  const int* item_row;  // constrained row i < r of the item
  const int* inst_loff; // per instance: offset of its rows in the subdomain's row results
};

// T^T v at glob slot j with composite positions (restrict)
__device__ __forceinline__ double xform_T_t_c(const XformDesc& x, int inst, int j, const double* v) {
  const int tr = x.inst_tr[inst];
  const int* cp = x.cpos + x.inst_pos[inst];
  const int n = x.tr_n[tr], r = x.tr_r[tr];
  const double* D = x.D + x.tr_off_d[tr];
  double s0 = j >= r ? v[cp[j]] : 0.0, s1 = 0.0;
  int i = 0;
  for (; i + 1 < r; i += 2) {
    s0 += D[i * n + j] * v[cp[i]];
    s1 += D[(i + 1) * n + j] * v[cp[i + 1]];
  }
  if (i < r) s0 += D[i * n + j] * v[cp[i]];
  return s0 + s1;
}

// y = T^T v on the glob blocks of one boundary position b (transform.cpp:94-149)
__device__ __forceinline__ double xform_T_t(const XformDesc& x, int inst, int j, const double* v) {
  const int tr = x.inst_tr[inst];
  const int* pos = x.tpos + x.inst_pos[inst];
  const int n = x.tr_n[tr], r = x.tr_r[tr];
  const int* perm = x.perm + x.tr_off_perm[tr];
  const double* D = x.D + x.tr_off_d[tr];
  double s = j >= r ? v[pos[perm[j]]] : 0.0;
  for (int i = 0; i < r; ++i) s += D[i * n + j] * v[pos[perm[i]]];
  return s;
}

// Schur apply, step 1 (schur.cpp:12-36 with S_s dense): WB_s = S_s * p[biface].
// Row-blocked: CTA (rb, s) forms rows [64 rb, 64 rb + 64) of S_s x_s.
// Lane l of warp w owns rows (2l, 2l+1) (one 16-byte load per column) and the
// columns w, w+8, ...; eight columns are in flight per thread, the eight warp
// partials are reduced in shared memory in a fixed order.  `in(i)` yields the
// input at interface dof i; xs holds nB doubles of shared memory.
template <class In>
__device__ __forceinline__ void schur_rows_body(const SubDesc& d, int r0, In in, double* xs) {
  __shared__ double2 part[8][32];
  for (int c = threadIdx.x; c < d.nB; c += blockDim.x) xs[c] = in(d.biface[c]);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* col0 = reinterpret_cast<const double2*>(d.S + r0) + lane;  // rows r0 + 2 lane, +1
  const size_t ld2 = d.PB / 2;
  double2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
  int c = w;
  for (; c + 56 < d.nB; c += 64) {
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = __ldg(col0 + (size_t)(c + 8 * q) * ld2);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double x = xs[c + 8 * q];
      acc[q & 3].x += v[q].x * x;
      acc[q & 3].y += v[q].y * x;
    }
  }
  for (; c < d.nB; c += 8) {
    const double2 v = __ldg(col0 + (size_t)c * ld2);
    const double x = xs[c];
    acc[0].x += v.x * x;
    acc[0].y += v.y * x;
  }
  part[w][lane] = make_double2((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x),
                               (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
  __syncthreads();
  if (threadIdx.x < 64) {
    const int l = threadIdx.x >> 1, h = threadIdx.x & 1;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += h ? part[q][l].y : part[q][l].x;
    const int r = r0 + threadIdx.x;
    if (r < d.nB) d.WB[r] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_schur_gemv_rows(const SubDesc* sd, const double* __restrict__ p,
                                                         const int* done) {
  if (done && *done) return;
  const SubDesc d = sd[blockIdx.y];
  const int r0 = blockIdx.x * 64;
  if (r0 >= d.nB) return;
  extern __shared__ double xs[];
  schur_rows_body(d, r0, [p](int i) { return p[i]; }, xs);
}

__device__ __forceinline__ void block_partial(double v, double* partials) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) partials[blockIdx.x] = v;
  }
}

__device__ __forceinline__ double sum_partials(const double* partials) {
  // fixed-order tree over kRed partials by one block of kRed threads
  __shared__ double red[kRed];
  red[threadIdx.x] = partials[threadIdx.x];
  __syncthreads();
  for (int s = kRed / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  return red[0];
}

// out[i] = sum over the copies of interface dof i of src[pos]; optional dot with `other`
// Sum of fv[idx[t]] over the CSR list of `at`, added in list order; the loads
// of up to eight entries are issued together, so the dependent chain is
// ptr -> index -> value instead of one round trip per entry.
template <class Index>
__device__ __forceinline__ double csr_sum(const int* __restrict__ ptr, const Index* __restrict__ idx, const double* fv,
                                          long long at) {
  const int b = ptr[at], e = ptr[at + 1];
  double s = 0.0;
  for (int t = b; t < e; t += 8) {
    long long k[8];
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) k[q] = t + q < e ? static_cast<long long>(idx[t + q]) : -1;
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = k[q] >= 0 ? fv[k[q]] : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (t + q < e) s += v[q];
  }
  return s;
}

__global__ void __launch_bounds__(256) k_sum_copies(i64 n, const int* __restrict__ ptr, const int* __restrict__ pos,
                                                    const double* __restrict__ src, double* out,
                                                    const double* other, double* partials, const int* done) {
  if (done && *done) return;
  double acc = 0.0;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  // two dofs per pass, their chains in flight together; sums and the dot
  // product are formed in the order of the one-dof loop
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += 2 * stride) {
    const i64 i1 = i + stride;
    const double s0 = csr_sum(ptr, pos, src, i);
    const double s1 = i1 < n ? csr_sum(ptr, pos, src, i1) : 0.0;
    const double o0 = other ? other[i] : 0.0, o1 = other && i1 < n ? other[i1] : 0.0;
    out[i] = s0;
    if (other) acc += s0 * o0;
    if (i1 < n) {
      out[i1] = s1;
      if (other) acc += s1 * o1;
    }
  }
  if (partials) block_partial(acc, partials);
}

// --- interface halo of the sharded engine ---------------------
__global__ void k_halo_pack(int n, const int* __restrict__ idx, const double* __restrict__ y, double* buf) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) buf[k] = y[idx[k]];
}

// y[dof[q]] = sum of the contributions of every rank holding dof[q], in
// ascending rank order (src < 0: this rank's own partial sum): the same value
// on every rank, deterministic.
__global__ void k_halo_sum(int n, const int* __restrict__ dof, const int* __restrict__ ptr, const int* __restrict__ src,
                           const double* __restrict__ recv, double* y) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int i = dof[q];
    double s = 0.0;
    for (int t = ptr[q]; t < ptr[q + 1]; ++t) s += src[t] < 0 ? y[i] : recv[src[t]];
    y[i] = s;
  }
}

// y[i] = 0 unless this rank owns interface dof i (before a completing sum)
__global__ void k_keep_owned(i64 n, const double* __restrict__ owned, double* y) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    if (owned[i] == 0.0) y[i] = 0.0;
}

__global__ void k_dot(i64 n, const double* a, const double* b, double* partials, const double* mask = nullptr) {
  double acc = 0.0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    if (!mask || mask[i] != 0.0) acc += a[i] * b[i];
  block_partial(acc, partials);
}

// alpha = rz / (p.q) (every CTA reduces the partials in the same fixed order),
// x += alpha p, r -= alpha q, partials of r.r.  Only CTA 0 writes the state
// fields nobody else reads here.
// Sharded: `owned` masks the r.r partials to the dofs this rank owns (the
// partials are then all-reduced, so every rank takes the same stopping decision).
__global__ void __launch_bounds__(kRed) k_alpha_axpy(i64 n, PcgState* st, double* x, double* r, const double* p,
                                                     const double* q, const double* ppq, double* prr, double* alphas,
                                                     const double* __restrict__ owned = nullptr) {
  if (st->done) return;
  const double pq = sum_partials(ppq);
  const double a = st->rz / pq;
  double acc = 0.0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    const double ri = r[i] - a * q[i];
    r[i] = ri;
    if (!owned || owned[i] != 0.0) acc += ri * ri;
  }
  block_partial(acc, prr);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->pq = pq;
    st->alpha = a;
    alphas[st->it] = a;
  }
}

// beta = rz_next / rz, p = z + beta p; the last CTA to finish commits the
// iteration (rz, it, residual, done), after every CTA has read the old state.
__global__ void __launch_bounds__(kRed) k_beta_update(i64 n, PcgState* st, double* p, const double* z,
                                                      const double* prz, const double* prr, double* betas) {
  if (st->done) return;
  const double rz_next = sum_partials(prz);
  __syncthreads();
  const double rr = sum_partials(prr);
  const double beta = rz_next / st->rz;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&st->arrive, 1u) == gridDim.x - 1) {
      st->arrive = 0;
      st->beta = beta;
      betas[st->it] = beta;
      st->rz = rz_next;
      st->it += 1;
      const double cur = st->precond_residual ? sqrt(fmax(rz_next, 0.0)) : sqrt(rr);
      st->relres = cur / st->ref;
      if (st->relres <= st->tol || st->it >= st->max_it) st->done = 1;
      __threadfence();
    }
  }
}

// restrict_residual (bddc_operator.cpp:52-68) restricted to the interface:
// FV_s = P_F T_s^T (w_s * r|_s), pads zero.  `in(i)` yields r at interface dof
// i; v holds nB doubles of shared memory.
template <class In>
__device__ __forceinline__ void restrict_body(const SubDesc& d, const XformDesc& x, In in, double* v) {
  for (int b = threadIdx.x; b < d.nB; b += blockDim.x) v[b] = d.bw[b] * in(d.biface[b]);
  for (int q = threadIdx.x; q < d.NF; q += blockDim.x) d.FV[q] = 0.0;
  __syncthreads();
  for (int b = threadIdx.x; b < d.nB; b += blockDim.x) {
    const int inst = d.bglob[b];
    const double y = inst < 0 ? v[b] : xform_T_t_c(x, inst, d.bslot[b], v);
    d.FV[d.posF[b]] = y;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_restrict(const SubDesc* sd, XformDesc x, const double* __restrict__ r, const int* done) {
  if (done && *done) return;
  extern __shared__ double sm[];
  restrict_body(sd[blockIdx.x], x, [r](int i) { return r[i]; }, sm);
}

// prolong (bddc_operator.cpp:87-99): WB_s = w_s * T_s x_s   (then summed over copies)
// The constrained rows of the glob transforms (dot products over the glob) are
// formed first, one warp per row, into shared memory; every other boundary
// position is a copy.  q: the substructure's index among the owned ones.
__device__ __forceinline__ void prolong_body(const SubDesc& d, const XformDesc& x, int q, double* sm) {
  double* xn = sm;
  double* yrow = sm + d.nB;
  for (int b = threadIdx.x; b < d.nB; b += blockDim.x) xn[b] = d.FV[d.posF[b]];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = x.item_ptr[q], i1 = x.item_ptr[q + 1];
  for (int it = i0 + warp; it < i1; it += blockDim.x >> 5) {
    const int inst = x.item_inst[it], i = x.item_row[it];
    const int tr = x.inst_tr[inst];
    const int* pos = x.tpos + x.inst_pos[inst];
    const int n = x.tr_n[tr];
    const double* D = x.D + x.tr_off_d[tr] + i * n;
    double s = 0.0;
    for (int jj = lane; jj < n; jj += 32) s += D[jj] * xn[pos[jj]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) yrow[x.inst_loff[inst] + i] = s;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < d.nB; b += blockDim.x) {
    const int inst = d.bglob[b];
    double xo = xn[b];
    if (inst >= 0) {
      const int tr = x.inst_tr[inst];
      const int i = x.iperm[x.tr_off_perm[tr] + d.bslot[b]];
      xo = i < x.tr_r[tr] ? yrow[x.inst_loff[inst] + i] : xn[x.tpos[x.inst_pos[inst] + i]];
    }
    d.WB[b] = d.bw[b] * xo;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_prolong(const SubDesc* sd, XformDesc x, const int* done) {
  if (done && *done) return;
  extern __shared__ double sm[];
  prolong_body(sd[blockIdx.x], x, blockIdx.x, sm);
}

// root right-hand side: sum of the leaves' coarse residuals (deterministic CSR)
__global__ void k_root_gather(int n_root, int NR, const int* __restrict__ ptr, const long long* __restrict__ src,
                              const double* __restrict__ fv, double* xr, const int* done) {
  if (done && *done) return;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < NR; k += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (k < n_root)
      for (int t = ptr[k]; t < ptr[k + 1]; ++t) s += fv[src[t]];
    xr[k] = s;
  }
}

// F_s column transform: X = S T (glob columns), other columns copied
__global__ void k_colxform(const SubDesc* sd, XformDesc x, double* Xarena, const long long* xoff) {
  const SubDesc d = sd[blockIdx.y];
  double* X = Xarena + xoff[blockIdx.y];
  const int c = blockIdx.x;
  if (c >= d.PB) return;
  const int inst = c < d.nB ? d.bglob[c] : -1;
  if (inst < 0) {
    for (int b = threadIdx.x; b < d.PB; b += blockDim.x) X[(size_t)c * d.PB + b] = d.S[(size_t)c * d.PB + b];
    return;
  }
  const int j = d.bslot[c];
  const int tr = x.inst_tr[inst];
  const int* pos = x.tpos + x.inst_pos[inst];
  const int n = x.tr_n[tr], r = x.tr_r[tr];
  const int* perm = x.perm + x.tr_off_perm[tr];
  const double* D = x.D + x.tr_off_d[tr];
  for (int b = threadIdx.x; b < d.PB; b += blockDim.x) {
    double s = j >= r ? d.S[(size_t)pos[perm[j]] * d.PB + b] : 0.0;
    for (int i = 0; i < r; ++i) s += D[i * n + j] * d.S[(size_t)pos[perm[i]] * d.PB + b];
    X[(size_t)c * d.PB + b] = s;
  }
}

// F = P_F (T^T X) P_F^T with identity pads
__global__ void k_rowxform_scatter(const SubDesc* sd, XformDesc x, const double* Xarena, const long long* xoff) {
  const SubDesc d = sd[blockIdx.y];
  const double* X = Xarena + xoff[blockIdx.y];
  const int c = blockIdx.x;
  if (c < d.nB) {
    const double* col = X + (size_t)c * d.PB;
    const size_t fc = (size_t)d.posF[c] * d.ldF;
    for (int b = threadIdx.x; b < d.nB; b += blockDim.x) {
      const int inst = d.bglob[b];
      const double v = inst < 0 ? col[b] : xform_T_t(x, inst, d.bslot[b], col);
      d.F[fc + d.posF[b]] = v;
    }
  }
  // the padding positions of F get identity entries in k_pad_identity
}

// F = P_F (T^T S T) P_F^T in one pass (factor mode: ld F = NF): CTA (c, s)
// forms kXformCols columns of S T in shared memory (a glob column combines
// r + 1 columns of S; when the CTA's columns share one glob instance the r
// pivot columns are read once for all of them), applies T^T on the rows and
// writes the whole F columns, padding rows included; columns beyond nB are the
// padding columns (unit vectors).  Every entry of F is written: no scratch X,
// no memset.
constexpr int kXformCols = 4;  // F columns per CTA in k_xform_fused

__global__ void __launch_bounds__(256) k_xform_fused(const SubDesc* sd, XformDesc x) {
  const SubDesc d = sd[blockIdx.y];
  extern __shared__ double y[];  // [kXformCols][nB]: columns of S T
  const int c0 = blockIdx.x * kXformCols, nE = d.nE, nC = d.nB - d.nE;
  const size_t ld = d.ldF;
  int inst[kXformCols];
#pragma unroll
  for (int k = 0; k < kXformCols; ++k) inst[k] = c0 + k < d.nB ? d.bglob[c0 + k] : -2;
  bool same = inst[0] >= 0;
#pragma unroll
  for (int k = 1; k < kXformCols; ++k) same = same && inst[k] == inst[0];
  if (same) {
    // the CTA's columns belong to one glob instance: the r pivot columns of S
    // are read once for all of them (S T column j = S e_{cp[j]} [j >= r] + sum_i D_ij S e_{cp[i]})
    const int tr = x.inst_tr[inst[0]];
    const int* cp = x.cpos + x.inst_pos[inst[0]];  // cp[i] = tpos[perm[i]]
    const int n = x.tr_n[tr], r = x.tr_r[tr];
    const double* D = x.D + x.tr_off_d[tr];
    int j[kXformCols];
#pragma unroll
    for (int k = 0; k < kXformCols; ++k) j[k] = d.bslot[c0 + k];
    for (int b = threadIdx.x; b < d.nB; b += blockDim.x) {
      double acc[kXformCols];
#pragma unroll
      for (int k = 0; k < kXformCols; ++k) acc[k] = j[k] >= r ? d.S[(size_t)cp[j[k]] * d.PB + b] : 0.0;
      for (int i = 0; i < r; ++i) {
        const double sv = d.S[(size_t)cp[i] * d.PB + b];
#pragma unroll
        for (int k = 0; k < kXformCols; ++k) acc[k] += D[i * n + j[k]] * sv;
      }
#pragma unroll
      for (int k = 0; k < kXformCols; ++k) y[k * d.nB + b] = acc[k];
    }
  } else {
    for (int k = 0; k < kXformCols; ++k) {
      const int c = c0 + k;
      if (c >= d.nB) break;
      double* yk = y + k * d.nB;
      if (inst[k] < 0) {
        const double* sc = d.S + (size_t)c * d.PB;
        for (int b = threadIdx.x; b < d.nB; b += blockDim.x) yk[b] = sc[b];
      } else {
        const int jj = d.bslot[c];
        const int tr = x.inst_tr[inst[k]];
        const int* cp = x.cpos + x.inst_pos[inst[k]];
        const int n = x.tr_n[tr], r = x.tr_r[tr];
        const double* D = x.D + x.tr_off_d[tr];
        for (int b = threadIdx.x; b < d.nB; b += blockDim.x) {
          double acc = jj >= r ? d.S[(size_t)cp[jj] * d.PB + b] : 0.0;
          for (int i = 0; i < r; ++i) acc += D[i * n + jj] * d.S[(size_t)cp[i] * d.PB + b];
          yk[b] = acc;
        }
      }
    }
  }
  __syncthreads();
  // T^T on the rows of all the CTA's columns at once (the row's D and cp loads
  // are shared by the columns)
  const int ncol = min(kXformCols, d.nB - c0);
  if (ncol == kXformCols) {
    double* fcol[kXformCols];
#pragma unroll
    for (int k = 0; k < kXformCols; ++k) fcol[k] = d.F + (size_t)d.posF[c0 + k] * ld;
    for (int b = threadIdx.x; b < d.nB; b += blockDim.x) {
      const int ib = d.bglob[b], fb = d.posF[b];
      if (ib < 0) {
#pragma unroll
        for (int k = 0; k < kXformCols; ++k) fcol[k][fb] = y[k * d.nB + b];
        continue;
      }
      const int tr = x.inst_tr[ib], jb = d.bslot[b];
      const int* cp = x.cpos + x.inst_pos[ib];
      const int n = x.tr_n[tr], r = x.tr_r[tr];
      const double* D = x.D + x.tr_off_d[tr];
      double acc[kXformCols];
      const int cj = jb >= r ? cp[jb] : 0;
#pragma unroll
      for (int k = 0; k < kXformCols; ++k) acc[k] = jb >= r ? y[k * d.nB + cj] : 0.0;
      for (int i = 0; i < r; ++i) {
        const double dd = D[i * n + jb];
        const int ci = cp[i];
#pragma unroll
        for (int k = 0; k < kXformCols; ++k) acc[k] += dd * y[k * d.nB + ci];
      }
#pragma unroll
      for (int k = 0; k < kXformCols; ++k) fcol[k][fb] = acc[k];
    }
#pragma unroll
    for (int k = 0; k < kXformCols; ++k) {
      for (int q = nE + threadIdx.x; q < d.PE; q += blockDim.x) fcol[k][q] = 0.0;
      for (int q = d.PE + nC + threadIdx.x; q < d.NF; q += blockDim.x) fcol[k][q] = 0.0;
    }
    return;
  }
  for (int k = 0; k < kXformCols; ++k) {
    const int c = c0 + k;
    if (c < d.nB) {
      const double* yk = y + k * d.nB;
      double* fcol = d.F + (size_t)d.posF[c] * ld;
      for (int b = threadIdx.x; b < d.nB; b += blockDim.x) {
        const int ib = d.bglob[b];
        fcol[d.posF[b]] = ib < 0 ? yk[b] : xform_T_t_c(x, ib, d.bslot[b], yk);
      }
      for (int q = nE + threadIdx.x; q < d.PE; q += blockDim.x) fcol[q] = 0.0;
      for (int q = d.PE + nC + threadIdx.x; q < d.NF; q += blockDim.x) fcol[q] = 0.0;
    } else {
      const int kp = c - d.nB, npe = d.PE - nE;  // padding column kp: [nE, PE) then [PE + nC, NF)
      const int q = kp < npe ? nE + kp : d.PE + nC + (kp - npe);
      if (q >= d.NF) break;
      double* fcol = d.F + (size_t)q * ld;
      for (int rr = threadIdx.x; rr < d.NF; rr += blockDim.x) fcol[rr] = rr == q ? 1.0 : 0.0;
    }
  }
}

__global__ void k_pad_identity(double* Farena, const long long* foff, const int* NF, const int* pad_sub,
                               const int* pads, int npads) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < npads; t += gridDim.x * blockDim.x) {
    const int q = pads[t], s = pad_sub[t];
    Farena[foff[s] + (size_t)q * NF[s] + q] = 1.0;
  }
}

// Explicit leaf mode (few leaf fronts: the sweeps would leave most SMs idle).
// The transformed leaf front is augmented to [[F_ee, F_ec, I], [F_ce, F_cc, 0],
// [I, 0, 0]] and only the e block is eliminated; the trailing block then holds
//   [[S_cc, -W^T], [-W, -F_ee^{-1}]],  W = F_ee^{-1} F_ec,
// and both leaf sweeps of the preconditioner become parallel GEMVs with
// E = [-F_ee^{-1} | -W]  (PE x (PE + M), column-major, ld PE).
struct LeafX {
  const double* a;  // augmented front (ld n)
  double* E;
  double* FV;       // F-layout vector: right-hand side in, solution out
  double* FV2;      // forward result: [u = F_ee^{-1} b_e | y_c = b_c - W^T b_e]
  const int* cmap;  // M: root index of each coarse slot or -1
  int n, PE, M;
};

__global__ void k_aug_identity(const LeafX* ds) {
  const LeafX d = ds[blockIdx.y];
  double* a = const_cast<double*>(d.a);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d.PE; i += gridDim.x * blockDim.x)
    a[(size_t)i * d.n + d.PE + d.M + i] = 1.0;
}

// E from the lower triangle of the trailing block (element (r, c), r >= c, at
// a[(PE + c) n + PE + r]; trailing index: coarse slots [0, M), augmented [M, M + PE)).
__global__ void k_leaf_explicit_copy(const LeafX* ds) {
  const LeafX d = ds[blockIdx.y];
  const long total = (long)d.PE * (d.PE + d.M);
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(t % d.PE), j = static_cast<int>(t / d.PE);
    int r, c;
    if (j < d.PE) {
      r = d.M + max(i, j);
      c = d.M + min(i, j);
    } else {
      r = d.M + i;
      c = j - d.PE;
    }
    d.E[(size_t)j * d.PE + i] = d.a[(size_t)(d.PE + c) * d.n + d.PE + r];
  }
}

// forward: warp per column j of E (symmetric -F_ee^{-1}: column == row), b_e
// staged in smem (bs: PE doubles).  Column block cb = columns [8 cb, 8 cb + 8).
__device__ __forceinline__ void leaf_fwd_body(const LeafX& d, int cb, double* bs) {
  const int cols = d.PE + d.M;
  if (cb * 8 < cols) {
    for (int k = threadIdx.x; k < d.PE; k += blockDim.x) bs[k] = d.FV[k];
    __syncthreads();
    const int j = cb * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (j < cols) {
      // lane reads double2 k = lane + 32 t; eight loads in flight per lane
      const double2* col = reinterpret_cast<const double2*>(d.E + (size_t)j * d.PE);
      const double2* b2 = reinterpret_cast<const double2*>(bs);
      const int half = d.PE / 2;  // PE is a multiple of 64
      double s0 = 0.0, s1 = 0.0;
      for (int k0 = 0; k0 < half; k0 += 256) {
        double2 v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int k = k0 + 32 * t + lane;
          v[t] = k < half ? __ldg(col + k) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int k = k0 + 32 * t + lane;
          if (k < half) {
            const double2 bb = b2[k];
            s0 += v[t].x * bb.x;
            s1 += v[t].y * bb.y;
          }
        }
      }
      double s = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) d.FV2[j] = j < d.PE ? -s : d.FV[j] + s;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_leaf_fwd_explicit(const LeafX* ds, const int* done) {
  if (done && *done) return;
  extern __shared__ double bs[];
  leaf_fwd_body(ds[blockIdx.y], blockIdx.x, bs);
}

// backward: x_e = u - W x_c.  Row block rb: rows [64 rb, 64 rb + 64) of the
// F-layout vector; the four 64-thread groups split the coarse slots, partials
// reduced in a fixed order.  Coarse slots take the root values (xc: M doubles).
__device__ __forceinline__ void leaf_bwd_body(const LeafX& d, int rb, const double* __restrict__ croot, double* xc) {
  __shared__ double part[4][64];
  const int r0 = rb * 64;
  if (r0 < d.PE + d.M) {
    for (int c = threadIdx.x; c < d.M; c += blockDim.x) xc[c] = d.cmap[c] >= 0 ? croot[d.cmap[c]] : 0.0;
    __syncthreads();
    const int g = threadIdx.x >> 6, i = r0 + (threadIdx.x & 63);
    if (r0 >= d.PE) {  // coarse slots (PE is a multiple of 64)
      if (g == 0) d.FV[i] = xc[i - d.PE];
    } else {
      const double* w = d.E + (size_t)d.PE * d.PE + i;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int c = g;
      for (; c + 28 < d.M; c += 32) {  // eight loads in flight
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldg(w + (size_t)(c + 4 * q) * d.PE);
        s0 += v[0] * xc[c] + v[4] * xc[c + 16];
        s1 += v[1] * xc[c + 4] + v[5] * xc[c + 20];
        s2 += v[2] * xc[c + 8] + v[6] * xc[c + 24];
        s3 += v[3] * xc[c + 12] + v[7] * xc[c + 28];
      }
      for (; c + 12 < d.M; c += 16) {
        s0 += w[(size_t)c * d.PE] * xc[c];
        s1 += w[(size_t)(c + 4) * d.PE] * xc[c + 4];
        s2 += w[(size_t)(c + 8) * d.PE] * xc[c + 8];
        s3 += w[(size_t)(c + 12) * d.PE] * xc[c + 12];
      }
      for (; c < d.M; c += 4) s0 += w[(size_t)c * d.PE] * xc[c];
      part[g][threadIdx.x & 63] = (s0 + s1) + (s2 + s3);
      __syncthreads();
      if (g == 0)
        d.FV[i] = d.FV2[i] + ((part[0][threadIdx.x] + part[1][threadIdx.x]) + (part[2][threadIdx.x] + part[3][threadIdx.x]));
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_leaf_bwd_explicit(const LeafX* ds, const double* __restrict__ croot,
                                                           const int* done) {
  if (done && *done) return;
  extern __shared__ double xc[];
  leaf_bwd_body(ds[blockIdx.y], blockIdx.x, croot, xc);
}

// A child of a coarse front: its Schur complement onto its coarse slots is the
// lower triangle of the trailing block, a[(p + lo) ld + p + hi], hi >= lo.
struct AsmChild {
  const double* a;
  int ld;
  int p;
};

// A coarse front (a box of the primal tree, or the root): logical slots are the
// rows [0, ne) (eliminated here) and [PE, PE + nc) (passed up); rows are padded
// to NF.  Entry lists of row r: [ptr[pos0 + r], ptr[pos0 + r + 1]), ascending by child.
struct AsmFront {
  double* out;
  long ld;  // NF, or 2 NF for the augmented root [[R, .], [I, 0]]
  int ne, nc, PE, NF;
  long long pos0;
};

// Extend-add of the children's Schur complements into the lower triangle of
// each front (the reference's sparse assembly of the stabilized operator,
// bddc_operator.cpp:7-36, restricted to the primal unknowns):
// one thread per entry, the two rows' entry lists merged by child in a fixed
// order (deterministic, no atomics).
__global__ void k_front_assemble(const AsmFront* fr, const int* __restrict__ ptr, const int* __restrict__ child,
                                 const int* __restrict__ cidx, const AsmChild* __restrict__ kids) {
  const AsmFront f = fr[blockIdx.y];
  const int n = f.ne + f.nc;
  const long total = (long)n * (n + 1) / 2;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total; t += (long)gridDim.x * blockDim.x) {
    int i1 = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((long)i1 * (i1 + 1) / 2 > t) --i1;
    while ((long)(i1 + 1) * (i1 + 2) / 2 <= t) ++i1;
    const int i2 = static_cast<int>(t - (long)i1 * (i1 + 1) / 2);
    const int r1 = i1 < f.ne ? i1 : f.PE + i1 - f.ne, r2 = i2 < f.ne ? i2 : f.PE + i2 - f.ne;
    double s = 0.0;
    int a = ptr[f.pos0 + r1], b = ptr[f.pos0 + r2];
    const int ae = ptr[f.pos0 + r1 + 1], be = ptr[f.pos0 + r2 + 1];
    while (a < ae && b < be) {
      const int ca = child[a], cb = child[b];
      if (ca < cb) {
        ++a;
      } else if (cb < ca) {
        ++b;
      } else {
        const int c1 = cidx[a], c2 = cidx[b];
        const int hi = c1 >= c2 ? c1 : c2, lo = c1 >= c2 ? c2 : c1;
        const AsmChild k = kids[ca];
        s += k.a[(size_t)(k.p + lo) * k.ld + k.p + hi];
        ++a;
        ++b;
      }
    }
    f.out[(size_t)r2 * f.ld + r1] = s;
  }
}

// Identity on the padding rows; with ld > NF also the augmented identity block
// (eliminating R then leaves -R^{-1} in the trailing block).
__global__ void k_front_pads(const AsmFront* fr) {
  const AsmFront f = fr[blockIdx.y];
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < f.NF; q += (long)gridDim.x * blockDim.x) {
    if ((q >= f.ne && q < f.PE) || q >= f.PE + f.nc) f.out[(size_t)q * f.ld + q] = 1.0;
    if (f.ld > f.NF && q < f.ld - f.NF) f.out[(size_t)q * f.ld + f.NF + q] = 1.0;
  }
}

// x = -T b with T = -R^{-1} (full symmetric, NR x NR): one warp per output, reading
// one column of T (coalesced; symmetric so column == row).
__global__ void __launch_bounds__(256) k_root_gemv(int NR, const double* __restrict__ T, const double* __restrict__ b,
                                                   double* __restrict__ x, const int* done) {
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < NR; c += warps) {
    const double* col = T + (size_t)c * NR;
    double s0 = 0.0, s1 = 0.0;
    int r = lane;
    for (; r + 32 < NR; r += 64) {
      s0 += col[r] * b[r];
      s1 += col[r + 32] * b[r + 32];
    }
    if (r < NR) s0 += col[r] * b[r];
    double s = s0 + s1;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) x[c] = -s;
  }
}

// Small roots: every CTA gathers the whole root right-hand side (deterministic
// CSR sums, as k_root_gather) into shared memory, then applies -R^{-1}.
__global__ void __launch_bounds__(256) k_root_gather_gemv(int n_root, int NR, const int* __restrict__ ptr,
                                                          const long long* __restrict__ src,
                                                          const double* __restrict__ fv, const double* __restrict__ T,
                                                          double* __restrict__ x, const int* done) {
  if (done && *done) return;
  extern __shared__ double bs[];
  for (int k = threadIdx.x; k < NR; k += blockDim.x) {
    double s = 0.0;
    if (k < n_root)
      for (int t = ptr[k]; t < ptr[k + 1]; ++t) s += fv[src[t]];
    bs[k] = s;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < NR; c += warps) {
    const double* col = T + (size_t)c * NR;
    double s0 = 0.0, s1 = 0.0;
    int r = lane;
    for (; r + 32 < NR; r += 64) {
      s0 += col[r] * bs[r];
      s1 += col[r + 32] * bs[r + 32];
    }
    if (r < NR) s0 += col[r] * bs[r];
    double s = s0 + s1;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) x[c] = -s;
  }
}

// ---------------------------------------------------------------------------
// Fused coarse stage of the preconditioner apply (explicit primal-tree levels
// and a small root inverse on one GPU): the level gathers and forward GEMVs,
// the root gather + -R^{-1} GEMV and the level backward GEMVs are phases of
// ONE launch separated by grid barriers, instead of four to six dependent
// launches of a few microseconds of work each (cfg3/cfg4: 48 us of a 323/451 us
// apply).  Every CTA forms the gathered right-hand side it needs itself (the
// deterministic CSR sums of k_root_gather, so results are bit-identical to the
// separate launches); the grid is at most the co-resident CTAs.
// ---------------------------------------------------------------------------
constexpr int kCoarseLevels = 4;
struct CoarseLevelArgs {
  const LeafX* lx;         // explicit fronts of the level
  const int* ptr;          // gather CSR over the level's vector positions
  const long long* src;
  const double* vbase;     // the level's vector arena (LeafX::FV points into it)
  const double* fvsrc;     // children's forward results
  const double* up;        // parent's solution (backward)
  int nfr, ncb, nrb;       // fronts, 8-column blocks and 64-row blocks per front
};
struct CoarseArgs {
  CoarseLevelArgs lv[kCoarseLevels];
  int nlev;
  int n_root, NR;
  const int* root_ptr;
  const long long* root_src;
  const double* root_fvsrc;
  const double* Rinv;
  double* xroot;
  unsigned* bar;  // [0] arrivals, [1] CTAs done (the last one zeroes both)
};

__device__ __forceinline__ void coarse_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256, 3) k_coarse_explicit(const __grid_constant__ CoarseArgs a, const int* done) {
  if (done && *done) return;
  extern __shared__ double bs[];
  __shared__ double tail[8];
  unsigned phase = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the later phases' matrices (-R^{-1}, the levels' W blocks) do not depend on
  // the vector: their lines are requested into L2 now, behind the first
  // phase's own loads, so the phases after the barriers do not start cold
  {
    const size_t gtid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, gn = (size_t)gridDim.x * blockDim.x;
    const char* rinv = reinterpret_cast<const char*>(a.Rinv);
    for (size_t o = gtid * 128; o < (size_t)a.NR * a.NR * sizeof(double); o += gn * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rinv + o));
    for (int l = 0; l < a.nlev; ++l)
      for (int f = 0; f < a.lv[l].nfr; ++f) {
        const LeafX d = a.lv[l].lx[f];
        const char* w = reinterpret_cast<const char*>(d.E + (size_t)d.PE * d.PE);
        for (size_t o = gtid * 128; o < (size_t)d.PE * d.M * sizeof(double); o += gn * 128)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(w + o));
      }
  }
  for (int l = 0; l < a.nlev; ++l) {
    const CoarseLevelArgs& L = a.lv[l];
    for (int u = blockIdx.x; u < L.nfr * L.ncb; u += gridDim.x) {
      const LeafX d = L.lx[u / L.ncb];
      const int cb = u % L.ncb, cols = d.PE + d.M;
      if (cb * 8 >= cols) continue;
      const long long off = d.FV - L.vbase;
      // the column of E does not depend on the vector: its loads (the whole
      // column when PE <= 512) are in flight while the right-hand side is gathered
      const int j = cb * 8 + warp;
      const double2* col = reinterpret_cast<const double2*>(d.E + (size_t)min(j, cols - 1) * d.PE);
      const int half = d.PE / 2;
      double2 v0[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int k = 32 * t + lane;
        v0[t] = k < half ? __ldg(col + k) : make_double2(0.0, 0.0);
      }
      for (int k = threadIdx.x; k < d.PE; k += blockDim.x) bs[k] = csr_sum(L.ptr, L.src, L.fvsrc, off + k);
      if (lane == 0 && j >= d.PE && j < cols) tail[warp] = csr_sum(L.ptr, L.src, L.fvsrc, off + j);
      __syncthreads();
      if (j < cols) {
        const double2* b2 = reinterpret_cast<const double2*>(bs);
        double s0 = 0.0, s1 = 0.0;
        for (int k0 = 0; k0 < half; k0 += 256) {
          double2 v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int k = k0 + 32 * t + lane;
            v[t] = k0 == 0 ? v0[t] : (k < half ? __ldg(col + k) : make_double2(0.0, 0.0));
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int k = k0 + 32 * t + lane;
            if (k < half) {
              const double2 bb = b2[k];
              s0 += v[t].x * bb.x;
              s1 += v[t].y * bb.y;
            }
          }
        }
        double s = s0 + s1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) d.FV2[j] = j < d.PE ? -s : tail[warp] + s;
      }
      __syncthreads();
    }
    coarse_barrier(a.bar, ++phase * gridDim.x);
  }
  // root: every CTA gathers the whole right-hand side, then its columns of -R^{-1}
  if (blockIdx.x * 8 < a.NR) {
    for (int k0 = threadIdx.x; k0 < a.NR; k0 += 4 * blockDim.x) {  // four independent chains per thread
      double s[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + q * blockDim.x;
        s[q] = k < a.n_root ? csr_sum(a.root_ptr, a.root_src, a.root_fvsrc, k) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (k0 + q * blockDim.x < a.NR) bs[k0 + q * blockDim.x] = s[q];
    }
    __syncthreads();
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < a.NR; c += warps) {
      const double* col = a.Rinv + (size_t)c * a.NR;
      double s0 = 0.0, s1 = 0.0;
      int r = lane;
      for (; r + 32 < a.NR; r += 64) {
        s0 += col[r] * bs[r];
        s1 += col[r + 32] * bs[r + 32];
      }
      if (r < a.NR) s0 += col[r] * bs[r];
      double s = s0 + s1;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) a.xroot[c] = -s;
    }
  }
  for (int l = a.nlev - 1; l >= 0; --l) {
    coarse_barrier(a.bar, ++phase * gridDim.x);
    const CoarseLevelArgs& L = a.lv[l];
    for (int u = blockIdx.x; u < L.nfr * L.nrb; u += gridDim.x) leaf_bwd_body(L.lx[u / L.nrb], u % L.nrb, L.up, bs);
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(a.bar + 1, 1u) == gridDim.x - 1) {
    a.bar[0] = 0u;
    a.bar[1] = 0u;
    __threadfence();
  }
}

__global__ void k_extract_boundary(const SubDesc* sd, const double* MV, const long long* mvoff, const int* PI) {
  const SubDesc d = sd[blockIdx.x];
  for (int b = threadIdx.x; b < d.nB; b += blockDim.x) d.WB[b] = MV[mvoff[blockIdx.x] + PI[blockIdx.x] + b];
}

__global__ void k_scatter_solution(long long nmv, const long long* gdof, const double* MV, i64 niface,
                                   const long long* igdof, const double* uiface, double* u) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nmv; t += (long long)gridDim.x * blockDim.x)
    if (gdof[t] >= 0) u[gdof[t]] = MV[t];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < niface; i += (long long)gridDim.x * blockDim.x)
    u[igdof[i]] = uiface[i];
}

__global__ void k_insert_boundary(const SubDesc* sd, double* MV, const long long* mvoff, const int* PI,
                                  const double* __restrict__ u_iface) {
  const SubDesc d = sd[blockIdx.x];
  for (int b = threadIdx.x; b < d.nB; b += blockDim.x) MV[mvoff[blockIdx.x] + PI[blockIdx.x] + b] = u_iface[d.biface[b]];
}

// restrict / prolong at one boundary position (s, b): the same arithmetic as
// restrict_body / prolong_body, spread over every boundary copy instead of one
// CTA per substructure (the persistent PCG's latency-bound regime).
template <class In>
__device__ __forceinline__ void restrict_at(const SubDesc& d, const XformDesc& x, int b, In in) {
  const int inst = d.bglob[b];
  double y;
  if (inst < 0) {
    y = d.bw[b] * in(d.biface[b]);
  } else {
    const int tr = x.inst_tr[inst];
    const int* cp = x.cpos + x.inst_pos[inst];
    const int n = x.tr_n[tr], r = x.tr_r[tr], j = d.bslot[b];
    const double* D = x.D + x.tr_off_d[tr];
    double s0 = j >= r ? d.bw[cp[j]] * in(d.biface[cp[j]]) : 0.0, s1 = 0.0;
    int i = 0;
    for (; i + 1 < r; i += 2) {
      s0 += D[i * n + j] * (d.bw[cp[i]] * in(d.biface[cp[i]]));
      s1 += D[(i + 1) * n + j] * (d.bw[cp[i + 1]] * in(d.biface[cp[i + 1]]));
    }
    if (i < r) s0 += D[i * n + j] * (d.bw[cp[i]] * in(d.biface[cp[i]]));
    y = s0 + s1;
  }
  d.FV[d.posF[b]] = y;
}

// prolong, constrained rows: item k = row i of a glob instance of owned
// substructure item_sub[k]; one warp per item (dot product over the glob).
__device__ __forceinline__ void prolong_item(const SubDesc& d, const XformDesc& x, int k, double* yglob) {
  const int lane = threadIdx.x & 31;
  const int inst = x.item_inst[k], i = x.item_row[k];
  const int tr = x.inst_tr[inst];
  const int* pos = x.tpos + x.inst_pos[inst];
  const int n = x.tr_n[tr];
  const double* D = x.D + x.tr_off_d[tr] + i * n;
  double s = 0.0;
  for (int jj = lane; jj < n; jj += 32) s += D[jj] * d.FV[d.posF[pos[jj]]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) yglob[k] = s;
}

// Position-parallel restrict / prolong (every boundary copy of the owned
// substructures; wpos = (owned index, boundary position)).
__global__ void __launch_bounds__(256) k_restrict_pos(const SubDesc* sd, XformDesc x, const int2* __restrict__ wpos,
                                                      int nw, const double* __restrict__ r, const int* done) {
  if (done && *done) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nw; e += gridDim.x * blockDim.x) {
    const int2 sb = wpos[e];
    restrict_at(sd[sb.x], x, sb.y, [r](int i) { return r[i]; });
  }
}

__global__ void __launch_bounds__(256) k_prolong_items(const SubDesc* sd, XformDesc x, const int* __restrict__ item_sub,
                                                       int nitems, double* yglob, const int* done) {
  if (done && *done) return;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nitems; k += (gridDim.x * blockDim.x) >> 5)
    prolong_item(sd[item_sub[k]], x, k, yglob);
}

__global__ void __launch_bounds__(256) k_prolong_copy(const SubDesc* sd, const int2* __restrict__ wpos,
                                                      const int* __restrict__ wsrc, int nw,
                                                      const double* __restrict__ fv, const double* __restrict__ yglob,
                                                      const int* done) {
  if (done && *done) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nw; e += gridDim.x * blockDim.x) {
    const int2 sb = wpos[e];
    const SubDesc& d = sd[sb.x];
    const int src = wsrc[e];
    d.WB[sb.y] = d.bw[sb.y] * (src >= 0 ? fv[src] : yglob[-1 - src]);
  }
}

// Prolongation in one launch: the first pos_blocks CTAs copy the boundary
// positions that take a leaf-vector entry, the others form the constrained rows
// of the glob transforms (one warp per item, as prolong_item) and write the
// weighted value straight to the item's own boundary position (item_e) -- the
// same products as k_prolong_items + k_prolong_copy without the dependency
// between two launches.
__global__ void __launch_bounds__(256) k_prolong_fused(const SubDesc* sd, XformDesc x, const int2* __restrict__ wpos,
                                                       const int* __restrict__ wsrc, int nw, int pos_blocks,
                                                       const int* __restrict__ item_sub,
                                                       const int* __restrict__ item_e, int nitems,
                                                       const double* __restrict__ fv, const int* done) {
  if (done && *done) return;
  if (static_cast<int>(blockIdx.x) < pos_blocks) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nw; e += pos_blocks * blockDim.x) {
      const int src = wsrc[e];
      if (src < 0) continue;
      const int2 sb = wpos[e];
      const SubDesc& d = sd[sb.x];
      d.WB[sb.y] = d.bw[sb.y] * fv[src];
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const int warps = ((gridDim.x - pos_blocks) * blockDim.x) >> 5;
  for (int k = ((blockIdx.x - pos_blocks) * blockDim.x + threadIdx.x) >> 5; k < nitems; k += warps) {
    const SubDesc& d = sd[item_sub[k]];
    const int inst = x.item_inst[k], i = x.item_row[k];
    const int tr = x.inst_tr[inst];
    const int* pos = x.tpos + x.inst_pos[inst];
    const int n = x.tr_n[tr];
    const double* D = x.D + x.tr_off_d[tr] + i * n;
    double s = 0.0;
    for (int jj = lane; jj < n; jj += 32) s += D[jj] * d.FV[d.posF[pos[jj]]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const int2 sb = wpos[item_e[k]];
      d.WB[sb.y] = d.bw[sb.y] * s;
    }
  }
}

// Leaf forward, one kFwdTile-column tile of E per call: b_e staged once, each
// warp owns kFwdTile / 8 columns and keeps two of them (up to 16 loads) in
// flight.  16-column tiles give the 27 fronts of configs 1-2 756 work units
// (189 with 64-column tiles), about one per CTA of the grid (3 per SM).
constexpr int kFwdTile = 16;
__device__ __forceinline__ void leaf_fwd_tile(const LeafX& d, int t, double* bs) {
  const int cols = d.PE + d.M;
  if (t * kFwdTile >= cols) return;  // uniform over the CTA
  for (int k = threadIdx.x; k < d.PE; k += blockDim.x) bs[k] = d.FV[k];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = d.PE / 2;
  const double2* b2 = reinterpret_cast<const double2*>(bs);
  for (int u = 0; u < kFwdTile / 8; u += 2) {
    const int j0 = t * kFwdTile + warp + 8 * u, j1 = j0 + 8;
    const double2* c0 = reinterpret_cast<const double2*>(d.E + (size_t)min(j0, cols - 1) * d.PE);
    const double2* c1 = reinterpret_cast<const double2*>(d.E + (size_t)min(j1, cols - 1) * d.PE);
    double a0 = 0.0, a1 = 0.0, e0 = 0.0, e1 = 0.0;
    for (int k0 = 0; k0 < half; k0 += 256) {
      double2 v[8], w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = k0 + 32 * q + lane;
        v[q] = k < half ? __ldg(c0 + k) : make_double2(0.0, 0.0);
        w[q] = k < half ? __ldg(c1 + k) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = k0 + 32 * q + lane;
        if (k < half) {
          const double2 bb = b2[k];
          a0 += v[q].x * bb.x;
          a1 += v[q].y * bb.y;
          e0 += w[q].x * bb.x;
          e1 += w[q].y * bb.y;
        }
      }
    }
    double s0 = a0 + a1, s1 = e0 + e1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) {
      if (j0 < cols) d.FV2[j0] = j0 < d.PE ? -s0 : d.FV[j0] + s0;
      if (j1 < cols) d.FV2[j1] = j1 < d.PE ? -s1 : d.FV[j1] + s1;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Persistent PCG (pcg.cpp:28-77) for the latency-bound regime: explicit leaf
// operators and a small root inverse on one GPU.  One cooperative launch runs
// every iteration; grid barriers replace kernel boundaries and the scalars
// (alpha, beta, rz, the stopping test) are formed redundantly by every CTA
// from the same partials in the same order, so no CTA waits on another for
// them.  p and r are double-buffered so that the updates p = z + beta p and
// r -= alpha q fold into the phases that read them:
//   A  q_s = S_s (z + beta p)                 (and p' = z + beta p)
//   B  q = sum of copies, partial p'.q
//   C  alpha; x += alpha p'; r' = r - alpha q (partials r'.r'); restrict(r')
//   D  leaf forward   E  root gather + R^{-1}   F  leaf backward
//   G  prolong        H  z = sum of copies, partial r'.z
// ---------------------------------------------------------------------------
struct PcgPersist {
  const SubDesc* sd;
  XformDesc xf;
  const LeafX* lx;
  const int2* wpos;  // every boundary copy: (owned substructure index, boundary position)
  int nw;
  const int* wsrc;   // per boundary copy: leaf-vector index, or -1 - constrained item
  const int* wsrcg;  // the same, indexed by the global boundary position (phase H's gather)
  const double* bwg; // averaging weight per global boundary position
  const int* item_sub;
  int nitems;
  double* yglob;     // constrained rows of the prolongation
  double* FVall;     // leaf vectors (zeroed before the restriction writes them)
  long long nfv;
  int ns, nrb_schur, ncb_fwd, nrb_bwd;
  // root
  int n_root, NR;
  const int* root_ptr;
  const long long* root_src;
  const double* Rinv;
  const double* fvsrc;  // leaf forward results (root_src offsets)
  double* xroot;
  // interface
  i64 n;
  const int* icp;
  const int* icpos;
  const double* WB;
  double *x, *z, *q;
  double* p[2];
  double* r[2];
  double* part;  // 3 x G partials: p.q, r.r, r.z
  PcgState* st;
  double* alphas;
  double* betas;
  unsigned long long* trace;  // optional: %globaltimer at each phase end (CTA 0), 9 per iteration
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double grid_sum(const double* part, int G) {
  // every CTA: the same fixed-order sum of the G partials (thread sums, warp
  // shuffles, then the warps' sums in order)
  __shared__ double red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < G; i += blockDim.x) v += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double out = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) out += red[w];
  __syncthreads();
  return out;
}

__device__ __forceinline__ void cta_partial(double v, double* slot) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) *slot = v;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_pcg_persistent(PcgPersist P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  const int G = gridDim.x, me = blockIdx.x;
  const i64 gt = (i64)me * blockDim.x + threadIdx.x, gs = (i64)G * blockDim.x;
  double* part_pq = P.part;
  double* part_rr = P.part + G;
  double* part_rz = P.part + 2 * G;
  // scalars: identical in every CTA
  double rz = P.st->rz, beta = 0.0;
  int it = P.st->it;
  const int max_it = P.st->max_it, precond_residual = P.st->precond_residual;
  const double ref = P.st->ref, tol = P.st->tol;
  int done = P.st->done, cur = 0;
  while (!done) {
    const double* pold = P.p[cur];
    double* pnew = P.p[cur ^ 1];
    const double* rold = P.r[cur];
    double* rnew = P.r[cur ^ 1];
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 8] = gtimer();
    // A
    for (int vb = me; vb < P.nrb_schur * P.ns; vb += G) {
      const SubDesc& d = P.sd[vb / P.nrb_schur];
      const int r0 = (vb % P.nrb_schur) * 64;
      if (r0 < d.nB) {
        const double* z = P.z;
        const double b = beta;
        schur_rows_body(d, r0, [z, pold, b](int i) { return z[i] + b * pold[i]; }, sm);
      }
    }
    for (i64 i = gt; i < P.n; i += gs) pnew[i] = P.z[i] + beta * pold[i];
    for (i64 i = gt; i < P.nfv; i += gs) P.FVall[i] = 0.0;
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 0] = gtimer();
    // B
    {
      double acc = 0.0;
      for (i64 i = gt; i < P.n; i += gs) {
        double s = 0.0;
        for (int t = P.icp[i]; t < P.icp[i + 1]; ++t) s += P.WB[P.icpos[t]];
        P.q[i] = s;
        acc += s * pnew[i];
      }
      cta_partial(acc, part_pq + me);
    }
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 1] = gtimer();
    // C
    const double alpha = rz / grid_sum(part_pq, G);
    {
      double acc = 0.0;
      for (i64 i = gt; i < P.n; i += gs) {
        P.x[i] += alpha * pnew[i];
        const double ri = rold[i] - alpha * P.q[i];
        rnew[i] = ri;
        acc += ri * ri;
      }
      cta_partial(acc, part_rr + me);
    }
    {
      const double* q = P.q;
      const double a = alpha;
      for (i64 w = gt; w < P.nw; w += gs) {
        const int2 sb = P.wpos[w];
        restrict_at(P.sd[sb.x], P.xf, sb.y, [rold, q, a](int i) { return rold[i] - a * q[i]; });
      }
    }
    if (me == 0 && threadIdx.x == 0) P.alphas[it] = alpha;
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 2] = gtimer();
    // D
    for (int vb = me; vb < P.ncb_fwd * P.ns; vb += G) leaf_fwd_tile(P.lx[vb / P.ncb_fwd], vb % P.ncb_fwd, sm);
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 3] = gtimer();
    // E: every CTA gathers the root right-hand side, then its columns of -R^{-1}
    if (me * 8 < P.NR) {
      for (int k = threadIdx.x; k < P.NR; k += blockDim.x) {
        double s = 0.0;
        if (k < P.n_root)
          for (int t = P.root_ptr[k]; t < P.root_ptr[k + 1]; ++t) s += P.fvsrc[P.root_src[t]];
        sm[k] = s;
      }
      __syncthreads();
      const int lane = threadIdx.x & 31;
      for (int c = (me * blockDim.x + threadIdx.x) >> 5; c < P.NR; c += (G * blockDim.x) >> 5) {
        const double* col = P.Rinv + (size_t)c * P.NR;
        double s0 = 0.0, s1 = 0.0;
        int rr = lane;
        for (; rr + 32 < P.NR; rr += 64) {
          s0 += col[rr] * sm[rr];
          s1 += col[rr + 32] * sm[rr + 32];
        }
        if (rr < P.NR) s0 += col[rr] * sm[rr];
        double sum = s0 + s1;
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) P.xroot[c] = -sum;
      }
      __syncthreads();
    }
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 4] = gtimer();
    // F
    for (int vb = me; vb < P.nrb_bwd * P.ns; vb += G) leaf_bwd_body(P.lx[vb / P.nrb_bwd], vb % P.nrb_bwd, P.xroot, sm);
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 5] = gtimer();
    // G
    for (int k = (me * blockDim.x + threadIdx.x) >> 5; k < P.nitems; k += (G * blockDim.x) >> 5)
      prolong_item(P.sd[P.item_sub[k]], P.xf, k, P.yglob);
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 6] = gtimer();
    // H: the weighted prolongation of every copy is formed where the copies
    // are summed (same products, same order as writing WB and summing it)
    {
      double acc = 0.0;
      for (i64 i = gt; i < P.n; i += gs) {
        double s = 0.0;
        for (int t = P.icp[i]; t < P.icp[i + 1]; ++t) {
          const int g = P.icpos[t], src = P.wsrcg[g];
          s += __dmul_rn(P.bwg[g], src >= 0 ? P.FVall[src] : P.yglob[-1 - src]);  // rounded product, no FMA
        }
        P.z[i] = s;
        acc += s * rnew[i];
      }
      cta_partial(acc, part_rz + me);
    }
    grid.sync();
    if (P.trace && me == 0 && threadIdx.x == 0 && it < 64) P.trace[(size_t)it * 9 + 7] = gtimer();
    // beta and the stopping test (pcg.cpp:49-70)
    const double rz_next = grid_sum(part_rz, G);
    const double rr = grid_sum(part_rr, G);
    beta = rz_next / rz;
    rz = rz_next;
    if (me == 0 && threadIdx.x == 0) P.betas[it] = beta;
    ++it;
    const double res = precond_residual ? sqrt(fmax(rz_next, 0.0)) : sqrt(rr);
    const double relres = res / ref;
    done = (relres <= tol || it >= max_it) ? 1 : 0;
    cur ^= 1;
    if (done && me == 0 && threadIdx.x == 0) {
      P.st->rz = rz;
      P.st->beta = beta;
      P.st->alpha = alpha;
      P.st->it = it;
      P.st->relres = relres;
      P.st->done = 1;
    }
  }
  // the final iterate lives in x; p/r buffers need no copy back
}

}  // namespace

// ---------------------------------------------------------------------------
// Device state
// ---------------------------------------------------------------------------
struct DeviceState {
  // sharding: comm == nullptr is the single-GPU engine
  std::shared_ptr<Comm> comm;
  std::vector<int> owner;       // rank per substructure
  std::vector<int> act, own;    // active (owned + ghosts) and owned substructures, ascending
  std::vector<char> is_act, is_own;
  int n_act = 0, n_own = 0;
  // interface halo: this rank's partial interface sums are completed by
  // neighbour send/recv of the dofs it shares (ascending interface index per
  // peer); dot products run over the dofs it owns (lowest rank holding a copy)
  // and all-reduce kRed partials
  struct Halo {
    std::vector<int> peers, peer_off;   // peer_off: offsets into send/recv buffers
    std::vector<int> shared;            // interface indices, concatenated per peer
    std::vector<char> touched, owned_h;
    DBuf<int> pack, dof, ptr, src;
    DBuf<double> sendbuf, recvbuf, owned;
    int nsum = 0;
  } halo;
  std::vector<Segment> ghost_send, ghost_recv;  // S of ghost substructures (analysis)
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr, ef0 = nullptr, ef1 = nullptr, s0 = nullptr, s1 = nullptr, s2 = nullptr;
  cudaEvent_t eg0 = nullptr, eg1 = nullptr;  // eigen stage of a step (its hub stage starts behind the analysis)
  cudaStream_t copy_st = nullptr;            // host->device copies of an end-to-end step's inputs
  cudaEvent_t ecopy = nullptr;
  bool inputs_pending = false;
  DBuf<double> ufree;
  int nsub = 0;
  i64 niface = 0;
  std::vector<int> nI, nB, PI, PB, NM;
  std::vector<long long> m_off, dm_off, s_off, wb_off, mv_off;
  int max_NM = 0, max_PI = 0, max_PB = 0, max_nB = 0;
  bool prepared = false;
  struct HostStage {
    std::vector<int> lnode, pos, eke, biface, icp, icpos;
    std::vector<double> ke, escale, mv, bw;
  } h;
  DBuf<double> M, DinvM, S, MV, MV0, WB;
  DBuf<int> minfo, asm_lnode, asm_pos, asm_eke, asm_ipos, asm_dofq;
  DBuf<double> asm_ke, asm_escale;
  DBuf<AsmDesc> asmdesc;
  AsmMesh asm_mesh{};
  DBuf<TrailDesc> mtrail;
  DBuf<FrontDesc> mfront;
  DBuf<SolveDesc> msolve;
  DBuf<long long> d_mvoff;
  DBuf<int> d_PI;
  // interface maps
  DBuf<int> biface, bposF, bglob, bslot, icopy_ptr, icopy_pos;
  DBuf<double> bw;
  std::vector<int> h_posF;   // host copy of bposF (W^c entry points)
  ChangeOfVariables h_cov;   // the change of variables of the last set_constraints
  DBuf<double> rhs;  // condensed rhs (interface)
  DBuf<long long> sol_gdof, iface_gdof;
  // preconditioner
  bool have_prec = false;
  std::vector<int> NF, PE, nE, nC;
  std::vector<long long> f_off, df_off, fv_off;
  int max_NF = 0, max_PE = 0, max_M = 0;
  bool leaf_explicit = false;  // explicit leaf mode (k_leaf_*_explicit)
  std::vector<int> NA;         // F leading dimension (NF, or NF + PE augmented)
  int max_NA = 0, max_MA = 0;
  DBuf<double> F, DinvF, FV, FV2, Xtmp, E;  // F, DinvF, E, Xtmp: views into `stage`
  StageArena stage;
  DBuf<LeafX> leafx;
  DBuf<long long> d_xoff;
  DBuf<int> finfo;
  DBuf<FrontDesc> ffront;
  DBuf<SolveDesc> fsolve_fwd, fsolve_bwd;
  DBuf<SubDesc> subdesc;
  // transforms
  DBuf<int> inst_tr, inst_pos, tpos, tr_n, tr_r, tr_off_perm, tr_off_d, perm, iperm, cmap;
  DBuf<int> cpos, item_ptr, item_inst, item_row, inst_loff;
  int max_rows = 0;  // most constrained transform rows of one subdomain (prolong smem)
  DBuf<double> trD;
  XformDesc xf{};
  // root: the top front of the primal tree (all primal unknowns when the tree
  // has depth 0)
  int n_root = 0, NR = 0, n_primal = 0;
  DBuf<double> R, DinvR, xroot, xroot2, Rinv;
  bool root_inv = false;
  DBuf<TrailDesc> rtrail;
  DBuf<int> rinfo, root_ptr, root_child, root_c, d_NF, d_PE, pads, pad_sub;
  DBuf<long long> root_src, d_foff;
  DBuf<AsmChild> root_kids;
  DBuf<AsmFront> root_afront;
  DBuf<FrontDesc> rfront;
  DBuf<SolveDesc> rsolve;
  // primal tree levels below the root (coarse_tree.hpp), deepest first
  struct TreeLevel {
    DBuf<double> A, Dinv, V;  // fronts, diagonal-tile inverses, vectors
    DBuf<FrontDesc> fronts;
    DBuf<SolveDesc> fwd, bwd;
    DBuf<AsmFront> afronts;
    DBuf<AsmChild> kids;
    DBuf<int> info, ptr, child, cidx, cmap;
    DBuf<long long> src;
    int nfr = 0, max_NF = 0, max_PE = 0, max_M = 0, max_slots = 0;
    long long arena = 0;
    std::vector<int> NF, PE, nown, nupd;
    // explicit level (few fronts): augmented fronts [[F, I], [I, 0]] (ld NA =
    // NF + PE) whose elimination leaves E = [-F_ee^{-1} | -W]; both sweeps of
    // the level become GEMVs (k_leaf_*_explicit), forward results in V2
    bool expl = false;
    int max_NA = 0, max_MA = 0;
    std::vector<long long> xa_off, xe_off;
    long long xa_size = 0, xe_size = 0;
    DBuf<double> E, V2;
    DBuf<LeafX> lx;
  };
  std::vector<std::unique_ptr<TreeLevel>> tree;
  // fused coarse stage (k_coarse_explicit): explicit levels + small root inverse
  bool coarse_fused = false;
  CoarseArgs coarse_args{};
  int coarse_grid = 0, coarse_smem = 0;
  DBuf<unsigned> coarse_bar;
  int tree_depth = 0;
  double tree_apply_bytes = 0, tree_factor_bytes = 0;
  double* leaf_croot = nullptr;  // where the leaves' backward sweeps read their coarse values
  // pcg
  DBuf<double> vx, vr, vz, vp, vq, vb, part_a, part_b, alphas, betas;
  DBuf<double> vp2, vr2, part3;  // persistent PCG: second p/r buffers, 3 x G partials
  DBuf<int2> wpos;
  UploadBatch up_index, up_desc;  // set_constraints' small uploads (one copy each)
  int nw = 0;
  DBuf<int> wsrc, wsrcg, item_sub, item_e;
  DBuf<double> yglob;
  int nitems = 0;
  DBuf<PcgState> pst;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int pcg_grid = 0;
  std::size_t pcg_smem = 0;
  long long graph_kernels = 0;
  // adaptive pair machinery
  PairEngine pairs;

  // the step's host inputs (DeviceState::h) are page-locked in place once they
  // are built, so the end-to-end step's host->device copies are asynchronous
  // DMA transfers instead of staged pageable copies
  std::vector<void*> pinned;
  template <class T>
  void pin(std::vector<T>& v) {
    if (v.empty()) return;
    if (cudaHostRegister(v.data(), v.size() * sizeof(T), cudaHostRegisterDefault) == cudaSuccess)
      pinned.push_back(v.data());
    else
      cudaGetLastError();  // stays pageable (the copies are then staged)
  }
  ~DeviceState() {
    for (void* p : pinned) cudaHostUnregister(p);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    for (cudaEvent_t e : {ef0, ef1, s0, s1, s2, eg0, eg1, ecopy})
      if (e) cudaEventDestroy(e);
    if (copy_st) cudaStreamDestroy(copy_st);
    if (st) cudaStreamDestroy(st);
  }
};

Engine::Engine(const Model& m) : m_(m), d_(new DeviceState) {
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    throw Error(kCudaError, "no CUDA device: the B200 path has no CPU fallback");
  CK(cudaStreamCreateWithFlags(&d_->st, cudaStreamNonBlocking));
  CK(cudaEventCreate(&d_->e0));
  CK(cudaEventCreate(&d_->e1));
  CK(cudaEventCreate(&d_->ef0));
  CK(cudaEventCreate(&d_->ef1));
  CK(cudaEventCreate(&d_->s0));
  CK(cudaEventCreate(&d_->s1));
  CK(cudaEventCreate(&d_->s2));
  CK(cudaEventCreate(&d_->eg0));
  CK(cudaEventCreate(&d_->eg1));
  CK(cudaEventCreateWithFlags(&d_->ecopy, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&d_->copy_st, cudaStreamNonBlocking));
}

Engine::~Engine() = default;


void Engine::set_shard(std::shared_ptr<Comm> comm, const std::vector<int>& owner) {
  DeviceState& D = *d_;
  if (D.prepared) throw Error(kError, "set_shard must precede any device work");
  if (owner.size() != m_.subs.size()) throw Error(kError, "owner: one rank per substructure");
  for (int r : owner)
    if (r < 0 || r >= comm->world()) throw Error(kError, "owner rank out of range");
  D.comm = std::move(comm);
  D.owner = owner;
}

bool Engine::sharded() const { return d_->comm != nullptr; }

cudaStream_t Engine::stream() const { return d_->st; }
i64 Engine::interface_size() const { return static_cast<i64>(m_.maps.interface_dofs.size()); }
int Engine::root_size() const { return d_->n_root; }

namespace {
// device memory is tight (large runs): stage arenas are released after use
double free_bytes() {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 0.0;
  return double(fr);
}

// bytes a grow-only buffer needs beyond its current capacity
template <class T>
double growth(const DBuf<T>& b, long long n) {
  return n > (long long)b.cap ? double(n - (long long)b.cap) * sizeof(T) : 0.0;
}

constexpr double kMemMargin = 1.5e9;  // headroom kept free for small buffers and the runtime

double elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms * 1e-3;
}
}  // namespace

// ---------------------------------------------------------------------------
// prepare: host staging of the inputs (CSR, positions, maps, loads) and device
// allocations; upload_inputs: the host->device copies of those inputs;
// analysis: A_s -> dense fronts -> partial Cholesky (eliminate the interior),
// interface Schur complements, condensed rhs (spaces.cpp:108-147, schur.cpp:38-55).
// ---------------------------------------------------------------------------
namespace {
// Halo plan and ghost Schur-complement messages of a sharded engine
// (paper_0910_5863_b200/shard.py HaloPlan is the same plan in Python, the
// checker of this one: tests/test_multirank.py).
void build_halo(DeviceState& D, const Model& m) {
  auto& H = D.halo;
  const i64 n = D.niface;
  const HaloPlan plan = halo_plan(m, D.owner, D.comm->rank(), D.comm->world());
  H.peers = plan.peers;
  H.peer_off = plan.peer_off;
  H.shared = plan.shared;
  H.touched = plan.touched;
  H.owned_h = plan.owned;
  const std::vector<int>& dofs = plan.sum_dof;
  const std::vector<int>& ptr = plan.sum_ptr;
  const std::vector<int>& src = plan.sum_src;
  H.nsum = static_cast<int>(dofs.size());
  cudaStream_t st = D.st;
  auto up = [&](DBuf<int>& b, const std::vector<int>& v) {
    if (v.empty()) b.alloc(1); else b.upload(v, st);
  };
  up(H.pack, H.shared);
  up(H.dof, dofs);
  up(H.ptr, ptr);
  up(H.src, src);
  H.sendbuf.alloc(std::max<std::size_t>(H.shared.size(), 1));
  H.recvbuf.alloc(std::max<std::size_t>(H.shared.size(), 1));
  std::vector<double> ow(std::max<i64>(n, 1), 0.0);
  for (i64 i = 0; i < n; ++i) ow[i] = H.owned_h[i] ? 1.0 : 0.0;
  H.owned.upload(ow, st);
  // ghosts: the owner of each face pair's neighbour sends its S (copy_trailing_full
  // layout, PB^2 doubles) instead of this rank re-factoring the neighbour
  D.ghost_send.clear();
  D.ghost_recv.clear();
  std::vector<std::vector<int>> needs(D.nsub);  // ranks needing substructure s as a ghost
  for (const auto& pr : face_pairs(m)) {
    const int r = D.owner[std::min(pr.first, pr.second)];
    for (int s : {pr.first, pr.second})
      if (D.owner[s] != r) needs[s].push_back(r);
  }
  for (int s = 0; s < D.nsub; ++s) {
    std::sort(needs[s].begin(), needs[s].end());
    needs[s].erase(std::unique(needs[s].begin(), needs[s].end()), needs[s].end());
  }
  for (int s = 0; s < D.nsub; ++s) {  // ascending s on both sides: the k-th messages match
    const std::size_t nb = (std::size_t)D.PB[s] * D.PB[s];
    if (D.is_own[s])
      for (int r : needs[s]) D.ghost_send.push_back(Segment{r, D.S.p + D.s_off[s], nb});
    if (D.is_act[s] && !D.is_own[s]) D.ghost_recv.push_back(Segment{D.owner[s], D.S.p + D.s_off[s], nb});
  }
}

// Complete this rank's partial sums of an interface vector on every dof it
// touches (identical values on every rank holding the dof).
void halo_exchange(DeviceState& D, double* y) {
  auto& H = D.halo;
  cudaStream_t st = D.st;
  const int ns = static_cast<int>(H.shared.size());
  if (ns) {
    k_halo_pack<<<std::max(1, std::min(1024, (ns + 255) / 256)), 256, 0, st>>>(ns, H.pack.p, y, H.sendbuf.p);
    count_launch(1);
  }
  std::vector<Segment> sends, recvs;
  for (std::size_t k = 0; k < H.peers.size(); ++k) {
    const std::size_t off = H.peer_off[k], cnt = H.peer_off[k + 1] - H.peer_off[k];
    sends.push_back(Segment{H.peers[k], H.sendbuf.p + off, cnt});
    recvs.push_back(Segment{H.peers[k], H.recvbuf.p + off, cnt});
  }
  D.comm->exchange(sends, recvs, st);
  if (H.nsum) {
    k_halo_sum<<<std::max(1, std::min(1024, (H.nsum + 255) / 256)), 256, 0, st>>>(H.nsum, H.dof.p, H.ptr.p, H.src.p,
                                                                                 H.recvbuf.p, y);
    count_launch(1);
  }
}

// The complete vector on every rank (host-facing results): owned values, summed.
void complete_interface(DeviceState& D, double* y) {
  if (!D.comm) return;
  k_keep_owned<<<kRed, 256, 0, D.st>>>(D.niface, D.halo.owned.p, y);
  count_launch(1);
  D.comm->allreduce(y, D.niface, D.st);
}
}  // namespace

void Engine::prepare() {
  DeviceState& D = *d_;
  if (D.prepared) return;
  const Model& m = m_;
  ensure_sweep_workspace(D.st);
  D.nsub = static_cast<int>(m.subs.size());
  D.niface = interface_size();
  const int ns = D.nsub;
  // shard sets: owned substructures, plus the ghosts this rank's face pairs
  // need (a pair belongs to the owner of its lower substructure, shard.py)
  D.is_own.assign(ns, 1);
  D.is_act.assign(ns, 1);
  if (D.comm) {
    const int rank = D.comm->rank();
    for (int s = 0; s < ns; ++s) D.is_own[s] = D.owner[s] == rank;
    D.is_act = D.is_own;
    for (const auto& pr : face_pairs(m))
      if (D.owner[std::min(pr.first, pr.second)] == rank) D.is_act[pr.first] = D.is_act[pr.second] = 1;
  }
  D.act.clear();
  D.own.clear();
  for (int s = 0; s < ns; ++s) {
    if (D.is_act[s]) D.act.push_back(s);
    if (D.is_own[s]) D.own.push_back(s);
  }
  D.n_act = static_cast<int>(D.act.size());
  D.n_own = static_cast<int>(D.own.size());
  D.nI.resize(ns);
  D.nB.resize(ns);
  D.PI.resize(ns);
  D.PB.resize(ns);
  D.NM.resize(ns);
  D.m_off.resize(ns);
  D.dm_off.resize(ns);
  D.s_off.resize(ns);
  D.wb_off.assign(ns, 0);
  D.mv_off.resize(ns);
  long long mo = 0, dmo = 0, so = 0, wbo = 0, mvo = 0;
  for (int s = 0; s < ns; ++s) {
    const Subdomain& S = m.subs[s];
    D.nI[s] = static_cast<int>(S.interior.size());
    D.nB[s] = static_cast<int>(S.boundary.size());
    // leaf fronts for the owned substructures; the ghosts (neighbours this
    // rank's face pairs need) hold only their Schur complement S, received from
    // the owner after its factorization (exchange_ghost_schur)
    const bool a = D.is_act[s], o = D.is_own[s];
    D.PI[s] = o ? rup(D.nI[s], kTile) : 0;
    D.PB[s] = a ? rup(std::max(D.nB[s], 1), kTile) : 0;
    D.NM[s] = o ? D.PI[s] + D.PB[s] : 0;
    D.m_off[s] = mo;
    mo += (long long)D.NM[s] * D.NM[s];
    D.dm_off[s] = dmo;
    dmo += (long long)(D.PI[s] / kTile) * kTile * kTile;
    D.s_off[s] = so;
    so += (long long)D.PB[s] * D.PB[s];
    D.mv_off[s] = mvo;
    mvo += D.NM[s];
    if (D.is_own[s]) {
      D.wb_off[s] = wbo;
      wbo += D.nB[s];
    }
    if (!a) continue;
    D.max_NM = std::max(D.max_NM, D.NM[s]);
    D.max_PI = std::max(D.max_PI, D.PI[s]);
    D.max_PB = std::max(D.max_PB, D.PB[s]);
    D.max_nB = std::max(D.max_nB, D.nB[s]);
  }
  cudaStream_t st = D.st;
  D.M.alloc(std::max<long long>(mo, 1));
  D.DinvM.alloc(std::max<long long>(dmo, 1));
  D.S.alloc(std::max<long long>(so, 1));
  D.MV.alloc(std::max<long long>(mvo, 1));
  D.MV0.alloc(std::max<long long>(mvo, 1));
  D.WB.alloc(std::max<long long>(wbo, 1));
  // host staging of the assembly inputs: element data, local numbering and
  // dense positions per substructure, loads in front layout
  std::vector<long long> lnode_off(ns, 0), pos_off(ns, 0), ipos_off(ns, 0);
  long long ipos_n = 0;
  auto& H = D.h;
  H.lnode.clear();
  H.pos.clear();
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    lnode_off[s] = H.lnode.size();
    pos_off[s] = H.pos.size();
    H.lnode.insert(H.lnode.end(), S.lnode.begin(), S.lnode.end());
    std::vector<int> p(S.dim());
    for (int r = 0; r < D.nI[s]; ++r) p[S.interior[r]] = r;
    for (int b = 0; b < D.nB[s]; ++b) p[S.boundary[b]] = D.PI[s] + b;
    H.pos.insert(H.pos.end(), p.begin(), p.end());
    ipos_off[s] = ipos_n;
    ipos_n += D.NM[s];
  }
  H.ke.clear();
  for (const auto& k : m.ke_ref) H.ke.insert(H.ke.end(), k.begin(), k.end());
  H.eke = m.element_ke;
  H.escale = m.mesh.element_scale;
  H.mv.assign(std::max<long long>(mvo, 1), 0.0);
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    for (int r = 0; r < D.nI[s]; ++r) H.mv[D.mv_off[s] + r] = S.load[S.interior[r]];
    for (int b = 0; b < D.nB[s]; ++b) H.mv[D.mv_off[s] + D.PI[s] + b] = S.load[S.boundary[b]];
  }
  // interface maps and averaging weights (spaces.cpp:71-86); the weights use
  // every copy of a dof, the copy lists only this rank's copies
  H.biface.assign(std::max<long long>(wbo, 1), 0);
  H.bw.assign(std::max<long long>(wbo, 1), 0.0);
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    for (int b = 0; b < D.nB[s]; ++b) {
      const i64 g = S.global_dof[S.boundary[b]];
      H.biface[D.wb_off[s] + b] = static_cast<int>(m.maps.global_to_interface[g]);
      double tot = 0.0;
      for (i64 t = m.maps.copy_ptr[g]; t < m.maps.copy_ptr[g + 1]; ++t)
        tot += m.subs[m.maps.copy_sub[t]].diag[m.maps.copy_local[t]];
      H.bw[D.wb_off[s] + b] = S.diag[S.boundary[b]] / tot;
    }
  }
  std::vector<std::vector<int>> lists(D.niface);
  for (int s : D.own)
    for (int b = 0; b < D.nB[s]; ++b) lists[H.biface[D.wb_off[s] + b]].push_back(static_cast<int>(D.wb_off[s] + b));
  H.icp.assign(D.niface + 1, 0);
  H.icpos.clear();
  for (i64 i = 0; i < D.niface; ++i) {
    H.icp[i + 1] = H.icp[i] + static_cast<int>(lists[i].size());
    H.icpos.insert(H.icpos.end(), lists[i].begin(), lists[i].end());
  }
  D.asm_lnode.alloc(std::max<std::size_t>(H.lnode.size(), 1));
  D.asm_pos.alloc(std::max<std::size_t>(H.pos.size(), 1));
  D.asm_ipos.alloc(std::max<long long>(ipos_n, 1));
  D.asm_dofq.alloc(std::max<std::size_t>(H.pos.size(), 1));
  D.asm_eke.alloc(std::max<std::size_t>(H.eke.size(), 1));
  D.asm_ke.alloc(std::max<std::size_t>(H.ke.size(), 1));
  D.asm_escale.alloc(std::max<std::size_t>(H.escale.size(), 1));
  D.asm_mesh = AsmMesh{D.asm_ke.p, D.asm_eke.p, H.escale.empty() ? nullptr : D.asm_escale.p, m.mesh.ne[0],
                       m.mesh.ne[1], m.mesh.epe, m.mesh.ncomp};
  D.biface.alloc(std::max<long long>(wbo, 1));
  D.bw.alloc(std::max<long long>(wbo, 1));
  D.icopy_ptr.alloc(H.icp.size());
  D.icopy_pos.alloc(std::max<std::size_t>(H.icpos.size(), 1));
  D.minfo.alloc(std::max(D.n_own, 1));
  D.rhs.alloc(std::max<i64>(D.niface, 1));
  // descriptors: leaf fronts and interface operators over the owned
  // substructures (compacted, in ascending order)
  std::vector<AsmDesc> ad;
  std::vector<FrontDesc> fd;
  std::vector<SolveDesc> sv;
  std::vector<TrailDesc> td;
  for (int q = 0; q < D.n_own; ++q) {
    const int s = D.own[q];
    const Subdomain& S = m.subs[s];
    ad.push_back(AsmDesc{D.M.p + D.m_off[s], D.asm_lnode.p + lnode_off[s], D.asm_pos.p + pos_off[s], D.NM[s], D.nI[s],
                         D.PI[s], D.nB[s], S.origin[0], S.origin[1], S.origin[2], D.asm_ipos.p + ipos_off[s],
                         D.asm_dofq.p + pos_off[s], static_cast<int>(S.lnode.size()), S.dim()});
    fd.push_back(FrontDesc{D.M.p + D.m_off[s], D.DinvM.p + D.dm_off[s], D.NM[s], D.PI[s], D.minfo.p + q, 0,
                           D.nI[s], D.nB[s]});
    sv.push_back(SolveDesc{D.M.p + D.m_off[s], D.DinvM.p + D.dm_off[s], D.MV.p + D.mv_off[s], D.NM[s], D.PI[s],
                           nullptr, nullptr, D.nI[s], D.nB[s]});
    td.push_back(TrailDesc{D.M.p + D.m_off[s], D.S.p + D.s_off[s], D.NM[s], D.PI[s]});
  }
  std::vector<SubDesc> sd;
  std::vector<long long> mvo_own;
  std::vector<int> pi_own;
  for (int s : D.own) {
    sd.push_back(SubDesc{D.S.p + D.s_off[s], nullptr, nullptr, D.biface.p + D.wb_off[s], D.bw.p + D.wb_off[s],
                         nullptr, nullptr, nullptr, D.WB.p + D.wb_off[s], D.nB[s], D.PB[s], 0, 0, 0, 0});
    mvo_own.push_back(D.mv_off[s]);
    pi_own.push_back(D.PI[s]);
  }
  auto up = [&](auto& buf, const auto& v) {
    if (v.empty()) buf.alloc(1); else buf.upload(v, st);
  };
  up(D.asmdesc, ad);
  up(D.mfront, fd);
  up(D.msolve, sv);
  up(D.mtrail, td);
  up(D.subdesc, sd);
  up(D.d_mvoff, mvo_own);
  up(D.d_PI, pi_own);
  D.pairs.attach(m, D.S.p, D.s_off, D.PB, D.nB, st);
  D.pairs.set_region([this](std::size_t n) {
    bool lost = false;
    double* base = d_->stage.region(true, n, &lost);
    if (lost) invalidate_preconditioner();
    return base;
  });
  if (D.comm) {
    D.pairs.set_shard(D.comm, D.owner);
    build_halo(D, m);
  }
  D.prepared = true;
  D.pin(H.ke);
  D.pin(H.eke);
  D.pin(H.escale);
  D.pin(H.lnode);
  D.pin(H.pos);
  D.pin(H.mv);
  D.pin(H.biface);
  D.pin(H.bw);
  D.pin(H.icp);
  D.pin(H.icpos);
  upload_inputs();
  CK(cudaStreamSynchronize(st));
}

double Engine::upload_inputs(bool on_copy_stream) {
  DeviceState& D = *d_;
  auto& H = D.h;
  cudaStream_t st = on_copy_stream ? D.copy_st : D.st;
  double bytes = 0;
  auto cp = [&](void* dst, const void* src, std::size_t n) {
    if (n) CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
    bytes += double(n);
  };
  cp(D.asm_ke.p, H.ke.data(), H.ke.size() * sizeof(double));
  cp(D.asm_eke.p, H.eke.data(), H.eke.size() * sizeof(int));
  cp(D.asm_escale.p, H.escale.data(), H.escale.size() * sizeof(double));
  cp(D.asm_lnode.p, H.lnode.data(), H.lnode.size() * sizeof(int));
  cp(D.asm_pos.p, H.pos.data(), H.pos.size() * sizeof(int));
  cp(D.MV0.p, H.mv.data(), H.mv.size() * sizeof(double));
  cp(D.biface.p, H.biface.data(), H.biface.size() * sizeof(int));
  cp(D.bw.p, H.bw.data(), H.bw.size() * sizeof(double));
  cp(D.icopy_ptr.p, H.icp.data(), H.icp.size() * sizeof(int));
  cp(D.icopy_pos.p, H.icpos.data(), H.icpos.size() * sizeof(int));
  return bytes;
}

namespace {
// Leaf fronts from the reference element matrices: the
// inverse layout maps, then every block-lower entry of every front.
void assemble_fronts(DeviceState& D) {
  const int na = D.n_own;
  cudaStream_t st = D.st;
  if (!na) {
    if (D.inputs_pending) CK(cudaStreamWaitEvent(st, D.ecopy, 0));
    D.inputs_pending = false;
    return;
  }
  // the zero-fill needs only the front shapes: it runs while an end-to-end
  // step's inputs are still arriving on the copy stream (Engine::step)
  const int bx = static_cast<int>(std::max<long>(1, std::min<long>(D.max_NM, (16L * sm_count() + na - 1) / na)));
  k_zero_fronts<<<dim3(bx, na), 256, 0, st>>>(D.asmdesc.p);
  if (D.inputs_pending) {
    CK(cudaStreamWaitEvent(st, D.ecopy, 0));
    D.inputs_pending = false;
  }
  CK(cudaMemsetAsync(D.asm_ipos.p, 0xff, D.asm_ipos.n * sizeof(int), st));
  k_front_maps<<<dim3(16, na), 256, 0, st>>>(D.asmdesc.p);
  k_assemble_sparse<<<dim3(bx, na), 256, 0, st>>>(D.asmdesc.p, D.asm_mesh);
  count_launch(3);
}
}  // namespace

void Engine::analysis() {
  analysis_launch();
  analysis_finish();
}

void Engine::analysis_launch() {
  NvtxRange nvtx("bddc:analysis");
  prepare();
  DeviceState& D = *d_;
  const int na = D.n_own;
  cudaStream_t st = D.st;
  CK(cudaEventRecord(D.e0, st));
  D.minfo.zero(st);
  assemble_fronts(D);
  CK(cudaGetLastError());
  CK(cudaEventRecord(D.ef0, st));
  partial_cholesky(D.mfront.p, na, D.max_NM, D.max_PI, D.max_PB, st);
  CK(cudaEventRecord(D.ef1, st));
  CK(cudaGetLastError());
  copy_trailing_full(D.mtrail.p, na, D.max_PB, st);
  CK(cudaGetLastError());
  if (D.comm) D.comm->exchange(D.ghost_send, D.ghost_recv, st);  // S of the ghost substructures
  // condensed rhs: forward sweep on [f_I; f_B], then sum the boundary rows over copies
  CK(cudaMemcpyAsync(D.MV.p, D.MV0.p, D.MV.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  front_forward(D.msolve.p, na, D.max_NM, st);
  if (D.n_own) {
    k_extract_boundary<<<D.n_own, 256, 0, st>>>(D.subdesc.p, D.MV.p, D.d_mvoff.p, D.d_PI.p);
    count_launch(1);
  }
  k_sum_copies<<<kRed, 256, 0, st>>>(D.niface, D.icopy_ptr.p, D.icopy_pos.p, D.WB.p, D.rhs.p, nullptr, nullptr, nullptr);
  count_launch(1);
  CK(cudaGetLastError());
  if (D.comm) halo_exchange(D, D.rhs.p);  // interface neighbour exchange
  CK(cudaEventRecord(D.e1, st));
}

// waits for analysis_launch's work, checks the pivots
void Engine::analysis_finish() {
  DeviceState& D = *d_;
  times_.analysis = elapsed(D.e0, D.e1);
  times_.leaf_factor = elapsed(D.ef0, D.ef1);
  std::vector<int> info(std::max(D.n_own, 1));
  CK(cudaMemcpy(info.data(), D.minfo.p, info.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (int q = 0; q < D.n_own; ++q)
    if (info[q]) throw Error(kNotPositiveDefinite, "factorize: A_II of substructure " + std::to_string(D.own[q]) +
                                                       " is not positive definite");
  double fl = 0;
  for (int s : D.own) {
    const double ni = D.nI[s], nb = D.nB[s];
    fl += ni * ni * ni / 3.0 + ni * ni * nb + ni * nb * nb;
  }
  times_.flops_leaf = fl;
}

double Engine::schur_bytes() const {
  double b = 0;
  for (int s : d_->own) b += double(d_->nB[s]) * d_->nB[s] * 8.0;
  return b;
}

double Engine::pcg_bytes_per_iteration() const {
  const DeviceState& D = *d_;
  double b = schur_bytes();
  if (D.NF.size() == std::size_t(D.nsub))
    for (int s : D.own) {
      const double e = D.nE[s], c = D.nC[s];
      // explicit: E = [-F_ee^{-1} | -W] forward, W backward; factor: L twice
      b += (D.leaf_explicit ? e * (e + c) + e * c : 2.0 * (e * (e + 1) / 2 + e * c)) * 8.0;
    }
  b += double(D.n_root) * D.n_root * 8.0;  // R^{-1} GEMV, or both triangular root sweeps
  b += D.tree_apply_bytes;                  // both sweeps of every primal tree front
  // the W^c vectors of the apply ("about 6 * 8 * wc_dim"): here the
  // leaf vectors [e | c] only, the interiors being eliminated -- restriction
  // (write), forward sweep (read, write), backward sweep (read, write),
  // prolongation (read)
  if (D.NF.size() == std::size_t(D.nsub))
    for (int s : D.own) b += 6.0 * 8.0 * (D.nE[s] + D.nC[s]);
  return b;
}

double Engine::leaf_front_bytes() const {
  const DeviceState& D = *d_;
  double b = 0;
  if (D.NF.size() == std::size_t(D.nsub))
    for (int s : D.own) {
      const double e = D.nE[s], c = D.nC[s];
      b += (D.leaf_explicit ? e * e + c * e : e * (e + 1) / 2 + c * e) * 8.0;
    }
  b += double(D.n_root) * (D.n_root + 1) / 2 * 8.0 + D.tree_factor_bytes;
  return b;
}

// ---------------------------------------------------------------------------
// set_constraints: change of variables, transformed leaf fronts, dense root
// ---------------------------------------------------------------------------
void Engine::set_constraints(const ConstraintSet& cs) {
  NvtxRange nvtx("bddc:set_constraints");
  DeviceState& D = *d_;
  const Model& m = m_;
  const int ns = D.nsub;
  cudaStream_t st = D.st;
  CK(cudaEventRecord(D.e0, st));
  HostTimer ht("set_constraints");
  const ChangeOfVariables cov = change_of_variables(cs, m);
  ht.mark("change_of_variables");
  // boundary position of each local dof (owned substructures)
  std::vector<std::vector<int>> bpos_of(ns);
  const int no = D.n_own;
#pragma omp parallel for schedule(dynamic, 4) if (no >= 64)
  for (int q = 0; q < no; ++q) {
    const int s = D.own[q];
    bpos_of[s].assign(m.subs[s].dim(), -1);
    for (int b = 0; b < D.nB[s]; ++b) bpos_of[s][m.subs[s].boundary[b]] = b;
  }
  ht.mark("bpos");
  // transforms (flat) and per-subdomain instances
  // sizes and offsets first (sequential, cheap), then the fill in parallel
  const int ntr = static_cast<int>(cov.transforms.size());
  std::vector<int> tr_n(ntr), tr_r(ntr), tr_off_perm(ntr), tr_off_d(ntr), tr_inst0(ntr + 1, 0);
  std::vector<int> inst_tr, inst_pos;
  int np_total = 0, nd_total = 0, ntpos = 0;
  for (int k = 0; k < ntr; ++k) {
    const GlobTransform& gt = cov.transforms[k];
    tr_n[k] = gt.n;
    tr_r[k] = gt.rank;
    tr_off_perm[k] = np_total;
    tr_off_d[k] = nd_total;
    np_total += gt.n;
    nd_total += gt.rank * gt.n;
    int ninst = 0;
    for (int sq : m.globs[gt.glob].subdomains) {
      if (!D.is_own[sq]) continue;  // instances of this rank's substructures only
      inst_tr.push_back(k);
      inst_pos.push_back(ntpos);
      ntpos += gt.n;
      ++ninst;
    }
    tr_inst0[k + 1] = tr_inst0[k] + ninst;
  }
  std::vector<int> perm(np_total), iperm(np_total), tpos(ntpos);
  std::vector<int> bglob(D.WB.n, -1), bslot(D.WB.n, -1);
#pragma omp parallel for schedule(dynamic, 16) if (ntr >= 512)
  for (int k = 0; k < ntr; ++k) {
    const GlobTransform& gt = cov.transforms[k];
    const int n = gt.n, r = gt.rank;
    for (int i = 0; i < n; ++i) {
      perm[tr_off_perm[k] + i] = gt.perm[i];
      iperm[tr_off_perm[k] + gt.perm[i]] = i;
    }
    const auto& dofs = m.glob_dofs[gt.glob];
    int inst = tr_inst0[k];
    for (int s : m.globs[gt.glob].subdomains) {
      if (!D.is_own[s]) continue;
      for (int a = 0; a < n; ++a) {
        const int b = bpos_of[s][m.maps.local_of(dofs[a], s)];
        tpos[inst_pos[inst] + a] = b;
        bglob[D.wb_off[s] + b] = inst;
        bslot[D.wb_off[s] + b] = a;
      }
      ++inst;
    }
  }
  ht.mark("transforms");
  // composite slot positions and the per-subdomain constrained-row work lists
  std::vector<int> cpos(tpos.size()), inst_loff(inst_tr.size()), item_ptr(no + 1, 0), item_inst, item_row;
  {
    std::vector<int> inst_sub(inst_tr.size());
    for (std::size_t k = 0, inst = 0; k < cov.transforms.size(); ++k)
      for (int s : m.globs[cov.transforms[k].glob].subdomains)
        if (D.is_own[s]) inst_sub[inst++] = s;
    std::vector<std::vector<int>> by_sub(ns);
    const int ninst = static_cast<int>(inst_tr.size());
#pragma omp parallel for schedule(static) if (ninst >= 1024)
    for (int inst = 0; inst < ninst; ++inst) {
      const int tr = inst_tr[inst];
      for (int i = 0; i < tr_n[tr]; ++i) cpos[inst_pos[inst] + i] = tpos[inst_pos[inst] + perm[tr_off_perm[tr] + i]];
    }
    for (int inst = 0; inst < ninst; ++inst) by_sub[inst_sub[inst]].push_back(inst);
    D.max_rows = 0;
    for (int q = 0; q < no; ++q) {  // compacted over the owned substructures (k_prolong's blocks)
      const int s = D.own[q];
      int off = 0;
      for (int inst : by_sub[s]) {
        inst_loff[inst] = off;
        for (int i = 0; i < tr_r[inst_tr[inst]]; ++i) {
          item_inst.push_back(inst);
          item_row.push_back(i);
        }
        off += tr_r[inst_tr[inst]];
      }
      item_ptr[q + 1] = static_cast<int>(item_inst.size());
      D.max_rows = std::max(D.max_rows, off);
    }
  }
  ht.mark("items");
  // coarse dofs per subdomain: corners (ascending corner id), then explicit dofs (group order)
  std::vector<std::vector<int>> coarse_b(ns), coarse_root(ns);
  const i64 ncd = m.maps.corner_dof_count;
#pragma omp parallel for schedule(dynamic, 4) if (no >= 64)
  for (int q = 0; q < no; ++q) {
    const int s = D.own[q];
    const Subdomain& S = m.subs[s];
    std::vector<std::pair<i64, int>> cors;
    for (int b = 0; b < D.nB[s]; ++b) {
      const i64 cid = m.maps.corner_dof_of_global[S.global_dof[S.boundary[b]]];
      if (cid >= 0) cors.emplace_back(cid, b);
    }
    std::sort(cors.begin(), cors.end());
    for (auto& [cid, b] : cors) {
      coarse_b[s].push_back(b);
      coarse_root[s].push_back(static_cast<int>(cid));
    }
  }
  for (std::size_t g = 0; g < cov.groups.size(); ++g)
    for (std::size_t t = 0; t < cov.group_subs[g].size(); ++t) {
      const int s = cov.group_subs[g][t];
      if (!D.is_own[s]) continue;
      coarse_b[s].push_back(bpos_of[s][cov.group_local[g][t]]);
      coarse_root[s].push_back(static_cast<int>(ncd + g));
    }
  D.n_primal = static_cast<int>(ncd + cov.groups.size());
  ht.mark("coarse");
  // F layout
  D.NF.assign(ns, 0);
  D.PE.assign(ns, 0);
  D.nE.assign(ns, 0);
  D.nC.assign(ns, 0);
  D.f_off.assign(ns, 0);
  D.df_off.assign(ns, 0);
  D.fv_off.assign(ns, 0);
  std::vector<int> posF(D.WB.n, 0), cmap, pads, pad_sub;
  std::vector<long long> cmap_off(ns), pad_off(ns + 1), xoff;
  long long fo = 0, dfo = 0, fvo = 0, xo = 0;
  D.max_NF = D.max_PE = D.max_M = D.max_NA = D.max_MA = 0;
  D.NA.assign(ns, 0);
  std::vector<long long> e_off(ns);
  long long eo = 0;
  {
    // explicit leaf mode when the leaf fronts cannot fill the SMs (BDDC_B200_LEAF
    // = explicit | factor overrides)
    const char* env = std::getenv("BDDC_B200_LEAF");
    const std::string mode = env ? env : "";
    D.leaf_explicit = mode == "explicit" || (mode != "factor" && no < sm_count());
  }
  for (int s : D.own) {
    const int nB = D.nB[s], nC = static_cast<int>(coarse_b[s].size()), nE = nB - nC;
    D.nE[s] = nE;
    D.nC[s] = nC;
    D.PE[s] = rup(nE, kTile);
    D.NF[s] = D.PE[s] + rup(std::max(nC, 1), kTile);
    D.NA[s] = D.leaf_explicit ? D.NF[s] + D.PE[s] : D.NF[s];
    D.f_off[s] = fo;
    fo += (long long)D.NA[s] * D.NA[s];
    e_off[s] = eo;
    if (D.leaf_explicit) eo += (long long)D.PE[s] * D.NF[s];
    D.df_off[s] = dfo;
    dfo += (long long)(D.PE[s] / kTile) * kTile * kTile;
    D.fv_off[s] = fvo;
    fvo += D.NF[s];
    xoff.push_back(xo);  // compacted (k_colxform's blocks)
    xo += (long long)D.PB[s] * D.PB[s];
    D.max_NF = std::max(D.max_NF, D.NF[s]);
    D.max_PE = std::max(D.max_PE, D.PE[s]);
    D.max_M = std::max(D.max_M, D.NF[s] - D.PE[s]);
    D.max_NA = std::max(D.max_NA, D.NA[s]);
    D.max_MA = std::max(D.max_MA, D.NA[s] - D.PE[s]);
    cmap_off[s] = cmap.size();
    for (int c = 0; c < D.NF[s] - D.PE[s]; ++c) cmap.push_back(c < nC ? coarse_root[s][c] : -1);
    pad_off[s] = pads.size();
    for (int q = nE; q < D.PE[s]; ++q) {
      pads.push_back(q);
      pad_sub.push_back(s);
    }
    for (int q = D.PE[s] + nC; q < D.NF[s]; ++q) {
      pads.push_back(q);
      pad_sub.push_back(s);
    }
  }
  pad_off[ns] = pads.size();
  // row of each boundary dof in its leaf front [e | c] (independent per substructure)
#pragma omp parallel for schedule(dynamic, 16) if (no >= 64)
  for (int q = 0; q < no; ++q) {
    const int s = D.own[q];
    const int nB = D.nB[s], nC = D.nC[s];
    std::vector<int> is_coarse(nB, -1);
    for (int c = 0; c < nC; ++c) is_coarse[coarse_b[s][c]] = c;
    int e = 0;
    for (int b = 0; b < nB; ++b)
      posF[D.wb_off[s] + b] = is_coarse[b] >= 0 ? D.PE[s] + is_coarse[b] : e++;
  }
  ht.mark("f_layout");
  // primal tree over the substructure lattice (coarse_tree.hpp); its top front
  // is the root.  Depth 0 = one dense root over all primal unknowns (always
  // when sharded: the root is then gathered over the ranks).
  CoarseTree plan;
  {
    std::vector<CoarseLeaf> leaves(no);
    for (int q = 0; q < no; ++q) {
      const int s = D.own[q];
      leaves[q].coarse = coarse_root[s];
      for (int a = 0; a < 3; ++a) leaves[q].coord[a] = m.subs[s].origin[a] / m.mesh.epe;
      leaves[q].src0 = D.fv_off[s] + D.PE[s];
    }
    int depth = 0;
    int maxd = coarse_tree_max_depth(m.mesh.sub);
    // Sharded: every rank plans the same boxes from the bounds of each primal
    // unknown over ALL substructures and keeps the fronts of its own boxes; the
    // top front is summed over the ranks.  The depth is chosen on the global
    // symbolic plan, so every rank takes the same one; a partition whose blocks
    // cut through the depth-1 boxes keeps the dense root (depth 0).
    CoarseBounds bounds;
    std::vector<CoarseLeaf> all_leaves;
    if (D.comm) {
      maxd = coarse_tree_shard_depth(m.mesh.sub, D.owner, maxd);
      all_leaves = primal_leaves(m, cov, &bounds);
    }
    const std::vector<CoarseLeaf>& cost_leaves = D.comm ? all_leaves : leaves;
    const char* env = std::getenv("BDDC_B200_ROOT_DEPTH");
    if (env && *env) {
      depth = std::max(0, std::min(std::atoi(env), maxd));
    } else if (maxd > 0) {
      // candidate depths planned symbolically in parallel, the cheapest kept
      std::vector<double> cost(maxd + 1);
      std::vector<CoarseTree> cand(maxd + 1);
#pragma omp parallel for schedule(static, 1) if (cost_leaves.size() >= 256)
      for (int d = 0; d <= maxd; ++d) {
        cand[d] = plan_coarse_tree(cost_leaves, m.mesh.sub, D.n_primal, d, kRootInverseMax, true);
        cost[d] = coarse_tree_cost(cand[d], kTreeApplies, kRootInverseMax);
      }
      for (int d = 1; d <= maxd; ++d)
        if (cost[d] < cost[depth]) depth = d;
      if (!D.comm) plan = std::move(cand[depth]);
      ht.mark("tree_depths");
    }
    if (plan.leaf_box.empty() && plan.top.empty())
      plan = plan_coarse_tree(leaves, m.mesh.sub, D.n_primal, depth, kRootInverseMax, false,
                              D.comm ? &bounds : nullptr);
    else
      complete_coarse_tree(plan, leaves);
    ht.mark("tree_plan");
    for (int q = 0; q < no; ++q) {
      const int s = D.own[q];
      for (int c = 0; c < D.nC[s]; ++c) cmap[cmap_off[s] + c] = plan.leaf_cmap[q][c];
    }
  }
  D.tree_depth = plan.depth;
  if (const char* e = std::getenv("BDDC_B200_PROFILE"); e && *e && *e != '0') {
    std::string line = "[profile] primal tree: " + std::to_string(D.n_primal) + " unknowns, depth " +
                       std::to_string(plan.depth);
    for (const auto& L : plan.levels) {
      long long own = 0;
      for (const auto& f : L.fronts) own += static_cast<long long>(f.own.size());
      line += ", " + std::to_string(L.fronts.size()) + " fronts (" + std::to_string(own) + " eliminated, max " +
              std::to_string(L.max_NF) + " rows)";
    }
    line += ", top " + std::to_string(plan.top.size()) + ", est " + std::to_string(plan.flops / 1e9) + " GF";
    std::fprintf(stderr, "%s\n", line.c_str());
  }
  D.n_root = static_cast<int>(plan.top.size());
  D.NR = rup(std::max(D.n_root, 1), kTile);
  // root front; up to kRootInverseMax rows it is augmented to [[R, .], [I, 0]] so
  // that the factorization leaves -R^{-1} and every apply is one parallel GEMV
  {
    const char* env = std::getenv("BDDC_B200_ROOT");  // inverse | sweep (testing override)
    const std::string mode = env ? env : "";
    D.root_inv = mode == "inverse" || (mode != "sweep" && D.NR <= kRootInverseMax);
  }
  ht.mark("index_build");
  // uploads: the index arrays in one copy (batch A), then the descriptors that
  // point into them and into the arenas (batch B)
  UploadBatch& UA = D.up_index;
  UploadBatch& UB = D.up_desc;
  UA.add(D.bposF, posF);
  D.h_posF = posF;
  UA.add(D.bglob, bglob);
  UA.add(D.bslot, bslot);
  auto up_i = [&](DBuf<int>& b, const std::vector<int>& v) { UA.add(b, v); };
  up_i(D.inst_tr, inst_tr);
  up_i(D.inst_pos, inst_pos);
  up_i(D.tpos, tpos);
  up_i(D.tr_n, tr_n);
  up_i(D.tr_r, tr_r);
  up_i(D.tr_off_perm, tr_off_perm);
  up_i(D.tr_off_d, tr_off_d);
  up_i(D.perm, perm);
  up_i(D.iperm, iperm);
  up_i(D.cmap, cmap);
  // the transforms' rows (D[i][j] = t_perm[i][j] = t[perm[i]][j]; 70 MB on cfg5)
  // are written straight into the upload blob
  UA.add_fill(D.trD, static_cast<std::size_t>(nd_total), [&](double* dst) {
#pragma omp parallel for schedule(dynamic, 16) if (ntr >= 512)
    for (int k = 0; k < ntr; ++k) {
      const GlobTransform& gt = cov.transforms[k];
      std::memcpy(dst + tr_off_d[k], gt.D.data(), sizeof(double) * std::size_t(gt.rank) * gt.n);
    }
  });
  up_i(D.cpos, cpos);
  up_i(D.item_ptr, item_ptr);
  up_i(D.item_inst, item_inst);
  up_i(D.item_row, item_row);
  up_i(D.inst_loff, inst_loff);
  {
    // position-parallel restrict / prolong: per boundary copy of the owned
    // substructures, the leaf-vector index it copies or the constrained item
    // it takes (prolong_body's two cases)
    // boundary copies in owned order; the (substructure, position) list is
    // fixed by the model, so it is uploaded once
    std::vector<long long> w0(no + 1, 0);
    for (int q = 0; q < no; ++q) w0[q + 1] = w0[q] + D.nB[D.own[q]];
    if (D.nw != static_cast<int>(w0[no]) || D.wpos.n == 0 || !D.wpos.owned) {
      std::vector<int2> wp(w0[no]);
      for (int q = 0; q < no; ++q)
        for (int b = 0; b < D.nB[D.own[q]]; ++b) wp[w0[q] + b] = make_int2(q, b);
      D.wpos.release();
      D.wpos.upload(wp, st);
      D.nw = static_cast<int>(w0[no]);
    }
    std::vector<int> wsrc(std::max<long long>(w0[no], 1)), isub(item_inst.size()),
        item_e(std::max<std::size_t>(item_inst.size(), 1), 0);
    std::vector<int> wsrcg(std::max<std::size_t>(D.WB.n, 1), 0);  // unowned positions: never summed by phase H
#pragma omp parallel for schedule(dynamic, 16) if (no >= 64)
    for (int q = 0; q < no; ++q) {
      const int s = D.own[q];
      for (int k = item_ptr[q]; k < item_ptr[q + 1]; ++k) isub[k] = q;
      for (int b = 0; b < D.nB[s]; ++b) {
        const long long w = D.wb_off[s] + b;
        const int inst = bglob[w];
        int src = static_cast<int>(D.fv_off[s]) + posF[w];
        if (inst >= 0) {
          const int tr = inst_tr[inst];
          const int i = iperm[tr_off_perm[tr] + bslot[w]];
          if (i < tr_r[tr]) {
            src = -1 - (item_ptr[q] + inst_loff[inst] + i);
            item_e[item_ptr[q] + inst_loff[inst] + i] = static_cast<int>(w0[q] + b);
          }
          else
            src = static_cast<int>(D.fv_off[s]) + posF[D.wb_off[s] + tpos[inst_pos[inst] + i]];
        }
        wsrc[w0[q] + b] = src;
        wsrcg[w] = src;
      }
    }
    up_i(D.wsrc, wsrc);
    up_i(D.wsrcg, wsrcg);
    up_i(D.item_sub, isub);
    up_i(D.item_e, item_e);
    D.nitems = static_cast<int>(item_inst.size());
    D.yglob.alloc(std::max(D.nitems, 1));
  }
  UA.add(D.d_xoff, xoff);
  D.tree.resize(plan.levels.size());
  for (auto& T : D.tree)
    if (!T) T.reset(new DeviceState::TreeLevel);
  for (std::size_t l = 0; l < plan.levels.size(); ++l) {
    DeviceState::TreeLevel& T = *D.tree[l];
    const CoarseTree::Level& P = plan.levels[l];
    up_i(T.ptr, P.ptr);
    up_i(T.child, P.child);
    up_i(T.cidx, P.cidx);
    up_i(T.cmap, P.cmap);
    UA.add(T.src, P.src);
  }
  up_i(D.root_ptr, plan.top_ptr);
  up_i(D.root_child, plan.top_child);
  up_i(D.root_c, plan.top_cidx);
  UA.add(D.root_src, plan.top_src);
  UA.add(D.d_foff, D.f_off);
  up_i(D.d_NF, D.NA);  // leading dimensions of the F fronts
  up_i(D.d_PE, D.PE);
  up_i(D.pads, pads);
  up_i(D.pad_sub, pad_sub);
  UA.flush(st);
  ht.mark("upload_index");
  D.xf = XformDesc{D.inst_tr.p, D.inst_pos.p, D.tpos.p, D.tr_n.p, D.tr_r.p, D.tr_off_perm.p, D.tr_off_d.p,
                   D.perm.p, D.iperm.p, D.trD.p, D.cpos.p, D.item_ptr.p, D.item_inst.p, D.item_row.p,
                   D.inst_loff.p};
  // Preconditioner arenas: views into the stage arena (shared with the pair
  // stage).  [F | DinvF | E | Xtmp], with the root and the primal tree over the
  // transform scratch Xtmp (dead once F is formed).
  for (std::size_t l = 0; l < plan.levels.size(); ++l) {
    DeviceState::TreeLevel& T = *D.tree[l];
    const CoarseTree::Level& P = plan.levels[l];
    const char* env = std::getenv("BDDC_B200_TREE");  // explicit | factor (testing override)
    const std::string mode = env ? env : "";
    T.expl = mode == "explicit" || (mode != "factor" && static_cast<int>(P.fronts.size()) < sm_count());
    T.xa_off.assign(P.fronts.size(), 0);
    T.xe_off.assign(P.fronts.size(), 0);
    T.xa_size = T.xe_size = 0;
    T.max_NA = T.max_MA = 0;
    for (std::size_t f = 0; f < P.fronts.size(); ++f) {
      const CoarseTree::Front& F = P.fronts[f];
      const long long NA = T.expl ? (long long)F.NF + F.PE : F.NF;
      T.xa_off[f] = T.xa_size;
      T.xa_size += NA * NA;
      T.xe_off[f] = T.xe_size;
      if (T.expl) T.xe_size += (long long)F.PE * F.NF;
      T.max_NA = std::max<int>(T.max_NA, static_cast<int>(NA));
      T.max_MA = std::max<int>(T.max_MA, static_cast<int>(NA - F.PE));
    }
  }
  {
    const long long ldR0 = D.root_inv ? 2LL * D.NR : D.NR;
    RegionPlan lead, scratch, late;
    lead.add(D.F, fo);
    lead.add(D.DinvF, dfo);
    if (D.leaf_explicit) lead.add(D.E, eo);
    if (D.leaf_explicit) scratch.add(D.Xtmp, xo);  // factor mode: k_xform_fused needs no scratch
    late.add(D.R, ldR0 * ldR0);
    late.add(D.DinvR, (long long)D.NR * kTile);
    if (D.root_inv) late.add(D.Rinv, (long long)D.NR * D.NR);
    for (std::size_t l = 0; l < plan.levels.size(); ++l) {
      late.add(D.tree[l]->A, D.tree[l]->xa_size);
      late.add(D.tree[l]->Dinv, plan.levels[l].d_size);
      if (D.tree[l]->expl) late.add(D.tree[l]->E, D.tree[l]->xe_size);
    }
    const std::size_t total = lead.total() + std::max(scratch.total(), late.total());
    const double room = total <= D.stage.capacity() ? 0.0 : double(D.stage.capacity()) * 8.0 + free_bytes();
    if (total > D.stage.capacity() && double(total) * 8.0 > room)
      throw Error(kError, "preconditioner needs " + std::to_string(total * 8.0 / 1e9) + " GB (root " +
                              std::to_string(D.n_root) + " primal unknowns); " + std::to_string(room / 1e9) +
                              " GB available");
    bool lost = false;
    double* base = D.stage.region(false, total, &lost);
    lead.place(base);
    scratch.place(base + lead.total());
    late.place(base + lead.total());
  }
  ht.mark("regions");
  D.FV.alloc(std::max<long long>(fvo, 1));
  D.FV.zero(st);
  if (D.leaf_explicit) {
    D.FV2.alloc(std::max<long long>(fvo, 1));
    D.FV2.zero(st);
  }
  D.finfo.alloc(std::max(no, 1));
  D.finfo.zero(st);
  std::vector<SubDesc> sd(no);
  std::vector<FrontDesc> fd(no);
  std::vector<SolveDesc> fw(no), bw(no);
  for (int q = 0; q < no; ++q) {
    const int s = D.own[q];
    sd[q] = SubDesc{D.S.p + D.s_off[s], D.F.p + D.f_off[s], D.FV.p + D.fv_off[s], D.biface.p + D.wb_off[s],
                    D.bw.p + D.wb_off[s], D.bposF.p + D.wb_off[s], D.bglob.p + D.wb_off[s],
                    D.bslot.p + D.wb_off[s], D.WB.p + D.wb_off[s], D.nB[s], D.PB[s], D.NF[s], D.PE[s], D.NA[s],
                    D.nE[s]};
    fd[q] = FrontDesc{D.F.p + D.f_off[s], D.DinvF.p + D.df_off[s], D.NA[s], D.PE[s], D.finfo.p + q,
                      D.leaf_explicit ? D.NF[s] : 0, D.leaf_explicit ? 0 : D.nE[s], D.leaf_explicit ? 0 : D.nC[s]};
    fw[q] = SolveDesc{D.F.p + D.f_off[s], D.DinvF.p + D.df_off[s], D.FV.p + D.fv_off[s], D.NF[s], D.PE[s],
                      nullptr, nullptr, D.nE[s], D.nC[s]};
  }
  auto up_v = [&](auto& b, const auto& v) { UB.add(b, v); };
  up_v(D.subdesc, sd);
  up_v(D.ffront, fd);
  up_v(D.fsolve_fwd, fw);
  // primal tree levels (deepest first): fronts, vectors, gathers, backward maps
  D.tree_apply_bytes = D.tree_factor_bytes = 0;
  for (std::size_t l = 0; l < plan.levels.size(); ++l) {
    DeviceState::TreeLevel& T = *D.tree[l];
    const CoarseTree::Level& P = plan.levels[l];
    T.nfr = static_cast<int>(P.fronts.size());
    T.max_NF = P.max_NF;
    T.max_PE = P.max_PE;
    T.max_M = P.max_M;
    T.arena = P.arena;
    T.V.alloc(std::max<long long>(P.arena, 1));
    if (T.expl) T.V2.alloc(std::max<long long>(P.arena, 1));
    T.info.alloc(T.nfr);
    T.info.zero(st);
    T.NF.assign(T.nfr, 0);
    T.PE.assign(T.nfr, 0);
    T.nown.assign(T.nfr, 0);
    T.nupd.assign(T.nfr, 0);
    T.max_slots = 0;
    for (int f = 0; f < T.nfr; ++f) {
      const CoarseTree::Front& F = P.fronts[f];
      T.NF[f] = F.NF;
      T.PE[f] = F.PE;
      T.nown[f] = static_cast<int>(F.own.size());
      T.nupd[f] = static_cast<int>(F.upd.size());
      T.max_slots = std::max(T.max_slots, T.nown[f] + T.nupd[f]);
      const double e = T.nown[f], c = T.nupd[f];
      // explicit: E (e x (e + c)) forward, W (e x c) backward; else L twice
      D.tree_apply_bytes += (T.expl ? e * (e + c) + e * c : 2.0 * (e * (e + 1) / 2 + e * c)) * 8.0;
      D.tree_factor_bytes += (T.expl ? e * e + e * c : e * (e + 1) / 2 + e * c) * 8.0;
    }
  }
  // Larger roots are factored in place and solved by triangular sweeps (over
  // the whole GPU for the largest ones).
  const long ldR = D.root_inv ? 2L * D.NR : D.NR;
  D.xroot.alloc(D.NR);
  D.xroot2.alloc(D.NR);
  D.rinfo.alloc(1);
  D.rinfo.zero(st);
  double* const top_x = D.root_inv ? D.xroot2.p : D.xroot.p;  // the root's solution
  for (std::size_t l = 0; l < plan.levels.size(); ++l) {
    DeviceState::TreeLevel& T = *D.tree[l];
    const CoarseTree::Level& P = plan.levels[l];
    double* const up = l + 1 < plan.levels.size() ? D.tree[l + 1]->V.p : top_x;
    std::vector<FrontDesc> fdl(T.nfr);
    std::vector<SolveDesc> fwl(T.nfr), bwl(T.nfr);
    std::vector<AsmFront> afl(T.nfr);
    std::vector<LeafX> lxl;
    for (int f = 0; f < T.nfr; ++f) {
      const CoarseTree::Front& F = P.fronts[f];
      const int NA = T.expl ? F.NF + F.PE : F.NF;
      double* a = T.A.p + T.xa_off[f];
      fdl[f] = FrontDesc{a, T.Dinv.p + F.d_off, NA, F.PE, T.info.p + f, T.expl ? F.NF : 0};
      fwl[f] = SolveDesc{a, T.Dinv.p + F.d_off, T.V.p + F.fv_off, F.NF, F.PE, nullptr, nullptr,
                         static_cast<int>(F.own.size()), static_cast<int>(F.upd.size())};
      bwl[f] = fwl[f];
      bwl[f].cmap = T.cmap.p + F.cmap_off;
      bwl[f].croot = up;
      afl[f] = AsmFront{a, NA, T.nown[f], T.nupd[f], F.PE, F.NF, F.fv_off};
      if (T.expl)
        lxl.push_back(LeafX{a, T.E.p + T.xe_off[f], T.V.p + F.fv_off, T.V2.p + F.fv_off, T.cmap.p + F.cmap_off, NA,
                            F.PE, F.NF - F.PE});
    }
    up_v(T.fronts, fdl);
    up_v(T.fwd, fwl);
    up_v(T.bwd, bwl);
    up_v(T.afronts, afl);
    if (T.expl) up_v(T.lx, lxl);
    std::vector<AsmChild> kids;
    if (l == 0) {
      for (int q = 0; q < no; ++q) {
        const int s = D.own[q];
        kids.push_back(AsmChild{D.F.p + D.f_off[s], D.NA[s], D.PE[s]});
      }
    } else {
      const DeviceState::TreeLevel& C = *D.tree[l - 1];
      for (std::size_t f = 0; f < plan.levels[l - 1].fronts.size(); ++f) {
        const CoarseTree::Front& F = plan.levels[l - 1].fronts[f];
        kids.push_back(AsmChild{C.A.p + C.xa_off[f], C.expl ? F.NF + F.PE : F.NF, F.PE});
      }
    }
    up_v(T.kids, kids);
  }
  {
    std::vector<AsmChild> kids;
    if (plan.levels.empty()) {
      for (int q = 0; q < no; ++q) {
        const int s = D.own[q];
        kids.push_back(AsmChild{D.F.p + D.f_off[s], D.NA[s], D.PE[s]});
      }
    } else {
      const DeviceState::TreeLevel& C = *D.tree.back();
      for (std::size_t f = 0; f < plan.levels.back().fronts.size(); ++f) {
        const CoarseTree::Front& F = plan.levels.back().fronts[f];
        kids.push_back(AsmChild{C.A.p + C.xa_off[f], C.expl ? F.NF + F.PE : F.NF, F.PE});
      }
    }
    up_v(D.root_kids, kids);
    std::vector<AsmFront> af{AsmFront{D.R.p, ldR, D.n_root, 0, D.NR, D.NR, 0}};
    up_v(D.root_afront, af);
  }
  D.leaf_croot = plan.levels.empty() ? top_x : D.tree[0]->V.p;
  for (int q = 0; q < no; ++q) {
    bw[q] = fw[q];
    bw[q].cmap = D.cmap.p + cmap_off[D.own[q]];
    bw[q].croot = D.leaf_croot;
  }
  up_v(D.fsolve_bwd, bw);
  if (D.leaf_explicit) {
    std::vector<LeafX> lx(no);
    for (int q = 0; q < no; ++q) {
      const int s = D.own[q];
      lx[q] = LeafX{D.F.p + D.f_off[s], D.E.p + e_off[s], D.FV.p + D.fv_off[s], D.FV2.p + D.fv_off[s],
                    D.cmap.p + cmap_off[s], D.NA[s], D.PE[s], D.NF[s] - D.PE[s]};
    }
    up_v(D.leafx, lx);
  }
  {
    std::vector<FrontDesc> rf{
        FrontDesc{D.R.p, D.DinvR.p, static_cast<int>(ldR), D.NR, D.rinfo.p, D.root_inv ? D.NR : 0}};
    up_v(D.rfront, rf);
    std::vector<TrailDesc> rt{TrailDesc{D.R.p, D.Rinv.p, static_cast<int>(ldR), D.NR}};
    up_v(D.rtrail, rt);
    std::vector<SolveDesc> rs{SolveDesc{D.R.p, D.DinvR.p, D.xroot.p, D.NR, D.NR, nullptr, nullptr}};
    up_v(D.rsolve, rs);
  }
  ht.mark("descriptors");
  UB.flush(st);
  ht.mark("upload_desc");
  // coarse stage of the apply as one launch (k_coarse_explicit) when every
  // level is explicit and the root inverse is small; BDDC_B200_COARSE=split keeps
  // the separate launches (parity-tested both ways)
  {
    const char* env = std::getenv("BDDC_B200_COARSE");
    bool ok = !(env && std::string(env) == "split") && !D.comm && D.root_inv && !D.tree.empty() &&
              D.tree.size() <= static_cast<std::size_t>(kCoarseLevels) && D.NR <= 4096;
    int words = D.NR;
    for (auto& T : D.tree) {
      ok = ok && T->expl && T->max_NF <= 4096;
      words = std::max(words, std::max(T->max_PE, T->max_M));
    }
    D.coarse_fused = ok;
    if (ok) {
      CoarseArgs& A = D.coarse_args;
      A = CoarseArgs{};
      A.nlev = static_cast<int>(D.tree.size());
      long units = (D.NR + 7) / 8;
      const double* fvsrc = D.leaf_explicit ? D.FV2.p : D.FV.p;
      for (int l = 0; l < A.nlev; ++l) {
        DeviceState::TreeLevel& T = *D.tree[l];
        CoarseLevelArgs& L = A.lv[l];
        L.lx = T.lx.p;
        L.ptr = T.ptr.p;
        L.src = T.src.p;
        L.vbase = T.V.p;
        L.fvsrc = fvsrc;
        L.up = l + 1 < A.nlev ? D.tree[l + 1]->V.p : top_x;
        L.nfr = T.nfr;
        L.ncb = (T.max_NF + 7) / 8;
        L.nrb = T.max_NF / kTile;
        units = std::max(units, (long)L.nfr * L.ncb);
        fvsrc = T.V2.p;
      }
      A.n_root = D.n_root;
      A.NR = D.NR;
      A.root_ptr = D.root_ptr.p;
      A.root_src = D.root_src.p;
      A.root_fvsrc = fvsrc;
      A.Rinv = D.Rinv.p;
      A.xroot = top_x;
      if (D.coarse_bar.n == 0) {
        D.coarse_bar.alloc(2);
        D.coarse_bar.zero(st);
      }
      A.bar = D.coarse_bar.p;
      D.coarse_smem = words * static_cast<int>(sizeof(double));
      const int per_sm = per_device(reinterpret_cast<const void*>(&k_coarse_explicit), [] {
        int n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_coarse_explicit, 256, 4096 * sizeof(double));
        return std::max(1, std::min(n, 3));
      });
      D.coarse_grid = static_cast<int>(std::min<long>(units, (long)per_sm * sm_count()));
    }
  }
  StageProfiler prof("set_constraints", st);
  // F = P (T^T S T) P^T, pads identity
  if (!D.leaf_explicit) {
    if (no) {
      CK(static_cast<cudaError_t>(per_device(reinterpret_cast<const void*>(&k_xform_fused), [] {
        return static_cast<int>(
            cudaFuncSetAttribute(k_xform_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      })));
      k_xform_fused<<<dim3((D.max_PB + 2 * kTile + kXformCols - 1) / kXformCols, no), 256,
                      kXformCols * D.max_nB * sizeof(double), st>>>(D.subdesc.p, D.xf);
      count_launch(1);
    }
  } else {
    D.F.zero(st);
    if (no) {
      k_colxform<<<dim3(D.max_PB, no), 128, 0, st>>>(D.subdesc.p, D.xf, D.Xtmp.p, D.d_xoff.p);
      k_rowxform_scatter<<<dim3(D.max_PB, no), 128, 0, st>>>(D.subdesc.p, D.xf, D.Xtmp.p, D.d_xoff.p);
    }
    if (!pads.empty())
      k_pad_identity<<<std::min<int>(1024, (static_cast<int>(pads.size()) + 255) / 256), 256, 0, st>>>(
          D.F.p, D.d_foff.p, D.d_NF.p, D.pad_sub.p, D.pads.p, static_cast<int>(pads.size()));
    count_launch(3);
  }
  if (D.leaf_explicit && no) {
    k_aug_identity<<<dim3((D.max_PE + 255) / 256, no), 256, 0, st>>>(D.leafx.p);
    count_launch(1);
  }
  CK(cudaGetLastError());
  prof.mark("xform");
  partial_cholesky(D.ffront.p, no, D.max_NA, D.max_PE, D.max_MA, st);
  if (D.leaf_explicit && no) {
    k_leaf_explicit_copy<<<dim3(256, no), 256, 0, st>>>(D.leafx.p);
    count_launch(1);
  }
  CK(cudaGetLastError());
  prof.mark(D.leaf_explicit ? "cholF+explicit" : "cholF");
  // primal tree, deepest level first: extend-add of the children's Schur
  // complements, identity pads, batched partial Cholesky
  for (std::size_t l = 0; l < D.tree.size(); ++l) {
    DeviceState::TreeLevel& T = *D.tree[l];
    T.A.zero(st);
    const long pairs = (long)T.max_slots * (T.max_slots + 1) / 2;
    k_front_assemble<<<dim3(static_cast<unsigned>(std::min<long>(1024, (pairs + 255) / 256)), T.nfr), 256, 0, st>>>(
        T.afronts.p, T.ptr.p, T.child.p, T.cidx.p, T.kids.p);
    k_front_pads<<<dim3(std::max(1, std::min(64, (T.max_NF + 255) / 256)), T.nfr), 256, 0, st>>>(T.afronts.p);
    count_launch(2);
    partial_cholesky(T.fronts.p, T.nfr, T.max_NA, T.max_PE, T.max_MA, st);
    if (T.expl) {
      k_leaf_explicit_copy<<<dim3(64, T.nfr), 256, 0, st>>>(T.lx.p);
      count_launch(1);
    }
  }
  if (!D.tree.empty()) prof.mark("tree");
  // this rank's contributions (+ the identity blocks on rank 0), then the
  // gather of the root front: an allreduce of its first N_R columns
  const bool identity = !D.comm || D.comm->rank() == 0;
  D.R.zero(st);
  {
    const long pairs = (long)D.n_root * (D.n_root + 1) / 2;
    k_front_assemble<<<static_cast<unsigned>(std::max<long>(1, std::min<long>(1024, (pairs + 255) / 256))), 256, 0,
                       st>>>(D.root_afront.p, D.root_ptr.p, D.root_child.p, D.root_c.p, D.root_kids.p);
    count_launch(1);
    if (identity) {
      k_front_pads<<<std::max(1, std::min(1024, (D.NR + 255) / 256)), 256, 0, st>>>(D.root_afront.p);
      count_launch(1);
    }
  }
  if (D.comm) D.comm->allreduce(D.R.p, (size_t)ldR * D.NR, st);
  prof.mark("root_asm");
  partial_cholesky(D.rfront.p, 1, static_cast<int>(ldR), D.NR, D.root_inv ? D.NR : 0, st);
  if (D.root_inv) {
    copy_trailing_full(D.rtrail.p, 1, D.NR, st);
  }
  prof.mark(D.root_inv ? "cholR+inverse" : "cholR");
  CK(cudaGetLastError());
  CK(cudaEventRecord(D.e1, st));
  times_.preconditioner = elapsed(D.e0, D.e1);
  std::vector<int> info(std::max(no, 1));
  CK(cudaMemcpy(info.data(), D.finfo.p, info.size() * sizeof(int), cudaMemcpyDeviceToHost));
  for (int q = 0; q < no; ++q)
    if (info[q]) throw Error(kNotPositiveDefinite, "factorize: transformed leaf front " + std::to_string(D.own[q]) +
                                                       " is not positive definite");
  int rinfo = 0;
  CK(cudaMemcpy(&rinfo, D.rinfo.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (rinfo) throw Error(kNotPositiveDefinite, "factorize: root front is not positive definite");
  for (auto& T : D.tree) {
    std::vector<int> ti(T->nfr);
    CK(cudaMemcpy(ti.data(), T->info.p, ti.size() * sizeof(int), cudaMemcpyDeviceToHost));
    for (int v : ti)
      if (v) throw Error(kNotPositiveDefinite, "factorize: primal tree front is not positive definite");
  }
  D.have_prec = true;
  D.h_cov = cov;
  // invalidate a captured PCG graph (pointers changed)
  if (D.gexec) {
    cudaGraphExecDestroy(D.gexec);
    D.gexec = nullptr;
  }
  if (D.graph) {
    cudaGraphDestroy(D.graph);
    D.graph = nullptr;
  }
}

// ---------------------------------------------------------------------------
// operator applications
// ---------------------------------------------------------------------------
namespace {
// Sharded: this rank's copies are summed, then the interface neighbour
// exchange (halo send/recv) completes every dof this rank touches, and the dot
// product is taken over the dofs it owns (partials all-reduced).
void finish_interface(DeviceState& D, double* y, const double* dot_with, double* partials, const int* done) {
  cudaStream_t st = D.st;
  if (!D.comm) return;
  halo_exchange(D, y);
  if (partials) {  // owned dofs only, then the kRed partials summed over the ranks
    k_dot<<<kRed, 256, 0, st>>>(D.niface, dot_with, y, partials, D.halo.owned.p);
    count_launch(1);
    D.comm->allreduce(partials, kRed, st);
  }
  (void)done;
}

// stages: kPreRestrict (restrict_residual), kPreSolve (coarse_solve on the leaf
// vectors), kPreProlong (prolong + copy sum); the PCG runs all three
enum : int { kPreRestrict = 1, kPreSolve = 2, kPreProlong = 4, kPreAll = 7 };
void launch_precond(DeviceState& D, const double* r, double* z, const double* dot_with, double* partials,
                    const int* done, StageProfiler* prof = nullptr, int stages = kPreAll) {
  cudaStream_t st = D.st;
  const int ns = D.n_own;
  const int smem_b = D.max_nB * sizeof(double);
  auto mark = [&](const char* s) {
    if (prof) prof->mark(s);
  };
  const int nw = D.nw;
  const int pos_blocks = std::max(1, std::min(8 * sm_count(), (nw + 255) / 256));  // one position per thread when resident
  if (ns && (stages & kPreRestrict)) k_restrict_pos<<<pos_blocks, 256, 0, st>>>(D.subdesc.p, D.xf, D.wpos.p, nw, r, done);
  count_launch(3);  // restrict, prolong, copy sum
  mark("restrict");
  if (stages & kPreSolve) {
  if (D.leaf_explicit && ns) {
    k_leaf_fwd_explicit<<<dim3((D.max_NF + 7) / 8, ns), 256, D.max_PE * sizeof(double), st>>>(D.leafx.p, done);
    count_launch(1);
  } else if (!D.leaf_explicit) {
    front_forward(D.fsolve_fwd.p, ns, D.max_NF, st, done);
  }
  mark("leaf_fwd");
  const double* fvsrc = D.leaf_explicit ? D.FV2.p : D.FV.p;
  if (D.coarse_fused) {
    k_coarse_explicit<<<D.coarse_grid, 256, D.coarse_smem, st>>>(D.coarse_args, done);
    count_launch(1);
    mark("root_coarse");
  } else {
  // primal tree, deepest level first: gather the children's coarse residuals,
  // forward sweep
  for (auto& T : D.tree) {
    k_root_gather<<<std::max(1, std::min<int>(1024, static_cast<int>((T->arena + 255) / 256))), 256, 0, st>>>(
        static_cast<int>(T->arena), static_cast<int>(T->arena), T->ptr.p, T->src.p, fvsrc, T->V.p, done);
    count_launch(1);
    if (T->expl) {
      k_leaf_fwd_explicit<<<dim3((T->max_NF + 7) / 8, T->nfr), 256, T->max_PE * sizeof(double), st>>>(T->lx.p, done);
      count_launch(1);
      fvsrc = T->V2.p;
    } else {
      front_forward(T->fwd.p, T->nfr, T->max_NF, st, done);
      fvsrc = T->V.p;
    }
  }
  if (!D.tree.empty()) mark("tree_fwd");
  if (D.root_inv && !D.comm && D.NR <= 1024) {
    // small root, one GPU: gather and apply in one launch
    k_root_gather_gemv<<<(D.NR + 7) / 8, 256, D.NR * sizeof(double), st>>>(D.n_root, D.NR, D.root_ptr.p,
                                                                         D.root_src.p, fvsrc, D.Rinv.p,
                                                                         D.xroot2.p, done);
    count_launch(1);
    mark("root_gemv");
  } else {
  k_root_gather<<<std::max(1, std::min(1024, (D.NR + 255) / 256)), 256, 0, st>>>(
      D.n_root, D.NR, D.root_ptr.p, D.root_src.p, fvsrc, D.xroot.p, done);
  count_launch(1);
  if (D.comm) D.comm->allreduce(D.xroot.p, D.NR, st);  // root right-hand side of every rank
  mark("root_gather");
  if (D.root_inv) {
    k_root_gemv<<<std::min(1184, (D.NR + 7) / 8), 256, 0, st>>>(D.NR, D.Rinv.p, D.xroot.p, D.xroot2.p, done);
    count_launch(1);
    mark("root_gemv");
  } else {
    front_forward(D.rsolve.p, 1, D.NR, st, done);
    mark("root_fwd");
    front_backward(D.rsolve.p, 1, D.NR, st, done);
    mark("root_bwd");
  }
  }
  for (std::size_t l = D.tree.size(); l-- > 0;) {
    DeviceState::TreeLevel& T = *D.tree[l];
    if (T.expl) {
      double* up = l + 1 < D.tree.size() ? D.tree[l + 1]->V.p : (D.root_inv ? D.xroot2.p : D.xroot.p);
      k_leaf_bwd_explicit<<<dim3(T.max_NF / kTile, T.nfr), 256, std::max(T.max_M, 1) * sizeof(double), st>>>(T.lx.p, up,
                                                                                                          done);
      count_launch(1);
    } else {
      front_backward(T.bwd.p, T.nfr, T.max_NF, st, done);
    }
  }
  if (!D.tree.empty()) mark("tree_bwd");
  }  // separate coarse launches
  if (D.leaf_explicit && ns) {
    k_leaf_bwd_explicit<<<dim3(D.max_NF / kTile, ns), 256, D.max_M * sizeof(double), st>>>(D.leafx.p, D.leaf_croot,
                                                                                          done);
    count_launch(1);
  } else if (!D.leaf_explicit) {
    front_backward(D.fsolve_bwd.p, ns, D.max_NF, st, done);
  }
  mark("leaf_bwd");
  }  // kPreSolve
  if (!(stages & kPreProlong)) return;
  if (ns) {
    const int item_blocks = D.nitems ? std::max(1, std::min(4 * sm_count(), (D.nitems + 7) / 8)) : 0;
    k_prolong_fused<<<pos_blocks + item_blocks, 256, 0, st>>>(D.subdesc.p, D.xf, D.wpos.p, D.wsrc.p, nw, pos_blocks,
                                                             D.item_sub.p, D.item_e.p, D.nitems, D.FV.p, done);
  }
  mark("prolong");
  k_sum_copies<<<kRed, 256, 0, st>>>(D.niface, D.icopy_ptr.p, D.icopy_pos.p, D.WB.p, z, D.comm ? nullptr : dot_with,
                                     D.comm ? nullptr : partials, done);
  finish_interface(D, z, dot_with, partials, done);
  mark("sum_copies");
}

void launch_schur(DeviceState& D, const double* x, double* y, const double* dot_with, double* partials,
                  const int* done) {
  cudaStream_t st = D.st;
  if (D.n_own)
    k_schur_gemv_rows<<<dim3((D.max_nB + 63) / 64, D.n_own), 256, D.max_nB * sizeof(double), st>>>(D.subdesc.p, x,
                                                                                                  done);
  count_launch(2);
  k_sum_copies<<<kRed, 256, 0, st>>>(D.niface, D.icopy_ptr.p, D.icopy_pos.p, D.WB.p, y, D.comm ? nullptr : dot_with,
                                     D.comm ? nullptr : partials, done);
  finish_interface(D, y, dot_with, partials, done);
}

void ensure_vectors(DeviceState& D) {
  const i64 n = std::max<i64>(D.niface, 1);
  if (D.vx.n == std::size_t(n)) return;
  D.vx.alloc(n);
  D.vr.alloc(n);
  D.vz.alloc(n);
  D.vp.alloc(n);
  D.vq.alloc(n);
  D.vb.alloc(n);
  D.part_a.alloc(kRed);
  D.part_b.alloc(kRed);
  D.pst.alloc(1);
}
}  // namespace

void Engine::leaf_front(int s, std::vector<double>* out, std::vector<int>* pos, int* ld) {
  prepare();
  DeviceState& D = *d_;
  *ld = D.NM[s];
  const Subdomain& S = m_.subs[s];
  if (!D.is_own[s]) throw Error(kError, "substructure not owned by this shard");
  std::size_t off = 0;
  for (int q : D.own) {
    if (q == s) break;
    off += m_.subs[q].dim();
  }
  pos->assign(D.h.pos.begin() + off, D.h.pos.begin() + off + S.dim());
  if (!out) return;
  cudaStream_t st = D.st;
  assemble_fronts(D);
  k_mirror_upper<<<256, 256, 0, st>>>(D.M.p + D.m_off[s], D.NM[s]);
  count_launch(1);
  CK(cudaGetLastError());
  out->resize((size_t)D.NM[s] * D.NM[s]);
  CK(cudaMemcpyAsync(out->data(), D.M.p + D.m_off[s], out->size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

void Engine::schur_apply(const double* x, double* y) {
  NvtxRange nvtx("bddc:schur_apply");
  DeviceState& D = *d_;
  ensure_vectors(D);
  const std::size_t bytes = D.niface * sizeof(double);
  CK(cudaMemcpyAsync(D.vp.p, x, bytes, cudaMemcpyHostToDevice, D.st));
  launch_schur(D, D.vp.p, D.vq.p, nullptr, nullptr, nullptr);
  complete_interface(D, D.vq.p);
  CK(cudaMemcpyAsync(y, D.vq.p, bytes, cudaMemcpyDeviceToHost, D.st));
  CK(cudaStreamSynchronize(D.st));
  CK(cudaGetLastError());
}

void Engine::precond_apply(const double* r, double* z) {
  NvtxRange nvtx("bddc:precond_apply");
  DeviceState& D = *d_;
  if (!D.have_prec) throw Error(kError, "preconditioner not set up");
  ensure_vectors(D);
  const std::size_t bytes = D.niface * sizeof(double);
  CK(cudaMemcpyAsync(D.vr.p, r, bytes, cudaMemcpyHostToDevice, D.st));
  launch_precond(D, D.vr.p, D.vz.p, nullptr, nullptr, nullptr);
  complete_interface(D, D.vz.p);
  CK(cudaMemcpyAsync(z, D.vz.p, bytes, cudaMemcpyDeviceToHost, D.st));
  CK(cudaStreamSynchronize(D.st));
  CK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// BddcPreconditioner::{restrict_residual, coarse_solve, prolong} on W^c vectors
// (bddc_operator.cpp:52-99; bddc_operator.hpp:40-48).  The stages of the
// preconditioner apply run on the device exactly as inside precond_apply; the
// host maps between W^c (maps.local_to_wc) and the device layouts: boundary
// dof b of substructure s in transformed variables lives at leaf-vector
// position fv_off[s] + posF[b] (explicit dof k = glob slot k, as
// transform.cpp:94-149), interior dof r at MV position mv_off[s] + r.  Not a
// hot path: the PCG uses the fused apply.
// ---------------------------------------------------------------------------
namespace {
void require_wc(const DeviceState& D) {
  if (!D.have_prec) throw Error(kError, "preconditioner not set up");
  if (D.comm) throw Error(kUnsupported, "W^c entry points are single-GPU (the sharded engine exchanges interface vectors)");
}

/// Means over the equality groups (GroupProjector::apply, transform.cpp:12-46).
void project_groups(const ChangeOfVariables& cov, std::vector<double>& wc) {
  for (const auto& g : cov.groups) {
    double sum = 0.0;
    for (i64 id : g) sum += wc[id];
    const double mean = sum / static_cast<double>(g.size());
    for (i64 id : g) wc[id] = mean;
  }
}

/// y = T_s x (transpose = false) or T_s^T x on the boundary values of
/// substructure s, given per local dof (ChangeOfVariables::basis, transform.cpp:94-149).
void apply_transforms(const Model& m, const ChangeOfVariables& cov, int s, std::vector<double>& local, bool transpose) {
  for (const GlobTransform& gt : cov.transforms) {
    const auto& subs = m.globs[gt.glob].subdomains;
    if (!std::binary_search(subs.begin(), subs.end(), s)) continue;
    const std::vector<double> t = gt.dense_t();
    const auto& dofs = m.glob_dofs[gt.glob];
    const int n = gt.n;
    std::vector<int> loc(n);
    std::vector<double> x(n), y(n, 0.0);
    for (int a = 0; a < n; ++a) {
      loc[a] = m.maps.local_of(dofs[a], s);
      x[a] = local[loc[a]];
    }
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b) {
        if (transpose)
          y[b] += t[std::size_t(a) * n + b] * x[a];
        else
          y[a] += t[std::size_t(a) * n + b] * x[b];
      }
    for (int a = 0; a < n; ++a) local[loc[a]] = y[a];
  }
}
}  // namespace

void Engine::restrict_residual(const double* r, double* wc_out) {
  DeviceState& D = *d_;
  require_wc(D);
  ensure_vectors(D);
  const Model& m = m_;
  CK(cudaMemcpyAsync(D.vr.p, r, D.niface * sizeof(double), cudaMemcpyHostToDevice, D.st));
  CK(cudaMemsetAsync(D.FV.p, 0, D.FV.n * sizeof(double), D.st));
  launch_precond(D, D.vr.p, D.vz.p, nullptr, nullptr, nullptr, nullptr, kPreRestrict);
  std::vector<double> fv(D.FV.n);
  CK(cudaMemcpyAsync(fv.data(), D.FV.p, fv.size() * sizeof(double), cudaMemcpyDeviceToHost, D.st));
  CK(cudaStreamSynchronize(D.st));
  std::vector<double> wc(m.maps.wc_dim, 0.0);
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    for (int b = 0; b < D.nB[s]; ++b)  // scatter-add: corners are summed over their substructures
      wc[m.maps.local_to_wc[s][S.boundary[b]]] += fv[D.fv_off[s] + D.h_posF[D.wb_off[s] + b]];
  }
  project_groups(D.h_cov, wc);
  std::copy(wc.begin(), wc.end(), wc_out);
}

void Engine::coarse_solve(const double* wc_in, double* wc_out) {
  DeviceState& D = *d_;
  require_wc(D);
  ensure_vectors(D);
  const Model& m = m_;
  cudaStream_t st = D.st;
  std::vector<double> rhs(wc_in, wc_in + m.maps.wc_dim);
  project_groups(D.h_cov, rhs);
  // local transformed residuals: a W^c entry shared by several substructures
  // (corners) goes to its first holder, so that summing the copies gives R^T rhs
  std::vector<char> taken(m.maps.wc_dim, 0);
  std::vector<std::vector<double>> loc(D.nsub);
  std::vector<double> mv(D.MV.n, 0.0);
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    loc[s].assign(S.dim(), 0.0);
    for (int l = 0; l < S.dim(); ++l) {
      const i64 id = m.maps.local_to_wc[s][l];
      if (!taken[id]) loc[s][l] = rhs[id];
      taken[id] = 1;
    }
    for (int r = 0; r < D.nI[s]; ++r) mv[D.mv_off[s] + r] = loc[s][S.interior[r]];
  }
  // interiors eliminated exactly: y_I = L^{-1} r_I, g_B = -A_BI A_II^{-1} r_I
  CK(cudaMemcpyAsync(D.MV.p, mv.data(), mv.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  front_forward(D.msolve.p, D.n_own, D.max_NM, st);
  CK(cudaMemcpyAsync(mv.data(), D.MV.p, mv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<double> fv(D.FV.n, 0.0);
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    std::vector<double> g(S.dim(), 0.0);
    for (int b = 0; b < D.nB[s]; ++b) g[S.boundary[b]] = mv[D.mv_off[s] + D.PI[s] + b];
    apply_transforms(m, D.h_cov, s, g, true);  // T_s^T g_B
    for (int b = 0; b < D.nB[s]; ++b)
      fv[D.fv_off[s] + D.h_posF[D.wb_off[s] + b]] = loc[s][S.boundary[b]] + g[S.boundary[b]];
  }
  CK(cudaMemcpyAsync(D.FV.p, fv.data(), fv.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  launch_precond(D, D.vr.p, D.vz.p, nullptr, nullptr, nullptr, nullptr, kPreSolve);
  CK(cudaMemcpyAsync(fv.data(), D.FV.p, fv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // x_B = T_s x~_B into the boundary part of MV, then x_I = L^{-T}(y_I - L_BI^T x_B)
  std::vector<double> wc(m.maps.wc_dim, 0.0);
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    std::vector<double> x(S.dim(), 0.0);
    for (int b = 0; b < D.nB[s]; ++b) {
      const double v = fv[D.fv_off[s] + D.h_posF[D.wb_off[s] + b]];
      x[S.boundary[b]] = v;
      wc[m.maps.local_to_wc[s][S.boundary[b]]] = v;
    }
    apply_transforms(m, D.h_cov, s, x, false);
    for (int b = 0; b < D.nB[s]; ++b) mv[D.mv_off[s] + D.PI[s] + b] = x[S.boundary[b]];
  }
  CK(cudaMemcpyAsync(D.MV.p, mv.data(), mv.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  front_backward(D.msolve.p, D.n_own, D.max_NM, st);
  CK(cudaMemcpyAsync(mv.data(), D.MV.p, mv.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    for (int r = 0; r < D.nI[s]; ++r) wc[m.maps.local_to_wc[s][S.interior[r]]] = mv[D.mv_off[s] + r];
  }
  std::copy(wc.begin(), wc.end(), wc_out);
}

void Engine::prolong(const double* wc, double* z) {
  DeviceState& D = *d_;
  require_wc(D);
  ensure_vectors(D);
  const Model& m = m_;
  std::vector<double> fv(D.FV.n, 0.0);
  for (int s : D.own) {
    const Subdomain& S = m.subs[s];
    for (int b = 0; b < D.nB[s]; ++b)
      fv[D.fv_off[s] + D.h_posF[D.wb_off[s] + b]] = wc[m.maps.local_to_wc[s][S.boundary[b]]];
  }
  CK(cudaMemcpyAsync(D.FV.p, fv.data(), fv.size() * sizeof(double), cudaMemcpyHostToDevice, D.st));
  launch_precond(D, D.vr.p, D.vz.p, nullptr, nullptr, nullptr, nullptr, kPreProlong);
  CK(cudaMemcpyAsync(z, D.vz.p, D.niface * sizeof(double), cudaMemcpyDeviceToHost, D.st));
  CK(cudaStreamSynchronize(D.st));
  CK(cudaGetLastError());
}

Engine::OpTimes Engine::time_operators(int reps) {
  DeviceState& D = *d_;
  if (!D.have_prec) throw Error(kError, "preconditioner not set up");
  ensure_vectors(D);
  reps = std::max(reps, 1);
  OpTimes o;
  // deterministic nonzero inputs
  CK(cudaMemcpyAsync(D.vp.p, D.rhs.p, D.niface * sizeof(double), cudaMemcpyDeviceToDevice, D.st));
  CK(cudaMemcpyAsync(D.vr.p, D.rhs.p, D.niface * sizeof(double), cudaMemcpyDeviceToDevice, D.st));
  launch_schur(D, D.vp.p, D.vq.p, nullptr, nullptr, nullptr);  // warm
  launch_precond(D, D.vr.p, D.vz.p, nullptr, nullptr, nullptr);
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  CK(cudaEventRecord(e0, D.st));
  for (int r = 0; r < reps; ++r) launch_schur(D, D.vp.p, D.vq.p, nullptr, nullptr, nullptr);
  CK(cudaEventRecord(e1, D.st));
  for (int r = 0; r < reps; ++r) launch_precond(D, D.vr.p, D.vz.p, nullptr, nullptr, nullptr);
  CK(cudaEventRecord(e2, D.st));
  CK(cudaEventSynchronize(e2));
  o.schur = elapsed(e0, e1) / reps;
  o.precond = elapsed(e1, e2) / reps;
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
  CK(cudaEventDestroy(e2));
  std::vector<std::pair<std::string, double>> stages;
  for (int r = 0; r < reps; ++r) {
    StageProfiler prof("precond_apply", D.st, &stages);
    launch_precond(D, D.vr.p, D.vz.p, nullptr, nullptr, nullptr, &prof);
  }
  for (const auto& [name, sec] : stages) {
    const double v = sec / reps;
    if (name == "restrict") o.restrict_ += v;
    else if (name == "leaf_fwd") o.leaf_fwd += v;
    else if (name == "tree_fwd") o.tree_fwd += v;
    else if (name.rfind("root", 0) == 0) o.root += v;
    else if (name == "tree_bwd") o.tree_bwd += v;
    else if (name == "leaf_bwd") o.leaf_bwd += v;
    else if (name == "prolong") o.prolong += v;
    else if (name == "sum_copies") o.sum_copies += v;
  }
  if (D.NF.size() == std::size_t(D.nsub))
    for (int s : D.own) {
      const double e = D.nE[s], c = D.nC[s];
      o.leaf_sweep_bytes += (D.leaf_explicit ? e * (e + c) : e * (e + 1) / 2 + e * c) * 8.0;
    }
  CK(cudaGetLastError());
  return o;
}

void Engine::rhs(double* out) {
  DeviceState& D = *d_;
  complete_interface(D, D.rhs.p);  // sharded: every dof (still valid for pcg)
  CK(cudaMemcpyAsync(out, D.rhs.p, D.niface * sizeof(double), cudaMemcpyDeviceToHost, D.st));
  CK(cudaStreamSynchronize(D.st));
}

// InterfaceProblem::recover (schur.cpp:57-75): x_I = A_II^{-1}(f_I - A_IB x_B),
// as the forward sweep of the loads followed by the backward sweep with x_B.
void Engine::recover_device(const double* d_uiface, double* d_ufree) {
  DeviceState& D = *d_;
  const Model& m = m_;
  cudaStream_t st = D.st;
  // sharded: interiors of the owned substructures; the interface values from
  // rank 0; the rest zero, summed over ranks
  const bool iface_here = !D.comm || D.comm->rank() == 0;
  if (D.sol_gdof.n == 0) {
    std::vector<long long> g(D.MV.n, -1), ig(m.maps.interface_dofs.begin(), m.maps.interface_dofs.end());
    for (int s : D.own) {
      const Subdomain& S = m.subs[s];
      for (int r = 0; r < D.nI[s]; ++r) g[D.mv_off[s] + r] = S.global_dof[S.interior[r]];
    }
    D.sol_gdof.upload(g, st);
    if (ig.empty()) ig.push_back(0);
    D.iface_gdof.upload(ig, st);
  }
  if (D.comm) CK(cudaMemsetAsync(d_ufree, 0, m.free_count * sizeof(double), st));
  CK(cudaMemcpyAsync(D.MV.p, D.MV0.p, D.MV.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  front_forward(D.msolve.p, D.n_own, D.max_NM, st);
  if (D.n_own) k_insert_boundary<<<D.n_own, 256, 0, st>>>(D.subdesc.p, D.MV.p, D.d_mvoff.p, D.d_PI.p, d_uiface);
  front_backward(D.msolve.p, D.n_own, D.max_NM, st);
  k_scatter_solution<<<256, 256, 0, st>>>(static_cast<long long>(D.MV.n), D.sol_gdof.p, D.MV.p,
                                          iface_here ? D.niface : 0, D.iface_gdof.p, d_uiface, d_ufree);
  count_launch(2);
  CK(cudaGetLastError());
  if (D.comm) D.comm->allreduce(d_ufree, m.free_count, st);
}

void Engine::recover(const double* u_interface, double* u_free) {
  DeviceState& D = *d_;
  ensure_vectors(D);
  DBuf<double> uf;
  uf.alloc(std::max<i64>(m_.free_count, 1));
  CK(cudaMemcpyAsync(D.vx.p, u_interface, D.niface * sizeof(double), cudaMemcpyHostToDevice, D.st));
  recover_device(D.vx.p, uf.p);
  CK(cudaMemcpyAsync(u_free, uf.p, m_.free_count * sizeof(double), cudaMemcpyDeviceToHost, D.st));
  CK(cudaStreamSynchronize(D.st));
}

namespace {
// The persistent PCG kernel covers the latency-bound layout: one GPU, explicit
// leaf operators, a small root inverse, no primal tree (BDDC_B200_PCG=graph
// keeps the per-iteration CUDA graph).
bool persistent_pcg(DeviceState& D) {
  if (D.comm || !D.leaf_explicit || !D.root_inv || D.NR > 1024 || !D.tree.empty() || D.n_own == 0) return false;
  if (const char* e = std::getenv("BDDC_B200_PCG"); e && std::string(e) == "graph") return false;
  const std::size_t words = std::max<std::size_t>({(std::size_t)D.max_nB + D.max_rows, (std::size_t)D.max_PE,
                                                   (std::size_t)D.NR, (std::size_t)D.max_M, 1});
  const std::size_t smem = words * sizeof(double);
  if (smem > 200 * 1024) return false;
  if (smem != D.pcg_smem || D.pcg_grid == 0) {  // occupancy queried once per shared-memory size
    CK(static_cast<cudaError_t>(per_device(reinterpret_cast<const void*>(&k_pcg_persistent), [] {
      return static_cast<int>(
          cudaFuncSetAttribute(k_pcg_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    })));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_persistent, 256, smem));
    D.pcg_smem = smem;
    const int cap = 3;  // CTAs per SM (measured: 3 beats 1, 2 and 4 on cfg1-2)
    D.pcg_grid = per_sm < 1 ? -1 : sm_count() * std::min(per_sm, cap);
  }
  return D.pcg_grid > 0;
}
}  // namespace

PcgOut Engine::pcg(const double* b, double* x, double tol, int max_it, bool precond_residual) {
  NvtxRange nvtx("bddc:pcg");
  DeviceState& D = *d_;
  if (!D.have_prec) throw Error(kError, "preconditioner not set up");
  ensure_vectors(D);
  cudaStream_t st = D.st;
  const i64 n = D.niface;
  const std::size_t bytes = n * sizeof(double);
  if (D.alphas.n < std::size_t(max_it + 1)) {
    D.alphas.alloc(max_it + 1);
    D.betas.alloc(max_it + 1);
  }
  CK(cudaEventRecord(D.e0, st));
  if (b)
    CK(cudaMemcpyAsync(D.vb.p, b, bytes, cudaMemcpyHostToDevice, st));
  else
    CK(cudaMemcpyAsync(D.vb.p, D.rhs.p, bytes, cudaMemcpyDeviceToDevice, st));
  // r = b, x = 0, z = M r, p = z, rz = r.z   (pcg.cpp:32-41)
  CK(cudaMemcpyAsync(D.vr.p, D.vb.p, bytes, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemsetAsync(D.vx.p, 0, bytes, st));
  {
    StageProfiler prof("precond_apply", st);
    launch_precond(D, D.vr.p, D.vz.p, D.vr.p, D.part_a.p, nullptr, &prof);
    if (prof.on()) {
      StageProfiler prof2("schur_apply", st);
      launch_schur(D, D.vz.p, D.vq.p, nullptr, nullptr, nullptr);
      prof2.mark("schur");
    }
  }
  CK(cudaMemcpyAsync(D.vp.p, D.vz.p, bytes, cudaMemcpyDeviceToDevice, st));
  k_dot<<<kRed, 256, 0, st>>>(n, D.vb.p, D.vb.p, D.part_b.p, D.comm ? D.halo.owned.p : nullptr);
  count_launch(1);
  if (D.comm) D.comm->allreduce(D.part_b.p, kRed, st);
  std::vector<double> pa(kRed), pb(kRed);
  CK(cudaMemcpyAsync(pa.data(), D.part_a.p, kRed * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(pb.data(), D.part_b.p, kRed * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // same fixed-order tree as sum_partials
  auto tree = [](std::vector<double> v) {
    for (int s = kRed / 2; s > 0; s >>= 1)
      for (int i = 0; i < s; ++i) v[i] += v[i + s];
    return v[0];
  };
  const double rz = tree(pa), bb = tree(pb);
  PcgState h{};
  h.rz = rz;
  h.bnorm = std::sqrt(bb);
  h.ref = precond_residual ? std::sqrt(std::max(rz, 0.0)) : h.bnorm;
  h.tol = tol;
  h.max_it = max_it;
  h.precond_residual = precond_residual ? 1 : 0;
  h.it = 0;
  h.relres = 1.0;
  h.done = (h.ref == 0.0 || h.relres <= tol || max_it <= 0) ? 1 : 0;
  PcgOut out;
  if (h.ref == 0.0) {  // zero right hand side
    out.relative_residual = 0.0;
    if (x) std::memset(x, 0, bytes);
    return out;
  }
  CK(cudaMemcpyAsync(D.pst.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  PcgState hs = h;
  if (D.comm) {
    // sharded: the iteration runs eagerly (its exchanges may synchronize the
    // host); every rank holds the same complete vectors and scalars, so the
    // iterations stay in lockstep
    while (!hs.done) {
      launch_schur(D, D.vp.p, D.vq.p, D.vp.p, D.part_a.p, nullptr);
      k_alpha_axpy<<<kRed, kRed, 0, st>>>(n, D.pst.p, D.vx.p, D.vr.p, D.vp.p, D.vq.p, D.part_a.p, D.part_b.p,
                                           D.alphas.p, D.halo.owned.p);
      D.comm->allreduce(D.part_b.p, kRed, st);  // r.r over the owned dofs of every rank
      launch_precond(D, D.vr.p, D.vz.p, D.vr.p, D.part_a.p, nullptr);
      k_beta_update<<<kRed, kRed, 0, st>>>(n, D.pst.p, D.vp.p, D.vz.p, D.part_a.p, D.part_b.p, D.betas.p);
      count_launch(2);
      CK(cudaMemcpyAsync(&hs, D.pst.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  } else if (persistent_pcg(D)) {
    // one cooperative launch for the whole iteration (k_pcg_persistent)
    const int G = D.pcg_grid;
    D.vp2.alloc(n);
    D.vr2.alloc(n);
    D.part3.alloc(3 * (size_t)G);
    PcgPersist P{};
    P.sd = D.subdesc.p;
    P.xf = D.xf;
    P.lx = D.leafx.p;
    P.wpos = D.wpos.p;
    P.nw = D.nw;
    P.FVall = D.FV.p;
    P.nfv = static_cast<long long>(D.FV.n);
    P.ns = D.n_own;
    P.nrb_schur = (D.max_nB + 63) / 64;
    P.ncb_fwd = (D.max_NF + kFwdTile - 1) / kFwdTile;
    P.wsrc = D.wsrc.p;
    P.wsrcg = D.wsrcg.p;
    P.bwg = D.bw.p;
    P.item_sub = D.item_sub.p;
    P.nitems = D.nitems;
    P.yglob = D.yglob.p;
    P.nrb_bwd = D.max_NF / kTile;
    P.n_root = D.n_root;
    P.NR = D.NR;
    P.root_ptr = D.root_ptr.p;
    P.root_src = D.root_src.p;
    P.Rinv = D.Rinv.p;
    P.fvsrc = D.FV2.p;
    P.xroot = D.xroot2.p;
    P.n = n;
    P.icp = D.icopy_ptr.p;
    P.icpos = D.icopy_pos.p;
    P.WB = D.WB.p;
    P.x = D.vx.p;
    P.z = D.vz.p;
    P.q = D.vq.p;
    P.p[0] = D.vp.p;
    P.p[1] = D.vp2.p;
    P.r[0] = D.vr.p;
    P.r[1] = D.vr2.p;
    P.part = D.part3.p;
    P.st = D.pst.p;
    P.alphas = D.alphas.p;
    P.betas = D.betas.p;
    const char* pe = std::getenv("BDDC_B200_PROFILE");
    const bool trace = pe && *pe && *pe != '0';
    DBuf<unsigned long long> tr;
    if (trace) {
      tr.alloc(64 * 9);
      tr.zero(st);
      P.trace = tr.p;
    }
    void* args[] = {&P};
    CK(cudaLaunchCooperativeKernel((void*)k_pcg_persistent, dim3(G), dim3(256), args, D.pcg_smem, st));
    count_launch(1);
    CK(cudaMemcpyAsync(&hs, D.pst.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (trace) {
      std::vector<unsigned long long> t(64 * 9);
      CK(cudaMemcpy(t.data(), tr.p, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      const char* names[8] = {"schur", "copysum_q", "alpha_restrict", "leaf_fwd", "root", "leaf_bwd", "prolong",
                              "copysum_z"};
      double acc[8] = {0};
      const int its = std::min(hs.it, 64);
      for (int i = 0; i < its; ++i) {
        unsigned long long prev = t[i * 9 + 8];
        for (int k = 0; k < 8; ++k) {
          acc[k] += double(t[i * 9 + k] - prev) * 1e-3;
          prev = t[i * 9 + k];
        }
      }
      std::string line = "[profile] persistent pcg grid=" + std::to_string(G) + " us/iteration:";
      for (int k = 0; k < 8; ++k) line += std::string(" ") + names[k] + "=" + std::to_string(acc[k] / std::max(its, 1));
      std::fprintf(stderr, "%s\n", line.c_str());
    }
  } else {
    // capture one iteration as a graph (pcg.cpp:49-70)
    if (!D.gexec) {
      const long long before = launch_count();
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      const int* done = &D.pst.p->done;
      launch_schur(D, D.vp.p, D.vq.p, D.vp.p, D.part_a.p, done);
      k_alpha_axpy<<<kRed, kRed, 0, st>>>(n, D.pst.p, D.vx.p, D.vr.p, D.vp.p, D.vq.p, D.part_a.p, D.part_b.p,
                                           D.alphas.p);
      launch_precond(D, D.vr.p, D.vz.p, D.vr.p, D.part_a.p, done);
      k_beta_update<<<kRed, kRed, 0, st>>>(n, D.pst.p, D.vp.p, D.vz.p, D.part_a.p, D.part_b.p, D.betas.p);
      CK(cudaStreamEndCapture(st, &D.graph));
      CK(cudaGraphInstantiate(&D.gexec, D.graph, 0));
      D.graph_kernels = launch_count() - before + 2;  // + k_alpha_axpy, k_beta_update
      count_launch(-(launch_count() - before));
    }
    const int chunk = 8;
    while (!hs.done) {
      for (int c = 0; c < chunk; ++c) CK(cudaGraphLaunch(D.gexec, st));
      count_launch(chunk * D.graph_kernels);
      CK(cudaMemcpyAsync(&hs, D.pst.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  }
  CK(cudaEventRecord(D.e1, st));
  times_.pcg = elapsed(D.e0, D.e1);
  times_.pcg_iterations = hs.it;
  CK(cudaGetLastError());
  out.iterations = hs.it;
  out.relative_residual = hs.relres;
  out.converged = hs.relres <= tol;
  out.alphas.resize(hs.it);
  out.betas.resize(hs.it);
  if (hs.it) {
    CK(cudaMemcpy(out.alphas.data(), D.alphas.p, hs.it * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out.betas.data(), D.betas.p, hs.it * sizeof(double), cudaMemcpyDeviceToHost));
  }
  out.condition_estimate = lanczos_condition_estimate(out.alphas, out.betas);
  complete_interface(D, D.vx.p);  // sharded: the whole solution on every rank
  if (x) CK(cudaMemcpyAsync(x, D.vx.p, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return out;
}

StepOut Engine::step(const StepSpec& sp, ConstraintSet& cs, double* u_free_host) {
  NvtxRange nvtx("bddc:step");
  DeviceState& D = *d_;
  prepare();
  StepOut out;
  const long long l0 = launch_count();
  cudaStream_t st = D.st;
  CK(cudaStreamSynchronize(st));
  HostTimer ht("step");
  CK(cudaEventRecord(D.s0, st));
  if (sp.e2e) {
    // the inputs go over on their own stream, behind the step's start event;
    // the assembly waits for them after the fronts' zero-fill (assemble_fronts)
    CK(cudaStreamWaitEvent(D.copy_st, D.s0, 0));
    out.h2d_bytes = upload_inputs(true);
    CK(cudaEventRecord(D.ecopy, D.copy_st));
    D.inputs_pending = true;
  }
  // the leaf factorization runs on the device while the host builds the base
  // constraints and prepares the face-pair problems
  analysis_launch();
  ht.mark("launch");
  cs = arithmetic_constraints(m_, sp.edges, sp.faces);
  ht.mark("base_constraints");
  EnrichOptions o;
  o.tau = sp.tau;
  o.max_vectors = sp.max_vectors;
  o.keep_edge_constraints = sp.keep_edge;
  o.fixed_count = sp.fixed_count;
  const bool adaptive = sp.adaptive || sp.fixed_count >= 0;
  std::shared_ptr<PairPrep> prep;
  if (adaptive) prep = D.pairs.prepare(cs, o);
  ht.mark("pair_prep");
  // the hub stage of the eigenproblems is enqueued behind the analysis before
  // the host waits for it (stream order gives it the S_s it reads), so the
  // device does not idle while the pivots are checked and the first chunk of
  // pair descriptors is built
  if (adaptive) {
    CK(cudaEventRecord(D.eg0, st));
    D.pairs.start(prep);
  }
  ht.mark("hubs_launch");
  analysis_finish();
  ht.mark("analysis_wait");
  if (adaptive) {
    out.omega_tilde = D.pairs.enrich(cs, o, prep).omega_tilde;
    CK(cudaEventRecord(D.eg1, st));
    times_.eigen = elapsed(D.eg0, D.eg1);
  }
  ht.mark("eigen");
  out.constraint_rows = cs.row_count(m_);
  set_constraints(cs);
  ht.mark("set_constraints");
  CK(cudaEventRecord(D.s1, st));
  out.pcg = pcg(nullptr, nullptr, sp.tol, sp.max_it, false);
  ht.mark("pcg");
  if (sp.e2e) {
    if (D.ufree.n == 0) D.ufree.alloc(std::max<i64>(m_.free_count, 1));
    recover_device(D.vx.p, D.ufree.p);
    CK(cudaMemcpyAsync(u_free_host, D.ufree.p, m_.free_count * sizeof(double), cudaMemcpyDeviceToHost, st));
    out.d2h_bytes = double(m_.free_count) * sizeof(double);
  }
  CK(cudaEventRecord(D.s2, st));
  out.seconds = elapsed(D.s0, D.s2);
  out.setup_seconds = elapsed(D.s0, D.s1);
  out.solve_seconds = elapsed(D.s1, D.s2);
  out.launches = launch_count() - l0;
  return out;
}

EnrichOutcome Engine::enrich(ConstraintSet& cs, const EnrichOptions& o) {
  CK(cudaEventRecord(d_->e0, d_->st));
  EnrichOutcome out = d_->pairs.enrich(cs, o);
  CK(cudaEventRecord(d_->e1, d_->st));
  times_.eigen = elapsed(d_->e0, d_->e1);
  return out;
}


void Engine::invalidate_preconditioner() {
  DeviceState& D = *d_;
  D.have_prec = false;
  if (D.gexec) {
    cudaGraphExecDestroy(D.gexec);
    D.gexec = nullptr;
  }
  if (D.graph) {
    cudaGraphDestroy(D.graph);
    D.graph = nullptr;
  }
}

}  // namespace b200
