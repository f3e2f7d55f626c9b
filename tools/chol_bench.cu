// Micro-benchmark of the batched partial Cholesky schedules (dense.cu):
//   tools/chol_bench BATCH N P [AUG] [REPS]
// Factors BATCH copies of one seeded SPD front (N x N, first P columns
// eliminated; AUG > 0 appends the identity-augmented rows as the root/explicit
// fronts do) with BDDC_B200_CHOL=dag and =tiled, prints the event-timed mean
// per call and the largest difference between the two results.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDENSE_TRACE \
//          -I paper_0910_5863_b200/csrc/cuda tools/chol_bench.cu \
//          paper_0910_5863_b200/csrc/cuda/dense.cu -o tools/chol_bench
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "dense.cuh"

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: chol_bench BATCH N P [AUG] [REPS]\n");
    return 2;
  }
  const int batch = std::atoi(argv[1]), n0 = std::atoi(argv[2]), p = std::atoi(argv[3]);
  const int aug = argc > 4 ? std::atoi(argv[4]) : 0;
  const int reps = argc > 5 ? std::atoi(argv[5]) : 20;
  // front [[A, .], [I, 0]] when aug: rows n0 .. n0 + p - 1 hold the identity
  const int n = aug ? n0 + p : n0;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> g;
  std::vector<double> B((size_t)n0 * n0), A((size_t)n * n, 0.0);
  for (auto& x : B) x = g(rng);
  for (int i = 0; i < n0; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0;
      for (int k = 0; k < n0; ++k) s += B[(size_t)k * n0 + i] * B[(size_t)k * n0 + j];
      if (i == j) s += n0;
      A[(size_t)j * n + i] = s;
      A[(size_t)i * n + j] = s;
    }
  if (aug)
    for (int q = 0; q < p; ++q) A[(size_t)q * n + n0 + q] = 1.0;
  const size_t fsz = (size_t)n * n;
  double *pristine, *work, *dinv;
  int* info;
  CK(cudaMalloc(&pristine, fsz * batch * sizeof(double)));
  CK(cudaMalloc(&work, fsz * batch * sizeof(double)));
  CK(cudaMalloc(&dinv, (size_t)(p / 64) * 4096 * batch * sizeof(double)));
  CK(cudaMalloc(&info, batch * sizeof(int)));
  for (int b = 0; b < batch; ++b)
    CK(cudaMemcpy(pristine + b * fsz, A.data(), fsz * sizeof(double), cudaMemcpyHostToDevice));
  std::vector<b200::FrontDesc> ds(batch);
  for (int b = 0; b < batch; ++b)
    ds[b] = b200::FrontDesc{work + b * fsz, dinv + (size_t)b * (p / 64) * 4096, n, p, info + b, aug ? n0 : 0};
  b200::FrontDesc* dd;
  CK(cudaMalloc(&dd, batch * sizeof(b200::FrontDesc)));
  CK(cudaMemcpy(dd, ds.data(), batch * sizeof(b200::FrontDesc), cudaMemcpyHostToDevice));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<double> out[2];
  const char* modes[2] = {"dag", "tiled"};
  const double flops = batch * ((double)p * p * p / 3 + (double)p * p * (n - p) + (double)p * (n - p) * (n - p));
  for (int m = 0; m < 2; ++m) {
    setenv("BDDC_B200_CHOL", modes[m], 1);
    double tot = 0;
    for (int r = 0; r < reps + 3; ++r) {
      CK(cudaMemcpyAsync(work, pristine, fsz * batch * sizeof(double), cudaMemcpyDeviceToDevice, st));
      CK(cudaMemsetAsync(info, 0, batch * sizeof(int), st));
      CK(cudaEventRecord(e0, st));
      b200::partial_cholesky(dd, batch, n, p, n - p, st);
      CK(cudaEventRecord(e1, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 3) tot += ms;
    }
    out[m].resize(fsz * batch);
    CK(cudaMemcpy(out[m].data(), work, fsz * batch * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<int> inf(batch);
    CK(cudaMemcpy(inf.data(), info, batch * sizeof(int), cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int x : inf) bad |= x != 0;
    const double us = tot / reps * 1e3;
    std::printf("%-5s batch %d n %d p %d aug %d: %.1f us  %.2f TF/s  info %s\n", modes[m], batch, n, p, aug, us,
                flops / (us * 1e-6) * 1e-12, bad ? "FAIL" : "ok");
  }
  // per-column timeline of front 0 (dataflow schedule)
  setenv("BDDC_B200_CHOL", "dag", 1);
  CK(cudaMemcpyAsync(work, pristine, fsz * batch * sizeof(double), cudaMemcpyDeviceToDevice, st));
  b200::chol_trace(true, nullptr);
  b200::partial_cholesky(dd, batch, n, p, n - p, st);
  CK(cudaStreamSynchronize(st));
  unsigned long long tr[144];
  b200::chol_trace(false, tr);
  std::printf("front 0 timeline (us: accumulated / published):");
  for (int j = 0; j < p / 64 && j < 64; ++j)
    std::printf(" %d:%.1f/%.1f", j, (tr[2 * j] - tr[0]) * 1e-3, (tr[2 * j + 1] - tr[0]) * 1e-3);
  std::printf("\npanel phases (us):");
  for (int q = 1; q < 16; ++q) std::printf(" %.2f", (tr[128 + q] - tr[128]) * 1e-3);
  std::printf("\n");
  for (int m = 0; m < 2; ++m) {
    setenv("BDDC_B200_CHOL", modes[m], 1);
    CK(cudaMemcpyAsync(work, pristine, fsz * batch * sizeof(double), cudaMemcpyDeviceToDevice, st));
    b200::chol_trace(true, nullptr);
    b200::partial_cholesky(dd, batch, n, p, n - p, st);
    CK(cudaStreamSynchronize(st));
    b200::chol_trace(false, tr);
    std::printf("%s panel phases again (us):", modes[m]);
    for (int q = 1; q < 16; ++q) std::printf(" %.2f", (tr[128 + q] - tr[128]) * 1e-3);
    std::printf("\n");
  }
  // lower triangle outside the eliminated diagonal tiles (those keep the unfactored update)
  double dmax = 0, amax = 0;
  for (int b = 0; b < batch; ++b)
    for (int c = 0; c < n; ++c)
      for (int r = c; r < n; ++r) {
        if (c < p && r / 64 == c / 64) continue;
        const size_t i = b * fsz + (size_t)c * n + r;
        dmax = std::fmax(dmax, std::fabs(out[0][i] - out[1][i]));
        amax = std::fmax(amax, std::fabs(out[1][i]));
      }
  std::printf("max |dag - tiled| / max|tiled| = %.3e\n", dmax / amax);
  return 0;
}
