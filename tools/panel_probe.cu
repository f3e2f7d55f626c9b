// Cycle probe of the 64x64 panel factorization pieces (dense.cu internals):
//   tools/panel_probe   -> clock64 per chol16 call and per panel_factor call
#include "../paper_0910_5863_b200/csrc/cuda/dense.cu"

namespace b200 {
namespace {
__global__ void k_probe(const double* src, long long* cyc, double* out) {
  extern __shared__ __align__(16) double sm[];
  double* L = sm;
  double* V = sm + 64 * LDS;
  __shared__ double rdp[64];
  const int tid = threadIdx.x;
  for (int it = 0; it < 4; ++it) {
    for (int e = tid; e < 64 * 64; e += blockDim.x) L[(e / 64) * LDS + e % 64] = src[e];
    __syncthreads();
    long long t0 = clock64();
    if (tid < 32) chol16(L, rdp, tid & 31);
    __syncthreads();
    long long t1 = clock64();
    for (int e = tid; e < 64 * 64; e += blockDim.x) L[(e / 64) * LDS + e % 64] = src[e];
    __syncthreads();
    long long t2 = clock64();
    panel_factor<128>(L, V, out);
    __syncthreads();
    long long t3 = clock64();
    if (tid == 0 && it == 3) {
      cyc[0] = t1 - t0;
      cyc[1] = t3 - t2;
    }
  }
}
}  // namespace
}  // namespace b200

int main() {
  double h[64 * 64];
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) h[j * 64 + i] = (i == j ? 100.0 : 0.0) + 1.0 / (1 + i + j);
  double *d, *out;
  long long* c;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&out, sizeof(h));
  cudaMalloc(&c, 16);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const int smem = 2 * 64 * b200::LDS * 8;
  cudaFuncSetAttribute(b200::k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  b200::k_probe<<<1, 128, smem>>>(d, c, out);
  long long hc[2];
  cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
  printf("chol16 %lld cycles, panel_factor<128> %lld cycles (%s)\n", hc[0], hc[1],
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
