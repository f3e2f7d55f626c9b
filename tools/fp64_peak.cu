#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_k4(double* out, int iters){
  double a0=threadIdx.x*1e-3, b0=1.0+threadIdx.x*1e-4;
  double c[8][4]={};
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<8;j++){
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
        : "+d"(c[j][0]),"+d"(c[j][1]),"+d"(c[j][2]),"+d"(c[j][3]) : "d"(a0),"d"(a0),"d"(b0));
    }
  }
  double s=0; for(int j=0;j<8;j++) for(int q=0;q<4;q++) s+=c[j][q];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void dmma_k16(double* out, int iters){
  double a0=threadIdx.x*1e-3, b0=1.0+threadIdx.x*1e-4;
  double c[4][4]={};
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<4;j++){
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
        : "+d"(c[j][0]),"+d"(c[j][1]),"+d"(c[j][2]),"+d"(c[j][3]) : "d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(a0),"d"(b0),"d"(b0),"d"(b0),"d"(b0));
    }
  }
  double s=0; for(int j=0;j<4;j++) for(int q=0;q<4;q++) s+=c[j][q];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void dfma(double* out, int iters){
  double a=threadIdx.x*1e-3, b=1.0+threadIdx.x*1e-4;
  double c[16]={};
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<16;j++) c[j]=fma(a,c[j],b);
  }
  double s=0; for(int j=0;j<16;j++) s+=c[j];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p,dev);
  printf("%s SMs %d cc %d.%d clock %d\n",p.name,p.multiProcessorCount,p.major,p.minor,p.clockRate);
  double* out; cudaMalloc(&out, 1<<26);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks=p.multiProcessorCount*4, threads=256, iters=20000;
  for(int rep=0;rep<2;rep++){
  float ms;
  cudaEventRecord(e0); dmma_k4<<<blocks,threads>>>(out,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms,e0,e1);
  double fl=2.0*16*8*4*8.0*iters*(double)blocks*threads/32;
  printf("dmma m16n8k4: %.2f TFLOP/s\n", fl/ms/1e9);
  cudaEventRecord(e0); dmma_k16<<<blocks,threads>>>(out,iters/4); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms,e0,e1);
  fl=2.0*16*8*16*4.0*(iters/4)*(double)blocks*threads/32;
  printf("dmma m16n8k16: %.2f TFLOP/s\n", fl/ms/1e9);
  cudaEventRecord(e0); dfma<<<blocks,threads>>>(out,iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms,e0,e1);
  fl=2.0*16*(double)iters*blocks*threads;
  printf("dfma: %.2f TFLOP/s\n", fl/ms/1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
