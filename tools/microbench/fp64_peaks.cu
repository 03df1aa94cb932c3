// Microbenchmarks for the FP64 design decisions of the sigma kernels:
// DMMA (mma.sync f64) vs DFMA issue throughput, shared-memory fp64 atomicAdd
// (CAS loop on sm_100a) throughput, and global RED.F64 throughput.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void k_dmma(double* out, int iters){
  double a0=threadIdx.x*1e-9, b0=1.0;
  double c[4][4]={};
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<4;j++)
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+d"(c[j][0]),"+d"(c[j][1]),"+d"(c[j][2]),"+d"(c[j][3]) : "d"(a0),"d"(a0),"d"(b0));
  }
  double s=0; for(int j=0;j<4;j++) s+=c[j][0]+c[j][1]+c[j][2]+c[j][3];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_dfma(double* out, int iters){
  double a=threadIdx.x*1e-9, b=1.0000001;
  double c[8]={};
  for(int i=0;i<iters;i++){
#pragma unroll
    for(int j=0;j<8;j++) c[j]=fma(a,b,c[j]);
  }
  double s=0; for(int j=0;j<8;j++) s+=c[j];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_satom(double* out, const unsigned* idx, int n, int nrow){
  extern __shared__ double s[];
  for(int i=threadIdx.x;i<nrow;i+=blockDim.x) s[i]=0;
  __syncthreads();
  for(int i=threadIdx.x;i<n;i+=blockDim.x){ unsigned t=idx[i]; atomicAdd(&s[t%nrow], 1.0); }
  __syncthreads();
  for(int i=threadIdx.x;i<nrow;i+=blockDim.x) out[blockIdx.x*nrow+i]=s[i];
}
__global__ void k_gred(double* out, const unsigned* idx, int n, int nrow){
  for(int i=threadIdx.x;i<n;i+=blockDim.x){ unsigned t=idx[i]; atomicAdd(&out[blockIdx.x*nrow + t%nrow], 1.0); }
}
int main(){
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 64<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int warps : {4,8,12,16,32}){
    int iters=20000; int thr=warps*32;
    k_dmma<<<nsm,thr>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_dmma<<<nsm,thr>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops=2.0*16*8*4*4*(double)iters*warps*nsm;
    printf("DMMA m16n8k4 warps/SM=%d: %.2f TFLOP/s\n", warps, flops/ms/1e9);
  }
  for(int warps : {4,8,16,32}){
    int iters=20000; int thr=warps*32;
    k_dfma<<<nsm,thr>>>(out,100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_dfma<<<nsm,thr>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops=2.0*8*(double)iters*thr*nsm;
    printf("DFMA warps/SM=%d: %.2f TFLOP/s\n", warps, flops/ms/1e9);
  }
  int n=1<<22; unsigned* idx; CK(cudaMalloc(&idx, n*4));
  unsigned* h=(unsigned*)malloc(n*4); unsigned long long x=88172645463325252ull;
  for(int i=0;i<n;i++){ x^=x<<13; x^=x>>7; x^=x<<17; h[i]=(unsigned)x; }
  cudaMemcpy(idx,h,n*4,cudaMemcpyHostToDevice);
  int nrow=12870; size_t sm=nrow*8; cudaFuncSetAttribute(k_satom, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for(int thr : {256,512,1024}){
    k_satom<<<nsm,thr,sm>>>(out,idx,n,nrow); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); k_satom<<<nsm,thr,sm>>>(out,idx,n,nrow); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    printf("smem f64 atomicAdd (CAS) thr=%d: %.3f Gatom/s total, %.3f atom/clk/SM @1.9GHz\n", thr, (double)n*nsm/ms/1e6, (double)n*nsm/(ms*1e-3)/nsm/1.9e9);
  }
  CK(cudaMemset(out,0,nsm*nrow*8));
  for(int thr : {256,1024}){
    cudaEventRecord(e0); k_gred<<<nsm,thr>>>(out,idx,n,nrow); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    printf("global RED.F64 thr=%d: %.3f Gred/s total\n", thr, (double)n*nsm/ms/1e6);
  }
  return 0;
}
