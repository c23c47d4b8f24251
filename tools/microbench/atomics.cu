// Microbenchmark: accumulation primitives available to the type-1 spreader on sm_100a.
// Measures per-SM throughput of shared-memory integer atomics (native ATOMS.ADD), fp64 shared
// atomicAdd (compiles to an ATOMS.CAST.SPIN.64 CAS loop), non-atomic shared RMW, global fp64 RED
// (L2 atomic unit) and the FP64 FMA pipe. Results decide the K1 design ("K1").
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

template<int MODE>
__global__ void __launch_bounds__(1024) k_smem(double* out, int iters, int words){
  extern __shared__ unsigned char sm[];
  unsigned* su=(unsigned*)sm; double* sd=(double*)sm;
  int nthr=blockDim.x;
  for(int i=threadIdx.x;i<words;i+=nthr) su[i]=0;
  __syncthreads();
  uint32_t s=hsh(threadIdx.x*7919u+blockIdx.x*104729u);
  double acc=0;
  int mask_u=words-1, mask_d=words/2-1;
  for(int it=0;it<iters;++it){
    s=s*1664525u+1013904223u;
    if(MODE==0){ atomicAdd(&su[(s>>8)&mask_u], s); }
    else if(MODE==1){ atomicAdd(&sd[(s>>8)&mask_d], (double)(s&255)); }
    else if(MODE==2){ int a=(s>>8)&mask_d; sd[a]+= (double)(s&255); }
    else if(MODE==3){ // 5 consecutive cells per op (a footprint row), integer atomics
      int a=(s>>8)&(mask_u-7); 
      #pragma unroll
      for(int c=0;c<5;++c) atomicAdd(&su[a+c], s+c); }
    else if(MODE==4){ // int64 fixed-point accumulation (survey §7 step 4(d)): 64-bit integer shared atomics
      unsigned long long* sl=(unsigned long long*)sm; atomicAdd(&sl[(s>>8)&mask_d], (unsigned long long)s); }
    else if(MODE==5){ // fp32 shared atomicAdd (native RED/ATOMS.ADD.F32)
      float* sf=(float*)sm; atomicAdd(&sf[(s>>8)&mask_u], (float)(s&255)); }
  }
  __syncthreads();
  if(threadIdx.x==0){ double t=0; for(int i=0;i<64;++i) t+=su[i]; out[blockIdx.x]=t+acc; }
}

__global__ void __launch_bounds__(1024) k_gred(double* grid, int iters, int cells){
  uint32_t s=hsh(threadIdx.x*7919u+blockIdx.x*104729u);
  for(int it=0;it<iters;++it){ s=s*1664525u+1013904223u; atomicAdd(&grid[(s>>8)%cells], (double)(s&255)); }
}

__global__ void __launch_bounds__(1024) k_dfma(double* out, int iters){
  double a0=threadIdx.x, a1=a0+1, a2=a0+2, a3=a0+3, a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  const double b=1.0000001, c=1e-9;
  for(int it=0;it<iters;++it){
    a0=fma(a0,b,c);a1=fma(a1,b,c);a2=fma(a2,b,c);a3=fma(a3,b,c);a4=fma(a4,b,c);a5=fma(a5,b,c);a6=fma(a6,b,c);a7=fma(a7,b,c);
  }
  if(a0+a1+a2+a3+a4+a5+a6+a7==12345.0) out[0]=1;
}

__global__ void k_read(const double2* __restrict__ x, size_t n, double* out){
  double acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ double2 v=__ldg(&x[i]); acc+=v.x+v.y; }
  if(acc==1234.5) out[0]=acc;
}

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  int clk_khz=0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  int nsm=p.multiProcessorCount; printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_mhz_attr\":%.0f}\n",p.name,nsm,clk_khz/1e3);
  double* out; CK(cudaMalloc(&out, 1<<20));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int smem=200*1024;
  CK(cudaFuncSetAttribute(k_smem<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_smem<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_smem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_smem<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_smem<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int words=32768; // 128 KB region
  const char* names[6]={"smem_u32_atomicAdd","smem_f64_atomicAdd_CAS","smem_f64_nonatomic_RMW","smem_u32_atomicAdd_5consec",
                        "smem_u64_atomicAdd_fixedpoint","smem_f32_atomicAdd"};
  for(int mode=0;mode<6;++mode){
    for(int thr: {256,1024}){
      int iters=4096;
      for(int rep=0;rep<2;++rep){
        cudaEventRecord(e0);
        if(mode==0) k_smem<0><<<nsm,thr,smem>>>(out,iters,words);
        if(mode==1) k_smem<1><<<nsm,thr,smem>>>(out,iters,words);
        if(mode==2) k_smem<2><<<nsm,thr,smem>>>(out,iters,words);
        if(mode==3) k_smem<3><<<nsm,thr,smem>>>(out,iters,words);
        if(mode==4) k_smem<4><<<nsm,thr,smem>>>(out,iters,words);
        if(mode==5) k_smem<5><<<nsm,thr,smem>>>(out,iters,words);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms,e0,e1);
        double ops=(double)nsm*thr*iters*(mode==3?5:1);
        if(rep==1) printf("{\"test\":\"%s\",\"threads\":%d,\"Gops\":%.1f,\"ops_per_sm_per_ns\":%.3f}\n",names[mode],thr,ops/ms/1e6,ops/ms/1e6/nsm);
      }
    }
  }
  for(int cells: {4096, 44100, 1<<20, 1<<24}){
    double* g; CK(cudaMalloc(&g, (size_t)cells*8)); cudaMemset(g,0,(size_t)cells*8);
    int iters=2048;
    for(int rep=0;rep<2;++rep){
      cudaEventRecord(e0); k_gred<<<nsm*2,1024>>>(g,iters,cells); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms,e0,e1); double ops=(double)nsm*2*1024*iters;
      if(rep==1) printf("{\"test\":\"global_RED_f64\",\"cells\":%d,\"Gops\":%.1f}\n",cells,ops/ms/1e6);
    }
    cudaFree(g);
  }
  for(int rep=0;rep<2;++rep){
    int iters=1<<14; cudaEventRecord(e0); k_dfma<<<nsm*4,512>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1); double f=(double)nsm*4*512*iters*8;
    if(rep==1) printf("{\"test\":\"dfma\",\"TFMA_per_s\":%.3f,\"TFLOPS\":%.2f}\n",f/ms/1e9,2*f/ms/1e9);
  }
  size_t n=(size_t)1<<28; double2* x; CK(cudaMalloc(&x,n*16)); cudaMemset(x,0,n*16);
  for(int rep=0;rep<3;++rep){
    cudaEventRecord(e0); k_read<<<nsm*8,512>>>(x,n,out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1); if(rep==2) printf("{\"test\":\"hbm_read_double2\",\"GBps\":%.0f}\n",n*16/ms/1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
