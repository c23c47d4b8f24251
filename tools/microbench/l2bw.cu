// Microbenchmark: L2-resident vs HBM bandwidth on the B200 (decides whether K1's binned records
// may round-trip through L2 instead of HBM).  Prints one JSON line per case.
//   read   : every thread streams 16-byte loads over a buffer of S bytes, many passes (L2 hits when
//            S fits in L2; ld.global.cg so L1 is bypassed)
//   rw     : each CTA writes a 16-byte-per-thread slice and reads another CTA's slice of a ring of S
//            bytes (the record hand-off pattern: written by one SM, read by another)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void __launch_bounds__(512) k_read(const float4 *__restrict__ buf, size_t n16, int passes, float *out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; ++p) {
    // each pass starts at a CTA-dependent offset so consecutive passes do not hit the same SM's lines
    const size_t off = ((size_t)p * 7919 * blockDim.x) % n16;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
      size_t j = i + off;
      if (j >= n16) j -= n16;
      const float4 v = __ldcg(buf + j);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void __launch_bounds__(512) k_rw(float4 *__restrict__ buf, size_t n16, int passes, float *out) {
  float acc = 0.f;
  const size_t per = n16 / gridDim.x;  // slice per CTA
  for (int p = 0; p < passes; ++p) {
    float4 *w = buf + (size_t)((blockIdx.x + p) % gridDim.x) * per;
    const float4 *r = buf + (size_t)((blockIdx.x + p + gridDim.x / 2) % gridDim.x) * per;
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) __stcg(w + i, make_float4(p, i, 1.f, 2.f));
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) {
      const float4 v = __ldcg(r + i);
      acc += v.x + v.w;
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *out;
  CK(cudaMalloc(&out, 4));
  const size_t maxb = (size_t)4 << 30;
  float4 *buf;
  CK(cudaMalloc(&buf, maxb));
  CK(cudaMemset(buf, 0, maxb));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t sizes[] = {(size_t)8 << 20, (size_t)16 << 20, (size_t)32 << 20, (size_t)48 << 20, (size_t)64 << 20,
                          (size_t)96 << 20, (size_t)128 << 20, (size_t)1 << 30, (size_t)4 << 30};
  for (size_t S : sizes) {
    const size_t n16 = S / 16;
    const int passes = (int)std::max<size_t>(1, ((size_t)16 << 30) / S);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_read<<<sms * 4, 512>>>(buf, n16, passes, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("{\"case\":\"read\",\"MB\":%zu,\"GBs\":%.1f}\n", S >> 20, (double)S * passes / (ms * 1e6));
    }
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_rw<<<sms, 512>>>(buf, n16, passes, out);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const size_t per = (n16 / sms) * 16;
      if (rep) printf("{\"case\":\"write+read\",\"MB\":%zu,\"GBs\":%.1f}\n", S >> 20,
                      2.0 * per * sms * passes / (ms * 1e6));
    }
  }
  return 0;
}
