// Device-side copy of efgp_data/philox.py + efgp_data/configs.py: seeded synthetic inputs for the
// five BASELINE workloads, generated directly in HBM (used for N = 1e9, where a host generator
// and a 24 GB host->device copy would dominate).  Input generation only: no EFGP arithmetic.
// Bitwise identical to the numpy generator for uniforms (integer arithmetic); normals and test
// functions go through CUDA's libm (a few ulp from numpy's).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += W0; k1 += W1; }
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

__device__ __forceinline__ double uniform(uint32_t seed, uint32_t stream, uint64_t rec, int k) {
  uint32_t c[4] = {(uint32_t)(rec & 0xFFFFFFFFu), stream, (uint32_t)(k / 2), (uint32_t)(rec >> 32)};
  philox10(c, seed, 0u);
  const uint64_t hi = c[2 * (k % 2)], lo = c[2 * (k % 2) + 1];
  return (double)((hi << 21) + (lo >> 11)) * 0x1p-53;
}

__device__ __forceinline__ double normal(uint32_t seed, uint32_t stream, uint64_t rec, int k) {
  const double u1 = uniform(seed, stream, rec, k), u2 = uniform(seed, stream, rec, k + 1);
  return sqrt(-2.0 * log1p(-u1)) * cos(2.0 * 3.141592653589793 * u2);
}

__device__ double testfunc(int cfg, const double *x) {
  const double pi = 3.141592653589793;
  switch (cfg) {
    case 1: { const double c = cos(2 * pi * x[0]); return sin(6 * pi * x[0]) + c * c; }
    case 2: case 5: return sin(6 * pi * x[0]) * cos(4 * pi * x[1]);
    case 3: { const double a = x[0] - 0.5, b = x[1] - 0.5; return exp(-(a * a + b * b) / 0.02); }
    case 4: return sin(4 * pi * x[0]) * sin(4 * pi * x[1]) * sin(4 * pi * x[2]);
  }
  return 0.0;
}

__global__ void k_points(int cfg, uint32_t seed, int d, int64_t start, int64_t count, double noise,
                         double *__restrict__ x, double *__restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t rec = (uint64_t)(start + i);
    double xc[3];
    if (cfg == 3) {  // 3-component mixture, sd 0.1, clamped to [0,1]^2
      const double means[3][2] = {{0.3, 0.3}, {0.7, 0.5}, {0.5, 0.8}};
      int comp = (int)floor(3.0 * uniform(seed, 3u, rec, 0));
      comp = comp > 2 ? 2 : comp;
      for (int k = 0; k < d; ++k) {
        const double v = means[comp][k] + 0.1 * normal(seed, 0u, rec, 2 * k);
        xc[k] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
      }
    } else {
      for (int k = 0; k < d; ++k) xc[k] = uniform(seed, 0u, rec, k);
    }
    for (int k = 0; k < d; ++k) x[i * d + k] = xc[k];
    if (y) y[i] = testfunc(cfg, xc) + noise * normal(seed, 1u, rec, 0);
  }
}

__global__ void k_targets(uint32_t seed, int d, int64_t start, int64_t count, double *__restrict__ xt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < d; ++k) xt[i * d + k] = uniform(seed, 2u, (uint64_t)(start + i), k);
}

}  // namespace

extern "C" {
// x: (count, d) device, y: (count) device or NULL.  Returns a cudaError_t value.
int efgp_datagen_points(int cfg, uint32_t seed, int d, int64_t start, int64_t count, double noise, double *x,
                        double *y, void *stream) {
  if (count <= 0) return 0;
  k_points<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(cfg, seed, d, start, count, noise, x, y);
  return (int)cudaGetLastError();
}
int efgp_datagen_targets(uint32_t seed, int d, int64_t start, int64_t count, double *xt, void *stream) {
  if (count <= 0) return 0;
  k_targets<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(seed, d, start, count, xt);
  return (int)cudaGetLastError();
}
}
