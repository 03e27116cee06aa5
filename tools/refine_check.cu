// Accuracy of the pair kernel's refined hardware rsqrt / rcp (pair.cu, PC_NEWTON = 3: one
// third-order step) against correctly rounded 1/sqrt(v) and 1/v, over random v spanning the
// pair kernel's r^2 and x + 3 ranges.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cmath>
__device__ double rs3(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  const double h = r2 * y;
  const double e = fma(-h, y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}
__device__ double rc3(double v) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
  const double e = fma(-v, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
__device__ double hw_rs(double r2) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2)); return y; }
__global__ void k(unsigned long long n, double* out) {
  double m0 = 0, m1 = 0, m2 = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    // v = 2^(-40 .. +8) with random mantissa (splitmix)
    unsigned long long z = i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u = (double)(z >> 11) * 0x1.0p-53;
    const double v = exp2(-40.0 + 48.0 * u);
    const double t = 1.0 / sqrt(v);
    m0 = fmax(m0, fabs(rs3(v) - t) / t);
    m2 = fmax(m2, fabs(hw_rs(v) - t) / t);
    const double w = 3.0 + 8.0 * u;
    const double c = 1.0 / w;
    m1 = fmax(m1, fabs(rc3(w) - c) / c);
  }
  atomicMax((unsigned long long*)&out[0], __double_as_longlong(m0));
  atomicMax((unsigned long long*)&out[1], __double_as_longlong(m1));
  atomicMax((unsigned long long*)&out[2], __double_as_longlong(m2));
}
int main() {
  double* d;
  cudaMalloc(&d, 3 * sizeof(double));
  cudaMemset(d, 0, 3 * sizeof(double));
  k<<<1184, 256>>>(1ull << 32, d);
  double h[3];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"samples\": %llu, \"rsqrt_refined_max_rel\": %.3e, \"rcp_refined_max_rel\": %.3e, \"rsqrt_hw_max_rel\": %.3e, \"ulp\": %.3e}\n",
         1ull << 32, h[0], h[1], h[2], 0x1.0p-53);
  return 0;
}
