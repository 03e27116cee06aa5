// Microbenchmarks used to pin the FP64 roofline denominators on B200 (sm_100a).
// DFMA peak, DMMA (mma.sync m8n8k4 f64) peak, and cuFFT D2Z/Z2D timings at the
// headline padded grid. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 probe_fp64.cu -lcufft
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cufft.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"", p.name, p.multiProcessorCount, p.major, p.minor);
  double* d; CK(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DFMA
  {
    int iters = 20000, threads = 512, blocks = sms * 4;
    dfma_kernel<<<blocks, threads>>>(d, 100, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 16.0 * iters * threads * (double)blocks;
    printf(", \"dfma_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  }
  // DMMA
  {
    int iters = 20000, threads = 256, blocks = sms * 8;
    dmma_kernel<<<blocks, threads>>>(d, 100); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256.0 * 8 * iters * (threads / 32) * (double)blocks;
    printf(", \"dmma_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  }
  // copy bandwidth (read + write)
  {
    size_t n = (size_t)1 << 28;  // 4 GiB per buffer of double2
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 0, n * 16);
    copy_kernel<<<sms * 8, 512>>>(a, b, n); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); copy_kernel<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf(", \"copy_gbs\": %.1f", 2.0 * n * 16 / (best * 1e-3) / 1e9);
    cudaFree(a); cudaFree(b);
  }
  // cuFFT at the headline padded grid (480,480,924)
  {
    int nx = 480, ny = 480, nz = 924;
    size_t nreal = (size_t)nx * ny * nz, ncplx = (size_t)nx * ny * (nz / 2 + 1);
    double* r; cufftDoubleComplex* c;
    CK(cudaMalloc(&r, nreal * 8)); CK(cudaMalloc(&c, ncplx * 16));
    cudaMemset(r, 0, nreal * 8);
    cufftHandle pf, pb;
    size_t ws;
    if (cufftPlan3d(&pf, nx, ny, nz, CUFFT_D2Z) != CUFFT_SUCCESS) { printf("plan fail\n"); return 1; }
    if (cufftPlan3d(&pb, nx, ny, nz, CUFFT_Z2D) != CUFFT_SUCCESS) { printf("plan fail\n"); return 1; }
    cufftGetSize(pf, &ws);
    float bf = 1e30f, bb = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); cufftExecD2Z(pf, r, c); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < bf) bf = ms;
      cudaEventRecord(e0); cufftExecZ2D(pb, c, r); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); if (ms < bb) bb = ms;
    }
    printf(", \"fft_d2z_480x480x924_ms\": %.3f, \"fft_z2d_ms\": %.3f, \"fft_workspace_mb\": %.1f", bf, bb, ws / 1e6);
    cufftDestroy(pf); cufftDestroy(pb);
    // 7-smooth alternative (480,480,900)?  900 = 2^2 3^2 5^2
    int nz2 = 900;
    cufftPlan3d(&pf, nx, ny, nz2, CUFFT_D2Z);
    bf = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); cufftExecD2Z(pf, r, c); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < bf) bf = ms;
    }
    printf(", \"fft_d2z_480x480x900_ms\": %.3f", bf);
    cufftDestroy(pf);
    cudaFree(r); cudaFree(c);
  }
  printf("}\n");
  return 0;
}
