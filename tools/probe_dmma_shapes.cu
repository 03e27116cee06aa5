// FP64 mma.sync shapes on B200 (sm_100a): throughput with NACC independent accumulator sets per warp
// and W warps per SM; prints TFLOP/s and cycles per instruction per SM sub-partition.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_dmma_shapes probe_dmma_shapes.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int SHAPE, int NACC>
__global__ void k(double* out, int iters) {
  double a[8], b[4], c[NACC][4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * (i + 1);
  for (int n = 0; n < NACC; ++n) for (int i = 0; i < 4; ++i) c[n][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int n = 0; n < NACC; ++n) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[n][0]), "+d"(c[n][1]) : "d"(a[0]), "d"(b[0]));
      else if (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[n][0]), "+d"(c[n][1]), "+d"(c[n][2]), "+d"(c[n][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[n][0]), "+d"(c[n][1]), "+d"(c[n][2]), "+d"(c[n][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[n][0]), "+d"(c[n][1]), "+d"(c[n][2]), "+d"(c[n][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int n = 0; n < NACC; ++n) for (int i = 0; i < 4; ++i) s += c[n][i];
  if (s == 12345.678) out[0] = s;
}

template <int SHAPE, int NACC>
void run(const char* name, double fma_per_inst, int sms, double* d, int warps_per_sm, double clk_ghz) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000, threads = 32 * warps_per_sm, blocks = sms;
  k<SHAPE, NACC><<<blocks, threads>>>(d, 10); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k<SHAPE, NACC><<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double ninst = (double)NACC * iters * warps_per_sm * blocks;
  const double tf = 2.0 * fma_per_inst * ninst / (best * 1e-3) / 1e12;
  const double cyc_per_inst_smsp = best * 1e-3 * clk_ghz * 1e9 / ((double)NACC * iters * warps_per_sm / 4.0);
  printf("{\"shape\": \"%s\", \"nacc\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f, \"cycles_per_inst_per_smsp\": %.2f}\n", name,
         NACC, warps_per_sm, tf, cyc_per_inst_smsp);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double clk = p.clockRate * 1e-6;
  double* d; CK(cudaMalloc(&d, 64));
  for (int w : {4, 8, 16}) {
    run<0, 1>("m8n8k4", 256, sms, d, w, clk);
    run<0, 3>("m8n8k4", 256, sms, d, w, clk);
    run<0, 8>("m8n8k4", 256, sms, d, w, clk);
    run<1, 1>("m16n8k4", 512, sms, d, w, clk);
    run<1, 8>("m16n8k4", 512, sms, d, w, clk);
    run<2, 1>("m16n8k8", 1024, sms, d, w, clk);
    run<2, 8>("m16n8k8", 1024, sms, d, w, clk);
    run<3, 1>("m16n8k16", 2048, sms, d, w, clk);
    run<3, 8>("m16n8k16", 2048, sms, d, w, clk);
  }
  return 0;
}
