// fp64_peak.cu -- measure the FP64 roofline denominators on the box:
// SIMT DFMA throughput and FP64 tensor-core (mma.sync m8n8k4 .f64 = SASS DMMA)
// throughput.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, double a, double b) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(acc[i][0], acc[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int blocks_per_sm : {4, 8}) {
    int grid = sms * blocks_per_sm, threads = 256;
    for (int k = 0; k < 2; ++k) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (k == 0) dfma_kernel<<<grid, threads>>>(out, 1.0000001, 1e-9);
        else dmma_kernel<<<grid, threads>>>(out, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = (k == 0) ? 2.0 * 8 * ITERS * double(grid) * threads
                              : 2.0 * 8 * ITERS * double(grid) * (threads / 32) * 256;
      printf("%s blocks/SM=%d: %.3f ms, %.2f TFLOP/s\n", k == 0 ? "DFMA (SIMT)" : "DMMA m8n8k4", blocks_per_sm, ms,
             flops / ms / 1e9);
    }
  }
  // sustained: the DMMA kernel back to back for ~4 s (the power cap settles), rate
  // of the last second -- the denominator for kernels timed inside long runs
  {
    const int grid = sms * 8, threads = 256;
    const double flops = 2.0 * 8 * ITERS * double(grid) * (threads / 32) * 256;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    int n = 0;
    float total = 0.f;
    while (total < 3000.f) {  // ~3 s of warm load
      cudaEventRecord(e0);
      for (int i = 0; i < 50; ++i) dmma_kernel<<<grid, threads>>>(out, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      total += ms;
      n += 50;
    }
    cudaEventRecord(t0);
    for (int i = 0; i < 250; ++i) dmma_kernel<<<grid, threads>>>(out, 1.0000001, 1e-9);
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    printf("DMMA m8n8k4 sustained (after %d launches / %.1f s): %.2f TFLOP/s over %d launches (%.3f ms each)\n", n,
           total / 1e3, 250 * flops / ms / 1e9, 250, ms / 250);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
