// Host enqueue cost of hmat_matvec from C (no Python): c1's shape (2D, L = 3,
// b = 64, r = 8), device x / y, N calls back to back, then one synchronise.
//   nvcc -O2 -Iinclude scripts/host_overhead_c.cu -Lpaper_2008_12441_b200 -lhmat \
//        -Xlinker -rpath,$PWD/paper_2008_12441_b200 -o /tmp/host_overhead_c
#include <chrono>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

#include "hmat.h"

int main() {
  const int dim = 2, depth = 3, leaf = 64, rank = 8, W = 3 * rank;
  const long long N = 64LL * 64;
  std::vector<double> panel(N * W, 0.01), D(N * leaf, 0.01);
  std::vector<const double*> U(depth, panel.data()), V(depth, panel.data());
  hmat_t H = nullptr;
  if (hmat_create(depth, dim, leaf, rank, U.data(), V.data(), D.data(), nullptr, &H) != HMAT_OK) {
    std::printf("create failed: %s\n", hmat_last_error());
    return 1;
  }
  double *x, *y;
  cudaMalloc(&x, N * sizeof(double));
  cudaMalloc(&y, N * sizeof(double));
  cudaMemset(x, 0, N * sizeof(double));
  for (int i = 0; i < 100; ++i) hmat_matvec(H, x, y, 1);
  cudaDeviceSynchronize();
  const int calls = 20000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < calls; ++i) hmat_matvec(H, x, y, 1);
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  auto t2 = std::chrono::steady_clock::now();
  const double enq = std::chrono::duration<double, std::micro>(t1 - t0).count() / calls;
  const double wall = std::chrono::duration<double, std::micro>(t2 - t0).count() / calls;
  std::printf("c1 shape from C: host enqueue %.2f us/call, wall incl. GPU %.2f us/call\n", enq, wall);
  // host cost alone: a burst short enough not to fill the launch queue
  {
    cudaDeviceSynchronize();
    auto b0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 100; ++i) hmat_matvec(H, x, y, 1);
    auto b1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    std::printf("host cost of a call (burst of 100, queue not full): %.2f us\n",
                std::chrono::duration<double, std::micro>(b1 - b0).count() / 100);
  }
  // GPU time alone: 100 matvecs captured in a CUDA graph, replayed
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  hmat_set_stream(H, s);
  hmat_matvec(H, x, y, 1);
  cudaStreamSynchronize(s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 100; ++i) hmat_matvec(H, x, y, 1);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::printf("graph replay: %.2f us per matvec on the GPU (%s)\n", 1e3 * ms / 2000, cudaGetErrorString(cudaGetLastError()));
  hmat_destroy(H);
  return 0;
}
