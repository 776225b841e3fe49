#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
struct Big { char b[3600]; };
struct Small { char b[64]; };
__global__ void kbig(const __grid_constant__ Big a) { if (a.b[threadIdx.x] == 42) printf("x"); }
__global__ void ksmall(const __grid_constant__ Small a) { if (a.b[threadIdx.x] == 42) printf("x"); }
int main() {
  Big b = {}; Small s = {};
  cudaStream_t st; cudaStreamCreate(&st);
  for (int i = 0; i < 100; ++i) { kbig<<<296, 288, 0, st>>>(b); ksmall<<<296, 288, 0, st>>>(s); }
  cudaDeviceSynchronize();
  const int n = 20000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) kbig<<<296, 288, 0, st>>>(b);
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  auto t2 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) ksmall<<<296, 288, 0, st>>>(s);
  auto t3 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  auto t4 = std::chrono::steady_clock::now();
  int v = 0;
  auto t5 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) { cudaPointerAttributes at; cudaPointerGetAttributes(&at, &b); v += at.type; }
  auto t6 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) { int d; cudaGetDevice(&d); cudaSetDevice(d); }
  auto t7 = std::chrono::steady_clock::now();
  auto us = [&](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count() / n; };
  printf("launch 3.6KB param: enqueue %.2f us (wall %.2f); 64B param: enqueue %.2f us (wall %.2f); cudaPointerGetAttributes %.2f us; get+setDevice %.2f us (%d)\n",
         us(t0, t1), us(t0, t2), us(t2, t3), us(t2, t4), us(t5, t6), us(t6, t7), v);
}
