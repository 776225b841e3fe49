// kernels_aux.cu -- one-time helpers of the C ABI (not on the per-matvec path).
//
// transpose_leaf_blocks: D^T for the transposed product H^T x (GEMV "T",
// PAPER.md:961-969): H^T has the same block structure with U and V exchanged
// and every dense leaf block transposed, so the expand kernel runs unchanged on
// (V, U, D^T).
#include "kernels.h"

namespace hmat {
namespace {

__global__ void transpose_leaf_blocks_kernel(const double* __restrict__ D, double* __restrict__ Dt, int64_t n_leaves,
                                             int b, int Dp) {
  const int64_t total = n_leaves * b * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / ((int64_t)b * b);
    const int rem = static_cast<int>(e - k * b * b);
    const int i = rem / b, j = rem - i * b;
    Dt[(k * b + j) * Dp + i] = D[(k * b + i) * Dp + j];
  }
}

}  // namespace

cudaError_t launch_transpose_leaf_blocks(const double* D, double* Dt, int64_t n_leaves, int b, int Dp,
                                         cudaStream_t s) {
  const int64_t total = n_leaves * b * b;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  if (grid < 1) grid = 1;
  transpose_leaf_blocks_kernel<<<static_cast<int>(grid), 256, 0, s>>>(D, Dt, n_leaves, b, Dp);
  return cudaGetLastError();
}

}  // namespace hmat
