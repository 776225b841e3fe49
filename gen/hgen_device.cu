/*
 * hgen_device.cu -- device side of the seeded input generator (gen/hgen.h).
 * TEST/BENCH INFRASTRUCTURE: writes the same synthetic inputs as
 * gen/hgen_host.c straight into device memory (needed for the 125 GB config,
 * which cannot be staged through host RAM).  Built with -fmad=false so every
 * value is bit-identical to the host generator.  Holds no H-matvec arithmetic.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include "hgen.h"

namespace {

__global__ void fill_rowmajor_kernel(uint64_t st, int is_x, int64_t row_begin, int64_t nrows,
                                     int64_t ncols_total, int64_t col_begin, int64_t ncols, double scale,
                                     double* out, int64_t ld) {
  int64_t total = nrows * ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t rr = e / ncols, col = e - rr * ncols;
    uint64_t idx = (uint64_t)((row_begin + rr) * ncols_total + col_begin + col);
    out[rr * ld + col] = is_x ? hgen_uniform11(st, idx) : hgen_normal(st, idx) * scale;
  }
}

__global__ void fill_x_kernel(uint64_t st, int64_t N, int64_t row_begin, int64_t nrows, int nrhs,
                              double* out, int64_t ld) {
  int64_t total = nrows * nrhs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t col = e / nrows, rr = e - col * nrows;
    out[col * ld + rr] = hgen_uniform11(st, (uint64_t)(col * N + row_begin + rr));
  }
}

int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

extern "C" {

/* Device twin of hgen_fill_rowmajor: out is a device pointer, ld in doubles. */
int hgen_dev_fill_rowmajor(uint64_t seed, int tag, int level, uint64_t vec, int64_t row_begin,
                           int64_t row_end, int64_t ncols, double scale, double* out, int64_t ld,
                           void* stream) {
  int64_t nrows = row_end - row_begin;
  if (nrows <= 0 || ncols <= 0) return 0;
  uint64_t st = hgen_stream(seed, (uint64_t)tag, (uint64_t)level, vec);
  fill_rowmajor_kernel<<<grid_for(nrows * ncols), 256, 0, (cudaStream_t)stream>>>(
      st, tag == HGEN_TAG_X, row_begin, nrows, ncols, 0, ncols, scale, out, ld);
  return (int)cudaGetLastError();
}

/* Columns [col_begin, col_begin + ncols) of a canonical panel with ncols_total
 * columns (e.g. one neighbour block of the standard-admissibility dense panel). */
int hgen_dev_fill_cols(uint64_t seed, int tag, int level, uint64_t vec, int64_t row_begin, int64_t row_end,
                       int64_t ncols_total, int64_t col_begin, int64_t ncols, double scale, double* out,
                       int64_t ld, void* stream) {
  int64_t nrows = row_end - row_begin;
  if (nrows <= 0 || ncols <= 0) return 0;
  uint64_t st = hgen_stream(seed, (uint64_t)tag, (uint64_t)level, vec);
  fill_rowmajor_kernel<<<grid_for(nrows * ncols), 256, 0, (cudaStream_t)stream>>>(
      st, tag == HGEN_TAG_X, row_begin, nrows, ncols_total, col_begin, ncols, scale, out, ld);
  return (int)cudaGetLastError();
}

/* Device twin of hgen_fill_x. */
int hgen_dev_fill_x(uint64_t seed, uint64_t vec, int64_t N, int64_t row_begin, int64_t row_end,
                    int nrhs, double* out, int64_t ld, void* stream) {
  int64_t nrows = row_end - row_begin;
  if (nrows <= 0 || nrhs <= 0) return 0;
  uint64_t st = hgen_stream(seed, HGEN_TAG_X, 0, vec);
  fill_x_kernel<<<grid_for(nrows * nrhs), 256, 0, (cudaStream_t)stream>>>(st, N, row_begin, nrows,
                                                                           nrhs, out, ld);
  return (int)cudaGetLastError();
}

}  // extern "C"
