/*
 * hgen_host.c -- host side of the seeded input generator (gen/hgen.h).
 * TEST/BENCH INFRASTRUCTURE: fills canonical panels with the synthetic inputs
 * of DESIGN.md §3; none of the H-matvec arithmetic lives here.
 * Build: gcc -O2 -fopenmp -ffp-contract=off (no fma, no contraction), so the
 * bits equal those of gen/hgen_device.cu (nvcc -fmad=false).
 */
#include <math.h>
#include <stdint.h>
#include "hgen.h"

/* Value of element idx of the stream (seed, tag, level, vec).  X draws are
 * U(-1,1); U, V, D draws are N(0,1) * scale. */
double hgen_value(uint64_t seed, int tag, int level, uint64_t vec, uint64_t idx, double scale) {
  uint64_t st = hgen_stream(seed, (uint64_t)tag, (uint64_t)level, vec);
  if (tag == HGEN_TAG_X) return hgen_uniform11(st, idx);
  return hgen_normal(st, idx) * scale;
}

/* Rows [row_begin,row_end) of a canonical row-major panel with ncols columns:
 * out[(row-row_begin)*ld + col] = value(idx = row*ncols + col). */
void hgen_fill_rowmajor(uint64_t seed, int tag, int level, uint64_t vec,
                        int64_t row_begin, int64_t row_end, int64_t ncols,
                        double scale, double* out, int64_t ld) {
  uint64_t st = hgen_stream(seed, (uint64_t)tag, (uint64_t)level, vec);
#pragma omp parallel for schedule(static)
  for (int64_t row = row_begin; row < row_end; ++row) {
    double* o = out + (row - row_begin) * ld;
    for (int64_t col = 0; col < ncols; ++col) {
      uint64_t idx = (uint64_t)(row * ncols + col);
      o[col] = (tag == HGEN_TAG_X) ? hgen_uniform11(st, idx) : hgen_normal(st, idx) * scale;
    }
  }
}

/* Rows [row_begin,row_end) of the N x nrhs column-major x block of timing
 * vector `vec`: out[col*ld + (row-row_begin)] = U(-1,1) draw idx = col*N + row. */
void hgen_fill_x(uint64_t seed, uint64_t vec, int64_t N, int64_t row_begin, int64_t row_end,
                 int nrhs, double* out, int64_t ld) {
  uint64_t st = hgen_stream(seed, HGEN_TAG_X, 0, vec);
  for (int col = 0; col < nrhs; ++col) {
#pragma omp parallel for schedule(static)
    for (int64_t row = row_begin; row < row_end; ++row)
      out[(int64_t)col * ld + (row - row_begin)] = hgen_uniform11(st, (uint64_t)((int64_t)col * N + row));
  }
}

/* Exposed for the distribution tests. */
double hgen_log_host(double u) { return hgen_log(u); }
double hgen_cos2pi_host(double u) { return hgen_cos2pi(u); }
