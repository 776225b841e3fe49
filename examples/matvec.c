/*
 * matvec.c -- the C ABI from plain C (no C++, no torch): build a small weak-
 * admissibility H-matrix from host panels, multiply host vectors, check two
 * properties that need no reference implementation, print the result.
 *
 *   make && gcc -std=c99 -O2 -Iinclude examples/matvec.c \
 *        -Lpaper_2008_12441_b200 -lhmat -Wl,-rpath,$PWD/paper_2008_12441_b200 -lm -o matvec
 *   ./matvec            (needs a B200)
 *
 * Checks: linearity H(2x + x') = 2Hx + Hx' (every product is linear in x), and
 * the dense part alone: with U = V = 0 the product is the block-diagonal D x
 * (eq:hmat-vec-add), computed here by hand.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hmat.h"

#define CHECK(call)                                                         \
  do {                                                                      \
    hmat_status st_ = (call);                                               \
    if (st_ != HMAT_OK) {                                                   \
      fprintf(stderr, "%s failed (%d): %s\n", #call, st_, hmat_last_error()); \
      return 1;                                                             \
    }                                                                       \
  } while (0)

static double urand(uint64_t* s) { /* xorshift64*, uniform in [-1, 1) */
  *s ^= *s >> 12;
  *s ^= *s << 25;
  *s ^= *s >> 27;
  return (double)((*s * 2685821657736338717ull) >> 11) * 0x1.0p-52 - 1.0;
}

int main(void) {
  const int dim = 2, depth = 3, leaf = 16, rank = 4;
  const int c = 1 << dim, W = (c - 1) * rank;
  int64_t N = leaf;
  for (int l = 0; l < depth; ++l) N *= c;
  uint64_t seed = 88172645463325252ull;
  double* U[3];
  double* V[3];
  double* Z[3];  /* zero panels */
  for (int l = 0; l < depth; ++l) {
    U[l] = malloc(sizeof(double) * N * W);
    V[l] = malloc(sizeof(double) * N * W);
    Z[l] = calloc((size_t)(N * W), sizeof(double));
    for (int64_t i = 0; i < N * W; ++i) {
      U[l][i] = 0.1 * urand(&seed);
      V[l][i] = 0.1 * urand(&seed);
    }
  }
  double* D = malloc(sizeof(double) * N * leaf);
  for (int64_t i = 0; i < N * leaf; ++i) D[i] = urand(&seed) / 8;
  double *x = malloc(sizeof(double) * N), *x2 = malloc(sizeof(double) * N), *xc = malloc(sizeof(double) * N);
  double *y = malloc(sizeof(double) * N), *y2 = malloc(sizeof(double) * N), *yc = malloc(sizeof(double) * N);
  for (int64_t i = 0; i < N; ++i) {
    x[i] = urand(&seed);
    x2[i] = urand(&seed);
    xc[i] = 2 * x[i] + x2[i];
  }

  hmat_t H = NULL, H0 = NULL;
  CHECK(hmat_create(depth, dim, leaf, rank, (const double* const*)U, (const double* const*)V, D, NULL, &H));
  CHECK(hmat_matvec(H, x, y, 1)); /* host pointers: returns with y complete */
  CHECK(hmat_matvec(H, x2, y2, 1));
  CHECK(hmat_matvec(H, xc, yc, 1));
  double err = 0, nrm = 0;
  for (int64_t i = 0; i < N; ++i) {
    err = fmax(err, fabs(yc[i] - (2 * y[i] + y2[i])));
    nrm = fmax(nrm, fabs(yc[i]));
  }
  printf("N = %lld, |H(2x+x') - (2Hx+Hx')|_max / |.|_max = %.2e\n", (long long)N, err / nrm);

  /* U = V = 0: only the leaf-diagonal blocks remain */
  CHECK(hmat_create(depth, dim, leaf, rank, (const double* const*)Z, (const double* const*)Z, D, NULL, &H0));
  CHECK(hmat_matvec(H0, x, y, 1));
  double derr = 0;
  for (int64_t i = 0; i < N; ++i) {
    const int64_t k = i / leaf;
    double acc = 0;
    for (int j = 0; j < leaf; ++j) acc += D[i * leaf + j] * x[k * leaf + j];
    derr = fmax(derr, fabs(y[i] - acc));
  }
  printf("dense part alone: max |y - D x| = %.2e\n", derr);
  CHECK(hmat_destroy(H));
  CHECK(hmat_destroy(H0));
  const int ok = err / nrm < 1e-13 && derr < 1e-13;
  printf("%s\n", ok ? "ok" : "FAILED");
  return ok ? 0 : 1;
}
