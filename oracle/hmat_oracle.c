/*
 * hmat_oracle.c -- the CPU ORACLE for the weak-admissibility H-matvec y = Hx.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code with the CUDA path (paper_2008_12441_b200/csrc); its only
 * shared dependency is the seeded input generator gen/hgen.h, used by
 * oracle_rows_generated() and the generated form of oracle_matvec_rows_par()
 * to produce factor entries on demand (full-size operators without factor
 * memory).  oracle_matvec_rows_par() is also the all-cores block loop timed as
 * the CPU baseline; it is bit-identical to oracle_matvec().
 *
 * Plain, slow, obviously correct fp64 loops, written from the paper:
 *   - structure: Def 2.4 (\label{def:hmat}) on the 2^d-ary
 *     domain tree of an ideal domain under weak
 *     admissibility, BASELINE variant (DESIGN.md reading
 *     R1): every pair of distinct siblings at levels 1..L is a rank-r block
 *     U_ts V_ts^T, only leaf-diagonal blocks are dense;
 *   - matvec: y = 0, then for every block y_t += D x_s or y_t += U (V^T x_s),
 *     eq:hmat-vec-add.
 * Built with gcc -O2 -ffp-contract=off (no contraction; R11).
 *
 * Canonical panel layout (the C-ABI's input format):
 *   c = 2^d, N = b c^L, m_l = N / c^l, W = (c-1) r, all row-major, Morton rows.
 *   U_l (N x W): row i, columns [q r, (q+1) r) = row i - t m_l of U_{t, s_q},
 *                t = i / m_l, s_q = q-th sibling of t (ascending, skip self).
 *   V_l (N x W): row j, columns [q r, (q+1) r) = row j - s m_l of V_{t_q, s},
 *                s = j / m_l, t_q = q-th sibling of s.
 *   D   (N x b): row i = row i - k b of D_k, k = i / b.
 *   x, y: N x nrhs column-major, leading dimension N.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "../gen/hgen.h"

/* ---- tree / sibling indexing (R6) ---------- */

/* q-th sibling of node t (siblings of t = the other children of t's parent,
 * in ascending child order, skipping t itself). */
int64_t oracle_sibling(int c, int64_t t, int q) {
  int64_t parent = t / c;
  int me = (int)(t % c);
  int child = q < me ? q : q + 1;
  return parent * c + child;
}

/* slot of sibling s in t's sibling list: the q with oracle_sibling(t,q) = s. */
int oracle_slot(int c, int64_t t, int64_t s) {
  for (int q = 0; q < c - 1; ++q)
    if (oracle_sibling(c, t, q) == s) return q;
  return -1;
}

static int64_t ipow(int64_t a, int e) {
  int64_t p = 1;
  while (e-- > 0) p *= a;
  return p;
}

/* ---- block enumeration by recursion on Def 2.4 -------------------------
 * Visits the H-matrix structure of K on Omega x Omega: starting from the root
 * pair (both domains are the root, level 0), each child pair (t, s) at level
 * l+1 of a hierarchical pair is
 *   - admissible (t != s, disjoint domains)  -> low-rank block (kind 1),
 *   - else (t == s) if l+1 == L (leaf)       -> dense block     (kind 0),
 *   - else                                   -> hierarchical, recurse.
 * The callback receives (kind, level, t, s). */
typedef void (*block_fn)(void* ctx, int kind, int level, int64_t t, int64_t s);

static void visit(int c, int L, int level, int64_t node, block_fn fn, void* ctx) {
  /* node is a diagonal (hierarchical) pair (node, node) at `level` */
  for (int a = 0; a < c; ++a) {
    for (int bb = 0; bb < c; ++bb) {
      int64_t t = node * c + a, s = node * c + bb;
      if (t != s) fn(ctx, 1, level + 1, t, s);
      else if (level + 1 == L) fn(ctx, 0, level + 1, t, s);
      else visit(c, L, level + 1, t, fn, ctx);
    }
  }
}

static void visit_root(int c, int L, block_fn fn, void* ctx) {
  if (L == 0) fn(ctx, 0, 0, 0, 0); /* the root is a leaf: one dense block */
  else visit(c, L, 0, 0, fn, ctx);
}

/* The paper-strict reading of Def 2.4 (R1): the three
 * conditions checked in the paper's order -- (1) a child pair whose domains are
 * leaves is dense, (2) else an admissible pair is low rank, (3) else recurse.
 * So every child pair of a leaf-parent is a dense b x b block. */
static void visit_strict(int c, int L, int level, int64_t node, block_fn fn, void* ctx) {
  for (int a = 0; a < c; ++a) {
    for (int bb = 0; bb < c; ++bb) {
      int64_t t = node * c + a, s = node * c + bb;
      if (level + 1 == L) fn(ctx, 0, level + 1, t, s);   /* leaves: dense */
      else if (t != s) fn(ctx, 1, level + 1, t, s);      /* admissible: low rank */
      else visit_strict(c, L, level + 1, t, fn, ctx);    /* hierarchical */
    }
  }
}

static void visit_root_v(int strict, int c, int L, block_fn fn, void* ctx) {
  if (L == 0) fn(ctx, 0, 0, 0, 0);
  else if (strict) visit_strict(c, L, 0, 0, fn, ctx);
  else visit(c, L, 0, 0, fn, ctx);
}

typedef struct { int64_t lowrank, dense, lowrank_level1; } census_t;

static void census_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  census_t* cs = (census_t*)ctx;
  (void)t; (void)s;
  if (kind == 1) { cs->lowrank++; if (level == 1) cs->lowrank_level1++; }
  else cs->dense++;
}

/* Counts blocks by walking the structure (not by formula). */
void oracle_block_census(int d, int L, int64_t* n_lowrank, int64_t* n_dense, int64_t* n_lowrank_level1) {
  census_t cs = {0, 0, 0};
  visit_root(1 << d, L, census_cb, &cs);
  *n_lowrank = cs.lowrank; *n_dense = cs.dense; *n_lowrank_level1 = cs.lowrank_level1;
}

typedef struct { int c, L, b; int64_t N; int32_t* count; } cover_t;

static void cover_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  cover_t* cv = (cover_t*)ctx;
  (void)kind;
  int64_t m = cv->N / ipow(cv->c, level);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) cv->count[(t * m + i) * cv->N + (s * m + j)] += 1;
}

/* count[i*N + j] = number of blocks covering entry (i, j) (must be 1). */
void oracle_cover_count_v(int strict, int d, int L, int b, int32_t* count) {
  cover_t cv;
  cv.c = 1 << d; cv.L = L; cv.b = b; cv.N = (int64_t)b * ipow(cv.c, L); cv.count = count;
  memset(count, 0, sizeof(int32_t) * (size_t)(cv.N * cv.N));
  visit_root_v(strict, cv.c, L, cover_cb, &cv);
}

void oracle_cover_count(int d, int L, int b, int32_t* count) { oracle_cover_count_v(0, d, L, b, count); }

void oracle_block_census_strict(int d, int L, int64_t* n_lowrank, int64_t* n_dense, int64_t* n_lowrank_level1) {
  census_t cs = {0, 0, 0};
  visit_root_v(1, 1 << d, L, census_cb, &cs);
  *n_lowrank = cs.lowrank; *n_dense = cs.dense; *n_lowrank_level1 = cs.lowrank_level1;
}

/* ---- the matvec, eq:hmat-vec-add ----------------------------------------
 * y = 0; for every dense block D_k: y_k += D_k x_k; for
 * every low-rank block (t, s) at level l: z = V_ts^T x_s, y_t += U_ts z.
 * level_mask bit (l-1) selects level l; dense selects the leaf blocks (test
 * hook for the per-level decomposition y = y_D + sum_l y_l). */
void oracle_matvec_masked(int d, int L, int b, int r, const double* const* U, const double* const* V,
                          const double* D, const double* x, double* y, int nrhs,
                          uint64_t level_mask, int dense) {
  const int c = 1 << d;
  const int64_t N = (int64_t)b * ipow(c, L);
  const int W = (c - 1) * r;
  double* z = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int k = 0; k < nrhs; ++k) {
    const double* xk = x + (int64_t)k * N;
    double* yk = y + (int64_t)k * N;
    for (int64_t i = 0; i < N; ++i) yk[i] = 0.0;
    if (dense) {
      for (int64_t leaf = 0; leaf < N / b; ++leaf)
        for (int i = 0; i < b; ++i)
          for (int j = 0; j < b; ++j)
            yk[leaf * b + i] += D[(leaf * b + i) * b + j] * xk[leaf * b + j];
    }
    for (int l = 1; l <= L; ++l) {
      if (!((level_mask >> (l - 1)) & 1ull)) continue;
      const int64_t m = N / ipow(c, l);
      const double* Ul = U[l - 1];
      const double* Vl = V[l - 1];
      for (int64_t t = 0; t < ipow(c, l); ++t) {
        for (int q = 0; q < c - 1; ++q) {
          int64_t s = oracle_sibling(c, t, q); /* block (t, s) */
          int qs = oracle_slot(c, s, t);        /* t's slot in s's list: V_ts columns */
          for (int a = 0; a < r; ++a) z[a] = 0.0;
          for (int64_t j = 0; j < m; ++j)       /* z = V_ts^T x_s */
            for (int a = 0; a < r; ++a)
              z[a] += Vl[(s * m + j) * W + qs * r + a] * xk[s * m + j];
          for (int64_t i = 0; i < m; ++i)       /* y_t += U_ts z */
            for (int a = 0; a < r; ++a)
              yk[t * m + i] += Ul[(t * m + i) * W + q * r + a] * z[a];
        }
      }
    }
  }
  free(z);
}

void oracle_matvec(int d, int L, int b, int r, const double* const* U, const double* const* V,
                   const double* D, const double* x, double* y, int nrhs) {
  oracle_matvec_masked(d, L, b, r, U, V, D, x, y, nrhs, ~0ull, 1);
}

/* ---- the transposed product H^T x (GEMV "T", PAPER.md:961-969 remark) ------
 * Every block contributes its transpose: for a dense D_k, y_k += D_k^T x_k; for
 * a low-rank block (t, s): w = U_ts^T x_t, y_s += V_ts w. */
void oracle_matvec_t(int d, int L, int b, int r, const double* const* U, const double* const* V,
                     const double* D, const double* x, double* y, int nrhs) {
  const int c = 1 << d;
  const int64_t N = (int64_t)b * ipow(c, L);
  const int W = (c - 1) * r;
  double* w = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int k = 0; k < nrhs; ++k) {
    const double* xk = x + (int64_t)k * N;
    double* yk = y + (int64_t)k * N;
    for (int64_t i = 0; i < N; ++i) yk[i] = 0.0;
    for (int64_t leaf = 0; leaf < N / b; ++leaf)
      for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j)
          yk[leaf * b + j] += D[(leaf * b + i) * b + j] * xk[leaf * b + i];
    for (int l = 1; l <= L; ++l) {
      const int64_t m = N / ipow(c, l);
      const double* Ul = U[l - 1];
      const double* Vl = V[l - 1];
      for (int64_t t = 0; t < ipow(c, l); ++t) {
        for (int q = 0; q < c - 1; ++q) {
          int64_t s = oracle_sibling(c, t, q);
          int qs = oracle_slot(c, s, t);
          for (int a = 0; a < r; ++a) w[a] = 0.0;
          for (int64_t i = 0; i < m; ++i)       /* w = U_ts^T x_t */
            for (int a = 0; a < r; ++a)
              w[a] += Ul[(t * m + i) * W + q * r + a] * xk[t * m + i];
          for (int64_t j = 0; j < m; ++j)       /* y_s += V_ts w */
            for (int a = 0; a < r; ++a)
              yk[s * m + j] += Vl[(s * m + j) * W + qs * r + a] * w[a];
        }
      }
    }
  }
  free(w);
}

/* ---- paper-strict structure (f2): dense leaf-parent blocks ------------------
 * U, V hold levels 1..L-1 (canonical layout); Dc is N x (c b): row i of
 * leaf-parent p = i / (c b) holds row i - p c b of the dense (c b) x (c b)
 * diagonal block of p, i.e. the c dense leaf blocks D_{t,s} of t's row. */
void oracle_matvec_strict(int d, int L, int b, int r, const double* const* U, const double* const* V,
                          const double* Dc, const double* x, double* y, int nrhs) {
  const int c = 1 << d;
  const int64_t N = (int64_t)b * ipow(c, L);
  const int W = (c - 1) * r;
  const int cb = (L >= 1 ? c : 1) * b;  /* L = 0: the root is a leaf (b x b) */
  double* z = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int k = 0; k < nrhs; ++k) {
    const double* xk = x + (int64_t)k * N;
    double* yk = y + (int64_t)k * N;
    for (int64_t i = 0; i < N; ++i) yk[i] = 0.0;
    /* dense blocks: every child pair (t, s) of each leaf-parent */
    for (int64_t p = 0; p < N / cb; ++p)
      for (int64_t i = 0; i < cb; ++i)
        for (int64_t j = 0; j < cb; ++j)
          yk[p * cb + i] += Dc[(p * cb + i) * cb + j] * xk[p * cb + j];
    for (int l = 1; l <= L - 1; ++l) {
      const int64_t m = N / ipow(c, l);
      const double* Ul = U[l - 1];
      const double* Vl = V[l - 1];
      for (int64_t t = 0; t < ipow(c, l); ++t) {
        for (int q = 0; q < c - 1; ++q) {
          int64_t s = oracle_sibling(c, t, q);
          int qs = oracle_slot(c, s, t);
          for (int a = 0; a < r; ++a) z[a] = 0.0;
          for (int64_t j = 0; j < m; ++j)
            for (int a = 0; a < r; ++a) z[a] += Vl[(s * m + j) * W + qs * r + a] * xk[s * m + j];
          for (int64_t i = 0; i < m; ++i)
            for (int a = 0; a < r; ++a) yk[t * m + i] += Ul[(t * m + i) * W + q * r + a] * z[a];
        }
      }
    }
  }
  free(z);
}

/* ---- dense assembly + brute-force matvec (small N) --------------------- */

typedef struct {
  int c, L, b, r, W, strict; int64_t N;
  const double* const* U; const double* const* V; const double* D; double* A;
} assemble_t;

static void assemble_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  assemble_t* as = (assemble_t*)ctx;
  const int64_t N = as->N;
  if (kind == 0 && !as->strict) { /* dense leaf block D_t, t == s */
    for (int i = 0; i < as->b; ++i)
      for (int j = 0; j < as->b; ++j)
        as->A[(t * as->b + i) * N + (s * as->b + j)] = as->D[(t * as->b + i) * as->b + j];
    return;
  }
  if (kind == 0) { /* strict: dense leaf-pair block D_ts from the leaf-parent panel */
    const int cb = (as->L >= 1 ? as->c : 1) * as->b;
    const int64_t p0 = (t * as->b) / cb * cb; /* first row of the leaf-parent */
    for (int i = 0; i < as->b; ++i)
      for (int j = 0; j < as->b; ++j)
        as->A[(t * as->b + i) * N + (s * as->b + j)] = as->D[(t * as->b + i) * cb + (s * as->b - p0) + j];
    return;
  }
  const int64_t m = N / ipow(as->c, level);
  const int q = oracle_slot(as->c, t, s), qs = oracle_slot(as->c, s, t);
  const double* Ul = as->U[level - 1];
  const double* Vl = as->V[level - 1];
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) {
      double acc = 0.0; /* (U_ts V_ts^T)[i, j] */
      for (int a = 0; a < as->r; ++a)
        acc += Ul[(t * m + i) * as->W + q * as->r + a] * Vl[(s * m + j) * as->W + qs * as->r + a];
      as->A[(t * m + i) * N + (s * m + j)] = acc;
    }
}

/* A (N x N row-major) = the matrix the blocks define. */
void oracle_assemble_v(int strict, int d, int L, int b, int r, const double* const* U, const double* const* V,
                       const double* D, double* A) {
  assemble_t as;
  as.c = 1 << d; as.L = L; as.b = b; as.r = r; as.W = (as.c - 1) * r; as.strict = strict;
  as.N = (int64_t)b * ipow(as.c, L);
  as.U = U; as.V = V; as.D = D; as.A = A;
  memset(A, 0, sizeof(double) * (size_t)(as.N * as.N));
  visit_root_v(strict, as.c, L, assemble_cb, &as);
}

void oracle_assemble(int d, int L, int b, int r, const double* const* U, const double* const* V,
                     const double* D, double* A) {
  oracle_assemble_v(0, d, L, b, r, U, V, D, A);
}

/* y = A x by the definition of a matrix-vector product (brute force). */
void oracle_dense_matvec(int64_t N, const double* A, const double* x, double* y, int nrhs) {
  for (int k = 0; k < nrhs; ++k)
    for (int64_t i = 0; i < N; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < N; ++j) acc += A[i * N + j] * x[(int64_t)k * N + j];
      y[(int64_t)k * N + i] = acc;
    }
}

/* ---- the block loop on all host cores (SURVEY §8(d) "oracle_allcores") ----
 * The arithmetic of oracle_matvec_masked (eq:hmat-vec-add),
 * element for element in the same order, so the output is BIT-IDENTICAL to the
 * one-thread block loop for any thread count:
 *   y_i = 0;  y_i += D_k[i, j] x_{k b + j}  for j = 0..b-1          (dense leaf)
 *   for l = 1..L, q = 0..c-2, a = 0..r-1:  y_i += U_{t,s_q}[i, a] z_{t,q}[a]
 *   with z_{t,q}[a] = sum_{j = 0..m-1} V_{t,s_q}[j, a] x_{s_q m + j}  (V_ts^T x_s)
 * Only the distribution of the work over threads differs: per level, (A) every
 * z_{t,q}[a] of the level's targets is an independent dot product (one thread
 * each), then (B) every row i adds its sum over q and a.  Rows [r0, r1) of y
 * only (an aligned shard, a chunk); y is (r1 - r0) x nrhs column-major with
 * leading dimension ldy, x the full N x nrhs block (ld N).
 * Factor entries come from the canonical panels (U, V, D non-NULL) or, with
 * U == NULL, straight from the seeded generator (gen/hgen.h):
 * U_l / V_l entry (row, col) = normal(stream(seed, U|V, l), row W + col) / sqrt(m_l),
 * D entry (row, col) = normal(stream(seed, D, 0), row b + col) / 8 -- the values
 * hgen_fill_rowmajor writes, so both sources give the same y bits.  The
 * generated form needs no factor memory: full-size operators (124.55 GB at
 * BASELINE configs[3]) are checked in full on the host. */
#define ORACLE_ZCAP ((int64_t)1 << 25) /* doubles of z per target chunk (256 MB) */

void oracle_matvec_rows_par(int d, int L, int b, int r, const double* const* U, const double* const* V,
                            const double* D, uint64_t seed, const double* x, int nrhs, int64_t r0, int64_t r1,
                            double* y, int64_t ldy, uint64_t level_mask, int dense, int nthreads) {
  const int c = 1 << d;
  const int64_t N = (int64_t)b * ipow(c, L);
  const int W = (c - 1) * r;
  const int gen = (U == NULL);
  const int nt = nthreads > 0 ? nthreads : 1;
  const uint64_t stD = hgen_stream(seed, HGEN_TAG_D, 0, 0);
  if (r1 <= r0) return;
  /* x and y with the right-hand sides innermost (xr[j nrhs + k], yr[(i - r0) nrhs + k]):
   * a data layout only -- column-major blocks put the nrhs values of one row
   * N doubles apart, on the same cache set */
  const int64_t nl = r1 - r0;
  double* xr = (double*)malloc(sizeof(double) * (size_t)N * (size_t)nrhs);
  double* yr = (double*)malloc(sizeof(double) * (size_t)nl * (size_t)nrhs);
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t j = 0; j < N; ++j)
    for (int k = 0; k < nrhs; ++k) xr[j * nrhs + k] = x[(int64_t)k * N + j];
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t i = r0; i < r1; ++i) { /* y = 0, then the dense leaf block */
    const int64_t leaf = i / b;
    double* yi = yr + (i - r0) * nrhs;
    for (int k = 0; k < nrhs; ++k) yi[k] = 0.0;
    if (!dense) continue;
    for (int j = 0; j < b; ++j) {
      const double dv = gen ? hgen_normal(stD, (uint64_t)(i * b + j)) * 0.125 : D[i * b + j];
      const double* xj = xr + (leaf * b + j) * nrhs;
      for (int k = 0; k < nrhs; ++k) yi[k] += dv * xj[k];
    }
  }
  const int64_t per_t = (int64_t)W * nrhs; /* z doubles per target: [q][a][k] */
  double* Z = (double*)malloc(sizeof(double) * (size_t)(per_t < ORACLE_ZCAP ? ORACLE_ZCAP : per_t));
  for (int l = 1; l <= L; ++l) {
    if (!((level_mask >> (l - 1)) & 1ull)) continue;
    const int64_t m = N / ipow(c, l);
    const double scale = 1.0 / sqrt((double)m);
    const uint64_t stU = hgen_stream(seed, HGEN_TAG_U, (uint64_t)l, 0);
    const uint64_t stV = hgen_stream(seed, HGEN_TAG_V, (uint64_t)l, 0);
    const double* Ul = gen ? NULL : U[l - 1];
    const double* Vl = gen ? NULL : V[l - 1];
    const int64_t t_lo = r0 / m, t_hi = (r1 - 1) / m + 1;
    int64_t chunk = ORACLE_ZCAP / per_t;
    if (chunk < 1) chunk = 1;
    for (int64_t tc = t_lo; tc < t_hi; tc += chunk) {
      const int64_t te = tc + chunk < t_hi ? tc + chunk : t_hi;
      const int64_t items = (te - tc) * (c - 1) * r;
      /* (A) z_{t,q}[a] = V_{t,s_q}[:, a]^T x_{s_q}, one dot product per item */
#pragma omp parallel for num_threads(nt) schedule(dynamic, 1)
      for (int64_t it = 0; it < items; ++it) {
        const int64_t t = tc + it / ((int64_t)(c - 1) * r);
        const int q = (int)((it / r) % (c - 1));
        const int a = (int)(it % r);
        const int64_t s = oracle_sibling(c, t, q); /* block (t, s) */
        const int qs = oracle_slot(c, s, t);       /* t's slot in s's list: V_ts columns */
        double* z = Z + (((t - tc) * (c - 1) + q) * r + a) * (int64_t)nrhs;
        for (int k = 0; k < nrhs; ++k) z[k] = 0.0;
        for (int64_t j = 0; j < m; ++j) {
          const int64_t idx = (s * m + j) * W + qs * r + a;
          const double v = gen ? hgen_normal(stV, (uint64_t)idx) * scale : Vl[idx];
          const double* xj = xr + (s * m + j) * nrhs;
          for (int k = 0; k < nrhs; ++k) z[k] += v * xj[k];
        }
      }
      /* (B) y_i += U_{t,s_q}[i, :] z_{t,q} for every row of these targets */
      const int64_t i_lo = tc * m > r0 ? tc * m : r0, i_hi = te * m < r1 ? te * m : r1;
#pragma omp parallel for num_threads(nt) schedule(static)
      for (int64_t i = i_lo; i < i_hi; ++i) {
        const int64_t t = i / m;
        double* yi = yr + (i - r0) * nrhs;
        for (int q = 0; q < c - 1; ++q)
          for (int a = 0; a < r; ++a) {
            const int64_t idx = i * W + q * r + a;
            const double u = gen ? hgen_normal(stU, (uint64_t)idx) * scale : Ul[idx];
            const double* z = Z + (((t - tc) * (c - 1) + q) * r + a) * (int64_t)nrhs;
            for (int k = 0; k < nrhs; ++k) yi[k] += u * z[k];
          }
      }
    }
  }
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t i = r0; i < r1; ++i)
    for (int k = 0; k < nrhs; ++k) y[(int64_t)k * ldy + (i - r0)] = yr[(i - r0) * nrhs + k];
  free(Z);
  free(xr);
  free(yr);
}

/* ---- sampled rows at any size, factors generated on demand ---------------
 * y[rows[n], :] for the H-matrix whose panels are the seeded synthetic inputs
 * (gen/hgen.h), computed row by row from eq:hmat-vec-add:
 *   y_i = sum_j D_k[i, j] x_{k b + j}
 *       + sum_l sum_q U_{t,s_q}[i, :] (V_{t,s_q}^T x_{s_q}),  t = i / m_l.
 * Only the factor entries these rows touch are generated.  The z vectors of
 * node t at level l are reused when consecutive sample rows share t; the sum
 * over j in V^T x may be split across OpenMP threads. */
void oracle_rows_generated(int d, int L, int b, int r, uint64_t seed, const double* x, int nrhs,
                           int64_t nrows, const int64_t* rows, double* yrows) {
  const int c = 1 << d;
  const int64_t N = (int64_t)b * ipow(c, L);
  const int W = (c - 1) * r;
  const uint64_t stD = hgen_stream(seed, HGEN_TAG_D, 0, 0);
  /* zc[l][(q * nrhs + k) * r + a] = (V_{t,s_q}^T x_{s_q, k})[a] for t = last_t[l] */
  double* zc = (double*)malloc(sizeof(double) * (size_t)(L + 1) * (size_t)W * (size_t)nrhs + 8);
  int64_t* last_t = (int64_t*)malloc(sizeof(int64_t) * (size_t)(L + 1));
  for (int l = 0; l <= L; ++l) last_t[l] = -1;
  for (int64_t n = 0; n < nrows; ++n) {
    const int64_t i = rows[n];
    const int64_t leaf = i / b;
    for (int k = 0; k < nrhs; ++k) {
      double acc = 0.0;
      for (int j = 0; j < b; ++j)
        acc += hgen_normal(stD, (uint64_t)(i * b + j)) * 0.125 * x[(int64_t)k * N + leaf * b + j];
      yrows[(int64_t)k * nrows + n] = acc;
    }
    for (int l = 1; l <= L; ++l) {
      const int64_t m = N / ipow(c, l);
      const double scale = 1.0 / sqrt((double)m);
      const uint64_t stU = hgen_stream(seed, HGEN_TAG_U, (uint64_t)l, 0);
      const uint64_t stV = hgen_stream(seed, HGEN_TAG_V, (uint64_t)l, 0);
      const int64_t t = i / m;
      double* z = zc + (size_t)l * (size_t)W * (size_t)nrhs;
      if (last_t[l] != t) {
        for (int q = 0; q < c - 1; ++q) {
          const int64_t s = oracle_sibling(c, t, q);
          const int qs = oracle_slot(c, s, t);
          for (int k = 0; k < nrhs; ++k)
            for (int a = 0; a < r; ++a) {
              double za = 0.0;
#pragma omp parallel for reduction(+ : za) schedule(static)
              for (int64_t j = 0; j < m; ++j)
                za += hgen_normal(stV, (uint64_t)((s * m + j) * W + qs * r + a)) * scale *
                      x[(int64_t)k * N + s * m + j];
              z[(q * nrhs + k) * r + a] = za;
            }
        }
        last_t[l] = t;
      }
      for (int q = 0; q < c - 1; ++q)
        for (int k = 0; k < nrhs; ++k) {
          double acc = 0.0;
          for (int a = 0; a < r; ++a)
            acc += hgen_normal(stU, (uint64_t)(i * W + q * r + a)) * scale * z[(q * nrhs + k) * r + a];
          yrows[(int64_t)k * nrows + n] += acc;
        }
    }
  }
  free(zc);
  free(last_t);
}

/* ===========================================================================
 * STANDARD admissibility: Def 2.4 with the standard admissibility
 * condition eq:standard-ad-cond, rho = sqrt(d), on the ideal
 * domain [0,1]^d with a non-periodic boundary (the paper's load-balance case,
 * PAPER.md:606-629; R17).
 *
 * A level-l node k is the box of side h = 2^-l with integer coordinates
 * (k decoded from Morton bits: bit j of coordinate i is bit j d + i of k).
 * Two level-l boxes with coordinate differences D_i have
 *   diam = sqrt(d) h,  dist = h sqrt(sum_i g_i^2),  g_i = max(0, |D_i| - 1),
 * so min(diam, diam) <= rho dist  <=>  d h^2 <= d h^2 sum_i g_i^2
 *                                 <=>  sum_i g_i^2 >= 1   (exact integers).
 *
 * Canonical panels (the input format of hmat_create_standard):
 *   M = 6^d - 3^d slots per node: for target t (child position tau of its
 *   parent) the candidate sources s are the children sigma of the parent's
 *   3^d neighbours eps in {-1,0,1}^d; slots enumerate the pairs (eps, sigma)
 *   in increasing order of (sum_i (eps_i+1) 3^i) 2^d + sum_i sigma_i 2^i,
 *   skipping those where s is a neighbour of t; pairs outside the domain keep
 *   their slot (zero factors).
 *   U_l row i, columns [q r, (q+1) r): row i - t m_l of U_{t,s}, s = slot q of t.
 *   V_l row j, columns [q r, (q+1) r): row j - s m_l of V_{t,s}, t = slot q of s.
 *   Dn row i (leaf t), columns [e b, (e+1) b): row i - t b of D_{t,s},
 *   s = t + eps, e = sum_i (eps_i + 1) 3^i (neighbours incl. t; zero if absent).
 * =========================================================================*/

static void morton_decode(int d, int64_t k, int level, int64_t* x) {
  for (int i = 0; i < d; ++i) x[i] = 0;
  for (int j = 0; j < level; ++j)
    for (int i = 0; i < d; ++i) x[i] |= ((k >> (j * d + i)) & 1) << j;
}

/* standard admissibility of two level-l boxes (eq:standard-ad-cond, rho = sqrt(d)) */
static int std_admissible(int d, const int64_t* xt, const int64_t* xs) {
  int64_t sum_g2 = 0;
  for (int i = 0; i < d; ++i) {
    int64_t D = xt[i] - xs[i];
    if (D < 0) D = -D;
    int64_t g = D - 1 > 0 ? D - 1 : 0;
    sum_g2 += g * g;
  }
  return d * 1 <= d * sum_g2; /* diam^2 <= rho^2 dist^2, both divided by h^2 */
}

static int std_neighbour(int d, const int64_t* xt, const int64_t* xs) {
  for (int i = 0; i < d; ++i) {
    int64_t D = xt[i] - xs[i];
    if (D < -1 || D > 1) return 0;
  }
  return 1;
}

int oracle_std_slots(int d) {
  int p6 = 1, p3 = 1;
  for (int i = 0; i < d; ++i) { p6 *= 6; p3 *= 3; }
  return p6 - p3;
}

/* slot of source s in target t's list (both at `level`), -1 if s is not a
 * candidate (its parent is not a neighbour of t's parent, or s neighbours t). */
int oracle_std_slot(int d, int level, int64_t t, int64_t s) {
  int64_t xt[3], xs[3];
  morton_decode(d, t, level, xt);
  morton_decode(d, s, level, xs);
  int64_t eps_t[3], sig_t[3];
  for (int i = 0; i < d; ++i) {
    eps_t[i] = (xs[i] >> 1) - (xt[i] >> 1);
    sig_t[i] = xs[i] & 1;
    if (eps_t[i] < -1 || eps_t[i] > 1) return -1;
  }
  if (std_neighbour(d, xt, xs)) return -1;
  int c = 1 << d, p3 = 1;
  for (int i = 0; i < d; ++i) p3 *= 3;
  int target_code = 0, mul = 1, sc = 0;
  for (int i = 0; i < d; ++i) { target_code += (int)(eps_t[i] + 1) * mul; mul *= 3; }
  for (int i = 0; i < d; ++i) sc |= (int)sig_t[i] << i;
  target_code = target_code * c + sc;
  /* count valid (eps, sigma) pairs before target_code, for t's child position */
  int q = 0;
  for (int code = 0; code < target_code; ++code) {
    int e = code / c, sg = code % c, rem = e;
    int64_t xc[3];
    for (int i = 0; i < d; ++i) {
      int ei = rem % 3 - 1;
      rem /= 3;
      xc[i] = 2 * ((xt[i] >> 1) + ei) + ((sg >> i) & 1);
    }
    if (!std_neighbour(d, xt, xc)) ++q;
  }
  (void)p3;
  return q;
}

/* Def 2.4 recursion with standard admissibility over hierarchical pairs (P_t, P_s). */
static void visit_std(int d, int L, int level, int64_t pt, int64_t ps, block_fn fn, void* ctx) {
  const int c = 1 << d;
  for (int a = 0; a < c; ++a)
    for (int bb = 0; bb < c; ++bb) {
      int64_t t = pt * c + a, s = ps * c + bb;
      int64_t xt[3], xs[3];
      morton_decode(d, t, level + 1, xt);
      morton_decode(d, s, level + 1, xs);
      if (std_admissible(d, xt, xs)) fn(ctx, 1, level + 1, t, s);
      else if (level + 1 == L) fn(ctx, 0, level + 1, t, s);
      else visit_std(d, L, level + 1, t, s, fn, ctx);
    }
}

static void visit_root_std(int d, int L, block_fn fn, void* ctx) {
  if (L == 0) fn(ctx, 0, 0, 0, 0);
  else visit_std(d, L, 0, 0, 0, fn, ctx);
}

typedef struct { int64_t lowrank, dense; int level; int64_t target; int64_t target_lowrank; } std_census_t;

static void std_census_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  std_census_t* cs = (std_census_t*)ctx;
  (void)s;
  if (kind == 1) {
    cs->lowrank++;
    if (level == cs->level && t == cs->target) cs->target_lowrank++;
  } else {
    cs->dense++;
  }
}

/* totals, and the number of low-rank blocks of target `target` at `level` */
void oracle_std_census(int d, int L, int level, int64_t target, int64_t* n_lowrank, int64_t* n_dense,
                       int64_t* n_target) {
  std_census_t cs = {0, 0, level, target, 0};
  visit_root_std(d, L, std_census_cb, &cs);
  *n_lowrank = cs.lowrank; *n_dense = cs.dense; *n_target = cs.target_lowrank;
}

void oracle_std_cover_count(int d, int L, int b, int32_t* count) {
  cover_t cv;
  cv.c = 1 << d; cv.L = L; cv.b = b; cv.N = (int64_t)b * ipow(cv.c, L); cv.count = count;
  memset(count, 0, sizeof(int32_t) * (size_t)(cv.N * cv.N));
  visit_root_std(d, L, cover_cb, &cv);
}

static int std_neighbour_index(int d, int64_t t, int64_t s, int level) {
  int64_t xt[3], xs[3];
  morton_decode(d, t, level, xt);
  morton_decode(d, s, level, xs);
  int e = 0, mul = 1;
  for (int i = 0; i < d; ++i) { e += (int)(xs[i] - xt[i] + 1) * mul; mul *= 3; }
  return e;
}

typedef struct {
  int d, L, b, r, M, ND; int64_t N;
  const double* const* U; const double* const* V; const double* Dn; double* A;
} std_assemble_t;

static void std_assemble_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  std_assemble_t* as = (std_assemble_t*)ctx;
  const int64_t N = as->N;
  if (kind == 0) {
    const int e = std_neighbour_index(as->d, t, s, level);
    for (int i = 0; i < as->b; ++i)
      for (int j = 0; j < as->b; ++j)
        as->A[(t * as->b + i) * N + (s * as->b + j)] = as->Dn[(t * as->b + i) * (as->ND * as->b) + e * as->b + j];
    return;
  }
  const int64_t m = N / ipow(1 << as->d, level);
  const int qt = oracle_std_slot(as->d, level, t, s), qs = oracle_std_slot(as->d, level, s, t);
  const int W = as->M * as->r;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int a = 0; a < as->r; ++a)
        acc += as->U[level - 1][(t * m + i) * W + qt * as->r + a] * as->V[level - 1][(s * m + j) * W + qs * as->r + a];
      as->A[(t * m + i) * N + (s * m + j)] = acc;
    }
}

void oracle_std_assemble(int d, int L, int b, int r, const double* const* U, const double* const* V,
                         const double* Dn, double* A) {
  std_assemble_t as;
  as.d = d; as.L = L; as.b = b; as.r = r; as.M = oracle_std_slots(d);
  as.ND = (int)ipow(3, d); as.N = (int64_t)b * ipow(1 << d, L);
  as.U = U; as.V = V; as.Dn = Dn; as.A = A;
  memset(A, 0, sizeof(double) * (size_t)(as.N * as.N));
  visit_root_std(d, L, std_assemble_cb, &as);
}

/* y = H x, eq:hmat-vec-add over the standard-admissibility blocks */
typedef struct {
  int d, b, r, M, ND, nrhs; int64_t N;
  const double* const* U; const double* const* V; const double* Dn; const double* x; double* y; double* z;
} std_mv_t;

static void std_mv_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  std_mv_t* mv = (std_mv_t*)ctx;
  const int64_t N = mv->N;
  for (int k = 0; k < mv->nrhs; ++k) {
    const double* xk = mv->x + (int64_t)k * N;
    double* yk = mv->y + (int64_t)k * N;
    if (kind == 0) { /* y_t += D_ts x_s */
      const int e = std_neighbour_index(mv->d, t, s, level);
      for (int i = 0; i < mv->b; ++i)
        for (int j = 0; j < mv->b; ++j)
          yk[t * mv->b + i] += mv->Dn[(t * mv->b + i) * (mv->ND * mv->b) + e * mv->b + j] * xk[s * mv->b + j];
      continue;
    }
    const int64_t m = N / ipow(1 << mv->d, level);
    const int qt = oracle_std_slot(mv->d, level, t, s), qs = oracle_std_slot(mv->d, level, s, t);
    const int W = mv->M * mv->r;
    const double* Ul = mv->U[level - 1];
    const double* Vl = mv->V[level - 1];
    for (int a = 0; a < mv->r; ++a) mv->z[a] = 0.0;
    for (int64_t j = 0; j < m; ++j)   /* z = V_ts^T x_s */
      for (int a = 0; a < mv->r; ++a) mv->z[a] += Vl[(s * m + j) * W + qs * mv->r + a] * xk[s * m + j];
    for (int64_t i = 0; i < m; ++i)   /* y_t += U_ts z */
      for (int a = 0; a < mv->r; ++a) yk[t * m + i] += Ul[(t * m + i) * W + qt * mv->r + a] * mv->z[a];
  }
}

void oracle_std_matvec(int d, int L, int b, int r, const double* const* U, const double* const* V,
                       const double* Dn, const double* x, double* y, int nrhs) {
  std_mv_t mv;
  mv.d = d; mv.b = b; mv.r = r; mv.M = oracle_std_slots(d); mv.ND = (int)ipow(3, d); mv.nrhs = nrhs;
  mv.N = (int64_t)b * ipow(1 << d, L);
  mv.U = U; mv.V = V; mv.Dn = Dn; mv.x = x; mv.y = y;
  mv.z = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int64_t i = 0; i < mv.N * nrhs; ++i) y[i] = 0.0;
  visit_root_std(d, L, std_mv_cb, &mv);
  free(mv.z);
}

/* y = H^T x over the standard-admissibility blocks (GEMV "T"):
 * H^T = sum over the blocks (t, s) of Def 2.4 of (H_ts)^T placed at (s, t), so
 * every block contributes its transpose: dense y_s += D_ts^T x_t; low rank
 * w = U_ts^T x_t, y_s += V_ts w. */
static void std_mv_t_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  std_mv_t* mv = (std_mv_t*)ctx;
  const int64_t N = mv->N;
  for (int k = 0; k < mv->nrhs; ++k) {
    const double* xk = mv->x + (int64_t)k * N;
    double* yk = mv->y + (int64_t)k * N;
    if (kind == 0) { /* y_s += D_ts^T x_t */
      const int e = std_neighbour_index(mv->d, t, s, level);
      for (int i = 0; i < mv->b; ++i)
        for (int j = 0; j < mv->b; ++j)
          yk[s * mv->b + j] += mv->Dn[(t * mv->b + i) * (mv->ND * mv->b) + e * mv->b + j] * xk[t * mv->b + i];
      continue;
    }
    const int64_t m = N / ipow(1 << mv->d, level);
    const int qt = oracle_std_slot(mv->d, level, t, s), qs = oracle_std_slot(mv->d, level, s, t);
    const int W = mv->M * mv->r;
    const double* Ul = mv->U[level - 1];
    const double* Vl = mv->V[level - 1];
    for (int a = 0; a < mv->r; ++a) mv->z[a] = 0.0;
    for (int64_t i = 0; i < m; ++i)   /* w = U_ts^T x_t */
      for (int a = 0; a < mv->r; ++a) mv->z[a] += Ul[(t * m + i) * W + qt * mv->r + a] * xk[t * m + i];
    for (int64_t j = 0; j < m; ++j)   /* y_s += V_ts w */
      for (int a = 0; a < mv->r; ++a) yk[s * m + j] += Vl[(s * m + j) * W + qs * mv->r + a] * mv->z[a];
  }
}

void oracle_std_matvec_t(int d, int L, int b, int r, const double* const* U, const double* const* V,
                         const double* Dn, const double* x, double* y, int nrhs) {
  std_mv_t mv;
  mv.d = d; mv.b = b; mv.r = r; mv.M = oracle_std_slots(d); mv.ND = (int)ipow(3, d); mv.nrhs = nrhs;
  mv.N = (int64_t)b * ipow(1 << d, L);
  mv.U = U; mv.V = V; mv.Dn = Dn; mv.x = x; mv.y = y;
  mv.z = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int64_t i = 0; i < mv.N * nrhs; ++i) y[i] = 0.0;
  visit_root_std(d, L, std_mv_t_cb, &mv);
  free(mv.z);
}

/* ---- standard admissibility, Def 2.4 read LITERALLY (leaf check first) ------
 * PAPER.md:316-339 checks the three conditions "in the given order": (1) a child
 * pair with a leaf is dense, (2) else an admissible pair is low rank, (3) else
 * recurse.  So at the leaf level EVERY child pair of a hierarchical (touching)
 * parent pair is dense -- the near field AND the leaf-level interaction list --
 * and low-rank blocks exist at levels 2..L-1 only.  (R17 checks
 * admissibility first, like R1 for the weak structure; this is the literal
 * alternative, SURVEY §8 f3 with the f2 reading.)
 * Panels: U, V as the standard canonical panels (levels 1..L-1 used); the dense
 * blocks of leaf-parent p (level L-1) against its neighbour p + eps form one
 * (c b) x (c b) block, stored like the standard near field one level up:
 *   Dc (N x 3^d c b): row i of leaf-parent p, columns [e c b, (e+1) c b) = row
 *   i - p c b of the dense block of (p, p + eps), e = sum_i (eps_i + 1) 3^i;
 *   the leaf pair (t, s), t in p, s in p + eps, is its sub-block at column
 *   offset (s - c (p + eps)) b. */
static void visit_std_strict(int d, int L, int level, int64_t pt, int64_t ps, block_fn fn, void* ctx) {
  const int c = 1 << d;
  for (int a = 0; a < c; ++a)
    for (int bb = 0; bb < c; ++bb) {
      int64_t t = pt * c + a, s = ps * c + bb;
      int64_t xt[3], xs[3];
      morton_decode(d, t, level + 1, xt);
      morton_decode(d, s, level + 1, xs);
      if (level + 1 == L) fn(ctx, 0, level + 1, t, s);                 /* (1) leaves: dense */
      else if (std_admissible(d, xt, xs)) fn(ctx, 1, level + 1, t, s); /* (2) admissible: low rank */
      else visit_std_strict(d, L, level + 1, t, s, fn, ctx);          /* (3) hierarchical */
    }
}

static void visit_root_std_strict(int d, int L, block_fn fn, void* ctx) {
  if (L == 0) fn(ctx, 0, 0, 0, 0);
  else visit_std_strict(d, L, 0, 0, 0, fn, ctx);
}

void oracle_std_census_strict(int d, int L, int64_t* n_lowrank, int64_t* n_dense) {
  std_census_t cs = {0, 0, -1, -1, 0};
  visit_root_std_strict(d, L, std_census_cb, &cs);
  *n_lowrank = cs.lowrank; *n_dense = cs.dense;
}

void oracle_std_cover_count_strict(int d, int L, int b, int32_t* count) {
  cover_t cv;
  cv.c = 1 << d; cv.L = L; cv.b = b; cv.N = (int64_t)b * ipow(cv.c, L); cv.count = count;
  memset(count, 0, sizeof(int32_t) * (size_t)(cv.N * cv.N));
  visit_root_std_strict(d, L, cover_cb, &cv);
}

/* column of entry (row of t, column j of s) of a leaf pair in the Dc panel */
static int64_t std_strict_dcol(int d, int L, int b, int64_t t, int64_t s, int j) {
  const int c = 1 << d;
  if (L == 0) return j; /* the root is the only leaf: Dc is N x b */
  const int64_t pt = t / c, ps = s / c;
  const int e = std_neighbour_index(d, pt, ps, L - 1);
  return (int64_t)e * c * b + (s - ps * c) * b + j;
}

typedef struct {
  int d, L, b, r, M, ND, nrhs, c; int64_t N, ldd;
  const double* const* U; const double* const* V; const double* Dc; const double* x; double* y; double* z;
  double* A;
} std_strict_t;

static void std_strict_assemble_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  std_strict_t* as = (std_strict_t*)ctx;
  const int64_t N = as->N;
  if (kind == 0) {
    for (int i = 0; i < as->b; ++i)
      for (int j = 0; j < as->b; ++j)
        as->A[(t * as->b + i) * N + (s * as->b + j)] =
            as->Dc[(t * as->b + i) * as->ldd + std_strict_dcol(as->d, as->L, as->b, t, s, j)];
    return;
  }
  const int64_t m = N / ipow(as->c, level);
  const int qt = oracle_std_slot(as->d, level, t, s), qs = oracle_std_slot(as->d, level, s, t);
  const int W = as->M * as->r;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int a = 0; a < as->r; ++a)
        acc += as->U[level - 1][(t * m + i) * W + qt * as->r + a] * as->V[level - 1][(s * m + j) * W + qs * as->r + a];
      as->A[(t * m + i) * N + (s * m + j)] = acc;
    }
}

static void std_strict_init(std_strict_t* st, int d, int L, int b, int r, const double* const* U,
                            const double* const* V, const double* Dc) {
  st->d = d; st->L = L; st->b = b; st->r = r; st->c = 1 << d;
  st->M = oracle_std_slots(d); st->ND = (int)ipow(3, d);
  st->N = (int64_t)b * ipow(st->c, L);
  st->ldd = L == 0 ? b : (int64_t)st->ND * st->c * b;
  st->U = U; st->V = V; st->Dc = Dc;
}

void oracle_std_assemble_strict(int d, int L, int b, int r, const double* const* U, const double* const* V,
                                const double* Dc, double* A) {
  std_strict_t as;
  std_strict_init(&as, d, L, b, r, U, V, Dc);
  as.A = A;
  memset(A, 0, sizeof(double) * (size_t)(as.N * as.N));
  visit_root_std_strict(d, L, std_strict_assemble_cb, &as);
}

/* y = H x, eq:hmat-vec-add over the literal-order blocks */
static void std_strict_mv_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  std_strict_t* mv = (std_strict_t*)ctx;
  const int64_t N = mv->N;
  for (int k = 0; k < mv->nrhs; ++k) {
    const double* xk = mv->x + (int64_t)k * N;
    double* yk = mv->y + (int64_t)k * N;
    if (kind == 0) { /* y_t += D_ts x_s */
      for (int i = 0; i < mv->b; ++i)
        for (int j = 0; j < mv->b; ++j)
          yk[t * mv->b + i] += mv->Dc[(t * mv->b + i) * mv->ldd + std_strict_dcol(mv->d, mv->L, mv->b, t, s, j)] *
                               xk[s * mv->b + j];
      continue;
    }
    const int64_t m = N / ipow(mv->c, level);
    const int qt = oracle_std_slot(mv->d, level, t, s), qs = oracle_std_slot(mv->d, level, s, t);
    const int W = mv->M * mv->r;
    const double* Ul = mv->U[level - 1];
    const double* Vl = mv->V[level - 1];
    for (int a = 0; a < mv->r; ++a) mv->z[a] = 0.0;
    for (int64_t j = 0; j < m; ++j)   /* z = V_ts^T x_s */
      for (int a = 0; a < mv->r; ++a) mv->z[a] += Vl[(s * m + j) * W + qs * mv->r + a] * xk[s * m + j];
    for (int64_t i = 0; i < m; ++i)   /* y_t += U_ts z */
      for (int a = 0; a < mv->r; ++a) yk[t * m + i] += Ul[(t * m + i) * W + qt * mv->r + a] * mv->z[a];
  }
}

void oracle_std_matvec_strict(int d, int L, int b, int r, const double* const* U, const double* const* V,
                              const double* Dc, const double* x, double* y, int nrhs) {
  std_strict_t mv;
  std_strict_init(&mv, d, L, b, r, U, V, Dc);
  mv.nrhs = nrhs; mv.x = x; mv.y = y;
  mv.z = (double*)malloc(sizeof(double) * (size_t)(r > 0 ? r : 1));
  for (int64_t i = 0; i < mv.N * nrhs; ++i) y[i] = 0.0;
  visit_root_std_strict(d, L, std_strict_mv_cb, &mv);
  free(mv.z);
}

/* Sampled rows of the SEEDED standard-admissibility operator (gen/hgen.h, the
 * canonical standard panels above, entries generated on demand), so that full
 * bench-size operators (s2: 55.6 GB of factors) can be checked row by row:
 * y_i = sum over the blocks (t, s) of Def 2.4 (standard admissibility,
 * PAPER.md:279-297, 316-339) whose target t contains row i of
 *   dense (leaf level):  D_ts[i - t b, :] x_s                (eq:prod-dx)
 *   low rank (level l):  U_ts[i - t m_l, :] (V_ts^T x_s)      (eq:prod-uvx)
 * The blocks are found by the same recursion as visit_std, restricted to the
 * child that holds row i at every level. */
typedef struct {
  int d, L, b, r, M, ND, nrhs; int64_t N, i; uint64_t seed;
  const double* x; double* yi;  /* yi[k] = y[i, k] */
} std_row_t;

static void std_row_cb(void* ctx, int kind, int level, int64_t t, int64_t s) {
  std_row_t* rw = (std_row_t*)ctx;
  const int64_t N = rw->N, i = rw->i;
  if (kind == 0) { /* dense neighbour block D_ts, Dn row i, columns [e b, (e+1) b) */
    const int e = std_neighbour_index(rw->d, t, s, level);
    const uint64_t stD = hgen_stream(rw->seed, HGEN_TAG_D, 0, 0);
    const int64_t ld = (int64_t)rw->ND * rw->b;
    for (int k = 0; k < rw->nrhs; ++k) {
      double acc = 0.0;
      for (int j = 0; j < rw->b; ++j)
        acc += hgen_normal(stD, (uint64_t)(i * ld + e * rw->b + j)) * 0.125 * rw->x[(int64_t)k * N + s * rw->b + j];
      rw->yi[k] += acc;
    }
    return;
  }
  const int64_t m = N / ipow(1 << rw->d, level);
  const double scale = 1.0 / sqrt((double)m);
  const int W = rw->M * rw->r;
  const int qt = oracle_std_slot(rw->d, level, t, s), qs = oracle_std_slot(rw->d, level, s, t);
  const uint64_t stU = hgen_stream(rw->seed, HGEN_TAG_U, (uint64_t)level, 0);
  const uint64_t stV = hgen_stream(rw->seed, HGEN_TAG_V, (uint64_t)level, 0);
  for (int k = 0; k < rw->nrhs; ++k)
    for (int a = 0; a < rw->r; ++a) {
      double za = 0.0; /* (V_ts^T x_s)[a] */
#pragma omp parallel for reduction(+ : za) schedule(static)
      for (int64_t j = 0; j < m; ++j)
        za += hgen_normal(stV, (uint64_t)((s * m + j) * W + qs * rw->r + a)) * scale * rw->x[(int64_t)k * N + s * m + j];
      rw->yi[k] += hgen_normal(stU, (uint64_t)(i * W + qt * rw->r + a)) * scale * za;
    }
}

static void visit_std_row(int d, int L, int level, int64_t pt, int64_t ps, int64_t i, int64_t N, block_fn fn,
                          void* ctx) {
  const int c = 1 << d;
  const int64_t t = i / (N / ipow(c, level + 1)); /* the child of pt holding row i */
  for (int bb = 0; bb < c; ++bb) {
    const int64_t s = ps * c + bb;
    int64_t xt[3], xs[3];
    morton_decode(d, t, level + 1, xt);
    morton_decode(d, s, level + 1, xs);
    if (std_admissible(d, xt, xs)) fn(ctx, 1, level + 1, t, s);
    else if (level + 1 == L) fn(ctx, 0, level + 1, t, s);
    else visit_std_row(d, L, level + 1, t, s, i, N, fn, ctx);
  }
  (void)pt;
}

void oracle_std_rows_generated(int d, int L, int b, int r, uint64_t seed, const double* x, int nrhs,
                               int64_t nrows, const int64_t* rows, double* yrows) {
  std_row_t rw;
  rw.d = d; rw.L = L; rw.b = b; rw.r = r; rw.M = oracle_std_slots(d); rw.ND = (int)ipow(3, d);
  rw.nrhs = nrhs; rw.N = (int64_t)b * ipow(1 << d, L); rw.seed = seed; rw.x = x;
  double* yi = (double*)malloc(sizeof(double) * (size_t)nrhs);
  for (int64_t n = 0; n < nrows; ++n) {
    for (int k = 0; k < nrhs; ++k) yi[k] = 0.0;
    rw.i = rows[n];
    rw.yi = yi;
    if (L == 0) std_row_cb(&rw, 0, 0, 0, 0);
    else visit_std_row(d, L, 0, 0, 0, rw.i, rw.N, std_row_cb, &rw);
    for (int k = 0; k < nrhs; ++k) yrows[(int64_t)k * nrows + n] = yi[k];
  }
  free(yi);
}
