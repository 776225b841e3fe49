// kernels_aux.cu -- one-time helpers of the C ABI (not on the per-matvec path).
//
// transpose_leaf_blocks: D^T for the transposed product H^T x (GEMV "T",
// PAPER.md:961-969): H^T has the same block structure with U and V exchanged
// and every dense leaf block transposed, so the expand kernel runs unchanged on
// (V, U, D^T).
#include "comm.h"
#include "geometry.cuh"
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

// Standard admissibility: H^T's near-field block (t, t + eps) is
// (H_{t+eps, t})^T, and H_{t+eps, t} sits in the rows of leaf t + eps, panel
// e' = nd - 1 - e (the offset -eps).  So panel e of D^T, row i of leaf t,
// column j = panel e' of D, row j of leaf t + eps, column i (zero when t + eps
// lies outside the domain).
__global__ void transpose_near_field_kernel(const double* __restrict__ D, double* __restrict__ Dt,
                                            int64_t n_leaves, int64_t lbase, int d, int L, int b, int Dp,
                                            int64_t d_stride, int nd) {
  const int64_t total = n_leaves * nd * b * b;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = o / ((int64_t)nd * b * b);
    int rem = static_cast<int>(o - t * nd * b * b);
    const int e = rem / (b * b);
    rem -= e * b * b;
    const int i = rem / b, j = rem - i * b;
    int x[3];
    geo::morton_decode(d, lbase + t, L, x);
    if (!((geo::near_mask(d, x, 1 << L) >> e) & 1u)) continue;
    const int64_t s = geo::neighbour(d, x, e, L) - lbase;  // local leaf of the neighbour
    if (s < 0 || s >= n_leaves) continue;  // on another rank: its product arrives via the exchange
    Dt[e * d_stride + (t * b + i) * Dp + j] = D[(nd - 1 - e) * d_stride + (s * b + j) * Dp + i];
  }
}

// H^T, P > 1: c_{S,T}[kk][j] = sum_i D_{S,T}[i][j] x_S[kk][i] for this rank's
// outgoing cross near-field pairs {pair, local leaf S, e} (T = S + eps_e) ->
// entries [pair][kk][bpad] of the packed buffer's second part
__global__ void std_tpack_kernel(double* __restrict__ out, const double* __restrict__ D, int64_t d_stride, int Dp,
                                 const double* __restrict__ x, int64_t ldx, const int64_t* __restrict__ tpack,
                                 int64_t n_pairs, int cap, int nr, int b, int bpad) {
  const int64_t total = n_pairs * nr * b;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t it = o / ((int64_t)nr * b);
    const int rem = static_cast<int>(o - it * nr * b);
    const int kk = rem / b, j = rem - kk * b;
    const int64_t pair = tpack[3 * it], leaf = tpack[3 * it + 1];
    const int e = static_cast<int>(tpack[3 * it + 2]);
    const double* blk = D + e * d_stride + leaf * b * Dp + j;
    const double* xs = x + kk * ldx + leaf * b;
    double v = 0.0;
    for (int i = 0; i < b; ++i) v = fma(blk[(int64_t)i * Dp], xs[i], v);
    out[(pair * cap + kk) * bpad + j] = v;
  }
}

// H^T, P > 1: y_T += alpha * sum over T's incoming pairs (ascending) of c_{S,T}
__global__ void std_tadd_kernel(double* __restrict__ y, int64_t ldy, double alpha, const double* __restrict__ in,
                                const int64_t* __restrict__ leaf, const int64_t* __restrict__ off,
                                const int64_t* __restrict__ pairs, int64_t n_leaves, int cap, int nr, int b,
                                int bpad) {
  const int64_t total = n_leaves * nr * b;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t it = o / ((int64_t)nr * b);
    const int rem = static_cast<int>(o - it * nr * b);
    const int kk = rem / b, j = rem - kk * b;
    double v = 0.0;
    for (int64_t q = off[it]; q < off[it + 1]; ++q) v += in[(pairs[q] * cap + kk) * bpad + j];
    y[kk * ldy + leaf[it] * b + j] += alpha * v;
  }
}

// x of this rank's boundary leaves -> halo entries [h][kk][bpad] of the packed buffer
__global__ void std_pack_x_kernel(double* __restrict__ halo, const double* __restrict__ x, int64_t ldx,
                                  const int64_t* __restrict__ pack, int64_t n_pack, int cap, int nr, int b,
                                  int bpad) {
  const int64_t total = n_pack * nr * b;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t it = o / ((int64_t)nr * b);
    const int rem = static_cast<int>(o - it * nr * b);
    const int kk = rem / b, j = rem - kk * b;
    const int64_t h = pack[2 * it], leaf = pack[2 * it + 1];
    halo[(h * cap + kk) * bpad + j] = x[kk * ldx + leaf * b + j];
  }
}

// received z entries [e][kk][r] -> Zt rows [row][kk][Wp] at columns q r .. q r + r - 1
__global__ void std_unpack_z_kernel(double* __restrict__ zt, const double* __restrict__ xchg,
                                    const int64_t* __restrict__ unpack, int64_t n_unpack, int cap, int nr, int Wp,
                                    int r) {
  const int64_t total = n_unpack * nr * r;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t it = o / ((int64_t)nr * r);
    const int rem = static_cast<int>(o - it * nr * r);
    const int kk = rem / r, aa = rem - kk * r;
    const int64_t e = unpack[2 * it], rq = unpack[2 * it + 1];
    const int64_t row = rq >> 8;
    const int q = static_cast<int>(rq & 255);
    zt[(row * cap + kk) * Wp + q * r + aa] = xchg[(e * cap + kk) * r + aa];
  }
}

// buf += add, elementwise (the tree exchange's combine, comm.h)
__global__ void add_inplace_kernel(double* __restrict__ buf, const double* __restrict__ add, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] += add[i];
}

int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : g > 148 * 16 ? 148 * 16 : g);
}

}  // namespace

cudaError_t launch_add_inplace(double* buf, const double* add, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  add_inplace_kernel<<<grid_for(static_cast<int64_t>(n)), 256, 0, s>>>(buf, add, static_cast<int64_t>(n));
  return cudaGetLastError();
}

cudaError_t launch_std_pack_x(double* halo, const double* x, int64_t ldx, const int64_t* pack, int64_t n_pack, int cap,
                              int nr, int b, int bpad, cudaStream_t s) {
  if (n_pack == 0) return cudaSuccess;
  std_pack_x_kernel<<<grid_for(n_pack * nr * b), 256, 0, s>>>(halo, x, ldx, pack, n_pack, cap, nr, b, bpad);
  return cudaGetLastError();
}

cudaError_t launch_std_unpack_z(double* zt, const double* xchg, const int64_t* unpack, int64_t n_unpack, int cap,
                                int nr, int Wp, int r, cudaStream_t s) {
  if (n_unpack == 0) return cudaSuccess;
  std_unpack_z_kernel<<<grid_for(n_unpack * nr * r), 256, 0, s>>>(zt, xchg, unpack, n_unpack, cap, nr, Wp, r);
  return cudaGetLastError();
}

cudaError_t launch_transpose_near_field(const double* D, double* Dt, int64_t n_leaves, int64_t lbase, int d, int L,
                                        int b, int Dp, int64_t d_stride, int nd, cudaStream_t s) {
  const int64_t total = n_leaves * nd * b * b;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 32) grid = 148 * 32;
  if (grid < 1) grid = 1;
  transpose_near_field_kernel<<<static_cast<int>(grid), 256, 0, s>>>(D, Dt, n_leaves, lbase, d, L, b, Dp, d_stride,
                                                                     nd);
  return cudaGetLastError();
}

cudaError_t launch_std_tpack(double* out, const double* D, int64_t d_stride, int Dp, const double* x, int64_t ldx,
                             const int64_t* tpack, int64_t n_pairs, int cap, int nr, int b, int bpad,
                             cudaStream_t s) {
  const int64_t total = n_pairs * nr * b;
  if (total == 0) return cudaSuccess;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  std_tpack_kernel<<<static_cast<int>(grid), 256, 0, s>>>(out, D, d_stride, Dp, x, ldx, tpack, n_pairs, cap, nr, b,
                                                          bpad);
  return cudaGetLastError();
}

cudaError_t launch_std_tadd(double* y, int64_t ldy, double alpha, const double* in, const int64_t* leaf,
                            const int64_t* off, const int64_t* pairs, int64_t n_leaves, int cap, int nr, int b,
                            int bpad, cudaStream_t s) {
  const int64_t total = n_leaves * nr * b;
  if (total == 0) return cudaSuccess;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  std_tadd_kernel<<<static_cast<int>(grid), 256, 0, s>>>(y, ldy, alpha, in, leaf, off, pairs, n_leaves, cap, nr, b,
                                                         bpad);
  return cudaGetLastError();
}

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
