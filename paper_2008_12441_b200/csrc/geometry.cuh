// geometry.cuh -- Morton boxes of the ideal domain [0,1]^d
// for the standard-admissibility path: a level-l node k is the
// box with integer coordinates x (bit j of x_i = bit j d + i of k, so the low d
// bits of k are the child position inside the parent).
#pragma once
#include <cstdint>

namespace hmat {
namespace geo {

__device__ __forceinline__ void morton_decode(int d, int64_t k, int level, int x[3]) {
  x[0] = x[1] = x[2] = 0;
  for (int j = 0; j < level; ++j)
    for (int i = 0; i < d; ++i) x[i] |= static_cast<int>((k >> (j * d + i)) & 1) << j;
}

__device__ __forceinline__ int64_t morton_encode(int d, const int x[3], int level) {
  int64_t k = 0;
  for (int j = 0; j < level; ++j)
    for (int i = 0; i < d; ++i) k |= static_cast<int64_t>((x[i] >> j) & 1) << (j * d + i);
  return k;
}

// Near-field offsets eps in {-1,0,1}^d are numbered e = sum_i (eps_i + 1) 3^i.
// Bit e of the result: the neighbour x + eps lies inside the n^d grid.
__device__ __forceinline__ uint32_t near_mask(int d, const int x[3], int n) {
  uint32_t m = 0;
  int nd = 1;
  for (int i = 0; i < d; ++i) nd *= 3;
  for (int e = 0; e < nd; ++e) {
    int rem = e;
    bool ok = true;
    for (int i = 0; i < d; ++i) {
      const int xi = x[i] + rem % 3 - 1;
      rem /= 3;
      ok = ok && xi >= 0 && xi < n;
    }
    if (ok) m |= 1u << e;
  }
  return m;
}

// Morton index of the level-`level` box x + eps(e) (caller checked it exists).
__device__ __forceinline__ int64_t neighbour(int d, const int x[3], int e, int level) {
  int y[3] = {x[0], x[1], x[2]};
  for (int i = 0; i < d; ++i) {
    y[i] += e % 3 - 1;
    e /= 3;
  }
  return morton_encode(d, y, level);
}

}  // namespace geo
}  // namespace hmat
