// geometry.cuh -- Morton boxes of the ideal domain [0,1]^d
// for the standard-admissibility path: a level-l node k is the
// box with integer coordinates x (bit j of x_i = bit j d + i of k, so the low d
// bits of k are the child position inside the parent).
#pragma once
#include <cstdint>

// host + device: tests/test_geometry_host.py compiles these for the CPU and
// checks the bit-arithmetic forms against decode / encode exhaustively
#define HMAT_GEO_FN __host__ __device__ __forceinline__

namespace hmat {
namespace geo {

HMAT_GEO_FN void morton_decode(int d, int64_t k, int level, int x[3]) {
  x[0] = x[1] = x[2] = 0;
  for (int j = 0; j < level; ++j)
    for (int i = 0; i < d; ++i) x[i] |= static_cast<int>((k >> (j * d + i)) & 1) << j;
}

HMAT_GEO_FN int64_t morton_encode(int d, const int x[3], int level) {
  int64_t k = 0;
  for (int j = 0; j < level; ++j)
    for (int i = 0; i < d; ++i) k |= static_cast<int64_t>((x[i] >> j) & 1) << (j * d + i);
  return k;
}

// Near-field offsets eps in {-1,0,1}^d are numbered e = sum_i (eps_i + 1) 3^i.
// Bit e of the result: the neighbour x + eps lies inside the n^d grid.
HMAT_GEO_FN uint32_t near_mask(int d, const int x[3], int n) {
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
HMAT_GEO_FN int64_t neighbour(int d, const int x[3], int e, int level) {
  int y[3] = {x[0], x[1], x[2]};
  for (int i = 0; i < d; ++i) {
    y[i] += e % 3 - 1;
    e /= 3;
  }
  return morton_encode(d, y, level);
}

// Bits of dimension i in a d-dimensional Morton index (bit j d + i for all j).
HMAT_GEO_FN uint64_t dilated_mask(int d, int i) {
  if (d == 1) return ~0ull;
  if (d == 2) return i == 0 ? 0x5555555555555555ull : 0xAAAAAAAAAAAAAAAAull;
  return i == 0 ? 0x9249249249249249ull : i == 1 ? 0x2492492492492492ull : 0x4924924924924924ull;
}

// Morton index of the level-`level` box x(k) + eps(e), computed on k's
// interleaved bits (dilated-integer increment / decrement per dimension: the
// carry or borrow runs through the other dimensions' bits), or -1 when it lies
// outside the 2^level grid.  Equal to neighbour(d, decode(k), e, level) where
// near_mask has bit e, without the decode / encode loops.
HMAT_GEO_FN int64_t neighbour_k(int d, int64_t k, int e, int level) {
  const uint64_t lvm = level * d >= 64 ? ~0ull : (1ull << (level * d)) - 1;
  uint64_t r = static_cast<uint64_t>(k);
  for (int i = 0; i < d; ++i) {
    const uint64_t M = dilated_mask(d, i) & lvm;
    const int off = e % 3 - 1;
    e /= 3;
    uint64_t part = r & M;
    if (off > 0) {
      if (part == M) return -1;
      part = ((part | ~M) + 1) & M;
    } else if (off < 0) {
      if (part == 0) return -1;
      part = (part - 1) & M;
    }
    r = (r & ~M) | part;
  }
  return static_cast<int64_t>(r);
}

// Pattern of the near-field offsets e whose digit i (eps_i + 1) is 0, in d dims.
HMAT_GEO_FN uint32_t digit_zero_pattern(int d, int i) {
  if (d == 1) return 0x1u;
  if (d == 2) return i == 0 ? 0x49u : 0x7u;
  return i == 0 ? 0x1249249u : i == 1 ? 0x1C0E07u : 0x1FFu;
}

// near_mask of the level-`level` box with Morton index k, from k's bits: in
// dimension i the offsets -1 (digit 0) are out when the coordinate is 0 (its
// dilated bits all clear) and +1 (digit 2) when it is 2^level - 1 (all set).
HMAT_GEO_FN uint32_t near_mask_k(int d, int64_t k, int level) {
  const uint64_t lvm = level * d >= 64 ? ~0ull : (1ull << (level * d)) - 1;
  uint32_t m = d == 1 ? 0x7u : d == 2 ? 0x1FFu : 0x7FFFFFFu;
  int shift = 2;  // 2 * 3^i
  for (int i = 0; i < d; ++i) {
    const uint64_t M = dilated_mask(d, i) & lvm;
    const uint64_t part = static_cast<uint64_t>(k) & M;
    const uint32_t z0 = digit_zero_pattern(d, i);
    if (part == 0) m &= ~z0;
    if (part == M) m &= ~(z0 << shift);
    shift *= 3;
  }
  return m;
}

}  // namespace geo
}  // namespace hmat
