// Host-side check of the Morton bit-arithmetic helpers in csrc/geometry.cuh
// (tests/test_geometry_host.py builds and runs it; no GPU): for d = 1, 2, 3 and
// every box k of small levels, near_mask_k equals near_mask of the decoded
// coordinates, and neighbour_k equals the decode / offset / encode form for
// every near-field offset e (-1 exactly where the neighbour leaves the grid).
#include <cstdio>
#include "geometry.cuh"

using namespace hmat::geo;

int main() {
  long checked = 0, bad = 0;
  for (int d = 1; d <= 3; ++d) {
    const int nd = d == 1 ? 3 : d == 2 ? 9 : 27;
    const int lmax = d == 1 ? 10 : d == 2 ? 6 : 4;
    for (int level = 0; level <= lmax; ++level) {
      const int64_t nk = int64_t(1) << (level * d);
      for (int64_t k = 0; k < nk; ++k) {
        int x[3];
        morton_decode(d, k, level, x);
        const uint32_t m = near_mask(d, x, 1 << level);
        if (near_mask_k(d, k, level) != m) {
          if (bad++ < 10) printf("near_mask_k d=%d level=%d k=%ld\n", d, level, (long)k);
        }
        for (int e = 0; e < nd; ++e) {
          const int64_t want = ((m >> e) & 1u) ? neighbour(d, x, e, level) : -1;
          if (neighbour_k(d, k, e, level) != want) {
            if (bad++ < 10) printf("neighbour_k d=%d level=%d k=%ld e=%d\n", d, level, (long)k, e);
          }
          ++checked;
        }
      }
    }
  }
  printf("checked %ld bad %ld\n", checked, bad);
  return bad ? 1 : 0;
}
