// std_exchange.cpp -- see std_exchange.h.
#include "std_exchange.h"

#include <algorithm>

namespace hmat {

namespace {

void decode(int d, int64_t k, int level, int64_t x[3]) {
  x[0] = x[1] = x[2] = 0;
  for (int j = 0; j < level; ++j)
    for (int i = 0; i < d; ++i) x[i] |= ((k >> (j * d + i)) & 1) << j;
}

int64_t encode(int d, const int64_t x[3], int level) {
  int64_t k = 0;
  for (int j = 0; j < level; ++j)
    for (int i = 0; i < d; ++i) k |= ((x[i] >> j) & 1) << (j * d + i);
  return k;
}

// box x + eps(e) at `level` (e = sum_i (eps_i + 1) 3^i), -1 outside the domain
int64_t shifted(int d, const int64_t x[3], int e, int level) {
  int64_t y[3] = {x[0], x[1], x[2]};
  const int64_t n = int64_t(1) << level;
  for (int i = 0; i < d; ++i) {
    y[i] += e % 3 - 1;
    e /= 3;
    if (y[i] < 0 || y[i] >= n) return -1;
  }
  return encode(d, y, level);
}

}  // namespace

std::string std_exchange_build(const Plan& p, StdExchange* out) {
  if (p.adm != 1) return "std_exchange_build: not a standard-admissibility plan";
  struct Tables {
    int16_t code[3][8][kStdMaxSlots], slot[3][8][kStdMaxCodes];
    Tables() { std_slot_tables(code, slot); }
  };
  static const Tables tab;  // built once; thread-safe static initialisation
  const auto& code = tab.code;
  const auto& slot = tab.slot;
  StdExchange X;
  const int d = p.d, c = p.c, M = p.M, nd = p.nd, L = p.L;
  const int64_t Nl = p.N_loc, row0 = p.row0;
  X.bpad = p.b + (p.b & 1);
  // rank owning row i; a node of m rows lies inside one rank iff m <= N_loc
  auto owner = [&](int64_t row) { return row / Nl; };
  const int me = p.rank;

  // ---- z entries: levels 2..L (level 1 has no admissible pair) ----
  int64_t off = 0;
  for (int l = 2; l <= L; ++l) {
    X.src_off[l] = off;
    off += std::max<int64_t>(1, Nl / p.m[l]) * M;
  }
  X.src_entry.assign(static_cast<size_t>(off), -1);
  for (int l = 2; l <= L; ++l) {
    const int64_t m = p.m[l], nodes = int64_t(1) << (d * l);
    const bool whole = m <= Nl;  // nodes of this level lie inside one rank
    const int64_t base = row0 / m, cnt = std::max<int64_t>(1, Nl / m);
    for (int64_t t = 0; t < nodes; ++t) {
      const int tau = static_cast<int>(t & (c - 1));
      int64_t xp[3];
      decode(d, t >> d, l - 1, xp);
      const bool t_here = t >= base && t < base + cnt;
      for (int q = 0; q < M; ++q) {
        const int cd = code[d - 1][tau][q];
        if (cd < 0) continue;
        const int e = cd / c, sigma = cd % c;
        const int64_t ps = shifted(d, xp, e, l - 1);
        if (ps < 0) continue;  // partner outside the domain: no block
        const int64_t s = ps * c + sigma;
        if (whole && owner(t * m) == owner(s * m)) continue;  // both inside one rank
        const int64_t entry = X.E++;
        const bool s_here = s >= base && s < base + cnt;
        if (s_here) {
          const int qs = slot[d - 1][sigma][(nd - 1 - e) * c + tau];  // slot of t in s's list
          X.src_entry[static_cast<size_t>(X.src_off[l] + (s - base) * M + qs)] = static_cast<int32_t>(entry);
        }
        if (t_here) X.unpack.insert(X.unpack.end(), {entry, (p.zt_off[l] + (t - base)) * 256 + q});
      }
    }
  }
  if (X.E > (int64_t(1) << 31) - 1) return "unsupported: too many cross-rank blocks";

  // ---- halo leaves: x of a leaf whose near field reaches another rank ----
  const int64_t leaves = p.N / p.b;
  const int64_t lbase = row0 / p.b, lcnt = Nl / p.b;
  X.halo_of.assign(static_cast<size_t>(lcnt * nd), -1);
  std::vector<int64_t> hidx(static_cast<size_t>(leaves), -1);
  for (int64_t s = 0; s < leaves; ++s) {
    int64_t xs[3];
    decode(d, s, L, xs);
    const int64_t os = owner(s * p.b);
    for (int e = 0; e < nd; ++e) {
      const int64_t t = shifted(d, xs, e, L);
      if (t >= 0 && owner(t * p.b) != os) {
        hidx[static_cast<size_t>(s)] = X.Hn++;
        break;
      }
    }
    if (hidx[static_cast<size_t>(s)] >= 0 && os == me) X.pack.insert(X.pack.end(), {hidx[static_cast<size_t>(s)], s - lbase});
  }
  for (int64_t t = lbase; t < lbase + lcnt; ++t) {
    int64_t xt[3];
    decode(d, t, L, xt);
    for (int e = 0; e < nd; ++e) {
      const int64_t s = shifted(d, xt, e, L);
      if (s >= 0 && owner(s * p.b) != me) X.halo_of[static_cast<size_t>((t - lbase) * nd + e)] =
          static_cast<int32_t>(hidx[static_cast<size_t>(s)]);
    }
  }
  // ---- H^T: cross near-field pairs (S, T) carrying c_{S,T} = (D_{S,T})^T x_S ----
  std::vector<std::vector<int64_t>> incoming(static_cast<size_t>(lcnt));
  for (int64_t s = 0; s < leaves; ++s) {
    int64_t xs[3];
    decode(d, s, L, xs);
    const int64_t os = owner(s * p.b);
    for (int e = 0; e < nd; ++e) {
      const int64_t t = shifted(d, xs, e, L);
      if (t < 0 || owner(t * p.b) == os) continue;
      const int64_t pair = X.Hp++;
      if (os == me) X.tpack.insert(X.tpack.end(), {pair, s - lbase, e});
      if (owner(t * p.b) == me) incoming[static_cast<size_t>(t - lbase)].push_back(pair);
    }
  }
  X.tadd_off.push_back(0);
  for (int64_t t = 0; t < lcnt; ++t) {
    const auto& v = incoming[static_cast<size_t>(t)];
    if (v.empty()) continue;
    X.tadd_leaf.push_back(t);
    X.tadd_pair.insert(X.tadd_pair.end(), v.begin(), v.end());
    X.tadd_off.push_back(static_cast<int64_t>(X.tadd_pair.size()));
  }
  *out = std::move(X);
  return "";
}

}  // namespace hmat
