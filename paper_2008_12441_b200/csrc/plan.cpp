// plan.cpp -- see plan.h.
#include "plan.h"

#include <algorithm>
#include <cstdio>

namespace hmat {

namespace {

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Largest divisor R of b with R <= rmax and R * width_doubles * 8 <= cap (>= 1).
int pick_rows(int b, int rmax, int64_t width_doubles, int64_t cap) {
  int best = 1;
  for (int R = 1; R <= std::min(b, rmax); ++R)
    if (b % R == 0 && R * width_doubles * 8 <= cap) best = R;
  return best;
}

}  // namespace

void std_slot_tables(int16_t code[3][8][kStdMaxSlots], int16_t slot[3][8][kStdMaxCodes]) {
  for (int d = 1; d <= 3; ++d) {
    const int c = 1 << d;
    int nd = 1;
    for (int i = 0; i < d; ++i) nd *= 3;
    for (int tau = 0; tau < 8; ++tau) {
      for (int q = 0; q < kStdMaxSlots; ++q) code[d - 1][tau][q] = -1;
      for (int k = 0; k < kStdMaxCodes; ++k) slot[d - 1][tau][k] = -1;
      if (tau >= c) continue;
      int q = 0;
      // candidates: child sigma of the parent's neighbour eps, in increasing
      // code = e 2^d + sigma; a candidate is in the list unless it touches the
      // box (offset 2 eps + sigma - tau in {-1,0,1}^d)
      for (int cd = 0; cd < nd * c; ++cd) {
        const int e = cd / c, sigma = cd % c;
        int rem = e;
        bool touches = true;
        for (int i = 0; i < d; ++i) {
          const int eps = rem % 3 - 1;
          rem /= 3;
          const int off = 2 * eps + ((sigma >> i) & 1) - ((tau >> i) & 1);
          touches = touches && off >= -1 && off <= 1;
        }
        if (touches) continue;
        code[d - 1][tau][q] = static_cast<int16_t>(cd);
        slot[d - 1][tau][cd] = static_cast<int16_t>(q);
        ++q;
      }
    }
  }
}

std::string plan_build(int depth, int dim, int leaf, int rank, int P, int shard, const PlanOptions& opt,
                       Plan* out) {
  char msg[256];
  if (dim < 1 || dim > 3) return "dim must be 1, 2 or 3 (ideal domains, PAPER.md:243-246)";
  if (depth < 0 || depth >= kMaxLevels) {
    snprintf(msg, sizeof msg, "depth must be in [0, %d]", kMaxLevels - 1);
    return msg;
  }
  if (leaf < 1) return "leaf_size must be >= 1";
  if (rank < 1) return "rank must be >= 1";
  Plan p;
  p.d = dim;
  p.c = 1 << dim;
  p.L = depth;
  p.b = leaf;
  p.r = rank;
  p.adm = opt.adm;
  p.dmma_off = opt.dmma_off;
  p.dmma_min = opt.dmma_min;
  p.dbg = opt.dbg;
  p.expand_chunk = opt.expand_chunk;
  p.project_dyn = opt.project_dyn;
  p.snake = opt.snake;
  p.pdl = opt.pdl;
  p.lpar = opt.lpar;
  p.early = opt.early;
  p.eshape = opt.eshape;
  p.dmma_ileave = opt.dmma_ileave;
  p.project_chunk = opt.project_chunk;
  p.aflush = opt.aflush;
  p.dmma_upol = opt.dmma_upol;
  p.dmma_pchunk = opt.dmma_pchunk;
  p.dmma_pchunk16 = opt.dmma_pchunk16;
  if (p.adm == 0) {
    p.M = p.c - 1;  // siblings (weak admissibility)
    p.nd = 1;
  } else {
    int p6 = 1, p3 = 1;
    for (int i = 0; i < dim; ++i) {
      p6 *= 6;
      p3 *= 3;
    }
    p.M = p6 - p3;  // interaction list (standard admissibility)
    p.nd = p3;      // near-field neighbours incl. self
  }
  p.W = p.M * rank;
  // N = b c^L must stay below 2^62
  int64_t N = leaf;
  for (int l = 0; l < depth; ++l) {
    if (N > (int64_t(1) << 62) / p.c) return "N = leaf_size * 2^(dim*depth) overflows 2^62";
    N *= p.c;
  }
  p.N = N;
  int64_t cl = 1;
  for (int l = 0; l <= depth; ++l) {
    p.m[l] = N / cl;
    if (l < depth) cl *= p.c;
  }
  const int64_t leaves = N / leaf;  // c^L
  if (P < 1 || (P & (P - 1)) != 0) return "nranks must be a power of two";
  if (P > leaves) return "nranks must not exceed the number of leaves 2^(dim*depth)";
  if (shard < 0 || shard >= P) return "rank id out of range [0, nranks)";
  if (p.W > 4 * kConsumerThreads) return "unsupported: slots * rank must be <= 1024";
  if (p.adm != 0 && P > 1 && opt.peer)
    return "unsupported: standard admissibility with the in-kernel peer exchange (use NCCL or the split-phase API)";
  p.P = P;
  p.rank = shard;
  p.N_loc = N / P;
  p.row0 = p.N_loc * shard;
  p.Wp = p.W + (p.W & 1);
  p.Dp = leaf + (leaf & 1);
  p.panel_stride = round_up(p.N_loc * p.Wp, 16);
  p.d_stride = round_up(p.N_loc * p.Dp, 16);

  // Levels whose parent spans more than one shard need the exchange
  // (Steps 2-4): c^{l-1} < P.
  // (Standard admissibility: no exchange levels; its cross-rank pairs travel in
  // the packed buffer of std_exchange.h and every level keeps local Zt rows,
  // one row for a node that spans ranks.)
  p.cross = 0;
  int64_t cpow = 1;  // c^{l-1}
  for (int l = 1; l <= depth && p.adm == 0; ++l) {
    if (cpow < P) p.cross = l;
    cpow *= p.c;
  }
  int64_t off_loc = 0, off_ex = 0;
  cpow = p.c;  // c^l
  for (int l = 1; l <= depth; ++l) {
    if (l <= p.cross) {
      p.zt_off[l] = off_ex;
      p.zt_tbase[l] = 0;
      p.zt_count[l] = cpow;
      off_ex += cpow;
    } else {
      p.zt_off[l] = off_loc;
      p.zt_tbase[l] = p.row0 / p.m[l];
      p.zt_count[l] = std::max<int64_t>(1, p.N_loc / p.m[l]);
      off_loc += p.zt_count[l];
    }
    if (l < depth) cpow *= p.c;
  }
  p.z_local_rows = off_loc;
  p.z_exch_rows = off_ex;

  // Pipeline geometry: stages of R rows with R | b, so every stage lies in one
  // node at every level (m_l = b c^{L-l}).
  const int64_t cap = opt.stage_cap_bytes;
  p.Rp = pick_rows(leaf, kConsumerThreads, p.Wp, cap);
  // expand: one stage holds U_l rows, or all nd dense blocks of the tile's rows
  // (standard admissibility: 3^d near-field blocks; a larger cap keeps Re >= 8)
  // A wide dense leaf block (paper-strict structure: 2^d b columns) travels in
  // column chunks of 64 (one tensor-TMA box each), so the stages stay U-sized
  // and the item keeps 64 rows.
  // Standard admissibility: the 3^d near-field blocks travel in 3 stages of
  // 3^(d-1) neighbours (d >= 2), so a dense stage is not larger than a U stage.
  p.ndc = (p.adm == 0 && leaf > 64 && leaf % 64 == 0) ? leaf / 64 : (p.adm && p.d >= 2 ? 3 : 1);
  p.dc = p.adm ? leaf : leaf / p.ndc;
  p.dgs = p.adm ? p.nd / p.ndc : 1;  // dense blocks (neighbours) per dense stage
  const int64_t dcp = p.dc + (p.dc & 1);
  p.Re = pick_rows(leaf, kConsumerThreads, std::max<int64_t>(p.Wp, int64_t(p.dgs) * dcp),
                   p.adm ? std::max<int64_t>(cap, 48 * 1024) : cap);
  p.tpr = 1;
  while (p.tpr * 2 <= 32 && p.tpr * 2 * p.Re <= kConsumerThreads) p.tpr *= 2;
  p.xs_p = static_cast<int>(round_up(p.Rp + 2, 2));
  p.xs_e = static_cast<int>(round_up(p.dc + 2, 2));
  p.stages_p = int64_t(depth) * (p.N_loc / p.Rp);
  p.items_e = p.N_loc / p.Re;
  const int np = p.Wp / 2;  // column pairs owned by project's consumer threads
  const int rg = np <= kConsumerThreads ? kConsumerThreads / np : 1;
  const int64_t bar_bytes = 1024;  // mbarriers + flag (256 B) + 2 x 32 neighbour entries
  p.grid_p_max = 0;
  for (int li = 0; li < 4; ++li) {
    const int64_t NR = int64_t(1) << li;
    if (NR > std::max(1, opt.max_nr)) break;  // widest SIMT pass allowed
    Plan::Layout& y = p.lay[li];
    y.stage_bytes_p = round_up(int64_t(p.Rp) * p.Wp * 8 + NR * p.xs_p * 8, 128);
    const int64_t zrows = opt.peer ? P : 1;  // peer exchange: one z row per rank on exchange levels
    y.stage_bytes_e = round_up(std::max(int64_t(p.Re) * p.Wp * 8 + int64_t(p.Wp) * NR * 8 * zrows,
                                        int64_t(p.dgs) * (int64_t(p.Re) * (p.dc + (p.dc & 1)) * 8 + NR * p.xs_e * 8)),
                               128);
    const int64_t red_bytes = round_up(2 * int64_t(rg) * p.Wp * NR * 8, 128);  // two alternating buffers
    // the requested CTAs per SM, or fewer if two pipeline stages do not fit
    for (int ctas = std::max(1, opt.ctas_per_sm); ctas >= 1; --ctas) {
      const int64_t budget = std::min<int64_t>(opt.smem_budget, 227 * 1024 / ctas - 1024);
      y.nstage_p = static_cast<int>(std::min<int64_t>(opt.max_stages_p, (budget - red_bytes - bar_bytes) / y.stage_bytes_p));
      y.nstage_e = static_cast<int>(std::min<int64_t>(opt.max_stages_e, (budget - bar_bytes) / y.stage_bytes_e));
      y.ctas_per_sm = ctas;
      if (y.nstage_p >= 2 && y.nstage_e >= 2) break;
    }
    if (y.nstage_p < 2 || y.nstage_e < 2) {
      if (li == 0) return "unsupported: pipeline stages do not fit in shared memory";
      break;  // wider right-hand-side passes do not fit: cap the pass width
    }
    p.max_nr = static_cast<int>(NR);
    y.red_off_p = y.nstage_p * y.stage_bytes_p;
    y.bar_off_p = y.red_off_p + red_bytes;
    y.bar_off_e = y.nstage_e * y.stage_bytes_e;
    y.smem_p = y.bar_off_p + bar_bytes;
    y.smem_e = y.bar_off_e + bar_bytes;
    const int64_t slots = int64_t(opt.num_sms) * y.ctas_per_sm;
    y.grid_p_slots = static_cast<int>(slots);
    y.grid_p = static_cast<int>(std::min<int64_t>(slots, depth > 0 ? p.N_loc / p.Rp : 0));
    y.grid_e = static_cast<int>(std::min<int64_t>(slots, p.items_e));
    p.grid_p_max = std::max(p.grid_p_max, y.grid_p);
  }
  // DMMA layouts (1 project CTA per SM: 2 stages of ~77 KB; 2 expand CTAs per SM)
  // W % 32 == 0: 4 column groups of W/32 M-tiles, 32-column expand chunks;
  // W % 16 == 0: 2 column groups of W/16 M-tiles (<= 7), 16-column chunks
  p.dkr = kDmmaKR;
  // expand k-chunk of a level stage: 32 columns (W % 32 == 0), the whole level at
  // W = 48 (the c2 / c4 shape: a third of the stages of 16-column chunks), else 16;
  // dense stages are 32 columns of D (kernels_dmma.cu KD)
  p.dkc = opt.dmma_kc > 0 ? opt.dmma_kc : p.W % 32 == 0 ? 32 : p.W % 48 == 0 ? 48 : 16;
  if (p.W % p.dkc != 0 || (p.dkc != 16 && p.dkc != 32 && p.dkc != 48)) p.dkc = p.W % 32 == 0 ? 32 : 16;
  // The project's column slice: the whole panel (weak admissibility), or for the
  // standard structure (W = M r, up to 1024 columns) the widest divisor WS of W
  // one CTA's register-resident node tile takes (WS % 16 == 0, WS <= 224 if
  // WS % 32 == 0, else <= 112); the slices are CTAs of a 2-D grid (one GPU only:
  // the boundary exchange of P > 1 stays on the SIMT kernels).
  int ws = p.W;
  if (p.adm) {
    ws = 0;
    for (int cand = 16; cand <= 224 && cand <= p.W; cand += 16)
      if (p.W % cand == 0 && (cand % 32 == 0 || cand <= 112)) ws = cand;
  }
  p.wslice = ws;
  p.nslice = ws > 0 ? p.W / ws : 0;
  p.dmma_ok = ws > 0 && p.W % 16 == 0 && (ws % 32 == 0 ? ws <= 224 : ws <= 112) &&
              leaf % kDmmaRE == 0 && leaf % p.dkr == 0 && p.N_loc % kDmmaRE == 0;
  if (p.dmma_ok) {
    p.vp = ws + ((4 - ws % 16) + 16) % 16;
    p.dnw = (ws % 32 != 0 && opt.dmma_nw == 8) ? 8 : 16;
    for (int li = 0; li < 4; ++li) {
      Plan::DmmaLayout& d = p.dl[li];
      d.nb = li == 3 ? 8 : 16 << li;
      // project warps: 64 / 32 wide as p.dnw; 16 wide: 8 (W % 32 == 0) or 4; 8 wide:
      // 4 or 2 (kernels_dmma.cu)
      // 8 wide, W = 48: 3 warps of 16 columns (5 CTAs per SM: more warps in flight than
      // 2 warps of 24; c2 4 rhs project 0.562 -> 0.533 ms, c4 8 rhs total unchanged)
      const int nw8 = opt.dmma8_nw > 0 && ws == 48 && 48 % (8 * opt.dmma8_nw) == 0 ? opt.dmma8_nw : 2;
      d.nw = d.nb == 8 ? (ws % 32 == 0 ? 4 : nw8) : d.nb == 16 ? (ws % 32 == 0 ? 8 : 4) : p.dnw;
      // V rows + the nb x columns (pitch dkr + 4 = 4 mod 16 doubles)
      d.dstage_p = round_up(int64_t(p.dkr) * p.vp * 8 + int64_t(d.nb) * (p.dkr + 4) * 8, 128);
      const int64_t kd = p.dkc == 16 ? 16 : 32;  // dense-stage columns (kernels_dmma.cu KD)
      d.dstage_e = round_up(std::max(int64_t(kDmmaRE) * (p.dkc + 4) * 8 + int64_t(p.dkc) * d.nb * 8,
                                     int64_t(kDmmaRE) * (kd + 4) * 8 + int64_t(d.nb) * (kd + 4) * 8),
                            128);
      // project CTAs per SM: 16 warps' worth (1 CTA of 16, 2 of 8, 4 of 4), fewer if
      // two stages do not fit (64 / 32 wide keep their measured budgets)
      int ctas = d.nb == 16 && opt.dmma16_ctas > 0 ? std::min(opt.dmma16_ctas, 16 / d.nw) : 16 / d.nw;
      const int cap_p = d.nb == 16 && opt.dmma16_max_stages > 0 ? opt.dmma16_max_stages : opt.dmma_max_stages_p;
      for (;; --ctas) {
        const int64_t pbudget = d.nb <= 16 ? 227 * 1024 / ctas - 1024 : (p.dnw == 8 ? 112 * 1024 : 226 * 1024);
        d.dns_p = static_cast<int>(std::min<int64_t>(std::max(2, cap_p), (pbudget - bar_bytes) / d.dstage_p));
        if (d.dns_p >= 2 || ctas == 1) break;
      }
      if (d.nb == 8) {
        // 8 wide: next to no math per stage, so the pass is a stream; a slot is
        // refilled only when all (2 or 4) warps are done with it, so about
        // ctas (stages - 1) stages per SM are in flight -- pick the split of the
        // shared memory that maximises it (ties: more CTAs) among >= 3 CTAs per
        // SM where they fit (c4, 8 rhs: 2 CTAs x 7 stages 12.0 ms, 3 x 4 10.7,
        // 6 x 2 10.7), or HMAT_DMMA8_CTAS
        int best = -1;
        for (int c = 16 / d.nw; c >= 1; --c) {
          if (opt.dmma8_ctas <= 0 && c < 3 && best >= 0) break;
          if (opt.dmma8_ctas > 0 && c != opt.dmma8_ctas) continue;
          const int64_t budget = 227 * 1024 / c - 1024;
          const int ns = static_cast<int>(std::min<int64_t>(opt.dmma8_max_stages, (budget - bar_bytes) / d.dstage_p));
          if (ns >= 2 && c * (ns - 1) > best) {
            best = c * (ns - 1);
            ctas = c;
            d.dns_p = ns;
          }
        }
      }
      // expand ring: 5 stages of 16-column chunks, 3 of wider ones (64 / 32 rhs);
      // narrow passes (<= 16 rhs) carry little math per stage, so deeper rings
      // keep more bytes in flight (HMAT_DMMA_STAGES_E caps them)
      const int cap_e = d.nb <= 16 && opt.dmma_stages_e_narrow > 0 ? opt.dmma_stages_e_narrow : (p.dkc == 16 ? 5 : 3);
      // CTAs per SM: 2 (112 KB each), or at 16 wide under weak admissibility 3
      // (A/B r02, ms per 16-rhs product, 2 -> 3 CTAs: c4 26.05 -> 25.37, c3 7.68 ->
      // 7.48, c2 1.233 -> 1.223; not the standard structure: s2 10.34 -> 10.82);
      // HMAT_DMMA_E_CTAS = 1..3 sets it for <= 16-wide passes
      const int ctas_e = d.nb <= 16 && opt.dmma_e_ctas >= 1 && opt.dmma_e_ctas <= 3 ? opt.dmma_e_ctas
                         : d.nb == 16 && !p.adm && opt.dmma_e_ctas == 0            ? 3
                                                                                   : 2;
      const int64_t ebudget = ctas_e == 2 ? 112 * 1024 : 227 * 1024 / ctas_e - 1024;
      d.dns_e = static_cast<int>(std::min<int64_t>(cap_e, (ebudget - bar_bytes) / d.dstage_e));
      d.dsmem_p = d.dns_p * d.dstage_p + bar_bytes;
      d.dsmem_e = d.dns_e * d.dstage_e + bar_bytes;
      d.dgrid_p = static_cast<int>(std::min<int64_t>(int64_t(opt.num_sms) * ctas, depth > 0 ? p.N_loc / p.dkr : 0));
      d.dgrid_e = static_cast<int>(std::min<int64_t>(int64_t(opt.num_sms) * ctas_e, p.N_loc / kDmmaRE));
      d.dgrid_e_gen = static_cast<int>(std::min<int64_t>(int64_t(opt.num_sms) * std::min(ctas_e, 2), p.N_loc / kDmmaRE));
      // (a 32-wide project pass with W % 32 != 0 needs the 8-warp grid: kernels_dmma.cu)
      const bool narrow_on = d.nb == kDmmaNB || (d.nb == 32   ? opt.dmma_narrow >= 1
                                                 : d.nb == 16 ? opt.dmma_narrow >= 2
                                                              : opt.dmma_narrow >= 3);
      d.ok = d.dns_p >= 2 && d.dns_e >= 2 && narrow_on && (d.nb != 32 || ws % 32 == 0 || p.dnw == 8);
      p.dgrid_p_max = std::max(p.dgrid_p_max, d.dgrid_p);
    }
    if (!p.dl[2].ok) p.dmma_ok = false;
  }
  *out = p;
  return "";
}

}  // namespace hmat
