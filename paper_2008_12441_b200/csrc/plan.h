// plan.h -- host-side plan of one H-matrix shard: validation, Morton/level
// arithmetic, device layout, the persistent-kernel schedule and the
// cross-GPU exchange layout.  Pure host code (testable without a GPU through
// hmat_plan_query()).
//
// Notation: c = 2^d children per node, L levels below the root,
// b points per leaf, N = b c^L, m_l = N / c^l rows per level-l node, W = (c-1) r
// panel width.  A shard owns the contiguous Morton rows [row0, row0 + N_loc),
// N_loc = N / P: whole subtrees at the partition level (PAPER.md:434-448,
// §3.1 process-tree rules; block-row factor placement PAPER.md:526-531).
#pragma once
#include <cstdint>
#include <string>

namespace hmat {

constexpr int kMaxLevels = 48;   // L <= 47
constexpr int kMaxNR = 8;        // right-hand sides per streaming pass
constexpr int kConsumerThreads = 256;
constexpr int kThreads = 32 + kConsumerThreads;  // 1 producer warp + 8 consumer warps

// standard admissibility: interaction-list slot tables (6^d - 3^d <= 189 slots,
// 3^d 2^d <= 216 (neighbour, child) codes)
constexpr int kStdMaxSlots = 192;
constexpr int kStdMaxCodes = 216;
// Host enumeration of the canonical slot order (include/hmat.h, standard panels):
// code[d-1][tau][q] = e 2^d + sigma of slot q, slot[d-1][tau][code] = q or -1.
void std_slot_tables(int16_t code[3][8][kStdMaxSlots], int16_t slot[3][8][kStdMaxCodes]);

// FP64 tensor-core (DMMA) path for many right-hand sides (kernels_dmma.cu)
constexpr int kDmmaNB = 64;   // right-hand sides per pass
constexpr int kDmmaKR = 32;   // project: V rows per stage
constexpr int kDmmaRE = 64;   // expand: rows per item
constexpr int kDmmaKC = 32;   // expand: k-columns per stage
constexpr int kDmmaXP = 36;   // smem pitch of staged x columns (= 4 mod 16 doubles)
constexpr int kDmmaAP = kDmmaKC + 4;  // smem pitch of staged U / D row chunks

struct Plan {
  // problem
  int d = 0, c = 0, L = 0, b = 0, r = 0, W = 0;
  // admissibility: 0 = weak (M = c-1 sibling slots, one dense leaf-diagonal
  // panel), 1 = standard (M = 6^d - 3^d interaction slots, nd = 3^d dense
  // near-field panels, one per neighbour offset); W = M r
  int adm = 0, M = 0, nd = 1;
  int64_t d_stride = 0;             // doubles between consecutive dense panels
  int64_t N = 0;
  int64_t m[kMaxLevels + 1] = {};   // m[l] = N / c^l
  // shard
  int P = 1, rank = 0;
  int64_t N_loc = 0, row0 = 0;
  // device layout (doubles)
  int Wp = 0, Dp = 0;               // row pitches of U/V panels and D (even => 16-B rows)
  int64_t panel_stride = 0;         // doubles between consecutive level panels (128-B multiple)
  // z storage per level l (target-major, per rhs-pass): Zt_l[t][rhs][col], Wp*NR per target
  // levels 1..cross live in the exchange buffer (all c^l targets), others in the
  // local buffer (this shard's targets only).
  int cross = 0;                    // levels 1..cross need the cross-GPU exchange (c^{l-1} < P)
  int64_t zt_off[kMaxLevels + 1] = {};    // offset in units of (Wp*kMaxNR) doubles
  int64_t zt_tbase[kMaxLevels + 1] = {};  // global index of the first stored target
  int64_t zt_count[kMaxLevels + 1] = {};
  int64_t z_local_rows = 0;         // targets stored in the local z buffer
  int64_t z_exch_rows = 0;          // targets stored in the exchange buffer
  // schedule
  int Rp = 0, Re = 0;               // rows per pipeline stage: project / expand (both divide b)
  int tpr = 0;
  int ndc = 1, dc = 0;              // expand: dense stages per item: weak = column chunks of dc columns,
  int dgs = 1;                      //   standard = groups of dgs near-field blocks                      // expand: threads per row
  int64_t stages_p = 0;             // L * N_loc / Rp
  int64_t items_e = 0;              // N_loc / Re
  int xs_p = 0, xs_e = 0;           // doubles reserved per rhs for x chunks in a stage
  // shared-memory layout and grid per right-hand-side capacity NR = 1, 2, 4, 8
  struct Layout {
    int ctas_per_sm = 0;
    int nstage_p = 0, nstage_e = 0;
    int64_t stage_bytes_p = 0, stage_bytes_e = 0;
    int64_t red_off_p = 0, bar_off_p = 0, bar_off_e = 0;  // byte offsets
    int64_t smem_p = 0, smem_e = 0;                        // dynamic smem per CTA
    int grid_p = 0, grid_e = 0;                            // persistent grids
    int grid_p_slots = 0;                                  // CTA slots (#SM x CTAs per SM)
  } lay[4];
  int grid_p_max = 0;               // partial-sum slots to allocate
  int max_nr = 1;                   // widest SIMT pass (<= kMaxNR) whose stages fit in smem
  // DMMA path (nrhs >= a threshold, W % 32 == 0, W <= 224, 64 | b)
  bool dmma_ok = false;
  int dmma_off = 0, dmma_min = 3, dbg = 0, expand_chunk = -1, project_dyn = 1, snake = 1, pdl = 2, lpar = 1, early = 1, eshape = 1, dmma_ileave = 1, project_chunk = 4, aflush = 1, dmma_upol = 1, dmma_pchunk = 32, dmma_pchunk16 = 16;  // from PlanOptions
  int vp = 0;                       // smem pitch of staged V rows (= 4 mod 16 doubles)
  int wslice = 0, nslice = 0;       // tensor-core project: column slice width / count (W = wslice nslice)
  int dkr = kDmmaKR;                // project: V rows (the GEMM's k) per stage
  int dkc = kDmmaKC;                // expand: k-columns per level stage (32; 48 at W = 48; else 16)
  int dnw = 16;                     // project: warps per CTA (16 at 1 CTA/SM, or 8 at 2 CTAs/SM)
  // one layout per pass width: dl[0] = 16 right-hand sides, dl[1] = 32, dl[2] = 64
  struct DmmaLayout {
    bool ok = false;
    int nb = 0;
    int nw = 0;                     // project warps per CTA
    int dns_p = 0, dns_e = 0;
    int64_t dstage_p = 0, dstage_e = 0, dsmem_p = 0, dsmem_e = 0;
    int dgrid_p = 0, dgrid_e = 0;
    int dgrid_e_gen = 0;            // expand grid of the general (not plain-product) variant: its
                                    // registers fit 2 CTAs per SM, not 3 (kernels_dmma.cu)
  } dl[4];                          // pass widths 16, 32, 64, and (dl[3]) 8
  int dgrid_p_max = 0;              // partial-sum / ticket slots to allocate (max over dl)
  // the layout of a pass of `nr` right-hand sides: the narrowest that holds them
  const DmmaLayout& dmma_layout(int nr) const {
    return nr <= 8 && dl[3].ok ? dl[3] : nr <= 16 && dl[0].ok ? dl[0] : nr <= 32 && dl[1].ok ? dl[1] : dl[2];
  }
};

// index into Plan::lay of a right-hand-side capacity 1, 2, 4 or 8
inline int nr_index(int nr_cap) { return nr_cap <= 1 ? 0 : nr_cap <= 2 ? 1 : nr_cap <= 4 ? 2 : 3; }

struct PlanOptions {
  int num_sms = 148;
  int ctas_per_sm = 2;
  int stage_cap_bytes = 36 * 1024;  // upper bound on the factor bytes of one stage
  int smem_budget = 200 * 1024;     // dynamic smem per CTA for the pipeline
  int max_stages_p = 3;             // project: measured best at 3 stages x 2 CTAs per SM (early slot release)
  int max_stages_e = 3;             // expand: measured best at 3 stages x 2 CTAs per SM
  int adm = 0;                      // structure: 0 = weak, 1 = standard admissibility
  int peer = 0;                     // P > 1 with the in-kernel peer exchange (expand stages hold P z rows)
  // per-call switches, read once at hmat_create (HMAT_* environment)
  int dmma_off = 0, dmma_min = 3;   // tensor-core path off / from this many rhs (measured crossover, 8-wide passes)
  int dbg = 0;                      // diagnostics (HMAT_DEBUG_SKIP)
  int expand_chunk = -1;            // expand items per dynamic chunk (-1 = default, 0 = static)
  int project_dyn = 1;              // project's last level in dynamic chunks
  int snake = 1;                    // project: alternate the stream direction per level
  int dmma_nw = 8;                  // DMMA project warps per CTA when W % 32 != 0 (8 or 16)
  int max_nr = 4;                   // widest SIMT right-hand-side pass (1, 2, 4 or 8): 8-wide passes
                                    // measured slower than two 4-wide ones (c3: 16.7 vs 14.2 ms)
  int dmma_max_stages_p = 3;        // DMMA project: pipeline depth cap
  int dmma_narrow = 3;              // DMMA narrow last passes: 0 = none, 1 = 32 wide, 2 = 32 or 16, 3 = 32, 16 or 8 wide
  int dmma_kc = 0;                  // DMMA expand k-columns per level stage (0 = auto: 32 / 48 / 16)
  int pdl = 2;                      // PDL: 0 off, 1 expand after project, 2 also project after the previous kernel
  int lpar = 1;                     // project: level-parallel mode for small operators
  int early = 1;                    // project: release a ring slot before the FMAs (1 rhs)
  int eshape = 1;                   // expand: compile-time consumer shapes (1 rhs, ExpShape)
  int dmma_ileave = 1;              // tensor-core expand: interleaved item order over the CTAs
  int project_chunk = 4;            // project: minimum stages per dynamic chunk of the last level
  int aflush = 1;                   // project: asynchronous node flushes (no CTA barrier per node)
  int dmma_upol = 1;                // tensor-core expand: L2 policy of the U / D boxes (0 first, 1 normal)
  int dmma8_ctas = 0;               // 8-wide tensor-core project: CTAs per SM (0 = auto)
  int dmma8_nw = 3;                 // 8-wide tensor-core project, W = 48: warps per CTA (2, 3 or 6; other W % 32 != 0: 2)
  int dmma8_max_stages = 8;         // 8-wide tensor-core project: ring depth cap
  int dmma_pchunk = 32;             // 8-wide tensor-core project: stages per level-interleaved chunk
  int dmma_pchunk16 = 16;           // 16-wide tensor-core project: the same (0 = level after level)
  int dmma_stages_e_narrow = 0;     // <= 16-wide tensor-core expand: ring depth cap (0: 5 / 3 as wider passes)
  int dmma16_ctas = 0;              // 16-wide tensor-core project: CTAs per SM (0 = auto: 16 warps' worth)
  int dmma16_max_stages = 0;        // 16-wide tensor-core project: ring depth cap (0 = dmma_max_stages_p)
  int dmma_e_ctas = 0;              // <= 16-wide tensor-core expand: CTAs per SM, 1-3 (0 = auto: 3 at 16 wide, weak; else 2)
};

// Validates arguments and fills `plan`.  Returns "" on success, else a message.
std::string plan_build(int depth, int dim, int leaf, int rank, int P, int shard, const PlanOptions& opt,
                       Plan* plan);

// q-th sibling of node t (ascending child order, skipping t) and the slot of
// sibling s in t's list (R6).
inline int64_t sibling_of(int c, int64_t t, int q) {
  int me = static_cast<int>(t % c);
  return (t / c) * c + (q < me ? q : q + 1);
}
inline int slot_of(int c, int64_t t, int64_t s) {
  int me = static_cast<int>(t % c), other = static_cast<int>(s % c);
  return other < me ? other : other - 1;
}

}  // namespace hmat
