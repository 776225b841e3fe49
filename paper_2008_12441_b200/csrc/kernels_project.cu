// kernels_project.cu -- Step 1 (source-side local computation) and the
// on-chip part of Step 2 (tree-reduction) of the H-matvec.
//
// For every level l and every source node s, z_{t,s} = V_{t,s}^T x_s
// (eq:prod-vx) for the c-1 targets t = siblings of s.  In the
// source-major V_l panel the rows of s are one contiguous m_l x W block, so the
// whole step is a segmented transposed GEMV over the level-major stream
// V_1 | V_2 | ... | V_L.
//
// Structure (persistent, warp-specialised):
//   * grid = #SM x CTAs/SM; each level's N_loc / Rp stages are split evenly
//     over the CTAs, CTA b owning [SL b / G, SL (b+1) / G) of every level, so
//     every CTA streams the same bytes and the same mix of coarse levels (one
//     node flush per many stages) and fine levels (one flush per stage).
//   * warp 0 (one elected lane) issues 1-D bulk TMA copies of each stage --
//     Rp rows of V_l (Rp * Wp doubles, contiguous) and the matching x segment --
//     into an nstage-deep shared-memory ring guarded by full/empty mbarriers.
//   * warps 1..8 own fixed columns of the panel and accumulate rows in
//     registers for as long as the node continues; at the node's end they
//     reduce across row groups in shared memory and write z.
//   * A node cut by a CTA-range boundary writes one partial per CTA; the last
//     CTA to arrive (atomic ticket) sums the partials in CTA order, so the
//     result is deterministic (the in-GPU analogue of the
//     paper's tree-reduction to the group leader).
//   * z is scattered target-major: Zt_l[t][slot(t -> s) r + a], the layout the
//     expand kernel reads (and, for levels above the partition level, the
//     packed exchange buffer of Steps 2-4).
#include "device_utils.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace hmat {
namespace {

constexpr int CT = kConsumerThreads;
constexpr int NCW = CT / 32;
constexpr int kEarlyRows = 7;  // rows per consumer thread and stage on the early-release path

// CTA owning stage k under the even split [S b / G, S (b+1) / G).
__device__ __forceinline__ int64_t owner_of(int64_t k, int64_t S, int64_t G) { return ((k + 1) * G - 1) / S; }

// z value (column col = q r + a of source node sg, rhs kk) -> Zt_l of target
// t = q-th sibling of sg, at slot(t -> sg).
// Standard admissibility: slot tables of the interaction lists,
// written by init_std_tables() from the host enumeration (plan.cpp):
//   c_std_code[d-1][tau][q]     = e * 2^d + sigma of slot q of a box with child
//                                 position tau (e = near-field index of the parent's
//                                 neighbour eps, sigma = child position of the source)
//   c_std_slot[d-1][tau][code]  = the inverse (-1 if the code is a neighbour).
__constant__ int16_t c_std_code[3][8][kStdMaxSlots];
__constant__ int16_t c_std_slot[3][8][kStdMaxCodes];

// z value of column col = q r + a of source node sg at `level` -> Zt of target
// t = slot q of sg, at slot(t -> sg).  nbr[e] = Morton index of sg's parent's
// neighbour e (-1 outside the domain), computed once per node.
template <int NR>
__device__ __forceinline__ void scatter_z_std(const StreamArgs& a, const LevelArgs& lv, int64_t sg,
                                              const int64_t* nbr, int col, int kk, double v) {
  const int d = a.d, c = a.c;
  const int q = col / a.r, aa = col - q * a.r;
  const int tau = static_cast<int>(sg & (c - 1));
  const int code = c_std_code[d - 1][tau][q];
  const int e = code >> d, sigma = code & (c - 1);
  const int64_t pt = nbr[e];
  if (pt < 0) return;  // the interaction partner lies outside the domain
  if (lv.xent) {       // P > 1: a cross-rank pair goes to the packed buffer
    const int32_t ent = lv.xent[(sg - lv.tbase) * (a.W / a.r) + q];
    if (ent >= 0) {
      a.xchg[((int64_t)ent * NR + kk) * a.r + aa] = v;
      return;
    }
  }
  const int64_t t = pt * c + sigma;
  const int nd = d == 1 ? 3 : d == 2 ? 9 : 27;
  const int qt = c_std_slot[d - 1][sigma][(nd - 1 - e) * c + tau];  // eps -> -eps, sigma <-> tau
  lv.zt[(t - lv.tbase) * (int64_t)a.Wp * NR + (int64_t)kk * a.Wp + qt * a.r + aa] = v;
}

// nbr[e] for the parent of source node sg at `level` (threads 0..nd-1).
__device__ __forceinline__ void std_parent_neighbours(const StreamArgs& a, int64_t sg, int level, int t,
                                                      int64_t* nbr) {
  if (t < a.nd) nbr[t] = geo::neighbour_k(a.d, sg >> a.d, t, level - 1);
}

template <int NR>
__device__ __forceinline__ void scatter_z(const StreamArgs& a, const LevelArgs& lv, int64_t sg, int col, int kk,
                                          double v) {
  const int d = __ffs(a.c) - 1;  // c = 2^d
  const int q = col / a.r, aa = col - q * a.r;
  const int me = static_cast<int>(sg & (a.c - 1));
  const int64_t t = ((sg >> d) << d) + (q < me ? q : q + 1);
  const int tc = static_cast<int>(t & (a.c - 1));
  const int qt = me < tc ? me : me - 1;
  lv.zt[(t - lv.tbase) * (int64_t)a.Wp * NR + (int64_t)kk * a.Wp + qt * a.r + aa] = v;  // [t][rhs][col]
}

// Compile-time consumer shapes (SH > 0, single rhs, one column pair per thread):
// the stage's row offsets become immediates and only the last row of a thread
// can fall outside the stage.  SH = 1: W = 48 (2D, r = 16: the c2 / c4 panels),
// 64-row stages; SH = 2: W = 224 (3D, r = 32: c3), 16-row stages.  SH = 0: any
// shape, from the runtime plan.
template <int SH>
struct ProjShape {
  static constexpr int NP = SH == 1 ? 24 : SH == 2 ? 112 : 0;  // column pairs (Wp / 2)
  static constexpr int RP = SH == 1 ? 64 : SH == 2 ? 16 : 0;   // rows per stage
  static constexpr int RG = NP ? kConsumerThreads / (NP ? NP : 1) : 0;  // row groups
  static constexpr int ROWS = NP ? (RP + RG - 1) / (RG ? RG : 1) : 0;   // rows per thread
  static constexpr int D = SH == 1 ? 2 : SH == 2 ? 3 : 0;               // dimension
  static constexpr int R = SH == 1 ? 16 : SH == 2 ? 32 : 0;             // rank
};

// scatter_z with the dimension and rank known at compile time (ProjShape)
template <int NR, int D, int R>
__device__ __forceinline__ void scatter_z_c(const StreamArgs& a, const LevelArgs& lv, int64_t sg, int col, int kk,
                                            double v) {
  constexpr int C = 1 << D, WP = (C - 1) * R;
  const int q = col / R, aa = col % R;
  const int me = static_cast<int>(sg & (C - 1));
  const int64_t t = ((sg >> D) << D) + (q < me ? q : q + 1);
  const int tc = static_cast<int>(t & (C - 1));
  const int qt = me < tc ? me : me - 1;
  lv.zt[(t - lv.tbase) * (int64_t)(WP * NR) + kk * WP + qt * R + aa] = v;  // [t][rhs][col]
}

template <int NR, int PAIRS, int SH = 0>
__global__ void __launch_bounds__(kThreads, 2) project_kernel(const __grid_constant__ StreamArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t G = gridDim.x, bid = blockIdx.x;
  const int Rp = a.Rp, W = a.W, Wp = a.Wp, L = a.L;
  const int64_t SL = a.N_loc / Rp;      // stages per level
  // Level-parallel mode (a.lpar, small operators): CTA b serves ONE stage of ONE
  // level -- the (b / SL)-th active level, stage b % SL -- so the levels' stage
  // loads and node flushes run side by side instead of one after the other in
  // every CTA (the whole pass is a few latencies long).  Otherwise each level is
  // split evenly over the GL CTAs.
  const bool lpar = a.lpar != 0;
  const int64_t GL = lpar ? SL : (G < SL ? G : SL);  // CTAs sharing a level
  const int64_t GS = lpar ? SL : G;                  // partial / ticket slots per level
  int my_level = 0;
  int64_t jb = bid;                                  // this CTA's index among GL
  if (lpar) {
    int nth = static_cast<int>(bid / SL);
    jb = bid - int64_t(nth) * SL;
    for (int l = 1; l <= L; ++l)
      if (((a.level_mask >> (l - 1)) & 1ull) && nth-- == 0) {
        my_level = l;
        break;
      }
  }
  const int NS = a.nstage_p;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off_p);
  uint64_t* empty = full + NS;
  volatile int* flag = reinterpret_cast<volatile int*>(empty + NS);
  volatile int* chunk_q = reinterpret_cast<volatile int*>(smem + a.bar_off_p + 768);  // [NS] chunk ids
  // asynchronous node flush (see the consumers): per reduction buffer, "all
  // consumer warps wrote their partials" and "its summing warps are done"
  uint64_t* rfull = reinterpret_cast<uint64_t*>(smem + a.bar_off_p + 160);
  uint64_t* rempty = rfull + 2;
  // summing warps per node: enough warps for the W NR outputs
  const int nsw = min(NCW, (W * NR + 31) / 32);
  // The last active level (a.dyn_level; 0 = none) is handed out dynamically in
  // chunks of a.dyn_chunk stages (whole nodes: no partial sums) from a global
  // counter, so CTAs that streamed the earlier levels faster take more of it
  // and all end together; the other levels keep the even static split.
  const int dyn_level = a.dyn_level;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      dev::mbar_init(&full[i], 1);
      dev::mbar_init(&empty[i], NCW);
    }
    for (int i = 0; i < 2; ++i) {
      dev::mbar_init(&rfull[i], NCW);
      dev::mbar_init(&rempty[i], nsw);
    }
    dev::fence_mbar_init();
  }
  __syncthreads();
  // PDL: wait for the previous kernel (e.g. the last product's expand, which may
  // have written this x) before any global access; let expand launch early
  if (a.pdl_p) dev::pdl_wait();
  if (a.pdl) dev::pdl_launch_dependents();  // expand may launch as SMs free up
  const dev::CtaTrace trace_scope(a.trace, bid);
  if (lpar ? my_level == 0 : bid >= GL) return;
  // every level is split evenly over the GL CTAs, so each CTA streams the same
  // mix of coarse and fine levels (fine levels flush a node per stage)
  const int64_t k0 = SL * jb / GL, k1 = SL * (jb + 1) / GL;  // this CTA's stages of each level

  if (warp == 0) {
    // ---------------- producer: one lane streams V_l rows + x segments -------
    if (lane == 0) {
      const uint64_t pol_stream = dev::policy_evict_first();
      const uint64_t pol_keep = dev::policy_evict_last();
      const uint32_t vbytes = static_cast<uint32_t>(Rp * Wp * 8);
      int slot = 0;
      uint32_t phase = 0;
      int next_c = -1;  // dynamic level: the chunk claimed ahead (its atomic's latency hidden)
      for (int l = 1; l <= L; ++l) {
        if (!((a.level_mask >> (l - 1)) & 1ull) || (lpar && l != my_level)) continue;
        const double* Vl = a.V + (l - 1) * a.panel_stride;
        const bool dyn = l == dyn_level;
        const bool rev = a.snake && !dyn && !(l & 1);  // even levels: the range backwards
        int64_t rk0 = k0, rk1 = k1;
        int chunk = -1;
        for (bool first_range = true;; first_range = false) {
        if (dyn) {
          const int c = next_c >= 0 ? next_c : atomicAdd(a.sched_p, 1);
          // claim the following chunk now: its round trip overlaps this chunk's copies
          next_c = int64_t(c) * a.dyn_chunk < SL ? atomicAdd(a.sched_p, 1) : -1;
          if (int64_t(c) * a.dyn_chunk >= SL) {
            // end of work: an empty phase with chunk id -1 tells the consumers
            dev::mbar_wait(&empty[slot], phase ^ 1);
            chunk_q[slot] = -1;
            dev::mbar_arrive(&full[slot]);
            if (++slot == NS) {
              slot = 0;
              phase ^= 1;
            }
            if (atomicAdd(a.sched_p + 1, 1) == static_cast<int>(GL) - 1) {  // re-arm for the next launch
              a.sched_p[0] = 0;
              a.sched_p[1] = 0;
            }
            break;
          }
          chunk = c;
          rk0 = int64_t(c) * a.dyn_chunk;
          rk1 = rk0 + a.dyn_chunk < SL ? rk0 + a.dyn_chunk : SL;
        } else if (!first_range) {
          break;
        }
        const int64_t dk = rev ? -1 : 1;
        int64_t k = rev ? rk1 - 1 : rk0;
        for (int64_t n = rk1 - rk0; n > 0; --n, k += dk) {
          // the stage's addresses first, then wait for the slot (the refill
          // latency is on the stream's critical path)
          const int64_t i0 = k * Rp;
          unsigned char* st = smem + slot * a.stage_bytes_p;
          uint32_t total = vbytes;
          int64_t lo[NR];
          uint32_t xb[NR];
#pragma unroll
          for (int kk = 0; kk < NR; ++kk) {
            if (kk < a.nr) {
              const int64_t start = kk * a.ldx + i0;
              lo[kk] = start & ~int64_t(1);
              xb[kk] = static_cast<uint32_t>((((start + Rp + 1) & ~int64_t(1)) - lo[kk]) * 8);
              total += xb[kk];
            }
          }
          dev::mbar_wait(&empty[slot], phase ^ 1);  // fresh barrier: parity 1 passes at once
          if (dyn && k == rk0) chunk_q[slot] = chunk;  // the chunk travels with its first stage
          dev::mbar_arrive_expect_tx(&full[slot], total);
          dev::bulk_g2s(st, Vl + i0 * Wp, vbytes, &full[slot], pol_stream);
#pragma unroll
          for (int kk = 0; kk < NR; ++kk)
            if (kk < a.nr)
              dev::bulk_g2s(st + vbytes + kk * a.xs_p * 8, a.x + lo[kk], xb[kk], &full[slot], pol_keep);
          if (++slot == NS) {
            slot = 0;
            phase ^= 1;
          }
        }
        }
      }
    }
    return;
  }

  // ---------------- consumers ------------------------------------------------
  const int t = tid - 32;
  // each thread owns column pair(s) cp (columns 2cp, 2cp+1; Wp is even) and,
  // when the pairs fit in one pass (PAIRS == 1), the rows rho, rho+RG, ...
  using Sh = ProjShape<SH>;
  const int NP = SH ? Sh::NP : Wp >> 1;
  const int RG = SH ? Sh::RG : PAIRS == 1 ? CT / NP : 1;
  const int rho = PAIRS == 1 ? t / NP : 0;
  const int cp0 = PAIRS == 1 ? t - rho * NP : t;
  const bool active = PAIRS == 1 ? rho < RG : true;
  // single rhs, one column pair per thread, at most 8 rows per thread per stage:
  // the early-release path (a.early, HMAT_PROJECT_EARLY)
  const bool early = SH || (NR == 1 && PAIRS == 1 && a.early && Rp <= kEarlyRows * RG);
  const int64_t red_elems = (int64_t)RG * Wp * NR;  // one of two alternating buffers
  double* red_base = reinterpret_cast<double*>(smem + a.red_off_p);
  int64_t* nbr_base = reinterpret_cast<int64_t*>(smem + a.bar_off_p + 256);  // 2 x 32 entries
  int red_buf = 0;
  // async flush phases (all threads): bit b = rfull[b]'s, bit 2 + b = rempty[b]'s
  // (one register: a per-buffer array indexed at run time would live in local memory)
  uint32_t ph_bits = 0u;
  int nflush = 0;                                   // async flushes so far (rotates the summing warps)
  const int cw = warp - 1;                          // consumer warp index
  const bool async_flush = a.aflush != 0;
  double2 acc[PAIRS][NR];
#pragma unroll
  for (int j = 0; j < PAIRS; ++j)
#pragma unroll
    for (int kk = 0; kk < NR; ++kk) acc[j][kk] = make_double2(0.0, 0.0);

  int slot = 0;
  uint32_t phase = 0;
  for (int l = 1; l <= L; ++l) {
    if (!((a.level_mask >> (l - 1)) & 1ull) || (lpar && l != my_level)) continue;
    const LevelArgs& lv = a.lv[l];
    const bool dyn = l == dyn_level;
    // Even levels stream the CTA's range backwards: the x segments read last at
    // level l - 1 (still in L2, evict_last) are the first ones read at level l,
    // instead of a cyclic sweep through more x than L2 holds (all misses).
    const bool rev = a.snake && !dyn && !(l & 1);
    const int64_t sg0 = a.row0 / lv.m;
    // node cursor: seg stages per local node, sl = node index, pos = stage in node
    const int64_t seg = lv.seg_rows / Rp;
    int64_t rk0 = k0, rk1 = k1;
    for (bool first_range = true;; first_range = false) {
    bool peeked = false;
    if (dyn) {  // the next stage is the first of the producer's next chunk (or the end mark)
      dev::mbar_wait(&full[slot], phase);
      const int c = chunk_q[slot];
      if (c < 0) {
        if (++slot == NS) {
          slot = 0;
          phase ^= 1;
        }
        break;
      }
      rk0 = int64_t(c) * a.dyn_chunk;
      rk1 = rk0 + a.dyn_chunk < SL ? rk0 + a.dyn_chunk : SL;
      peeked = true;
    } else if (!first_range) {
      break;
    }
    // (32-bit cursors: stages per level and per node fit; fewer live registers)
    const int dk = rev ? -1 : 1;
    int64_t k = rev ? rk1 - 1 : rk0;
    int64_t sl = k / seg;
    const int pos0 = static_cast<int>(k - sl * seg);
    int left = rev ? pos0 + 1 : static_cast<int>(seg) - pos0;  // stages to the node's end, stream order
    for (int n = static_cast<int>(rk1 - rk0); n > 0; --n, k += dk) {
      if (!peeked) dev::mbar_wait(&full[slot], phase);
      peeked = false;
      const int64_t i0 = k * Rp;
      const unsigned char* st = smem + slot * a.stage_bytes_p;
      const double2* V2 = reinterpret_cast<const double2*>(st);
      const double* xs = reinterpret_cast<const double*>(st + (SH ? Sh::RP * Sh::NP * 16 : Rp * Wp * 8));
      int xo[NR];
#pragma unroll
      for (int kk = 0; kk < NR; ++kk)  // (one rhs, even stage rows: the segment starts aligned)
        xo[kk] = SH ? 0 : kk * a.xs_p + static_cast<int>((kk * a.ldx + i0) & 1);
      if (SH) {
        // compile-time shape: immediate row offsets; rows below the last one are
        // always inside the stage
        constexpr int RWS = Sh::ROWS > 0 ? Sh::ROWS : 1;
        double2 v[RWS];
        double xv[RWS];
        const double2* vp = V2 + rho * Sh::NP + cp0;
        const double* xp = xs + rho;
#pragma unroll
        for (int i = 0; i < RWS; ++i) {
          const bool last = (i + 1) * Sh::RG > Sh::RP;  // may pass the stage's end
          const int off = last ? min(i * Sh::RG, Sh::RP - 1 - rho) : i * Sh::RG;
          v[i] = vp[off * Sh::NP];
          xv[i] = xp[off];
        }
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&empty[slot]);
        if (active && !(a.dbg & 1)) {
#pragma unroll
          for (int i = 0; i < RWS; ++i) {
            const bool last = (i + 1) * Sh::RG > Sh::RP;
            const double xi = (!last || rho + i * Sh::RG < Sh::RP) ? xv[i] : 0.0;
            acc[0][0].x = fma(v[i].x, xi, acc[0][0].x);
            acc[0][0].y = fma(v[i].y, xi, acc[0][0].y);
          }
        }
      } else if (NR == 1 && PAIRS == 1 && early) {
        // early release: the thread's rows of the stage (<= kEarlyRows) go to
        // registers, the slot is handed back to the producer, then the FMAs run --
        // the ring slot is held for the shared-memory loads only, not for the math
        double2 v[kEarlyRows];
        double xv[kEarlyRows];
#pragma unroll
        for (int i = 0; i < kEarlyRows; ++i) {
          const int row = min(rho + i * RG, Rp - 1);  // clamped: in-bounds, unused beyond Rp
          v[i] = V2[row * NP + cp0];
          xv[i] = xs[xo[0] + row];
        }
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&empty[slot]);
        if (active && !(a.dbg & 1)) {
#pragma unroll
          for (int i = 0; i < kEarlyRows; ++i) {
            const double xi = rho + i * RG < Rp ? xv[i] : 0.0;
            acc[0][0].x = fma(v[i].x, xi, acc[0][0].x);
            acc[0][0].y = fma(v[i].y, xi, acc[0][0].y);
          }
        }
      } else if (active && !(a.dbg & 1)) {
#pragma unroll 4
        for (int row = rho; row < Rp; row += RG) {
          double xv[NR];
#pragma unroll
          for (int kk = 0; kk < NR; ++kk) xv[kk] = xs[xo[kk] + row];
#pragma unroll
          for (int j = 0; j < PAIRS; ++j) {
            const int cp = cp0 + j * CT;
            if (PAIRS == 1 || cp < NP) {
              const double2 v = V2[row * NP + cp];
#pragma unroll
              for (int kk = 0; kk < NR; ++kk) {
                acc[j][kk].x = fma(v.x, xv[kk], acc[j][kk].x);
                acc[j][kk].y = fma(v.y, xv[kk], acc[j][kk].y);
              }
            }
          }
        }
      }
      if (!(SH || (NR == 1 && PAIRS == 1 && early))) {
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&empty[slot]);
      }
      if (++slot == NS) {
        slot = 0;
        phase ^= 1;
      }
      const bool node_end = --left == 0;
      const int64_t this_sl = sl;
      if (node_end) {
        left = static_cast<int>(seg);
        sl += dk;
      }
      if (!node_end && n != 1) continue;
      if ((a.dbg & 4) && node_end) continue;  // diagnostics: skip node flushes entirely (wrong z)

      // ---- end of a (local) node, or end of this CTA's range of the level ----
      const int64_t sa = this_sl * seg, sb = sa + seg;  // the node's stages
      const bool complete = sa >= rk0 && sb <= rk1;
      const int64_t sg = sg0 + this_sl;                 // global source node
      const int rb = red_buf;
      double* red = red_base + rb * red_elems;
      int64_t* nbr = nbr_base + rb * 32;  // standard admissibility: parent's neighbours
      red_buf ^= 1;  // alternate buffers: one barrier per complete node suffices
      // the buffer is free once the summing warps of its last asynchronous use
      // are done (a fresh barrier's parity 1 passes at once)
      dev::mbar_wait(&rempty[rb], ((ph_bits >> (2 + rb)) & 1u) ^ 1u);
      if (a.adm) std_parent_neighbours(a, sg, l, t, nbr);
      if (active) {
#pragma unroll
        for (int j = 0; j < PAIRS; ++j) {
          const int cp = cp0 + j * CT;
          if (PAIRS == 1 || cp < NP) {
#pragma unroll
            for (int kk = 0; kk < NR; ++kk) {
              reinterpret_cast<double2*>(red + ((int64_t)rho * NR + kk) * Wp)[cp] = acc[j][kk];
              acc[j][kk] = make_double2(0.0, 0.0);
            }
          }
        }
      }
      if (complete && async_flush) {
        // Asynchronous flush of a complete node: every warp posts its partials
        // and moves on to the next stage; only this node's nsw summing warps
        // (rotating, so the work spreads over all warps) wait for the other
        // warps' partials, sum the RG row groups and scatter z.  No CTA-wide
        // barrier per node: at the finest level (one node per stage) the
        // barrier held every warp to the slowest one each stage.
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&rfull[rb]);
        const int rel = (cw - nflush * nsw % NCW + NCW) % NCW;
        if (rel < nsw) {
          dev::mbar_wait(&rfull[rb], (ph_bits >> rb) & 1u);
          for (int o = rel * 32 + lane; o < W * NR; o += nsw * 32) {
            const int kk = o / W, col = o - kk * W;
            double v = 0.0;
            for (int g = 0; g < RG; ++g) v += red[((int64_t)g * NR + kk) * Wp + col];
            if (kk < a.nr) {
              if constexpr (SH != 0) scatter_z_c<NR, Sh::D, Sh::R>(a, lv, sg, col, kk, v);
              else if (a.adm) scatter_z_std<NR>(a, lv, sg, nbr, col, kk, v);
              else scatter_z<NR>(a, lv, sg, col, kk, v);
            }
          }
          __syncwarp();
          if (lane == 0) dev::mbar_arrive(&rempty[rb]);
        }
        ph_bits ^= 5u << rb;  // flip bits rb and 2 + rb
        ++nflush;
        continue;
      }
      dev::named_bar_sync(1, CT);
      if (complete && (a.dbg & 8)) continue;  // diagnostics: barrier only, no reduction / store
      if (complete) {
        for (int o = t; o < W * NR; o += CT) {
          const int kk = o / W, col = o - kk * W;
          double v = 0.0;
          for (int g = 0; g < RG; ++g) v += red[((int64_t)g * NR + kk) * Wp + col];
          if (kk < a.nr) {
            if (a.adm) scatter_z_std<NR>(a, lv, sg, nbr, col, kk, v);
            else scatter_z<NR>(a, lv, sg, col, kk, v);
          }
        }
      } else {
        // partial node sum of this CTA: slot 0 if the node holds our first
        // stage of the level, slot 1 otherwise (it then holds our last one)
        const int myslot = sa <= k0 ? 0 : 1;
        double* pp = a.part + (((int64_t)(l - 1) * GS + jb) * 2 + myslot) * (int64_t)Wp * NR;
        for (int o = t; o < W * NR; o += CT) {
          const int kk = o / W, col = o - kk * W;
          double v = 0.0;
          for (int g = 0; g < RG; ++g) v += red[((int64_t)g * NR + kk) * Wp + col];
          pp[(int64_t)kk * Wp + col] = v;
        }
        __threadfence();
        dev::named_bar_sync(1, CT);
        const int64_t b0 = owner_of(sa, SL, GL), b1 = owner_of(sb - 1, SL, GL);
        int* ticket = a.cnt + (int64_t)(l - 1) * GS + b1;
        if (t == 0) {
          const int prev = atomicAdd(ticket, 1);
          *flag = (prev == static_cast<int>(b1 - b0)) ? 1 : 0;
        }
        dev::named_bar_sync(1, CT);
        if (*flag) {
          __threadfence();
          // partial i = 0..nb: CTA b0 + i's slot (slot0 for i = 0, slot 0 after);
          // consecutive CTAs' slot-0 partials are 2 ps doubles apart
          const int slot0 = (sa == SL * b0 / GL) ? 0 : 1;
          const int64_t ps = (int64_t)Wp * NR, nb = b1 - b0;
          const double* p0 = a.part + (((int64_t)(l - 1) * GS + b0) * 2 + slot0) * ps;
          const double* p1 = a.part + (((int64_t)(l - 1) * GS + b0 + 1) * 2) * ps;
          const int WN = W * NR;
          // few outputs (W NR < CT): spl threads per output, thread s summing the
          // partials i = s mod spl in order, then the spl sums in order (smem)
          const int spl = WN < CT ? CT / WN : 1;
          if (spl > 1) {
            if (t < spl * WN) {
              const int o = t % WN, s = t / WN;
              const int kk = o / W, col = o - kk * W;
              const int64_t off = (int64_t)kk * Wp + col;
              double v = 0.0;
              if (s == 0) {
                v = dev::ld_cg(p0 + off);
                v = dev::sum_cg(v, p1 + (spl - 1) * 2 * ps + off, spl * 2 * ps, nb / spl);
              } else if (s <= nb) {
                v = dev::sum_cg(v, p1 + (s - 1) * 2 * ps + off, spl * 2 * ps, (nb - s) / spl + 1);
              }
              red[t] = v;
            }
            dev::named_bar_sync(1, CT);
          }
          for (int o = t; o < WN; o += CT) {
            const int kk = o / W, col = o - kk * W;
            double v = 0.0;
            if (spl > 1) {
              for (int s = 0; s < spl; ++s) v += red[s * WN + o];
            } else {
              const int64_t off = (int64_t)kk * Wp + col;
              v = dev::sum_cg(dev::ld_cg(p0 + off), p1 + off, 2 * ps, nb);
            }
            if (kk < a.nr) {
              if (a.adm) scatter_z_std<NR>(a, lv, sg, nbr, col, kk, v);
              else scatter_z<NR>(a, lv, sg, col, kk, v);
            }
          }
          if (t == 0) *ticket = 0;  // re-arm for the next launch
        }
        dev::named_bar_sync(1, CT);  // *flag is rewritten by the next partial node
      }
    }
    }
  }
  if (a.peer) peer_push<CT>(a, t, GL, flag);
}

template <int NR, int PAIRS, int SH>
cudaError_t launch_sh(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if (a.pdl_p) return launch_pdl(project_kernel<NR, PAIRS, SH>, a, grid, kThreads, smem, s);
  project_kernel<NR, PAIRS, SH><<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

// compile-time shape of this launch (ProjShape), 0 = generic
int project_shape(const StreamArgs& a, int nr_cap) {
  if (nr_cap != 1 || !a.early || a.adm || a.lpar) return 0;
  if (a.Wp == 2 * ProjShape<1>::NP && a.Rp == ProjShape<1>::RP && a.d == ProjShape<1>::D && a.r == ProjShape<1>::R)
    return 1;
  if (a.Wp == 2 * ProjShape<2>::NP && a.Rp == ProjShape<2>::RP && a.d == ProjShape<2>::D && a.r == ProjShape<2>::R)
    return 2;
  return 0;
}

template <int NR>
cudaError_t launch_nr(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if (NR == 1) {
    const int sh = project_shape(a, NR);
    if (sh == 1) return launch_sh<NR, 1, 1>(a, grid, smem, s);
    if (sh == 2) return launch_sh<NR, 1, 2>(a, grid, smem, s);
  }
  if ((a.Wp >> 1) <= CT) return launch_sh<NR, 1, 0>(a, grid, smem, s);
  return launch_sh<NR, 2, 0>(a, grid, smem, s);
}

template <int NR>
cudaError_t configure_nr(int64_t smem) {
  cudaError_t e = cudaFuncSetAttribute(project_kernel<NR, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (NR == 1) {
    if ((e = cudaFuncSetAttribute(project_kernel<NR, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) ||
        (e = cudaFuncSetAttribute(project_kernel<NR, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
      return e;
  }
  return cudaFuncSetAttribute(project_kernel<NR, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace

cudaError_t launch_project(const StreamArgs& a, int nr_cap, int grid, int64_t smem, cudaStream_t s) {
  switch (nr_cap) {
    case 1: return launch_nr<1>(a, grid, smem, s);
    case 2: return launch_nr<2>(a, grid, smem, s);
    case 4: return launch_nr<4>(a, grid, smem, s);
    default: return launch_nr<8>(a, grid, smem, s);
  }
}

cudaError_t init_std_tables(const int16_t* code, const int16_t* slot) {
  cudaError_t e = cudaMemcpyToSymbol(c_std_code, code, sizeof(int16_t) * 3 * 8 * kStdMaxSlots);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_std_slot, slot, sizeof(int16_t) * 3 * 8 * kStdMaxCodes);
}

cudaError_t configure_project(int64_t smem) {
  cudaError_t e;
  if ((e = configure_nr<1>(smem))) return e;
  if ((e = configure_nr<2>(smem))) return e;
  if ((e = configure_nr<4>(smem))) return e;
  return configure_nr<8>(smem);
}

}  // namespace hmat
