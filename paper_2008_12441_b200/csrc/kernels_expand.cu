// kernels_expand.cu -- Step 5 (target-side local computation) of the
// H-matvec, fused over all sibling blocks, all levels and
// the dense leaf-diagonal blocks so that y is written exactly once:
//
//   y_i = sum_{l=1..L} U_l[i, :] . Zt_l[t_l(i), :]      (eq:prod-yuz, all q)
//       + D_k[i, :] . x_k                                (eq:prod-ydz / eq:prod-dx)
//
// with t_l(i) = i / m_l, Zt_l[t] = concat_q z_{t, s_q} (written by project),
// k = i / b the leaf of row i.  (Under weak admissibility the dense blocks are
// leaf-diagonal and never cross a shard, so their source
// x_k is local and the paper's z_local = d_p x_p pass-through is not needed.)
//
// Structure (persistent, warp-specialised): CTA b owns an even, contiguous
// range of row tiles ("items") of Re rows (Re | b).  Per item the producer lane
// streams, by 1-D bulk TMA, U_1 rows + Zt_1 row, ..., U_L rows + Zt_L row,
// D rows + the leaf's x segment through an nstage-deep smem ring.  Consumer
// threads own (row, column-subset) pairs: tpr threads per row, interleaved
// columns visited in a row-rotated order (bank-conflict-free for the row
// pitches used here), fp64 FMAs into registers, a shuffle reduction across
// the tpr lanes, one store of y per row and rhs.
#include "device_utils.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace hmat {

cudaError_t configure_project(int64_t smem);

namespace {

constexpr int CT = kConsumerThreads;
constexpr int NCW = CT / 32;

// Order of an item's stages: levels 1..L, then the dense block (L + 1).  With
// the peer exchange the levels 1..cross wait for other ranks' flags, so they go
// last: local levels and the dense block first (overlap).
// Stages L+1 .. L+ndc are the dense block's column chunks.
__device__ __forceinline__ int level_order(const StreamArgs& a, int li) {
  if (!a.peer) return li;
  const int nloc = a.L + a.ndc - a.cross;
  return li <= nloc ? li + a.cross : li - nloc;
}

// Compile-time consumer shapes (1 rhs, weak admissibility, one dense stage,
// no peer exchange): tpr threads per row, NJU U / NJD D column pairs per
// thread.  The per-thread smem offsets are then a base register plus
// immediates, so a U stage is NJU x (2 LDS.128 + 2 DFMA) and little else --
// fewer issue slots and less power per byte streamed (the kernel runs under
// the board's power cap next to project).  SH = 1: W = 48 (c1, c2, c4), SH = 2:
// W = 224 (c3); both with b = 64.  SH = 3: standard admissibility in 2-D with
// r = 16, b = 64, one GPU (s2): W = 27 r = 432, one row per warp (Re = 8), the
// 3 x 3 near-field blocks in 3 dense stages of 3.
template <int SH>
struct ExpShape {
  static constexpr int TPR = SH == 1 ? 4 : SH == 2 ? 16 : 32;
  static constexpr int NJU = SH == 1 ? 6 : SH == 2 ? 7 : 0;
  static constexpr int NJD = SH == 1 ? 8 : SH == 2 ? 2 : 1;
};
constexpr int kStd2NP = 27 * 16 / 2;  // SH = 3: U column pairs

template <int NR, int SH = 0>
__global__ void __launch_bounds__(kThreads, 2) expand_kernel(const __grid_constant__ StreamArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t G = gridDim.x, bid = blockIdx.x;
  // items [item0, item0 + items_e) of the shard (item0 > 0: one of the row
  // chunks of a host-y product, whose copy out overlaps the next chunk)
  const int64_t ib = a.item0;
  const int64_t j0 = ib + a.items_e * bid / G, j1 = ib + a.items_e * (bid + 1) / G;
  const int Re = a.Re, W = a.W, Wp = a.Wp, Dp = a.Dp, b = a.b, L = a.L;
  const int NS = a.nstage_e;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off_e);
  uint64_t* empty = full + NS;
  volatile int* chunk_q = reinterpret_cast<volatile int*>(smem + a.bar_off_e + 512);  // [NS] chunk ids
  const bool dyn = a.chunk_e > 0;
  const int64_t nchunks = dyn ? (a.items_e + a.chunk_e - 1) / a.chunk_e : 0;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      dev::mbar_init(&full[i], 1);
      dev::mbar_init(&empty[i], NCW);
    }
    dev::fence_mbar_init();
  }
  __syncthreads();
  if (a.pdl) dev::pdl_wait();  // project (Zt, x staging) complete and visible
  if (a.pdl_p) dev::pdl_launch_dependents();  // the next product's project may launch as SMs free up
  const dev::CtaTrace trace_scope(a.trace, bid);

  if (warp == 0) {
    // ---------------- producer (the whole warp: lane e owns dense block e) ----
    const uint64_t pol_stream = dev::policy_evict_first();
    const uint64_t pol_keep = dev::policy_evict_last();
    int slot = 0;
    uint32_t phase = 0;
    const int64_t ipl = b / Re;                        // items per leaf
    int64_t leaf0 = 0, in_leaf = 0;
    // dense source of lane e: the leaf itself (weak) or its near-field
    // neighbour e (standard; -1 when it lies outside the domain)
    int64_t leaf_idx = 0;
    const int dd = __ffs(a.c) - 1;  // c = 2^d
    // (P > 1, standard: a neighbour on another rank -- local row offset < 0 or
    // >= N_loc -- is read from the packed buffer's halo entry, whose rhs
    // columns are bpad apart).  kNone: this lane has no dense block.
    // The lane's x source: xsrc + kk xld for rhs kk.
    constexpr int64_t kNone = INT64_MIN;
    const double* xsrc = a.x;
    int64_t xld = a.ldx;
    auto dense_source = [&]() -> int64_t {
      xsrc = a.x;
      xld = a.ldx;
      if (!a.adm) return lane == 0 ? leaf0 : kNone;
      if (lane >= a.nd) return kNone;
      const int64_t nb = geo::neighbour_k(a.d, leaf_idx, lane, L);
      if (nb < 0) return kNone;
      if (a.halo_of) {
        const int h = a.halo_of[(leaf_idx - a.row0 / b) * a.nd + lane];
        if (h >= 0 && a.skip_remote) return kNone;  // H^T: that product arrives in the exchange
        if (h >= 0) {
          xsrc = a.xchg + a.halo_base;
          xld = a.bpad;
          return (int64_t)h * NR * a.bpad;
        }
      }
      return nb * b - a.row0;
    };
    int64_t src = kNone;
    bool peers_ready = false;
    const uint32_t db = static_cast<uint32_t>(Re * Dp * 8);
    const int64_t dblk = db + int64_t(NR) * a.xs_e * 8;
    // Work: the static range [j0, j1), or (a.chunk_e > 0) chunks of chunk_e items
    // taken from a global counter -- the CTAs that stream faster take more
    // chunks, so they all finish within one chunk of each other (no tail).  The
    // first stage of a chunk carries its id to the consumers (chunk_q[slot]).
    int64_t cj0 = j0, cj1 = j1;
    int chunk = -1;
    bool first_range = true, first_stage = false;
    auto next_range = [&]() -> bool {
      if (!dyn) {
        const bool r = first_range && j0 < j1;
        first_range = false;
        return r;
      }
      int c = 0;
      if (lane == 0) c = atomicAdd(a.sched, 1);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (c >= nchunks) {
        // end of work: an empty phase with chunk id -1 tells the consumers
        dev::mbar_wait(&empty[slot], phase ^ 1);
        if (lane == 0) {
          chunk_q[slot] = -1;
          dev::mbar_arrive(&full[slot]);
          // the last CTA to run out re-arms the counters for the next launch
          if (atomicAdd(a.sched + 1, 1) == static_cast<int>(G) - 1) {
            a.sched[0] = 0;
            a.sched[1] = 0;
          }
        }
        return false;
      }
      chunk = c;
      cj0 = ib + int64_t(c) * a.chunk_e;
      cj1 = cj0 + a.chunk_e < ib + a.items_e ? cj0 + a.chunk_e : ib + a.items_e;
      first_stage = true;
      return true;
    };
    while (next_range()) {
    leaf0 = (cj0 * Re / b) * b;
    in_leaf = (cj0 * Re - leaf0) / Re;
    leaf_idx = (a.row0 + leaf0) / b;
    src = dense_source();
    for (int64_t j = cj0; j < cj1; ++j) {
      const int64_t i0 = j * Re;
      for (int li = 1; li <= L + a.ndc; ++li) {
        const int l = level_order(a, li);
        const bool is_d = (l > L);
        if (is_d ? !a.dense : !((a.level_mask >> (l - 1)) & 1ull)) continue;
        // Everything about the stage is computed BEFORE waiting for its slot:
        // the slot's refill latency (release -> copies issued) is on the
        // critical path of the stream, the address arithmetic is not.
        unsigned char* st = smem + slot * a.stage_bytes_e;
        if (!is_d) {
          const uint32_t ub = static_cast<uint32_t>(Re * Wp * 8);
          const uint32_t zb = static_cast<uint32_t>(Wp * NR * 8);
          const LevelArgs& lv = a.lv[l];
          // target node of the item at level l: m_l = b c^{L-l}, so the leaf's
          // index shifted right by d (L - l) bits (no 64-bit division)
          const int64_t tg = leaf_idx >> (dd * (L - l));
          const double* zrow = lv.zt + (tg - lv.tbase) * (int64_t)Wp * NR;
          const double* usrc = a.U + (l - 1) * a.panel_stride + i0 * Wp;
          dev::mbar_wait(&empty[slot], phase ^ 1);  // fresh barrier: parity 1 passes at once
          if (lane == 0 && first_stage) chunk_q[slot] = chunk;
          first_stage = false;
          if (lane == 0) {
            if (a.peer && l <= a.cross) {
              // peer exchange: the P ranks' contributions sit in this rank's
              // mailbox slots; wait once for every rank's flag of this pass
              const int par = static_cast<int>(a.epoch & 1);
              const double* mb = a.mbox[a.rank] + (int64_t)par * a.P * a.mb;
              if (!peers_ready) {
                peer_wait_flags(a);  // bounded; a timeout is reported through a.err
                dev::fence_proxy_async_global();
                peers_ready = true;
              }
              const int64_t off = zrow - a.zex_base;
              dev::mbar_arrive_expect_tx(&full[slot], ub + a.P * zb);
              dev::bulk_g2s(st, usrc, ub, &full[slot], pol_stream);
              for (int g = 0; g < a.P; ++g)
                dev::bulk_g2s(st + ub + g * zb, mb + g * a.mb + off, zb, &full[slot], pol_keep);
            } else {
              dev::mbar_arrive_expect_tx(&full[slot], ub + zb);
              dev::bulk_g2s(st, usrc, ub, &full[slot], pol_stream);
              dev::bulk_g2s(st + ub, zrow, zb, &full[slot], pol_keep);
            }
          }
        } else if (a.ndc > 1 && !a.adm) {
          // column chunk h of the (weak) dense block: the Re x dc box of D
          // (tensor TMA) + the chunk's x segment per rhs; lane 0 issues
          const int h = l - L - 1;
          uint32_t total = static_cast<uint32_t>(Re * a.dc * 8);
          int64_t lo[NR];
          uint32_t xb[NR];
#pragma unroll
          for (int kk = 0; kk < NR; ++kk) {
            if (kk < a.nr) {
              const int64_t start = kk * a.ldx + leaf0 + h * a.dc;
              lo[kk] = start & ~int64_t(1);
              xb[kk] = static_cast<uint32_t>((((start + a.dc + 1) & ~int64_t(1)) - lo[kk]) * 8);
              total += xb[kk];
            }
          }
          dev::mbar_wait(&empty[slot], phase ^ 1);
          if (lane == 0) {
            if (first_stage) chunk_q[slot] = chunk;
            dev::mbar_arrive_expect_tx(&full[slot], total);
            dev::tma_load_2d(st, &a.tm_dse, h * a.dc, static_cast<int>(i0), &full[slot], pol_stream);
#pragma unroll
            for (int kk = 0; kk < NR; ++kk)
              if (kk < a.nr)
                dev::bulk_g2s(st + Re * a.dc * 8 + kk * a.xs_e * 8, a.x + lo[kk], xb[kk], &full[slot], pol_keep);
          }
          first_stage = false;
        } else {
          // one stage holds the dense blocks e of group h = l - L - 1 (weak: the
          // single leaf block; standard: neighbours [h dgs, (h+1) dgs)), block e
          // at byte offset (e - h dgs) * dblk followed by its source x segment
          // (16-byte aligned superset per rhs); lanes issue their own blocks
          const int e0 = (l - L - 1) * a.dgs;
          const bool lane_on = src != kNone && lane >= e0 && lane < e0 + a.dgs;
          uint32_t mine = 0;
          int64_t lo[NR];
          uint32_t xb[NR];
          if (lane_on) {
            mine = db;
#pragma unroll
            for (int kk = 0; kk < NR; ++kk) {
              if (kk < a.nr) {
                const int64_t start = kk * xld + src;
                lo[kk] = start & ~int64_t(1);
                xb[kk] = static_cast<uint32_t>((((start + b + 1) & ~int64_t(1)) - lo[kk]) * 8);
                mine += xb[kk];
              }
            }
          }
          const uint32_t total = __reduce_add_sync(0xffffffffu, mine);
          dev::mbar_wait(&empty[slot], phase ^ 1);
          if (lane == 0 && first_stage) chunk_q[slot] = chunk;
          first_stage = false;
          if (lane == 0) dev::mbar_arrive_expect_tx(&full[slot], total);
          __syncwarp();
          if (lane_on) {
            unsigned char* se = st + (lane - e0) * dblk;
            dev::bulk_g2s(se, a.D + lane * a.d_stride + i0 * Dp, db, &full[slot], pol_stream);
#pragma unroll
            for (int kk = 0; kk < NR; ++kk)
              if (kk < a.nr)
                dev::bulk_g2s(se + db + kk * a.xs_e * 8, xsrc + lo[kk], xb[kk], &full[slot], pol_keep);
          }
        }
        if (++slot == NS) {
          slot = 0;
          phase ^= 1;
        }
      }
      if (++in_leaf == ipl) {
        in_leaf = 0;
        leaf0 += b;
        ++leaf_idx;
        src = dense_source();
      }
    }
    }
    return;
  }

  // ---------------- consumers ------------------------------------------------
  // tpr threads per row; thread p of row ri owns the column pairs
  // cp = p + tpr*jj (columns 2cp, 2cp+1), visited in a row-rotated order so the
  // 16-byte smem reads of a warp's rows fall in different bank halves.
  const int t = tid - 32;
  const int tpr = a.tpr;
  const int ri = t / tpr, p = t - ri * tpr;
  const bool active = ri < Re;
  const int NP = Wp >> 1, NPD = Dp >> 1;
  const int njU = (NP + tpr - 1) / tpr;
  const int njD = (NPD + tpr - 1) / tpr;
  const int rotU = ri % njU, rotD = ri % njD;
  // The thread's U column pairs in visiting order, fixed for the whole kernel
  // (kMaxJ of them at most on the fast path; -1 = none): the stage loop is then
  // a straight run of 2 LDS.128 + 2 DFMA per pair.  The consumers' per-stage
  // time is on the stream's critical path (a slot is refilled only after every
  // warp has read it), so their instruction count per stage matters.
  constexpr int kMaxJ = 8;
  const bool fastU = NR <= 4 && njU <= kMaxJ && !(W & 1);  // (NR = 8: registers; odd W: padding column)
  int coff[kMaxJ];
#pragma unroll
  for (int n = 0; n < kMaxJ; ++n) {
    if constexpr (NR <= 4) {
      const int jj = n < njU ? (rotU + n) % njU : 0;
      const int cp = p + tpr * jj;
      coff[n] = (n < njU && cp < NP) ? cp : -1;
    } else {
      coff[n] = -1;
    }
  }
  const int64_t ipl = b / Re;
  int64_t leaf0 = 0, in_leaf = 0;
  int64_t leaf_idx = 0;
  uint32_t nmask = 1u, hmask = 0u;  // neighbours present / read from the halo buffer (P > 1)
  const int64_t lbase = a.row0 / b;
  auto halo_mask = [&]() -> uint32_t {
    uint32_t m = 0u;
    if (a.halo_of)
      for (int e = 0; e < a.nd; ++e) m |= (a.halo_of[(leaf_idx - lbase) * a.nd + e] >= 0 ? 1u : 0u) << e;
    return m;
  };
  // H^T with P > 1: remote neighbours' blocks are skipped (added after the kernel)
  auto present = [&]() -> uint32_t {
    const uint32_t m = geo::near_mask_k(a.d, leaf_idx, L);
    return a.skip_remote ? m & ~hmask : m;
  };
  int slot = 0;
  uint32_t phase = 0;
  int64_t cj0 = j0, cj1 = j1;
  bool first_range = true, peeked = false;
  auto next_range = [&]() -> bool {
    if (!dyn) {
      const bool r = first_range && j0 < j1;
      first_range = false;
      return r;
    }
    // the next stage is the first of the producer's next chunk (or the end mark)
    dev::mbar_wait(&full[slot], phase);
    const int c = chunk_q[slot];
    if (c < 0) return false;
    cj0 = ib + int64_t(c) * a.chunk_e;
    cj1 = cj0 + a.chunk_e < ib + a.items_e ? cj0 + a.chunk_e : ib + a.items_e;
    peeked = true;
    return true;
  };
  if constexpr (SH == 3) {
    // one row per warp, lane p: U pairs p + 32 n (n < 6) and p + 192 (p < 24);
    // D pair p of each present near-field block.  Consecutive lanes read
    // consecutive 16-byte pairs of one row: conflict-free without rotation.
    constexpr int NPc = kStd2NP, NFULL = NPc / 32, NTAIL = NPc - 32 * NFULL, REc = CT / 32, NPDc = 32;
    const uint32_t ub0 = (ri * NPc + p) * 16;
    const uint32_t zd = (REc - ri) * NPc * 16;
    const bool tail = p < NTAIL;
    const uint32_t db0 = (ri * NPDc + p) * 16;
    const uint32_t xd = (REc - ri) * NPDc * 16;
    const uint32_t dblk = static_cast<uint32_t>(REc * NPDc * 16 + a.xs_e * 8);
    const bool skip = a.dbg & 2;
    const int ipl2 = b / REc;
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&empty[slot]);
      if (++slot == NS) {
        slot = 0;
        phase ^= 1;
      }
    };
    while (next_range()) {
      int64_t lf = (a.row0 + cj0 * REc) / b;  // the item's leaf
      int il = static_cast<int>((cj0 * REc) % b) / REc;
      uint32_t nm = geo::near_mask_k(2, lf, L);
      for (int64_t j = cj0; j < cj1; ++j) {
        double acc = 0.0, acc2 = 0.0;
        for (int l = 1; l <= L + 3; ++l) {
          const bool is_d = l > L;
          if (is_d ? !a.dense : !((a.level_mask >> (l - 1)) & 1ull)) continue;
          if (!peeked) dev::mbar_wait(&full[slot], phase);
          peeked = false;
          if (!skip) {
            const unsigned char* st = smem + slot * a.stage_bytes_e;
            if (!is_d) {
              const unsigned char* su = st + ub0;
              const unsigned char* sz = su + zd;
#pragma unroll
              for (int n = 0; n < NFULL; ++n) {
                const double2 u = *reinterpret_cast<const double2*>(su + n * 512);
                const double2 z = *reinterpret_cast<const double2*>(sz + n * 512);
                acc = fma(u.x, z.x, acc);
                acc2 = fma(u.y, z.y, acc2);
              }
              if (tail) {
                const double2 u = *reinterpret_cast<const double2*>(su + NFULL * 512);
                const double2 z = *reinterpret_cast<const double2*>(sz + NFULL * 512);
                acc = fma(u.x, z.x, acc);
                acc2 = fma(u.y, z.y, acc2);
              }
            } else {
              const uint32_t m3 = nm >> ((l - L - 1) * 3);
              const unsigned char* sd = st + db0;
#pragma unroll
              for (int e = 0; e < 3; ++e) {
                if ((m3 >> e) & 1u) {
                  const double2 dv = *reinterpret_cast<const double2*>(sd + e * dblk);
                  const double2 xv = *reinterpret_cast<const double2*>(sd + e * dblk + xd);
                  acc = fma(dv.x, xv.x, acc);
                  acc2 = fma(dv.y, xv.y, acc2);
                }
              }
            }
          }
          release();
        }
        acc += acc2;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (p == 0) {
          double* yp = a.y + j * REc + ri;  // y = alpha (H x) + beta y (GEMV)
          *yp = a.beta == 0.0 ? a.alpha * acc : a.alpha * acc + a.beta * *yp;
        }
        if (++il == ipl2) {
          il = 0;
          ++lf;
          nm = geo::near_mask_k(2, lf, L);
        }
      }
    }
    return;
  } else if constexpr (SH != 0) {
    using S = ExpShape<SH>;
    constexpr int TPR = S::TPR, NJU = S::NJU, NJD = S::NJD;
    constexpr int NPc = TPR * NJU, NPDc = TPR * NJD, REc = CT / TPR;
    // Pair cp of row ri sits at byte (ri NP + cp) 16 of a U stage, pair cp of
    // the z row at (Re NP + cp) 16 = the U offset + (Re - ri) NP 16; the same
    // for D and the x segment.  Thread p of row ri reads pairs p + TPR n.  With
    // TPR = 4 a quarter-warp phase of LDS.128 holds rows 2k and 2k + 1, whose
    // pitches are multiples of 128 B: the odd row starts one pair group later
    // (n = 1, ..., NJ - 1, then 0) so the phase's 8 reads hit 8 bank groups.
    const int odd = TPR == 4 ? (ri & 1) : 0;
    const uint32_t ub0 = (ri * NPc + p) * 16 + odd * TPR * 16;
    const uint32_t ul = odd ? ub0 - TPR * 16 : ub0 + (NJU - 1) * TPR * 16;
    const uint32_t zd = (REc - ri) * NPc * 16;
    const uint32_t db0 = (ri * NPDc + p) * 16 + odd * TPR * 16;
    const uint32_t dl = odd ? db0 - TPR * 16 : db0 + (NJD - 1) * TPR * 16;
    const uint32_t xd = (REc - ri) * NPDc * 16;
    const bool skip = a.dbg & 2;
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&empty[slot]);
      if (++slot == NS) {
        slot = 0;
        phase ^= 1;
      }
    };
    while (next_range()) {
      for (int64_t j = cj0; j < cj1; ++j) {
        double acc = 0.0, acc2 = 0.0;  // two chains: even / odd columns
        for (int l = 1; l <= L; ++l) {
          if (!((a.level_mask >> (l - 1)) & 1ull)) continue;
          if (!peeked) dev::mbar_wait(&full[slot], phase);
          peeked = false;
          if (!skip) {
            const unsigned char* st = smem + slot * a.stage_bytes_e;
            const unsigned char* su = st + ub0;
            const unsigned char* sz = su + zd;
#pragma unroll
            for (int n = 0; n < NJU - 1; ++n) {
              const double2 u = *reinterpret_cast<const double2*>(su + n * TPR * 16);
              const double2 z = *reinterpret_cast<const double2*>(sz + n * TPR * 16);
              acc = fma(u.x, z.x, acc);
              acc2 = fma(u.y, z.y, acc2);
            }
            const double2 u = *reinterpret_cast<const double2*>(st + ul);
            const double2 z = *reinterpret_cast<const double2*>(st + ul + zd);
            acc = fma(u.x, z.x, acc);
            acc2 = fma(u.y, z.y, acc2);
          }
          release();
        }
        if (a.dense) {
          if (!peeked) dev::mbar_wait(&full[slot], phase);
          peeked = false;
          if (!skip) {
            const unsigned char* st = smem + slot * a.stage_bytes_e;
            const unsigned char* sd = st + db0;
            const unsigned char* sx = sd + xd;
#pragma unroll
            for (int n = 0; n < NJD - 1; ++n) {
              const double2 dv = *reinterpret_cast<const double2*>(sd + n * TPR * 16);
              const double2 xv = *reinterpret_cast<const double2*>(sx + n * TPR * 16);
              acc = fma(dv.x, xv.x, acc);
              acc2 = fma(dv.y, xv.y, acc2);
            }
            const double2 dv = *reinterpret_cast<const double2*>(st + dl);
            const double2 xv = *reinterpret_cast<const double2*>(st + dl + xd);
            acc = fma(dv.x, xv.x, acc);
            acc2 = fma(dv.y, xv.y, acc2);
          }
          release();
        }
        acc += acc2;
#pragma unroll
        for (int off = TPR >> 1; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (p == 0) {
          double* yp = a.y + j * REc + ri;  // y = alpha (H x) + beta y (GEMV)
          *yp = a.beta == 0.0 ? a.alpha * acc : a.alpha * acc + a.beta * *yp;
        }
      }
    }
  } else {  // generic shapes
  while (next_range()) {
  leaf0 = (cj0 * Re / b) * b;
  in_leaf = (cj0 * Re - leaf0) / Re;
  leaf_idx = (a.row0 + leaf0) / b;
  if (a.adm) {
    hmask = halo_mask();
    nmask = present();
  }
  for (int64_t j = cj0; j < cj1; ++j) {
    const int64_t i0 = j * Re;
    double acc[NR], acc2[NR];  // two chains: even / odd columns
#pragma unroll
    for (int kk = 0; kk < NR; ++kk) acc[kk] = acc2[kk] = 0.0;
    for (int li = 1; li <= L + a.ndc; ++li) {
      const int l = level_order(a, li);
      const bool is_d = (l > L);
      if (is_d ? !a.dense : !((a.level_mask >> (l - 1)) & 1ull)) continue;
      if (!peeked) dev::mbar_wait(&full[slot], phase);
      peeked = false;
      const unsigned char* st = smem + slot * a.stage_bytes_e;
      if (active && !(a.dbg & 2)) {
        if (!is_d) {
          const double2* U2 = reinterpret_cast<const double2*>(st) + ri * NP;
          const double* Zs = reinterpret_cast<const double*>(st + Re * Wp * 8);
          // peer exchange levels: the stage holds the P ranks' rows, summed here in rank order
          const int nz = (a.peer && l <= a.cross) ? a.P : 1;
          if (NR <= 4 && fastU && nz == 1) {
            const double2* Z2 = reinterpret_cast<const double2*>(Zs);
#pragma unroll
            for (int n = 0; n < kMaxJ; ++n) {
              if (coff[n] >= 0) {
                const double2 u = U2[coff[n]];
#pragma unroll
                for (int kk = 0; kk < NR; ++kk) {
                  const double2 z = Z2[kk * NP + coff[n]];
                  acc[kk] = fma(u.x, z.x, acc[kk]);
                  acc2[kk] = fma(u.y, z.y, acc2[kk]);
                }
              }
            }
          } else {
          int jj = rotU;
          for (int n = 0; n < njU; ++n) {
            const int cp = p + tpr * jj;
            if (cp < NP) {
              double2 u = U2[cp];
              if (2 * cp + 1 >= W) u.y = 0.0;  // padding column of an odd W
#pragma unroll
              for (int kk = 0; kk < NR; ++kk) {  // Zt row layout [rhs][col]
                double2 z = reinterpret_cast<const double2*>(Zs + kk * Wp)[cp];
                for (int g = 1; g < nz; ++g) {
                  const double2 zg = reinterpret_cast<const double2*>(Zs + (int64_t)g * Wp * NR + kk * Wp)[cp];
                  z.x += zg.x;
                  z.y += zg.y;
                }
                acc[kk] = fma(u.x, z.x, acc[kk]);
                acc2[kk] = fma(u.y, z.y, acc2[kk]);
              }
            }
            if (++jj == njU) jj = 0;
          }
          }
        } else if (a.ndc > 1 && !a.adm) {
          // column chunk h: D box [Re][dc] + x[leaf0 + h dc, + dc)
          const int NPC = a.dc >> 1;
          const double2* D2 = reinterpret_cast<const double2*>(st) + ri * NPC;
          const double* xs = reinterpret_cast<const double*>(st + Re * a.dc * 8);
          int xo[NR];
#pragma unroll
          for (int kk = 0; kk < NR; ++kk) xo[kk] = kk * a.xs_e + static_cast<int>((kk * a.ldx + leaf0) & 1);
          for (int cp = p; cp < NPC; cp += tpr) {
            const double2 dv = D2[cp];
#pragma unroll
            for (int kk = 0; kk < NR; ++kk) {
              acc[kk] = fma(dv.x, xs[xo[kk] + 2 * cp], acc[kk]);
              acc2[kk] = fma(dv.y, xs[xo[kk] + 2 * cp + 1], acc2[kk]);
            }
          }
        } else {
          const int64_t dblk = int64_t(Re) * Dp * 8 + int64_t(NR) * a.xs_e * 8;
          const int e0 = (l - L - 1) * a.dgs;
          for (int e = e0; e < e0 + a.dgs; ++e) {  // dense blocks present in this stage
            if (!((nmask >> e) & 1u)) continue;
            const unsigned char* se = st + (e - e0) * dblk;
            const double2* D2 = reinterpret_cast<const double2*>(se) + ri * NPD;
            const double* xs = reinterpret_cast<const double*>(se + Re * Dp * 8);
            const int64_t src0 = (a.adm && (b & 1)) ? geo::neighbour_k(a.d, leaf_idx, e, L) * b - a.row0 : leaf0;
            // halo segments start 16-byte aligned (bpad even): no parity offset
            const bool halo = (hmask >> e) & 1u;
            int xo[NR];
#pragma unroll
            for (int kk = 0; kk < NR; ++kk)
              xo[kk] = kk * a.xs_e + (halo ? 0 : static_cast<int>((kk * a.ldx + src0) & 1));
            int jj = rotD;
            for (int n = 0; n < njD; ++n) {
              const int cp = p + tpr * jj;
              if (cp < NPD) {
                const double2 dv = D2[cp];
                const bool odd_ok = 2 * cp + 1 < b;  // padding column of an odd b
#pragma unroll
                for (int kk = 0; kk < NR; ++kk) {
                  acc[kk] = fma(dv.x, xs[xo[kk] + 2 * cp], acc[kk]);
                  if (odd_ok) acc2[kk] = fma(dv.y, xs[xo[kk] + 2 * cp + 1], acc2[kk]);
                }
              }
              if (++jj == njD) jj = 0;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&empty[slot]);
      if (++slot == NS) {
        slot = 0;
        phase ^= 1;
      }
    }
#pragma unroll
    for (int kk = 0; kk < NR; ++kk) {
      acc[kk] += acc2[kk];
      for (int off = tpr >> 1; off >= 1; off >>= 1) acc[kk] += __shfl_xor_sync(0xffffffffu, acc[kk], off);
    }
    if (active && p == 0) {
#pragma unroll
      for (int kk = 0; kk < NR; ++kk)
        if (kk < a.nr) {
          double* yp = a.y + kk * a.ldy + i0 + ri;  // y = alpha (H x) + beta y (GEMV)
          *yp = a.beta == 0.0 ? a.alpha * acc[kk] : a.alpha * acc[kk] + a.beta * *yp;
        }
    }
    if (++in_leaf == ipl) {
      in_leaf = 0;
      leaf0 += b;
      if (a.adm) {
        ++leaf_idx;
        hmask = halo_mask();
        nmask = present();
      }
    }
  }
  }
  }
}

template <int NR, int SH>
cudaError_t launch_sh(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if (!a.pdl) {
    expand_kernel<NR, SH><<<grid, kThreads, smem, s>>>(a);
    return cudaGetLastError();
  }
  return launch_pdl(expand_kernel<NR, SH>, a, grid, kThreads, smem, s);
}

template <int SH>
bool shape_is(const StreamArgs& a) {
  using S = ExpShape<SH>;
  return a.tpr == S::TPR && a.Re * S::TPR == CT && a.W == a.Wp && a.Wp == 2 * S::TPR * S::NJU &&
         a.b == a.Dp && a.Dp == 2 * S::TPR * S::NJD;
}

// compile-time consumer shape of this launch (ExpShape), 0 = generic
int expand_shape(const StreamArgs& a, int nr_cap) {
  if (nr_cap != 1 || a.peer || !a.eshape) return 0;
  if (a.adm)  // standard, 2-D, r = 16, b = 64, one GPU (no halo, nothing skipped)
    return a.d == 2 && a.r == 16 && a.b == 64 && a.Dp == 64 && a.W == 2 * kStd2NP && a.Wp == a.W && a.tpr == 32 &&
                   a.Re * 32 == CT && a.ndc == 3 && a.dgs == 3 && a.nd == 9 && !a.halo_of && !a.skip_remote
               ? 3
               : 0;
  if (a.ndc != 1) return 0;
  if (shape_is<1>(a)) return 1;
  if (shape_is<2>(a)) return 2;
  return 0;
}

template <int NR>
cudaError_t launch_nr(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if constexpr (NR == 1) {
    const int sh = expand_shape(a, NR);
    if (sh == 1) return launch_sh<1, 1>(a, grid, smem, s);
    if (sh == 2) return launch_sh<1, 2>(a, grid, smem, s);
    if (sh == 3) return launch_sh<1, 3>(a, grid, smem, s);
  }
  return launch_sh<NR, 0>(a, grid, smem, s);
}

}  // namespace

cudaError_t launch_expand(const StreamArgs& a, int nr_cap, int grid, int64_t smem, cudaStream_t s) {
  switch (nr_cap) {
    case 1: return launch_nr<1>(a, grid, smem, s);
    case 2: return launch_nr<2>(a, grid, smem, s);
    case 4: return launch_nr<4>(a, grid, smem, s);
    default: return launch_nr<8>(a, grid, smem, s);
  }
}

cudaError_t configure_kernels(int64_t smem_p, int64_t smem_e) {
  cudaError_t e = configure_project(smem_p);
  if (e != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(expand_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e))) return e;
  if ((e = cudaFuncSetAttribute(expand_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e))) return e;
  if ((e = cudaFuncSetAttribute(expand_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e))) return e;
  if ((e = cudaFuncSetAttribute(expand_kernel<1, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e))) return e;
  if ((e = cudaFuncSetAttribute(expand_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e))) return e;
  if ((e = cudaFuncSetAttribute(expand_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e))) return e;
  return cudaFuncSetAttribute(expand_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_e);
}

}  // namespace hmat
