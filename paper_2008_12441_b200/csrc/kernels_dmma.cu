// kernels_dmma.cu -- the many-right-hand-side H-matvec on the FP64 tensor cores
// (BASELINE configs[4]: 64 right-hand sides).
//
// With NB = 64 right-hand sides the two steps become dense contractions:
//   project (Step 1, eq:prod-vx):  Z_s (W x NB) = V_s^T (W x m) X_s (m x NB)
//   expand  (Step 5, eq:prod-yuz, eq:prod-ydz):      Y_tile (64 x NB) = sum_l U_l[tile] (64 x W) Zt_l[t] (W x NB)
//                                                                       + D[tile] (64 x b) X_leaf (b x NB)
// computed with warp-level mma.sync.m8n8k4.f64 (SASS DMMA; tcgen05 has no
// f64 kind on sm_100a).  A pass is NB = 64 columns wide, or NB = 32 / 16 when at
// most 32 / 16 right-hand sides remain (a pass computes all NB columns, so a
// narrower one cuts the work of a few rhs).  Measured on this B200: DMMA 37.1 TFLOP/s, DFMA 36.5
// (scripts/fp64_peak.cu), so the tensor path's gain is issue slots and
// operand reuse, not a higher peak.
//
// Operands reach shared memory by 1-D bulk TMA copies into padded pitches
// (row pitch = 4 mod 16 doubles), which makes every m8n8k4 fragment load
// conflict-free; Zt is stored "fragment-major" (the exact order in which the
// expand kernel's B fragments are read), so one copy per stage brings it in.
// Pipelines, CTA splits and the deterministic ticketed reduction of node
// partials are the same as in the single-vector kernels.
#include "device_utils.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace hmat {
namespace {

// project: 16 warps (4 per SM sub-partition) or 8, no producer warp (launch_p)
constexpr int kThreadsE = 256;  // expand: 8 warps, no producer warp
constexpr int RE = kDmmaRE;   // expand: rows per item

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Fragment-major position of element (w, n) of one target's Zt block (W x NB):
// k-step kb = w/4, N-tile pair np = n/16, lane = (n%8)*4 + w%4, half = (n/8)%2.
template <int NB>
__device__ __forceinline__ int64_t zfrag(int w, int n) {
  if constexpr (NB == 8)  // one N-tile: [k-step][lane], one double per lane
    return (int64_t)(w >> 2) * 32 + (n & 7) * 4 + (w & 3);
  return ((((int64_t)(w >> 2) * (NB / 16) + (n >> 4)) * 32 + (n & 7) * 4 + (w & 3)) << 1) + ((n >> 3) & 1);
}

__device__ __forceinline__ int64_t owner_of(int64_t k, int64_t S, int64_t G) { return ((k + 1) * G - 1) / S; }

// Standard admissibility: the interaction-list slot tables (the
// same as kernels_project.cu's, written by init_std_tables_dmma).
__constant__ int16_t c_std_code_d[3][8][kStdMaxSlots];
__constant__ int16_t c_std_slot_d[3][8][kStdMaxCodes];

// Column w = q r + aa of source node sg's z at `level`, standard admissibility:
// target t = slot q of sg (child sigma of the parent's neighbour e), into t's
// column qt r + aa (qt = slot of sg in t's list).  nullptr when the partner box
// lies outside the domain (the block does not exist).  P > 1: a pair with an
// entry in the packed cross-rank buffer (std_exchange.h) goes there instead,
// rhs n at + n r (xs = r; xs = 0: the fragment-major Zt column, + zfrag(0, n)).
template <int NB>
__device__ __forceinline__ double* zt_column_std(const StreamArgs& a, const LevelArgs& lv, int64_t sg, int level,
                                                 int q, int aa, int& xs) {
  xs = 0;
  const int d = a.d, c = a.c;
  const int tau = static_cast<int>(sg & (c - 1));
  const int code = c_std_code_d[d - 1][tau][q];
  const int e = code >> d, sigma = code & (c - 1);
  const int64_t pt = geo::neighbour_k(d, sg >> d, e, level - 1);  // the parent's neighbour e
  if (pt < 0) return nullptr;
  if (lv.xent) {
    const int32_t ent = lv.xent[(sg - lv.tbase) * (a.W / a.r) + q];
    if (ent >= 0) {
      xs = a.r;
      return a.xchg + (int64_t)ent * NB * a.r + aa;
    }
  }
  const int64_t t = pt * c + sigma;
  const int nd = d == 1 ? 3 : d == 2 ? 9 : 27;
  const int qt = c_std_slot_d[d - 1][sigma][(nd - 1 - e) * c + tau];  // eps -> -eps, sigma <-> tau
  return lv.zt + (t - lv.tbase) * (int64_t)a.W * NB + zfrag<NB>(qt * a.r + aa, 0);
}

// Column w = q r + aa of source node sg's z goes to target t = sib(sg, q), into
// t's column qt r + aa (qt = slot of sg in t's list).  Returns the Zt block of t
// with the column's fragment-major base folded in: element (w, n) then sits at
// + zfrag(0, n) (zfrag is additive in its w and n parts).
template <int NB>
__device__ __forceinline__ double* zt_column(const StreamArgs& a, const LevelArgs& lv, int64_t sg, int q, int aa) {
  const int d = __ffs(a.c) - 1;
  const int me = static_cast<int>(sg & (a.c - 1));
  const int64_t t = ((sg >> d) << d) + (q < me ? q : q + 1);
  const int tc = static_cast<int>(t & (a.c - 1));
  const int qt = me < tc ? me : me - 1;
  return lv.zt + (t - lv.tbase) * (int64_t)a.W * NB + zfrag<NB>(qt * a.r + aa, 0);
}

// ============================ project ========================================
// KR: V rows (the GEMM's k) per stage; the staged x columns have pitch KR + 4
// (= 4 mod 16 doubles: conflict-free B-fragment loads).
// The W x NB accumulator tile is split over 16 warps as MG column groups (MT
// M-tiles of 8 columns each) x NG = 8 / NT rhs groups (NT N-tiles of 8 rhs),
// MG NG = 16: NT = 2 (MG = 4, MT = W/32) when W % 32 == 0, else NT = 1 (MG = 2,
// MT = W/16).  Each of the SM's 4 sub-partitions runs exactly 4 warps (a
// W/16-warp split leaves 3 or 4 warps per sub-partition: with W = 224 the
// tensor pipe then idles 1/8).
// No producer warp: a stage is two tensor-TMA copies (the KR x VP block of V
// rows, padding columns out of bounds = zero-filled, and the NB x (KR+4) block
// of x), issued by the LAST warp to finish reading the slot (smem counter), so
// all 16 warps compute and each gets 128 registers.
// NW warps per CTA: 16 (one CTA per SM) or 8 (two CTAs per SM, used for
// W % 32 != 0 so that a warp still holds 2 N-tiles: MT + 2 fragment loads per
// 2 MT DMMAs instead of MT + 1 per MT).
template <int KR, int MT, int NT, int NW, int NB>
__global__ void __launch_bounds__(NW * 32, 16 / NW) project_dmma_kernel(const __grid_constant__ StreamArgs a) {
  constexpr int XPP = KR + 4;
  constexpr int NG = NB / 8 / NT, MG = NW / NG;
  static_assert(NG * MG == NW, "warp grid");
  constexpr int NCW = NW;
  constexpr int CTP = NCW * 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // Column slices (a.nslice > 1, the standard structure's wide panels) are the
  // fastest-varying part of the CTA index: the CTAs resident at any time hold all
  // slices of neighbouring row ranges, so a stage's x rows are shared through L2
  // by the slices instead of being swept once per slice.
  const int NSL = a.nslice > 0 ? a.nslice : 1;
  const int64_t G = gridDim.x / NSL, bid = blockIdx.x / NSL;
  const int slice = static_cast<int>(blockIdx.x % NSL);
  const int Wp = a.Wp, L = a.L;
  const int VP = a.vp;                     // smem pitch of V rows (= 4 mod 16)
  // column slice of this CTA: [c0, c0 + WS) of the W panel columns (a panel wider
  // than one CTA's register-resident node tile, standard admissibility: W = M r)
  const int WS = a.wslice, c0 = slice * WS;
  const int64_t SL = a.N_loc / KR;
  const int64_t GL = G < SL ? G : SL;
  const int NS = a.nstage_p;
  const int64_t vbytes = (int64_t)KR * VP * 8;
  const uint32_t stage_tx = static_cast<uint32_t>(vbytes + NB * XPP * 8);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off_p);
  int* done = reinterpret_cast<int*>(full + NS);           // readers finished, per slot
  volatile int* flag = reinterpret_cast<volatile int*>(done + NS);
  const int64_t k0 = SL * bid / (GL > 0 ? GL : 1), k1 = SL * (bid + 1) / (GL > 0 ? GL : 1);
  const uint64_t pol_stream = dev::policy_evict_first();
  const uint64_t pol_keep = dev::policy_evict_last();
  // Stage order: the CTA's range [k0, k1) in chunks of CH stages (a.pchunk; 0 =
  // one chunk), every active level of a chunk before the next chunk, so the x
  // rows of a chunk are re-read by the other levels from L2 instead of once per
  // level from DRAM (8 rhs at c4: 9 x 1.07 GB).  A level's accumulators carry
  // over between chunks through a small per-CTA global buffer (a.accbuf, L2).
  // Within a level the stages keep their order, so the sums are bit-identical.
  const int64_t CH = a.pchunk > 0 ? a.pchunk : (k1 > k0 ? k1 - k0 : 1);
  int first_l = 1;
  while (first_l <= L && !((a.level_mask >> (first_l - 1)) & 1ull)) ++first_l;
  // the refill cursor (chunk [cb, ce), level lr, stage kr): identical in every warp
  int lr = 0;
  int64_t cb = k0, ce = k0 + CH < k1 ? k0 + CH : k1, kr = ce;
  auto advance = [&]() {
    if (++kr < ce) return;
    for (++lr; lr <= L && !((a.level_mask >> (lr - 1)) & 1ull); ++lr) {
    }
    if (lr > L) {  // next chunk
      cb = ce;
      ce = cb + CH < k1 ? cb + CH : k1;
      lr = cb < k1 ? first_l : L + 1;
    }
    kr = cb;
  };
  const bool no_x = (a.dbg & 64) != 0;  // (diagnostics: the ring without its x boxes -- wrong results)
  // (diagnostics, bit 7: V boxes exactly Wp wide, no out-of-bounds columns -- wrong
  // results; unsliced panels only, where Wp <= vp and the box fits the slot)
  const uint32_t vtx = static_cast<uint32_t>((a.dbg & 128) && NSL == 1 && Wp <= VP ? (int64_t)KR * Wp * 8 : vbytes);
  auto issue = [&](int sl) {  // one thread: the next stage into slot sl
    dev::mbar_arrive_expect_tx(&full[sl], no_x ? vtx : stage_tx - static_cast<uint32_t>(vbytes) + vtx);
    dev::tma_load_3d(smem + sl * a.stage_bytes_p, &a.tm_v, c0, static_cast<int>(kr * KR), lr - 1, &full[sl],
                     pol_stream);
    if (!no_x)
      dev::tma_load_2d(smem + sl * a.stage_bytes_p + vbytes, &a.tm_x, static_cast<int>(kr * KR), 0, &full[sl],
                       pol_keep);
  };
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      dev::mbar_init(&full[i], 1);
      done[i] = 0;
    }
    dev::fence_mbar_init();
  }
  __syncthreads();
  if (a.pdl_p) dev::pdl_wait();  // the previous kernel (e.g. last product's expand) complete
  if (a.pdl) dev::pdl_launch_dependents();  // expand may launch as SMs free up
  const dev::CtaTrace trace_scope(a.trace, blockIdx.x);
  if (bid >= GL) return;
  advance();  // first stage
  for (int i = 0; i < NS && lr <= L; ++i) {
    if (tid == 0) issue(i);
    advance();
  }

  const int mg = warp % MG, ng = warp / MG;  // columns [mg 8 MT, (mg+1) 8 MT), rhs [8 NT ng, 8 NT (ng+1))
  const int g = lane >> 2, tq = lane & 3;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int slot = 0;
  uint32_t phase = 0;
  constexpr int NACC = MT * NT * 2;
  // 8-wide passes with few fragments per stage: release a slot before its DMMAs
  constexpr bool EARLY = NB == 8 && (MT + NT) * (KR / 4) <= 32;
  double* accb = a.accbuf + ((int64_t)bid * L * (NW * 32) + tid) * NACC;  // + (l-1) NW 32 NACC
  for (int64_t ck0 = k0; ck0 < k1; ck0 += CH) {
  const int64_t ck1 = ck0 + CH < k1 ? ck0 + CH : k1;
  for (int l = 1; l <= L; ++l) {
    if (!((a.level_mask >> (l - 1)) & 1ull)) continue;
    const LevelArgs& lv = a.lv[l];
    const int64_t seg = lv.seg_rows / KR;
    int64_t sl = ck0 / seg, pos = ck0 - sl * seg;
    const int64_t sg0 = a.row0 / lv.m;
    if (ck0 > k0) {  // this level's running sums from the previous chunk
      double* ab = accb + (int64_t)(l - 1) * (NW * 32) * NACC;
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          acc[i][j][0] = ab[(i * NT + j) * 2];
          acc[i][j][1] = ab[(i * NT + j) * 2 + 1];
        }
    }
    for (int64_t k = ck0; k < ck1; ++k) {
      dev::mbar_wait(&full[slot], phase);
      const double* Vs = reinterpret_cast<const double*>(smem + slot * a.stage_bytes_p) + mg * 8 * MT + g;
      const double* Xs = reinterpret_cast<const double*>(smem + slot * a.stage_bytes_p + vbytes) +
                         (ng * 8 * NT + g) * XPP + tq;
      if constexpr (EARLY) {
        // 8 wide: the whole stage's fragments to registers, the slot handed back,
        // then the DMMAs -- the slot is held for the loads only, so its refill
        // (the pass is a stream: little math per byte) starts a DMMA chain earlier
        double af[KR / 4][MT], bf[KR / 4][NT];
#pragma unroll
        for (int ks = 0; ks < KR / 4; ++ks) {
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) af[ks][mt] = Vs[(ks * 4 + tq) * VP + mt * 8];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) bf[ks][nt] = Xs[nt * 8 * XPP + ks * 4];
        }
        // every lane's loads are ordered before lane 0's release (syncwarp), and
        // the last warp's acquire orders them all before its refill
        __syncwarp();
        if (lane == 0) {
          const int prev = dev::atom_add_acq_rel_cta(&done[slot], 1);
          if (prev == NCW - 1) {
            done[slot] = 0;
            if (lr <= L) {
              dev::fence_proxy_async_smem();
              issue(slot);
            }
          }
        }
#pragma unroll
        for (int ks = 0; ks < KR / 4; ++ks)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[ks][mt], bf[ks][nt]);
      } else {
      // (diagnostics, HMAT_DEBUG_SKIP bit 5: the ring without the math -- wrong results)
      if (!(a.dbg & 32))
#pragma unroll
      for (int ks = 0; ks < KR / 4; ++ks) {
        double av[MT], bv[NT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) av[mt] = Vs[(ks * 4 + tq) * VP + mt * 8];  // A = V^T
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bv[nt] = Xs[nt * 8 * XPP + ks * 4];         // B = X
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], av[mt], bv[nt]);
      }
      // release the slot: the last of the 16 warps refills it with the stage
      // NS ahead (its smem reads are complete: their values fed the DMMAs)
      __syncwarp();
      if (lane == 0) {
        const int prev = atomicAdd(&done[slot], 1);
        if (prev == NCW - 1) {
          done[slot] = 0;
          if (lr <= L) {
            dev::fence_proxy_async_smem();
            issue(slot);
          }
        }
      }
      }
      if (lr <= L) advance();
      if (++slot == NS) {
        slot = 0;
        phase ^= 1;
      }
      const bool node_end = (pos + 1 == seg);
      const int64_t this_sl = sl;
      if (++pos == seg) {
        pos = 0;
        ++sl;
      }
      if (!node_end && k + 1 != k1) continue;

      // ---- node flush ----
      const int64_t sa = this_sl * seg, sb = sa + seg;
      const bool complete = sa >= k0 && sb <= k1;
      const int64_t sg = sg0 + this_sl;
      if (complete) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          // column w = q r + aa; rhs n = 8 NT ng + 8 nt + 2 tq + h
          const int w = c0 + (mg * MT + mt) * 8 + g;
          const int q = w / a.r;
          int xs = 0;
          double* zc =
              a.adm ? zt_column_std<NB>(a, lv, sg, l, q, w - q * a.r, xs) : zt_column<NB>(a, lv, sg, q, w - q * a.r);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int n = (ng * NT + nt) * 8 + tq * 2 + h;
              if (n < a.nr && zc) zc[xs ? n * xs : zfrag<NB>(0, n)] = acc[mt][nt][h];
              acc[mt][nt][h] = 0.0;
            }
        }
      } else {
        const int myslot = sa <= k0 ? 0 : 1;
        double* pp = a.part + (((int64_t)(l - 1) * G + bid) * 2 + myslot) * (int64_t)Wp * NB;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int w = c0 + (mg * MT + mt) * 8 + g;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              pp[(int64_t)w * NB + (ng * NT + nt) * 8 + tq * 2 + h] = acc[mt][nt][h];
              acc[mt][nt][h] = 0.0;
            }
        }
        __threadfence();
        dev::named_bar_sync(1, CTP);
        const int64_t b0 = owner_of(sa, SL, GL), b1 = owner_of(sb - 1, SL, GL);
        int* ticket = a.cnt + ((int64_t)(l - 1) * G + b1) * NSL + slice;  // per column slice
        if (tid == 0) {
          const int prev = atomicAdd(ticket, 1);
          *flag = (prev == static_cast<int>(b1 - b0)) ? 1 : 0;
        }
        dev::named_bar_sync(1, CTP);
        if (*flag) {
          __threadfence();
          const int slot0 = (sa == SL * b0 / GL) ? 0 : 1;
          // thread: rhs n = tid % NB, columns w = tid / NB, + CTP / NB, ... (CTP is a multiple of NB)
          const int n = tid % NB, wstep = CTP / NB;
          const int64_t zn = zfrag<NB>(0, n);
          const int w0 = c0 + tid / NB;
          const int nwt = w0 < c0 + WS ? (c0 + WS - w0 + wstep - 1) / wstep : 0;  // this thread's columns
          const int64_t ps = (int64_t)Wp * NB;
          const double* p0 = a.part + (((int64_t)(l - 1) * G + b0) * 2 + slot0) * ps;
          const double* p1 = a.part + (((int64_t)(l - 1) * G + b0 + 1) * 2) * ps;
          const int64_t cnt = b1 - b0;
          // 2 columns at a time, 8 partials deep: 16 loads in flight per thread (a
          // node spanning ~100 CTAs -- the coarsest level of a small operator -- is
          // otherwise a long serial chain of L2 round trips in one CTA); each
          // column's sum keeps the CTA order
          for (int j0 = 0; j0 < nwt; j0 += 2) {
            double v[2];
            int64_t off[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              off[u] = (int64_t)(w0 + (j0 + u) * wstep) * NB + n;
              v[u] = j0 + u < nwt ? dev::ld_cg(p0 + off[u]) : 0.0;
            }
            for (int64_t i = 0; i < cnt; i += 8) {
              double t[2][8];
#pragma unroll
              for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int s = 0; s < 8; ++s)
                  t[u][s] = (j0 + u < nwt && i + s < cnt) ? dev::ld_cg(p1 + off[u] + (i + s) * 2 * ps) : 0.0;
#pragma unroll
              for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int s = 0; s < 8; ++s)
                  if (i + s < cnt) v[u] += t[u][s];
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (j0 + u < nwt && n < a.nr) {
                const int w = w0 + (j0 + u) * wstep, q = w / a.r, aa = w - q * a.r;
                int xs = 0;
                double* zc = a.adm ? zt_column_std<NB>(a, lv, sg, l, q, aa, xs) : zt_column<NB>(a, lv, sg, q, aa);
                if (zc) zc[xs ? n * xs : zn] = v[u];
              }
            }
          }
          if (tid == 0) *ticket = 0;
        }
        dev::named_bar_sync(1, CTP);
      }
    }
    if (ck1 < k1) {  // the next chunk continues this level's open node
      double* ab = accb + (int64_t)(l - 1) * (NW * 32) * NACC;
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          ab[(i * NT + j) * 2] = acc[i][j][0];
          ab[(i * NT + j) * 2 + 1] = acc[i][j][1];
          acc[i][j][0] = acc[i][j][1] = 0.0;
        }
    }
  }
  }
  if (a.peer) peer_push<NW * 32>(a, tid, GL, flag);  // this rank's exchange levels -> every mailbox
}

// ============================ expand =========================================
// CTA item: RE = 64 rows x NB rhs over WM x WN warps: warp (wm, wn) owns rows
// [wm*8*MT, (wm+1)*8*MT) (MT M-tiles) and NTW N-tiles of rhs from wn*NTW*8:
// NB = 64: 4 x 2 warps, MT = 2, NTW = 4; NB = 32: 4 x 2, MT = 2, NTW = 2;
// NB = 16: 8 x 1, MT = 1, NTW = 2.  A stage is one k-chunk of KC
// columns: the RE x (KC+4) box of U_l (tm_u) + the chunk of the target's
// fragment-major Zt (one bulk copy), or of D (tm_d) + the (KC+4) x NB box of
// the leaf's x (tm_xe); the extra 4 columns / rows give the conflict-free
// pitch AP = XP = KC + 4 and are never read.  As in project, no producer warp:
// the last of the 8 warps to finish a slot refills it.
// KC: k-columns per stage (32, or 16 when W % 32 != 0); the staged U / D row
// chunks and x columns have pitch KC + 4 (= 4 mod 16 doubles).
// WF: weak admissibility with every level and the dense block active (the
// plain product; a.level_mask full, a.dense): the stage sequence is then fixed
// -- kcw chunks per level, kcd for the leaf block -- and the cursor walk and the
// per-stage level checks compile away.  (Per stage and warp they outnumbered
// the DMMAs of a narrow pass.)
template <int KC, int NB, bool WF>
__global__ void __launch_bounds__(kThreadsE, 2) expand_dmma_kernel(const __grid_constant__ StreamArgs a) {
  constexpr int NCW = kThreadsE / 32;
  constexpr int WM = NB <= 16 ? 8 : 4, WN = NCW / WM;  // warp grid over rows x rhs
  constexpr int MT = RE / 8 / WM;                      // M-tiles (8 rows) per warp
  constexpr int NTW = NB / 8 / WN;                     // N-tiles per warp (NTW / 2 fragment-major pairs)
  static_assert((NTW == 1 || NTW % 2 == 0) && MT * WM * 8 == RE, "expand warp grid");
  // level stages: KC columns of U (pitch AP = KC + 4); dense stages: KD columns
  // of D (pitch APD) and the KD x NB box of x (pitch XP): KD = 16 with KC = 16, else 32
  constexpr int KD = KC == 16 ? 16 : 32;
  constexpr int AP = KC + 4, APD = KD + 4, XP = KD + 4;
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t G = gridDim.x, bid = blockIdx.x;
  const int W = a.W, b = a.b, L = a.L;
  // items [ib, ib + items) of the shard (a row chunk of a host-y product, or all)
  const int64_t ib = a.item0;
  const int64_t items = a.e_items > 0 ? a.e_items : a.N_loc / RE;
  // item order: interleaved (CTA b takes items b, b + G, b + 2G, ...: the G CTAs
  // work on G consecutive tiles at any time, so the coarse levels' Zt chunks they
  // share stay in L2 -- a handful of nodes instead of one per CTA, which at c5
  // (296 x 4 coarse levels x 114 KB) exceeded L2 and re-read Zt from DRAM), or
  // contiguous ranges (a.dmma_ileave = 0)
  const bool ilv = a.dmma_ileave != 0;
  const int64_t j0 = ilv ? bid : items * bid / G, j1 = ilv ? items : items * (bid + 1) / G;
  const int64_t jst = ilv ? G : 1;
  const int NS = a.nstage_e;
  const int kcw = W / KC, kcd = b / KD;      // k-chunks per level / for the dense block
  const int64_t abytes = (int64_t)RE * AP * 8, abytes_d = (int64_t)RE * APD * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off_e);
  int* done = reinterpret_cast<int*>(full + NS);
  // U / D boxes: read once, but each 36-column box overlaps the next chunk's
  // first 4 columns, so a policy that keeps them in L2 a little longer saves the
  // re-read (a.dmma_upol: 0 evict_first, 1 evict_normal)
  const uint64_t pol_stream = a.dmma_upol == 1 ? dev::policy_evict_normal() : dev::policy_evict_first();
  const uint64_t pol_keep = dev::policy_evict_last();
  // Dense stages: the leaf-diagonal block (weak, stage L + 1), or the 3^d
  // near-field blocks of the tile's leaf (standard admissibility, stages L + 1 + e
  // for the neighbours e inside the domain, one GPU).  nmask: the present ones.
  const int ndn = !WF && a.adm ? a.nd : 1;
  const int64_t lbase = a.row0 / b;
  // (P > 1: a neighbour on another rank -- halo_of >= 0 -- is read from the
  // packed buffer's halo x, map tm_xh; H^T skips it: its product arrives in the
  // exchange and is added after the kernel)
  auto near_of = [&](int64_t item) -> uint32_t {
    if (WF || !a.adm) return 1u;
    uint32_t m = geo::near_mask_k(a.d, lbase + item * RE / b, L);
    if (a.halo_of && a.skip_remote) {
      const int32_t* ho = a.halo_of + (item * RE / b) * a.nd;
      for (int e = 0; e < a.nd; ++e)
        if (ho[e] >= 0) m &= ~(1u << e);
    }
    return m;
  };
  auto level_on = [&](int l, uint32_t nmask) -> bool {
    if constexpr (WF) return true;
    return l > L ? a.dense != 0 && ((nmask >> (l - L - 1)) & 1u) : ((a.level_mask >> (l - 1)) & 1ull) != 0;
  };
  // refill cursor (item jr, level lr in 1..L+ndn (> L: dense), chunk kcr): identical in every warp
  int64_t jr = j0;
  int lr = 1, kcr = 0;
  uint32_t pmask = jr < j1 ? near_of(ib + jr) : 1u;
  bool any = false;
  for (int l = 1; l <= L + ndn; ++l) any = any || level_on(l, a.adm ? 1u << ((a.nd - 1) / 2) : 1u);  // (self)
  if (!any) jr = j1;
  while (jr < j1 && !level_on(lr, pmask)) ++lr;
  auto advance = [&]() {
    if (++kcr < (lr > L ? kcd : kcw)) return;
    kcr = 0;
    if constexpr (WF) {
      if (++lr > L + 1) {
        lr = 1;
        jr += jst;
      }
    } else {
      do {
        if (++lr > L + ndn) {
          lr = 1;
          jr += jst;
          pmask = jr < j1 ? near_of(ib + jr) : 1u;
        }
      } while (jr < j1 && !level_on(lr, pmask));
    }
  };
  auto issue = [&](int sl) {  // one thread: stage (jr, lr, kcr) into slot sl
    unsigned char* st = smem + sl * a.stage_bytes_e;
    const int i0 = static_cast<int>((ib + jr) * RE);
    if (lr > L) {
      dev::mbar_arrive_expect_tx(&full[sl], static_cast<uint32_t>(abytes_d + NB * XP * 8));
      if (!WF && a.adm) {  // near-field block e: panel e of the D-role panels, x of neighbour leaf e
        const int e = lr - L - 1;
        dev::tma_load_3d(st, &a.tm_d, kcr * KD, i0, e, &full[sl], pol_stream);
        const int h = a.halo_of ? a.halo_of[(i0 / b) * a.nd + e] : -1;
        if (h >= 0) {  // remote neighbour: its x from the halo region, rows h NB .. h NB + NB - 1
          dev::tma_load_2d(st + abytes_d, &a.tm_xh, kcr * KD, h * NB, &full[sl], pol_keep);
        } else {
          const int64_t nleaf = geo::neighbour_k(a.d, lbase + i0 / b, e, L) - lbase;
          dev::tma_load_2d(st + abytes_d, &a.tm_xe, static_cast<int>(nleaf * b) + kcr * KD, 0, &full[sl], pol_keep);
        }
      } else {
        dev::tma_load_2d(st, &a.tm_d, kcr * KD, i0, &full[sl], pol_stream);
        dev::tma_load_2d(st + abytes_d, &a.tm_xe, (i0 / b) * b + kcr * KD, 0, &full[sl], pol_keep);
      }
    } else {
      const LevelArgs& lv = a.lv[lr];
      const double* zt = lv.zt + ((a.row0 + i0) / lv.m - lv.tbase) * (int64_t)W * NB;
      dev::mbar_arrive_expect_tx(&full[sl], static_cast<uint32_t>(abytes + KC * NB * 8));
      dev::tma_load_3d(st, &a.tm_u, kcr * KC, i0, lr - 1, &full[sl], pol_stream);
      // a node of at most one tile is read once: stream it; coarser nodes' Zt is shared
      dev::bulk_g2s(st + abytes, zt + (int64_t)kcr * KC * NB, KC * NB * 8, &full[sl], lv.m <= RE ? pol_stream : pol_keep);
    }
  };
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      dev::mbar_init(&full[i], 1);
      done[i] = 0;
    }
    dev::fence_mbar_init();
  }
  __syncthreads();
  if (a.pdl) dev::pdl_wait();  // project (Zt) complete and visible
  if (a.pdl_p) dev::pdl_launch_dependents();  // the next product's project may launch early
  const dev::CtaTrace trace_scope(a.trace, bid);
  for (int i = 0; i < NS && jr < j1; ++i) {
    if (tid == 0) issue(i);
    advance();
  }

  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, tq = lane & 3;
  int slot = 0;
  uint32_t phase = 0;
  for (int64_t j = j0; j < j1; j += jst) {
    const int64_t i0 = (ib + j) * RE;
    double acc[MT][NTW][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int k = 0; k < NTW; ++k) acc[i][k][0] = acc[i][k][1] = 0.0;
    const uint32_t cmask = near_of(ib + j);
    for (int l = 1; l <= L + ndn; ++l) {
      const bool is_d = (l > L);
      if (!level_on(l, cmask)) continue;
      const int nkc = is_d ? kcd : kcw;
      for (int kc = 0; kc < nkc; ++kc) {
        dev::mbar_wait(&full[slot], phase);
        const double* As = reinterpret_cast<const double*>(smem + slot * a.stage_bytes_e);
        const double* Bs = reinterpret_cast<const double*>(smem + slot * a.stage_bytes_e + (is_d ? abytes_d : abytes));
        // two copies of the k loop (U / Zt stage, D / x stage), so the compiler
        // does not if-convert the B loads of both layouts into every k-step
        if (!is_d) {
#pragma unroll
          for (int ks = 0; ks < KC / 4; ++ks) {
            double av[MT], bv[NTW];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) av[mt] = As[(wm * 8 * MT + mt * 8 + g) * AP + ks * 4 + tq];
            // fragment-major Zt chunk: k-step ks, N-tile pairs wn*NTW/2 .. + NTW/2 - 1
            // (NB = 8: the one N-tile, a double per lane)
            if constexpr (NTW == 1) {
              bv[0] = Bs[ks * 32 + lane];
            } else {
#pragma unroll
              for (int np = 0; np < NTW / 2; ++np) {
                const double2 v =
                    reinterpret_cast<const double2*>(Bs)[(ks * (NB / 16) + wn * (NTW / 2) + np) * 32 + lane];
                bv[np * 2] = v.x;
                bv[np * 2 + 1] = v.y;
              }
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
              for (int nt = 0; nt < NTW; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], av[mt], bv[nt]);
          }
        } else {
#pragma unroll
          for (int ks = 0; ks < KD / 4; ++ks) {
            double av[MT], bv[NTW];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) av[mt] = As[(wm * 8 * MT + mt * 8 + g) * APD + ks * 4 + tq];
#pragma unroll
            for (int nt = 0; nt < NTW; ++nt) bv[nt] = Bs[((wn * NTW + nt) * 8 + g) * XP + ks * 4 + tq];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
              for (int nt = 0; nt < NTW; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], av[mt], bv[nt]);
          }
        }
        // release: the last of the NCW warps refills the slot NS stages ahead
        __syncwarp();
        if (lane == 0) {
          const int prev = atomicAdd(&done[slot], 1);
          if (prev == NCW - 1) {
            done[slot] = 0;
            if (jr < j1) {
              dev::fence_proxy_async_smem();
              issue(slot);
            }
          }
        }
        if (jr < j1) advance();
        if (++slot == NS) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int64_t row = i0 + wm * 8 * MT + mt * 8 + g;
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = (wn * NTW + nt) * 8 + tq * 2 + h;
          if (n < a.nr) {
            double* yp = a.y + n * a.ldy + row;
            *yp = a.beta == 0.0 ? a.alpha * acc[mt][nt][h] : a.alpha * acc[mt][nt][h] + a.beta * *yp;
          }
        }
    }
  }
}

template <int MT, int NT, int NW, int NB>
void launch_p(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  const int gs = grid * (a.nslice > 0 ? a.nslice : 1);  // column slices fastest (kernel)
  if (a.pdl_p)
    launch_pdl(project_dmma_kernel<kDmmaKR, MT, NT, NW, NB>, a, gs, NW * 32, smem, s);
  else
    project_dmma_kernel<kDmmaKR, MT, NT, NW, NB><<<gs, NW * 32, smem, s>>>(a);
}

template <int MT, int NT, int NW, int NB>
cudaError_t set_p(int64_t smem) {
  return cudaFuncSetAttribute(project_dmma_kernel<kDmmaKR, MT, NT, NW, NB>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// The warp grid of a project pass (plan.cpp: dmma_project_warps picks NW):
//   NB = 64: W % 32 == 0: NT = 2, MT = W / 32, NW = 16; W % 16 == 0: MT = W / 16,
//            NT = 2 with NW = 8 (two CTAs per SM) or NT = 1 with NW = 16
//   NB = 32: NT = 1; W % 32 == 0: MT = W / 32, NW = 16; W % 16 == 0: MT = W / 16, NW = 8
template <int NB>
void launch_p_nb(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  constexpr int NT64 = NB == 64 ? 2 : 1;
  if (a.wslice % 32 == 0) {
    switch (a.wslice / 32) {
      case 1: launch_p<1, NT64, 16, NB>(a, grid, smem, s); break;
      case 2: launch_p<2, NT64, 16, NB>(a, grid, smem, s); break;
      case 3: launch_p<3, NT64, 16, NB>(a, grid, smem, s); break;
      case 4: launch_p<4, NT64, 16, NB>(a, grid, smem, s); break;
      case 5: launch_p<5, NT64, 16, NB>(a, grid, smem, s); break;
      case 6: launch_p<6, NT64, 16, NB>(a, grid, smem, s); break;
      default: launch_p<7, NT64, 16, NB>(a, grid, smem, s); break;
    }
  } else if (a.dnw == 8) {  // 2 column groups (W/16 M-tiles) x NB/8/NT rhs groups, 2 CTAs per SM
    switch (a.wslice / 16) {
      case 1: launch_p<1, NT64, 8, NB>(a, grid, smem, s); break;
      case 3: launch_p<3, NT64, 8, NB>(a, grid, smem, s); break;
      case 5: launch_p<5, NT64, 8, NB>(a, grid, smem, s); break;
      default: launch_p<7, NT64, 8, NB>(a, grid, smem, s); break;
    }
  } else if constexpr (NB == 64) {  // (NB = 32 needs dnw = 8 here: plan.cpp)
    switch (a.wslice / 16) {
      case 1: launch_p<1, 1, 16, 64>(a, grid, smem, s); break;
      case 3: launch_p<3, 1, 16, 64>(a, grid, smem, s); break;
      case 5: launch_p<5, 1, 16, 64>(a, grid, smem, s); break;
      default: launch_p<7, 1, 16, 64>(a, grid, smem, s); break;
    }
  }
}

template <int NB>
cudaError_t set_p_nb(int64_t smem) {
  constexpr int NT64 = NB == 64 ? 2 : 1;
  cudaError_t e;
  if ((e = set_p<1, NT64, 16, NB>(smem)) || (e = set_p<2, NT64, 16, NB>(smem)) || (e = set_p<3, NT64, 16, NB>(smem)) ||
      (e = set_p<4, NT64, 16, NB>(smem)) || (e = set_p<5, NT64, 16, NB>(smem)) || (e = set_p<6, NT64, 16, NB>(smem)) ||
      (e = set_p<7, NT64, 16, NB>(smem)) || (e = set_p<1, NT64, 8, NB>(smem)) || (e = set_p<3, NT64, 8, NB>(smem)) ||
      (e = set_p<5, NT64, 8, NB>(smem)) || (e = set_p<7, NT64, 8, NB>(smem)))
    return e;
  return cudaSuccess;
}

// NB = 16: NT = 1 (2 rhs groups); W % 32 == 0: MT = W / 32 over 4 column groups,
// NW = 8; W % 16 == 0: MT = W / 16 over 2 column groups, NW = 4
void launch_p16(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if (a.wslice % 32 == 0) {
    switch (a.wslice / 32) {
      case 1: launch_p<1, 1, 8, 16>(a, grid, smem, s); break;
      case 2: launch_p<2, 1, 8, 16>(a, grid, smem, s); break;
      case 3: launch_p<3, 1, 8, 16>(a, grid, smem, s); break;
      case 4: launch_p<4, 1, 8, 16>(a, grid, smem, s); break;
      case 5: launch_p<5, 1, 8, 16>(a, grid, smem, s); break;
      case 6: launch_p<6, 1, 8, 16>(a, grid, smem, s); break;
      default: launch_p<7, 1, 8, 16>(a, grid, smem, s); break;
    }
  } else {
    switch (a.wslice / 16) {
      case 1: launch_p<1, 1, 4, 16>(a, grid, smem, s); break;
      case 3: launch_p<3, 1, 4, 16>(a, grid, smem, s); break;
      case 5: launch_p<5, 1, 4, 16>(a, grid, smem, s); break;
      default: launch_p<7, 1, 4, 16>(a, grid, smem, s); break;
    }
  }
}

// NB = 8: one rhs group (NT = 1); W % 32 == 0: MT = W / 32 over 4 column groups,
// NW = 4; W % 16 == 0: MT = W / 16 over 2 column groups, NW = 2
void launch_p8(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if (a.wslice % 32 == 0) {
    switch (a.wslice / 32) {
      case 1: launch_p<1, 1, 4, 8>(a, grid, smem, s); break;
      case 2: launch_p<2, 1, 4, 8>(a, grid, smem, s); break;
      case 3: launch_p<3, 1, 4, 8>(a, grid, smem, s); break;
      case 4: launch_p<4, 1, 4, 8>(a, grid, smem, s); break;
      case 5: launch_p<5, 1, 4, 8>(a, grid, smem, s); break;
      case 6: launch_p<6, 1, 4, 8>(a, grid, smem, s); break;
      default: launch_p<7, 1, 4, 8>(a, grid, smem, s); break;
    }
  } else if (a.dnw == 3 && a.wslice == 48) {
    launch_p<2, 1, 3, 8>(a, grid, smem, s);
  } else if (a.dnw == 6 && a.wslice == 48) {
    launch_p<1, 1, 6, 8>(a, grid, smem, s);
  } else {
    switch (a.wslice / 16) {
      case 1: launch_p<1, 1, 2, 8>(a, grid, smem, s); break;
      case 3: launch_p<3, 1, 2, 8>(a, grid, smem, s); break;
      case 5: launch_p<5, 1, 2, 8>(a, grid, smem, s); break;
      default: launch_p<7, 1, 2, 8>(a, grid, smem, s); break;
    }
  }
}

cudaError_t set_p8(int64_t smem) {
  cudaError_t e;
  if ((e = set_p<1, 1, 4, 8>(smem)) || (e = set_p<2, 1, 4, 8>(smem)) || (e = set_p<3, 1, 4, 8>(smem)) ||
      (e = set_p<4, 1, 4, 8>(smem)) || (e = set_p<5, 1, 4, 8>(smem)) || (e = set_p<6, 1, 4, 8>(smem)) ||
      (e = set_p<7, 1, 4, 8>(smem)) || (e = set_p<1, 1, 2, 8>(smem)) || (e = set_p<3, 1, 2, 8>(smem)) ||
      (e = set_p<5, 1, 2, 8>(smem)) || (e = set_p<7, 1, 2, 8>(smem)) || (e = set_p<2, 1, 3, 8>(smem)) ||
      (e = set_p<1, 1, 6, 8>(smem)))
    return e;
  return cudaSuccess;
}

cudaError_t set_p16(int64_t smem) {
  cudaError_t e;
  if ((e = set_p<1, 1, 8, 16>(smem)) || (e = set_p<2, 1, 8, 16>(smem)) || (e = set_p<3, 1, 8, 16>(smem)) ||
      (e = set_p<4, 1, 8, 16>(smem)) || (e = set_p<5, 1, 8, 16>(smem)) || (e = set_p<6, 1, 8, 16>(smem)) ||
      (e = set_p<7, 1, 8, 16>(smem)) || (e = set_p<1, 1, 4, 16>(smem)) || (e = set_p<3, 1, 4, 16>(smem)) ||
      (e = set_p<5, 1, 4, 16>(smem)) || (e = set_p<7, 1, 4, 16>(smem)))
    return e;
  return cudaSuccess;
}

template <int KC, int NB, bool WF>
void launch_e_wf(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if (a.pdl)
    launch_pdl(expand_dmma_kernel<KC, NB, WF>, a, grid, kThreadsE, smem, s);
  else
    expand_dmma_kernel<KC, NB, WF><<<grid, kThreadsE, smem, s>>>(a);
}

template <int KC, int NB>
void launch_e_kc(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  const uint64_t all_lv = a.L >= 64 ? ~0ull : (1ull << a.L) - 1;
  const bool wf = !a.adm && a.dense && (a.level_mask & all_lv) == all_lv && !(a.dbg & 16);
  if (wf)
    launch_e_wf<KC, NB, true>(a, grid, smem, s);
  else  // (the general variant's ~100 registers fit 2 CTAs per SM: a grid of 3 per SM would run a second wave)
    launch_e_wf<KC, NB, false>(a, a.grid_e_gen > 0 && a.grid_e_gen < grid ? a.grid_e_gen : grid, smem, s);
}

template <int NB>
void launch_e(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  if (a.dkc == 16)
    launch_e_kc<16, NB>(a, grid, smem, s);
  else if (a.dkc == 48)
    launch_e_kc<48, NB>(a, grid, smem, s);
  else
    launch_e_kc<32, NB>(a, grid, smem, s);
}

template <int NB, bool WF>
cudaError_t set_e_wf(int64_t smem) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(expand_dmma_kernel<16, NB, WF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) ||
      (e = cudaFuncSetAttribute(expand_dmma_kernel<48, NB, WF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
    return e;
  return cudaFuncSetAttribute(expand_dmma_kernel<32, NB, WF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int NB>
cudaError_t set_e(int64_t smem) {
  const cudaError_t e = set_e_wf<NB, false>(smem);
  return e != cudaSuccess ? e : set_e_wf<NB, true>(smem);
}

// Wait for the P ranks' flags of this pass, then exchange[o] = sum over ranks g
// (in rank order) of slot g of this rank's mailbox: the summed exchange levels
// the tensor-core expand reads.  Bounded wait: a timeout is reported through
// the handle's error word (peer_wait_flags), never a trap or a hung GPU.
__global__ void peer_sum_kernel(const __grid_constant__ StreamArgs a, double* __restrict__ out) {
  const int par = static_cast<int>(a.epoch & 1);
  const double* mb = a.mbox[a.rank] + (int64_t)par * a.P * a.mb;
  if (threadIdx.x == 0) peer_wait_flags(a);
  __syncthreads();
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < a.exch; o += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int g = 0; g < a.P; ++g) v += dev::ld_cg(mb + (int64_t)g * a.mb + o);
    out[o] = v;
  }
}

// Standard admissibility, P > 1: received z entries [e][NB][r] of the packed
// buffer -> this rank's fragment-major Zt rows (the SIMT path's
// std_unpack_z_kernel for the tensor-core layout)
template <int NB>
__global__ void std_unpack_z_dmma_kernel(double* __restrict__ zt, const double* __restrict__ xchg,
                                         const int64_t* __restrict__ unpack, int64_t n_unpack, int nr, int W, int r) {
  const int64_t total = n_unpack * nr * r;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t it = o / ((int64_t)nr * r);
    const int rem = static_cast<int>(o - it * nr * r);
    const int n = rem / r, aa = rem - n * r;
    const int64_t e = unpack[2 * it], rq = unpack[2 * it + 1];
    const int64_t row = rq >> 8;
    const int q = static_cast<int>(rq & 255);
    zt[row * (int64_t)W * NB + zfrag<NB>(q * r + aa, n)] = xchg[(e * NB + n) * r + aa];
  }
}

}  // namespace

cudaError_t launch_std_unpack_z_dmma(double* zt, const double* xchg, const int64_t* unpack, int64_t n_unpack, int nb,
                                     int nr, int W, int r, cudaStream_t s) {
  if (n_unpack == 0) return cudaSuccess;
  int64_t g = (n_unpack * nr * r + 255) / 256;
  const int grid = static_cast<int>(g < 1 ? 1 : g > 148 * 16 ? 148 * 16 : g);
  switch (nb) {
    case 8: std_unpack_z_dmma_kernel<8><<<grid, 256, 0, s>>>(zt, xchg, unpack, n_unpack, nr, W, r); break;
    case 16: std_unpack_z_dmma_kernel<16><<<grid, 256, 0, s>>>(zt, xchg, unpack, n_unpack, nr, W, r); break;
    case 32: std_unpack_z_dmma_kernel<32><<<grid, 256, 0, s>>>(zt, xchg, unpack, n_unpack, nr, W, r); break;
    default: std_unpack_z_dmma_kernel<64><<<grid, 256, 0, s>>>(zt, xchg, unpack, n_unpack, nr, W, r); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_project_dmma(const StreamArgs& a, int nb, int grid, int64_t smem, cudaStream_t s) {
  if (nb == 8)
    launch_p8(a, grid, smem, s);
  else if (nb == 16)
    launch_p16(a, grid, smem, s);
  else if (nb == 32)
    launch_p_nb<32>(a, grid, smem, s);
  else
    launch_p_nb<64>(a, grid, smem, s);
  return cudaGetLastError();
}

cudaError_t launch_expand_dmma(const StreamArgs& a, int nb, int grid, int64_t smem, cudaStream_t s) {
  if (nb == 8)
    launch_e<8>(a, grid, smem, s);
  else if (nb == 16)
    launch_e<16>(a, grid, smem, s);
  else if (nb == 32)
    launch_e<32>(a, grid, smem, s);
  else
    launch_e<64>(a, grid, smem, s);
  return cudaGetLastError();
}

cudaError_t launch_peer_sum(const StreamArgs& a, double* out, cudaStream_t s) {
  if (a.exch <= 0) return cudaSuccess;
  int64_t grid = (a.exch + 255) / 256;
  if (grid > 148) grid = 148;
  peer_sum_kernel<<<static_cast<int>(grid), 256, 0, s>>>(a, out);
  return cudaGetLastError();
}

cudaError_t init_std_tables_dmma(const int16_t* code, const int16_t* slot) {
  cudaError_t e = cudaMemcpyToSymbol(c_std_code_d, code, sizeof(int16_t) * 3 * 8 * kStdMaxSlots);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(c_std_slot_d, slot, sizeof(int16_t) * 3 * 8 * kStdMaxCodes);
}

cudaError_t configure_dmma(int nb, int64_t smem_p, int64_t smem_e) {
  cudaError_t e;
  if (nb == 8) {
    if ((e = set_p8(smem_p))) return e;
    return set_e<8>(smem_e);
  }
  if (nb == 16) {
    if ((e = set_p16(smem_p))) return e;
    return set_e<16>(smem_e);
  }
  if (nb == 32) {
    if ((e = set_p_nb<32>(smem_p))) return e;
    return set_e<32>(smem_e);
  }
  if ((e = set_p_nb<64>(smem_p)) || (e = set_p<1, 1, 16, 64>(smem_p)) || (e = set_p<3, 1, 16, 64>(smem_p)) ||
      (e = set_p<5, 1, 16, 64>(smem_p)) || (e = set_p<7, 1, 16, 64>(smem_p)))
    return e;
  return set_e<64>(smem_e);
}

}  // namespace hmat
