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
//   * grid = min(#SM x CTAs/SM, #stages); CTA b owns the contiguous stage range
//     [S b / G, S (b+1) / G) of the L * N_loc / Rp stages, so every CTA streams
//     the same number of bytes.
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
#include "kernels.h"

namespace hmat {
namespace {

constexpr int CT = kConsumerThreads;
constexpr int NCW = CT / 32;
constexpr int MAXCPT = 4;  // columns per consumer thread when W > CT

// CTA owning stage k under the even split [S b / G, S (b+1) / G).
__device__ __forceinline__ int64_t owner_of(int64_t k, int64_t S, int64_t G) { return ((k + 1) * G - 1) / S; }

// z value (column col = q r + a of source node sg, rhs kk) -> Zt_l of target
// t = q-th sibling of sg, at slot(t -> sg).
template <int NR>
__device__ __forceinline__ void scatter_z(const StreamArgs& a, const LevelArgs& lv, int64_t sg, int col, int kk,
                                          double v) {
  const int d = __ffs(a.c) - 1;  // c = 2^d
  const int q = col / a.r, aa = col - q * a.r;
  const int me = static_cast<int>(sg & (a.c - 1));
  const int64_t t = ((sg >> d) << d) + (q < me ? q : q + 1);
  const int tc = static_cast<int>(t & (a.c - 1));
  const int qt = me < tc ? me : me - 1;
  lv.zt[(t - lv.tbase) * (int64_t)a.Wp * NR + (int64_t)(qt * a.r + aa) * NR + kk] = v;
}

template <int NR>
__global__ void __launch_bounds__(kThreads, 1) project_kernel(const __grid_constant__ StreamArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t G = gridDim.x, bid = blockIdx.x;
  const int64_t S = a.stages_p;
  const int64_t k0 = S * bid / G, k1 = S * (bid + 1) / G;
  const int Rp = a.Rp, W = a.W, Wp = a.Wp;
  const int64_t SL = a.N_loc / Rp;  // stages per level
  const int NS = a.nstage_p;
  double* red = reinterpret_cast<double*>(smem + a.red_off_p);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off_p);
  uint64_t* empty = full + NS;
  volatile int* flag = reinterpret_cast<volatile int*>(empty + NS);

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      dev::mbar_init(&full[i], 1);
      dev::mbar_init(&empty[i], NCW);
    }
    dev::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer: one lane streams V_l rows + x segments -------
    if (lane == 0) {
      const uint64_t pol_stream = dev::policy_evict_first();
      const uint64_t pol_keep = dev::policy_evict_last();
      const uint32_t vbytes = static_cast<uint32_t>(Rp * Wp * 8);
      int it = 0;
      int64_t l = k0 / SL + 1, kl = k0 - (l - 1) * SL;  // level and stage-in-level of k
      for (int64_t k = k0; k < k1;) {
        if (!((a.level_mask >> (l - 1)) & 1ull)) {  // masked level: skip it
          k += SL - kl;
          ++l;
          kl = 0;
          continue;
        }
        const int slot = it % NS;
        if (it >= NS) dev::mbar_wait(&empty[slot], ((it / NS) & 1) ^ 1);
        const int64_t i0 = kl * Rp;
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
        dev::mbar_arrive_expect_tx(&full[slot], total);
        dev::bulk_g2s(st, a.V + (l - 1) * a.panel_stride + i0 * Wp, vbytes, &full[slot], pol_stream);
#pragma unroll
        for (int kk = 0; kk < NR; ++kk)
          if (kk < a.nr)
            dev::bulk_g2s(st + vbytes + kk * a.xs_p * 8, a.x + lo[kk], xb[kk], &full[slot], pol_keep);
        ++it;
        ++k;
        if (++kl == SL) {
          kl = 0;
          ++l;
        }
      }
    }
    return;
  }

  // ---------------- consumers ------------------------------------------------
  const int t = tid - 32;
  const int RG = W <= CT ? CT / W : 1;
  const int rho = W <= CT ? t / W : 0;
  const int col0 = W <= CT ? t % W : t;
  const bool active = rho < RG;
  const int cpt = W <= CT ? 1 : (W + CT - 1) / CT;
  double acc[MAXCPT][NR];
#pragma unroll
  for (int j = 0; j < MAXCPT; ++j)
#pragma unroll
    for (int kk = 0; kk < NR; ++kk) acc[j][kk] = 0.0;

  int it = 0;
  int64_t l = k0 / SL + 1, kl = k0 - (l - 1) * SL;
  // node (segment) cursor of the current level: seg_stages stages per local
  // node, sl = local node index, pos = stage index inside the node
  int64_t seg_stages = 0, sl = 0, pos = 0, sg0 = 0;
  int64_t cur_level = -1;
  for (int64_t k = k0; k < k1;) {
    if (!((a.level_mask >> (l - 1)) & 1ull)) {
      k += SL - kl;
      ++l;
      kl = 0;
      continue;
    }
    if (l != cur_level) {  // entering a level: one set of divisions per level
      cur_level = l;
      seg_stages = a.lv[l].seg_rows / Rp;
      sl = kl / seg_stages;
      pos = kl - sl * seg_stages;
      sg0 = a.row0 / a.lv[l].m;
    }
    const int slot = it % NS;
    dev::mbar_wait(&full[slot], (it / NS) & 1);
    const int64_t i0 = kl * Rp;
    const unsigned char* st = smem + slot * a.stage_bytes_p;
    const double* Vs = reinterpret_cast<const double*>(st);
    const double* xs = reinterpret_cast<const double*>(st + Rp * Wp * 8);
    int xo[NR];
#pragma unroll
    for (int kk = 0; kk < NR; ++kk) xo[kk] = kk * a.xs_p + static_cast<int>((kk * a.ldx + i0) & 1);
    if (active) {
#pragma unroll 4
      for (int row = rho; row < Rp; row += RG) {
        double xv[NR];
#pragma unroll
        for (int kk = 0; kk < NR; ++kk) xv[kk] = kk < a.nr ? xs[xo[kk] + row] : 0.0;
#pragma unroll
        for (int j = 0; j < MAXCPT; ++j) {
          const int col = col0 + j * CT;
          if (j < cpt && col < W) {
            const double v = Vs[row * Wp + col];
#pragma unroll
            for (int kk = 0; kk < NR; ++kk) acc[j][kk] = fma(v, xv[kk], acc[j][kk]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) dev::mbar_arrive(&empty[slot]);
    ++it;
    const bool node_end = (pos + 1 == seg_stages);
    const bool range_end = (k + 1 == k1);
    const int64_t this_l = l, this_sl = sl;
    // advance the cursors to the next stage
    ++k;
    if (++pos == seg_stages) {
      pos = 0;
      ++sl;
    }
    if (++kl == SL) {
      kl = 0;
      ++l;
    }
    if (!node_end && !range_end) continue;

    // ---- end of a (local) node at this level, or end of this CTA's range ----
    const LevelArgs& lv = a.lv[this_l];
    const int64_t sa = (this_l - 1) * SL + this_sl * seg_stages, sb = sa + seg_stages;
    const bool complete = sa >= k0 && sb <= k1;
    const int64_t sg = sg0 + this_sl;                           // global source node
    if (active) {
#pragma unroll
      for (int j = 0; j < MAXCPT; ++j) {
        const int col = col0 + j * CT;
        if (j < cpt && col < W) {
#pragma unroll
          for (int kk = 0; kk < NR; ++kk) {
            red[((int64_t)rho * Wp + col) * NR + kk] = acc[j][kk];
            acc[j][kk] = 0.0;
          }
        }
      }
    }
    dev::named_bar_sync(1, CT);
    if (complete) {
      for (int o = t; o < W * NR; o += CT) {
        const int col = o / NR, kk = o - col * NR;
        double v = 0.0;
        for (int g = 0; g < RG; ++g) v += red[((int64_t)g * Wp + col) * NR + kk];
        if (kk < a.nr) scatter_z<NR>(a, lv, sg, col, kk, v);
      }
      dev::named_bar_sync(1, CT);
    } else {
      // partial node sum of this CTA: slot 0 if the node holds our first
      // stage, slot 1 otherwise (it then holds our last stage)
      const int myslot = sa <= k0 ? 0 : 1;
      double* pp = a.part + (bid * 2 + myslot) * (int64_t)Wp * NR;
      for (int o = t; o < W * NR; o += CT) {
        const int col = o / NR, kk = o - col * NR;
        double v = 0.0;
        for (int g = 0; g < RG; ++g) v += red[((int64_t)g * Wp + col) * NR + kk];
        pp[(int64_t)col * NR + kk] = v;
      }
      __threadfence();
      dev::named_bar_sync(1, CT);
      const int64_t b0 = owner_of(sa, S, G), b1 = owner_of(sb - 1, S, G);
      if (t == 0) {
        const int prev = atomicAdd(&a.cnt[b1], 1);
        *flag = (prev == static_cast<int>(b1 - b0)) ? 1 : 0;
      }
      dev::named_bar_sync(1, CT);
      if (*flag) {
        __threadfence();
        const int64_t kb0 = S * b0 / G;
        const int slot0 = (sa == kb0) ? 0 : 1;
        for (int o = t; o < W * NR; o += CT) {
          const int col = o / NR, kk = o - col * NR;
          double v = 0.0;
          for (int64_t bb = b0; bb <= b1; ++bb) {
            const int sl_b = bb == b0 ? slot0 : 0;
            v += dev::ld_cg(a.part + (bb * 2 + sl_b) * (int64_t)Wp * NR + (int64_t)col * NR + kk);
          }
          if (kk < a.nr) scatter_z<NR>(a, lv, sg, col, kk, v);
        }
        if (t == 0) a.cnt[b1] = 0;  // re-arm the ticket for the next launch
      }
      dev::named_bar_sync(1, CT);
    }
  }
}

template <int NR>
cudaError_t launch_nr(const StreamArgs& a, int grid, int64_t smem, cudaStream_t s) {
  project_kernel<NR><<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
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

cudaError_t configure_project(int64_t smem) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(project_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  if ((e = cudaFuncSetAttribute(project_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  if ((e = cudaFuncSetAttribute(project_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem))) return e;
  return cudaFuncSetAttribute(project_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace hmat
