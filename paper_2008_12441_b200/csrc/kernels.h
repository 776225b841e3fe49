// kernels.h -- parameter blocks and launchers of the sm_100a H-matvec kernels.
//
//   project  Step 1 + on-chip Step 2: z_ts = V_ts^T x_s for
//            every sibling block at every level (eq:prod-vx), as per-CTA
//            contiguous row ranges streamed by bulk TMA, with a deterministic
//            last-CTA reduction of node sums that cross CTA ranges; results
//            scattered target-major (Zt_l[t][slot(t->s)]).
//   expand   Step 5: y_i = sum_l U_l[i,:] . Zt_l[t(i)] +
//            D_k[i,:] . x_k (eq:prod-yuz, eq:prod-ydz), fused over siblings,
//            levels and the dense leaf blocks so y is written once.
#pragma once
#include <cuda.h>  // CUtensorMap (type only; maps are encoded through the runtime's driver entry point)
#include <cuda_runtime.h>

#include <cstdint>

#include "plan.h"

namespace hmat {

struct LevelArgs {
  int64_t m;         // rows per node at this level (global)
  int64_t seg_rows;  // rows of one local segment = min(m, N_loc)
  double* zt;        // Zt_l (target-major, pitch Wp*NR), already offset for this pass
  int64_t tbase;     // global index of zt's first target (= first local source node)
  // standard admissibility, P > 1 (std_exchange.h): [source node - tbase][M] ->
  // entry of the packed cross-rank buffer, or -1 for a pair inside this rank
  const int32_t* xent;
};

struct StreamArgs {
  // panels
  const double* U;   // level-major, level l at U + (l-1)*panel_stride, rows pitch Wp
  const double* V;
  const double* D;   // N_loc x Dp
  int64_t panel_stride;
  // vectors (16-byte aligned base, column-major)
  const double* x;
  int64_t ldx;
  double* y;
  int64_t ldy;
  int nr;            // active right-hand sides in this pass (<= NR template)
  double alpha, beta;  // y = alpha op(H) x + beta y (beta == 0: y is not read)
  // shape
  int L, c, r, W, Wp, Dp, b;
  int d, adm, nd;        // dim; admissibility (0 weak, 1 standard); dense panels
  int64_t d_stride;      // doubles between dense panels (standard: one per neighbour offset)
  int64_t N_loc, row0;
  uint64_t level_mask;
  int dense;
  // project schedule
  int Rp, nstage_p;
  int64_t stage_bytes_p, stages_p;
  double* part;      // [L][grid_p][2][Wp*NR] partial node sums
  int* cnt;          // [L][grid_p] arrival tickets
  // expand schedule
  int Re, tpr, nstage_e;
  int ndc, dc;       // expand: dense stages per item (weak, ndc > 1: column chunks of dc columns, box tm_dse;
  int dgs;           //   standard: groups of dgs near-field blocks)
  int64_t chunk_e;   // expand: 0 = static item ranges; > 0 = dynamic chunks of chunk_e items
  int* sched;        // expand: [next chunk, CTAs done] (re-armed by the last CTA)
  int dyn_level;     // project: the level handed out in dynamic chunks (0 = none)
  int64_t dyn_chunk; // project: stages per chunk (a multiple of the level's node size)
  int* sched_p;      // project: [next chunk, CTAs done]
  int64_t stage_bytes_e, items_e;
  int64_t item0;     // expand: first item of this launch (row chunks of a host-y product; 0 = from the start)
  int64_t e_items;   // tensor-core expand: items of this launch (0 = all)
  int xs_p, xs_e;
  int vp;              // DMMA project: smem pitch of staged V rows
  int dkr;             // DMMA project: V rows per stage (32)
  int dkc;             // DMMA expand: k-columns per level stage (32; 48 at W = 48; else 16)
  int dnw;             // DMMA project: warps per CTA (16, or 8 with two CTAs per SM)
  int dbg;             // diagnostics only (HMAT_DEBUG_SKIP): bit 0 skips project's math, bit 1 expand's
  int snake;           // project: even levels stream their range backwards (x tail reused from L2)
  int pdl;             // expand launched as a programmatic dependent of project (HMAT_PDL)
  int lpar;            // project: level-parallel mode (one stage of one level per CTA)
  int pdl_p;           // project launched as a programmatic dependent of the previous kernel
  // in-kernel peer exchange (HMAT_EXCHANGE_PEER): the last project
  // CTA pushes this rank's exchange levels into slot `rank` of every rank's
  // mailbox and raises its flag there; expand sums the P slots in rank order
  int peer, P, rank;
  double* const* mbox;       // [P] device pointers: each rank's mailbox base (peer memory)
  int64_t mb;                // doubles per slot (this pass's exchange levels, padded)
  uint64_t epoch;            // pass counter (identical on all ranks)
  unsigned int* done;        // project CTAs finished (last one pushes)
  unsigned int* err;         // host-mapped error word: a flag wait that timed out (peer.cuh)
  int64_t peer_timeout_ns;   // bound on a flag wait (HMAT_PEER_TIMEOUT_MS)
  int early;                 // project: release a ring slot before the FMAs (HMAT_PROJECT_EARLY)
  int eshape;                // expand: compile-time consumer shapes, 1 rhs (HMAT_EXPAND_SHAPE)
  int dmma_ileave;           // tensor-core expand: interleaved item order (HMAT_DMMA_ILEAVE)
  int skip_remote;           // standard H^T, P > 1: expand skips near-field blocks of remote neighbours
  int wslice, nslice;        // tensor-core project: column slices of the panel (gridDim.y = nslice)
  int aflush;                // project: asynchronous node flushes (HMAT_PROJECT_AFLUSH)
  int dmma_upol;             // tensor-core expand: L2 policy of the U / D boxes (HMAT_DMMA_UPOL)
  int grid_e_gen;            // tensor-core expand: grid of the general variant (<= the plan's grid)
  int64_t pchunk;            // tensor-core project: stages per chunk of the level interleave (0 = off)
  double* accbuf;            // tensor-core project: [grid][L][W NB] running sums between chunks
  const double* zex_base;    // local exchange buffer (offsets of the exchange levels)
  int64_t exch;              // doubles of this pass's exchange levels
  int cross;                 // levels 1..cross are exchange levels
  // standard admissibility, P > 1 (std_exchange.h): the packed cross-rank buffer
  // [E][NR][r] z entries then [Hn][NR][bpad] halo x; halo_of[local leaf][nd] =
  // halo index of near-field neighbour e (-1: local or outside the domain)
  double* xchg;
  const int32_t* halo_of;
  int64_t halo_base;         // doubles before the halo x region (E r NR)
  int bpad;
  unsigned long long* trace; // optional per-CTA [start ns, end ns, SM id] (hmat_cta_trace)
  int64_t red_off_p;   // byte offsets inside the dynamic shared memory
  int64_t bar_off_p, bar_off_e;
  LevelArgs lv[kMaxLevels + 1];
  // DMMA project (tensor TMA, one copy per operand per stage):
  //   tm_v  3-D map over the V-role panels [L][N_loc][Wp], box [1][dkr][vp]
  //         (the vp - Wp padding columns are out of bounds: zero-filled);
  //   tm_x  2-D map over this pass's x columns [nr][N_loc] (ld = ldx), box
  //         [64][dkr + 4]: the staged x block with the conflict-free pitch.
  alignas(64) CUtensorMap tm_v;
  alignas(64) CUtensorMap tm_x;
  // DMMA expand: tm_u 3-D over the U-role panels, box [1][64][KC+4]; tm_d 2-D
  // over the D-role panel [N_loc][Dp], box [64][KC+4]; tm_xe like tm_x with box
  // [64][KC+4]
  alignas(64) CUtensorMap tm_u;
  alignas(64) CUtensorMap tm_d;
  alignas(64) CUtensorMap tm_xe;
  // SIMT expand with ndc > 1: 2-D map over the D-role panel [N_loc][Dp], box [Re][dc]
  alignas(64) CUtensorMap tm_dse;
  // DMMA expand, standard admissibility, P > 1: 2-D map over the packed buffer's
  // halo x [Hn NB][bpad] (row h NB + n: halo leaf h, rhs n), box [NB][KC+4]
  alignas(64) CUtensorMap tm_xh;
};

// Launch one project pass (template NR chosen from args.nr).  grid = plan.grid_p.
cudaError_t launch_project(const StreamArgs& a, int nr_cap, int grid, int64_t smem, cudaStream_t s);
// Launch one expand pass.  grid = plan.grid_e.
cudaError_t launch_expand(const StreamArgs& a, int nr_cap, int grid, int64_t smem, cudaStream_t s);
// FP64 tensor-core (DMMA) passes of kDmmaNB right-hand sides (kernels_dmma.cu).
// Launch `kernel(a)` as a programmatic dependent of the previous kernel on `s`
// (PDL: its CTAs may start while that kernel's last CTAs finish; the kernel
// calls griddepcontrol.wait before reading what the previous one wrote).
template <typename Kernel>
cudaError_t launch_pdl(Kernel kernel, const StreamArgs& a, int grid, int threads, int64_t smem, cudaStream_t s,
                       int grid_y = 1) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid), static_cast<unsigned>(grid_y));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

// nb: the pass width (32 or 64 right-hand sides; plan.h DmmaLayout).
cudaError_t launch_project_dmma(const StreamArgs& a, int nb, int grid, int64_t smem, cudaStream_t s);
cudaError_t launch_expand_dmma(const StreamArgs& a, int nb, int grid, int64_t smem, cudaStream_t s);
// standard admissibility, P > 1: received z entries [e][nb][r] -> fragment-major Zt rows
cudaError_t launch_std_unpack_z_dmma(double* zt, const double* xchg, const int64_t* unpack, int64_t n_unpack, int nb,
                                     int nr, int W, int r, cudaStream_t s);
cudaError_t configure_dmma(int nb, int64_t smem_p, int64_t smem_e);
// PEER exchange on the tensor-core path: wait for the P ranks' flags of this
// pass, then out[0..a.exch) = the rank-ordered sum of this rank's P mailbox slots.
cudaError_t launch_peer_sum(const StreamArgs& a, double* out, cudaStream_t s);
// Standard admissibility: upload the interaction-list slot tables (plan.h
// std_slot_tables) to the project kernel's constant memory (per device).
cudaError_t init_std_tables(const int16_t* code, const int16_t* slot);
// Standard admissibility, P > 1 (std_exchange.h): copy this rank's boundary-leaf
// x into the packed buffer (before project) / the received z entries of its
// targets into its Zt rows (after the exchange, before expand).
cudaError_t launch_std_pack_x(double* xchg_halo, const double* x, int64_t ldx, const int64_t* pack, int64_t n_pack,
                              int cap, int nr, int b, int bpad, cudaStream_t s);
cudaError_t launch_std_unpack_z(double* zt, const double* xchg, const int64_t* unpack, int64_t n_unpack, int cap,
                                int nr, int Wp, int r, cudaStream_t s);
// Standard admissibility: the transposed near-field panels of H^T (one-time
// helper); leaves lbase .. lbase + n_leaves - 1 of this rank, blocks whose
// neighbour lies on another rank stay zero (their products travel in the exchange).
cudaError_t launch_transpose_near_field(const double* D, double* Dt, int64_t n_leaves, int64_t lbase, int d, int L,
                                        int b, int Dp, int64_t d_stride, int nd, cudaStream_t s);
// Standard admissibility, H^T with P > 1 (std_exchange.h): the products
// c_{S,T} = (D_{S,T})^T x_S of this rank's outgoing cross near-field pairs into the
// packed buffer (before project), and y_T += alpha sum c_{S,T} of the incoming
// ones in pair order (after expand).
cudaError_t launch_std_tpack(double* out, const double* D, int64_t d_stride, int Dp, const double* x, int64_t ldx,
                             const int64_t* tpack, int64_t n_pairs, int cap, int nr, int b, int bpad, cudaStream_t s);
cudaError_t launch_std_tadd(double* y, int64_t ldy, double alpha, const double* in, const int64_t* leaf,
                            const int64_t* off, const int64_t* pairs, int64_t n_leaves, int cap, int nr, int b,
                            int bpad, cudaStream_t s);
// D^T of every dense leaf block (for H^T x); one-time helper.
cudaError_t launch_transpose_leaf_blocks(const double* D, double* Dt, int64_t n_leaves, int b, int Dp, cudaStream_t s);
// Standard admissibility on the tensor-core path: the slot tables of the
// interaction lists (as init_std_tables) for kernels_dmma.cu's constant memory.
cudaError_t init_std_tables_dmma(const int16_t* code, const int16_t* slot);
// Opt the kernels into large dynamic shared memory (once per device).
cudaError_t configure_kernels(int64_t smem_p, int64_t smem_e);  // max over layouts

}  // namespace hmat
