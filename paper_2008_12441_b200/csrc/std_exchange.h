// std_exchange.h -- the cross-GPU exchange of the standard-admissibility
// H-matvec with P > 1 ranks owning contiguous Morton slices.
//
// Under standard admissibility a node interacts with the children of its
// parent's 3^d neighbours, so blocks (t, s) whose
// target and source sit on different ranks exist at every level along the
// slice boundaries, and the dense near field of a boundary leaf needs x of its
// neighbour leaves on other ranks: the O((N/P)^{(d-1)/d}) halo of
// PAPER.md:1061-1068.  Both travel in ONE packed buffer per pass, the same on
// every rank ("global packed cross array"):
//
//   [E z entries][cap rhs][r]        entry (l, t, q): z_{t, s_q} = V_{t,s_q}^T x_{s_q}
//   [Hn halo leaves][cap rhs][bpad]  x of a leaf some other rank needs
//
// Entries are numbered by a global enumeration (levels 2..L, targets in Morton
// order, slots in order; halo leaves in Morton order), so every rank computes
// the same numbering from the plan alone.  Each rank writes what it owns (its
// sources' complete or partial z, its leaves' x), zeros elsewhere; the buffer is
// summed over the ranks (ncclAllReduce, or the caller in the split-phase API);
// each rank then copies the z entries of its targets into its local Zt rows and
// reads halo x directly from the buffer.  A pair is "cross" unless target and
// source lie inside the same rank (pairs touching a node that spans ranks are
// always cross: its z is a sum of per-rank partials).
//
// The transposed product H^T (GEMV "T") has the same
// interaction pairs (the relation is symmetric), so the z entries and their
// tables serve it unchanged with U and V swapping roles.  Its near field is
// y_T += (D_{S,T})^T x_S, and for S on another rank the block D_{S,T} lives
// there (row block S): instead of the halo x, the buffer's second part carries
// one product per cross near-field pair, computed by the rank owning S,
//   [Hp pairs][cap rhs][bpad]        c_{S,T} = (D_{S,T})^T x_S,
// and the rank owning T adds its incoming c's to y_T after the expand kernel
// (which skips the remote blocks), in pair order: deterministic.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "plan.h"

namespace hmat {

struct StdExchange {
  int64_t E = 0;   // global z entries
  int64_t Hn = 0;  // global halo leaves
  int bpad = 0;    // leaf_size rounded up to even (16-byte aligned x segments)
  // this rank
  // project: entry of (local source node, slot q of the source) or -1 (local pair),
  // per level l in 2..L at src_off[l]: [node - sbase][M]
  std::vector<int32_t> src_entry;
  int64_t src_off[kMaxLevels + 1] = {};
  // expand: z entries of this rank's targets -> its Zt rows: {entry, zt_row * 256 + q}
  std::vector<int64_t> unpack;
  // x of this rank's leaves other ranks need: {halo index, local leaf}
  std::vector<int64_t> pack;
  // [local leaf][3^d]: halo index of neighbour e, -1 when local / outside the domain
  std::vector<int32_t> halo_of;
  // H^T: cross near-field pairs (S, T), owner(S) != owner(T), numbered over leaves S
  // in Morton order then neighbour e (T = S + eps_e)
  int64_t Hp = 0;
  std::vector<int64_t> tpack;     // this rank's outgoing pairs: {pair, local leaf S, e}
  std::vector<int64_t> tadd_leaf; // this rank's leaves T with incoming pairs (local index)
  std::vector<int64_t> tadd_off;  // CSR offsets into tadd_pair (size tadd_leaf + 1)
  std::vector<int64_t> tadd_pair; // incoming pair indices, ascending per leaf
  // doubles of the packed buffer for a pass of `cap` right-hand sides
  int64_t halo_base(int cap, int r) const { return (E * r * cap + 1) / 2 * 2; }  // 16-byte aligned
  int64_t doubles(int cap, int r) const { return halo_base(cap, r) + Hn * bpad * cap; }
  int64_t doubles_t(int cap, int r) const { return halo_base(cap, r) + Hp * bpad * cap; }  // H^T
  int64_t doubles_max(int cap, int r) const { return halo_base(cap, r) + (Hn > Hp ? Hn : Hp) * bpad * cap; }
};

// Requires p.adm == 1 (standard admissibility).  Returns "" on success.
std::string std_exchange_build(const Plan& p, StdExchange* out);

}  // namespace hmat
