/*
 * hmat.h -- C ABI of the B200-native weak-admissibility H-matrix-vector
 * product y = H x (arXiv 2008.12441, Li, Poulson & Ying, "Distributed-memory
 * H-matrix algebra I").  Implemented by paper_2008_12441_b200/libhmat.so
 * (sm_100a kernels + host plan; NCCL loaded on demand for nranks > 1).
 *
 * The operation (eq:hmat-vec-add): y is initialised to zero
 * and, for every block K_{t x s} of H holding data, y_t += D_ts x_s (dense) or
 * y_t += U_ts (V_ts^T x_s) (low rank).  The structure is Def 2.4
 * on the 2^dim-ary domain tree of an ideal dim-dimensional
 * domain under weak admissibility, in
 * the reading of DESIGN.md R1: every node t at levels 1..depth has a rank-`rank`
 * block U_ts V_ts^T against each of its 2^dim - 1 siblings s; the leaf-diagonal
 * blocks D_k (leaf_size x leaf_size) are dense; nothing else holds data.
 *
 * Notation: c = 2^dim, L = depth, b = leaf_size, r = rank, N = b c^L,
 * m_l = N / c^l (rows of a level-l node), W = (c-1) r.  Points are in Morton
 * (Z-) order so every tree node is a contiguous index range: node k of level l
 * owns rows [k m_l, (k+1) m_l).  Siblings of t are the other children of t's
 * parent, in ascending child order; slot(t -> s) is s's position in that list.
 *
 * CANONICAL PANELS (the input format; row-major, Morton rows):
 *   U[l-1]  N_loc x W  row i, columns [q r, (q+1) r): row i - t m_l of U_{t,s_q}
 *           where t = i / m_l and s_q is t's q-th sibling (target-major).
 *   V[l-1]  N_loc x W  row j, columns [q r, (q+1) r): row j - s m_l of V_{t_q,s}
 *           where s = j / m_l and t_q is s's q-th sibling (source-major).
 *   D       N_loc x b  row i: row i - k b of D_k, k = i / b.
 * Block K_{t x s} = U_ts V_ts^T with U_ts in R^{|t| x r}, V_ts in R^{|s| x r}
 * (PAPER.md:327-334).  With nranks = P > 1, rank g passes only its Morton
 * rows [g N/P, (g+1) N/P) of every panel (the paper's block-row placement, U on
 * the target side, V on the source side; dense blocks on
 * their single owner).
 *
 * VECTORS: x and y are N_loc x nrhs column-major with leading dimension N_loc
 * (block-row distributed exactly like the panels).  They may
 * be device pointers (on H's device) or host pointers; host vectors are copied
 * in/out by the call (a host y of 4 MB or more leaves in row chunks while the
 * expand kernel computes the next ones: HMAT_Y_CHUNKS, default 4, launches the
 * expand once per chunk).  x and y must not alias.  y is overwritten.
 *
 * STREAMS AND SYNCHRONISATION: work is enqueued on H's stream.  With device
 * x/y the call returns without waiting (like a BLAS handle); with a host x or
 * y it returns after y is complete.  With nranks > 1 hmat_matvec is a
 * collective: every rank calls it with the same nrhs in the same order.
 *
 * CUDA GRAPHS: with device x/y (16-byte aligned), profiling off, and one GPU or
 * the NCCL / TREE exchange, a call enqueues only kernels, memsets and NCCL calls
 * on H's stream, so it may be stream-captured (set H's stream to the capturing
 * stream with hmat_set_stream, and make one uncaptured call first: buffers are
 * allocated lazily) and replayed; the kernels re-arm their own work counters.
 * Host vectors and the PEER exchange (a host-side pass counter) are not
 * capture-safe.
 *
 * ERRORS: every entry point returns HMAT_OK or a negative hmat_status and sets
 * a thread-local message readable with hmat_last_error().  Argument checks
 * happen before any device work.  No C++ exception crosses this ABI.
 * Asynchronous device faults surface as HMAT_ERR_CUDA at a later call.
 * Asynchronous EXCHANGE failures surface as HMAT_ERR_NCCL at the next call on
 * H (or at hmat_synchronize / hmat_comm_info): an NCCL communicator error
 * (ncclCommGetAsyncError is polled on every call), or, with the PEER exchange,
 * a flag wait that timed out (HMAT_PEER_TIMEOUT_MS, default 10000): the waiting
 * kernel records the missing rank in a host-mapped error word and finishes
 * without trapping, so the CUDA context stays usable; that product's y is
 * invalid and the error is reported once.
 */
#ifndef HMAT_H
#define HMAT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hmat_s* hmat_t;

typedef enum {
  HMAT_OK = 0,
  HMAT_ERR_INVALID = -1,     /* bad argument (message says which) */
  HMAT_ERR_NOMEM = -2,       /* device allocation failed */
  HMAT_ERR_CUDA = -3,        /* CUDA runtime error (incl. asynchronous faults) */
  HMAT_ERR_NCCL = -4,        /* cross-GPU exchange error: NCCL load / init / collective /
                                asynchronous error, or a PEER flag wait that timed out */
  HMAT_ERR_UNSUPPORTED = -5  /* valid but outside the implemented envelope */
} hmat_status;

/* Multi-GPU placement of one rank (PAPER.md:413-501 process tree on an ideal
 * domain; block-row distribution of the vectors).  NULL =>
 * one GPU, the current device, N_loc = N, a library-owned stream (a blocking
 * stream, so it is ordered with work on the legacy default stream). */
typedef struct {
  int nranks;                 /* P: a power of two <= c^L                            */
  int rank;                   /* 0 <= rank < P; owns Morton rows [rank N/P, ...)     */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId (same on all ranks); P > 1 only */
  void* cuda_stream;          /* cudaStream_t to enqueue on; NULL => library-owned    */
  int device;                 /* CUDA ordinal of this rank's GPU                     */
  int exchange;               /* P > 1: one of HMAT_EXCHANGE_*                       */
} hmat_dist_t;

/* How ranks exchange the projected vectors of the levels whose parent spans
 * more than one GPU (Steps 2-4):
 *   NCCL     ncclAllReduce(sum) of the packed buffer inside hmat_matvec
 *            (needs nccl_unique_id);
 *   EXTERNAL the caller sums the buffer between hmat_project and hmat_expand;
 *   PEER     in-kernel over NVLink peer memory: the project
 *            kernel's last CTA writes this rank's contributions into slot
 *            `rank` of every rank's mailbox and raises a flag there; the expand
 *            kernel waits for the P flags and sums the P slots in rank order.
 *            Mailboxes are connected once with hmat_peer_export/_import (CUDA
 *            IPC, one process per GPU) or hmat_peer_connect_local (one process).
 *            No host or NCCL call per matvec.  On the many-rhs tensor-core
 *            path the project kernel pushes the same way and a small kernel
 *            sums the P slots in rank order before expand.  Not with
 *            standard admissibility.
 *   TREE     the paper's tree-structured Steps 2-4 over NCCL point-to-point
 *            (needs nccl_unique_id): log2 P rounds of recursive doubling on
 *            the hypercube of ranks, round j swapping the packed buffer with
 *            rank ^ 2^j (ncclSend/ncclRecv) and adding the partner's copy;
 *            every rank ends with bit-identical sums (IEEE addition is
 *            commutative), whatever algorithm NCCL would pick for an allreduce.
 *            The recommended exchange (bench.py's default for P > 1). */
#define HMAT_EXCHANGE_NCCL 0
#define HMAT_EXCHANGE_EXTERNAL 1
#define HMAT_EXCHANGE_PEER 2
#define HMAT_EXCHANGE_TREE 3

/* Build H from canonical panels (see above): the H-matrix of Def 2.4
 * on the ideal domain tree under weak
 * admissibility, factors U_ts V_ts^T,
 * O(r N log N) storage.  U and V are arrays of `depth`
 * pointers (ignored when depth == 0); each panel and D may be host (pageable or
 * pinned) or device memory; the library copies them into its own 128-byte
 * aligned per-level device panels, so the caller may free them on return.
 * With dist->nranks = P > 1 each rank passes its rows only.
 * HMAT_ERR_INVALID: dim not in {1,2,3}, depth < 0, leaf_size < 1, rank < 1,
 * N >= 2^62, a NULL pointer, P not a power of two, P > c^L, rank out of range.
 * HMAT_ERR_UNSUPPORTED if (2^dim - 1) * rank > 1024.  HMAT_ERR_NOMEM if the
 * panels do not fit.  HMAT_ERR_NCCL if the NCCL communicator cannot be made. */
hmat_status hmat_create(int depth, int dim, int leaf_size, int rank, const double* const* U,
                        const double* const* V, const double* D, const hmat_dist_t* dist, hmat_t* out);

/* Same as hmat_create but leaves the panels uninitialised
 * (zero); fill them in place through hmat_panel() (no second copy of a 125 GB
 * operator).  Same errors as hmat_create. */
hmat_status hmat_create_uninit(int depth, int dim, int leaf_size, int rank, const hmat_dist_t* dist,
                               hmat_t* out);

/* Device address of one of H's panels (the per-level factor layout of the
 * blocks U_ts, V_ts; dense leaf blocks):
 * kind 0 = U_level, 1 = V_level (level in 1..depth), 2 = D (level ignored; the
 * dense panel index with standard admissibility).  *rows = N_loc, *cols = W (or
 * b), *ld = row pitch in doubles (>= cols; padding columns are never read).
 * HMAT_ERR_INVALID for a bad kind or level.  The pointer stays valid until
 * hmat_destroy; writes must be complete before the next product is enqueued. */
hmat_status hmat_panel(hmat_t H, int kind, int level, double** ptr, int64_t* rows, int64_t* cols,
                       int64_t* ld);

/* y = H x for nrhs right-hand sides: eq:hmat-vec-add with
 * y initialised to zero, computed by the paper's five steps
 * (PAPER.md:652-663): project z_ts = V_ts^T x_s (Step 1, eq:prod-vx,
 * PAPER.md:701-713), on-chip and cross-GPU reduction / transfer / broadcast of
 * the z of blocks whose parent spans ranks (Steps 2-4), then
 * y_t = sum U_ts z_ts + D_t x_t (Step 5, eq:prod-yuz / eq:prod-ydz,
 * PAPER.md:907-959), expand fused over all levels and the dense leaf blocks.
 * x, y: N_loc x nrhs column-major, device or host.  1-2 rhs
 * run on the SIMT streaming kernels; from 3 rhs (HMAT_DMMA_MIN), where W % 16 == 0
 * (W <= 224, or <= 112 if W % 32 != 0) and 64 | leaf_size, on the FP64 tensor
 * cores in passes of 64 rhs, the last one 8, 16 or 32 wide when at most 8 / 16 /
 * 32 remain; standard admissibility from 5 rhs with W % 16 == 0 (any W up to
 * 1024: the project runs in column slices; with P > 1 the packed cross-rank buffer
 * of the standard structure serves both paths).  Other shapes: SIMT passes of up
 * to 4.  HMAT_ERR_INVALID: NULL H/x/y, nrhs < 1, x aliasing y.
 * With P > 1 a collective (same nrhs, same order on every rank); with the
 * EXTERNAL exchange use hmat_project / hmat_expand (HMAT_ERR_UNSUPPORTED). */
hmat_status hmat_matvec(hmat_t H, const double* x, double* y, int nrhs);

/* GEMV form y = alpha op(H) x + beta y ("do not initialize y
 * as a zero vector and modify eq:prod-yuz, eq:prod-yz, eq:prod-ydz
 * accordingly"), op(H) = H (trans = 0) or H^T (trans = 1).  H^T has H's block
 * structure with U and V exchanged and every dense leaf block transposed; the
 * first trans = 1 call builds D^T once (N_loc x leaf_size more device memory).
 * beta == 0: y is write-only (not read).  Same vectors/streams rules as
 * hmat_matvec. */
hmat_status hmat_gemv(hmat_t H, int trans, double alpha, const double* x, double beta, double* y, int nrhs);

/* STANDARD admissibility: Def 2.4 with eq:standard-ad-cond
 * (PAPER.md:279-297), rho = sqrt(d), on [0,1]^dim with a non-periodic boundary:
 * two same-level boxes are admissible iff they do not touch.  Every node t at
 * levels 2..depth has a rank-`rank` block against each box of its interaction
 * list (children of the parent's 3^dim neighbours that do not touch t; at most
 * M = 6^dim - 3^dim); dense blocks D_{t,s} join every pair of
 * touching leaves (3^dim per leaf, incl. t).  Box coordinates: Morton, bit j of
 * coordinate i = bit j dim + i of the node index.
 * Canonical panels:
 *   M slots per node: for a box with child position tau, the candidates are the
 *   children sigma of the parent's neighbours eps in {-1,0,1}^dim, enumerated in
 *   increasing (sum_i (eps_i+1) 3^i) 2^dim + sum_i sigma_i 2^i, skipping those
 *   that touch the box; candidates outside the domain keep their slot (unused).
 *   U[l-1], V[l-1]: N x (M rank), like the weak panels with "sibling q" replaced
 *   by "slot q" (U target-major, V source-major).
 *   Dn: N x (3^dim leaf_size): row i of leaf t, columns [e b, (e+1) b) = row
 *   i - t b of D_{t, t+eps}, e = sum_i (eps_i + 1) 3^i (ignored if outside).
 * hmat_gemv(trans = 1) applies H^T (the interaction relation is symmetric, so
 * U and V swap roles; the near-field panels of H^T, (D_{t+eps,t})^T, are built
 * once on the first transposed call: 3^dim N leaf_size more doubles).
 * nranks > 1 is supported with the NCCL, TREE and EXTERNAL exchanges, for H
 * and H^T: the cross-rank pairs along the slice boundaries and the near-field
 * halo (x for H, the products (D_{S,T})^T x_S for H^T) travel in one packed
 * buffer (hmat_std_exchange_query).  Not supported
 * (HMAT_ERR_UNSUPPORTED): the PEER exchange.  M rank <= 1024.
 * hmat_panel(kind 2, level e) returns dense panel e. */
hmat_status hmat_create_standard(int depth, int dim, int leaf_size, int rank, const double* const* U,
                                 const double* const* V, const double* Dn, const hmat_dist_t* dist, hmat_t* out);
hmat_status hmat_create_standard_uninit(int depth, int dim, int leaf_size, int rank, const hmat_dist_t* dist,
                                        hmat_t* out);

/* Standard admissibility with Def 2.4 read LITERALLY (the
 * three conditions "in the given order", leaf first; the literal alternative to
 * hmat_create_standard's reading, R17): at the leaf level every child
 * pair of two touching leaf-parents is dense (near field AND the leaf-level
 * interaction list), low-rank blocks exist at levels 2..depth-1.  U, V: depth-1
 * canonical standard panels (levels 1..depth-1); Dc: N_loc x (3^dim 2^dim
 * leaf_size): row i of leaf-parent p, columns [e 2^dim b, (e+1) 2^dim b) = row
 * i - p 2^dim b of the dense block of (p, p + eps), e = sum_i (eps_i + 1) 3^i.
 * This is the structure of hmat_create_standard(depth - 1, dim, 2^dim leaf_size,
 * ...) and is built as such (same envelope and errors); depth >= 1. */
hmat_status hmat_create_standard_strict(int depth, int dim, int leaf_size, int rank, const double* const* U,
                                        const double* const* V, const double* Dc, const hmat_dist_t* dist,
                                        hmat_t* out);

/* The paper-strict reading of Def 2.4 (conditions checked in
 * order, "leaf" first): every child pair of a leaf-parent is dense, so each
 * leaf-parent diagonal block (2^dim leaf_size square) is dense and low-rank
 * sibling blocks exist at levels 1..depth-1 only.  U, V: depth-1
 * canonical panels (levels 1..depth-1); Dc: N_loc x (2^dim leaf_size), row i
 * of leaf-parent p = i / (2^dim leaf_size) holds row i - p 2^dim leaf_size of
 * p's dense diagonal block.  This is the structure of hmat_create(depth - 1,
 * dim, 2^dim leaf_size, ...) and is built as such.  depth >= 1
 * (HMAT_ERR_INVALID otherwise); other errors as hmat_create. */
hmat_status hmat_create_strict(int depth, int dim, int leaf_size, int rank, const double* const* U,
                               const double* const* V, const double* Dc, const hmat_dist_t* dist, hmat_t* out);

/* Split-phase form (one pass of right-hand sides: nrhs <= the SIMT pass width,
 * 4 by default, or <= 64 where the tensor-core path takes the product: from 5
 * rhs when W % 16 == 0 within its limits and 64 | leaf_size), for
 * a caller-provided exchange (hmat_dist_t.exchange = HMAT_EXCHANGE_EXTERNAL: MPI,
 * torch.distributed, ...) or to overlap other work.  x, y, exchange are device
 * pointers on H's device; work is enqueued on H's stream.
 *   hmat_exchange_size: doubles of this pass's packed exchange buffer (level-
 *     major, target-major z of the levels whose parent spans > 1 rank; 0 when
 *     P = 1), per hmat_plan_query's layout.
 *   hmat_project: Step 1 + on-chip Step 2; writes this rank's
 *     contributions (partial node sums, zeros elsewhere) to exchange[0..count).
 *   the caller sums exchange over all ranks (Steps 2-4);
 *   hmat_expand: reads the summed exchange, Step 5: y = H x.
 * With HMAT_EXCHANGE_NCCL hmat_matvec does exactly this with an in-place
 * ncclAllReduce (HMAT_EXCHANGE_TREE: the recursive-doubling rounds).  With
 * HMAT_EXCHANGE_PEER `exchange` is ignored (may be NULL): the kernels exchange
 * through the connected mailboxes.  HMAT_ERR_INVALID: more than one pass of
 * rhs, host x / y, NULL exchange where count > 0. */
hmat_status hmat_exchange_size(hmat_t H, int nrhs, int64_t* count);
hmat_status hmat_project(hmat_t H, const double* x, int nrhs, double* exchange);
hmat_status hmat_expand(hmat_t H, const double* x, const double* exchange, double* y, int nrhs);

/* The split-phase form of the GEMV y = alpha op(H) x + beta y,
 * op = H (trans = 0: exactly the three calls above) or H^T (trans = 1; with
 * standard admissibility and P > 1 the buffer's second part carries the
 * products (D_{S,T})^T x_S of the cross-rank near-field pairs instead of halo
 * x, and hmat_expand_op adds the incoming ones after its kernel).  Same rules
 * and errors as above; HMAT_ERR_INVALID for trans not in {0, 1}. */
hmat_status hmat_exchange_size_op(hmat_t H, int trans, int nrhs, int64_t* count);
hmat_status hmat_project_op(hmat_t H, int trans, const double* x, int nrhs, double* exchange);
hmat_status hmat_expand_op(hmat_t H, int trans, double alpha, const double* x, const double* exchange, double beta,
                           double* y, int nrhs);

/* PEER exchange set-up (the fused Steps 2-4, over NVLink
 * peer memory; collective in spirit: every rank must connect before the first
 * product).  hmat_peer_export writes the 64-byte CUDA IPC handle of
 * H's mailbox; after gathering all ranks' handles (rank order), each rank calls
 * hmat_peer_import with them.  hmat_peer_connect_local connects the P handles of
 * ONE process directly (e.g. P shards on one GPU; only the split-phase calls
 * may then be used, projects of all ranks before any expand, since an expand
 * waits for every rank's project); ranks on other devices of the process get
 * peer access enabled (HMAT_ERR_UNSUPPORTED if the devices cannot reach each
 * other).  HMAT_ERR_INVALID: H not a PEER handle, ranks[g] not rank g's handle
 * of the same operator. */
hmat_status hmat_peer_export(hmat_t H, void* handle64);
hmat_status hmat_peer_import(hmat_t H, const void* handles);
hmat_status hmat_peer_connect_local(hmat_t H, const hmat_t* ranks);

/* Diagnostic form of eq:hmat-vec-add restricted to some
 * blocks: only the low-rank levels l with bit (l-1) of level_mask set and, if
 * dense != 0, the dense leaf blocks: y = y_D + sum_{l in mask} y_l.  Errors as
 * hmat_matvec. */
hmat_status hmat_matvec_parts(hmat_t H, const double* x, double* y, int nrhs, uint64_t level_mask,
                              int dense);

/* Frees everything H owns (device panels of PAPER.md:316-339, buffers, the
 * communicator; collective when P > 1).  Waits for H's
 * stream first.  hmat_destroy(NULL) is OK.  Always returns HMAT_OK. */
hmat_status hmat_destroy(hmat_t H);

/* Thread-local message of the last failing call on this thread ("" if none);
 * the text names the failed check or call (SPEC's "dimension mismatch -> error"
 * of the sequential matvec, PAPER.md:363-372 for the operation's shapes). */
const char* hmat_last_error(void);

/* N = b c^L, the global number of points of the domain tree,
 * or -1 if H is NULL. */
int64_t hmat_num_points(hmat_t H);

/* This rank's Morton rows [begin, end) = [rank N/P, (rank+1) N/P): the block-row
 * ownership of x, y and the panels.  HMAT_ERR_INVALID
 * for NULL arguments. */
hmat_status hmat_local_rows(hmat_t H, int64_t* begin, int64_t* end);

/* Make H enqueue on `stream` (a cudaStream_t on H's device) from now on; waits
 * for H's current stream first.  (Execution plumbing of the matvec of
 * PAPER.md:363-388; no paper counterpart.)  HMAT_ERR_INVALID if H is NULL. */
hmat_status hmat_set_stream(hmat_t H, void* stream);

/* Asynchronous host-pointer mode (enable = 1) for the products of
 * PAPER.md:363-388 with host vectors: hmat_matvec / hmat_gemv with a
 * host x or y return as soon as the work is enqueued.  x is copied in on a
 * copy stream, the kernels run on H's stream, y is copied out on another copy
 * stream; the staging buffers alternate between consecutive calls, so one
 * call's copies overlap its neighbours' kernels (a stream of matvecs runs at
 * the kernels' rate, not kernels + PCIe).  The caller keeps x and y valid and
 * unmodified until hmat_synchronize(H) returns (pinned host memory for real
 * overlap; pageable memory is correct but copies synchronously).  Device
 * pointers are unaffected.  Disabling drains the pipeline.  Default: off. */
hmat_status hmat_set_host_async(hmat_t H, int enable);

/* Wait for all work of H (copies in, kernels, copies out; the exchange of
 * PAPER.md:746-904 included), then report any asynchronous exchange error
 * (HMAT_ERR_NCCL, see ERRORS above). */
hmat_status hmat_synchronize(hmat_t H);

/* 128 bytes of a fresh ncclUniqueId for hmat_dist_t (call on one rank and
 * broadcast): the communicator of the cross-GPU Steps 2-4.
 * HMAT_ERR_NCCL if NCCL cannot be loaded, HMAT_ERR_INVALID for NULL. */
hmat_status hmat_nccl_unique_id(void* out128);

/* Diagnostic: runs the library's NCCL layer end to end on ONE GPU -- a fresh
 * unique id, a one-rank communicator on `device`, an in-place sum of `count`
 * doubles (the call every multi-GPU matvec makes on its packed exchange
 * buffer) checked unchanged (a one-rank sum is the
 * identity), then one round of the TREE exchange with this rank as its own
 * partner (ncclSend + ncclRecv in a group, then the add) checked to double
 * every value, destroy.  HMAT_ERR_NCCL / HMAT_ERR_CUDA on failure,
 * HMAT_ERR_INVALID for count < 1. */
hmat_status hmat_nccl_selftest(int device, int64_t count);

/* The communicator H exchanges over (Steps 2-4): *nranks
 * and *rank as NCCL reports them (ncclCommCount / ncclCommUserRank) for the
 * NCCL and TREE exchanges, else the plan's P and rank.  Also reports pending
 * asynchronous exchange errors (HMAT_ERR_NCCL).  HMAT_ERR_INVALID for NULL. */
hmat_status hmat_comm_info(hmat_t H, int* nranks, int* rank);

/* Kernel timing of the steps of PAPER.md:652-663: when enabled, CUDA events
 * bracket every kernel/collective of each matvec on H's stream.  hmat_profile_read() synchronises, returns the
 * accumulated milliseconds and launch counts per phase since the last read
 * (phase 0 = project, 1 = exchange, 2 = expand, 3 = host<->device copies) and
 * resets them.  ms and launches point to HMAT_NUM_PHASES entries.
 * HMAT_ERR_INVALID for NULL arguments. */
#define HMAT_NUM_PHASES 4
hmat_status hmat_profile(hmat_t H, int enable);
hmat_status hmat_profile_read(hmat_t H, double* ms, int64_t* launches);

/* Per-CTA trace (load-balance diagnostics of the balanced work split the paper
 * argues for).  hmat_cta_trace(H, 1) allocates a
 * device buffer; every later project / expand launch on H then records, per CTA
 * b, [start ns, end ns, SM id] (%globaltimer at the CTA's start and at its last
 * warp's exit; end is 0 for a CTA that did not run).  hmat_cta_trace(H, 0) frees
 * it.  hmat_cta_trace_read synchronises H's stream and copies the records of the
 * LAST launch of `kernel` (0 = project, 1 = expand) into out[3 * b + 0..2] for
 * b < min(grid, max_ctas, 8192); *n_ctas = that count.  HMAT_ERR_INVALID for a
 * bad kernel index or when tracing is off. */
hmat_status hmat_cta_trace(hmat_t H, int enable);
hmat_status hmat_cta_trace_read(hmat_t H, int kernel, int64_t* out, int max_ctas, int* n_ctas);

/* Launches of this library's kernels one hmat_matvec(nrhs) performs on this
 * rank (the steps of PAPER.md:652-663 as kernels): per pass of right-hand sides, project + expand, + pack / unpack with
 * standard admissibility and P > 1, + log2 P adds with the TREE exchange, + the
 * mailbox sum on the tensor-core path with the PEER exchange (NCCL's own kernels
 * and memsets not counted), for device x / y (a host y of 4 MB or more adds
 * HMAT_Y_CHUNKS - 1 expand launches per pass: VECTORS above).  -1 for NULL H or
 * nrhs < 1. */
int64_t hmat_launches_per_matvec(hmat_t H, int nrhs);

/* Host-only description of a shard's plan (no GPU needed). */
typedef struct {
  int64_t N, row_begin, row_end;
  int c, W, W_pitch;          /* W_pitch: row pitch (doubles) of panels and z rows  */
  int cross_levels;           /* levels 1..cross_levels go through the exchange     */
  int64_t exchange_rows;      /* targets in the exchange buffer (sum of c^l, l <= cross) */
  int64_t level_rows_offset[64]; /* first exchange row of level l (l = 1..cross)    */
  int Rp, Re, tpr, nstage_p, nstage_e, grid_p, grid_e;
  int64_t smem_p, smem_e;
  int max_nr;                 /* widest SIMT pass of right-hand sides                */
  int dmma;                   /* 1: the FP64 tensor-core path serves >= HMAT_DMMA_MIN (3) rhs */
  /* tensor-core pass layouts, [0] = 16, [1] = 32, [2] = 64, [3] = 8 rhs wide (ok = 0: unused) */
  int dmma_ok[4], dmma_grid_p[4], dmma_grid_e[4], dmma_stages_p[4], dmma_stages_e[4];
  int64_t dmma_smem_p[4], dmma_smem_e[4];
} hmat_plan_info_t;

/* Validates (depth, dim, leaf_size, rank, nranks, rank_id) exactly like
 * hmat_create (same HMAT_ERR_INVALID / _UNSUPPORTED) and describes the plan a
 * B200 (148 SMs) would use: the partition of PAPER.md:434-501 and the packed
 * exchange of Steps 2-4.  The exchange
 * buffer is level-major, then target-major: row (level_rows_offset[l] + t)
 * holds, in columns [q r, (q+1) r), z_{t, s_q} = V_{t,s_q}^T x_{s_q}, summed over
 * all ranks. */
hmat_status hmat_plan_query(int depth, int dim, int leaf_size, int rank, int nranks, int rank_id,
                            hmat_plan_info_t* info);

/* Standard admissibility with nranks > 1: the packed cross-rank exchange of
 * one rank (csrc/std_exchange.h), computed on the host exactly as
 * hmat_create_standard does, for tests without a GPU.  One pass of `cap`
 * right-hand sides exchanges the doubles
 *   [E entries][cap][rank]  z_{t,s} = V_{t,s}^T x_s of every interaction pair
 *                           (levels 2..depth) whose target and source are not
 *                           inside one rank, numbered by (level, target in
 *                           Morton order, slot of the target's list);
 *   [Hn halo leaves][cap][bpad]  x of every leaf whose near field reaches
 *                           another rank, in Morton order,
 * the second part starting at E rank cap rounded up to even; every rank writes
 * what it owns, zeros elsewhere, and the buffer is summed over the ranks.
 * (PAPER.md:606-629 for where the pairs lie; errors as hmat_plan_query.)
 * Tables of THIS rank (filled when the caller's array is non-NULL and its
 * capacity is large enough; the n_* fields always receive the lengths):
 *   src_entry  [node - first local node][M] per level l at src_off[l]: entry of
 *              (local source node, slot of its list), -1 for a pair inside the rank;
 *   unpack     pairs {entry, Zt row * 256 + slot}: entries of this rank's targets,
 *              Zt row = zt_row_offset[l] + target - first local node of level l;
 *   pack       pairs {halo index, local leaf}: this rank's leaves others need;
 *   halo_of    [local leaf][3^dim]: halo index of near-field neighbour e, or -1.
 * H^T (the second part holds [Hp pairs][cap][bpad] products instead of halo x):
 *   Hp         cross near-field pairs (S, T), owner(S) != owner(T), numbered over
 *              leaves S in Morton order, then neighbour e (T = S + eps_e);
 *   tpack      triples {pair, local leaf S, e}: this rank's outgoing pairs, whose
 *              product (D_{S,T})^T x_S it writes;
 *   tadd_leaf / tadd_off / tadd_pair  CSR of this rank's leaves T with incoming
 *              pairs (local leaf, offsets, ascending pair indices). */
typedef struct {
  int64_t E, Hn;
  int bpad, M;
  int64_t src_off[64], zt_row_offset[64];
  int32_t* src_entry; int64_t src_entry_cap, n_src_entry;
  int64_t* unpack;    int64_t unpack_cap, n_unpack;
  int64_t* pack;      int64_t pack_cap, n_pack;
  int32_t* halo_of;   int64_t halo_of_cap, n_halo_of;
  int64_t Hp;
  int64_t* tpack;     int64_t tpack_cap, n_tpack;
  int64_t* tadd_leaf; int64_t tadd_leaf_cap, n_tadd_leaf;
  int64_t* tadd_off;  int64_t tadd_off_cap, n_tadd_off;
  int64_t* tadd_pair; int64_t tadd_pair_cap, n_tadd_pair;
} hmat_std_exchange_t;
hmat_status hmat_std_exchange_query(int depth, int dim, int leaf_size, int rank, int nranks, int rank_id,
                                    hmat_std_exchange_t* q);

#ifdef __cplusplus
}
#endif

#endif /* HMAT_H */
