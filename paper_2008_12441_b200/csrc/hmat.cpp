// hmat.cpp -- the C ABI (include/hmat.h): validation, device memory, the
// per-matvec launch sequence and the optional NCCL exchange.
//
// One hmat_matvec = for each pass of <= 8 right-hand sides:
//   [P>1: zero the exchange buffer]
//   project  (Step 1 + on-chip Step 2)
//   [P>1: sum-allreduce of the packed exchange buffer = Steps 2-4 across GPUs,
//         PAPER.md:746-904]
//   expand   (Step 5, fused with the dense leaf blocks)
#include "hmat.h"

#include <cuda_runtime.h>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comm.h"
#include "std_exchange.h"
#include "kernels.h"
#include "plan.h"

namespace {

thread_local std::string g_err;

hmat_status fail(hmat_status s, const std::string& m) {
  g_err = m;
  return s;
}

hmat_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? HMAT_ERR_NOMEM : HMAT_ERR_CUDA;
}

#define CUDA_TRY(expr)                                   \
  do {                                                   \
    cudaError_t e_ = (expr);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr);  \
  } while (0)

int env_int(const char* name, int def) {
  const char* v = getenv(name);
  if (!v || !*v) return def;
  return atoi(v);
}

hmat::PlanOptions options_from_env(int num_sms) {
  hmat::PlanOptions o;
  o.num_sms = num_sms;
  o.ctas_per_sm = env_int("HMAT_CTAS_PER_SM", 2);
  o.stage_cap_bytes = env_int("HMAT_STAGE_KB", 36) * 1024;
  o.smem_budget = env_int("HMAT_SMEM_KB", 200) * 1024;
  o.max_stages_p = env_int("HMAT_MAX_STAGES_P", env_int("HMAT_MAX_STAGES", o.max_stages_p));
  o.max_stages_e = env_int("HMAT_MAX_STAGES_E", env_int("HMAT_MAX_STAGES", o.max_stages_e));
  o.max_nr = env_int("HMAT_MAX_NR", o.max_nr);
  o.dmma_max_stages_p = env_int("HMAT_DMMA_STAGES_P", o.dmma_max_stages_p);
  o.dmma_off = env_int("HMAT_DMMA_OFF", 0);
  o.dmma_min = env_int("HMAT_DMMA_MIN", 3);
  o.dbg = env_int("HMAT_DEBUG_SKIP", 0);
  o.expand_chunk = env_int("HMAT_EXPAND_CHUNK", -1);
  o.project_dyn = env_int("HMAT_PROJECT_DYN", 1);
  o.project_chunk = env_int("HMAT_PROJECT_CHUNK", 4);
  o.snake = env_int("HMAT_PROJECT_SNAKE", 1);
  o.pdl = env_int("HMAT_PDL", 2);
  o.lpar = env_int("HMAT_PROJECT_LPAR", 1);
  o.early = env_int("HMAT_PROJECT_EARLY", 1);
  o.eshape = env_int("HMAT_EXPAND_SHAPE", 1);
  o.dmma_ileave = env_int("HMAT_DMMA_ILEAVE", 1);
  o.aflush = env_int("HMAT_PROJECT_AFLUSH", 1);
  o.dmma_upol = env_int("HMAT_DMMA_UPOL", 1);
  o.dmma8_ctas = env_int("HMAT_DMMA8_CTAS", 0);
  o.dmma8_nw = env_int("HMAT_DMMA8_NW", o.dmma8_nw);
  o.dmma_pchunk = env_int("HMAT_DMMA_PCHUNK", 32);
  o.dmma_pchunk16 = env_int("HMAT_DMMA_PCHUNK16", 16);
  o.dmma_stages_e_narrow = env_int("HMAT_DMMA_STAGES_E", 0);
  o.dmma8_max_stages = env_int("HMAT_DMMA8_STAGES", o.dmma8_max_stages);
  o.dmma_nw = env_int("HMAT_DMMA_NW", o.dmma_nw);
  o.dmma_narrow = env_int("HMAT_DMMA_NARROW", o.dmma_narrow);
  o.dmma_kc = env_int("HMAT_DMMA_KC", 0);
  o.dmma16_ctas = env_int("HMAT_DMMA16_CTAS", 0);
  o.dmma16_max_stages = env_int("HMAT_DMMA16_STAGES", 0);
  o.dmma_e_ctas = env_int("HMAT_DMMA_E_CTAS", 0);
  return o;
}

hmat_status plan_status(const std::string& msg) {
  if (msg.rfind("unsupported", 0) == 0) return fail(HMAT_ERR_UNSUPPORTED, msg);
  return fail(HMAT_ERR_INVALID, msg);
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int nr_cap(int nr) { return nr <= 1 ? 1 : nr <= 2 ? 2 : nr <= 4 ? 4 : 8; }

cudaError_t configure_all(const hmat::Plan& p) {
  int64_t sp = 0, se = 0;
  for (int li = 0; li < 4 && (1 << li) <= p.max_nr; ++li) {  // layouts that fit
    sp = std::max(sp, p.lay[li].smem_p);
    se = std::max(se, p.lay[li].smem_e);
  }
  return hmat::configure_kernels(sp, se);
}


struct EventPair {
  int phase;
  cudaEvent_t a, b;
};

}  // namespace

struct hmat_s {
  hmat::Plan plan;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double* U = nullptr;
  double* V = nullptr;
  double* D = nullptr;
  double* zloc = nullptr;
  double* zex = nullptr;
  double* part = nullptr;
  int* cnt = nullptr;
  int* sched = nullptr;  // expand's dynamic chunk counters [next, done]
  double* xbuf = nullptr;
  double* ybuf = nullptr;
  size_t xcap = 0, ycap = 0;  // doubles
  // asynchronous host-pointer mode (hmat_set_host_async): double-buffered
  // staging, copies in / out on their own streams, ordered by events
  bool host_async = false;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  double* xb2[2] = {nullptr, nullptr};
  double* yb2[2] = {nullptr, nullptr};
  size_t xc2[2] = {0, 0}, yc2[2] = {0, 0};
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  bool comp_rec[2] = {false, false}, out_rec[2] = {false, false};
  int apar = 0;
  // blocking host-y calls: expand in row chunks, each chunk's y copied out on
  // s_y while the next chunk runs (HMAT_Y_CHUNKS)
  int y_chunks = 4;
  cudaStream_t s_y = nullptr;
  cudaEvent_t ev_y[8] = {};
  hmat::Comm* comm = nullptr;
  // DMMA (many right-hand sides) buffers, allocated on first use
  double* zloc_d = nullptr;
  double* zex_d = nullptr;
  double* part_d = nullptr;
  double* accbuf_d = nullptr;  // chunked tensor-core project: running sums between chunks
  int* cnt_d = nullptr;
  double* Dt = nullptr;  // D^T, built on the first transposed product
  // standard admissibility with P > 1: the packed cross-rank exchange (std_exchange.h)
  hmat::StdExchange* sx = nullptr;
  int32_t* xent_d = nullptr;
  int64_t* unpack_d = nullptr;
  int64_t* pack_d = nullptr;
  int32_t* halo_of_d = nullptr;
  int64_t* tpack_d = nullptr;   // H^T, P > 1: outgoing cross near-field pairs
  int64_t* tadd_leaf_d = nullptr;
  int64_t* tadd_off_d = nullptr;
  int64_t* tadd_pair_d = nullptr;
  bool external = false;  // P > 1 with a caller-provided exchange (split-phase API)
  // HMAT_EXCHANGE_TREE: recursive doubling over NCCL point-to-point; scratch buffer
  bool tree = false;
  double* xtmp = nullptr;
  size_t xtmp_cap = 0;
  // in-kernel peer exchange (HMAT_EXCHANGE_PEER): this rank's mailbox
  // [2 parities][P slots][mb] doubles + [2][P] uint64 flags, and the device
  // table of every rank's mailbox address (peer memory)
  bool peer = false, connected = false;
  double* mbox = nullptr;
  double** mbox_dev = nullptr;
  unsigned int* done = nullptr;
  // error word of the bounded flag waits (peer.cuh): host-mapped, written by a
  // kernel whose wait timed out, read (and cleared) by the next call
  unsigned int* err_host = nullptr;
  unsigned int* err_dev = nullptr;
  int64_t peer_timeout_ns = 0;
  int64_t mb = 0;
  uint64_t epoch = 0;
  std::vector<void*> opened;  // IPC mappings to close
  int zt_cap = 1;         // rhs width of the z-buffer layout last written (zeroed at create)
  int zt_nb_d = 0;        // tensor-core pass width of the DMMA z-buffer layout last written (0: never)
  bool prof = false;
  // per-CTA trace of the last project / expand launch (hmat_cta_trace)
  unsigned long long* trace = nullptr;
  int trace_n[2] = {0, 0};
  std::vector<EventPair> ev;
  std::vector<cudaEvent_t> pool;
  double ms[HMAT_NUM_PHASES] = {};
  int64_t nl[HMAT_NUM_PHASES] = {};
};

namespace {

void release(hmat_s* H) {
  if (!H) return;
  cudaSetDevice(H->device);
  if (H->stream) cudaStreamSynchronize(H->stream);
  cudaFree(H->trace);
  cudaFree(H->xtmp);
  cudaFree(H->U);
  cudaFree(H->V);
  cudaFree(H->D);
  cudaFree(H->zloc);
  cudaFree(H->zex);
  cudaFree(H->part);
  cudaFree(H->cnt);
  cudaFree(H->sched);
  cudaFree(H->xbuf);
  cudaFree(H->ybuf);
  for (int i = 0; i < 2; ++i) {
    if (H->s_in) cudaStreamSynchronize(H->s_in);
    if (H->s_out) cudaStreamSynchronize(H->s_out);
    cudaFree(H->xb2[i]);
    cudaFree(H->yb2[i]);
    if (H->ev_in[i]) cudaEventDestroy(H->ev_in[i]);
    if (H->ev_comp[i]) cudaEventDestroy(H->ev_comp[i]);
    if (H->ev_out[i]) cudaEventDestroy(H->ev_out[i]);
  }
  if (H->s_in) cudaStreamDestroy(H->s_in);
  if (H->s_out) cudaStreamDestroy(H->s_out);
  if (H->s_y) {
    cudaStreamSynchronize(H->s_y);
    cudaStreamDestroy(H->s_y);
  }
  for (cudaEvent_t ev : H->ev_y)
    if (ev) cudaEventDestroy(ev);
  cudaFree(H->zloc_d);
  cudaFree(H->zex_d);
  cudaFree(H->part_d);
  cudaFree(H->accbuf_d);
  cudaFree(H->cnt_d);
  cudaFree(H->Dt);
  cudaFree(H->xent_d);
  cudaFree(H->unpack_d);
  cudaFree(H->pack_d);
  cudaFree(H->halo_of_d);
  cudaFree(H->tpack_d);
  cudaFree(H->tadd_leaf_d);
  cudaFree(H->tadd_off_d);
  cudaFree(H->tadd_pair_d);
  delete H->sx;
  for (void* q : H->opened) cudaIpcCloseMemHandle(q);
  cudaFree(H->mbox);
  cudaFree(H->mbox_dev);
  cudaFree(H->done);
  if (H->err_host) cudaFreeHost(H->err_host);
  for (auto& e : H->ev) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : H->pool) cudaEventDestroy(e);
  hmat::comm_destroy(H->comm);
  if (H->own_stream && H->stream) cudaStreamDestroy(H->stream);
  delete H;
}

hmat_status validate_dist(const hmat_dist_t* dist, int* P, int* rank) {
  *P = 1;
  *rank = 0;
  if (!dist) return HMAT_OK;
  *P = dist->nranks;
  *rank = dist->rank;
  if (dist->exchange < HMAT_EXCHANGE_NCCL || dist->exchange > HMAT_EXCHANGE_TREE)
    return fail(HMAT_ERR_INVALID, "exchange must be HMAT_EXCHANGE_NCCL, _EXTERNAL, _PEER or _TREE");
  if (dist->nranks > 1 && (dist->exchange == HMAT_EXCHANGE_NCCL || dist->exchange == HMAT_EXCHANGE_TREE) &&
      !dist->nccl_unique_id)
    return fail(HMAT_ERR_INVALID, "nccl_unique_id is NULL with nranks > 1 and an NCCL exchange");
  if (dist->device < 0) return fail(HMAT_ERR_INVALID, "device ordinal must be >= 0");
  return HMAT_OK;
}

hmat_status create_common(int depth, int dim, int leaf, int rank, const hmat_dist_t* dist, hmat_t* out,
                          int adm = 0) {
  if (!out) return fail(HMAT_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int P, shard;
  hmat_status st = validate_dist(dist, &P, &shard);
  if (st != HMAT_OK) return st;
  hmat::Plan plan;
  const bool peer = dist && dist->nranks > 1 && dist->exchange == HMAT_EXCHANGE_PEER;
  hmat::PlanOptions opt0 = options_from_env(148);
  opt0.adm = adm;
  opt0.peer = peer;
  std::string msg = hmat::plan_build(depth, dim, leaf, rank, P, shard, opt0, &plan);
  if (!msg.empty()) return plan_status(msg);

  // ---- device work starts here ----
  int device = 0;
  if (dist) {
    device = dist->device;
    CUDA_TRY(cudaSetDevice(device));
  } else {
    CUDA_TRY(cudaGetDevice(&device));
  }
  int sms = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  hmat::PlanOptions opt = options_from_env(sms);
  opt.adm = adm;
  opt.peer = peer;
  msg = hmat::plan_build(depth, dim, leaf, rank, P, shard, opt, &plan);
  if (!msg.empty()) return plan_status(msg);

  hmat_s* H = new hmat_s;
  H->plan = plan;
  H->device = device;
  auto bail = [&](hmat_status s) {
    release(H);
    return s;
  };
  if (dist && dist->cuda_stream) {
    H->stream = static_cast<cudaStream_t>(dist->cuda_stream);
  } else {
    // blocking stream: ordered with work the caller put on the legacy default stream
    cudaError_t e = cudaStreamCreateWithFlags(&H->stream, cudaStreamDefault);
    if (e != cudaSuccess) return bail(cuda_fail(e, "cudaStreamCreate"));
    H->own_stream = true;
  }
  const hmat::Plan& p = H->plan;
  if (p.adm && p.P > 1) {  // the standard-admissibility exchange plan (host enumeration)
    H->sx = new hmat::StdExchange;
    std::string m = hmat::std_exchange_build(p, H->sx);
    if (!m.empty()) return bail(plan_status(m));
  }
  auto alloc = [&](void** ptr, size_t bytes, const char* what) -> cudaError_t {
    if (bytes == 0) bytes = 256;
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess) g_err = std::string("cudaMalloc(") + what + ")";
    return e;
  };
  cudaError_t e = cudaSuccess;
  const size_t panels = size_t(p.L) * size_t(p.panel_stride) * sizeof(double);
  const size_t zrow = size_t(p.Wp) * hmat::kMaxNR * sizeof(double);
  if ((e = alloc(reinterpret_cast<void**>(&H->U), panels, "U")) ||
      (e = alloc(reinterpret_cast<void**>(&H->V), panels, "V")) ||
      (e = alloc(reinterpret_cast<void**>(&H->D), size_t(p.nd) * p.d_stride * sizeof(double), "D")) ||
      (e = alloc(reinterpret_cast<void**>(&H->zloc), size_t(p.z_local_rows) * zrow, "z")) ||
      (e = alloc(reinterpret_cast<void**>(&H->zex),
                 H->sx ? size_t(H->sx->doubles_max(hmat::kMaxNR, p.r)) * sizeof(double) : size_t(p.z_exch_rows) * zrow,
                 "exchange")) ||
      (e = alloc(reinterpret_cast<void**>(&H->part), size_t(p.grid_p_max) * p.L * 2 * zrow, "partials")) ||
      (e = alloc(reinterpret_cast<void**>(&H->cnt), size_t(p.grid_p_max) * p.L * sizeof(int) + 256, "tickets")) ||
      (e = alloc(reinterpret_cast<void**>(&H->sched), 256, "schedule counters"))) {
    std::string what = g_err;
    return bail(cuda_fail(e, what.c_str()));
  }
  if ((e = cudaMemsetAsync(H->cnt, 0, size_t(p.grid_p_max) * p.L * sizeof(int) + 256, H->stream)) ||
      (e = cudaMemsetAsync(H->sched, 0, 256, H->stream)) ||
      (e = cudaMemsetAsync(H->U, 0, panels ? panels : 256, H->stream)) ||
      (e = cudaMemsetAsync(H->V, 0, panels ? panels : 256, H->stream)) ||
      (e = cudaMemsetAsync(H->D, 0, size_t(p.nd) * p.d_stride * sizeof(double), H->stream)) ||
      // z rows: padding columns (odd W) are multiplied by zero padding of U, so keep them finite
      (e = cudaMemsetAsync(H->zloc, 0, std::max<size_t>(256, size_t(p.z_local_rows) * zrow), H->stream)) ||
      (e = cudaMemsetAsync(H->zex, 0, std::max<size_t>(256, size_t(p.z_exch_rows) * zrow), H->stream)) ||
      (e = configure_all(p)) || (p.dmma_ok && (e = hmat::configure_dmma(64, p.dl[2].dsmem_p, p.dl[2].dsmem_e))) ||
      (p.dmma_ok && p.dl[1].ok && (e = hmat::configure_dmma(32, p.dl[1].dsmem_p, p.dl[1].dsmem_e))) ||
      (p.dmma_ok && p.dl[0].ok && (e = hmat::configure_dmma(16, p.dl[0].dsmem_p, p.dl[0].dsmem_e))) ||
      (p.dmma_ok && p.dl[3].ok && (e = hmat::configure_dmma(8, p.dl[3].dsmem_p, p.dl[3].dsmem_e))) ||
      (e = cudaStreamSynchronize(H->stream)))
    return bail(cuda_fail(e, "initialising device buffers"));
  H->y_chunks = std::max(1, std::min(8, env_int("HMAT_Y_CHUNKS", 4)));
  H->external = p.P > 1 && dist->exchange == HMAT_EXCHANGE_EXTERNAL;
  H->tree = p.P > 1 && dist->exchange == HMAT_EXCHANGE_TREE;
  H->peer = peer;
  if (peer) {
    // one slot holds the widest pass's exchange levels (SIMT: kMaxNR rhs; tensor-core: 64)
    H->mb = (p.z_exch_rows * p.Wp * (p.dmma_ok ? std::max(hmat::kMaxNR, hmat::kDmmaNB) : hmat::kMaxNR) + 15) / 16 * 16;
    const size_t mbytes = (size_t(2) * p.P * H->mb + size_t(2) * p.P) * sizeof(double);
    if ((e = cudaMalloc(reinterpret_cast<void**>(&H->mbox), mbytes)) ||
        (e = cudaMalloc(reinterpret_cast<void**>(&H->mbox_dev), size_t(p.P) * sizeof(double*))) ||
        (e = cudaMalloc(reinterpret_cast<void**>(&H->done), 256)) ||
        (e = cudaMemset(H->mbox, 0, mbytes)) || (e = cudaMemset(H->mbox_dev, 0, size_t(p.P) * sizeof(double*))) ||
        (e = cudaMemset(H->done, 0, 256)) ||
        (e = cudaHostAlloc(reinterpret_cast<void**>(&H->err_host), 64, cudaHostAllocMapped | cudaHostAllocPortable)))
      return bail(cuda_fail(e, "allocating the peer mailbox"));
    *reinterpret_cast<volatile unsigned int*>(H->err_host) = 0u;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&H->err_dev), H->err_host, 0)))
      return bail(cuda_fail(e, "mapping the peer error word"));
    H->peer_timeout_ns = int64_t(std::max(1, env_int("HMAT_PEER_TIMEOUT_MS", 10000))) * 1000000;
  }
  if (H->sx) {  // device copies of the exchange tables
    const hmat::StdExchange& X = *H->sx;
    auto up = [&](void** dst, const void* src, size_t bytes) -> cudaError_t {
      cudaError_t e2 = cudaMalloc(dst, bytes ? bytes : 256);
      if (e2 == cudaSuccess && bytes) e2 = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
      return e2;
    };
    if ((e = up(reinterpret_cast<void**>(&H->xent_d), X.src_entry.data(), X.src_entry.size() * sizeof(int32_t))) ||
        (e = up(reinterpret_cast<void**>(&H->unpack_d), X.unpack.data(), X.unpack.size() * sizeof(int64_t))) ||
        (e = up(reinterpret_cast<void**>(&H->pack_d), X.pack.data(), X.pack.size() * sizeof(int64_t))) ||
        (e = up(reinterpret_cast<void**>(&H->halo_of_d), X.halo_of.data(), X.halo_of.size() * sizeof(int32_t))) ||
        (e = up(reinterpret_cast<void**>(&H->tpack_d), X.tpack.data(), X.tpack.size() * sizeof(int64_t))) ||
        (e = up(reinterpret_cast<void**>(&H->tadd_leaf_d), X.tadd_leaf.data(), X.tadd_leaf.size() * sizeof(int64_t))) ||
        (e = up(reinterpret_cast<void**>(&H->tadd_off_d), X.tadd_off.data(), X.tadd_off.size() * sizeof(int64_t))) ||
        (e = up(reinterpret_cast<void**>(&H->tadd_pair_d), X.tadd_pair.data(), X.tadd_pair.size() * sizeof(int64_t))))
      return bail(cuda_fail(e, "uploading the standard-admissibility exchange tables"));
  }
  if (p.adm) {  // interaction-list slot tables for the project kernel's scatter
    int16_t code[3][8][hmat::kStdMaxSlots], slot[3][8][hmat::kStdMaxCodes];  // ~20 KB, per call
    hmat::std_slot_tables(code, slot);
    if ((e = hmat::init_std_tables(&code[0][0][0], &slot[0][0][0])) != cudaSuccess ||
        (p.dmma_ok && (e = hmat::init_std_tables_dmma(&code[0][0][0], &slot[0][0][0])) != cudaSuccess))
      return bail(cuda_fail(e, "init_std_tables"));
  }
  if (p.P > 1 && !H->external && !peer) {
    std::string m = hmat::comm_create(dist->nccl_unique_id, p.P, p.rank, &H->comm);
    if (!m.empty()) return bail(fail(HMAT_ERR_NCCL, m));
  }
  *out = H;
  return HMAT_OK;
}

cudaEvent_t take_event(hmat_s* H) {
  if (!H->pool.empty()) {
    cudaEvent_t e = H->pool.back();
    H->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(hmat_s* H, int phase, EventPair* ep) {
  if (!H->prof) return;
  ep->phase = phase;
  ep->a = take_event(H);
  ep->b = take_event(H);
  cudaEventRecord(ep->a, H->stream);
}

void prof_end(hmat_s* H, EventPair* ep) {
  if (!H->prof) return;
  cudaEventRecord(ep->b, H->stream);
  H->ev.push_back(*ep);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
// A tiled fp64 map of `rank` dims (innermost first), strides in bytes for
// dims 1..rank-1, zero fill out of bounds, no swizzle.
hmat_status encode_map(CUtensorMap* m, int rank, const void* base, const uint64_t* dims, const uint64_t* strides,
                       const uint32_t* box) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return fail(HMAT_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  cuuint64_t gd[3], gs[2];
  cuuint32_t bx[3], es[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    if (i + 1 < rank) gs[i] = strides[i];
  }
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), gd, gs, bx, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(HMAT_ERR_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string(r) + ")");
  return HMAT_OK;
}

bool use_dmma(const hmat::Plan& p, int nrhs) {
  if (!p.dmma_ok || p.dmma_off) return false;
  // standard admissibility: one SIMT pass serves up to 4 rhs faster than the
  // sliced tensor-core project (s2, 4 rhs: 9.9 vs 18.4 ms; 8 rhs: 19.9 vs 18.4)
  return nrhs >= (p.adm ? std::max(p.dmma_min, 5) : p.dmma_min);
}

hmat_status ensure_dmma(hmat_s* H) {
  if (H->cnt_d) return HMAT_OK;
  const hmat::Plan& p = H->plan;
  const size_t zrow = size_t(p.W) * hmat::kDmmaNB * sizeof(double);
  const size_t tickets = size_t(p.dgrid_p_max) * p.L * std::max(1, p.nslice) * sizeof(int) + 256;  // per slice
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&H->zloc_d), std::max<size_t>(256, size_t(p.z_local_rows) * zrow)));
  // exchange levels, or (standard admissibility, P > 1) the packed cross-rank buffer of a 64-wide pass
  const size_t zex_bytes = H->sx ? size_t(H->sx->doubles_max(hmat::kDmmaNB, p.r)) * sizeof(double)
                                 : size_t(p.z_exch_rows) * zrow;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&H->zex_d), std::max<size_t>(256, zex_bytes)));
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&H->part_d),
                      std::max<size_t>(256, size_t(p.dgrid_p_max) * p.L * 2 * p.Wp * hmat::kDmmaNB * sizeof(double))));
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&H->cnt_d), tickets));
  // chunked project passes (<= 16 wide): per CTA and level one W x 16 tile of sums
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&H->accbuf_d),
                      std::max<size_t>(256, size_t(p.dgrid_p_max) * p.L * p.W * 16 * sizeof(double))));
  CUDA_TRY(cudaMemsetAsync(H->cnt_d, 0, tickets, H->stream));
  return HMAT_OK;
}

hmat_status ensure_buf(double** buf, size_t* cap, size_t n) {
  if (*cap >= n) return HMAT_OK;
  cudaFree(*buf);
  *buf = nullptr;
  *cap = 0;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(buf), n * sizeof(double)));
  *cap = n;
  return HMAT_OK;
}

// Asynchronous failures of earlier work on H: a peer flag wait that timed out
// (the kernels' error word, cleared once reported) and NCCL's asynchronous
// communicator errors (ncclCommGetAsyncError).  Both map to HMAT_ERR_NCCL.
hmat_status check_async(hmat_s* H) {
  if (H->err_host) {
    volatile unsigned int* w = reinterpret_cast<volatile unsigned int*>(H->err_host);
    const unsigned int v = *w;
    if (v) {
      *w = 0u;
      return fail(HMAT_ERR_NCCL, "peer exchange: rank " + std::to_string((v >> 16) & 0x7fffu) +
                                     "'s flag of pass " + std::to_string(v & 0xffffu) + " (mod 2^16) not raised within " +
                                     std::to_string(H->peer_timeout_ns / 1000000) +
                                     " ms (late or missing peer; that product's y is invalid)");
    }
  }
  if (H->comm) {
    std::string m = hmat::comm_async_error(H->comm);
    if (!m.empty()) return fail(HMAT_ERR_NCCL, m);
  }
  return HMAT_OK;
}

}  // namespace

extern "C" {

hmat_status hmat_create_standard_uninit(int depth, int dim, int leaf_size, int rank, const hmat_dist_t* dist,
                                       hmat_t* out) {
  return create_common(depth, dim, leaf_size, rank, dist, out, 1);
}

hmat_status hmat_create_uninit(int depth, int dim, int leaf_size, int rank, const hmat_dist_t* dist, hmat_t* out) {
  return create_common(depth, dim, leaf_size, rank, dist, out);
}

}  // extern "C"

namespace {

hmat_status create_from_panels(int depth, int dim, int leaf_size, int rank, const double* const* U,
                               const double* const* V, const double* D, const hmat_dist_t* dist, hmat_t* out,
                               int adm) {
  if (!out) return fail(HMAT_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (depth > 0 && (!U || !V)) return fail(HMAT_ERR_INVALID, "U or V is NULL");
  if (!D) return fail(HMAT_ERR_INVALID, "D is NULL");
  for (int l = 0; depth > 0 && l < depth && l < hmat::kMaxLevels; ++l)
    if (!U[l] || !V[l]) return fail(HMAT_ERR_INVALID, "a U or V panel pointer is NULL");
  hmat_t H = nullptr;
  hmat_status st = create_common(depth, dim, leaf_size, rank, dist, &H, adm);
  if (st != HMAT_OK) return st;
  const hmat::Plan& p = H->plan;
  cudaError_t e = cudaSuccess;
  for (int l = 1; l <= p.L && e == cudaSuccess; ++l) {
    e = cudaMemcpy2DAsync(H->U + (l - 1) * p.panel_stride, p.Wp * sizeof(double), U[l - 1], p.W * sizeof(double),
                          p.W * sizeof(double), p.N_loc, cudaMemcpyDefault, H->stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(H->V + (l - 1) * p.panel_stride, p.Wp * sizeof(double), V[l - 1], p.W * sizeof(double),
                            p.W * sizeof(double), p.N_loc, cudaMemcpyDefault, H->stream);
  }
  if (e == cudaSuccess)
    for (int k = 0; k < p.nd && e == cudaSuccess; ++k)  // canonical N_loc x (nd b) -> nd panels
      e = cudaMemcpy2DAsync(H->D + k * p.d_stride, p.Dp * sizeof(double), D + k * p.b,
                            size_t(p.nd) * p.b * sizeof(double), p.b * sizeof(double), p.N_loc, cudaMemcpyDefault,
                            H->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(H->stream);
  if (e != cudaSuccess) {
    hmat_status s = cuda_fail(e, "copying panels");
    release(H);
    return s;
  }
  *out = H;
  return HMAT_OK;
}

}  // namespace

extern "C" {

hmat_status hmat_create(int depth, int dim, int leaf_size, int rank, const double* const* U, const double* const* V,
                        const double* D, const hmat_dist_t* dist, hmat_t* out) {
  return create_from_panels(depth, dim, leaf_size, rank, U, V, D, dist, out, 0);
}

hmat_status hmat_create_standard(int depth, int dim, int leaf_size, int rank, const double* const* U,
                                 const double* const* V, const double* Dn, const hmat_dist_t* dist, hmat_t* out) {
  return create_from_panels(depth, dim, leaf_size, rank, U, V, Dn, dist, out, 1);
}

hmat_status hmat_panel(hmat_t H, int kind, int level, double** ptr, int64_t* rows, int64_t* cols, int64_t* ld) {
  if (!H || !ptr) return fail(HMAT_ERR_INVALID, "NULL argument");
  const hmat::Plan& p = H->plan;
  if (kind == 0 || kind == 1) {
    if (level < 1 || level > p.L) return fail(HMAT_ERR_INVALID, "level out of range [1, depth]");
    *ptr = (kind == 0 ? H->U : H->V) + (level - 1) * p.panel_stride;
    if (cols) *cols = p.W;
    if (ld) *ld = p.Wp;
  } else if (kind == 2) {
    if (level < 0 || level >= p.nd) return fail(HMAT_ERR_INVALID, "dense panel index out of range");
    *ptr = H->D + level * p.d_stride;
    if (cols) *cols = p.b;
    if (ld) *ld = p.Dp;
  } else {
    return fail(HMAT_ERR_INVALID, "kind must be 0 (U), 1 (V) or 2 (D)");
  }
  if (rows) *rows = p.N_loc;
  return HMAT_OK;
}

}  // extern "C"

namespace {

// D^T panel for the transposed product, built on first use (one-time kernel).
hmat_status ensure_dt(hmat_s* H) {
  if (H->Dt) return HMAT_OK;
  const hmat::Plan& p = H->plan;
  const size_t bytes = size_t(p.nd) * p.d_stride * sizeof(double);
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&H->Dt), bytes));
  CUDA_TRY(cudaMemsetAsync(H->Dt, 0, bytes, H->stream));
  if (p.adm)  // standard admissibility: nd near-field panels of this rank's leaves
    CUDA_TRY(hmat::launch_transpose_near_field(H->D, H->Dt, p.N_loc / p.b, p.row0 / p.b, p.d, p.L, p.b, p.Dp,
                                               p.d_stride, p.nd, H->stream));
  else
    CUDA_TRY(hmat::launch_transpose_leaf_blocks(H->D, H->Dt, p.N_loc / p.b, p.b, p.Dp, H->stream));
  return HMAT_OK;
}

constexpr int kTraceCap = 8192;  // CTAs recorded per kernel

enum { kPhaseProject = 1, kPhaseExchange = 2, kPhaseExpand = 4, kPhaseAll = 7 };

// y = alpha op(H) x + beta y restricted to the selected parts (the whole path).
// `phases` selects project / exchange / expand (split-phase API: one pass only).
hmat_status run(hmat_t H, int trans, double alpha, const double* x, double beta, double* y, int nrhs,
                uint64_t level_mask, int dense, int phases = kPhaseAll, double* exch_out = nullptr,
                const double* exch_in = nullptr) {
  if (!H) return fail(HMAT_ERR_INVALID, "H is NULL");
  if (!x || (!y && (phases & kPhaseExpand))) return fail(HMAT_ERR_INVALID, "x or y is NULL");
  if (nrhs < 1) return fail(HMAT_ERR_INVALID, "nrhs must be >= 1");
  if (trans != 0 && trans != 1) return fail(HMAT_ERR_INVALID, "trans must be 0 (H) or 1 (H^T)");
  if (y && static_cast<const void*>(x) == static_cast<const void*>(y))
    return fail(HMAT_ERR_INVALID, "x and y alias");
  const hmat::Plan& p = H->plan;
  CUDA_TRY(cudaSetDevice(H->device));
  {
    hmat_status sa = check_async(H);
    if (sa != HMAT_OK) return sa;
  }
  if (trans) {
    hmat_status st = ensure_dt(H);
    if (st != HMAT_OK) return st;
  }
  const int64_t n = p.N_loc;
  const bool x_dev = is_device_ptr(x), y_dev = y ? is_device_ptr(y) : true;
  if (phases != kPhaseAll) {
    const int width = use_dmma(p, nrhs) ? hmat::kDmmaNB : p.max_nr;
    if (nrhs > width) return fail(HMAT_ERR_INVALID, "split-phase calls take at most one pass of right-hand sides");
    if (!x_dev || !y_dev) return fail(HMAT_ERR_INVALID, "split-phase calls need device x and y");
  } else if (p.P > 1 && H->external) {
    return fail(HMAT_ERR_UNSUPPORTED, "external exchange: use hmat_project / hmat_expand");
  }
  if (H->peer && !H->connected) return fail(HMAT_ERR_INVALID, "peer exchange: mailboxes not connected");
  const bool host_io = !x_dev || !y_dev;
  if (p.L < 64) level_mask &= (p.L == 0 ? 0ull : (~0ull >> (64 - p.L)));
  if (p.adm) level_mask &= ~1ull;  // standard admissibility: no admissible pair at level 1

  EventPair ep{};
  // ---- asynchronous host-pointer mode: x in on s_in, y out on s_out, the
  //      kernels on H's stream, staging buffers alternating between calls so
  //      call k's copies overlap calls k-1 / k+1's kernels
  const bool async_io = host_io && H->host_async && phases == kPhaseAll;
  const int par = H->apar;
  if (async_io) {
    H->apar ^= 1;
    if (!H->s_in) {
      CUDA_TRY(cudaStreamCreateWithFlags(&H->s_in, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamCreateWithFlags(&H->s_out, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        CUDA_TRY(cudaEventCreateWithFlags(&H->ev_in[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&H->ev_comp[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&H->ev_out[i], cudaEventDisableTiming));
      }
    }
    // x staging free once call k-2's kernels are done; y staging once its copy
    // out is done -- the kernels wait for that (below), the copy in only when it
    // writes y staging too (beta != 0), so x(k) streams in while y(k-2) streams out
    if (H->comp_rec[par]) CUDA_TRY(cudaStreamWaitEvent(H->s_in, H->ev_comp[par], 0));
    if (H->out_rec[par] && beta != 0.0 && !y_dev) CUDA_TRY(cudaStreamWaitEvent(H->s_in, H->ev_out[par], 0));
  }
  cudaStream_t s_copy_in = async_io ? H->s_in : H->stream;
  // ---- x: stage when it is host memory, misaligned, or its last column would
  //      be over-read by the 16-byte-granular bulk copies
  const double* xd = x;
  int64_t ldx = n;
  if (async_io && !x_dev) {
    const int64_t lds = n + (n & 1);
    hmat_status st = ensure_buf(&H->xb2[par], &H->xc2[par], size_t(lds) * nrhs + 2);
    if (st != HMAT_OK) return st;
    CUDA_TRY(cudaMemcpy2DAsync(H->xb2[par], lds * sizeof(double), x, n * sizeof(double), n * sizeof(double), nrhs,
                               cudaMemcpyDefault, s_copy_in));
    xd = H->xb2[par];
    ldx = lds;
  } else if (!x_dev || (reinterpret_cast<uintptr_t>(x) & 15) || ((n * nrhs) & 1)) {
    const int64_t lds = n + (n & 1);
    hmat_status st = ensure_buf(&H->xbuf, &H->xcap, size_t(lds) * nrhs + 2);
    if (st != HMAT_OK) return st;
    prof_begin(H, 3, &ep);
    CUDA_TRY(cudaMemcpy2DAsync(H->xbuf, lds * sizeof(double), x, n * sizeof(double), n * sizeof(double), nrhs,
                               cudaMemcpyDefault, H->stream));
    prof_end(H, &ep);
    xd = H->xbuf;
    ldx = lds;
  }
  double* yd = y;
  if (!y_dev) {
    hmat_status st = async_io ? ensure_buf(&H->yb2[par], &H->yc2[par], size_t(n) * nrhs)
                              : ensure_buf(&H->ybuf, &H->ycap, size_t(n) * nrhs);
    if (st != HMAT_OK) return st;
    yd = async_io ? H->yb2[par] : H->ybuf;
    if (beta != 0.0) {  // y is an input too
      prof_begin(H, 3, &ep);
      CUDA_TRY(cudaMemcpyAsync(yd, y, size_t(n) * nrhs * sizeof(double), cudaMemcpyDefault, s_copy_in));
      prof_end(H, &ep);
    }
  }
  if (async_io) {  // the kernels wait for this call's inputs and for y staging to be free
    CUDA_TRY(cudaEventRecord(H->ev_in[par], H->s_in));
    CUDA_TRY(cudaStreamWaitEvent(H->stream, H->ev_in[par], 0));
    if (H->out_rec[par] && !y_dev) CUDA_TRY(cudaStreamWaitEvent(H->stream, H->ev_out[par], 0));
  }

  hmat::StreamArgs a;
  memset(&a, 0, sizeof a);
  // H^T has H's block structure with U and V exchanged and D_k -> D_k^T
  // (the source-major V panel is the target-major panel of H^T and vice versa)
  a.U = trans ? H->V : H->U;
  a.V = trans ? H->U : H->V;
  a.D = trans ? H->Dt : H->D;
  a.alpha = alpha;
  a.beta = beta;
  a.panel_stride = p.panel_stride;
  a.ldx = ldx;
  a.ldy = n;
  a.L = p.L;
  a.d = p.d;
  a.adm = p.adm;
  a.nd = p.nd;
  a.d_stride = p.d_stride;
  a.c = p.c;
  a.r = p.r;
  a.W = p.W;
  a.Wp = p.Wp;
  a.Dp = p.Dp;
  a.b = p.b;
  a.N_loc = n;
  a.row0 = p.row0;
  a.level_mask = level_mask;
  a.dense = dense ? 1 : 0;
  a.Rp = p.Rp;
  a.stages_p = p.stages_p;
  a.part = H->part;
  a.cnt = H->cnt;
  a.Re = p.Re;
  a.ndc = p.ndc;
  a.dc = p.dc;
  a.dgs = p.dgs;
  if (p.ndc > 1 && !p.adm) {  // the dense block's column-chunk boxes [Re][dc]
    const uint64_t dims[2] = {uint64_t(p.Dp), uint64_t(p.N_loc)};
    const uint64_t strides[1] = {uint64_t(p.Dp) * 8};
    const uint32_t box[2] = {uint32_t(p.dc), uint32_t(p.Re)};
    hmat_status st3 = encode_map(&a.tm_dse, 2, a.D, dims, strides, box);
    if (st3 != HMAT_OK) return st3;
  }
  a.sched = H->sched;
  a.tpr = p.tpr;
  a.items_e = p.items_e;
  a.xs_p = p.xs_p;
  a.xs_e = p.xs_e;
  a.cross = p.cross;
  a.P = p.P;
  a.rank = p.rank;
  a.peer = H->peer ? 1 : 0;
  a.mbox = H->mbox_dev;
  a.mb = H->mb;
  a.done = H->done;
  a.err = H->err_dev;
  a.peer_timeout_ns = H->peer_timeout_ns;
  a.zex_base = H->zex;
  a.dbg = p.dbg;
  a.snake = p.snake;
  a.early = p.early;
  a.eshape = p.eshape;
  a.dmma_ileave = p.dmma_ileave;
  a.aflush = p.aflush;
  a.dmma_upol = p.dmma_upol;
  // PDL (expand's launch and prologue overlap project's tail) for whole products;
  // off while the per-kernel profiler brackets the kernels with events
  // and the CTA trace (its memsets sit between the kernels)
  a.pdl = p.pdl && !H->prof && !H->trace && phases == kPhaseAll;
  // project as a programmatic dependent of whatever kernel precedes it (it waits
  // for that kernel's completion before any global access): one GPU, no memset
  // or event wait of this call in between
  a.pdl_p = a.pdl && p.pdl >= 2 && p.P == 1 && !async_io ? 1 : 0;

  // A blocking call with y in host memory: the expand runs in row chunks of
  // whole leaves and each chunk's rows of y are copied out (on s_y) while the
  // next chunk computes, so only the last chunk's copy follows the kernels.
  // (Not with the standard structure's P > 1 exchange -- H^T adds to y after the
  // expand -- nor under the per-kernel profiler or the peer exchange.)
  // (Also in the streaming mode: there the copies go to s_out, and the last
  // product's copy-out -- the pipeline's drain -- overlaps its own expand.)
  // Only where the copy is worth the extra launches: from 4 MB of y (c1's 32 KB
  // took 2.4x longer per call in 4 launches).
  const bool y_big = size_t(n) * size_t(nrhs) * sizeof(double) >= (size_t(4) << 20);
  const int ychunks =
      (!y_dev && y_big && phases == kPhaseAll && !H->peer && !H->sx && !H->prof) ? H->y_chunks : 1;
  bool y_split = false;
  auto expand_rows = [&](auto&& launch, int64_t item_rows, bool dmma, int c0, int nr) -> cudaError_t {
    if (ychunks <= 1) return launch();
    cudaError_t e;
    cudaStream_t s_copy = async_io ? H->s_out : H->s_y;
    if (!async_io && !H->s_y) {
      if ((e = cudaStreamCreateWithFlags(&H->s_y, cudaStreamNonBlocking))) return e;
      s_copy = H->s_y;
    }
    if (!H->ev_y[0])
      for (cudaEvent_t& ev : H->ev_y)
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))) return e;
    const int64_t units = n / p.b, per = (units + ychunks - 1) / ychunks;  // leaves (b is a multiple of item_rows)
    int k = 0;
    for (int64_t u0 = 0; u0 < units; u0 += per, ++k) {
      const int64_t r0 = u0 * p.b, r1 = std::min(units, u0 + per) * p.b;
      a.item0 = r0 / item_rows;
      if (dmma)
        a.e_items = (r1 - r0) / item_rows;
      else
        a.items_e = (r1 - r0) / item_rows;
      if ((e = launch())) return e;
      if ((e = cudaEventRecord(H->ev_y[k], H->stream)) || (e = cudaStreamWaitEvent(s_copy, H->ev_y[k], 0)) ||
          (e = cudaMemcpy2DAsync(y + int64_t(c0) * n + r0, size_t(n) * sizeof(double), yd + int64_t(c0) * n + r0,
                                 size_t(n) * sizeof(double), size_t(r1 - r0) * sizeof(double), size_t(nr),
                                 cudaMemcpyDeviceToHost, s_copy)))
        return e;
    }
    a.item0 = 0;
    a.e_items = 0;
    a.items_e = p.items_e;
    y_split = true;
    return cudaSuccess;
  };

  // One pass of right-hand sides: [zero the exchange levels] project
  // [copy them out] [NCCL sum over ranks] [copy the caller's sum in] expand.
  auto pass = [&](double* zex, size_t exch, auto&& project, auto&& expand, bool has_project, int gp, int ge,
                  auto&& before_project, auto&& before_expand, auto&& after_expand) -> hmat_status {
    const size_t bytes = exch * sizeof(double);
    // optional per-CTA trace: zeroed slots, filled by the kernels
    auto trace = [&](int ph, int grid) -> cudaError_t {
      if (!H->trace) return cudaSuccess;
      a.trace = H->trace + (int64_t)ph * kTraceCap * 3;
      H->trace_n[ph] = grid < kTraceCap ? grid : kTraceCap;
      return grid <= kTraceCap ? cudaMemsetAsync(a.trace, 0, size_t(grid) * 3 * 8, H->stream) : cudaSuccess;
    };
    a.exch = int64_t(exch);
    if (phases & kPhaseProject) ++H->epoch;  // peer exchange: a new pass (same count on every rank)
    a.epoch = H->epoch;
    if (phases & kPhaseProject) {
      if (p.P > 1 && exch) CUDA_TRY(cudaMemsetAsync(zex, 0, bytes, H->stream));
      CUDA_TRY(before_project());
      if (has_project && level_mask) {
        CUDA_TRY(trace(0, gp));
        prof_begin(H, 0, &ep);
        CUDA_TRY(project());
        prof_end(H, &ep);
      }
      if (exch_out && exch) CUDA_TRY(cudaMemcpyAsync(exch_out, zex, bytes, cudaMemcpyDeviceToDevice, H->stream));
    }
    if ((phases & kPhaseExchange) && !H->external && !H->peer && p.P > 1 && exch) {
      prof_begin(H, 1, &ep);
      std::string m;
      if (H->tree) {
        hmat_status st = ensure_buf(&H->xtmp, &H->xtmp_cap, exch);
        if (st != HMAT_OK) return st;
        m = hmat::comm_tree_allreduce_sum(H->comm, zex, H->xtmp, exch, p.P, p.rank, H->stream);
      } else {
        m = hmat::comm_allreduce_sum(H->comm, zex, exch, H->stream);
      }
      if (!m.empty()) return fail(HMAT_ERR_NCCL, m);
      prof_end(H, &ep);
    }
    if (phases & kPhaseExpand) {
      if (exch_in && exch) CUDA_TRY(cudaMemcpyAsync(zex, exch_in, bytes, cudaMemcpyDeviceToDevice, H->stream));
      CUDA_TRY(before_expand());
      CUDA_TRY(trace(1, ge));
      prof_begin(H, 2, &ep);
      CUDA_TRY(expand());
      prof_end(H, &ep);
      CUDA_TRY(after_expand());
    }
    return HMAT_OK;
  };

  if (use_dmma(p, nrhs)) {
    hmat_status st = ensure_dmma(H);
    if (st != HMAT_OK) return st;
    a.vp = p.vp;
    a.dkr = p.dkr;
    a.dkc = p.dkc;
    a.part = H->part_d;
    a.cnt = H->cnt_d;
    if (p.L > 0) {  // V-role panels [L][N_loc][Wp], box [1][dkr][vp]
      const uint64_t dims[3] = {uint64_t(p.Wp), uint64_t(n), uint64_t(p.L)};
      const uint64_t strides[2] = {uint64_t(p.Wp) * 8, uint64_t(p.panel_stride) * 8};
      const bool vdiag = (p.dbg & 128) && p.nslice <= 1 && p.Wp <= p.vp;  // (bit 7: diagnostics, kernels_dmma.cu)
      const uint32_t box[3] = {uint32_t(vdiag ? p.Wp : p.vp), uint32_t(p.dkr), 1};
      hmat_status st3 = encode_map(&a.tm_v, 3, a.V, dims, strides, box);
      if (st3 != HMAT_OK) return st3;
      const uint32_t ubox[3] = {uint32_t(p.dkc + 4), uint32_t(hmat::kDmmaRE), 1};
      if ((st3 = encode_map(&a.tm_u, 3, a.U, dims, strides, ubox)) != HMAT_OK) return st3;
    }
    if (p.adm) {  // the nd near-field D-role panels [nd][N_loc][Dp], box [1][64][KC+4]
      const uint64_t dims[3] = {uint64_t(p.Dp), uint64_t(n), uint64_t(p.nd)};
      const uint64_t strides[2] = {uint64_t(p.Dp) * 8, uint64_t(p.d_stride) * 8};
      const uint32_t box[3] = {uint32_t((p.dkc == 16 ? 16 : 32) + 4), uint32_t(hmat::kDmmaRE), 1};
      hmat_status st3 = encode_map(&a.tm_d, 3, a.D, dims, strides, box);
      if (st3 != HMAT_OK) return st3;
    } else {  // D-role panel [N_loc][Dp], box [64][KC+4]
      const uint64_t dims[2] = {uint64_t(p.Dp), uint64_t(n)};
      const uint64_t strides[1] = {uint64_t(p.Dp) * 8};
      const uint32_t box[2] = {uint32_t((p.dkc == 16 ? 16 : 32) + 4), uint32_t(hmat::kDmmaRE)};  // dense stage columns
      hmat_status st3 = encode_map(&a.tm_d, 2, a.D, dims, strides, box);
      if (st3 != HMAT_OK) return st3;
    }
    for (int c0 = 0; c0 < nrhs; c0 += hmat::kDmmaNB) {
      a.nr = nrhs - c0 < hmat::kDmmaNB ? nrhs - c0 : hmat::kDmmaNB;
      a.wslice = p.wslice;
      a.nslice = p.nslice;
      a.accbuf = H->accbuf_d;
      // the pass width: 32 when at most 32 rhs remain (half the work), else 64
      const hmat::Plan::DmmaLayout& dl = p.dmma_layout(a.nr);
      const int nb = dl.nb;
      // standard admissibility: slots whose partner lies outside the domain are
      // never written and must read as zero; a pass of another width leaves values
      // at other positions of the fragment-major rows, so clear on a width change
      if (p.adm && H->zt_nb_d != nb && (phases & kPhaseProject)) {
        CUDA_TRY(cudaMemsetAsync(H->zloc_d, 0, std::max<size_t>(256, size_t(p.z_local_rows) * p.W * hmat::kDmmaNB * 8),
                                 H->stream));
        H->zt_nb_d = nb;
      }
      a.dnw = dl.nw;
      // 8-wide passes on narrow panels: level-interleaved chunks, so x (nb/W of
      // the V bytes per level: 1/6 at W = 48) is re-read from L2, not DRAM
      // (c4 8 rhs project 10.8 -> 10.0 ms, c2 0.66 -> 0.55 ms; at W = 224 or 16
      // rhs the chunk switches cost more than they save)
      // 16 wide: chunks of 16 stages, so the x rows of all CTAs' current chunks
      // (592 x 16 x 32 rows x 16 rhs: 39 MB) stay in L2 (c4 16 rhs project 13.0 ->
      // 12.0 ms, c2 0.80 -> 0.70 ms; 32-stage chunks: 78 MB, no gain)
      a.pchunk = nb == 8 && p.W <= 112 ? p.dmma_pchunk : nb == 16 && p.W <= 112 ? p.dmma_pchunk16 : 0;
      a.nstage_p = dl.dns_p;
      a.stage_bytes_p = dl.dstage_p;
      a.grid_e_gen = dl.dgrid_e_gen;
      a.bar_off_p = dl.dns_p * dl.dstage_p;
      a.nstage_e = dl.dns_e;
      a.stage_bytes_e = dl.dstage_e;
      a.bar_off_e = dl.dns_e * dl.dstage_e;
      a.x = xd + c0 * ldx;
      a.y = yd + c0 * n;
      {  // this pass's x columns [nr][N_loc] (ld = ldx), box [nb][dkr + 4] (rows >= nr zero-filled)
        const uint64_t dims[2] = {uint64_t(n), uint64_t(a.nr)};
        const uint64_t strides[1] = {uint64_t(ldx) * 8};
        const uint32_t box[2] = {uint32_t(p.dkr + 4), uint32_t(nb)};
        hmat_status st3 = encode_map(&a.tm_x, 2, a.x, dims, strides, box);
        if (st3 != HMAT_OK) return st3;
        const uint32_t xbox[2] = {uint32_t((p.dkc == 16 ? 16 : 32) + 4), uint32_t(nb)};
        if ((st3 = encode_map(&a.tm_xe, 2, a.x, dims, strides, xbox)) != HMAT_OK) return st3;
      }
      for (int l = 1; l <= p.L; ++l) {
        hmat::LevelArgs& lv = a.lv[l];
        lv.m = p.m[l];
        lv.seg_rows = p.m[l] < n ? p.m[l] : n;
        lv.zt = (l <= p.cross ? H->zex_d : H->zloc_d) + p.zt_off[l] * p.W * nb;
        lv.tbase = p.zt_tbase[l];
      }
      size_t exch = size_t(p.z_exch_rows) * p.W * nb;
      a.zex_base = H->zex_d;  // PEER: the project's last CTA pushes this region to every mailbox
      if (H->sx) {  // standard admissibility, P > 1: the packed cross-rank buffer (std_exchange.h)
        const hmat::StdExchange& X = *H->sx;
        exch = size_t(trans ? X.doubles_t(nb, p.r) : X.doubles(nb, p.r));
        a.skip_remote = trans ? 1 : 0;
        a.xchg = H->zex_d;
        a.halo_of = H->halo_of_d;
        a.halo_base = X.halo_base(nb, p.r);
        a.bpad = X.bpad;
        for (int l = 2; l <= p.L; ++l) a.lv[l].xent = H->xent_d + X.src_off[l];
        if (!trans && X.Hn > 0) {  // remote neighbours' x: [Hn nb][bpad], box [nb][KD + 4]
          const uint64_t dims[2] = {uint64_t(X.bpad), uint64_t(X.Hn) * nb};
          const uint64_t strides[1] = {uint64_t(X.bpad) * 8};
          const uint32_t box[2] = {uint32_t((p.dkc == 16 ? 16 : 32) + 4), uint32_t(nb)};
          hmat_status st3 = encode_map(&a.tm_xh, 2, H->zex_d + a.halo_base, dims, strides, box);
          if (st3 != HMAT_OK) return st3;
        }
      }
      auto before_project = [&]() -> cudaError_t {  // P > 1, standard: this rank's halo x (H^T: products)
        if (!H->sx) return cudaSuccess;
        if (trans)
          return hmat::launch_std_tpack(H->zex_d + a.halo_base, H->D, p.d_stride, p.Dp, a.x, ldx, H->tpack_d,
                                        int64_t(H->sx->tpack.size() / 3), nb, a.nr, p.b, a.bpad, H->stream);
        return hmat::launch_std_pack_x(H->zex_d + a.halo_base, a.x, ldx, H->pack_d, int64_t(H->sx->pack.size() / 2),
                                       nb, a.nr, p.b, a.bpad, H->stream);
      };
      auto before_expand = [&]() -> cudaError_t {
        // PEER: the rank-ordered sum of the P mailbox slots into the exchange levels,
        // when this pass ran a project (whose last CTA raised the flags)
        if (H->peer) return dl.dgrid_p > 0 && level_mask ? hmat::launch_peer_sum(a, H->zex_d, H->stream) : cudaSuccess;
        if (!H->sx) return cudaSuccess;  // standard, P > 1: the received z entries into Zt
        return hmat::launch_std_unpack_z_dmma(H->zloc_d, H->zex_d, H->unpack_d, int64_t(H->sx->unpack.size() / 2), nb,
                                              a.nr, p.W, p.r, H->stream);
      };
      auto after_expand = [&]() -> cudaError_t {  // standard H^T, P > 1: the incoming near-field products
        if (!H->sx || !trans || !dense) return cudaSuccess;
        return hmat::launch_std_tadd(a.y, n, alpha, H->zex_d + a.halo_base, H->tadd_leaf_d, H->tadd_off_d,
                                     H->tadd_pair_d, int64_t(H->sx->tadd_leaf.size()), nb, a.nr, p.b, a.bpad,
                                     H->stream);
      };
      hmat_status st2 = pass(
          H->zex_d, exch, [&] { return hmat::launch_project_dmma(a, nb, dl.dgrid_p, dl.dsmem_p, H->stream); },
          [&] {
            return expand_rows([&] { return hmat::launch_expand_dmma(a, nb, dl.dgrid_e, dl.dsmem_e, H->stream); },
                               hmat::kDmmaRE, true, c0, a.nr);
          },
          dl.dgrid_p > 0,
          dl.dgrid_p, dl.dgrid_e, before_project, before_expand, after_expand);
      if (st2 != HMAT_OK) return st2;
    }
  }
  for (int c0 = 0; !use_dmma(p, nrhs) && c0 < nrhs; c0 += p.max_nr) {
    const int nr = nrhs - c0 < p.max_nr ? nrhs - c0 : p.max_nr;
    const int cap = nr_cap(nr);
    const hmat::Plan::Layout& ly = p.lay[hmat::nr_index(cap)];
    a.nstage_p = ly.nstage_p;
    a.stage_bytes_p = ly.stage_bytes_p;
    a.nstage_e = ly.nstage_e;
    a.stage_bytes_e = ly.stage_bytes_e;
    a.red_off_p = ly.red_off_p;
    a.bar_off_p = ly.bar_off_p;
    a.bar_off_e = ly.bar_off_e;
    a.nr = nr;
    a.x = xd + c0 * ldx;
    a.y = yd + c0 * n;
    // expand's dynamic chunks of 1 item, 2 for standard admissibility (s2: 3.81 ->
    // 3.75 ms against static ranges, 3.89 with chunks of 1; A/B late r02); 0 =
    // static ranges when an item may have no stage at all (the chunk protocol
    // carries the chunk id in a chunk's first stage): no dense block and, under
    // standard admissibility, no active level >= 2 (level 1 holds no blocks)
    const uint64_t lv_all = p.L >= 64 ? ~0ull : (1ull << p.L) - 1;
    const bool std_stage = dense || (level_mask & lv_all & ~1ull);
    a.chunk_e = p.expand_chunk >= 0 ? p.expand_chunk : (p.adm ? (std_stage ? 2 : 0) : 1);
    if (!level_mask && !dense) a.chunk_e = 0;
    // project: the last active level in dynamic chunks of whole nodes (>= 4
    // stages), when it is local (no exchange) and has at least 2 chunks per CTA
    a.dyn_level = 0;
    a.sched_p = H->sched + 4;
    // small operators (every active level's stages fit the grid at once, one GPU):
    // level-parallel project, one stage of one level per CTA (kernels_project.cu)
    const int64_t SL = p.N_loc / p.Rp;
    const int nact = __builtin_popcountll(level_mask);
    a.lpar = p.lpar && p.P == 1 && nact >= 2 && SL * nact <= int64_t(ly.grid_p_slots) && SL <= p.grid_p_max ? 1 : 0;
    const int grid_p = a.lpar ? static_cast<int>(SL * nact) : ly.grid_p;
    if (level_mask && p.project_dyn && !a.lpar) {
      const int ll = 64 - __builtin_clzll(level_mask);
      const int64_t SLs = p.N_loc / p.Rp, seg = std::min<int64_t>(p.m[ll], p.N_loc) / p.Rp;
      int64_t ch = seg;
      while (ch < p.project_chunk) ch += seg;
      if (ll > p.cross && SLs / ch >= 2 * int64_t(ly.grid_p)) {
        a.dyn_level = ll;
        a.dyn_chunk = ch;
      }
    }
    for (int l = 1; l <= p.L; ++l) {
      hmat::LevelArgs& lv = a.lv[l];
      lv.m = p.m[l];
      lv.seg_rows = p.m[l] < n ? p.m[l] : n;
      lv.zt = (l <= p.cross ? H->zex : H->zloc) + p.zt_off[l] * p.Wp * cap;
      lv.tbase = p.zt_tbase[l];
    }
    size_t exch = size_t(p.z_exch_rows) * p.Wp * cap;
    if (H->sx) {  // standard admissibility, P > 1: the packed cross-rank buffer
      const hmat::StdExchange& X = *H->sx;
      // H^T: products of the cross near-field pairs instead of the halo x
      exch = size_t(trans ? X.doubles_t(cap, p.r) : X.doubles(cap, p.r));
      a.skip_remote = trans ? 1 : 0;
      a.xchg = H->zex;
      a.halo_of = H->halo_of_d;
      a.halo_base = X.halo_base(cap, p.r);
      a.bpad = X.bpad;
      for (int l = 2; l <= p.L; ++l) a.lv[l].xent = H->xent_d + X.src_off[l];
    }
    auto pack_x = [&]() -> cudaError_t {
      if (!H->sx) return cudaSuccess;
      if (trans)  // H^T: c_{S,T} = (D_{S,T})^T x_S of this rank's outgoing near-field pairs (forward D)
        return hmat::launch_std_tpack(H->zex + a.halo_base, H->D, p.d_stride, p.Dp, a.x, ldx, H->tpack_d,
                                      int64_t(H->sx->tpack.size() / 3), cap, nr, p.b, a.bpad, H->stream);
      return hmat::launch_std_pack_x(H->zex + a.halo_base, a.x, ldx, H->pack_d, int64_t(H->sx->pack.size() / 2), cap,
                                     nr, p.b, a.bpad, H->stream);
    };
    auto add_t = [&]() -> cudaError_t {  // H^T: the incoming near-field products, in pair order
      if (!H->sx || !trans || !dense) return cudaSuccess;
      return hmat::launch_std_tadd(a.y, n, alpha, H->zex + a.halo_base, H->tadd_leaf_d, H->tadd_off_d, H->tadd_pair_d,
                                   int64_t(H->sx->tadd_leaf.size()), cap, nr, p.b, a.bpad, H->stream);
    };
    auto unpack_z = [&]() -> cudaError_t {
      if (!H->sx) return cudaSuccess;
      return hmat::launch_std_unpack_z(H->zloc, H->zex, H->unpack_d, int64_t(H->sx->unpack.size() / 2), cap, nr,
                                       p.Wp, p.r, H->stream);
    };
    // Standard admissibility: slots whose partner lies outside the domain are
    // never written and must read as zero; after a pass with another rhs width
    // the buffer holds values at other positions, so clear it on a layout change.
    if (p.adm && H->zt_cap != cap && (phases & kPhaseProject)) {
      CUDA_TRY(cudaMemsetAsync(H->zloc, 0, std::max<size_t>(256, size_t(p.z_local_rows) * p.Wp * cap * 8),
                               H->stream));
      H->zt_cap = cap;
    }
    hmat_status st2 = pass(
        H->zex, exch, [&] { return hmat::launch_project(a, cap, grid_p, ly.smem_p, H->stream); },
        [&] {
          return expand_rows([&] { return hmat::launch_expand(a, cap, ly.grid_e, ly.smem_e, H->stream); }, p.Re, false,
                             c0, nr);
        },
        ly.grid_p > 0, grid_p,
        ly.grid_e, pack_x, unpack_z, add_t);
    if (st2 != HMAT_OK) return st2;
  }
  if (async_io) {  // y out on s_out once the kernels are done; no host wait
    CUDA_TRY(cudaEventRecord(H->ev_comp[par], H->stream));
    H->comp_rec[par] = true;
    if (!y_dev) {
      if (!y_split) {  // (row-chunked: the chunks' copies are already queued on s_out)
        CUDA_TRY(cudaStreamWaitEvent(H->s_out, H->ev_comp[par], 0));
        CUDA_TRY(cudaMemcpyAsync(y, yd, size_t(n) * nrhs * sizeof(double), cudaMemcpyDefault, H->s_out));
      }
      CUDA_TRY(cudaEventRecord(H->ev_out[par], H->s_out));
      H->out_rec[par] = true;
    }
    CUDA_TRY(cudaGetLastError());
    return HMAT_OK;
  }
  if (!y_dev && (phases & kPhaseExpand) && !y_split) {
    prof_begin(H, 3, &ep);
    CUDA_TRY(cudaMemcpyAsync(y, yd, size_t(n) * nrhs * sizeof(double), cudaMemcpyDefault, H->stream));
    prof_end(H, &ep);
  }
  if (host_io) {
    CUDA_TRY(cudaStreamSynchronize(H->stream));
    if (y_split) CUDA_TRY(cudaStreamSynchronize(H->s_y));
    hmat_status sa = check_async(H);
    if (sa != HMAT_OK) return sa;
  }
  CUDA_TRY(cudaGetLastError());
  return HMAT_OK;
}

}  // namespace

extern "C" {

hmat_status hmat_matvec_parts(hmat_t H, const double* x, double* y, int nrhs, uint64_t level_mask, int dense) {
  return run(H, 0, 1.0, x, 0.0, y, nrhs, level_mask, dense);
}

hmat_status hmat_matvec(hmat_t H, const double* x, double* y, int nrhs) {
  return run(H, 0, 1.0, x, 0.0, y, nrhs, ~0ull, 1);
}

hmat_status hmat_gemv(hmat_t H, int trans, double alpha, const double* x, double beta, double* y, int nrhs) {
  return run(H, trans, alpha, x, beta, y, nrhs, ~0ull, 1);
}

hmat_status hmat_exchange_size_op(hmat_t H, int trans, int nrhs, int64_t* count) {
  if (!H || !count || nrhs < 1) return fail(HMAT_ERR_INVALID, "NULL argument or nrhs < 1");
  if (trans != 0 && trans != 1) return fail(HMAT_ERR_INVALID, "trans must be 0 (H) or 1 (H^T)");
  const hmat::Plan& p = H->plan;
  if (use_dmma(p, nrhs)) {
    if (nrhs > hmat::kDmmaNB) return fail(HMAT_ERR_INVALID, "more than one pass of right-hand sides");
    const int nb = p.dmma_layout(nrhs).nb;
    *count = p.P > 1 ? (H->sx ? (trans ? H->sx->doubles_t(nb, p.r) : H->sx->doubles(nb, p.r))
                              : p.z_exch_rows * p.W * nb)
                     : 0;
  } else {
    if (nrhs > p.max_nr) return fail(HMAT_ERR_INVALID, "more than one pass of right-hand sides");
    const int cap = nr_cap(nrhs);
    *count = p.P > 1 ? (H->sx ? (trans ? H->sx->doubles_t(cap, p.r) : H->sx->doubles(cap, p.r))
                              : p.z_exch_rows * p.Wp * cap)
                     : 0;
  }
  return HMAT_OK;
}

hmat_status hmat_exchange_size(hmat_t H, int nrhs, int64_t* count) { return hmat_exchange_size_op(H, 0, nrhs, count); }

hmat_status hmat_project_op(hmat_t H, int trans, const double* x, int nrhs, double* exchange) {
  int64_t count = 0;
  hmat_status st = hmat_exchange_size_op(H, trans, nrhs, &count);
  if (st != HMAT_OK) return st;
  if (count && !exchange && !H->peer) return fail(HMAT_ERR_INVALID, "exchange is NULL");
  return run(H, trans, 1.0, x, 0.0, nullptr, nrhs, ~0ull, 1, kPhaseProject, exchange, nullptr);
}

hmat_status hmat_project(hmat_t H, const double* x, int nrhs, double* exchange) {
  return hmat_project_op(H, 0, x, nrhs, exchange);
}

hmat_status hmat_expand_op(hmat_t H, int trans, double alpha, const double* x, const double* exchange, double beta,
                           double* y, int nrhs) {
  int64_t count = 0;
  hmat_status st = hmat_exchange_size_op(H, trans, nrhs, &count);
  if (st != HMAT_OK) return st;
  if (count && !exchange && !H->peer) return fail(HMAT_ERR_INVALID, "exchange is NULL");
  return run(H, trans, alpha, x, beta, y, nrhs, ~0ull, 1, kPhaseExpand, nullptr, exchange);
}

hmat_status hmat_expand(hmat_t H, const double* x, const double* exchange, double* y, int nrhs) {
  return hmat_expand_op(H, 0, 1.0, x, exchange, 0.0, y, nrhs);
}

hmat_status hmat_create_strict(int depth, int dim, int leaf_size, int rank, const double* const* U,
                               const double* const* V, const double* Dc, const hmat_dist_t* dist, hmat_t* out) {
  // Def 2.4 read literally (leaves checked first): the leaf-parent diagonal
  // blocks (2^dim leaf_size square) are dense and low-rank blocks exist at
  // levels 1..depth-1 -- exactly the structure of depth-1 with leaf 2^dim leaf_size.
  if (out) *out = nullptr;
  if (depth < 1) return fail(HMAT_ERR_INVALID, "strict structure needs depth >= 1");
  if (dim < 1 || dim > 3) return fail(HMAT_ERR_INVALID, "dim must be 1, 2 or 3 (ideal domains, PAPER.md:243-246)");
  if (leaf_size < 1 || leaf_size > (1 << 28)) return fail(HMAT_ERR_INVALID, "leaf_size must be >= 1");
  return hmat_create(depth - 1, dim, leaf_size << dim, rank, U, V, Dc, dist, out);
}

hmat_status hmat_create_standard_strict(int depth, int dim, int leaf_size, int rank, const double* const* U,
                                        const double* const* V, const double* Dc, const hmat_dist_t* dist,
                                        hmat_t* out) {
  // Def 2.4 read literally under standard admissibility: at the leaf level every
  // child pair of two touching leaf-parents is dense, low-rank blocks exist at
  // levels 2..depth-1 -- the standard structure of depth-1 with leaf 2^dim leaf_size
  // (its near field = the touching leaf-parents' (2^dim b)^2 blocks).
  if (out) *out = nullptr;
  if (depth < 1) return fail(HMAT_ERR_INVALID, "strict structure needs depth >= 1");
  if (dim < 1 || dim > 3) return fail(HMAT_ERR_INVALID, "dim must be 1, 2 or 3 (ideal domains, PAPER.md:243-246)");
  if (leaf_size < 1 || leaf_size > (1 << 28)) return fail(HMAT_ERR_INVALID, "leaf_size must be >= 1");
  return hmat_create_standard(depth - 1, dim, leaf_size << dim, rank, U, V, Dc, dist, out);
}

hmat_status hmat_destroy(hmat_t H) {
  release(H);
  return HMAT_OK;
}

const char* hmat_last_error(void) { return g_err.c_str(); }

int64_t hmat_num_points(hmat_t H) { return H ? H->plan.N : -1; }

hmat_status hmat_local_rows(hmat_t H, int64_t* begin, int64_t* end) {
  if (!H || !begin || !end) return fail(HMAT_ERR_INVALID, "NULL argument");
  *begin = H->plan.row0;
  *end = H->plan.row0 + H->plan.N_loc;
  return HMAT_OK;
}

hmat_status hmat_set_host_async(hmat_t H, int enable) {
  if (!H) return fail(HMAT_ERR_INVALID, "H is NULL");
  CUDA_TRY(cudaSetDevice(H->device));
  if (H->host_async && !enable) {  // leaving the mode: drain the pipeline
    if (H->s_in) CUDA_TRY(cudaStreamSynchronize(H->s_in));
    CUDA_TRY(cudaStreamSynchronize(H->stream));
    if (H->s_out) CUDA_TRY(cudaStreamSynchronize(H->s_out));
  }
  H->host_async = enable != 0;
  return HMAT_OK;
}

hmat_status hmat_synchronize(hmat_t H) {
  if (!H) return fail(HMAT_ERR_INVALID, "H is NULL");
  CUDA_TRY(cudaSetDevice(H->device));
  if (H->s_in) CUDA_TRY(cudaStreamSynchronize(H->s_in));
  CUDA_TRY(cudaStreamSynchronize(H->stream));
  if (H->s_out) CUDA_TRY(cudaStreamSynchronize(H->s_out));
  return check_async(H);
}

hmat_status hmat_set_stream(hmat_t H, void* stream) {
  if (!H) return fail(HMAT_ERR_INVALID, "H is NULL");
  CUDA_TRY(cudaSetDevice(H->device));
  CUDA_TRY(cudaStreamSynchronize(H->stream));
  if (H->own_stream) cudaStreamDestroy(H->stream);
  H->own_stream = false;
  H->stream = static_cast<cudaStream_t>(stream);
  return HMAT_OK;
}

hmat_status hmat_nccl_unique_id(void* out128) {
  if (!out128) return fail(HMAT_ERR_INVALID, "out is NULL");
  std::string m = hmat::comm_unique_id(out128);
  if (!m.empty()) return fail(HMAT_ERR_NCCL, m);
  return HMAT_OK;
}

hmat_status hmat_nccl_selftest(int device, int64_t count) {
  if (count < 1) return fail(HMAT_ERR_INVALID, "count must be >= 1");
  CUDA_TRY(cudaSetDevice(device));
  char id[128];
  std::string m = hmat::comm_unique_id(id);
  if (!m.empty()) return fail(HMAT_ERR_NCCL, m);
  hmat::Comm* c = nullptr;
  m = hmat::comm_create(id, 1, 0, &c);
  if (!m.empty()) return fail(HMAT_ERR_NCCL, m);
  std::vector<double> h(static_cast<size_t>(count)), back(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) h[static_cast<size_t>(i)] = 0.5 * static_cast<double>(i) - 3.0;
  double* d = nullptr;
  cudaStream_t s = nullptr;
  const size_t bytes = static_cast<size_t>(count) * sizeof(double);
  cudaError_t e = cudaMalloc(&d, bytes);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) m = hmat::comm_allreduce_sum(c, d, static_cast<size_t>(count), s);
  if (e == cudaSuccess && m.empty()) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && m.empty()) e = cudaMemcpy(back.data(), d, bytes, cudaMemcpyDeviceToHost);
  bool same = back == h;
  // one TREE round with this rank as its own partner: the buffer doubles
  double* t = nullptr;
  std::vector<double> twice(static_cast<size_t>(count));
  if (e == cudaSuccess && m.empty()) e = cudaMalloc(&t, bytes);
  if (e == cudaSuccess && m.empty()) m = hmat::comm_swap_round(c, d, t, static_cast<size_t>(count), 0, s);
  if (e == cudaSuccess && m.empty()) e = hmat::launch_add_inplace(d, t, static_cast<size_t>(count), s);
  if (e == cudaSuccess && m.empty()) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && m.empty()) e = cudaMemcpy(twice.data(), d, bytes, cudaMemcpyDeviceToHost);
  if (s) cudaStreamDestroy(s);
  if (d) cudaFree(d);
  if (t) cudaFree(t);
  hmat::comm_destroy(c);
  if (e != cudaSuccess) return cuda_fail(e, "hmat_nccl_selftest");
  if (!m.empty()) return fail(HMAT_ERR_NCCL, m);
  if (!same) return fail(HMAT_ERR_NCCL, "one-rank ncclAllReduce changed the buffer");
  for (int64_t i = 0; i < count; ++i)
    if (twice[static_cast<size_t>(i)] != 2.0 * h[static_cast<size_t>(i)])
      return fail(HMAT_ERR_NCCL, "tree round (send/recv to self + add) gave a wrong value");
  return HMAT_OK;
}

hmat_status hmat_peer_export(hmat_t H, void* handle64) {
  if (!H || !handle64) return fail(HMAT_ERR_INVALID, "NULL argument");
  if (!H->peer) return fail(HMAT_ERR_INVALID, "H does not use the peer exchange");
  CUDA_TRY(cudaSetDevice(H->device));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  CUDA_TRY(cudaIpcGetMemHandle(&h, H->mbox));
  memcpy(handle64, &h, sizeof h);
  return HMAT_OK;
}

hmat_status hmat_peer_import(hmat_t H, const void* handles) {
  if (!H || !handles) return fail(HMAT_ERR_INVALID, "NULL argument");
  if (!H->peer) return fail(HMAT_ERR_INVALID, "H does not use the peer exchange");
  CUDA_TRY(cudaSetDevice(H->device));
  const int P = H->plan.P;
  std::vector<double*> ptrs(P);
  for (int g = 0; g < P; ++g) {
    if (g == H->plan.rank) {
      ptrs[g] = H->mbox;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + 64 * g, sizeof h);
    void* q = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
    H->opened.push_back(q);
    ptrs[g] = static_cast<double*>(q);
  }
  CUDA_TRY(cudaMemcpy(H->mbox_dev, ptrs.data(), P * sizeof(double*), cudaMemcpyHostToDevice));
  H->connected = true;
  return HMAT_OK;
}

hmat_status hmat_peer_connect_local(hmat_t H, const hmat_t* ranks) {
  if (!H || !ranks) return fail(HMAT_ERR_INVALID, "NULL argument");
  if (!H->peer) return fail(HMAT_ERR_INVALID, "H does not use the peer exchange");
  const int P = H->plan.P;
  std::vector<double*> ptrs(P);
  CUDA_TRY(cudaSetDevice(H->device));
  for (int g = 0; g < P; ++g) {
    if (!ranks[g] || !ranks[g]->peer || ranks[g]->plan.P != P || ranks[g]->plan.rank != g)
      return fail(HMAT_ERR_INVALID, "ranks[g] must be rank g's handle of the same peer-exchange operator");
    if (ranks[g]->mb != H->mb)
      return fail(HMAT_ERR_INVALID, "ranks[g]'s mailbox slot size differs (not the same operator)");
    if (ranks[g]->device != H->device) {  // this rank's kernels store into that device's memory
      int ok = 0;
      CUDA_TRY(cudaDeviceCanAccessPeer(&ok, H->device, ranks[g]->device));
      if (!ok) return fail(HMAT_ERR_UNSUPPORTED, "no peer access from this device to rank " + std::to_string(g) + "'s");
      cudaError_t pe = cudaDeviceEnablePeerAccess(ranks[g]->device, 0);
      if (pe == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else if (pe != cudaSuccess)
        return cuda_fail(pe, "cudaDeviceEnablePeerAccess");
    }
    ptrs[g] = ranks[g]->mbox;
  }
  CUDA_TRY(cudaMemcpy(H->mbox_dev, ptrs.data(), P * sizeof(double*), cudaMemcpyHostToDevice));
  H->connected = true;
  return HMAT_OK;
}

hmat_status hmat_comm_info(hmat_t H, int* nranks, int* rank) {
  if (!H || !nranks || !rank) return fail(HMAT_ERR_INVALID, "NULL argument");
  *nranks = H->plan.P;
  *rank = H->plan.rank;
  if (H->comm) {  // the NCCL communicator's own view
    CUDA_TRY(cudaSetDevice(H->device));
    std::string m = hmat::comm_info(H->comm, nranks, rank);
    if (!m.empty()) return fail(HMAT_ERR_NCCL, m);
  }
  return check_async(H);
}

hmat_status hmat_profile(hmat_t H, int enable) {
  if (!H) return fail(HMAT_ERR_INVALID, "H is NULL");
  H->prof = enable != 0;
  return HMAT_OK;
}

hmat_status hmat_cta_trace(hmat_t H, int enable) {
  if (!H) return fail(HMAT_ERR_INVALID, "H is NULL");
  CUDA_TRY(cudaSetDevice(H->device));
  CUDA_TRY(cudaStreamSynchronize(H->stream));
  if (enable && !H->trace) {
    CUDA_TRY(cudaMalloc(&H->trace, size_t(2) * kTraceCap * 3 * sizeof(unsigned long long)));
  } else if (!enable && H->trace) {
    cudaFree(H->trace);
    H->trace = nullptr;
  }
  H->trace_n[0] = H->trace_n[1] = 0;
  return HMAT_OK;
}

hmat_status hmat_cta_trace_read(hmat_t H, int kernel, int64_t* out, int max_ctas, int* n_ctas) {
  if (!H || !out || !n_ctas || (kernel != 0 && kernel != 1)) return fail(HMAT_ERR_INVALID, "bad argument");
  if (!H->trace) return fail(HMAT_ERR_INVALID, "tracing is not enabled (hmat_cta_trace)");
  CUDA_TRY(cudaSetDevice(H->device));
  CUDA_TRY(cudaStreamSynchronize(H->stream));
  const int n = H->trace_n[kernel] < max_ctas ? H->trace_n[kernel] : max_ctas;
  if (n > 0)
    CUDA_TRY(cudaMemcpy(out, H->trace + (int64_t)kernel * kTraceCap * 3, size_t(n) * 3 * 8, cudaMemcpyDeviceToHost));
  *n_ctas = n;
  return HMAT_OK;
}

hmat_status hmat_profile_read(hmat_t H, double* ms, int64_t* launches) {
  if (!H || !ms || !launches) return fail(HMAT_ERR_INVALID, "NULL argument");
  CUDA_TRY(cudaSetDevice(H->device));
  CUDA_TRY(cudaStreamSynchronize(H->stream));
  for (auto& e : H->ev) {
    float t = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&t, e.a, e.b));
    H->ms[e.phase] += t;
    H->nl[e.phase] += 1;
    H->pool.push_back(e.a);
    H->pool.push_back(e.b);
  }
  H->ev.clear();
  for (int i = 0; i < HMAT_NUM_PHASES; ++i) {
    ms[i] = H->ms[i];
    launches[i] = H->nl[i];
    H->ms[i] = 0;
    H->nl[i] = 0;
  }
  return HMAT_OK;
}

int64_t hmat_launches_per_matvec(hmat_t H, int nrhs) {
  if (!H || nrhs < 1) return -1;
  const hmat::Plan& p = H->plan;
  const int per = use_dmma(p, nrhs) ? hmat::kDmmaNB : p.max_nr;
  const int64_t passes = (nrhs + per - 1) / per;
  int per_pass = (p.stages_p > 0 ? 1 : 0) + 1;  // project (if any level) + expand
  if (H->sx) per_pass += 2;                     // standard admissibility, P > 1: pack x, unpack z
  if (H->peer && use_dmma(p, nrhs)) per_pass += 1;  // tensor-core path with PEER: the mailbox sum
  if (H->tree) {                                // one add kernel per recursive-doubling round
    for (int bit = 1; bit < p.P; bit <<= 1) ++per_pass;
  }
  return passes * per_pass;
}

hmat_status hmat_plan_query(int depth, int dim, int leaf_size, int rank, int nranks, int rank_id,
                            hmat_plan_info_t* info) {
  if (!info) return fail(HMAT_ERR_INVALID, "info is NULL");
  hmat::Plan p;
  std::string msg = hmat::plan_build(depth, dim, leaf_size, rank, nranks, rank_id, options_from_env(148), &p);
  if (!msg.empty()) return plan_status(msg);
  memset(info, 0, sizeof *info);
  info->N = p.N;
  info->row_begin = p.row0;
  info->row_end = p.row0 + p.N_loc;
  info->c = p.c;
  info->W = p.W;
  info->W_pitch = p.Wp;
  info->cross_levels = p.cross;
  info->exchange_rows = p.z_exch_rows;
  for (int l = 1; l <= p.cross && l < 64; ++l) info->level_rows_offset[l] = p.zt_off[l];
  info->Rp = p.Rp;
  info->Re = p.Re;
  info->tpr = p.tpr;
  info->nstage_p = p.lay[0].nstage_p;
  info->nstage_e = p.lay[0].nstage_e;
  info->grid_p = p.lay[0].grid_p;
  info->grid_e = p.lay[0].grid_e;
  info->smem_p = p.lay[0].smem_p;
  info->smem_e = p.lay[0].smem_e;
  info->max_nr = p.max_nr;
  info->dmma = use_dmma(p, p.dmma_min) ? 1 : 0;
  for (int i = 0; i < 4; ++i) {
    const hmat::Plan::DmmaLayout& d = p.dl[i];
    info->dmma_ok[i] = p.dmma_ok && d.ok ? 1 : 0;
    info->dmma_grid_p[i] = d.dgrid_p;
    info->dmma_grid_e[i] = d.dgrid_e;
    info->dmma_stages_p[i] = d.dns_p;
    info->dmma_stages_e[i] = d.dns_e;
    info->dmma_smem_p[i] = d.dsmem_p;
    info->dmma_smem_e[i] = d.dsmem_e;
  }
  return HMAT_OK;
}

hmat_status hmat_std_exchange_query(int depth, int dim, int leaf_size, int rank, int nranks, int rank_id,
                                    hmat_std_exchange_t* q) {
  if (!q) return fail(HMAT_ERR_INVALID, "q is NULL");
  hmat::PlanOptions opt = options_from_env(148);
  opt.adm = 1;
  hmat::Plan p;
  std::string msg = hmat::plan_build(depth, dim, leaf_size, rank, nranks, rank_id, opt, &p);
  if (!msg.empty()) return plan_status(msg);
  hmat::StdExchange X;
  if (nranks > 1) {
    msg = hmat::std_exchange_build(p, &X);
    if (!msg.empty()) return plan_status(msg);
  }
  auto give = [](const auto& v, auto* dst, int64_t cap, int64_t* n) {
    *n = int64_t(v.size());
    if (dst && cap >= *n) std::copy(v.begin(), v.end(), dst);
  };
  q->E = X.E;
  q->Hn = X.Hn;
  q->bpad = X.bpad;
  q->M = p.M;
  for (int l = 0; l <= depth && l < 64; ++l) {
    q->src_off[l] = X.src_off[l];
    q->zt_row_offset[l] = p.zt_off[l];
  }
  give(X.src_entry, q->src_entry, q->src_entry_cap, &q->n_src_entry);
  give(X.unpack, q->unpack, q->unpack_cap, &q->n_unpack);
  give(X.pack, q->pack, q->pack_cap, &q->n_pack);
  give(X.halo_of, q->halo_of, q->halo_of_cap, &q->n_halo_of);
  q->Hp = X.Hp;
  give(X.tpack, q->tpack, q->tpack_cap, &q->n_tpack);
  give(X.tadd_leaf, q->tadd_leaf, q->tadd_leaf_cap, &q->n_tadd_leaf);
  give(X.tadd_off, q->tadd_off, q->tadd_off_cap, &q->n_tadd_off);
  give(X.tadd_pair, q->tadd_pair, q->tadd_pair_cap, &q->n_tadd_pair);
  return HMAT_OK;
}

}  // extern "C"
