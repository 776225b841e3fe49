// comm.h -- the cross-GPU part of Steps 2-4 over NCCL.
//
// Only the projected vectors z of sibling blocks whose parent spans more than
// one GPU cross a device boundary: levels 1..cross of the packed, level-major,
// target-major exchange buffer (plan.h).  Each GPU writes its (possibly
// partial) contributions there; a sum over GPUs completes Step 2 (reduction of
// partial node sums), Step 3 (source -> target transfer) and Step 4
// (broadcast to every GPU of the target group) in one collective.  NCCL is
// loaded with dlopen so the single-GPU library has no NCCL dependency.
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace hmat {

struct Comm;

// Fills 128 bytes with a fresh ncclUniqueId.  Returns "" or an error message.
std::string comm_unique_id(void* out128);
// Creates the communicator (collective over all ranks).
std::string comm_create(const void* id128, int nranks, int rank, Comm** out);
// In-place sum of `count` doubles over all ranks, on `stream`.
std::string comm_allreduce_sum(Comm* c, double* buf, size_t count, cudaStream_t stream);
// The paper's tree-structured Steps 2-4 (reduce to group leaders, leader to
// leader, broadcast back) on the hypercube of the P = 2^k
// ranks: log2 P rounds of recursive doubling, round j swapping the whole packed
// buffer with rank ^ 2^j (ncclSend + ncclRecv in one group) and adding the
// partner's copy (launch_add_inplace).  IEEE addition is commutative, so both
// partners hold bit-identical sums after every round, and after the last one
// every rank holds the same total -- deterministic, unlike an allreduce whose
// algorithm NCCL picks.  tmp: count doubles of scratch.
std::string comm_tree_allreduce_sum(Comm* c, double* buf, double* tmp, size_t count, int nranks, int rank,
                                    cudaStream_t stream);
// One round: buf -> partner, partner's buf -> tmp (partner may be this rank).
std::string comm_swap_round(Comm* c, const double* buf, double* tmp, size_t count, int partner, cudaStream_t stream);
// ncclCommGetAsyncError: "" while the communicator is healthy (or still
// progressing), else the error (a peer died, a network/NVLink fault, ...).
std::string comm_async_error(Comm* c);
// ncclCommCount / ncclCommUserRank of the library's communicator.
std::string comm_info(Comm* c, int* nranks, int* rank);
void comm_destroy(Comm* c);

// buf[i] += add[i] (kernels_aux.cu)
cudaError_t launch_add_inplace(double* buf, const double* add, size_t n, cudaStream_t s);

}  // namespace hmat
