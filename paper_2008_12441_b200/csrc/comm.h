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
void comm_destroy(Comm* c);

}  // namespace hmat
