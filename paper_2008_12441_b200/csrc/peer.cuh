// peer.cuh -- the device side of the in-kernel NVLink peer exchange
// (HMAT_EXCHANGE_PEER): the push at the end of a project kernel
// (SIMT and tensor-core).
#pragma once
#include "device_utils.cuh"
#include "kernels.h"

namespace hmat {

// Peer exchange (the device-side Steps 2-4):
// the last CTA to finish pushes this rank's exchange levels (complete sums of
// its own sources, partial sums of sources spanning ranks, zeros elsewhere)
// into slot `rank` of every rank's mailbox over NVLink peer memory, then raises
// its flag there (system-scope release).  Readers sum the P slots in rank order,
// so the result is deterministic and equal on every rank.  Consumer threads only.
template <int NTH>  // threads taking part (all consumer threads of the CTA)
__device__ __forceinline__ void peer_push(const StreamArgs& a, int t, int64_t GL, volatile int* flag) {
  dev::named_bar_sync(1, NTH);
  __threadfence();
  if (t == 0) {
    const unsigned int prev = atomicAdd(a.done, 1u);
    *flag = (prev + 1 == static_cast<unsigned int>(GL)) ? 1 : 0;
  }
  dev::named_bar_sync(1, NTH);
  if (!*flag) return;
  __threadfence();
  const int par = static_cast<int>(a.epoch & 1);
  for (int p = 0; p < a.P; ++p) {
    double* dst = a.mbox[p] + ((int64_t)par * a.P + a.rank) * a.mb;
    for (int64_t o = t; o < a.exch; o += NTH) dst[o] = dev::ld_cg(a.zex_base + o);
  }
  __threadfence_system();
  dev::named_bar_sync(1, NTH);
  if (t == 0) {
    for (int p = 0; p < a.P; ++p) {
      uint64_t* fl = reinterpret_cast<uint64_t*>(a.mbox[p] + 2 * a.P * a.mb) + par * a.P + a.rank;
      dev::st_release_sys(fl, a.epoch);
    }
    *a.done = 0u;  // re-arm for the next pass
  }
}

// Bounded wait (one thread) for the P ranks' flags of this pass in this rank's
// mailbox.  Returns true when all are raised.  On timeout (a.peer_timeout_ns,
// HMAT_PEER_TIMEOUT_MS) it records the first missing rank in the handle's
// host-mapped error word -- the host reports it as HMAT_ERR_NCCL on the next
// call or at hmat_synchronize -- and returns false; the caller then finishes
// with whatever the mailbox holds (a wrong but finite y, flagged as an error):
// no __trap, so a late or missing peer never poisons the CUDA context.
__device__ __forceinline__ bool peer_wait_flags(const StreamArgs& a) {
  const int par = static_cast<int>(a.epoch & 1);
  const uint64_t* fl = reinterpret_cast<const uint64_t*>(a.mbox[a.rank] + 2 * a.P * a.mb) + par * a.P;
  const uint64_t t0 = dev::globaltimer_ns();
  for (int g = 0; g < a.P; ++g)
    while (dev::ld_acquire_sys(fl + g) != a.epoch) {
      __nanosleep(256);
      if (static_cast<int64_t>(dev::globaltimer_ns() - t0) > a.peer_timeout_ns) {
        // error word: bit 31 | missing rank << 16 | low 16 bits of the pass number
        // (a plain store: atomics on host-mapped memory need platform support, and
        // any waiter's report will do)
        *reinterpret_cast<volatile unsigned int*>(a.err) =
            0x80000000u | (static_cast<unsigned int>(g) << 16) | static_cast<unsigned int>(a.epoch & 0xffffu);
        __threadfence_system();
        return false;
      }
    }
  return true;
}

}  // namespace hmat
