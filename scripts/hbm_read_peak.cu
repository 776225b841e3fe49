// hbm_read_peak.cu -- what read-only HBM bandwidth can a kernel reach on this B200?
// The c4 matvec is a pure read stream (124.8 GB read, 0.27 GB written), so its
// ceiling is the read-only stream rate, not the copy figure in MEASURED_PEAKS.json.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/hbm_read_peak.cu -o /tmp/hbm_read_peak
//
// Variants: (1) LDG.128 grid-stride loads, unrolled; (2) 256-bit loads (sm_100);
// (3) 1-D bulk TMA (cp.async.bulk) into a shared-memory ring (the pattern the
// project / expand kernels use), for several stage sizes / depths / CTAs per SM.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <string>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__global__ void ldg128(const double2* __restrict__ p, int64_t n2, double* out) {
  double s = 0;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int U = 8;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
  }
  for (; i < n2; i += stride) { double2 v = __ldcs(p + i); s += v.x + v.y; }
  if (s == 123.456) out[0] = s;
}

__global__ void ldg256(const double* __restrict__ p, int64_t n4, double* out) {
  double s = 0;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  constexpr int U = 4;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    double v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(v[u][0]), "=d"(v[u][1]), "=d"(v[u][2]), "=d"(v[u][3])
                   : "l"(p + 4 * (i + u * stride)));
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u][0] + v[u][1] + v[u][2] + v[u][3];
  }
  if (s == 123.456) out[0] = s;
}

__global__ void fill_random(uint64_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = i * 0x9E3779B97F4A7C15ull + 12345;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    // a finite double in [1, 2) with random mantissa and random sign: like N(0,1) data
    p[i] = (z & 0x800FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// bulk TMA ring: warp 0 lane 0 produces, warps 1..C consume (sum 1 double per thread per stage)
__global__ void bulk_ring(const char* __restrict__ p, int64_t bytes, int stage_bytes, int nstage, double* out, int full_read,
                          const double* __restrict__ xv = nullptr, int xmode = 0, int nlev = 1, int inter = 0, int64_t lev_stride = 0) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (int64_t)stage_bytes * nstage);
  uint64_t* empty = full + nstage;
  const int ncw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) {
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sa(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sa(&empty[i])), "r"(ncw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t nst_all = bytes / stage_bytes;
  const int64_t nst = nst_all / nlev;  // stages per "level" chunk
  const int64_t s0 = nst * blockIdx.x / gridDim.x, s1 = nst * (blockIdx.x + 1) / gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int slot = 0;
  uint32_t phase = 0;
  const int rows = stage_bytes / 384;  // x: one double per 384-B "row"
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol, polx;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      if (xmode == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(polx));
      else polx = pol;
      for (int64_t it = 0; it < nlev * (s1 - s0); ++it) {
        // level-major (each CTA streams level 0's range, then level 1's ...) or
        // interleaved (stage s of every level, then stage s+1: like the expand kernel)
        const int lv = inter ? (int)(it % nlev) : (int)(it / (s1 - s0));
        const int64_t s = s0 + (inter ? it / nlev : it % (s1 - s0));
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&empty[slot])), "r"(phase ^ 1));
        const int64_t lo = (s * rows) & ~int64_t(1);
        const int xb = xmode ? (int)((((s * rows + rows + 1) & ~int64_t(1)) - lo) * 8) : 0;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&full[slot])), "r"(stage_bytes + xb));
        const int chunk = stage_bytes > 32768 ? 32768 : stage_bytes;
        const char* src = p + (lev_stride ? lv * lev_stride + s * (int64_t)stage_bytes : (lv * nst + s) * (int64_t)stage_bytes);
        for (int o = 0; o < stage_bytes; o += chunk) {
          const int n = stage_bytes - o < chunk ? stage_bytes - o : chunk;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(sa(smem + (int64_t)slot * stage_bytes + o)), "l"(src + o), "r"(n), "r"(sa(&full[slot])), "l"(pol) : "memory");
        }
        if (xmode)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(sa(smem + (int64_t)nstage * stage_bytes + 16 * nstage + slot * 1024)), "l"(xv + lo), "r"(xb), "r"(sa(&full[slot])), "l"(polx) : "memory");
        if (++slot == nstage) { slot = 0; phase ^= 1; }
      }
    }
    return;
  }
  double acc = 0;
  for (int64_t s = s0; s < s1 * nlev - s0 * (nlev - 1); ++s) {
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&full[slot])), "r"(phase));
    const double* st = reinterpret_cast<const double*>(smem + (int64_t)slot * stage_bytes);
    if (full_read) {
      const double2* s2 = reinterpret_cast<const double2*>(st);
      double2 a2 = make_double2(0, 0);
      for (int i = threadIdx.x - 32; i < stage_bytes / 16; i += blockDim.x - 32) { double2 v = s2[i]; a2.x = fma(v.x, 1.0001, a2.x); a2.y = fma(v.y, 0.9999, a2.y); }
      acc += a2.x + a2.y;
    } else {
      acc += st[threadIdx.x - 32];
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(sa(&empty[slot])));
    if (++slot == nstage) { slot = 0; phase ^= 1; }
  }
  if (acc == 123.456) out[0] = acc;
}

static int g_sustain = 100;
// expand-shaped stream: per 64-row item, 9 stages of 64 rows x 384 B (9 "U
// panels") + 1 stage of 64 rows x 512 B ("D"), `nslot` slots of `slot_bytes`.
// dsplit = 2: the D stage is two stages of 64 rows x 256 B columns halves... (as two 16 KB copies of rows 0..31 / 32..63)
__global__ void expand_ring(const char* __restrict__ p, int64_t rows, int nslot, int slot_bytes, int dsplit,
                            double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (int64_t)slot_bytes * nslot);
  uint64_t* empty = full + nslot;
  const int ncw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslot; ++i) {
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sa(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sa(&empty[i])), "r"(ncw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t items = rows / 64;
  const int64_t j0 = items * blockIdx.x / gridDim.x, j1 = items * (blockIdx.x + 1) / gridDim.x;
  const int64_t upanel = rows * 384, dbase = 9 * upanel;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = 9 + dsplit;
  int slot = 0;
  uint32_t phase = 0;
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int64_t j = j0; j < j1; ++j)
        for (int st = 0; st < nst; ++st) {
          asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&empty[slot])), "r"(phase ^ 1));
          const char* src;
          int n;
          if (st < 9) { src = p + st * upanel + j * 64 * 384; n = 64 * 384; }
          else { n = 64 * 512 / dsplit; src = p + dbase + j * 64 * 512 + (st - 9) * n; }
          asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(&full[slot])), "r"(n));
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(sa(smem + (int64_t)slot * slot_bytes)), "l"(src), "r"(n), "r"(sa(&full[slot])), "l"(pol) : "memory");
          if (++slot == nslot) { slot = 0; phase ^= 1; }
        }
    }
    return;
  }
  double acc = 0;
  for (int64_t j = j0; j < j1; ++j)
    for (int st = 0; st < nst; ++st) {
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra W;}" ::"r"(sa(&full[slot])), "r"(phase));
      const double2* s2 = reinterpret_cast<const double2*>(smem + (int64_t)slot * slot_bytes);
      const int n16 = (st < 9 ? 64 * 384 : 64 * 512 / dsplit) / 16;
      double2 a2 = make_double2(0, 0);
      for (int i = threadIdx.x - 32; i < n16; i += blockDim.x - 32) { double2 v = s2[i]; a2.x = fma(v.x, 1.0001, a2.x); a2.y = fma(v.y, 0.9999, a2.y); }
      acc += a2.x + a2.y;
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(sa(&empty[slot])));
      if (++slot == nslot) { slot = 0; phase ^= 1; }
    }
  if (acc == 123.456) out[0] = acc;
}

int main(int argc, char** argv) {
  if (argc > 2) g_sustain = atoi(argv[2]);
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int64_t bytes = 16ll << 30;  // 16 GiB, ~130x L2
  char* p;
  double* out;
  CK(cudaMalloc(&p, bytes));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(p, 0, bytes));
  const bool rnd = argc > 1;
  if (rnd) { fill_random<<<4096, 256>>>((uint64_t*)p, bytes / 8); CK(cudaDeviceSynchronize()); }
  printf("data: %s\n", rnd ? "random doubles" : "zeros");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_it = [&](auto launch, const char* name) {
    launch();
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // sustained: 100 back-to-back launches (~0.2 s, long enough for the power cap to act)
    cudaEventRecord(e0);
    for (int rep = 0; rep < g_sustain; ++rep) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms_all;
    cudaEventElapsedTime(&ms_all, e0, e1);
    cudaError_t e = cudaGetLastError();
    printf("%-48s burst %8.1f GB/s  sustained %8.1f GB/s %s\n", name, bytes / (best * 1e-3) / 1e9,
           (double)g_sustain * bytes / (ms_all * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  char name[128];
  if (g_sustain <= 100)
  for (int bpsm : {2, 4, 8})
    for (int th : {256, 512, 1024}) {
      if (bpsm * th > 2048) continue;
      snprintf(name, sizeof name, "ldg128 unroll8 grid=%dx%d thr=%d", nsm, bpsm, th);
      time_it([&] { ldg128<<<nsm * bpsm, th>>>((const double2*)p, bytes / 16, out); }, name);
    }
  if (g_sustain <= 100)
  for (int bpsm : {2, 4})
    for (int th : {256, 512}) {
      snprintf(name, sizeof name, "ldg256 unroll4 grid=%dx%d thr=%d", nsm, bpsm, th);
      time_it([&] { ldg256<<<nsm * bpsm, th>>>((const double*)p, bytes / 32, out); }, name);
    }
  CK(cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  double* xv;
  CK(cudaMalloc(&xv, bytes / 48 + 4096));  // one double per 384 B row
  CK(cudaMemset(xv, 0, bytes / 48 + 4096));
  struct Cfg { int stage_kb, nstage, cta_per_sm, xmode, nlev; };
  if (argc > 3 && std::string(argv[3]) == "expand") {
    CK(cudaFuncSetAttribute(expand_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const int64_t rows = 1ll << 24;  // 9 x 6.44 GB + 8.6 GB: the c4 expand stream
    CK(cudaFree(p));
    const int64_t big = rows * (9 * 384 + 512);
    CK(cudaMalloc(&p, big));
    fill_random<<<4096, 256>>>((uint64_t*)p, big / 8);
    CK(cudaDeviceSynchronize());
    struct E { int nslot, slot_kb, dsplit; };
    for (E c : std::vector<E>{{3, 33, 1}, {2, 33, 1}, {4, 25, 2}, {3, 25, 2}, {2, 32, 1}, {5, 17, 4}}) {
      const int sb = c.slot_kb * 1024;
      const int smem = sb * c.nslot + 16 * c.nslot;
      if ((smem + 1024) * 2 > 228 * 1024) continue;
      snprintf(name, sizeof name, "expand ring %d slots x %d KB, D in %d", c.nslot, c.slot_kb, c.dsplit);
      const int64_t tot = rows * (9 * 384 + 512);
      auto launch = [&] { expand_ring<<<nsm * 2, 288, smem>>>(p, rows, c.nslot, sb, c.dsplit, out); };
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int rep = 0; rep < 20; ++rep) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t er = cudaGetLastError();
      printf("%-48s sustained %8.1f GB/s (%.3f ms) %s\n", name, 20.0 * tot / (ms * 1e-3) / 1e9, ms / 20,
             er == cudaSuccess ? "" : cudaGetErrorString(er));
    }
    return 0;
  }
  if (argc > 3) {
    // TLB reach: the same 16 GiB of reads, spread over a 126 GB allocation (9 "levels" 14 GB apart)
    CK(cudaFree(p));
    const int64_t big = 126ll << 30;
    CK(cudaMalloc(&p, big));
    fill_random<<<4096, 256>>>((uint64_t*)p, big / 8);
    CK(cudaDeviceSynchronize());
    for (int inter : {0, 1}) {
      snprintf(name, sizeof name, "SPREAD 126GB 24KBx%d lev=9 inter=%d", inter ? 3 : 2, inter);
      const int ns = inter ? 3 : 2;
      time_it([&] { bulk_ring<<<nsm * 2, 288, 24576 * ns + 16 * ns + 1024 * ns>>>(p, bytes, 24576, ns, out, 1, xv, 0, 9, inter, 14ll << 30); }, name);
    }
    return 0;
  }
  struct Cfg2 { int stage_kb, nstage, cta_per_sm, xmode, nlev, inter; };
  for (Cfg2 c : std::vector<Cfg2>{{24, 2, 2, 1, 9, 0}, {24, 2, 2, 0, 10, 1}, {24, 3, 2, 0, 10, 1}, {32, 3, 2, 0, 10, 1},
                                  {16, 3, 2, 0, 10, 1}, {16, 4, 2, 0, 10, 1}, {24, 2, 2, 0, 3, 1}, {16, 3, 2, 1, 9, 0}}) {
    const int sb = c.stage_kb * 1024;
    const int smem = sb * c.nstage + 16 * c.nstage + 1024 * c.nstage;
    if ((smem + 1024) * c.cta_per_sm > 228 * 1024) continue;
    snprintf(name, sizeof name, "bulk ring %dKBx%d, %d CTA/SM, x=%d lev=%d inter=%d", c.stage_kb, c.nstage, c.cta_per_sm, c.xmode, c.nlev, c.inter);
    time_it([&] { bulk_ring<<<nsm * c.cta_per_sm, 288, smem>>>(p, bytes, sb, c.nstage, out, 1, xv, c.xmode, c.nlev, c.inter); }, name);
  }
  return 0;
}
