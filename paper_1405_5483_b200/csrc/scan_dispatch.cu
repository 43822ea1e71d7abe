// Kernel-family dispatch, the SMAG prepare kernel and launch bookkeeping.
#include <atomic>
#include <mutex>
#include <map>
#include <utility>

#include "kern_common.cuh"

namespace magb {
namespace {

std::atomic<unsigned long long> g_launches{0};

// The search's gather grid: one warp per CTA, launched as a programmatic
// dependent of the scan so it runs beside it (kern_common.cuh
// gather_warp_run).  The last gather warp of the final launch waits for the
// scan grid to complete (its candidate counts), then publishes the counters
// to the mapped host words and clears the next search's control words.
__global__ void __launch_bounds__(32, 16) mag_gather_kernel(const __grid_constant__ ScanArgs A) {
  const int lane = threadIdx.x & 31;
  gather_warp_run(A, lane);
  unsigned long long old = 0;
  if (lane == 0) {
    fence_release();
    old = atomicAdd(A.exits, 1ull);
  }
  old = __shfl_sync(kFull, old, 0);
  if (old + 1 != gridDim.x || !A.final_launch) return;
  if (lane == 0) diag_time(A, 3);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  fence_gpu();
  if (lane < 3) {
    const unsigned src = lane == 0 ? kCtrCands : (lane == 1 ? kCtrTotal : kCtrMax);
    const unsigned long long v = ld_gpu(reinterpret_cast<const uint64_t*>(A.counters) + src);
    reinterpret_cast<volatile unsigned long long*>(A.host_ctr)[1 + lane] = v;
  }
  if ((A.plan.diag & 2048) && lane < 4) {  // diagnostics timeline, ns after the first scan CTA started
    const uint64_t t0 = ~ld_gpu(reinterpret_cast<const uint64_t*>(A.counters) + kCtrTime);
    const uint64_t t = lane == 3 ? ld_gpu(reinterpret_cast<const uint64_t*>(A.counters) + kCtrTime + 4)
                                 : ld_gpu(reinterpret_cast<const uint64_t*>(A.counters) + kCtrTime + 1 + lane);
    reinterpret_cast<volatile unsigned long long*>(A.host_ctr)[4 + lane] = t - t0;
  }
  for (uint32_t i = lane; i < A.reset_words; i += 32) A.reset[i] = 0;
  __threadfence_system();
}

// SMAG prepare (encode_text qgram.cpp:29-37) on the device.
__global__ void mag_encode_kernel(const ScanPlan P, const uint8_t* __restrict__ text, uint64_t nq,
                                  const uint8_t* __restrict__ map, uint32_t* __restrict__ codes) {
  __shared__ uint8_t smap[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) smap[i] = map ? map[i] : 0;
  __syncthreads();
  const uint32_t q = P.q;
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nq; u += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t* g = text + u * q;
    uint32_t v;
    if (P.gram_mode == kGramExact) {
      v = smap[g[q - 1]];
      for (int i = static_cast<int>(q) - 2; i >= 0; --i) v = v * P.sigma_prime + smap[g[i]];
    } else {
      uint32_t x[4] = {0, 0, 0, 0};
      for (uint32_t i = 0; i < q; ++i) x[i >> 2] |= static_cast<uint32_t>(g[i]) << (8 * (i & 3));
      v = gram_slot(hash_gram_words(x[0], x[1], x[2], x[3]), P.table_bits);
    }
    codes[u] = v;
  }
}

}  // namespace

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

unsigned long long kernel_launch_count() { return g_launches.load(); }

cudaError_t allow_max_smem(const void* kernel, size_t need) {
  // The limit only ever grows to what a launch needs (not the device's
  // opt-in maximum): the driver sizes the shared-memory carveout, hence what
  // is left for L1, from it.
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = set[{kernel, dev}];
  if (cur >= need) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(need));
  if (e != cudaSuccess) return e;
  cur = need;
  return cudaSuccess;
}

namespace {
cudaError_t launch_scan_only(const ScanArgs& a, cudaStream_t stream, int grid) {
  if (a.plan.direct) return launch_direct(a, stream, grid);
  if (a.plan.roll) return launch_roll(a, stream, grid);
  if (a.plan.smag) return launch_staged_codes(a, stream, grid);
  if (a.plan.gram_mode == kGramHashed) return launch_staged_hashed(a, stream, grid);
  return launch_staged_exact(a, stream, grid);
}
}  // namespace

cudaError_t launch_scan(const ScanArgs& a, cudaStream_t stream, int grid) {
  cudaError_t e = launch_scan_only(a, stream, grid);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, mag_gather_kernel, a);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_encode(const ScanPlan& plan, const uint8_t* text, uint64_t n, const uint8_t* map,
                          uint32_t* codes, cudaStream_t stream) {
  const uint64_t nq = n / plan.q;
  if (nq == 0) return cudaSuccess;
  const int threads = 256;
  uint64_t blocks = (nq + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  (void)cudaGetLastError();
  mag_encode_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(plan, text, nq, map, codes);
  count_launch();
  return cudaGetLastError();
}

}  // namespace magb
