// Bandwidth probe (measurement aid, not product code): copy `bytes` from src to dst with
// (0) vectorised LDG/STG grid-stride, (1) cp.async.bulk 16 KB chunks through shared memory with
// a 4-deep pipeline per CTA (one CTA per SM), reporting what each path sustains on this B200.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_ldg(const uint4* __restrict__ s, uint4* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CHUNK, int NST>
__global__ void __launch_bounds__(32) k_bulk(const uint8_t* __restrict__ s, uint8_t* __restrict__ d, int64_t nchunks) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[NST];
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t it = 0;
  int64_t first = blockIdx.x;
  // prologue
  for (int k = 0; k < NST; ++k) {
    int64_t c = first + k * (int64_t)gridDim.x;
    if (c >= nchunks) break;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[k])), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su(sm + k * CHUNK)), "l"(s + c * CHUNK), "r"(CHUNK), "r"(su(&bar[k])) : "memory");
  }
  for (int64_t c = first; c < nchunks; c += gridDim.x, ++it) {
    const int st = it % NST;
    const uint32_t ph = (it / NST) & 1;
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su(&bar[st])), "r"(ph) : "memory");
    }
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + c * CHUNK), "r"(su(sm + st * CHUNK)), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    int64_t nc = c + NST * (int64_t)gridDim.x;
    if (nc < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su(sm + st * CHUNK)), "l"(s + nc * CHUNK), "r"(CHUNK), "r"(su(&bar[st])) : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

extern "C" int probe_copy(int mode, const void* src, void* dst, int64_t bytes, int sms, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) {
    k_ldg<<<sms * 8, 256, 0, s>>>((const uint4*)src, (uint4*)dst, bytes / 16);
  } else {
    constexpr int CH = 32768, NST = 6;
    auto k = k_bulk<CH, NST>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * NST);
    k<<<sms * (mode == 2 ? 2 : 1), 32, CH * NST, s>>>((const uint8_t*)src, (uint8_t*)dst, bytes / CH);
  }
  return (int)cudaGetLastError();
}
