// Data-movement floor of the streaming tile transforms (measurement aid, not product code).
//
// A unit reads n_in segments of s_in bytes and writes n_out segments of s_out bytes with 1-D
// cp.async.bulk copies through a per-CTA shared-memory ring (one thread drives the pipeline:
// loads run NST-1 units ahead, stores are bulk groups). Segment addressing:
//   kind 0 ("rows"):   segment a of unit u at base + (n_seg * (u / upr) + a) * row_bytes + (u % upr) * s
//                      (the 4 matrix rows of a tile row: X for encode, Y for decode)
//   kind 1 ("planes"): segment p of unit u at base + p * plane_bytes + u * s
//                      (r plane segments, contiguous along the unit index)
// Reports achieved GB/s of (in + out) bytes. Built by scripts/probes/pattern_probe.py.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

struct Pat {
  int kind, nseg;
  int64_t s, upr, row_bytes, plane_bytes;
};

__device__ __forceinline__ const uint8_t* seg_addr(const uint8_t* base, const Pat& p, int64_t u, int a) {
  if (p.kind == 0) return base + (p.nseg * (u / p.upr) + a) * p.row_bytes + (u % p.upr) * p.s;
  return base + a * p.plane_bytes + u * p.s;
}

__global__ void __launch_bounds__(32) k_pattern(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                Pat pin, Pat pout, int64_t nunits, int nst,
                                                uint32_t stage_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[32];
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t in_bytes = (uint32_t)(pin.nseg * pin.s);
  auto load = [&](int64_t u, int st) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(in_bytes));
    for (int a = 0; a < pin.nseg; ++a)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su(sm + st * stage_bytes + a * pin.s)), "l"(seg_addr(src, pin, u, a)),
                   "r"((uint32_t)pin.s), "r"(su(&bar[st])) : "memory");
  };
  // ring of nst stages: loads run L = nst - D units ahead, D store groups stay in flight
  const int D = nst / 2, L = nst - D;
  int64_t it = 0;
  for (int k = 0; k < L; ++k) {
    const int64_t u = blockIdx.x + k * (int64_t)gridDim.x;
    if (u < nunits) load(u, k);
  }
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
    const int st = (int)(it % nst);
    const uint32_t ph = (uint32_t)((it / nst) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su(&bar[st])), "r"(ph) : "memory");
    for (int a = 0; a < pout.nseg; ++a)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   ::"l"(seg_addr(dst, pout, u, a)), "r"(su(sm + st * stage_bytes + a * pout.s)),
                   "r"((uint32_t)pout.s) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // unit it + L goes into the stage of unit it - D: its stores must have read it
    switch (D) {
      case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
      case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
      case 3: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
      case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
      case 5: asm volatile("cp.async.bulk.wait_group.read 5;" ::: "memory"); break;
      case 6: asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory"); break;
      case 7: asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory"); break;
      default: asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory"); break;
    }
    const int64_t nu = u + L * (int64_t)gridDim.x;
    if (nu < nunits) load(nu, (int)((it + L) % nst));
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

extern "C" int probe_pattern(const void* src, void* dst, int in_kind, int in_nseg, int64_t in_s,
                             int64_t in_upr, int64_t in_row, int64_t in_plane, int out_kind,
                             int out_nseg, int64_t out_s, int64_t out_upr, int64_t out_row,
                             int64_t out_plane, int64_t nunits, int grid, int nst, void* stream) {
  Pat pin{in_kind, in_nseg, in_s, in_upr, in_row, in_plane};
  Pat pout{out_kind, out_nseg, out_s, out_upr, out_row, out_plane};
  int64_t ib = in_nseg * in_s, ob = out_nseg * out_s;
  uint32_t stage = (uint32_t)(((ib > ob ? ib : ob) + 1023) / 1024 * 1024);
  if (nst > 32 || nst < 2 || (int64_t)stage * nst > 220 * 1024) return -1;
  cudaFuncSetAttribute(k_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, stage * nst);
  k_pattern<<<grid, 32, stage * nst, (cudaStream_t)stream>>>((const uint8_t*)src, (uint8_t*)dst, pin,
                                                             pout, nunits, nst, stage);
  return (int)cudaGetLastError();
}
