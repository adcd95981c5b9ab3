// stl_fused_gemm.cu — slice GEMM with the decode fused into the epilogue (t = 4).
//
// Computes  Y[I*4 + a, J*4 + b] = sum_p dec[p][4a + b] * (A_p . B_p)[I, J]
// i.e. decode_tiles(_slice_products(x_enc, w_enc), d) (snf_operator.py:88-116) for the forward,
// and untile(g_u @ e_x) (toy_network.py:103,105) for the backward, without the fp32 slice
// products ever leaving L2.
//
// Schedule: CTA pairs (cta_group::2, see sm100_pair_pipeline.cuh) walk tiles in block-major,
// slice-minor order (tile = block * r + p), so the r slice tiles of one 256 x 256 output block
// run at the same time on r different pairs. Per tile, the 8 epilogue warps of each CTA
//   1. drain their 128 TMEM lanes (fp32) into an L2-resident scratch ring slot of the block
//      (and optionally into the forward cache planes), then free the TMEM buffer so the MMA
//      warp proceeds with the next tile;
//   2. publish the slice (per-block counter), wait until all r slices of the block are in L2;
//   3. decode 1/(2r) of the block: each thread reads r fp32 values per 4x4 tile from L2
//      (ld.global.cg) and applies the r x 16 decoder with FFMA, writing the output tile rows.
// Scratch slots are recycled only after every chunk of the block that used them is decoded.
// All waits are bounded (trap after 10 s), and the grid never exceeds one CTA per SM.
#include "sm100_pair_pipeline.cuh"
#include <cstdlib>
#include "stl_internal.h"

namespace stl {
namespace {

constexpr int kFBN = 256;           // N tile (J tiles per block)
constexpr int kFStages = 6;
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kFThreads = 128 + kEpiThreads;
constexpr int kBlockQuads = 256 * (kFBN / 4);  // 4-tile quads per output block
constexpr int kDecChunk = 8;

struct FusedArgs {
  int r, M, N, K;          // slice GEMM dims: M = I tiles, N = J tiles, K = contraction tiles
  const float* dec;        // r x 16 decoder
  void* y;                 // (4M) x (4N) output, leading dim ldy
  int64_t ldy;
  int y_bf16;
  void* cache;             // optional (r, M, N) planes copy of the slice products
  int cache_bf16;
  float* scratch;          // nslot x r x 256 x 256 fp32
  unsigned* written;       // per-block: CTA drains completed (target 2r)
  unsigned* decoded;       // per-block: decode chunks completed (target 2r)
  int nslot;
};

using FL = pair::Layout<kFBN, kFStages>;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
  if (ld_acquire(p) >= target) return;
  const uint64_t t0 = ptx::globaltimer_ns();
  while (ld_acquire(p) < target) {
    __nanosleep(128);
    if (ptx::globaltimer_ns() - t0 > 10000000000ull) __trap();
  }
}
__device__ __forceinline__ float4 ld_cg4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_cg4(float* p, float a, float b, float c, float d) {
  asm volatile("st.global.cg.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}
__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

template <typename T>
__device__ __forceinline__ void store16(T* dst, const float (&v)[16]);
template <>
__device__ __forceinline__ void store16<float>(float* dst, const float (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<float4*>(dst + 4 * i) =
        make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
template <>
__device__ __forceinline__ void store16<__nv_bfloat16>(__nv_bfloat16* dst, const float (&v)[16]) {
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
}

// Decode one 4-tile quad (row I, tiles J0..J0+3) of a block whose r slices sit in `slot`.
template <typename Ty>
__device__ __forceinline__ void decode_quad(const float* __restrict__ slot, int r, int rl,
                                            int jq, const float* __restrict__ sdec, Ty* dst,
                                            int64_t ldy) {
  float acc[4][16];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[t][c] = 0.f;
  const float* base = slot + static_cast<size_t>(rl) * kFBN + jq * 4;
  for (int p0 = 0; p0 < r; p0 += kDecChunk) {
    float4 v[kDecChunk];
#pragma unroll
    for (int j = 0; j < kDecChunk; ++j)
      v[j] = (p0 + j < r) ? ld_cg4(base + static_cast<size_t>(p0 + j) * 256 * kFBN)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < kDecChunk; ++j) {
      if (p0 + j >= r) break;
      const float vt[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
      const float4* cp = reinterpret_cast<const float4*>(sdec + (p0 + j) * 16);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 c4 = cp[i];
        const float cf[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int t = 0; t < 4; ++t) acc[t][4 * i + jj] = fmaf(cf[jj], vt[t], acc[t][4 * i + jj]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    float row[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) row[e] = acc[e >> 2][a * 4 + (e & 3)];
    store16(dst + a * ldy, row);
  }
}

template <bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kFThreads, 1)
    fused_gemm_decode_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB, FusedArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kFStages * FL::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FL::kRingBytes);
  uint64_t* empty = full + kFStages;
  uint64_t* tfull = empty + kFStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* sdec = reinterpret_cast<float*>(smem + FL::kRingBytes + FL::kBarBytes);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int r = args.r, M = args.M, N = args.N;
  const int m_tiles = (M + 255) / 256, n_tiles = (N + kFBN - 1) / kFBN;
  const int nblocks = m_tiles * n_tiles;
  const int total = nblocks * r;
  const int num_kb = (args.K + pair::kBK - 1) / pair::kBK;
  auto map = [=](int tile) {
    const int b = tile / r;
    return pair::TileCoord{tile - b * r, b / n_tiles, b - (b / n_tiles) * n_tiles};
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kFStages; ++s) {
      ptx::mbar_init(&full[s], 2);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 2 * kEpiWarps);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, 512);
  for (int i = threadIdx.x; i < r * 16; i += kFThreads) sdec[i] = args.dec[i];
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0)
      pair::produce<kFBN, kFStages, false, B_MN>(&tmA, &tmB, sA, sB, full, empty, rank, cluster,
                                                 nclusters, total, num_kb, map);
  } else if (warp == 1) {
    if (lane == 0 && rank == 0)
      pair::mma_loop<kFBN, kFStages, false, B_MN>(sA, sB, full, empty, tfull, tempty, tmem_base,
                                                  cluster, nclusters, total, num_kb);
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ epilogue
    const int ew = warp - 4;             // 0..7
    const int q = warp & 3;              // TMEM lane quadrant
    const int half = ew >> 2;            // column half of the 256-wide accumulator
    const int etid = threadIdx.x - 128;  // 0..255
    const unsigned target = 2u * static_cast<unsigned>(r);
    const size_t slot_elems = static_cast<size_t>(r) * 256 * kFBN;
    int it = 0;
    for (int tile = cluster; tile < total; tile += nclusters, ++it) {
      const pair::TileCoord tc = map(tile);
      const int b = tile / r;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      float* slot = args.scratch + static_cast<size_t>(b % args.nslot) * slot_elems;
      // Slot reuse guard: the block that last used this slot must be fully decoded.
      if (b >= args.nslot) {
        if (etid == 0) wait_count(&args.decoded[b - args.nslot], target);
        epi_bar();
      }
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      // 1. drain TMEM -> scratch (fp32) [+ cache planes]
      const int rl = static_cast<int>(rank) * 128 + q * 32 + lane;  // row within block
      float* srow = slot + (static_cast<size_t>(tc.p) * 256 + rl) * kFBN + half * 128;
      const int grow = tc.mb * 256 + rl;
      const int gcol0 = tc.nb * kFBN + half * 128;
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        uint32_t v[32];
        __syncwarp();
        ptx::tmem_ld_32x32b_x32(
            tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * kFBN + half * 128 + c, v);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          st_cg4(srow + c + 4 * i, __uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                 __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        if (args.cache != nullptr && grow < M) {
          const size_t off = (static_cast<size_t>(tc.p) * M + grow) * N + gcol0 + c;
          const int ncol = N - (gcol0 + c);
          if (ncol > 0) {
            if (args.cache_bf16) {
              __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(args.cache) + off;
              if (ncol >= 32 && (N & 7) == 0) {
                float tmp[16];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                  for (int e = 0; e < 16; ++e) tmp[e] = __uint_as_float(v[16 * h + e]);
                  store16(d + 16 * h, tmp);
                }
              } else {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                  if (e < ncol) d[e] = __float2bfloat16_rn(__uint_as_float(v[e]));
              }
            } else {
              float* d = reinterpret_cast<float*>(args.cache) + off;
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e < ncol) d[e] = __uint_as_float(v[e]);
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0));
      // 2. publish this CTA's half of slice p, then wait for the whole block
      __threadfence();
      epi_bar();
      if (etid == 0) {
        atomicAdd(&args.written[b], 1u);
        wait_count(&args.written[b], target);
      }
      epi_bar();
      // 3. decode chunk (2p + rank) of 2r
      const int chunk = 2 * tc.p + static_cast<int>(rank);
      const int q_lo = static_cast<int>((static_cast<int64_t>(chunk) * kBlockQuads) / (2 * r));
      const int q_hi = static_cast<int>((static_cast<int64_t>(chunk + 1) * kBlockQuads) / (2 * r));
      for (int qi = q_lo + etid; qi < q_hi; qi += kEpiThreads) {
        const int brl = qi / (kFBN / 4), jq = qi - brl * (kFBN / 4);
        const int I = tc.mb * 256 + brl, J0 = tc.nb * kFBN + jq * 4;
        if (I >= M || J0 >= N) continue;
        const int64_t yoff = static_cast<int64_t>(I) * 4 * args.ldy + static_cast<int64_t>(J0) * 4;
        if (args.y_bf16)
          decode_quad(slot, r, brl, jq, sdec, reinterpret_cast<__nv_bfloat16*>(args.y) + yoff,
                      args.ldy);
        else
          decode_quad(slot, r, brl, jq, sdec, reinterpret_cast<float*>(args.y) + yoff, args.ldy);
      }
      epi_bar();
      if (etid == 0) {
        __threadfence();
        atomicAdd(&args.decoded[b], 1u);
      }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_2sm(tmem_base, 512);
}

constexpr size_t kCounterBytes(int nblocks) { return ((size_t(2) * nblocks * 4) + 255) / 256 * 256; }

int fused_nslot(int r, int nblocks) {
  // slices in flight span ~2 rounds of tiles; keep a few blocks of slack
  int n = (2 * (sm_count() / 2) + r - 1) / r + 3;
  return n < nblocks ? n : nblocks;
}

}  // namespace

bool fused_decode_supported(int t, int r, int64_t M, int64_t N, int64_t K, int ab_dtype,
                            const void* a, const void* b, int b_layout) {
  if (t != 4 || ab_dtype != kBF16 || r < 1 || r > kMaxRank) return false;
  if (M <= 128 || N % 4 || K % 8 || (b_layout ? N % 8 : 0)) return false;
  if ((reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(b) & 15)) return false;
  return M < (1 << 30) && N < (1 << 30) && K < (1 << 30);
}

size_t fused_decode_scratch_bytes(int r, int64_t M, int64_t N) {
  const int nblocks = static_cast<int>(((M + 255) / 256) * ((N + kFBN - 1) / kFBN));
  return kCounterBytes(nblocks) +
         size_t(fused_nslot(r, nblocks)) * r * 256 * kFBN * sizeof(float);
}

cudaError_t fused_gemm_decode(const void* a, const void* b, int b_layout, int r, int64_t M,
                              int64_t N, int64_t K, const float* dec, void* y, int64_t ldy,
                              int y_dtype, void* cache, int cache_dtype, void* scratch,
                              cudaStream_t s) {
  const int nblocks = static_cast<int>(((M + 255) / 256) * ((N + kFBN - 1) / kFBN));
  unsigned* counters = static_cast<unsigned*>(scratch);
  cudaError_t e = cudaMemsetAsync(counters, 0, kCounterBytes(nblocks), s);
  if (e != cudaSuccess) return e;
  CUtensorMap ta, tb;
  bool ok = make_bf16_tmap(&ta, a, K, M, r, pair::kBK, 128);
  ok = ok && (b_layout ? make_bf16_tmap(&tb, b, N, K, r, pair::kBK, 64)
                       : make_bf16_tmap(&tb, b, K, N, r, pair::kBK, kFBN / 2));
  if (!ok) return cudaErrorInvalidValue;
  FusedArgs fa{};
  fa.r = r;
  fa.M = static_cast<int>(M);
  fa.N = static_cast<int>(N);
  fa.K = static_cast<int>(K);
  fa.dec = dec;
  fa.y = y;
  fa.ldy = ldy;
  fa.y_bf16 = y_dtype == kBF16;
  fa.cache = cache;
  fa.cache_bf16 = cache_dtype == kBF16;
  fa.written = counters;
  fa.decoded = counters + nblocks;
  fa.scratch = reinterpret_cast<float*>(static_cast<uint8_t*>(scratch) + kCounterBytes(nblocks));
  fa.nslot = fused_nslot(r, nblocks);
  const int smem = FL::kRingBytes + FL::kBarBytes + kMaxRank * 16 * 4 + 1024;
  const int64_t tiles = static_cast<int64_t>(nblocks) * r;
  int pairs = sm_count() / 2;
  static const int env_pairs = [] {
    const char* e = getenv("STL_FUSED_PAIRS");
    return e ? atoi(e) : 0;
  }();
  if (env_pairs > 0 && env_pairs < pairs) pairs = env_pairs;
  const int grid = 2 * static_cast<int>(tiles < pairs ? tiles : pairs);
  if (b_layout) {
    auto k = fused_gemm_decode_kernel<true>;
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    k<<<grid, kFThreads, smem, s>>>(ta, tb, fa);
  } else {
    auto k = fused_gemm_decode_kernel<false>;
    if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    k<<<grid, kFThreads, smem, s>>>(ta, tb, fa);
  }
  return cudaGetLastError();
}

}  // namespace stl
