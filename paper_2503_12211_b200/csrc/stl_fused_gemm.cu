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
#include <cstdio>
#include <cstdlib>
#include "stl_internal.h"

namespace stl {
namespace {

constexpr int kFBN = 256;           // N tile (J tiles per block)
constexpr int kFStages = 6;
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kFThreads = 128 + kEpiThreads;

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
  unsigned long long* dbg;  // optional [grid][4] phase timers (ns): tfull wait, drain, block wait, decode
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
__device__ __forceinline__ void epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

template <typename T>
__device__ __forceinline__ void store16(T* dst, const float (&v)[16]);
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

__device__ __forceinline__ float ld_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Decoder as mma B fragments (K = p, N = c), split hi + lo bf16: thread (g, q) holds
// B[2q, 2q+1][g] and B[2q+8, 2q+9][g] of every 16-wide K step and 8-wide N tile.
constexpr int kMaxKs = kMaxRank / 16;
struct DecFrags {
  uint32_t hi[kMaxKs][2][2], lo[kMaxKs][2][2];
};
__device__ __forceinline__ void load_dec_frags(const float* sdec, int r, DecFrags& f) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int ks = 0; ks < kMaxKs; ++ks)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p0 = ks * 16 + 2 * q + 8 * h;
        const int c = nt * 8 + g;
        const float d0 = p0 < r ? sdec[p0 * 16 + c] : 0.f;
        const float d1 = p0 + 1 < r ? sdec[(p0 + 1) * 16 + c] : 0.f;
        const float h0 = __bfloat162float(__float2bfloat16_rn(d0));
        const float h1 = __bfloat162float(__float2bfloat16_rn(d1));
        f.hi[ks][nt][h] = pack2(h0, h1);
        f.lo[ks][nt][h] = pack2(d0 - h0, d1 - h1);
      }
}

// Decode 16 consecutive tiles (block row rl, tiles j0..j0+15) of a block whose r slices sit in
// `slot` (fp32 planes 256 x 256): out tile[c] = sum_p Z[p][tile] * dec[p][c] on the tensor
// cores (m16n8k16: M = tiles, K = p, N = c), Z split hi + lo bf16.
template <typename Ty>
__device__ __forceinline__ void decode_mtile(const float* __restrict__ slot, int r, int rl,
                                             int j0, const DecFrags& f, Ty* __restrict__ y,
                                             int64_t ldy, int I, int J0, int Nvalid) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  const float* base = slot + static_cast<size_t>(rl) * kFBN + j0 + g;
  const int nks = (r + 15) >> 4;
#pragma unroll
  for (int ks = 0; ks < kMaxKs; ++ks) {
    if (ks >= nks) break;
    float v[2][4];  // [tile g / g+8][p = 2q, 2q+1, 2q+8, 2q+9]
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int p = ks * 16 + 2 * q + (h & 1) + 8 * (h >> 1);
      const bool ok = p < r;
      const float* src = base + static_cast<size_t>(p) * 256 * kFBN;
      v[0][h] = ok ? ld_cg(src) : 0.f;
      v[1][h] = ok ? ld_cg(src + 8) : 0.f;
    }
    uint32_t ah[4], al[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      // a0 = (tile g, p 2q..), a1 = (tile g+8, p 2q..), a2 = (g, 2q+8..), a3 = (g+8, 2q+8..)
      const int t = i & 1, hh = (i >> 1) * 2;
      const float x0 = v[t][hh], x1 = v[t][hh + 1];
      const float h0 = __bfloat162float(__float2bfloat16_rn(x0));
      const float h1 = __bfloat162float(__float2bfloat16_rn(x1));
      ah[i] = pack2(h0, h1);
      al[i] = pack2(x0 - h0, x1 - h1);
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      mma16816(acc[nt], ah, f.hi[ks][nt][0], f.hi[ks][nt][1]);
      mma16816(acc[nt], al, f.hi[ks][nt][0], f.hi[ks][nt][1]);
      mma16816(acc[nt], ah, f.lo[ks][nt][0], f.lo[ks][nt][1]);
    }
  }
  // C[tile][c]: (acc[nt][0], [1]) -> tile g, c = 8nt + 2q (+1); ([2], [3]) -> tile g + 8.
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int a = 2 * nt + (q >> 1), b = 2 * (q & 1);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int J = J0 + g + 8 * t;
      if (J >= Nvalid) continue;
      Ty* dst = y + (static_cast<int64_t>(I) * 4 + a) * ldy + static_cast<int64_t>(J) * 4 + b;
      if constexpr (sizeof(Ty) == 2) {
        *reinterpret_cast<uint32_t*>(dst) = pack2(acc[nt][2 * t], acc[nt][2 * t + 1]);
      } else {
        *reinterpret_cast<float2*>(dst) = make_float2(acc[nt][2 * t], acc[nt][2 * t + 1]);
      }
    }
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
    DecFrags dfr;
    load_dec_frags(sdec, r, dfr);
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
      const uint64_t t_a = ptx::globaltimer_ns();
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint64_t t_b = ptx::globaltimer_ns();
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
          *reinterpret_cast<float4*>(srow + c + 4 * i) =
              make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
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
      //    (cooperative-groups grid-sync pattern: CTA barrier, one gpu-scope fence + atomic).
      epi_bar();
      const uint64_t t_c = ptx::globaltimer_ns();
      if (etid == 0) {
        __threadfence();
        atomicAdd(&args.written[b], 1u);
        wait_count(&args.written[b], target);
      }
      epi_bar();
      const uint64_t t_d = ptx::globaltimer_ns();
      // 3. decode m-tiles [mt_lo, mt_hi) of the block's 256 x (256/16) m-tiles (16 tiles each)
      const int chunk = 2 * tc.p + static_cast<int>(rank);
      constexpr int kBlockMt = 256 * (kFBN / 16);
      const int mt_lo = static_cast<int>((static_cast<int64_t>(chunk) * kBlockMt) / (2 * r));
      const int mt_hi = static_cast<int>((static_cast<int64_t>(chunk + 1) * kBlockMt) / (2 * r));
      for (int mt = mt_lo + ew; mt < mt_hi; mt += kEpiWarps) {
        const int brl = mt / (kFBN / 16), j0 = (mt - brl * (kFBN / 16)) * 16;
        const int I = tc.mb * 256 + brl, J0 = tc.nb * kFBN + j0;
        if (I >= M || J0 >= N) continue;
        if (args.y_bf16)
          decode_mtile(slot, r, brl, j0, dfr, reinterpret_cast<__nv_bfloat16*>(args.y), args.ldy,
                       I, J0, N);
        else
          decode_mtile(slot, r, brl, j0, dfr, reinterpret_cast<float*>(args.y), args.ldy, I, J0,
                       N);
      }
      epi_bar();
      if (etid == 0) {
        __threadfence();
        atomicAdd(&args.decoded[b], 1u);
        if (args.dbg) {
          unsigned long long* d = args.dbg + 4 * blockIdx.x;
          d[0] += t_b - t_a;
          d[1] += t_c - t_b;
          d[2] += t_d - t_c;
          d[3] += ptx::globaltimer_ns() - t_d;
        }
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
  static const bool dbg_on = getenv("STL_FUSED_DEBUG") != nullptr;
  static unsigned long long* dbg = nullptr;
  if (dbg_on && !dbg) cudaMalloc(&dbg, 4 * 4096 * sizeof(unsigned long long));
  if (dbg_on) cudaMemsetAsync(dbg, 0, 4 * 4096 * sizeof(unsigned long long), s);
  fa.dbg = dbg_on ? dbg : nullptr;
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
  if (dbg_on) {
    unsigned long long h[4 * 296] = {};
    cudaMemcpyAsync(h, dbg, sizeof(unsigned long long) * 4 * grid, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double sum[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
    for (int i = 0; i < grid; ++i)
      for (int j = 0; j < 4; ++j) {
        sum[j] += h[4 * i + j];
        mx[j] = mx[j] > h[4 * i + j] ? mx[j] : h[4 * i + j];
      }
    fprintf(stderr, "[fused dbg] grid=%d tiles/pair=%.1f  avg us: tfull_wait=%.1f drain=%.1f "
            "block_wait=%.1f decode=%.1f | max: %.1f %.1f %.1f %.1f\n", grid,
            double(tiles) / (grid / 2), sum[0] / grid / 1e3, sum[1] / grid / 1e3,
            sum[2] / grid / 1e3, sum[3] / grid / 1e3, mx[0] / 1e3, mx[1] / 1e3, mx[2] / 1e3,
            mx[3] / 1e3);
  }
  return cudaGetLastError();
}

}  // namespace stl
