// stl_transform_mma.cu — t = 4 encode on the tensor cores (warp-level mma.sync), the fallback
// of the streaming encode (stl_stream.cu) for tile-column counts that are not multiples of 64
// (the T2T-ViT-7 layers).
//
// The per-tile change of basis is a GEMM with a tiny inner dimension:
//   encode  (encode_tiles, snf_operator.py:80-85):  C[tile][p] = sum_c X[tile][c] * E[p][c]
//   g_d (toy_network.py:100):                       R[p][c]   = sum_tiles Z[p][tile] * X[tile][c]
// On CUDA cores these cost r FMAs per element (~43 us of FFMA at 8192^2, as much as the HBM
// time), so they run as m16n8k16 bf16 MMAs with fp32 accumulation, leaving the kernels
// HBM-bound. Operands are loaded straight from global memory in fragment layout:
//   * X (bf16 activations): A-fragment element pairs (c = 2q, 2q+1) are two adjacent columns of
//     one tile row -> one 4-byte load, exact;
//   * fp32 operands (slice planes Z, the E/D coefficient matrices) are split into bf16 hi + lo
//     and both halves are multiplied (fp32-level accuracy, ~2^-16 relative);
//   * bf16 planes (the training cache y_enc) are exact in one MMA.
// One warp owns a row segment of 128 consecutive tiles (8 m-tiles of 16). Encode outputs are
// staged through shared memory per warp so every plane store is a coalesced 256/512-byte row.
// Reductions keep per-warp fragment accumulators, reduce warps in a fixed order into per-block
// partials, and a fixed-order tree sums the blocks -> deterministic.
#include "stl_internal.h"

namespace stl {
namespace {

constexpr int kWarpsM = 4;
constexpr int kThreadsM = 32 * kWarpsM;
constexpr int kTaskTiles = 128;   // tiles per warp task
constexpr int kMtPerTask = kTaskTiles / 16;

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}
// x (fp32 pair) -> hi, lo bf16x2 halves
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const float h0 = bf16_round(x0), h1 = bf16_round(x1);
  hi = pack2(h0, h1);
  lo = pack2(x0 - h0, x1 - h1);
}
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                    uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t ld_u32(const void* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}
__device__ __forceinline__ uint32_t ld_bf16_pair(const __nv_bfloat16* p0, const __nv_bfloat16* p1) {
  const uint32_t lo = *reinterpret_cast<const uint16_t*>(p0);
  const uint32_t hi = *reinterpret_cast<const uint16_t*>(p1);
  return lo | (hi << 16);
}

// ---------------------------------------------------------------------------------------------
// Reduction accumulator R[p][c] (p < 32, c < 16) as 2 x 2 m16n8 fragments per warp.
struct RedAcc {
  float acc[2][2][4];
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[i][j][k] = 0.f;
  }
  // One k-step over 16 tiles [jm, jm+16) of tile row I.
  //   A (M = p, K = tiles): planes Zp[p][tile] (bf16 exact, or fp32 split hi/lo)
  //   B (K = tiles, N = c): X tile values (bf16 matrix, exact)
  // K rows are permuted (k = 2q, 2q+1, 2q+8, 2q+9 <-> tiles 4q .. 4q+3; a consistent K
  // permutation of A and B leaves the product unchanged) so each thread's A elements are four
  // consecutive tiles of one plane: one 16-byte (fp32) or 8-byte (bf16) load.
  template <typename Tz>
  __device__ void step(const Tz* __restrict__ zrow, int64_t plane_stride, int P,
                       const __nv_bfloat16* __restrict__ xrow0, int64_t ldx) {
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    uint32_t b[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int c = 8 * nt + g;
      const __nv_bfloat16* xr = xrow0 + (c >> 2) * ldx + (c & 3) + 16 * q;
      b[nt][0] = ld_bf16_pair(xr, xr + 4);
      b[nt][1] = ld_bf16_pair(xr + 8, xr + 12);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      if (16 * mt >= P) break;
      const int p0 = 16 * mt + g, p1 = p0 + 8;
      if constexpr (sizeof(Tz) == 2) {
        uint2 u0 = make_uint2(0u, 0u), u1 = u0;
        if (p0 < P) u0 = *reinterpret_cast<const uint2*>(zrow + p0 * plane_stride + 4 * q);
        if (p1 < P) u1 = *reinterpret_cast<const uint2*>(zrow + p1 * plane_stride + 4 * q);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) mma(acc[mt][nt], u0.x, u1.x, u0.y, u1.y, b[nt][0], b[nt][1]);
      } else {
        float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
        if (p0 < P) v0 = *reinterpret_cast<const float4*>(zrow + p0 * plane_stride + 4 * q);
        if (p1 < P) v1 = *reinterpret_cast<const float4*>(zrow + p1 * plane_stride + 4 * q);
        uint32_t h0, l0, h1, l1, h2, l2, h3, l3;
        split2(v0.x, v0.y, h0, l0);  // a0: (p0, tiles 4q, 4q+1)
        split2(v1.x, v1.y, h1, l1);  // a1: (p1, tiles 4q, 4q+1)
        split2(v0.z, v0.w, h2, l2);  // a2: (p0, tiles 4q+2, 4q+3)
        split2(v1.z, v1.w, h3, l3);  // a3
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          mma(acc[mt][nt], h0, h1, h2, h3, b[nt][0], b[nt][1]);
          mma(acc[mt][nt], l0, l1, l2, l3, b[nt][0], b[nt][1]);
        }
      }
    }
  }
  // Fixed-order block reduction -> red_partial[blockIdx.x][P*16]. `sred` has kWarpsM*P*16 floats.
  __device__ void finish(float* sred, int P, float* __restrict__ red_partial) const {
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3, warp = threadIdx.x >> 5;
    float* mine = sred + warp * P * 16;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int c = 8 * nt + 2 * q, p0 = 16 * mt + g, p1 = p0 + 8;
        if (p0 < P) {
          mine[p0 * 16 + c] = acc[mt][nt][0];
          mine[p0 * 16 + c + 1] = acc[mt][nt][1];
        }
        if (p1 < P) {
          mine[p1 * 16 + c] = acc[mt][nt][2];
          mine[p1 * 16 + c + 1] = acc[mt][nt][3];
        }
      }
    __syncthreads();
    const int n = P * 16;
    for (int o = threadIdx.x; o < n; o += kThreadsM) {
      float s = sred[o];
#pragma unroll
      for (int w = 1; w < kWarpsM; ++w) s += sred[w * n + o];
      red_partial[static_cast<int64_t>(blockIdx.x) * n + o] = s;
    }
  }
};

// ---------------------------------------------------------------------------------------------
// encode: X (bf16) tiles -> P planes. RED: g_d += Zp (x) X over the same tiles.
template <typename Tout, bool RED, typename Tz>
__global__ void __launch_bounds__(kThreadsM)
    k_encode_mma(const __nv_bfloat16* __restrict__ x, int64_t ldx, int64_t br, int64_t bc,
                 const float* __restrict__ coef, int P, Tout* __restrict__ out,
                 const Tz* __restrict__ zred, float* __restrict__ red_partial) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int kStride = kTaskTiles + (sizeof(Tout) == 4 ? 4 : 8);  // padded staging row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int NT = (P + 7) >> 3;
  Tout* stage = reinterpret_cast<Tout*>(smem) + warp * (8 * NT) * kStride;
  float* sred = reinterpret_cast<float*>(smem + kWarpsM * (8 * NT) * kStride * sizeof(Tout));
  // E as B fragments (K = c, N = p): b0 = E[p][2q, 2q+1], b1 = E[p][2q+8, 2q+9], p = 8nt + g
  uint32_t bh[8][2], bl[8][2];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int p = 8 * nt + g;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = 2 * q + 8 * h;
      const float e0 = p < P ? coef[p * 16 + c] : 0.f, e1 = p < P ? coef[p * 16 + c + 1] : 0.f;
      split2(e0, e1, bh[nt][h], bl[nt][h]);
    }
  }
  RedAcc R;
  R.zero();
  const int64_t ntiles = br * bc;
  const int64_t tasks_per_row = (bc + kTaskTiles - 1) / kTaskTiles;
  const int64_t ntasks = br * tasks_per_row;
  for (int64_t task = static_cast<int64_t>(blockIdx.x) * kWarpsM + warp; task < ntasks;
       task += static_cast<int64_t>(gridDim.x) * kWarpsM) {
    const int64_t I = task / tasks_per_row;
    const int64_t J0 = (task - I * tasks_per_row) * kTaskTiles;
    const int64_t rem_mt = (bc - J0) >> 4;
    const int nmt = rem_mt < kMtPerTask ? static_cast<int>(rem_mt) : kMtPerTask;
    const __nv_bfloat16* xrow = x + I * 4 * ldx + J0 * 4;
    // A fragments for all m-tiles: a0 = X[tile g][c 2q..] (row q>>1, cols 2(q&1)..),
    // a1 = tile g+8, a2 = tile g rows 2+(q>>1), a3 = tile g+8 rows 2+(q>>1).
    uint32_t a[kMtPerTask][4];
#pragma unroll
    for (int mi = 0; mi < kMtPerTask; ++mi) {
      if (mi < nmt) {
        const __nv_bfloat16* base = xrow + (q >> 1) * ldx + (16 * mi + g) * 4 + 2 * (q & 1);
        a[mi][0] = ld_u32(base);
        a[mi][1] = ld_u32(base + 32);
        a[mi][2] = ld_u32(base + 2 * ldx);
        a[mi][3] = ld_u32(base + 2 * ldx + 32);
      } else {
        a[mi][0] = a[mi][1] = a[mi][2] = a[mi][3] = 0u;
      }
    }
#pragma unroll
    for (int mi = 0; mi < kMtPerTask; ++mi) {
      if (mi >= nmt) break;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        if (nt >= NT) break;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        mma(c, a[mi][0], a[mi][1], a[mi][2], a[mi][3], bh[nt][0], bh[nt][1]);
        mma(c, a[mi][0], a[mi][1], a[mi][2], a[mi][3], bl[nt][0], bl[nt][1]);
        // C[tile][p]: c0,c1 -> tile g, p = 8nt+2q (+1); c2,c3 -> tile g+8
        const int p = 8 * nt + 2 * q, t0 = 16 * mi + g;
        stage[p * kStride + t0] = static_cast<Tout>(c[0]);
        stage[(p + 1) * kStride + t0] = static_cast<Tout>(c[1]);
        stage[p * kStride + t0 + 8] = static_cast<Tout>(c[2]);
        stage[(p + 1) * kStride + t0 + 8] = static_cast<Tout>(c[3]);
      }
    }
    __syncwarp();
    // coalesced plane rows: lane writes tiles 4*lane .. 4*lane+3 of every plane
    const int tl = 4 * lane;
    if (tl < 16 * nmt) {
      Tout* dst = out + I * bc + J0 + tl;
      for (int p = 0; p < P; ++p) {
        const Tout* s = stage + p * kStride + tl;
        if constexpr (sizeof(Tout) == 2)
          *reinterpret_cast<uint2*>(dst + p * ntiles) = *reinterpret_cast<const uint2*>(s);
        else
          *reinterpret_cast<float4*>(dst + p * ntiles) = *reinterpret_cast<const float4*>(s);
      }
    }
    __syncwarp();
    if constexpr (RED) {
      const Tz* zrow = zred + I * bc + J0;
      for (int mi = 0; mi < nmt; ++mi)
        R.step(zrow + 16 * mi, ntiles, P, xrow + 16 * mi * 4, ldx);
    }
  }
  if constexpr (RED) R.finish(sred, P, red_partial);
}


int grid_m(int64_t ntasks, int cap) {
  int64_t g = (ntasks + kWarpsM - 1) / kWarpsM;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

template <typename K>
cudaError_t set_smem(K k, size_t smem) {
  if (smem <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename Tout, typename Tz, bool RED>
cudaError_t launch_enc(const void* m, int64_t ldm, int64_t br, int64_t bc, const float* coef,
                       int P, void* out, const void* rp, float* ro, float* rw, cudaStream_t s) {
  constexpr int kStride = kTaskTiles + (sizeof(Tout) == 4 ? 4 : 8);
  const size_t smem =
      kWarpsM * (8 * ((P + 7) / 8)) * kStride * sizeof(Tout) + (RED ? kWarpsM * P * 16 * 4 : 0);
  auto k = k_encode_mma<Tout, RED, Tz>;
  if (cudaError_t e = set_smem(k, smem)) return e;
  const int64_t ntasks = br * ((bc + kTaskTiles - 1) / kTaskTiles);
  const int grid = grid_m(ntasks, sm_count() * (RED ? 4 : 8));
  k<<<grid, kThreadsM, smem, s>>>(static_cast<const __nv_bfloat16*>(m), ldm, br, bc, coef, P,
                                  static_cast<Tout*>(out), static_cast<const Tz*>(rp), rw);
  if (RED) return sum_partials(rw, grid, P * 16, ro, s);
  return cudaGetLastError();
}

}  // namespace

// Tensor-core encode: bf16 X, t = 4, bc % 16 == 0. Returns cudaErrorNotSupported otherwise.
cudaError_t tiles_to_planes_mma(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                                const float* coef, int P, void* out, int odt, const void* rp,
                                int rdt, float* ro, float* rw, cudaStream_t s) {
  if (mdt != kBF16 || bc % 16 || ldm % 8 || P > 64 || !al16(m) || !al16(out))
    return cudaErrorNotSupported;
  if (rp && (P > 32 || !al16(rp))) return cudaErrorNotSupported;
  if (odt == kBF16) {
    if (!rp) return launch_enc<__nv_bfloat16, float, false>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
    if (rdt == kBF16)
      return launch_enc<__nv_bfloat16, __nv_bfloat16, true>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
    return launch_enc<__nv_bfloat16, float, true>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
  }
  if (!rp) return launch_enc<float, float, false>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
  if (rdt == kBF16)
    return launch_enc<float, __nv_bfloat16, true>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
  return launch_enc<float, float, true>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
}

}  // namespace stl
