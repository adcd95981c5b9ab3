// stl_transform_mma.cu — t = 4 tile transforms on the tensor cores (warp-level mma.sync).
//
// The per-tile change of basis is a GEMM with a tiny inner dimension:
//   encode  (encode_tiles, snf_operator.py:80-85):  C[tile][p] = sum_c X[tile][c] * E[p][c]
//   decode  (decode_tiles, snf_operator.py:88-96):  C[tile][c] = sum_p Z[p][tile] * D[p][c]
//   g_d / g_ex (toy_network.py:100,104):            R[p][c]   = sum_tiles Z[p][tile] * X[tile][c]
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

// ---------------------------------------------------------------------------------------------
// decode: Q planes (fp32 or bf16) -> tiles. RED: g_ex += Z (x) X' (X' = bf16 matrix).
template <typename Tz, typename Tout, bool RED, int KST>
__global__ void __launch_bounds__(kThreadsM)
    k_decode_mma(const Tz* __restrict__ z, int Q, int64_t br, int64_t bc,
                 const float* __restrict__ coef, Tout* __restrict__ out, int64_t ldo,
                 const __nv_bfloat16* __restrict__ xr, int64_t ldr, float* __restrict__ red_partial) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int kOutStride = 128 + (sizeof(Tout) == 2 ? 8 : 4);  // padded staged output row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  Tout* ostage = reinterpret_cast<Tout*>(smem) + warp * 4 * kOutStride;
  float* sred = reinterpret_cast<float*>(smem + kWarpsM * 4 * kOutStride * sizeof(Tout));
  // D as B fragments (K = p, N = c): b0 = D[16ks+2q, +1][c], b1 = D[16ks+2q+8, +9][c], c = 8nt+g
  uint32_t bh[KST][2][2], bl[KST][2][2];
#pragma unroll
  for (int ks = 0; ks < KST; ++ks)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 16 * ks + 2 * q + 8 * h, c = 8 * nt + g;
        const float d0 = p < Q ? coef[p * 16 + c] : 0.f;
        const float d1 = p + 1 < Q ? coef[(p + 1) * 16 + c] : 0.f;
        split2(d0, d1, bh[ks][nt][h], bl[ks][nt][h]);
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
    const Tz* zrow = z + I * bc + J0;
    // 32-tile groups; M rows permuted so thread (g, q) owns tiles 4g .. 4g+3 of the group:
    // m-tile A rows g, g+8 <-> tiles 4g, 4g+1; m-tile B rows g, g+8 <-> tiles 4g+2, 4g+3.
    const int ngroups = nmt >> 1;
    for (int gp = 0; gp < ngroups; gp += 2) {
      // issue the loads of two 32-tile groups before any math (memory-level parallelism)
      float vv[2][KST][4][4];  // [group][k-step][plane 2q, 2q+1, 2q+8, 2q+9][tile 4g + i]
#pragma unroll
      for (int gg = 0; gg < 2; ++gg) {
        const bool gok = gp + gg < ngroups;
        const Tz* zt = zrow + 32 * (gp + gg) + 4 * g;
#pragma unroll
        for (int ks = 0; ks < KST; ++ks)
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int p = 16 * ks + 2 * q + (h & 1) + 8 * (h >> 1);
            float* v = vv[gg][ks][h];
            if (gok && p < Q) {
              if constexpr (sizeof(Tz) == 2) {
                const uint2 u = *reinterpret_cast<const uint2*>(zt + p * ntiles);
                const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
                const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
                v[0] = f0.x; v[1] = f0.y; v[2] = f1.x; v[3] = f1.y;
              } else {
                const float4 f = *reinterpret_cast<const float4*>(zt + p * ntiles);
                v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
              }
            } else {
              v[0] = v[1] = v[2] = v[3] = 0.f;
            }
          }
      }
#pragma unroll
      for (int gg = 0; gg < 2; ++gg) {
      const int gi = gp + gg;
      if (gi >= ngroups) break;
      float acc[2][2][4] = {};  // [m-tile A/B][n-tile][frag]
#pragma unroll
      for (int ks = 0; ks < KST; ++ks) {
        float (&v)[4][4] = vv[gg][ks];
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          // a0 = (tile 4g+2m, planes 2q, 2q+1), a1 = (tile 4g+2m+1, ...), a2/a3: planes 2q+8, +9
          const int t0 = 2 * m, t1 = 2 * m + 1;
          if constexpr (sizeof(Tz) == 2) {
            const uint32_t a0 = pack2(v[0][t0], v[1][t0]), a1 = pack2(v[0][t1], v[1][t1]);
            const uint32_t a2 = pack2(v[2][t0], v[3][t0]), a3 = pack2(v[2][t1], v[3][t1]);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              mma(acc[m][nt], a0, a1, a2, a3, bh[ks][nt][0], bh[ks][nt][1]);
              mma(acc[m][nt], a0, a1, a2, a3, bl[ks][nt][0], bl[ks][nt][1]);
            }
          } else {
            uint32_t h0, l0, h1, l1, h2, l2, h3, l3;
            split2(v[0][t0], v[1][t0], h0, l0);
            split2(v[0][t1], v[1][t1], h1, l1);
            split2(v[2][t0], v[3][t0], h2, l2);
            split2(v[2][t1], v[3][t1], h3, l3);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              mma(acc[m][nt], h0, h1, h2, h3, bh[ks][nt][0], bh[ks][nt][1]);
              mma(acc[m][nt], l0, l1, l2, l3, bh[ks][nt][0], bh[ks][nt][1]);
              mma(acc[m][nt], h0, h1, h2, h3, bl[ks][nt][0], bl[ks][nt][1]);
            }
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int a = 2 * nt + (q >> 1), b = 2 * (q & 1);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            Tout* d = ostage + a * kOutStride + (4 * g + 2 * m + t) * 4 + b;
            if constexpr (sizeof(Tout) == 2)
              *reinterpret_cast<uint32_t*>(d) = pack2(acc[m][nt][2 * t], acc[m][nt][2 * t + 1]);
            else
              *reinterpret_cast<float2*>(d) = make_float2(acc[m][nt][2 * t], acc[m][nt][2 * t + 1]);
          }
        }
      __syncwarp();
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        Tout* dst = out + (I * 4 + a) * ldo + (J0 + 32 * gi) * 4 + 4 * lane;
        const Tout* src = ostage + a * kOutStride + 4 * lane;
        if constexpr (sizeof(Tout) == 2)
          *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(src);
        else
          *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
      }
      if constexpr (RED) {
        const __nv_bfloat16* xg = xr + I * 4 * ldr + (J0 + 32 * gi) * 4;
        R.step(zrow + 32 * gi, ntiles, Q, xg, ldr);
        R.step(zrow + 32 * gi + 16, ntiles, Q, xg + 64, ldr);
      }
      }
    }
  }
  if constexpr (RED) R.finish(sred, Q, red_partial);
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

template <typename Tz, typename Tout, bool RED, int KST>
cudaError_t launch_dec_k(const void* in, int Q, int64_t br, int64_t bc, const float* coef,
                         void* out, int64_t ldo, const void* rm, int64_t ldr, float* ro, float* rw,
                         cudaStream_t s) {
  constexpr int kOutStride = 128 + (sizeof(Tout) == 2 ? 8 : 4);
  const size_t smem = kWarpsM * 4 * kOutStride * sizeof(Tout) + (RED ? kWarpsM * Q * 16 * 4 : 0);
  auto k = k_decode_mma<Tz, Tout, RED, KST>;
  if (cudaError_t e = set_smem(k, smem)) return e;
  const int64_t ntasks = br * ((bc + kTaskTiles - 1) / kTaskTiles);
  const int grid = grid_m(ntasks, sm_count() * (RED ? 4 : 8));
  k<<<grid, kThreadsM, smem, s>>>(static_cast<const Tz*>(in), Q, br, bc, coef,
                                  static_cast<Tout*>(out), ldo,
                                  static_cast<const __nv_bfloat16*>(rm), ldr, rw);
  if (RED) return sum_partials(rw, grid, Q * 16, ro, s);
  return cudaGetLastError();
}

template <typename Tz, typename Tout, bool RED>
cudaError_t launch_dec(const void* in, int Q, int64_t br, int64_t bc, const float* coef, void* out,
                       int64_t ldo, const void* rm, int64_t ldr, float* ro, float* rw,
                       cudaStream_t s) {
  switch ((Q + 15) / 16) {
    case 1: return launch_dec_k<Tz, Tout, RED, 1>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
    case 2: return launch_dec_k<Tz, Tout, RED, 2>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
    case 3: return launch_dec_k<Tz, Tout, RED, 3>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
    default: return launch_dec_k<Tz, Tout, RED, 4>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
  }
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

// Tensor-core decode: t = 4, bc % 16 == 0, output bf16 (fp32 output keeps the FFMA path so
// the fp32 parity mode stays full precision); RED needs a bf16 second matrix.
cudaError_t planes_to_tiles_mma(const void* in, int idt, int Q, int64_t br, int64_t bc,
                                const float* coef, void* out, int odt, int64_t ldo, const void* rm,
                                int rdt, int64_t ldr, float* ro, float* rw, cudaStream_t s) {
  if (odt != kBF16 || bc % 32 || ldo % 8 || Q > 64 || !al16(in) || !al16(out))
    return cudaErrorNotSupported;
  if (rm && (rdt != kBF16 || Q > 32 || ldr % 8 || !al16(rm))) return cudaErrorNotSupported;
  if (idt == kF32) {
    if (rm) return launch_dec<float, __nv_bfloat16, true>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
    return launch_dec<float, __nv_bfloat16, false>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
  }
  if (rm) return launch_dec<__nv_bfloat16, __nv_bfloat16, true>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
  return launch_dec<__nv_bfloat16, __nv_bfloat16, false>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
}

}  // namespace stl
