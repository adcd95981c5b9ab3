// stl_transform2.cu — HBM-streaming t = 2 tile transforms (BASELINE configs[2]'s t = 2 points).
//
//   encode: planes[p][I][J] = sum_c E[p][c] tile(I, J)[c]   encode_tiles (snf_operator.py:80-85)
//   decode: tile(I, J)[c]   = sum_q Z[q][I][J] D[q][c]      decode_tiles (snf_operator.py:88-96)
// Tiles follow the reference layout contract (dense_core.py:98-108): element c = 2a + b of
// tile (I, J) is m[2I + a, 2J + b].
//
// At t = 2 a tile holds only 4 values, so the change of basis is 4 multiply-adds per output
// coefficient — far below what the FMA pipe sustains next to the HBM stream — and the planes
// are r/4 = 4..12x the matrix: the pass is purely HBM-bound. The design is therefore a register
// streaming kernel with high memory-level parallelism and no shared-memory staging: one thread
// owns 4 consecutive tiles of a tile row (2 matrix rows x 8 elements = two 16-byte loads or
// stores), a warp 128 tiles, so every plane access of a warp is one contiguous 256-byte (bf16)
// or 512-byte (fp32) run; the decode issues all of its plane loads before the first use. The
// coefficients sit in shared memory (warp-uniform reads: broadcast).
#include "stl_internal.h"

namespace stl {
namespace {

constexpr int kThreads2 = 256;

__device__ __forceinline__ void unpack8(const uint4 u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// PB = plane bound (a multiple of 8 >= P): the plane loops unroll fully. TPT = tiles per
// thread (8: 16-byte plane accesses; 4 when the tile columns are not a multiple of 8).
template <int TPT>
struct Rows2 {  // the 2 x (2 TPT) matrix elements of a thread's tiles, loaded as 16-byte words
  uint4 w[2][TPT / 4];
};
template <int TPT>
__device__ __forceinline__ void load_rows2(Rows2<TPT>& r, const __nv_bfloat16* src, int64_t ldm) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int h = 0; h < TPT / 4; ++h)
      r.w[a][h] = __ldcs(reinterpret_cast<const uint4*>(src + a * ldm) + h);
}

template <int PB, int TPT>
__global__ void __launch_bounds__(kThreads2)
    k_encode2(const __nv_bfloat16* __restrict__ m, int64_t ldm, int64_t br, int64_t bc,
              const float* __restrict__ coef, int P, __nv_bfloat16* __restrict__ out) {
  __shared__ float sc[PB * 4];
  for (int i = threadIdx.x; i < PB * 4; i += kThreads2) sc[i] = i < P * 4 ? coef[i] : 0.f;
  __syncthreads();
  const int64_t gpr = bc / TPT;  // thread groups per tile row
  const int64_t ngroups = br * gpr;
  const int64_t ntiles = br * bc;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads2;
  int64_t g = blockIdx.x * static_cast<int64_t>(kThreads2) + threadIdx.x;
  // software pipeline: the next group's rows are in flight while this group is computed
  Rows2<TPT> cur, nxt;
  if (g < ngroups) {
    const int64_t I = g / gpr;
    load_rows2<TPT>(cur, m + 2 * I * ldm + 2 * (g - I * gpr) * TPT, ldm);
  }
  for (; g < ngroups; g += stride) {
    const int64_t gn = g + stride;
    if (gn < ngroups) {
      const int64_t In = gn / gpr;
      load_rows2<TPT>(nxt, m + 2 * In * ldm + 2 * (gn - In * gpr) * TPT, ldm);
    }
    const int64_t I = g / gpr, J0 = (g - I * gpr) * TPT;
    float r0[2 * TPT], r1[2 * TPT];
#pragma unroll
    for (int h = 0; h < TPT / 4; ++h) {
      float f[8];
      unpack8(cur.w[0][h], f);
#pragma unroll
      for (int i = 0; i < 8; ++i) r0[8 * h + i] = f[i];
      unpack8(cur.w[1][h], f);
#pragma unroll
      for (int i = 0; i < 8; ++i) r1[8 * h + i] = f[i];
    }
    __nv_bfloat16* dst = out + I * bc + J0;
#pragma unroll 4
    for (int p = 0; p < P; ++p) {
      // re-read per use (volatile): hoisting 4 PB coefficients into registers would cost
      // occupancy, and a warp-uniform shared load is a broadcast
      const volatile float* vc = sc + 4 * p;
      const float e0 = vc[0], e1 = vc[1], e2 = vc[2], e3 = vc[3];
      uint32_t o[TPT / 2];
#pragma unroll
      for (int k = 0; k < TPT; k += 2) {  // tile J0 + k: (r0[2k], r0[2k+1]; r1[2k], r1[2k+1])
        const float v0 = fmaf(e0, r0[2 * k], fmaf(e1, r0[2 * k + 1], fmaf(e2, r1[2 * k], e3 * r1[2 * k + 1])));
        const float v1 = fmaf(e0, r0[2 * k + 2], fmaf(e1, r0[2 * k + 3], fmaf(e2, r1[2 * k + 2], e3 * r1[2 * k + 3])));
        o[k / 2] = pack2(v0, v1);
      }
      if constexpr (TPT == 8)
        __stcs(reinterpret_cast<uint4*>(dst + p * ntiles), make_uint4(o[0], o[1], o[2], o[3]));
      else
        __stcs(reinterpret_cast<uint2*>(dst + p * ntiles), make_uint2(o[0], o[1]));
    }
    cur = nxt;
  }
}

// A thread's TPT values of one plane, kept as the loaded words until used (bf16: 2 bytes per
// value in registers) and unpacked to fp32 at the multiply-adds.
template <typename Z, int TPT>
struct PlaneWords {
  static constexpr int kWords = TPT * static_cast<int>(sizeof(Z)) / 16;  // 16-byte words (0: 8 bytes)
  uint4 w[kWords > 0 ? kWords : 1];
};
template <typename Z, int TPT>
__device__ __forceinline__ void load_plane2(PlaneWords<Z, TPT>& z, const Z* p) {
  if constexpr (PlaneWords<Z, TPT>::kWords == 0) {
    const uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));
    z.w[0] = make_uint4(u.x, u.y, 0u, 0u);
  } else {
#pragma unroll
    for (int h = 0; h < PlaneWords<Z, TPT>::kWords; ++h)
      z.w[h] = __ldcs(reinterpret_cast<const uint4*>(p) + h);
  }
}
template <typename Z, int TPT>
__device__ __forceinline__ float plane_val(const PlaneWords<Z, TPT>& z, int k) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(z.w);
  if constexpr (sizeof(Z) == 2)
    return __uint_as_float((k & 1) ? (u[k >> 1] & 0xFFFF0000u) : (u[k >> 1] << 16));
  else
    return __uint_as_float(u[k]);
}

template <int PB, int TPT, typename Z>
__global__ void __launch_bounds__(kThreads2)
    k_decode2(const Z* __restrict__ in, int Q, int64_t br, int64_t bc,
              const float* __restrict__ coef, __nv_bfloat16* __restrict__ out, int64_t ldo) {
  constexpr int kChunk = sizeof(Z) == 2 ? 12 : (TPT == 8 ? 6 : 12);  // planes in flight together
  __shared__ float sc[(PB + kChunk) * 4];
  for (int i = threadIdx.x; i < (PB + kChunk) * 4; i += kThreads2) sc[i] = i < Q * 4 ? coef[i] : 0.f;
  __syncthreads();
  const int64_t gpr = bc / TPT;
  const int64_t ngroups = br * gpr;
  const int64_t ntiles = br * bc;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(kThreads2) + threadIdx.x; g < ngroups;
       g += static_cast<int64_t>(gridDim.x) * kThreads2) {
    const int64_t I = g / gpr, J0 = (g - I * gpr) * TPT;
    const Z* src = in + I * bc + J0;
    float acc[2 * TPT][2];  // [2k + b][a]: tile J0 + k, column b, row a
#pragma unroll
    for (int i = 0; i < 2 * TPT; ++i) acc[i][0] = acc[i][1] = 0.f;
#pragma unroll 1
    for (int q0 = 0; q0 < Q; q0 += kChunk) {
      PlaneWords<Z, TPT> z[kChunk];
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        if (q0 + j < Q) load_plane2<Z, TPT>(z[j], src + (q0 + j) * ntiles);
        else
#pragma unroll
          for (int h = 0; h < (PlaneWords<Z, TPT>::kWords > 0 ? PlaneWords<Z, TPT>::kWords : 1); ++h)
            z[j].w[h] = make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int j = 0; j < kChunk; ++j) {
        const int q = q0 + j;
        const volatile float* vc = sc + 4 * q;  // see k_encode2
        const float d0 = vc[0], d1 = vc[1], d2 = vc[2], d3 = vc[3];
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          const float v = plane_val<Z, TPT>(z[j], k);
          acc[2 * k][0] = fmaf(v, d0, acc[2 * k][0]);          // (a 0, b 0)
          acc[2 * k + 1][0] = fmaf(v, d1, acc[2 * k + 1][0]);  // (a 0, b 1)
          acc[2 * k][1] = fmaf(v, d2, acc[2 * k][1]);          // (a 1, b 0)
          acc[2 * k + 1][1] = fmaf(v, d3, acc[2 * k + 1][1]);  // (a 1, b 1)
        }
      }
    }
    __nv_bfloat16* dst = out + 2 * I * ldo + 2 * J0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int h = 0; h < TPT / 4; ++h)
        __stcs(reinterpret_cast<uint4*>(dst + a * ldo) + h,
               make_uint4(pack2(acc[8 * h][a], acc[8 * h + 1][a]), pack2(acc[8 * h + 2][a], acc[8 * h + 3][a]),
                          pack2(acc[8 * h + 4][a], acc[8 * h + 5][a]), pack2(acc[8 * h + 6][a], acc[8 * h + 7][a])));
  }
}

int grid2(int64_t ngroups) {
  const int64_t g = (ngroups + kThreads2 - 1) / kThreads2;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  return static_cast<int>(g < cap ? (g < 1 ? 1 : g) : cap);
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

template <int TPT>
cudaError_t encode2_launch(const __nv_bfloat16* x, int64_t ldm, int64_t br, int64_t bc,
                           const float* coef, int P, __nv_bfloat16* o, cudaStream_t s) {
  const int grid = grid2(br * (bc / TPT));
  if (P <= 16) k_encode2<16, TPT><<<grid, kThreads2, 0, s>>>(x, ldm, br, bc, coef, P, o);
  else if (P <= 32) k_encode2<32, TPT><<<grid, kThreads2, 0, s>>>(x, ldm, br, bc, coef, P, o);
  else k_encode2<64, TPT><<<grid, kThreads2, 0, s>>>(x, ldm, br, bc, coef, P, o);
  return cudaGetLastError();
}

template <int TPT, typename Z>
cudaError_t decode2_launch(const Z* z, int Q, int64_t br, int64_t bc, const float* coef,
                           __nv_bfloat16* o, int64_t ldo, cudaStream_t s) {
  const int grid = grid2(br * (bc / TPT));
  if (Q <= 24) k_decode2<24, TPT, Z><<<grid, kThreads2, 0, s>>>(z, Q, br, bc, coef, o, ldo);
  else if (Q <= 48) k_decode2<48, TPT, Z><<<grid, kThreads2, 0, s>>>(z, Q, br, bc, coef, o, ldo);
  else k_decode2<64, TPT, Z><<<grid, kThreads2, 0, s>>>(z, Q, br, bc, coef, o, ldo);
  return cudaGetLastError();
}

cudaError_t tiles_to_planes2(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                             const float* coef, int P, void* out, int odt, cudaStream_t s) {
  if (mdt != kBF16 || odt != kBF16 || bc % 4 || ldm % 8 || !al16(m) || !al16(out) || P < 1 ||
      P > kMaxRank)
    return cudaErrorNotSupported;
  const auto* x = static_cast<const __nv_bfloat16*>(m);
  auto* o = static_cast<__nv_bfloat16*>(out);
  return bc % 8 == 0 ? encode2_launch<8>(x, ldm, br, bc, coef, P, o, s)
                     : encode2_launch<4>(x, ldm, br, bc, coef, P, o, s);
}

cudaError_t planes_to_tiles2(const void* in, int idt, int Q, int64_t br, int64_t bc,
                             const float* coef, void* out, int odt, int64_t ldo, cudaStream_t s) {
  if ((idt != kBF16 && idt != kF32) || odt != kBF16 || bc % 4 || ldo % 8 || !al16(out) ||
      !al16(in) || Q < 1 || Q > kMaxRank)
    return cudaErrorNotSupported;
  auto* o = static_cast<__nv_bfloat16*>(out);
  if (idt == kBF16) {
    const cudaError_t e = planes_to_tiles2_tc(in, Q, br, bc, coef, out, ldo, s);
    if (e != cudaErrorNotSupported) return e;
    const auto* z = static_cast<const __nv_bfloat16*>(in);
    return bc % 8 == 0 ? decode2_launch<8>(z, Q, br, bc, coef, o, ldo, s)
                       : decode2_launch<4>(z, Q, br, bc, coef, o, ldo, s);
  }
  const auto* z = static_cast<const float*>(in);
  return bc % 8 == 0 ? decode2_launch<8>(z, Q, br, bc, coef, o, ldo, s)
                     : decode2_launch<4>(z, Q, br, bc, coef, o, ldo, s);
}

}  // namespace stl
