// stl_transform.cu — the per-tile change-of-basis kernels around the contraction.
//
//   tiles_to_planes : encode_tiles   (snf_operator.py:80-85; tile layout dense_core.py:98-108)
//                     out[p][I][J] = sum_c coef[p][c] * m[I*t + c/t, J*t + c%t]
//                     optional fused reduction  red[p][c] = sum_{I,J} planes[p][I][J]*tile[I,J][c]
//                     (g_d of _layer_backward, toy_network.py:100)
//   planes_to_tiles : decode_tiles   (snf_operator.py:88-96; untile dense_core.py:111-119)
//                     out[I*t + c/t, J*t + c%t] = sum_q coef[q][c] * in[q][I][J]
//                     optional fused reduction with the tiles of a second matrix
//                     (g_ex of _layer_backward, toy_network.py:104)
//   planes_to_planes: the r x r composite of stl_fused_step (snf_operator.py:175-188)
//
// "planes" = the GPU-native encoded layout: r slice planes (r, rows, cols), each plane a
// row-major (rows x cols) matrix — the operand layout of the slice GEMMs. The reference's
// fiber-contiguous (rows, cols, r) layout is converted at the Python boundary.
//
// These passes are HBM-bound (one read of the tiles, one write of r/t^2 as many coefficients);
// one thread owns one t x t tile, warps cover consecutive tile columns so every row segment
// and every plane store is coalesced. Reductions are deterministic: per-block partial sums
// in registers, a fixed-order second pass over blocks.
#include "stl_internal.h"

namespace stl {
namespace {

constexpr int kTB = 128;  // threads per block = tiles per block iteration

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Load one t-wide row segment (vectorised when the segment is 8 or 16 aligned bytes).
template <int T, typename E>
__device__ __forceinline__ void load_seg(const E* __restrict__ src, float* dst, bool vec) {
  if constexpr (T * sizeof(E) == 8) {
    if (vec) {
      const uint2 u = *reinterpret_cast<const uint2*>(src);
      const E* e = reinterpret_cast<const E*>(&u);
#pragma unroll
      for (int b = 0; b < T; ++b) dst[b] = to_f(e[b]);
      return;
    }
  } else if constexpr (T * sizeof(E) == 16) {
    if (vec) {
      const uint4 u = *reinterpret_cast<const uint4*>(src);
      const E* e = reinterpret_cast<const E*>(&u);
#pragma unroll
      for (int b = 0; b < T; ++b) dst[b] = to_f(e[b]);
      return;
    }
  }
#pragma unroll
  for (int b = 0; b < T; ++b) dst[b] = to_f(src[b]);
}

template <int T, typename E>
__device__ __forceinline__ void store_seg(E* __restrict__ dst, const float* src, bool vec) {
  if constexpr (T * sizeof(E) == 8 || T * sizeof(E) == 16) {
    if (vec) {
      E tmp[T];
#pragma unroll
      for (int b = 0; b < T; ++b) tmp[b] = from_f<E>(src[b]);
      if constexpr (T * sizeof(E) == 8)
        *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(tmp);
      else
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(tmp);
      return;
    }
  }
#pragma unroll
  for (int b = 0; b < T; ++b) dst[b] = from_f<E>(src[b]);
}

// Staged reduction red[p][c] += sum over this block's tiles of pv[p] * tv[c].
// sp: [kTB][SP] plane values, sx: [kTB][SX] tile values (odd strides: conflict-free).
template <int TT, int MAXO>
__device__ __forceinline__ void reduce_stage(const float* sp, int SP, const float* sx, int SX,
                                             int P, float (&racc)[MAXO]) {
  const int n = P * TT;
#pragma unroll
  for (int j = 0; j < MAXO; ++j) {
    const int o = threadIdx.x + j * kTB;
    if (o < n) {
      const int p = o / TT, c = o - (o / TT) * TT;
      float s = 0.f;
#pragma unroll 8
      for (int tl = 0; tl < kTB; ++tl) s = fmaf(sp[tl * SP + p], sx[tl * SX + c], s);
      racc[j] += s;
    }
  }
}

template <int T, typename Tin, typename Tout, bool RED, typename Tr>
__global__ void __launch_bounds__(kTB)
    k_tiles_to_planes(const Tin* __restrict__ m, int64_t ldm, int64_t br, int64_t bc,
                      const float* __restrict__ coef, int P, Tout* __restrict__ out,
                      const Tr* __restrict__ red_planes, float* __restrict__ red_partial,
                      int vec) {
  constexpr int TT = T * T;
  constexpr int MAXO = RED ? (kMaxRank * TT + kTB - 1) / kTB : 1;
  extern __shared__ float sm[];
  float* sc = sm;
  const int SX = TT + 1;
  const int SP = P | 1;
  float* sx = sc + P * TT;
  float* sp = sx + kTB * SX;
  for (int i = threadIdx.x; i < P * TT; i += kTB) sc[i] = coef[i];
  __syncthreads();
  const int64_t ntiles = br * bc;
  float racc[MAXO];
#pragma unroll
  for (int j = 0; j < MAXO; ++j) racc[j] = 0.f;

  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kTB; base < ntiles;
       base += static_cast<int64_t>(gridDim.x) * kTB) {
    const int64_t idx = base + threadIdx.x;
    const bool valid = idx < ntiles;
    float x[TT];
    if (valid) {
      const int64_t I = idx / bc, J = idx - (idx / bc) * bc;
      const Tin* src = m + I * T * ldm + J * T;
#pragma unroll
      for (int a = 0; a < T; ++a) load_seg<T>(src + a * ldm, x + a * T, vec);
#pragma unroll 4
      for (int p = 0; p < P; ++p) {
        const float* cp = sc + p * TT;
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < TT; ++c) acc = fmaf(cp[c], x[c], acc);
        out[p * ntiles + idx] = from_f<Tout>(acc);
      }
    } else {
#pragma unroll
      for (int c = 0; c < TT; ++c) x[c] = 0.f;
    }
    if constexpr (RED) {
      __syncthreads();
#pragma unroll
      for (int c = 0; c < TT; ++c) sx[threadIdx.x * SX + c] = x[c];
      for (int p = 0; p < P; ++p)
        sp[threadIdx.x * SP + p] = valid ? to_f(red_planes[p * ntiles + idx]) : 0.f;
      __syncthreads();
      reduce_stage<TT, MAXO>(sp, SP, sx, SX, P, racc);
    }
  }
  if constexpr (RED) {
    const int n = P * TT;
#pragma unroll
    for (int j = 0; j < MAXO; ++j) {
      const int o = threadIdx.x + j * kTB;
      if (o < n) red_partial[static_cast<int64_t>(blockIdx.x) * n + o] = racc[j];
    }
  }
}

template <int T, typename Tin, typename Tout, bool RED, typename Tr>
__global__ void __launch_bounds__(kTB)
    k_planes_to_tiles(const Tin* __restrict__ in, int Q, int64_t br, int64_t bc,
                      const float* __restrict__ coef, Tout* __restrict__ out, int64_t ldo,
                      const Tr* __restrict__ red_m, int64_t ldr, float* __restrict__ red_partial,
                      int vec_out, int vec_red) {
  constexpr int TT = T * T;
  constexpr int MAXO = RED ? (kMaxRank * TT + kTB - 1) / kTB : 1;
  extern __shared__ float sm[];
  float* sc = sm;
  const int SX = TT + 1;
  const int SP = Q | 1;
  float* sx = sc + Q * TT;
  float* sp = sx + kTB * SX;
  for (int i = threadIdx.x; i < Q * TT; i += kTB) sc[i] = coef[i];
  __syncthreads();
  const int64_t ntiles = br * bc;
  float racc[MAXO];
#pragma unroll
  for (int j = 0; j < MAXO; ++j) racc[j] = 0.f;

  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kTB; base < ntiles;
       base += static_cast<int64_t>(gridDim.x) * kTB) {
    const int64_t idx = base + threadIdx.x;
    const bool valid = idx < ntiles;
    int64_t I = 0, J = 0;
    if (valid) {
      I = idx / bc;
      J = idx - I * bc;
      float acc[TT];
#pragma unroll
      for (int c = 0; c < TT; ++c) acc[c] = 0.f;
#pragma unroll 4
      for (int q = 0; q < Q; ++q) {
        const float v = to_f(in[q * ntiles + idx]);
        if constexpr (RED) sp[threadIdx.x * SP + q] = v;  // staged below after a barrier
        const float* cq = sc + q * TT;
#pragma unroll
        for (int c = 0; c < TT; ++c) acc[c] = fmaf(cq[c], v, acc[c]);
      }
      Tout* dst = out + I * T * ldo + J * T;
#pragma unroll
      for (int a = 0; a < T; ++a) store_seg<T>(dst + a * ldo, acc + a * T, vec_out);
    }
    if constexpr (RED) {
      // sp rows of this thread were written above; other threads only read after the sync.
      float x[TT];
      if (valid) {
        const Tr* src = red_m + I * T * ldr + J * T;
#pragma unroll
        for (int a = 0; a < T; ++a) load_seg<T>(src + a * ldr, x + a * T, vec_red);
      } else {
#pragma unroll
        for (int c = 0; c < TT; ++c) x[c] = 0.f;
        for (int q = 0; q < Q; ++q) sp[threadIdx.x * SP + q] = 0.f;
      }
#pragma unroll
      for (int c = 0; c < TT; ++c) sx[threadIdx.x * SX + c] = x[c];
      __syncthreads();
      reduce_stage<TT, MAXO>(sp, SP, sx, SX, Q, racc);
      __syncthreads();
    }
  }
  if constexpr (RED) {
    const int n = Q * TT;
#pragma unroll
    for (int j = 0; j < MAXO; ++j) {
      const int o = threadIdx.x + j * kTB;
      if (o < n) red_partial[static_cast<int64_t>(blockIdx.x) * n + o] = racc[j];
    }
  }
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kTB)
    k_planes_to_planes(const Tin* __restrict__ in, int Q, int64_t ntiles,
                       const float* __restrict__ coef, int P, Tout* __restrict__ out) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < P * Q; i += kTB) sm[i] = coef[i];
  __syncthreads();
  // (the generic fallback of the fused-step remix: fp32 chains, r > 32, odd tile columns)
  // No per-thread array indexed by a runtime rank (it would live in local memory): each output
  // re-reads the thread's Q inputs, which stay in L1 after the first output.
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * kTB + threadIdx.x; idx < ntiles;
       idx += static_cast<int64_t>(gridDim.x) * kTB) {
    for (int p = 0; p < P; ++p) {
      float acc = 0.f;
      const float* cp = sm + p * Q;
#pragma unroll 4
      for (int q = 0; q < Q; ++q) acc = fmaf(cp[q], to_f(in[q * ntiles + idx]), acc);
      out[p * ntiles + idx] = from_f<Tout>(acc);
    }
  }
}

// out (r x r) = a (r x tt) . b^T (b is r x tt):  the fused-step composite e_x @ d.T.
__global__ void k_compose(const float* __restrict__ a, const float* __restrict__ b, int r, int tt,
                          float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r * r) return;
  const int p = i / r, q = i % r;
  float s = 0.f;
  for (int c = 0; c < tt; ++c) s = fmaf(a[p * tt + c], b[q * tt + c], s);
  out[i] = s;
}

int grid_for(int64_t ntiles, int cap) {
  int64_t g = (ntiles + kTB - 1) / kTB;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

template <int T, typename Tin, typename Tout, typename Tr>
cudaError_t t2p_launch(const void* m, int64_t ldm, int64_t br, int64_t bc, const float* coef,
                       int P, void* out, const void* red_planes, float* red_out, float* red_ws,
                       cudaStream_t s) {
  constexpr int TT = T * T;
  const int64_t ntiles = br * bc;
  const bool vec = (ldm % T == 0) && ((reinterpret_cast<uintptr_t>(m) % (T * sizeof(Tin))) == 0);
  if (red_planes) {
    const int grid = grid_for(ntiles, kRedBlocks);
    const size_t smem = sizeof(float) * (P * TT + kTB * (TT + 1) + kTB * (P | 1));
    auto k = k_tiles_to_planes<T, Tin, Tout, true, Tr>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kTB, smem, s>>>(static_cast<const Tin*>(m), ldm, br, bc, coef, P,
                              static_cast<Tout*>(out), static_cast<const Tr*>(red_planes), red_ws,
                              vec);
    if (cudaError_t e2 = sum_partials(red_ws, grid, P * TT, red_out, s)) return e2;
  } else {
    const int grid = grid_for(ntiles, sm_count() * 16);
    const size_t smem = sizeof(float) * P * TT;
    k_tiles_to_planes<T, Tin, Tout, false, float><<<grid, kTB, smem, s>>>(
        static_cast<const Tin*>(m), ldm, br, bc, coef, P, static_cast<Tout*>(out), nullptr,
        nullptr, vec);
  }
  return cudaGetLastError();
}

template <int T, typename Tin, typename Tout, typename Tr>
cudaError_t p2t_launch(const void* in, int Q, int64_t br, int64_t bc, const float* coef, void* out,
                       int64_t ldo, const void* red_m, int64_t ldr, float* red_out, float* red_ws,
                       cudaStream_t s) {
  constexpr int TT = T * T;
  const int64_t ntiles = br * bc;
  const bool vo = (ldo % T == 0) && ((reinterpret_cast<uintptr_t>(out) % (T * sizeof(Tout))) == 0);
  if (red_m) {
    const bool vr = (ldr % T == 0) && ((reinterpret_cast<uintptr_t>(red_m) % (T * sizeof(Tr))) == 0);
    const int grid = grid_for(ntiles, kRedBlocks);
    const size_t smem = sizeof(float) * (Q * TT + kTB * (TT + 1) + kTB * (Q | 1));
    auto k = k_planes_to_tiles<T, Tin, Tout, true, Tr>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    k<<<grid, kTB, smem, s>>>(static_cast<const Tin*>(in), Q, br, bc, coef,
                              static_cast<Tout*>(out), ldo, static_cast<const Tr*>(red_m), ldr,
                              red_ws, vo, vr);
    if (cudaError_t e2 = sum_partials(red_ws, grid, Q * TT, red_out, s)) return e2;
  } else {
    const int grid = grid_for(ntiles, sm_count() * 16);
    const size_t smem = sizeof(float) * Q * TT;
    k_planes_to_tiles<T, Tin, Tout, false, Tr><<<grid, kTB, smem, s>>>(
        static_cast<const Tin*>(in), Q, br, bc, coef, static_cast<Tout*>(out), ldo, nullptr, 0,
        nullptr, vo, 0);
  }
  return cudaGetLastError();
}

template <int T, typename Tr>
cudaError_t t2p_dispatch_r(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                           const float* coef, int P, void* out, int odt, const void* rp,
                           float* ro, float* rw, cudaStream_t s) {
  if (mdt == kBF16 && odt == kBF16)
    return t2p_launch<T, __nv_bfloat16, __nv_bfloat16, Tr>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
  if (mdt == kBF16 && odt == kF32)
    return t2p_launch<T, __nv_bfloat16, float, Tr>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
  if (mdt == kF32 && odt == kBF16)
    return t2p_launch<T, float, __nv_bfloat16, Tr>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
  return t2p_launch<T, float, float, Tr>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
}

template <int T>
cudaError_t t2p_dispatch(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                         const float* coef, int P, void* out, int odt, const void* rp, int rdt,
                         float* ro, float* rw, cudaStream_t s) {
  if (rp && rdt == kBF16)
    return t2p_dispatch_r<T, __nv_bfloat16>(m, mdt, ldm, br, bc, coef, P, out, odt, rp, ro, rw, s);
  return t2p_dispatch_r<T, float>(m, mdt, ldm, br, bc, coef, P, out, odt, rp, ro, rw, s);
}

template <int T, typename Tin, typename Tout>
cudaError_t p2t_red_dispatch(const void* in, int Q, int64_t br, int64_t bc, const float* coef,
                             void* out, int64_t ldo, const void* rm, int rdt, int64_t ldr,
                             float* ro, float* rw, cudaStream_t s) {
  if (rdt == kBF16)
    return p2t_launch<T, Tin, Tout, __nv_bfloat16>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
  return p2t_launch<T, Tin, Tout, float>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
}

template <int T>
cudaError_t p2t_dispatch(const void* in, int idt, int Q, int64_t br, int64_t bc,
                         const float* coef, void* out, int odt, int64_t ldo, const void* rm,
                         int rdt, int64_t ldr, float* ro, float* rw, cudaStream_t s) {
  if (idt == kBF16 && odt == kBF16)
    return p2t_red_dispatch<T, __nv_bfloat16, __nv_bfloat16>(in, Q, br, bc, coef, out, ldo, rm, rdt, ldr, ro, rw, s);
  if (idt == kBF16 && odt == kF32)
    return p2t_red_dispatch<T, __nv_bfloat16, float>(in, Q, br, bc, coef, out, ldo, rm, rdt, ldr, ro, rw, s);
  if (idt == kF32 && odt == kBF16)
    return p2t_red_dispatch<T, float, __nv_bfloat16>(in, Q, br, bc, coef, out, ldo, rm, rdt, ldr, ro, rw, s);
  return p2t_red_dispatch<T, float, float>(in, Q, br, bc, coef, out, ldo, rm, rdt, ldr, ro, rw, s);
}

}  // namespace

// Dispatch: the streaming kernels first (t = 4, aligned bf16), then the t = 4 register /
// tensor-core fallbacks, then the generic tile-size-templated FFMA kernels. F24 planes (a bf16
// path intermediate) are read by the streaming kernels only: if they decline, fail loudly
// instead of reading the 3-byte format as fp32.
cudaError_t tiles_to_planes(const void* m, int m_dtype, int64_t ldm, int64_t br, int64_t bc,
                            int t, const float* coef, int P, void* out, int out_dtype,
                            const void* red_planes, int red_dtype, float* red_out,
                            float* red_ws, cudaStream_t s) {
  if (br * bc == 0) return cudaSuccess;
  if (t == 4) {
    cudaError_t e = tiles_to_planes_stream(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype,
                                           red_planes, red_dtype, red_out, red_ws, s);
    if (e != cudaErrorNotSupported) return e;
  }
  if (t == 2 && !red_planes) {
    cudaError_t e = tiles_to_planes2(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype, s);
    if (e != cudaErrorNotSupported) return e;
  }
  if (red_planes && red_dtype == kF24) return cudaErrorNotSupported;
  if (t == 4) {
    cudaError_t e = tiles_to_planes_mma(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype,
                                        red_planes, red_dtype, red_out, red_ws, s);
    if (e != cudaErrorNotSupported) return e;
    e = tiles_to_planes4(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype, red_planes,
                         red_dtype, red_out, red_ws, s);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (t) {
    case 1: return t2p_dispatch<1>(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype, red_planes, red_dtype, red_out, red_ws, s);
    case 2: return t2p_dispatch<2>(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype, red_planes, red_dtype, red_out, red_ws, s);
    case 4: return t2p_dispatch<4>(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype, red_planes, red_dtype, red_out, red_ws, s);
    case 8: return t2p_dispatch<8>(m, m_dtype, ldm, br, bc, coef, P, out, out_dtype, red_planes, red_dtype, red_out, red_ws, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t planes_to_tiles(const void* in, int in_dtype, int Q, int64_t br, int64_t bc, int t,
                            const float* coef, void* out, int out_dtype, int64_t ldo,
                            const void* red_m, int red_dtype, int64_t ldr, float* red_out,
                            float* red_ws, cudaStream_t s) {
  if (br * bc == 0) return cudaSuccess;
  if (t == 4) {
    cudaError_t e = planes_to_tiles_stream(in, in_dtype, Q, br, bc, coef, out, out_dtype, ldo,
                                           red_m, red_dtype, ldr, red_out, red_ws, s);
    if (e != cudaErrorNotSupported) return e;
  }
  if (in_dtype == kF24) return cudaErrorNotSupported;
  if (t == 2 && !red_m) {
    cudaError_t e = planes_to_tiles2(in, in_dtype, Q, br, bc, coef, out, out_dtype, ldo, s);
    if (e != cudaErrorNotSupported) return e;
  }
  if (t == 4) {
    cudaError_t e = planes_to_tiles4(in, in_dtype, Q, br, bc, coef, out, out_dtype, ldo, red_m,
                                     red_dtype, ldr, red_out, red_ws, s);
    if (e != cudaErrorNotSupported) return e;
  }
  switch (t) {
    case 1: return p2t_dispatch<1>(in, in_dtype, Q, br, bc, coef, out, out_dtype, ldo, red_m, red_dtype, ldr, red_out, red_ws, s);
    case 2: return p2t_dispatch<2>(in, in_dtype, Q, br, bc, coef, out, out_dtype, ldo, red_m, red_dtype, ldr, red_out, red_ws, s);
    case 4: return p2t_dispatch<4>(in, in_dtype, Q, br, bc, coef, out, out_dtype, ldo, red_m, red_dtype, ldr, red_out, red_ws, s);
    case 8: return p2t_dispatch<8>(in, in_dtype, Q, br, bc, coef, out, out_dtype, ldo, red_m, red_dtype, ldr, red_out, red_ws, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t planes_to_planes(const void* in, int in_dtype, int Q, int64_t ntiles,
                             const float* coef, int P, void* out, int out_dtype, cudaStream_t s) {
  if (ntiles == 0) return cudaSuccess;
  const int grid = grid_for(ntiles, sm_count() * 16);
  const size_t smem = sizeof(float) * P * Q;
  if (in_dtype == kBF16 && out_dtype == kBF16)
    k_planes_to_planes<__nv_bfloat16, __nv_bfloat16><<<grid, kTB, smem, s>>>(
        static_cast<const __nv_bfloat16*>(in), Q, ntiles, coef, P, static_cast<__nv_bfloat16*>(out));
  else if (in_dtype == kBF16)
    k_planes_to_planes<__nv_bfloat16, float><<<grid, kTB, smem, s>>>(
        static_cast<const __nv_bfloat16*>(in), Q, ntiles, coef, P, static_cast<float*>(out));
  else if (out_dtype == kBF16)
    k_planes_to_planes<float, __nv_bfloat16><<<grid, kTB, smem, s>>>(
        static_cast<const float*>(in), Q, ntiles, coef, P, static_cast<__nv_bfloat16*>(out));
  else
    k_planes_to_planes<float, float><<<grid, kTB, smem, s>>>(
        static_cast<const float*>(in), Q, ntiles, coef, P, static_cast<float*>(out));
  return cudaGetLastError();
}

cudaError_t compose_coefs(const float* a, const float* b, int r, int tt, float* out,
                          cudaStream_t s) {
  k_compose<<<(r * r + 127) / 128, 128, 0, s>>>(a, b, r, tt, out);
  return cudaGetLastError();
}

}  // namespace stl
