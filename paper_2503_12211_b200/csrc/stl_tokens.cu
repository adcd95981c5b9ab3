// stl_tokens.cu — token-row plumbing around an STL layer whose token count is not a multiple
// of t (T2T-ViT's 197 tokens).
//
// An STL layer tiles t consecutive token rows, so a (B, T, C) activation with T % t == 1 is
// run as (B, Tp = T - 1 + t, C): t - 1 null rows appended per sample, and the layer's last t
// output rows of each sample folded back into one row with t learnable coefficients. Done with
// framework ops that is five to eight passes over the activations per layer (pad, cast, fold,
// concatenate, bias add, and their backward copies); here it is one pass each way:
//   stl_token_pad            x (B, T, C) fp32/bf16 -> bf16 (B, Tp, Cp), zero rows / columns
//   stl_token_unpad          g (B, Tp, Cp) bf16 -> (B, T, C) fp32/bf16 (the pad's backward)
//   stl_token_fold           y (B, Tp, N) -> (B, T, N): rows < T-1 copied, row T-1 = sum_i
//                            fold[i] y[T-1+i]; + bias
//   stl_token_fold_backward  g_out -> g_y (B, Tp, N), plus d bias and d fold as fixed-order
//                            per-block partial sums reduced by the deterministic tree
// All are 16-byte vectorised HBM streams (8 bf16 per thread), grid-stride over rows.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "stl_internal.h"

namespace stl {
namespace {

struct alignas(16) Bf8 {
  __nv_bfloat162 h[4];
};

__device__ __forceinline__ void bf8_to_f(const Bf8& v, float* f) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 p = __bfloat1622float2(v.h[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}

__device__ __forceinline__ Bf8 f_to_bf8(const float* f) {
  Bf8 v;
#pragma unroll
  for (int i = 0; i < 4; ++i) v.h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

__device__ __forceinline__ void load8(const float* p, float* f) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* f) {
  bf8_to_f(*reinterpret_cast<const Bf8*>(p), f);
}

__device__ __forceinline__ void store8(float* p, const float* f) {
  *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(f[4], f[5], f[6], f[7]);
}

__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* f) {
  *reinterpret_cast<Bf8*>(p) = f_to_bf8(f);
}

// out (B, Tp, Cp) bf16 <- x (B, T, C), zeros elsewhere. One thread per 8 output columns.
template <typename Tin>
__global__ void k_token_pad(const Tin* __restrict__ x, int64_t B, int64_t T, int64_t C,
                            __nv_bfloat16* __restrict__ out, int64_t Tp, int64_t Cp) {
  const int64_t vc = Cp / 8;
  const int64_t n = B * Tp * vc;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c8 = i % vc, row = i / vc;
    const int64_t b = row / Tp, j = row - b * Tp;
    float f[8];
    const int64_t c0 = c8 * 8;
    if (j < T && c0 + 8 <= C) {
      load8(x + (b * T + j) * C + c0, f);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        f[e] = (j < T && c0 + e < C) ? float(x[(b * T + j) * C + c0 + e]) : 0.f;
    }
    store8(out + row * Cp + c0, f);
  }
}

// out (B, T, C) <- g (B, Tp, Cp)[:, :T, :C]. One thread per 8 output columns (C % 8 == 0).
template <typename Tout>
__global__ void k_token_unpad(const __nv_bfloat16* __restrict__ g, int64_t B, int64_t Tp,
                              int64_t Cp, Tout* __restrict__ out, int64_t T, int64_t C) {
  const int64_t vc = C / 8;
  const int64_t n = B * T * vc;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c8 = i % vc, row = i / vc;
    const int64_t b = row / T, j = row - b * T;
    float f[8];
    load8(g + (b * Tp + j) * Cp + c8 * 8, f);
    store8(out + row * C + c8 * 8, f);
  }
}

// out (B, T, N) <- y (B, Tp, N): rows j < T-1 copied, row T-1 = sum_i fold[i] y[T-1+i]; + bias.
__global__ void k_token_fold(const __nv_bfloat16* __restrict__ y, int64_t B, int64_t Tp,
                             int64_t N, int t, const float* __restrict__ fold,
                             const float* __restrict__ bias, __nv_bfloat16* __restrict__ out,
                             int64_t T) {
  const int64_t vc = N / 8;
  const int64_t n = B * T * vc;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c0 = (i % vc) * 8, row = i / vc;
    const int64_t b = row / T, j = row - b * T;
    float f[8];
    const __nv_bfloat16* src = y + (b * Tp + j) * N + c0;
    load8(src, f);
    if (j == T - 1) {
      const float w0 = fold[0];
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] *= w0;
      for (int k = 1; k < t; ++k) {
        float h[8];
        load8(src + k * N, h);
        const float wk = fold[k];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = fmaf(wk, h[e], f[e]);
      }
    }
    if (bias) {
      float bb[8];
      load8(bias + c0, bb);
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] += bb[e];
    }
    store8(out + row * N + c0, f);
  }
}


// Backward of k_token_fold. Block `blk` owns output rows [blk*rpb, (blk+1)*rpb); a thread owns
// 8 columns (cpr = N / 8 rounded up to a warp multiple threads per row) of every ry-th row
// (ry = the block's row lanes). It writes g_y for its rows; the block writes its partial column
// sums of g_out (d bias: the row lanes summed in fixed order through shared memory) and, from
// the fold rows, partial d fold[k] = sum_n g_out[b, T-1, n] y[b, T-1+k, n], to
// part[blk * (N + t) + ...].
__global__ void k_token_fold_bwd(const __nv_bfloat16* __restrict__ gout,
                                 const __nv_bfloat16* __restrict__ y, int64_t B, int64_t Tp,
                                 int64_t N, int t, const float* __restrict__ fold, int64_t T,
                                 int64_t rpb, int cpr, __nv_bfloat16* __restrict__ gy,
                                 float* __restrict__ part) {
  extern __shared__ float s_bias[];  // [row lanes][N]
  __shared__ float s_fold[32][kFoldMaxT];
  const int ry = threadIdx.x / cpr, nry = blockDim.x / cpr;
  const int64_t c0 = int64_t(threadIdx.x - ry * cpr) * 8;
  const bool col_ok = c0 < N;
  const int64_t r0 = blockIdx.x * rpb;
  const int64_t r1 = min(r0 + rpb, B * T);
  float sb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  float sf[kFoldMaxT];
#pragma unroll
  for (int k = 0; k < kFoldMaxT; ++k) sf[k] = 0.f;
  if (col_ok) {
    constexpr int kU = 2;  // rows in flight per thread
    for (int64_t rb = r0 + ry; rb < r1; rb += kU * nry) {
      float gg[kU][8];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (rb + u * nry < r1) load8(gout + (rb + u * nry) * N + c0, gg[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t row = rb + u * nry;
        if (row >= r1) break;
        const float* g = gg[u];
        const int64_t b = row / T, j = row - b * T;
#pragma unroll
        for (int e = 0; e < 8; ++e) sb[e] += g[e];
        __nv_bfloat16* dst = gy + (b * Tp + j) * N + c0;
        if (j != T - 1) {
          store8(dst, g);
        } else {
          for (int k = 0; k < t; ++k) {
            const float wk = fold[k];
            float h[8], o[8];
            load8(y + (b * Tp + j + k) * N + c0, h);
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              o[e] = wk * g[e];
              acc = fmaf(g[e], h[e], acc);
            }
#pragma unroll
            for (int kk = 0; kk < kFoldMaxT; ++kk)
              if (kk == k) sf[kk] += acc;
            store8(dst + k * N, o);
          }
        }
      }
    }
    store8(s_bias + ry * N + c0, sb);
  }
  // fold partials: warp shuffle reduction, then the block's warps in fixed order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kFoldMaxT; ++k) {
    float v = sf[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_fold[warp][k] = v;
  }
  __syncthreads();
  float* out = part + blockIdx.x * (N + t);
  for (int64_t c = threadIdx.x; c < N; c += blockDim.x) {
    float v = s_bias[c];
    for (int r = 1; r < nry; ++r) v += s_bias[r * N + c];
    out[c] = v;
  }
  if (threadIdx.x < t) {
    float v = 0.f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) v += s_fold[w][threadIdx.x];
    out[N + threadIdx.x] = v;
  }
}

int grid_for(int64_t n, int threads) {
  const int64_t blocks = (n + threads - 1) / threads;
  const int64_t cap = int64_t(sm_count()) * 8;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

int64_t fold_blocks(int64_t rows) {
  const int64_t want = int64_t(sm_count()) * 6;
  int64_t nb = want < kRedBlocks ? want : kRedBlocks;
  if (nb > rows) nb = rows;
  return nb > 0 ? nb : 1;
}

}  // namespace

// Launchers; arguments validated by the C ABI wrappers in stl_capi.cu.
cudaError_t token_pad(const void* x, int dtype_in, int64_t B, int64_t T, int64_t C, void* out,
                      int64_t Tp, int64_t Cp, cudaStream_t s) {
  const int64_t n = B * Tp * (Cp / 8);
  if (n == 0) return cudaSuccess;
  auto* o = static_cast<__nv_bfloat16*>(out);
  if (dtype_in == kF32)
    k_token_pad<<<grid_for(n, 256), 256, 0, s>>>(static_cast<const float*>(x), B, T, C, o, Tp, Cp);
  else
    k_token_pad<<<grid_for(n, 256), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(x), B, T, C,
                                                 o, Tp, Cp);
  return cudaGetLastError();
}

cudaError_t token_unpad(const void* g, int64_t B, int64_t Tp, int64_t Cp, void* out,
                        int dtype_out, int64_t T, int64_t C, cudaStream_t s) {
  const int64_t n = B * T * (C / 8);
  if (n == 0) return cudaSuccess;
  auto* gi = static_cast<const __nv_bfloat16*>(g);
  if (dtype_out == kF32)
    k_token_unpad<<<grid_for(n, 256), 256, 0, s>>>(gi, B, Tp, Cp, static_cast<float*>(out), T, C);
  else
    k_token_unpad<<<grid_for(n, 256), 256, 0, s>>>(gi, B, Tp, Cp,
                                                   static_cast<__nv_bfloat16*>(out), T, C);
  return cudaGetLastError();
}

cudaError_t token_fold(const void* y, int64_t B, int64_t Tp, int64_t N, int t, const float* fold,
                       const float* bias, void* out, int64_t T, cudaStream_t s) {
  const int64_t n = B * T * (N / 8);
  if (n == 0) return cudaSuccess;
  k_token_fold<<<grid_for(n, 256), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(y), B, Tp, N, t,
                                                fold, bias, static_cast<__nv_bfloat16*>(out), T);
  return cudaGetLastError();
}

int64_t token_fold_ws_floats(int64_t B, int64_t T, int64_t N, int t) {
  return fold_blocks(B * T) * (N + t);
}

cudaError_t token_fold_backward(const void* gout, const void* y, int64_t B, int64_t Tp,
                                int64_t N, int t, const float* fold, int64_t T, void* g_y,
                                float* g_bias_fold, float* ws, cudaStream_t s) {
  const int64_t rows = B * T;
  if (rows == 0 || N == 0) return cudaMemsetAsync(g_bias_fold, 0, sizeof(float) * (N + t), s);
  const int64_t nb = fold_blocks(rows);
  const int64_t rpb = (rows + nb - 1) / nb;
  const int cpr = static_cast<int>(((N / 8 + 31) / 32) * 32);  // threads per row
  const int nry = cpr >= 256 ? 1 : 256 / cpr;                    // row lanes per block
  const size_t smem = sizeof(float) * nry * N;
  k_token_fold_bwd<<<static_cast<int>(nb), cpr * nry, smem, s>>>(
      static_cast<const __nv_bfloat16*>(gout), static_cast<const __nv_bfloat16*>(y), B, Tp, N, t,
      fold, T, rpb, cpr, static_cast<__nv_bfloat16*>(g_y), ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return sum_partials(ws, static_cast<int>(nb), static_cast<int>(N + t), g_bias_fold, s);
}

}  // namespace stl
