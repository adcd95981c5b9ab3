// stl_transform4.cu — vectorised t = 4 tile transforms (the production tile size).
//
// Same semantics as the generic kernels in stl_transform.cu (encode_tiles snf_operator.py:80-85,
// decode_tiles :88-96, and the g_d / g_ex reductions of _layer_backward toy_network.py:100,104),
// restructured for HBM throughput:
//   * one thread owns 4 horizontally adjacent 4x4 tiles: every tile row is one 32-byte (bf16)
//     or 64-byte (fp32) contiguous segment -> 16-byte vector loads/stores, and each plane write
//     is 4 consecutive coefficients (8 or 16 bytes);
//   * the r x 16 reductions  red[p][c] = sum_tiles plane[p][tile] * tile[c]  run on the tensor
//     cores with warp-level mma.sync m16n8k16 (bf16 in, fp32 accumulate): a warp stages its 128
//     tiles in shared memory (planes split hi+lo bf16, so the fp32 operand keeps ~16 mantissa
//     bits; the tile operand is bf16 data, exact) and reduces over K = tiles with ldmatrix fed
//     MMAs. Partials are combined in a fixed order -> deterministic.
#include "stl_internal.h"

namespace stl {
namespace {

constexpr int kThreads4 = 128;
constexpr int kChunk = 8;                      // planes loaded per batch
// Reducer staging: a warp stages 32 * TPT tiles per round (TPT tiles per lane), rows padded by
// 8 bf16 so ldmatrix row addresses spread over all banks.

template <typename T> struct Vec4;  // four consecutive elements
template <> struct Vec4<float> {
  __device__ static void load(const float* p, float (&v)[4]) {
    const float4 u = *reinterpret_cast<const float4*>(p);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  }
  __device__ static void store(float* p, const float (&v)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct Vec4<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, float (&v)[4]) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    v[0] = fa.x; v[1] = fa.y; v[2] = fb.x; v[3] = fb.y;
  }
  __device__ static void store(__nv_bfloat16* p, const float (&v)[4]) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
    __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = u;
  }
};

// Row segment of 4 tiles x 4 columns = 16 consecutive elements.
template <typename T>
__device__ __forceinline__ void load_row16(const T* p, float (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float w[4];
    Vec4<T>::load(p + 4 * i, w);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[4 * i + j] = w[j];
  }
}
template <typename T>
__device__ __forceinline__ void store_row16(T* p, const float (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float w[4] = {v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]};
    Vec4<T>::store(p + 4 * i, w);
  }
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Per-warp tensor-core reducer for red[p][c] (p < P <= 32, c < 16) over staged tiles.
// Staging (bf16, row stride kStageStride): hi[P] rows, lo[P] rows, x[16] rows, one zero row.
template <int TPT>
struct MmaReducer {
  static constexpr int kStageTiles = 32 * TPT;
  static constexpr int kStageStride = kStageTiles + 8;
  __nv_bfloat16* base;  // this warp's staging area
  int P;
  float acc[2][2][4];   // [m-tile (p 0-15, 16-31)][n-tile (c 0-7, 8-15)][fragment]

  __device__ static int stage_elems(int P) { return (2 * P + 16 + 1) * kStageStride; }

  __device__ void init(__nv_bfloat16* b, int P_) {
    base = b;
    P = P_;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[i][j][k] = 0.f;
    const int lane = threadIdx.x & 31;
    __nv_bfloat16* zero = base + (2 * P + 16) * kStageStride;
    for (int i = lane; i < kStageStride; i += 32) zero[i] = __float2bfloat16_rn(0.f);
  }
  __device__ __nv_bfloat16* hi(int p) const { return base + p * kStageStride; }
  __device__ __nv_bfloat16* lo(int p) const { return base + (P + p) * kStageStride; }
  __device__ __nv_bfloat16* xr(int c) const { return base + (2 * P + c) * kStageStride; }

  // Lane `lane` owns staged tiles TPT*lane .. TPT*lane+TPT-1.
  __device__ void stage_plane(int p, const float (&v)[TPT]) {
    const int col = TPT * (threadIdx.x & 31);
    uint32_t uh[TPT / 2], ul[TPT / 2];
#pragma unroll
    for (int i = 0; i < TPT / 2; ++i) {
      const float h0 = __bfloat162float(__float2bfloat16_rn(v[2 * i]));
      const float h1 = __bfloat162float(__float2bfloat16_rn(v[2 * i + 1]));
      uh[i] = pack_bf16(h0, h1);
      ul[i] = pack_bf16(v[2 * i] - h0, v[2 * i + 1] - h1);
    }
    if constexpr (TPT == 4) {
      *reinterpret_cast<uint2*>(hi(p) + col) = make_uint2(uh[0], uh[1]);
      *reinterpret_cast<uint2*>(lo(p) + col) = make_uint2(ul[0], ul[1]);
    } else {
      *reinterpret_cast<uint32_t*>(hi(p) + col) = uh[0];
      *reinterpret_cast<uint32_t*>(lo(p) + col) = ul[0];
    }
  }
  // x[tile][c] for the lane's TPT tiles.
  __device__ void stage_tiles(const float (&x)[TPT][16]) {
    const int col = TPT * (threadIdx.x & 31);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if constexpr (TPT == 4) {
        *reinterpret_cast<uint2*>(xr(c) + col) =
            make_uint2(pack_bf16(x[0][c], x[1][c]), pack_bf16(x[2][c], x[3][c]));
      } else {
        *reinterpret_cast<uint32_t*>(xr(c) + col) = pack_bf16(x[0][c], x[1][c]);
      }
    }
  }
  __device__ void accumulate() {
    __syncwarp();
    const int lane = threadIdx.x & 31;
    const int mi = lane >> 3;
    const uint32_t zero = ptx_addr(base + (2 * P + 16) * kStageStride);
    // B: rows c, 8 tiles per row; matrices (c0-7,k0-7) (c0-7,k8-15) (c8-15,k0-7) (c8-15,k8-15)
    const int bc = (lane & 7) + ((lane >> 4) << 3);
    const int bk = ((lane >> 3) & 1) * 8;
    // A: rows p, matrices (p0-7,k0-7) (p8-15,k0-7) (p0-7,k8-15) (p8-15,k8-15)
    const int ar = (lane & 7) + (mi & 1) * 8;
    const int ak = (mi >> 1) * 8;
    const int mts = P > 16 ? 2 : 1;
#pragma unroll
    for (int ks = 0; ks < kStageTiles / 16; ++ks) {
      uint32_t b[4];
      ldsm_x4(ptx_addr(xr(bc) + ks * 16 + bk), b);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        if (mt >= mts) break;
        const int p = mt * 16 + ar;
        uint32_t ah[4], al[4];
        ldsm_x4(p < P ? ptx_addr(hi(p) + ks * 16 + ak) : zero + 2 * ak, ah);
        ldsm_x4(p < P ? ptx_addr(lo(p) + ks * 16 + ak) : zero + 2 * ak, al);
        mma16816(acc[mt][0], ah, b[0], b[1]);
        mma16816(acc[mt][0], al, b[0], b[1]);
        mma16816(acc[mt][1], ah, b[2], b[3]);
        mma16816(acc[mt][1], al, b[2], b[3]);
      }
    }
    __syncwarp();
  }
  // Write this warp's [P][16] result into red (fp32, shared).
  __device__ void dump(float* red) const {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int c = nt * 8 + 2 * q;
        const int p0 = mt * 16 + g, p1 = p0 + 8;
        if (p0 < P) {
          red[p0 * 16 + c] = acc[mt][nt][0];
          red[p0 * 16 + c + 1] = acc[mt][nt][1];
        }
        if (p1 < P) {
          red[p1 * 16 + c] = acc[mt][nt][2];
          red[p1 * 16 + c + 1] = acc[mt][nt][3];
        }
      }
  }
  __device__ static uint32_t ptx_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
  }
};

// Shared-memory carve-up: coefficients (P*16 floats), per-warp reducer staging, final sums.
__host__ __device__ inline size_t coef_bytes(int P) { return ((P * 16 * 4) + 15) / 16 * 16; }
template <int TPT>
__host__ __device__ inline size_t stage_bytes(int P) {
  return size_t(4) * (2 * P + 17) * (32 * TPT + 8) * 2;
}
__host__ __device__ inline size_t red_bytes(int P) { return size_t(4) * P * 16 * 4; }

template <bool RED, int TPT>
__device__ __forceinline__ void finish_partial(MmaReducer<TPT>& R, unsigned char* smem, int P,
                                               float* __restrict__ red_partial) {
  if constexpr (RED) {
    float* red = reinterpret_cast<float*>(smem + coef_bytes(P) + stage_bytes<TPT>(P));
    const int warp = threadIdx.x >> 5;
    R.dump(red + warp * P * 16);
    __syncthreads();
    const int n = P * 16;
    for (int o = threadIdx.x; o < n; o += kThreads4)
      red_partial[static_cast<int64_t>(blockIdx.x) * n + o] =
          ((red[o] + red[n + o]) + red[2 * n + o]) + red[3 * n + o];
  }
}

// encode: out[p][I][J] = sum_c coef[p][c] * tile(I, J)[c];  RED: red[p][c] += planes[p] * tile.
template <typename Tin, typename Tout, bool RED, typename Tr>
__global__ void __launch_bounds__(kThreads4)
    k_encode4(const Tin* __restrict__ m, int64_t ldm, int64_t br, int64_t bc,
              const float* __restrict__ coef, int P, Tout* __restrict__ out,
              const Tr* __restrict__ red_planes, float* __restrict__ red_partial) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* sc = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < P * 16; i += kThreads4) sc[i] = coef[i];
  MmaReducer<4> R;
  if constexpr (RED) {
    __nv_bfloat16* st = reinterpret_cast<__nv_bfloat16*>(smem + coef_bytes(P)) +
                        (threadIdx.x >> 5) * MmaReducer<4>::stage_elems(P);
    R.init(st, P);
  }
  __syncthreads();
  const int64_t bq = bc >> 2, nq = br * bq, ntiles = br * bc;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads4; base < nq;
       base += static_cast<int64_t>(gridDim.x) * kThreads4) {
    const int64_t qd = base + threadIdx.x;
    const bool valid = qd < nq;
    float x[4][16];
    int64_t off = 0;
    if (valid) {
      const int64_t I = qd / bq, J0 = (qd - I * bq) * 4;
      off = I * bc + J0;
      const Tin* src = m + I * 4 * ldm + J0 * 4;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        float row[16];
        load_row16(src + a * ldm, row);
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e >> 2][a * 4 + (e & 3)] = row[e];
      }
#pragma unroll 2
      for (int p = 0; p < P; ++p) {
        const float4* cp = reinterpret_cast<const float4*>(sc + p * 16);
        float cf[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 c4 = cp[i];
          cf[4 * i] = c4.x; cf[4 * i + 1] = c4.y; cf[4 * i + 2] = c4.z; cf[4 * i + 3] = c4.w;
        }
        float o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float s = 0.f;
#pragma unroll
          for (int c = 0; c < 16; ++c) s = fmaf(cf[c], x[t][c], s);
          o[t] = s;
        }
        Vec4<Tout>::store(out + p * ntiles + off, o);
      }
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int c = 0; c < 16; ++c) x[t][c] = 0.f;
    }
    if constexpr (RED) {
      for (int p0 = 0; p0 < P; p0 += kChunk) {
        float v[kChunk][4];
#pragma unroll
        for (int j = 0; j < kChunk; ++j) {
          if (valid && p0 + j < P) {
            Vec4<Tr>::load(red_planes + (p0 + j) * ntiles + off, v[j]);
          } else {
            v[j][0] = v[j][1] = v[j][2] = v[j][3] = 0.f;
          }
        }
#pragma unroll
        for (int j = 0; j < kChunk; ++j)
          if (p0 + j < P) R.stage_plane(p0 + j, v[j]);
      }
      R.stage_tiles(x);
      R.accumulate();
    }
  }
  finish_partial<RED, 4>(R, smem, P, red_partial);
}

// decode: out tile(I, J)[c] = sum_q coef[q][c] * in[q][I][J];  RED: red[q][c] += in[q] * tile'.
// One thread owns TPT horizontally adjacent tiles (TPT = 2 keeps registers low enough for
// ~24 resident warps per SM, which this HBM-bound kernel needs to hide latency).
template <int TPT, typename T> struct VecN;
template <> struct VecN<2, float> {
  __device__ static void load(const float* p, float (&v)[2]) {
    const float2 u = *reinterpret_cast<const float2*>(p);
    v[0] = u.x; v[1] = u.y;
  }
};
template <> struct VecN<2, __nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, float (&v)[2]) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
    v[0] = f.x; v[1] = f.y;
  }
};
template <typename T> struct VecN<4, T> {
  __device__ static void load(const T* p, float (&v)[4]) { Vec4<T>::load(p, v); }
};
// a tile-row segment of TPT tiles (4*TPT elements)
template <int TPT, typename T>
__device__ __forceinline__ void store_seg4(T* p, const float (&v)[4 * TPT]) {
#pragma unroll
  for (int i = 0; i < TPT; ++i) {
    const float w[4] = {v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]};
    Vec4<T>::store(p + 4 * i, w);
  }
}
template <int TPT, typename T>
__device__ __forceinline__ void load_seg4(const T* p, float (&v)[4 * TPT]) {
#pragma unroll
  for (int i = 0; i < TPT; ++i) {
    float w[4];
    Vec4<T>::load(p + 4 * i, w);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[4 * i + j] = w[j];
  }
}

template <int TPT, typename Tin, typename Tout, bool RED, typename Tr>
__global__ void __launch_bounds__(kThreads4, RED ? 4 : 6)
    k_decode4(const Tin* __restrict__ in, int Q, int64_t br, int64_t bc,
              const float* __restrict__ coef, Tout* __restrict__ out, int64_t ldo,
              const Tr* __restrict__ red_m, int64_t ldr, float* __restrict__ red_partial) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int kCh = kChunk;
  float* sc = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < Q * 16; i += kThreads4) sc[i] = coef[i];
  MmaReducer<TPT> R;
  if constexpr (RED) {
    __nv_bfloat16* st = reinterpret_cast<__nv_bfloat16*>(smem + coef_bytes(Q)) +
                        (threadIdx.x >> 5) * MmaReducer<TPT>::stage_elems(Q);
    R.init(st, Q);
  }
  __syncthreads();
  const int64_t bq = bc / TPT, nq = br * bq, ntiles = br * bc;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kThreads4; base < nq;
       base += static_cast<int64_t>(gridDim.x) * kThreads4) {
    const int64_t qd = base + threadIdx.x;
    const bool valid = qd < nq;
    int64_t I = 0, J0 = 0, off = 0;
    if (valid) {
      I = qd / bq;
      J0 = (qd - I * bq) * TPT;
      off = I * bc + J0;
      float acc[TPT][16];
#pragma unroll
      for (int t = 0; t < TPT; ++t)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[t][c] = 0.f;
      for (int q0 = 0; q0 < Q; q0 += kCh) {
        float v[kCh][TPT];
#pragma unroll
        for (int j = 0; j < kCh; ++j) {
          if (q0 + j < Q) {
            VecN<TPT, Tin>::load(in + (q0 + j) * ntiles + off, v[j]);
          } else {
#pragma unroll
            for (int t = 0; t < TPT; ++t) v[j][t] = 0.f;
          }
        }
#pragma unroll
        for (int j = 0; j < kCh; ++j) {
          if (q0 + j >= Q) break;
          if constexpr (RED) R.stage_plane(q0 + j, v[j]);
          const float4* cp = reinterpret_cast<const float4*>(sc + (q0 + j) * 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 c4 = cp[i];
            const float cf[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
#pragma unroll
              for (int t = 0; t < TPT; ++t)
                acc[t][4 * i + jj] = fmaf(cf[jj], v[j][t], acc[t][4 * i + jj]);
          }
        }
      }
      Tout* dst = out + I * 4 * ldo + J0 * 4;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        float row[4 * TPT];
#pragma unroll
        for (int e = 0; e < 4 * TPT; ++e) row[e] = acc[e >> 2][a * 4 + (e & 3)];
        store_seg4<TPT>(dst + a * ldo, row);
      }
    } else if constexpr (RED) {
      float z[TPT];
#pragma unroll
      for (int t = 0; t < TPT; ++t) z[t] = 0.f;
      for (int q = 0; q < Q; ++q) R.stage_plane(q, z);
    }
    if constexpr (RED) {
      float x[TPT][16];
      if (valid) {
        const Tr* src = red_m + I * 4 * ldr + J0 * 4;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          float row[4 * TPT];
          load_seg4<TPT>(src + a * ldr, row);
#pragma unroll
          for (int e = 0; e < 4 * TPT; ++e) x[e >> 2][a * 4 + (e & 3)] = row[e];
        }
      } else {
#pragma unroll
        for (int t = 0; t < TPT; ++t)
#pragma unroll
          for (int c = 0; c < 16; ++c) x[t][c] = 0.f;
      }
      R.stage_tiles(x);
      R.accumulate();
    }
  }
  finish_partial<RED, TPT>(R, smem, Q, red_partial);
}

// out[o] = sum_b partial[b][o]: one block per output, fixed-order tree (deterministic).
__global__ void __launch_bounds__(256) k_sum_partials_tree(const float* __restrict__ partial,
                                                           int nblocks, int n,
                                                           float* __restrict__ out) {
  __shared__ float s[256];
  griddep_launch_dependents();
  griddep_wait();  // the partials of the preceding launch are complete (PDL)
  const int o = blockIdx.x;
  float v = 0.f;
  for (int b = threadIdx.x; b < nblocks; b += 256) v += partial[static_cast<int64_t>(b) * n + o];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[o] = s[0];
}

int grid4(int64_t nq, int cap) {
  int64_t g = (nq + kThreads4 - 1) / kThreads4;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

template <typename K>
cudaError_t prep(K k, size_t smem) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

template <typename Tin, typename Tout, typename Tr>
cudaError_t enc4_red(const void* m, int64_t ldm, int64_t br, int64_t bc, const float* coef, int P,
                     void* out, const void* rp, float* ro, float* rw, cudaStream_t s) {
  const int64_t nq = br * (bc / 4);
  const size_t smem = coef_bytes(P) + stage_bytes<4>(P) + red_bytes(P);
  auto k = k_encode4<Tin, Tout, true, Tr>;
  if (cudaError_t e = prep(k, smem)) return e;
  const int grid = grid4(nq, sm_count() * 3);
  k<<<grid, kThreads4, smem, s>>>(static_cast<const Tin*>(m), ldm, br, bc, coef, P,
                                  static_cast<Tout*>(out), static_cast<const Tr*>(rp), rw);
  k_sum_partials_tree<<<P * 16, 256, 0, s>>>(rw, grid, P * 16, ro);
  return cudaGetLastError();
}

template <typename Tin, typename Tout>
cudaError_t enc4(const void* m, int64_t ldm, int64_t br, int64_t bc, const float* coef, int P,
                 void* out, const void* rp, int rdt, float* ro, float* rw, cudaStream_t s) {
  const int64_t nq = br * (bc / 4);
  if (rp) {
    if (rdt == kBF16)
      return enc4_red<Tin, Tout, __nv_bfloat16>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
    return enc4_red<Tin, Tout, float>(m, ldm, br, bc, coef, P, out, rp, ro, rw, s);
  } else {
    const size_t smem = coef_bytes(P);
    auto k = k_encode4<Tin, Tout, false, float>;
    if (cudaError_t e = prep(k, smem)) return e;
    k<<<grid4(nq, sm_count() * 16), kThreads4, smem, s>>>(
        static_cast<const Tin*>(m), ldm, br, bc, coef, P, static_cast<Tout*>(out), nullptr,
        nullptr);
  }
  return cudaGetLastError();
}

template <typename Tin, typename Tout>
cudaError_t dec4(const void* in, int Q, int64_t br, int64_t bc, const float* coef, void* out,
                 int64_t ldo, const void* rm, int64_t ldr, float* ro, float* rw, cudaStream_t s) {
  constexpr int TPT = 2;
  const int64_t nq = br * (bc / TPT);
  if (rm) {
    const size_t smem = coef_bytes(Q) + stage_bytes<TPT>(Q) + red_bytes(Q);
    auto k = k_decode4<TPT, Tin, Tout, true, __nv_bfloat16>;
    if (cudaError_t e = prep(k, smem)) return e;
    const int grid = grid4(nq, sm_count() * 5);
    k<<<grid, kThreads4, smem, s>>>(static_cast<const Tin*>(in), Q, br, bc, coef,
                                    static_cast<Tout*>(out), ldo,
                                    static_cast<const __nv_bfloat16*>(rm), ldr, rw);
    k_sum_partials_tree<<<Q * 16, 256, 0, s>>>(rw, grid, Q * 16, ro);
  } else {
    const size_t smem = coef_bytes(Q);
    auto k = k_decode4<TPT, Tin, Tout, false, __nv_bfloat16>;
    if (cudaError_t e = prep(k, smem)) return e;
    k<<<grid4(nq, sm_count() * 16), kThreads4, smem, s>>>(
        static_cast<const Tin*>(in), Q, br, bc, coef, static_cast<Tout*>(out), ldo, nullptr, 0,
        nullptr);
  }
  return cudaGetLastError();
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// out[o] = sum_b partial[b][o], 32 outputs per block: warp w sums partials b = w, w + 16, ...
// of its lane's output (each warp load one 128-byte row segment, all of a thread's loads
// independent), then lane l of warp 0 adds the 16 warp sums in order — a fixed order
// (deterministic); 12 blocks for the r = 24 reductions instead of 384 one-output trees.
__global__ void __launch_bounds__(512) k_sum_partials_cols(const float* __restrict__ partial,
                                                           int nblocks, int n,
                                                           float* __restrict__ out) {
  __shared__ float s[16][33];
  griddep_launch_dependents();
  griddep_wait();  // the partials of the preceding launch are complete (PDL)
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int o = blockIdx.x * 32 + l;
  float v0 = 0.f, v1 = 0.f;
  if (o < n) {
    int b = w;
    for (; b + 16 < nblocks; b += 32) {
      v0 += partial[static_cast<int64_t>(b) * n + o];
      v1 += partial[static_cast<int64_t>(b + 16) * n + o];
    }
    if (b < nblocks) v0 += partial[static_cast<int64_t>(b) * n + o];
  }
  s[w][l] = v0 + v1;
  __syncthreads();
  if (w == 0 && o < n) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) t += s[k][l];
    out[o] = t;
  }
}

cudaError_t sum_partials(const float* partial, int nblocks, int n, float* out, cudaStream_t s) {
  return launch_pdl(k_sum_partials_cols, dim3((n + 31) / 32), dim3(512), 0, s, partial, nblocks,
                    n, out);
}

// Fast-path dispatch; returns cudaErrorNotSupported when the generic kernels must be used.
cudaError_t tiles_to_planes4(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                             const float* coef, int P, void* out, int odt, const void* rp,
                             int rdt, float* ro, float* rw, cudaStream_t s) {
  if (bc % 4 || ldm % 8 || !aligned16(m) || !aligned16(out)) return cudaErrorNotSupported;
  if (rp && (mdt != kBF16 || P > 32 || !aligned16(rp))) return cudaErrorNotSupported;
  if (mdt == kBF16 && odt == kBF16)
    return enc4<__nv_bfloat16, __nv_bfloat16>(m, ldm, br, bc, coef, P, out, rp, rdt, ro, rw, s);
  if (mdt == kBF16)
    return enc4<__nv_bfloat16, float>(m, ldm, br, bc, coef, P, out, rp, rdt, ro, rw, s);
  if (rp) return cudaErrorNotSupported;
  if (odt == kBF16)
    return enc4<float, __nv_bfloat16>(m, ldm, br, bc, coef, P, out, nullptr, 0, ro, rw, s);
  return enc4<float, float>(m, ldm, br, bc, coef, P, out, nullptr, 0, ro, rw, s);
}

__global__ void k_cast_f32_bf16(const float* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

cudaError_t cast_f32_to_bf16(const float* in, void* out, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int64_t g = (n + 255) / 256;
  if (g > sm_count() * 32) g = sm_count() * 32;
  k_cast_f32_bf16<<<static_cast<int>(g), 256, 0, s>>>(in, static_cast<__nv_bfloat16*>(out), n);
  return cudaGetLastError();
}

cudaError_t planes_to_tiles4(const void* in, int idt, int Q, int64_t br, int64_t bc,
                             const float* coef, void* out, int odt, int64_t ldo, const void* rm,
                             int rdt, int64_t ldr, float* ro, float* rw, cudaStream_t s) {
  if (bc % 4 || ldo % 8 || !aligned16(in) || !aligned16(out)) return cudaErrorNotSupported;
  if (rm && (rdt != kBF16 || Q > 32 || ldr % 8 || !aligned16(rm))) return cudaErrorNotSupported;
  if (idt == kF32 && odt == kBF16)
    return dec4<float, __nv_bfloat16>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
  if (idt == kF32 && odt == kF32)
    return dec4<float, float>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
  if (idt == kBF16 && odt == kBF16)
    return dec4<__nv_bfloat16, __nv_bfloat16>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
  return dec4<__nv_bfloat16, float>(in, Q, br, bc, coef, out, ldo, rm, ldr, ro, rw, s);
}

}  // namespace stl
