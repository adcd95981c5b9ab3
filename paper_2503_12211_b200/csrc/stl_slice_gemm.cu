// stl_slice_gemm.cu — the STL contraction: r independent slice GEMMs C_p = A_p · B_p.
//
// Reference semantics: `_slice_products` (snf_operator.py:107-116),
//   out[:, :, p] = x_enc[:, :, p] @ w_enc[:, :, p]   for every p,
// i.e. Claim 1 / Algorithm 1 step 2 of the paper.
//
// B200 design:
//   * persistent, warp-specialised kernel, one CTA per SM (grid = #SMs), static tile schedule
//     over (slice p, M-block, N-block);
//   * warp 0 lane 0 = TMA producer: 3-D tensor maps (inner, outer, slice) load 128x64 A and
//     BNx64 B boxes with 128-byte swizzle into a 4-stage shared-memory ring;
//   * warp 1 lane 0 = MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16,
//     bf16 operands straight from shared memory, fp32 accumulators in TMEM;
//   * warp 2 owns the TMEM allocation (2 x BN columns: accumulator double buffer so the
//     epilogue of tile i overlaps the main loop of tile i+1);
//   * warps 4..7 = epilogue: tcgen05.ld 32 lanes x 32 columns, fp32 (or bf16) stores.
// Both operands may be K-major or MN-major (the backward pass needs MN-major operands for
// g_u = g_enc_p W_p^T and g_w = u_p^T g_enc_p), selected by the UMMA instruction descriptor.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <vector>
#include "sm100_ptx.cuh"
#include "stl_internal.h"

namespace stl {

namespace {
constexpr int kBM = 128;
constexpr int kBK = 64;   // 64 bf16 = 128 bytes = one swizzle row
constexpr int kStages = 4;
constexpr int kThreads = 256;

struct EpiArgs {
  void* c;
  int c_bf16;
  int nostore;  // probe: skip the C stores (measures the mainloop alone)
  int unused;
  int r;
  int M, N, K;
  __nv_bfloat16* c2;  // optional bf16 copy of C (the forward's training cache)
};

template <int BN>
struct Smem {
  static constexpr uint32_t kABytes = kBM * kBK * 2;
  static constexpr uint32_t kBBytes = BN * kBK * 2;
  static constexpr uint32_t kBarOffset = kStages * (kABytes + kBBytes);
  static constexpr uint32_t kTotal = kBarOffset + 256 + 1024;  // barriers + alignment slack
};

__device__ __forceinline__ void store_row_chunk(float* dst, const uint32_t (&v)[32], int ncols,
                                                bool vec) {
  if (vec && ncols >= 32) {
    float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      d4[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                          __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) dst[i] = __uint_as_float(v[i]);
  }
}

__device__ __forceinline__ void store_row_chunk(__nv_bfloat16* dst, const uint32_t (&v)[32],
                                                int ncols, bool vec) {
  if (vec && ncols >= 32) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[8 * i + 2 * j]),
                                                 __uint_as_float(v[8 * i + 2 * j + 1]));
        w[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      d4[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) dst[i] = __float2bfloat16_rn(__uint_as_float(v[i]));
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    slice_gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB, EpiArgs args) {
  using S = Smem<BN>;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(kBM, BN, A_MN, B_MN);
  constexpr uint32_t kTmemCols = (2 * BN <= 256) ? 256 : 512;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * S::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = args.M, N = args.N, K = args.K;
  const int m_tiles = (M + kBM - 1) / kBM;
  const int n_tiles = (N + BN - 1) / BN;
  const int per_slice = m_tiles * n_tiles;
  const int total = args.r * per_slice;
  const int num_kb = (K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int p = tile / per_slice;
        const int rem = tile - p * per_slice;
        const int mb = rem / n_tiles;
        const int nb = rem - mb * n_tiles;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], S::kABytes + S::kBBytes);
          uint8_t* a = sA + stage * S::kABytes;
          uint8_t* b = sB + stage * S::kBBytes;
          if constexpr (!A_MN) {
            ptx::tma_load_3d(&tmA, &full[stage], a, kb * kBK, mb * kBM, p);
          } else {
#pragma unroll
            for (int j = 0; j < kBM / 64; ++j)
              ptx::tma_load_3d(&tmA, &full[stage], a + j * (64 * kBK * 2), mb * kBM + j * 64,
                               kb * kBK, p);
          }
          if constexpr (!B_MN) {
            ptx::tma_load_3d(&tmB, &full[stage], b, kb * kBK, nb * BN, p);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              ptx::tma_load_3d(&tmB, &full[stage], b + j * (64 * kBK * 2), nb * BN + j * 64,
                               kb * kBK, p);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(sA + stage * S::kABytes);
          const uint32_t b_addr = ptx::smem_u32(sB + stage * S::kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // K-major: step 16 elements = 32 bytes inside the 128-byte swizzle row.
            // MN-major: step 16 K-rows of 128 bytes; 64-wide MN atoms are 64*kBK*2 apart.
            const uint64_t ad = A_MN ? ptx::smem_desc_sw128(a_addr + k * 2048, 64 * kBK * 2, 1024)
                                     : ptx::smem_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::smem_desc_sw128(b_addr + k * 2048, 64 * kBK * 2, 1024)
                                     : ptx::smem_desc_sw128(b_addr + k * 32, 16, 1024);
            ptx::mma_bf16_ss(d_tmem, ad, bd, kIdesc, (kb | k) != 0 ? 1u : 0u);
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const bool c_vec = (N % 4 == 0) && ((reinterpret_cast<uintptr_t>(args.c) & 15) == 0) &&
                       (args.c_bf16 ? (N % 8 == 0) : true);
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      const int p = tile / per_slice;
      const int rem = tile - p * per_slice;
      const int mb = rem / n_tiles;
      const int nb = rem - mb * n_tiles;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int row = mb * kBM + q * 32 + lane;
      const size_t row_off = (static_cast<size_t>(p) * M + row) * static_cast<size_t>(N);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t v[32];
        __syncwarp();
        ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c,
                                v);
        ptx::tmem_ld_wait();
        const int col0 = nb * BN + c;
        if (row < M && col0 < N) {
          if (args.c_bf16)
            store_row_chunk(reinterpret_cast<__nv_bfloat16*>(args.c) + row_off + col0, v,
                            N - col0, c_vec);
          else
            store_row_chunk(reinterpret_cast<float*>(args.c) + row_off + col0, v, N - col0,
                            c_vec);
          if (args.c2) store_row_chunk(args.c2 + row_off + col0, v, N - col0, N % 8 == 0);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, kTmemCols);
}


// ==================================================================== CTA-pair variant
// cta_group::2: a cluster of 2 CTAs (one TPC) computes a 256 x BN tile. Each CTA stages its
// 128 rows of A and its BN/2 columns of B (half the B bytes per SM of the 1-CTA kernel, and
// 32 KB stages -> a 6-deep ring); the even CTA issues tcgen05.mma.cta_group::2 for both, and
// each CTA's epilogue drains its own 128 TMEM lanes.
// Output modes of the pair kernel: fp32 C; fp32 C plus a bf16 copy (c2); or F24 — fp32 rounded
// to 24 bits and stored as a 16-bit high plane set (c) followed by an 8-bit low plane set
// (c + 2 * r * M * N bytes), 3 bytes per element at ~2^-16 relative precision.
enum OutMode { kOutF32 = 0, kOutF32Bf16 = 1, kOutF24 = 2, kOutBf16 = 3 };

// Per-problem compile-time traits of the pair kernel: operand majorness and output mode.
template <bool A_MN_, bool B_MN_, int OUT_>
struct GemmKind {
  static constexpr bool A_MN = A_MN_, B_MN = B_MN_;
  static constexpr int OUT = OUT_;
};

// Epilogue staging of one output mode: 128 rows (the CTA's TMEM lanes) x 32 columns (64 for
// bf16 output), a primary part (fp32 or bf16 128 B rows, or F24 high 64 B rows) and a secondary
// part at kSecOff (the bf16 copy's 64 B rows, or F24 low 32 B rows).
template <int OUT>
struct OutStage {
  static constexpr uint32_t kSecOff = OUT == kOutF24 ? 128 * 64 : 128 * 128;
  static constexpr uint32_t kBytes =
      kSecOff + (OUT == kOutF32Bf16 ? 128 * 64 : (OUT == kOutF24 ? 128 * 32 : 0));
};

template <int BN, int OUT0, int OUT1, int ST = 0>
struct Smem2 {
  // ring depth chosen so ring + epilogue staging fits the 227 KB opt-in limit (ST > 0: forced)
  static constexpr bool kDual = OUT0 == kOutF32Bf16 || OUT1 == kOutF32Bf16;
  static constexpr int kStages = ST > 0 ? ST : (BN == 256 ? (kDual ? 5 : 6) : (kDual ? 7 : 8));
  static constexpr uint32_t kABytes = 128 * kBK * 2;
  static constexpr uint32_t kBBytes = (BN / 2) * kBK * 2;
  static constexpr uint32_t kRing = kStages * (kABytes + kBBytes);
  static constexpr uint32_t kBufBytes = OutStage<OUT0>::kBytes > OutStage<OUT1>::kBytes
                                            ? OutStage<OUT0>::kBytes
                                            : OutStage<OUT1>::kBytes;
  static constexpr uint32_t kBarOffset = kRing + 2 * kBufBytes;  // two staging buffers
  static constexpr uint32_t kTotal = kBarOffset + 512 + 1024;
};

// fp32 -> 24-bit round-to-nearest-even bit pattern (low 8 bits zero)
__device__ __forceinline__ uint32_t rne24(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u + 0x7Fu + ((u >> 8) & 1u)) & 0xFFFFFF00u;
}

// A group of up to two slice-GEMM problems sharing r, run by one persistent launch: tiles
// [0, total0) belong to problem 0, [total0, total) to problem 1 (the backward's g_w and g_u
// GEMMs: one launch, one tail, and the longer-K problem scheduled first).
struct GroupArgs {
  int M[2], N[2], K[2];
  int r;
  int total0, total;
  int nostore;
  Trace trace;  // probe: launch span
  // Tile order: rounds of nclusters tiles; -1 = every round left to right (round robin:
  // tile = cluster + k * nclusters); 0 / 1 = alternating directions (snake; round 0 left to
  // right when 0); 2 = left to right except the last round. For groups whose tiles have
  // different K (the backward's g_w and g_u) the host picks the order whose busiest cluster
  // has the fewest K-blocks (config 2: 352 -> 336 K-blocks against a mean of 332).
  int order;
};

// k-th tile of cluster c in the group's order (>= total: done).
__device__ __forceinline__ int group_tile(const GroupArgs& g, int c, int nc, int k) {
  bool rev;
  if (g.order < 0) rev = false;
  else if (g.order == 2) rev = k == (g.total + nc - 1) / nc - 1;
  else rev = ((k + g.order) & 1) != 0;
  return k * nc + (rev ? nc - 1 - c : c);
}

// Tile `tile` of a group: problem, slice, 256-row block, BN-column block.
template <int BN>
struct TileCoord {
  int prob, p, mb, nb, num_kb;
  __device__ __forceinline__ TileCoord(const GroupArgs& g, int tile) {
    prob = tile >= g.total0 ? 1 : 0;
    const int local = prob ? tile - g.total0 : tile;
    const int n_tiles = (g.N[prob] + BN - 1) / BN;
    const int per_slice = ((g.M[prob] + 255) / 256) * n_tiles;
    p = local / per_slice;
    const int rem = local - p * per_slice;
    mb = rem / n_tiles;
    nb = rem - mb * n_tiles;
    num_kb = (g.K[prob] + kBK - 1) / kBK;
  }
};

// TMA producer for one tile (both CTAs: each loads its 128 rows of A and BN/2 columns of B).
template <int BN, class Kd, class S>
__device__ __forceinline__ void tc2_produce(const CUtensorMap* tmA, const CUtensorMap* tmB,
                                            uint8_t* sA, uint8_t* sB, uint64_t* full,
                                            uint64_t* empty, int& stage, uint32_t& phase,
                                            const TileCoord<BN>& tc, uint32_t prank) {
  const bool leader = prank == 0;
  const int m0 = tc.mb * 256 + static_cast<int>(prank) * 128;
  const int n0 = tc.nb * BN + static_cast<int>(prank) * (BN / 2);
  for (int kb = 0; kb < tc.num_kb; ++kb) {
    ptx::mbar_wait(&empty[stage], phase ^ 1);
    if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (S::kABytes + S::kBBytes));
    uint8_t* a = sA + stage * S::kABytes;
    uint8_t* b = sB + stage * S::kBBytes;
    if constexpr (!Kd::A_MN) {
      ptx::tma_load_3d_2sm(tmA, &full[stage], a, kb * kBK, m0, tc.p);
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j)
        ptx::tma_load_3d_2sm(tmA, &full[stage], a + j * (64 * kBK * 2), m0 + j * 64, kb * kBK,
                             tc.p);
    }
    if constexpr (!Kd::B_MN) {
      ptx::tma_load_3d_2sm(tmB, &full[stage], b, kb * kBK, n0, tc.p);
    } else {
#pragma unroll
      for (int j = 0; j < BN / 128; ++j)
        ptx::tma_load_3d_2sm(tmB, &full[stage], b + j * (64 * kBK * 2), n0 + j * 64, kb * kBK,
                             tc.p);
    }
    if (!leader) ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&full[stage]), 0u));
    if (++stage == S::kStages) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// MMA issue for one tile (even CTA, one thread): num_kb x (kBK / 16) cta_group::2 MMAs.
template <int BN, class Kd, class S>
__device__ __forceinline__ void tc2_mma(uint8_t* sA, uint8_t* sB, uint64_t* full,
                                        uint64_t* empty, int& stage, uint32_t& phase,
                                        uint32_t d_tmem, int num_kb) {
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(256, BN, Kd::A_MN, Kd::B_MN);
  for (int kb = 0; kb < num_kb; ++kb) {
    ptx::mbar_wait(&full[stage], phase);
    ptx::tc_fence_after();
    const uint32_t a_addr = ptx::smem_u32(sA + stage * S::kABytes);
    const uint32_t b_addr = ptx::smem_u32(sB + stage * S::kBBytes);
#pragma unroll
    for (int k = 0; k < kBK / 16; ++k) {
      const uint64_t ad = Kd::A_MN ? ptx::smem_desc_sw128(a_addr + k * 2048, 64 * kBK * 2, 1024)
                                   : ptx::smem_desc_sw128(a_addr + k * 32, 16, 1024);
      const uint64_t bd = Kd::B_MN ? ptx::smem_desc_sw128(b_addr + k * 2048, 64 * kBK * 2, 1024)
                                   : ptx::smem_desc_sw128(b_addr + k * 32, 16, 1024);
      ptx::mma_bf16_ss_2sm(d_tmem, ad, bd, kIdesc, (kb | k) != 0 ? 1u : 0u);
    }
    ptx::mma_commit_2sm(&empty[stage], 0x3);
    if (++stage == S::kStages) {
      stage = 0;
      phase ^= 1;
    }
  }
}

// Epilogue for one tile (4 warps per CTA): TMEM -> registers -> swizzled smem staging of the
// CTA's 128 rows x 32 columns (each warp writes its 32 TMEM lanes) -> one TMA store per plane
// set and chunk, issued by one thread after a 128-thread barrier (few, large TMA ops: the TMA
// unit also feeds the mainloop). TMA clips rows >= M / cols >= N. Two staging buffers.
// BN = the accumulator's columns drained here; `col_base` = output column of its column 0.
template <int BN, class Kd, class S>
__device__ __forceinline__ void tc2_epilogue(const CUtensorMap* tmC, const CUtensorMap* tmC2,
                                             uint8_t* stage_base, uint32_t tmem_acc,
                                             int& chunk_no, int p, int col_base,
                                             int row_base, int M, int N, bool nostore, int q,
                                             int lane, bool issuer) {
  constexpr int OUT = Kd::OUT;
  constexpr uint32_t kSec = OutStage<OUT>::kSecOff;
  const int r = q * 32 + lane;  // staging row = TMEM lane
  // bf16 output drains 64 columns per chunk (128 B staging rows, half the barriers / stores)
  constexpr int kCols = OUT == kOutBf16 ? 64 : 32;
#pragma unroll 1
  for (int c = 0; c < BN; c += kCols, ++chunk_no) {
    uint32_t v[32], v2[32];
    __syncwarp();
    ptx::tmem_ld_32x32b_x32(tmem_acc + c, v);
    if constexpr (kCols == 64) ptx::tmem_ld_32x32b_x32(tmem_acc + c + 32, v2);
    uint8_t* sf = stage_base + (chunk_no & 1) * S::kBufBytes;
    ptx::tmem_ld_wait();
    const bool active = col_base + c < N && row_base < M && !nostore;  // CTA-uniform
    if (active) {
      if constexpr (OUT == kOutF24) {
        // high 16 bits: 64 B rows, 64B-swizzled; low 8 bits: 32 B rows, 32B-swizzled
        uint8_t* sh = sf + kSec;
        uint32_t hw[16], lw[8];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const uint32_t a = rne24(__uint_as_float(v[2 * e])),
                         b = rne24(__uint_as_float(v[2 * e + 1]));
          hw[e] = (a >> 16) | (b & 0xFFFF0000u);
          const uint32_t lo2 = ((a >> 8) & 0xFFu) | (b & 0xFF00u);  // two low bytes
          if (e & 1) lw[e >> 1] |= lo2 << 16;
          else lw[e >> 1] = lo2;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(sf + r * 64 + ((j ^ ((r >> 1) & 3)) << 4)) =
              make_uint4(hw[4 * j], hw[4 * j + 1], hw[4 * j + 2], hw[4 * j + 3]);
#pragma unroll
        for (int j = 0; j < 2; ++j)
          *reinterpret_cast<uint4*>(sh + r * 32 + ((j ^ ((r >> 2) & 1)) << 4)) =
              make_uint4(lw[4 * j], lw[4 * j + 1], lw[4 * j + 2], lw[4 * j + 3]);
      } else if constexpr (OUT == kOutBf16) {
        // bf16 only: 64 columns = 128 B rows, 128B-swizzled (16-byte chunk j at j ^ (r & 7))
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t* src = j < 4 ? v + 8 * j : v2 + 8 * (j - 4);
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(src[2 * e]),
                                                     __uint_as_float(src[2 * e + 1]));
            w[e] = *reinterpret_cast<uint32_t*>(&h);
          }
          *reinterpret_cast<uint4*>(sf + r * 128 + ((j ^ (r & 7)) << 4)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<float4*>(sf + r * 128 + ((j ^ (r & 7)) << 4)) =
              make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                          __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
      }
      if constexpr (OUT == kOutF32Bf16) {
        uint8_t* sh = sf + kSec;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[8 * j + 2 * e]),
                                                     __uint_as_float(v[8 * j + 2 * e + 1]));
            w[e] = *reinterpret_cast<uint32_t*>(&h);
          }
          *reinterpret_cast<uint4*>(sh + r * 64 + ((j ^ ((r >> 1) & 3)) << 4)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      ptx::fence_proxy_async_smem();
    }
    // the previous chunk's store must be done reading the other buffer (written next chunk)
    if (issuer) ptx::bulk_wait_read<0>();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (issuer && active) {
      ptx::tma_store_3d(tmC, sf, col_base + c, row_base, p);
      if constexpr (OUT == kOutF32Bf16 || OUT == kOutF24)
        ptx::tma_store_3d(tmC2, sf + kSec, col_base + c, row_base, p);
      ptx::bulk_commit();
    }
  }
}

template <int BN, class K0, class K1, int ST = 0>
__global__ void __launch_bounds__(kThreads, 1)
    slice_gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA0,
                          const __grid_constant__ CUtensorMap tmB0,
                          const __grid_constant__ CUtensorMap tmC0,
                          const __grid_constant__ CUtensorMap tmC20,
                          const __grid_constant__ CUtensorMap tmA1,
                          const __grid_constant__ CUtensorMap tmB1,
                          const __grid_constant__ CUtensorMap tmC1,
                          const __grid_constant__ CUtensorMap tmC21, GroupArgs args) {
  using S = Smem2<BN, K0::OUT, K1::OUT, ST>;
  constexpr int kSt = S::kStages;
  constexpr uint32_t kTmemCols = (2 * BN <= 256) ? 256 : 512;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kSt * S::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::kBarOffset);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t prank = ptx::cluster_ctarank();  // 0 (leader: issues the pair MMAs) or 1
  const bool leader = prank == 0;
  const int cluster = blockIdx.x / 2, nclusters = gridDim.x / 2;
  const int total = args.total;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA0);
    ptx::prefetch_tmap(&tmB0);
    if (args.total > args.total0) {
      ptx::prefetch_tmap(&tmA1);
      ptx::prefetch_tmap(&tmB1);
    }
  }
  if (warp == 1 && lane == 0) {
    trace_mark(args.trace, false);
    for (int s = 0; s < kSt; ++s) {
      ptx::mbar_init(&full[s], 2);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], 8);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_2sm(tmem_slot, kTmemCols);
  griddep_launch_dependents();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // operands of this launch are complete (PDL)

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int kk = 0, tile = group_tile(args, cluster, nclusters, 0); tile < total;
           tile = group_tile(args, cluster, nclusters, ++kk)) {
        const TileCoord<BN> tc(args, tile);
        if (tc.prob == 0)
          tc2_produce<BN, K0, S>(&tmA0, &tmB0, sA, sB, full, empty, stage, phase, tc, prank);
        else
          tc2_produce<BN, K1, S>(&tmA1, &tmB1, sA, sB, full, empty, stage, phase, tc, prank);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------------------ MMA issuer (even CTA)
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int kk = 0, tile = group_tile(args, cluster, nclusters, 0); tile < total;
           tile = group_tile(args, cluster, nclusters, ++kk), ++it) {
        const TileCoord<BN> tc(args, tile);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        if (tc.prob == 0)
          tc2_mma<BN, K0, S>(sA, sB, full, empty, stage, phase, d_tmem, tc.num_kb);
        else
          tc2_mma<BN, K1, S>(sA, sB, full, empty, stage, phase, d_tmem, tc.num_kb);
        ptx::mma_commit_2sm(&tfull[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    const bool issuer = warp == 4 && lane == 0;
    int chunk_no = 0;
    int it = 0;
    uint8_t* stage_base = smem + S::kRing;
    for (int kk = 0, tile = group_tile(args, cluster, nclusters, 0); tile < total;
         tile = group_tile(args, cluster, nclusters, ++kk), ++it) {
      const TileCoord<BN> tc(args, tile);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int row_base = tc.mb * 256 + static_cast<int>(prank) * 128;
      const uint32_t tmem_acc = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
      if (tc.prob == 0)
        tc2_epilogue<BN, K0, S>(&tmC0, &tmC20, stage_base, tmem_acc, chunk_no, tc.p, tc.nb * BN, row_base,
                                args.M[0], args.N[0], args.nostore, q, lane, issuer);
      else
        tc2_epilogue<BN, K1, S>(&tmC1, &tmC21, stage_base, tmem_acc, chunk_no, tc.p, tc.nb * BN, row_base,
                                args.M[1], args.N[1], args.nostore, q, lane, issuer);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0)
        ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&tempty[acc]), 0u));
    }
    if (issuer) ptx::bulk_wait_all();
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_2sm(tmem_base, kTmemCols);
  if (threadIdx.x == 0) trace_mark(args.trace, true);
}

// ------------------------------------------------------------------ host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool make_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t slices,
               uint32_t box_outer, uint64_t slice_bytes = 0) {
  return make_bf16_tmap(m, base, inner, outer, slices, 64, box_outer, slice_bytes);
}

template <int BN, bool A_MN, bool B_MN>
cudaError_t launch_tc(const SliceGemmProblem& pb, cudaStream_t s) {
  CUtensorMap ta, tb;
  const uint64_t M = pb.M, N = pb.N, K = pb.K, r = pb.r;
  bool ok = A_MN ? make_tmap(&ta, pb.a, M, K, r, kBK) : make_tmap(&ta, pb.a, K, M, r, kBM);
  ok = ok && (B_MN ? make_tmap(&tb, pb.b, N, K, r, kBK) : make_tmap(&tb, pb.b, K, N, r, BN));
  if (!ok) return cudaErrorInvalidValue;
  auto kern = slice_gemm_tc_kernel<BN, A_MN, B_MN>;
  const int smem = Smem<BN>::kTotal;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t tiles = r * ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int grid = static_cast<int>(tiles < sm_count() ? tiles : sm_count());
  EpiArgs ea{pb.c, pb.c_dtype == kBF16 ? 1 : 0, 0, 0, pb.r, static_cast<int>(M), static_cast<int>(N),
             static_cast<int>(K), static_cast<__nv_bfloat16*>(pb.c2)};
  kern<<<grid, kThreads, smem, s>>>(ta, tb, ea);
  return cudaGetLastError();
}


// 3-D (N, M, r) store map for 128-row x 32-column output chunks: es = 4 (fp32, 128B swizzle),
// 2 (16-bit, 64B swizzle) or 1 (8-bit, 32B swizzle).
bool make_out_tmap(CUtensorMap* m, const void* base, int es, uint64_t N, uint64_t M, uint64_t r,
                   uint32_t cols = 32, uint64_t slice_rows = 0) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {N, M, r};
  cuuint64_t strides[2] = {N * es, N * (slice_rows ? slice_rows : M) * es};
  cuuint32_t box[3] = {cols, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType dt = es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const uint32_t row_bytes = cols * es;  // the staging rows: 128, 64 or 32 bytes
  const CUtensorMapSwizzle sw = row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                  : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult res = fn(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

struct Tc2Maps {
  CUtensorMap a, b, c, c2;
};

template <int BN, class Kd>
bool make_tc2_maps(const SliceGemmProblem& pb, Tc2Maps* m) {
  const uint64_t M = pb.M, N = pb.N, K = pb.K, r = pb.r;
  // K-major A: one 128-row box per CTA
  bool ok = Kd::A_MN ? make_tmap(&m->a, pb.a, M, K, r, kBK) : make_tmap(&m->a, pb.a, K, M, r, 128);
  ok = ok && (Kd::B_MN ? make_tmap(&m->b, pb.b, N, K, r, kBK)
                       : make_tmap(&m->b, pb.b, K, N, r, BN / 2));
  if (Kd::OUT == kOutBf16) {
    ok = ok && make_out_tmap(&m->c, pb.c, 2, N, M, r, 64);  // 64-column chunks, 128 B rows
    m->c2 = m->c;
  } else if (Kd::OUT == kOutF24) {
    ok = ok && make_out_tmap(&m->c, pb.c, 2, N, M, r) &&
         make_out_tmap(&m->c2, static_cast<uint8_t*>(pb.c) + 2 * r * M * N, 1, N, M, r);
  } else {
    ok = ok && make_out_tmap(&m->c, pb.c, 4, N, M, r);
    if (Kd::OUT == kOutF32Bf16) ok = ok && make_out_tmap(&m->c2, pb.c2, 2, N, M, r);
    else m->c2 = m->c;
  }
  return ok;
}

int64_t tc2_tiles(const SliceGemmProblem& pb, int BN) {
  return static_cast<int64_t>(pb.r) * ((pb.M + 255) / 256) * ((pb.N + BN - 1) / BN);
}

// Launch config of the persistent CTA-pair kernels: clusters of 2 (one TPC), as many as can be
// co-resident, programmatic dependent launch.
struct PairLaunch {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  PairLaunch(int smem, cudaStream_t s) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
  }
  template <class Kern>
  int max_clusters(Kern kern) {
    cfg.gridDim = dim3(2 * (sm_count() / 2));
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = sm_count() / 2;
    return n;
  }
};

// One persistent launch over np (1 or 2) problems of kinds K0, K1.
template <int BN, class K0, class K1, int ST = 0>
cudaError_t launch_tc2_group(const SliceGemmProblem* pbs, int np, cudaStream_t s) {
  Tc2Maps m0, m1;
  bool ok = make_tc2_maps<BN, K0>(pbs[0], &m0);
  if (np > 1) ok = ok && make_tc2_maps<BN, K1>(pbs[1], &m1);
  else m1 = m0;
  if (!ok) return cudaErrorInvalidValue;
  auto kern = slice_gemm_tc2_kernel<BN, K0, K1, ST>;
  const int smem = Smem2<BN, K0::OUT, K1::OUT, ST>::kTotal;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (probe_env("STL_SMEM_MAX_CARVEOUT", 0))  // probe: let a transform CTA share the SM
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const int64_t t0 = tc2_tiles(pbs[0], BN);
  const int64_t tiles = t0 + (np > 1 ? tc2_tiles(pbs[1], BN) : 0);
  if (tiles <= 0) return cudaSuccess;
  if (tiles >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  PairLaunch L(smem, s);
  static const int max_clusters = L.max_clusters(kern);
  const int clusters = static_cast<int>(tiles < max_clusters ? tiles : max_clusters);
  L.cfg.gridDim = dim3(2 * clusters);
  GroupArgs ga{};
  for (int i = 0; i < 2; ++i) {
    const SliceGemmProblem& pb = pbs[i < np ? i : 0];
    ga.M[i] = static_cast<int>(pb.M);
    ga.N[i] = static_cast<int>(pb.N);
    ga.K[i] = static_cast<int>(pb.K);
  }
  ga.r = pbs[0].r;
  ga.total0 = static_cast<int>(t0);
  ga.total = static_cast<int>(tiles);
  ga.order = -1;
  if (np > 1 && pbs[0].K != pbs[1].K && probe_env("STL_GEMM_ORDER", 1)) {
    // per-cluster K-block load of each order; keep the best (ties: round robin)
    const int64_t kb0 = (pbs[0].K + kBK - 1) / kBK, kb1 = (pbs[1].K + kBK - 1) / kBK;
    const int64_t rounds = (tiles + clusters - 1) / clusters;
    int64_t best = -1;
    for (int order = -1; order <= 2; ++order) {
      std::vector<int64_t> load(clusters, 0);
      for (int c = 0; c < clusters; ++c)
        for (int64_t k = 0; k < rounds; ++k) {
          const bool rev = order < 0 ? false : order == 2 ? k == rounds - 1 : ((k + order) & 1) != 0;
          const int64_t t = k * clusters + (rev ? clusters - 1 - c : c);
          if (t < tiles) load[c] += t < t0 ? kb0 : kb1;
        }
      const int64_t mx = *std::max_element(load.begin(), load.end());
      if (best < 0 || mx < best) {
        best = mx;
        ga.order = order;
      }
    }
  }
  ga.nostore = probe_env("STL_GEMM_NOSTORE", 0);
  ga.trace = trace_next();
  if (probe_env("STL_GEMM_VERBOSE", 0))
    fprintf(stderr, "[tc2] max_clusters=%d clusters=%d tiles=%d BN=%d smem=%d\n", max_clusters,
            clusters, ga.total, BN, smem);
  return cudaLaunchKernelEx(&L.cfg, kern, m0.a, m0.b, m0.c, m0.c2, m1.a, m1.b, m1.c, m1.c2, ga);
}

template <int BN, bool A_MN, bool B_MN>
cudaError_t launch_tc2_any(const SliceGemmProblem& pb, cudaStream_t s) {
  if (pb.c_dtype == kBF16) {
    using Kd = GemmKind<A_MN, B_MN, kOutBf16>;
#ifdef STL_PROBES
    // probe: a 4-stage ring (161.5 KB) leaves room for a co-resident transform CTA
    if (BN == 256 && !A_MN && !B_MN && probe_env("STL_GEMM_STAGES", 0) == 4)
      return launch_tc2_group<BN, Kd, Kd, 4>(&pb, 1, s);
#endif
    return launch_tc2_group<BN, Kd, Kd>(&pb, 1, s);
  }
  if (pb.c_dtype == kF24) {
    using Kd = GemmKind<A_MN, B_MN, kOutF24>;
    return launch_tc2_group<BN, Kd, Kd>(&pb, 1, s);
  }
  if (pb.c2) {
    using Kd = GemmKind<A_MN, B_MN, kOutF32Bf16>;
    return launch_tc2_group<BN, Kd, Kd>(&pb, 1, s);
  }
  using Kd = GemmKind<A_MN, B_MN, kOutF32>;
  return launch_tc2_group<BN, Kd, Kd>(&pb, 1, s);
}

}  // namespace

bool make_bf16_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t slices, uint32_t box_inner, uint32_t box_outer,
                    uint64_t slice_bytes) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {inner, outer, slices};
  cuuint64_t strides[2] = {inner * 2, slice_bytes ? slice_bytes : inner * outer * 2};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult res = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS;
}

bool pdl_enabled() {
  static const bool on = [] {
    return probe_env("STL_PDL", 1) != 0;
  }();
  return on;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

bool slice_gemm_tc_supported(const SliceGemmProblem& pb) {
  if (pb.ab_dtype != kBF16) return false;
  if (pb.M <= 0 || pb.N <= 0 || pb.K <= 0 || pb.r <= 0) return false;
  if (pb.M > (1 << 30) || pb.N > (1 << 30) || pb.K > (1 << 30)) return false;
  // TMA: 16-byte aligned base and strides -> contiguous dim multiple of 8 bf16.
  const int64_t a_inner = pb.a_layout ? pb.M : pb.K;
  const int64_t b_inner = pb.b_layout ? pb.N : pb.K;
  if (a_inner % 8 || b_inner % 8) return false;
  if ((reinterpret_cast<uintptr_t>(pb.a) & 15) || (reinterpret_cast<uintptr_t>(pb.b) & 15))
    return false;
  return get_encode_fn() != nullptr;
}

bool slice_gemm_f24_supported(const SliceGemmProblem& pb) {
  return slice_gemm_tc_supported(pb) && pb.M > 128 && pb.N % 16 == 0 && !pb.c2 &&
         (reinterpret_cast<uintptr_t>(pb.c) & 15) == 0 && !probe_env("STL_GEMM_1CTA", 0);
}

namespace {
// CTA-pair kernel: M > 128 and C stored with TMA (16-byte aligned rows).
bool pair_eligible(const SliceGemmProblem& pb) {
  return pb.M > 128 && pb.N % 4 == 0 && (pb.c_dtype != kBF16 || (pb.N % 8 == 0 && !pb.c2)) &&
         (reinterpret_cast<uintptr_t>(pb.c) & 15) == 0 &&
         (!pb.c2 || (pb.N % 8 == 0 && (reinterpret_cast<uintptr_t>(pb.c2) & 15) == 0));
}
}  // namespace

bool slice_gemm_tc_group_supported(const SliceGemmProblem& p0, const SliceGemmProblem& p1) {
  const bool off = probe_env("STL_GEMM_NOGROUP", 0) || probe_env("STL_GEMM_1CTA", 0);
  if (off) return false;
  // the instantiated pair: g_w (A, B MN-major; fp32) with g_u (A K-major, B MN-major; F24/fp32)
  const bool kinds = p0.a_layout == 1 && p0.b_layout == 1 && p0.c_dtype == kF32 &&
                     p1.a_layout == 0 && p1.b_layout == 1 &&
                     (p1.c_dtype == kF32 || p1.c_dtype == kF24 || p1.c_dtype == kBF16);
  return kinds && slice_gemm_tc_supported(p0) && slice_gemm_tc_supported(p1) && p0.r == p1.r &&
         pair_eligible(p0) && pair_eligible(p1) && !p0.c2 && !p1.c2 && p0.N > 128 &&
         p1.N > 128 && (p1.c_dtype != kF24 || slice_gemm_f24_supported(p1));
}

cudaError_t slice_gemm_tc_group(const SliceGemmProblem& p0, const SliceGemmProblem& p1,
                                cudaStream_t s) {
  if (!slice_gemm_tc_group_supported(p0, p1)) return cudaErrorNotSupported;
  const SliceGemmProblem pbs[2] = {p0, p1};
  using K0 = GemmKind<true, true, kOutF32>;
  if (p1.c_dtype == kF24) return launch_tc2_group<256, K0, GemmKind<false, true, kOutF24>>(pbs, 2, s);
  if (p1.c_dtype == kBF16) return launch_tc2_group<256, K0, GemmKind<false, true, kOutBf16>>(pbs, 2, s);
  return launch_tc2_group<256, K0, GemmKind<false, true, kOutF32>>(pbs, 2, s);
}

cudaError_t slice_gemm_tc(const SliceGemmProblem& pb, cudaStream_t s) {
  const bool a_mn = pb.a_layout != 0, b_mn = pb.b_layout != 0;
  const int force1 = probe_env("STL_GEMM_1CTA", 0);
  // The pair kernel stores C with TMA (fp32 output, 16-byte aligned rows); other cases use the
  // 1-CTA kernel's direct-store epilogue.
  if (pb.c_dtype == kF24 && !slice_gemm_f24_supported(pb)) return cudaErrorNotSupported;
  if (!force1 && pair_eligible(pb)) {
    if (pb.N <= 128) {
      if (!a_mn && !b_mn) return launch_tc2_any<128, false, false>(pb, s);
      if (!a_mn && b_mn) return launch_tc2_any<128, false, true>(pb, s);
      if (a_mn && !b_mn) return launch_tc2_any<128, true, false>(pb, s);
      return launch_tc2_any<128, true, true>(pb, s);
    }
    if (!a_mn && !b_mn) return launch_tc2_any<256, false, false>(pb, s);
    if (!a_mn && b_mn) return launch_tc2_any<256, false, true>(pb, s);
    if (a_mn && !b_mn) return launch_tc2_any<256, true, false>(pb, s);
    return launch_tc2_any<256, true, true>(pb, s);
  }
  const bool narrow = pb.N <= 128;
  if (narrow) {
    if (!a_mn && !b_mn) return launch_tc<128, false, false>(pb, s);
    if (!a_mn && b_mn) return launch_tc<128, false, true>(pb, s);
    if (a_mn && !b_mn) return launch_tc<128, true, false>(pb, s);
    return launch_tc<128, true, true>(pb, s);
  }
  if (!a_mn && !b_mn) return launch_tc<256, false, false>(pb, s);
  if (!a_mn && b_mn) return launch_tc<256, false, true>(pb, s);
  if (a_mn && !b_mn) return launch_tc<256, true, false>(pb, s);
  return launch_tc<256, true, true>(pb, s);
}

// Split-K partial sums: out[p][i] = sum_s partial[p * S + s][i], fixed order (deterministic).
namespace {
__global__ void k_sum_splits(const float4* __restrict__ partial, int S, int64_t mn4, int64_t total4,
                             float4* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = i / mn4, o = i - p * mn4;
    const float4* src = partial + p * S * mn4 + o;
    float4 a = src[0];
    for (int k = 1; k < S; ++k) {
      const float4 b = src[k * mn4];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    out[i] = a;
  }
}
}  // namespace

cudaError_t slice_gemm_sum_splits(const float* partial, int r, int S, int64_t mn, float* out,
                                  cudaStream_t s) {
  if (mn % 4 || (reinterpret_cast<uintptr_t>(partial) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  const int64_t total4 = static_cast<int64_t>(r) * mn / 4;
  if (total4 == 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((total4 + 255) / 256, int64_t(sm_count()) * 8);
  k_sum_splits<<<static_cast<int>(blocks), 256, 0, s>>>(reinterpret_cast<const float4*>(partial),
                                                        S, mn / 4, total4,
                                                        reinterpret_cast<float4*>(out));
  return cudaGetLastError();
}

// ==================================================================== SIMT slice GEMM
// Generic fp32-accumulate batched GEMM for fp32 operands (the fp32 parity path: TF32 would
// miss the 1e-5 bar, SURVEY §7 hard part 3) and for shapes TMA cannot describe.
namespace {
template <typename T>
__device__ __forceinline__ float ldf(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ldf<float>(const float* p, int64_t i) {
  return __ldg(p + i);
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

constexpr int kSB = 64, kSK = 16;

template <typename T>
__global__ void __launch_bounds__(256)
    slice_gemm_simt_kernel(const T* __restrict__ A, int64_t sAm, int64_t sAk,
                           const T* __restrict__ B, int64_t sBk, int64_t sBn, void* C,
                           int c_bf16, int M, int N, int K) {
  __shared__ float As[kSK][kSB + 4];
  __shared__ float Bs[kSK][kSB + 4];
  const int p = blockIdx.z;
  const int64_t MK = static_cast<int64_t>(M) * K, KN = static_cast<int64_t>(K) * N;
  const T* Ap = A + p * MK;
  const T* Bp = B + p * KN;
  const int m0 = blockIdx.y * kSB, n0 = blockIdx.x * kSB;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kSK) {
    for (int i = threadIdx.x; i < kSK * kSB; i += 256) {
      // A tile: (m, k); B tile: (k, n). Index order chosen so the contiguous dim of the
      // common layouts maps to consecutive threads.
      const int kk = sAk == 1 ? (i % kSK) : (i / kSB);
      const int mm = sAk == 1 ? (i / kSK) : (i % kSB);
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? ldf(Ap, gm * sAm + gk * sAk) : 0.f;
      const int kb = sBk == 1 ? (i % kSK) : (i / kSB);
      const int nn = sBk == 1 ? (i / kSK) : (i % kSB);
      const int gn = n0 + nn, gk2 = k0 + kb;
      Bs[kb][nn] = (gn < N && gk2 < K) ? ldf(Bp, gk2 * sBk + gn * sBn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int64_t MN = static_cast<int64_t>(M) * N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      const int64_t off = p * MN + static_cast<int64_t>(gm) * N + gn;
      if (c_bf16)
        reinterpret_cast<__nv_bfloat16*>(C)[off] = __float2bfloat16_rn(acc[i][j]);
      else
        reinterpret_cast<float*>(C)[off] = acc[i][j];
    }
  }
}
}  // namespace

cudaError_t slice_gemm_simt(const SliceGemmProblem& pb, cudaStream_t s) {
  const int64_t M = pb.M, N = pb.N, K = pb.K;
  const int64_t sAm = pb.a_layout ? 1 : K, sAk = pb.a_layout ? M : 1;
  const int64_t sBk = pb.b_layout ? N : 1, sBn = pb.b_layout ? 1 : K;
  dim3 grid(static_cast<unsigned>((N + kSB - 1) / kSB), static_cast<unsigned>((M + kSB - 1) / kSB),
            static_cast<unsigned>(pb.r));
  const int cb = pb.c_dtype == kBF16 ? 1 : 0;
  if (pb.ab_dtype == kBF16)
    slice_gemm_simt_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(pb.a), sAm, sAk,
        static_cast<const __nv_bfloat16*>(pb.b), sBk, sBn, pb.c, cb, int(M), int(N), int(K));
  else
    slice_gemm_simt_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(pb.a), sAm, sAk,
                                                       static_cast<const float*>(pb.b), sBk, sBn,
                                                       pb.c, cb, int(M), int(N), int(K));
  return cudaGetLastError();
}

}  // namespace stl

#ifdef STL_PROBES
namespace stl {
namespace {
unsigned long long* g_trace = nullptr;
unsigned long long* g_trace_cta = nullptr;
int g_trace_n = 0;
constexpr int kTraceSlots = 4096;
}  // namespace
Trace trace_next() {
  static const int on = probe_env("STL_TRACE", 0);
  if (!on) return Trace{nullptr, 0, nullptr};
  if (!g_trace) {
    cudaMalloc(&g_trace, 2 * kTraceSlots * sizeof(unsigned long long));
    g_trace_n = kTraceSlots;  // forces a reset before first use
  }
  if (g_trace_n >= kTraceSlots) return Trace{nullptr, 0, nullptr};
  if (!g_trace_cta) cudaMalloc(&g_trace_cta, kTraceCtaSlots * 2048 * 4 * sizeof(unsigned long long));
  return Trace{g_trace, g_trace_n++, g_trace_cta};
}
}  // namespace stl

// probe-only exports (not in include/stl_b200.h): reset the trace slots, read them back
extern "C" __attribute__((visibility("default"))) int stl_trace_reset(void) {
  using namespace stl;
  if (!g_trace) cudaMalloc(&g_trace, 2 * kTraceSlots * sizeof(unsigned long long));
  static unsigned long long h[2 * kTraceSlots];
  for (int i = 0; i < kTraceSlots; ++i) { h[2 * i] = ~0ull; h[2 * i + 1] = 0; }
  g_trace_n = 0;
  return static_cast<int>(cudaMemcpy(g_trace, h, sizeof(h), cudaMemcpyHostToDevice));
}
extern "C" __attribute__((visibility("default"))) int stl_trace_read_cta(unsigned long long* out,
                                                                         int slot, int grid) {
  using namespace stl;
  if (!g_trace_cta || slot >= kTraceCtaSlots) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(out, g_trace_cta + static_cast<size_t>(slot) * grid * 4, grid * 4 * sizeof(unsigned long long),
             cudaMemcpyDeviceToHost);
  return grid;
}
extern "C" __attribute__((visibility("default"))) int stl_trace_read(unsigned long long* out, int n) {
  using namespace stl;
  if (!g_trace) return 0;
  const int k = n < g_trace_n ? n : g_trace_n;
  cudaDeviceSynchronize();
  cudaMemcpy(out, g_trace, 2 * k * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return k;
}
#endif
