// sm100_pair_pipeline.cuh — the CTA-pair (cta_group::2) TMA -> tcgen05 mainloop shared by the
// plain slice GEMM and the decode-fused slice GEMM.
//
// Roles (per CTA of the pair): warp 0 lane 0 = TMA producer (both CTAs), warp 1 lane 0 of the
// even CTA = MMA issuer, warp 2 = TMEM owner. A tile is 256 (M) x BN (N); each CTA stages its
// 128 A rows and BN/2 B columns per 64-wide K block. Tiles are visited in a caller-defined
// order (TileMap) so the fused kernel can schedule all r slices of an output block together.
#pragma once
#include "sm100_ptx.cuh"

namespace stl {
namespace pair {

constexpr int kBK = 64;  // 64 bf16 = one 128-byte swizzle row

template <int BN, int STAGES>
struct Layout {
  static constexpr uint32_t kABytes = 128 * kBK * 2;
  static constexpr uint32_t kBBytes = (BN / 2) * kBK * 2;
  static constexpr uint32_t kRingBytes = STAGES * (kABytes + kBBytes);
  // barriers: full[STAGES], empty[STAGES], tfull[2], tempty[2], tmem slot
  static constexpr uint32_t kBarBytes = (2 * STAGES + 4) * 8 + 16;
};

struct TileCoord {
  int p, mb, nb;
};

// Producer: both CTAs. `map(tile)` -> TileCoord.
template <int BN, int STAGES, bool A_MN, bool B_MN, class TileMap>
__device__ __forceinline__ void produce(const CUtensorMap* tmA, const CUtensorMap* tmB,
                                       uint8_t* sA, uint8_t* sB, uint64_t* full, uint64_t* empty,
                                       uint32_t rank, int first, int stride, int total,
                                       int num_kb, TileMap map) {
  using L = Layout<BN, STAGES>;
  const bool leader = rank == 0;
  int stage = 0;
  uint32_t phase = 0;
  for (int tile = first; tile < total; tile += stride) {
    const TileCoord tc = map(tile);
    const int m0 = tc.mb * 256 + static_cast<int>(rank) * 128;
    const int n0 = tc.nb * BN + static_cast<int>(rank) * (BN / 2);
    for (int kb = 0; kb < num_kb; ++kb) {
      ptx::mbar_wait(&empty[stage], phase ^ 1);
      if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (L::kABytes + L::kBBytes));
      uint8_t* a = sA + stage * L::kABytes;
      uint8_t* b = sB + stage * L::kBBytes;
      if constexpr (!A_MN) {
        ptx::tma_load_3d_2sm(tmA, &full[stage], a, kb * kBK, m0, tc.p);
      } else {
#pragma unroll
        for (int j = 0; j < 2; ++j)
          ptx::tma_load_3d_2sm(tmA, &full[stage], a + j * (64 * kBK * 2), m0 + j * 64, kb * kBK,
                               tc.p);
      }
      if constexpr (!B_MN) {
        ptx::tma_load_3d_2sm(tmB, &full[stage], b, kb * kBK, n0, tc.p);
      } else {
#pragma unroll
        for (int j = 0; j < BN / 128; ++j)
          ptx::tma_load_3d_2sm(tmB, &full[stage], b + j * (64 * kBK * 2), n0 + j * 64, kb * kBK,
                               tc.p);
      }
      if (!leader) ptx::mbar_arrive_cluster(ptx::mapa_shared(ptx::smem_u32(&full[stage]), 0));
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
}

// MMA issuer: even CTA only. Accumulator buffer `it & 1` at TMEM column (it & 1) * BN.
template <int BN, int STAGES, bool A_MN, bool B_MN>
__device__ __forceinline__ void mma_loop(uint8_t* sA, uint8_t* sB, uint64_t* full,
                                         uint64_t* empty, uint64_t* tfull, uint64_t* tempty,
                                         uint32_t tmem_base, int first, int stride, int total,
                                         int num_kb) {
  using L = Layout<BN, STAGES>;
  constexpr uint32_t kIdesc = ptx::idesc_bf16_f32(256, BN, A_MN, B_MN);
  int stage = 0;
  uint32_t phase = 0;
  int it = 0;
  for (int tile = first; tile < total; tile += stride, ++it) {
    const int acc = it & 1;
    const uint32_t acc_phase = (it >> 1) & 1;
    ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
    ptx::tc_fence_after();
    const uint32_t d_tmem = tmem_base + acc * BN;
    for (int kb = 0; kb < num_kb; ++kb) {
      ptx::mbar_wait(&full[stage], phase);
      ptx::tc_fence_after();
      const uint32_t a_addr = ptx::smem_u32(sA + stage * L::kABytes);
      const uint32_t b_addr = ptx::smem_u32(sB + stage * L::kBBytes);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) {
        const uint64_t ad = A_MN ? ptx::smem_desc_sw128(a_addr + k * 2048, 64 * kBK * 2, 1024)
                                 : ptx::smem_desc_sw128(a_addr + k * 32, 16, 1024);
        const uint64_t bd = B_MN ? ptx::smem_desc_sw128(b_addr + k * 2048, 64 * kBK * 2, 1024)
                                 : ptx::smem_desc_sw128(b_addr + k * 32, 16, 1024);
        ptx::mma_bf16_ss_2sm(d_tmem, ad, bd, kIdesc, (kb | k) != 0 ? 1u : 0u);
      }
      ptx::mma_commit_2sm(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    ptx::mma_commit_2sm(&tfull[acc]);
  }
}

}  // namespace pair
}  // namespace stl
