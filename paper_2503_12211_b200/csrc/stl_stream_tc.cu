// stl_stream_tc.cu — the t = 4 decode on the 5th-generation tensor cores (tcgen05 + TMEM).
//
//   tile(I, J)[c] = sum_p Z[p][I][J] D[p][c]          decode_tiles (snf_operator.py:88-96)
//
// The same HBM stream as k_stream<kDec> (stl_stream.cu): a unit is a 512-tile segment of one
// tile row, its P bf16 planes land in shared memory as one 4-D TMA box (64 tiles x Pb planes x 8
// chunks, 128-byte swizzle) and its 4 output matrix rows leave as 1-D bulk stores. What changes
// is who does the change of basis: instead of 16 consumer warps running mma.sync fragments, one
// thread issues UMMAs straight on the landed box —
//   D[tile m][n] = sum_p A[m][p] B[p][n],  A = the plane box read as an MN-major (tile-major)
//   SW128 operand (64-tile atoms Pb * 128 bytes apart, 8-plane groups 1024 bytes apart),
//   B = [D_hi | D_lo] (K-major, 32 columns: the decoder rows split into bf16 hi + lo),
// M = 128 tiles per MMA, N = 32, K = 16 planes per step, fp32 accumulation in TMEM — and eight
// epilogue warps read the accumulators back (tcgen05.ld), add the hi and lo columns, round to
// bf16 and stage the output rows for the bulk stores. The tensor pipe does the arithmetic the
// SM's issue slots did before, which matters inside the forward pipeline: after the slice GEMM
// the SMs clock lower and the mma.sync decode's consumers set its pace.
// Warp roles: 0 = TMA producer, 1 = MMA issuer (and TMEM owner), 2..9 = epilogue.
#include <cstdio>
#include "sm100_ptx.cuh"
#include "stl_internal.h"

namespace stl {
namespace {

constexpr int kT = 512;                 // tiles per unit
constexpr int kMB = kT / 128;           // UMMA M-blocks per unit
constexpr int kEpi = 8;                 // epilogue warps
constexpr int kThreads = 32 * (2 + kEpi);
constexpr uint32_t kOS = kT * 8;        // output staging row: 512 tiles x 4 bf16
constexpr uint32_t kOutBytes = 4 * kOS; // one unit's 4 matrix rows
constexpr uint32_t kBBytes = 32 * 128;  // B operand: 32 rows (hi, lo) x 128-byte swizzled K rows
constexpr uint32_t kTmemCols = 2 * kMB * 32;  // two accumulator sets of 4 x (128 x 32)
constexpr int kMaxSt = 8;
// encode: two accumulator sets of 2 M-blocks x N = 32 G columns, rounded up to a power of 2
template <int G> constexpr uint32_t kTmemColsEnc() { return 4 * 32 * G <= 256 ? 256u : 512u; }

struct TcArgs {
  __nv_bfloat16* out;
  int64_t ldo;
  const float* coef;  // D: P x 16
  int P, Pb;
  int64_t bc, upr, nunits;
  uint32_t nstages, nbuf;
};

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(dst)),
               "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* m, uint64_t* bar, uint32_t dst,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(ptx::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_wait_read_n(uint32_t n) {
  // the number of store groups that may still be reading shared memory (nbuf - 2: 0 or 1)
  if (n == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld_x32(uint32_t taddr, float (&v)[32]) {
  uint32_t (&u)[32] = reinterpret_cast<uint32_t(&)[32]>(v);
  ptx::tmem_ld_32x32b_x32(taddr, u);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void epi_bar(int grp, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(nthreads) : "memory");
}

// KS = K-steps of 16 planes. The box holds Pb = 8 ceil(P / 8) planes (>= 16; planes P..Pb-1 are
// TMA zero fill); step s reads planes off_s .. off_s + 15 of each 64-tile chunk, off_0 = 0 and
// the last step off = Pb - 16, so a step never reads past its chunk's planes (it may overlap
// the previous step's planes, whose B rows it then carries as zeros).
// EG = epilogue groups: 1 (all 8 warps per unit, each a half of the M-blocks) or 2 (4 warps per
// unit, alternate units: two units' read-back, staging and stores in flight).
template <int KS, int EG>
__global__ void __launch_bounds__(kThreads, 1)
    k_decode_tc(const __grid_constant__ CUtensorMap tm_in, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  const int Pb = a.Pb;
  const uint32_t kStage = static_cast<uint32_t>(Pb) * kT * 2;
  const uint32_t nst = a.nstages, nbuf = a.nbuf;
  const uint32_t s_out = nst * kStage;
  const uint32_t s_b = s_out + EG * nbuf * kOutBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + s_b + kBBytes);
  uint64_t* empty = full + kMaxSt;
  uint64_t* tfull = empty + kMaxSt;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nunits = static_cast<uint32_t>(a.nunits), upr = static_cast<uint32_t>(a.upr);
  constexpr int kGW = kEpi / EG;  // warps per epilogue group

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < nst; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kGW);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tm_in);
  if (warp == 1) ptx::tmem_alloc(tslot, kTmemCols);
  // B = [D_hi | D_lo]: row n < 16 holds the hi halves of decoder column n, row 16 + n the lo
  // halves; K runs along the 128-byte row (16 elements per step), 16-byte chunks XOR-swizzled
  // by (n & 7).
  for (int i = threadIdx.x; i < 32 * 64; i += kThreads) {
    const int n = i >> 6, k = i & 63, c = n & 15, st = k >> 4;
    const int pl = (st == 0 ? 0 : Pb - 16) + (k & 15);
    const float d = st < KS && pl < a.P && pl >= 16 * st ? a.coef[pl * 16 + c] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(d);
    const __nv_bfloat16 v = n < 16 ? hi : __float2bfloat16_rn(d - __bfloat162float(hi));
    const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
    *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
  }
  ptx::fence_proxy_async_smem();  // the generic-proxy B writes, before the UMMAs read them
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch_dependents();
  griddep_wait();  // the planes of this launch are complete (PDL)

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        const uint32_t st = it % nst, ph = (it / nst) & 1;
        const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
        ptx::mbar_wait(&empty[st], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[st], kStage);
        tma_load_4d(&tm_in, &full[st], sbase + st * kStage, 0, 0, static_cast<int>(J0 / 64),
                    static_cast<int>(I));
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 32, true, false);
      uint32_t it = 0;
      for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        const uint32_t st = it % nst, ph = (it / nst) & 1;
        const uint32_t buf = it & 1, bph = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[buf], bph ^ 1);
        ptx::mbar_wait(&full[st], ph);
        ptx::tc_fence_after();
        const uint32_t a0 = sbase + st * kStage;
#pragma unroll
        for (int mb = 0; mb < kMB; ++mb)
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            // tiles 128 mb .. +127 = chunks 2 mb, 2 mb + 1 (Pb * 128 bytes apart)
            const uint32_t off = ks == 0 ? 0u : static_cast<uint32_t>(Pb - 16);
            const uint64_t ad =
                ptx::smem_desc_sw128(a0 + (2 * mb * Pb + off) * 128, Pb * 128, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(sbase + s_b + ks * 32, 16, 1024);
            ptx::mma_bf16_ss(tmem + buf * (kMB * 32) + mb * 32, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
        ptx::mma_commit(&empty[st]);   // the stage's box is consumed
        ptx::mma_commit(&tfull[buf]);  // the unit's accumulators are ready
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int grp = ew / kGW, gw = ew % kGW;
    const uint32_t quarter = warp & 3;  // TMEM lanes 32 quarter .. +31 (warp id mod 4)
    constexpr int kMBW = kMB * 4 / kGW;  // M-blocks per warp
    const int mb0 = (gw >> 2) * kMBW;
    const bool issuer = gw == 0 && lane == 0;
    uint32_t it = grp, k = 0;
    for (uint32_t u = blockIdx.x + grp * gridDim.x; u < nunits; u += EG * gridDim.x, it += EG, ++k) {
      const uint32_t buf = it & 1, bph = (it >> 1) & 1;
      const uint32_t ob0 = s_out + (grp * nbuf + k % nbuf) * kOutBytes;
      const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
      ptx::mbar_wait(&tfull[buf], bph);
      ptx::tc_fence_after();
#pragma unroll
      // two M-blocks' accumulators per tcgen05.wait::ld (the loads' latencies overlap)
      static_assert(kMBW % 2 == 0, "M-blocks per warp");
#pragma unroll
      for (int j = 0; j < kMBW; j += 2) {
        float v[2][32];
#pragma unroll
        for (int h = 0; h < 2; ++h)
          tmem_ld_x32(tmem + ((quarter * 32) << 16) + buf * (kMB * 32) + (mb0 + j + h) * 32, v[h]);
        ptx::tmem_ld_wait();
        if (j == kMBW - 2) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t m = (mb0 + j + h) * 128 + quarter * 32 + lane;
#pragma unroll
          for (int r = 0; r < 4; ++r) {  // matrix row 4I + r: tile values c = 4r .. 4r + 3
            const uint32_t w0 = pack_bf16(v[h][4 * r] + v[h][16 + 4 * r], v[h][4 * r + 1] + v[h][17 + 4 * r]);
            const uint32_t w1 = pack_bf16(v[h][4 * r + 2] + v[h][18 + 4 * r], v[h][4 * r + 3] + v[h][19 + 4 * r]);
            *reinterpret_cast<uint2*>(smem + ob0 + r * kOS + m * 8) = make_uint2(w0, w1);
          }
        }
      }
      ptx::fence_proxy_async_smem();
      // the group's next staging buffer was last stored from nbuf of its units ago
      if (issuer) bulk_wait_read_n(nbuf - 2);
      epi_bar(grp, 32 * kGW);
      if (issuer) {
        const uint32_t Tw = min(static_cast<uint32_t>(a.bc) - J0, static_cast<uint32_t>(kT));
#pragma unroll
        for (int r = 0; r < 4; ++r)
          bulk_s2g(a.out + (4 * static_cast<int64_t>(I) + r) * a.ldo + 4 * static_cast<int64_t>(J0),
                   sbase + ob0 + r * kOS, Tw * 8);
        ptx::bulk_commit();
      }
    }
    if (issuer) ptx::bulk_wait_all();
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

template <int KS, int EG>
cudaError_t launch_tc(const CUtensorMap& tm, TcArgs a, cudaStream_t s) {
  const uint32_t kStage = static_cast<uint32_t>(a.Pb) * kT * 2;
  const uint32_t budget = 227 * 1024 - 1024 - kBBytes - 2 * (kMaxSt + 4) * 8 - 16;
  static const int nb_env = probe_env("STL_DEC_TC_NBUF", 0);
  static const int st_env = probe_env("STL_DEC_TC_STAGES", 0);
  a.nbuf = nb_env >= 2 && nb_env <= 6 ? nb_env : (EG == 2 ? 3 : 4);
  if (EG * a.nbuf * kOutBytes + 2 * kStage > budget) return cudaErrorNotSupported;
  uint32_t ns = (budget - EG * a.nbuf * kOutBytes) / kStage;
  a.nstages = ns > kMaxSt ? kMaxSt : ns;
  if (st_env >= 2 && static_cast<uint32_t>(st_env) < a.nstages) a.nstages = st_env;
  const uint32_t smem = a.nstages * kStage + EG * a.nbuf * kOutBytes + kBBytes +
                        2 * (kMaxSt + 4) * 8 + 16 + 1024;
  auto k = k_decode_tc<KS, EG>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  return launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(kThreads), smem, s, tm, a);
}

// ------------------------------------------------------------------ encode
//   planes[p][I][J] = sum_c E[p][c] tile(I, J)[c]     encode_tiles (snf_operator.py:80-85)
// A unit's 4 matrix rows land as 4 plain 4 KB rows (1-D bulk copies). Row a read as pairs of
// tiles is a K-major no-swizzle UMMA operand: MMA row i = tiles 2i, 2i + 1 (16 bytes: b = 0..3
// of each), 8-row core matrices 128 contiguous bytes (SBO = 128), and the two core matrices of a
// K-step are matrix rows a0, a0 + 1 (LBO = the row stride). So one K-step covers k = (a, parity,
// b) for two matrix rows and two steps the whole tile; B pairs each parity with its own output
// columns: n = 32 g + 16 par + 8 hl + pp (plane p = 8 g + pp, hl: encoder hi / lo half),
// B[n][(a, par', b)] = E_hl[p][4a + b] if par' == par else 0. M = 128 pairs (256 tiles), N = 32 G,
// K = 16; the epilogue adds hi + lo, packs the two tiles of a pair into one bf16x2 word and
// writes plane rows of the swizzled output box, which leaves by one TMA store.
constexpr uint32_t kERow = kT * 8;  // one matrix row of a unit: 512 tiles x 4 bf16

__device__ __forceinline__ uint64_t smem_desc_plain(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // version 1, layout 0 = SWIZZLE_NONE
  return d;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, uint32_t src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

struct TcEncArgs {
  const __nv_bfloat16* mat;
  int64_t ldm;
  const float* coef;  // E: P x 16
  int P;
  int64_t bc, upr, nunits;
  uint32_t nstages, nbuf, out_bytes;
};

// G = 8-plane groups (N = 32 G); EG epilogue groups as in the decode.
template <int G, int EG>
__global__ void __launch_bounds__(kThreads, 1)
    k_encode_tc(const __grid_constant__ CUtensorMap tm_out, TcEncArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  constexpr int N = 32 * G;
  constexpr uint32_t kStage = 4 * kERow;
  constexpr uint32_t kB = N * 128;
  constexpr int kGW = kEpi / EG;
  constexpr int kEMB = 2;  // M-blocks (128 tile pairs) per unit
  const uint32_t nst = a.nstages, nbuf = a.nbuf, ob_bytes = a.out_bytes;
  const uint32_t s_out = nst * kStage;
  const uint32_t s_b = s_out + EG * nbuf * ob_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + s_b + kB);
  uint64_t* empty = full + kMaxSt;
  uint64_t* tfull = empty + kMaxSt;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = a.P;
  const uint32_t nunits = static_cast<uint32_t>(a.nunits), upr = static_cast<uint32_t>(a.upr);
  const uint32_t bc = static_cast<uint32_t>(a.bc);

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < nst; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kGW);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tm_out);
  if (warp == 1) ptx::tmem_alloc(tslot, kTmemColsEnc<G>());
  for (int i = threadIdx.x; i < N * 32; i += kThreads) {
    const int n = i >> 5, k = i & 31;
    const int g = n >> 5, par = (n >> 4) & 1, hl = (n >> 3) & 1, p = 8 * g + (n & 7);
    const int ka = k >> 3, kpar = (k >> 2) & 1, kb = k & 3;
    const float e = kpar == par && p < P ? a.coef[p * 16 + 4 * ka + kb] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(e);
    const __nv_bfloat16 v = hl == 0 ? hi : __float2bfloat16_rn(e - __bfloat162float(hi));
    const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
    *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
  }
  for (int i = threadIdx.x; i < N * 32; i += kThreads) {  // K 32..63 of each B row: zero
    const int n = i >> 5, k = 32 + (i & 31);
    const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
    *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = __float2bfloat16_rn(0.f);
  }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch_dependents();
  griddep_wait();

  if (warp == 0) {
    // ---------------------------------------------------------------- producer: 4 matrix rows
    uint32_t it = 0;
    for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
      const uint32_t st = it % nst, ph = (it / nst) & 1;
      const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
      const uint32_t Tw = min(bc - J0, static_cast<uint32_t>(kT));
      ptx::mbar_wait(&empty[st], ph ^ 1);
      if (lane == 0) ptx::mbar_arrive_expect_tx(&full[st], 4 * Tw * 8);
      __syncwarp();
      if (lane < 4)
        bulk_g2s(sbase + st * kStage + lane * kERow,
                 a.mat + (4 * static_cast<int64_t>(I) + lane) * a.ldm + 4 * static_cast<int64_t>(J0),
                 Tw * 8, &full[st]);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N, false, false);
      uint32_t it = 0;
      for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
        const uint32_t st = it % nst, ph = (it / nst) & 1;
        const uint32_t buf = it & 1, bph = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[buf], bph ^ 1);
        ptx::mbar_wait(&full[st], ph);
        ptx::tc_fence_after();
        const uint32_t a0 = sbase + st * kStage;
#pragma unroll
        for (int mb = 0; mb < kEMB; ++mb)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            // pairs 128 mb .. +127 of matrix rows 2 ks, 2 ks + 1
            const uint64_t ad = smem_desc_plain(a0 + 2 * ks * kERow + mb * 2048, kERow, 128);
            const uint64_t bd = ptx::smem_desc_sw128(sbase + s_b + ks * 32, 16, 1024);
            ptx::mma_bf16_ss(tmem + buf * (kEMB * N) + mb * N, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
        ptx::mma_commit(&empty[st]);
        ptx::mma_commit(&tfull[buf]);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int grp = ew / kGW, gw = ew % kGW;
    const uint32_t quarter = warp & 3;
    constexpr int kMBW = kEMB * 4 / kGW;  // M-blocks per warp
    const int mb0 = (gw >> 2) * kMBW;
    const bool issuer = gw == 0 && lane == 0;
    uint32_t it = grp, k = 0;
    for (uint32_t u = blockIdx.x + grp * gridDim.x; u < nunits; u += EG * gridDim.x, it += EG, ++k) {
      const uint32_t buf = it & 1, bph = (it >> 1) & 1;
      const uint32_t ob0 = s_out + (grp * nbuf + k % nbuf) * ob_bytes;
      const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
      ptx::mbar_wait(&tfull[buf], bph);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int j = 0; j < kMBW; ++j) {
        const int mb = mb0 + j;
        // tiles 256 mb + 2 (32 quarter + lane) + {0, 1}: chunk 4 mb + quarter, bytes 4 lane
        const uint32_t chunk = 4 * mb + quarter;
        // two column groups (16 planes) per tcgen05.wait::ld (the loads' latencies overlap)
#pragma unroll
        for (int g0 = 0; g0 < G; g0 += 2) {
          constexpr int kB2 = 2;
          float v[kB2][32];
#pragma unroll
          for (int h = 0; h < kB2; ++h)
            if (g0 + h < G)
              tmem_ld_x32(tmem + ((quarter * 32) << 16) + buf * (kEMB * N) + mb * N + 32 * (g0 + h), v[h]);
          ptx::tmem_ld_wait();
          if (j == kMBW - 1 && g0 + 2 >= G) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
          }
#pragma unroll
          for (int h = 0; h < kB2; ++h)
#pragma unroll
            for (int pp = 0; pp < 8; ++pp) {
              const int p = 8 * (g0 + h) + pp;
              if (g0 + h < G && p < P) {
                const uint32_t row = chunk * P + p;
                const uint32_t byte = 4 * lane;
                const uint32_t off = row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
                *reinterpret_cast<uint32_t*>(smem + ob0 + off) =
                    pack_bf16(v[h][pp] + v[h][8 + pp], v[h][16 + pp] + v[h][24 + pp]);
              }
            }
        }
      }
      ptx::fence_proxy_async_smem();
      if (issuer) bulk_wait_read_n(nbuf - 2);
      epi_bar(grp, 32 * kGW);
      if (issuer) {
        tma_store_4d(&tm_out, sbase + ob0, 0, 0, static_cast<int>(J0 / 64), static_cast<int>(I));
        ptx::bulk_commit();
      }
    }
    if (issuer) ptx::bulk_wait_all();
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemColsEnc<G>());
  }
}

template <int G, int EG>
cudaError_t launch_enc_tc(const CUtensorMap& tm, TcEncArgs a, cudaStream_t s) {
  constexpr uint32_t kStage = 4 * kERow;
  constexpr uint32_t kB = 32 * G * 128;
  a.out_bytes = (static_cast<uint32_t>(a.P) * kT * 2 + 1023) / 1024 * 1024;
  const uint32_t budget = 227 * 1024 - 1024 - kB - 2 * (kMaxSt + 4) * 8 - 16;
  static const int nb_env = probe_env("STL_ENC_TC_NBUF", 0);
  static const int st_env = probe_env("STL_ENC_TC_STAGES", 0);
  a.nbuf = nb_env >= 2 && nb_env <= 6 ? nb_env : 2;
  if (EG * a.nbuf * a.out_bytes + 2 * kStage > budget) return cudaErrorNotSupported;
  const uint32_t ns = (budget - EG * a.nbuf * a.out_bytes) / kStage;
  a.nstages = ns > kMaxSt ? kMaxSt : ns;
  if (st_env >= 2 && static_cast<uint32_t>(st_env) < a.nstages) a.nstages = st_env;
  const uint32_t smem = a.nstages * kStage + EG * a.nbuf * a.out_bytes + kB +
                        2 * (kMaxSt + 4) * 8 + 16 + 1024;
  auto k = k_encode_tc<G, EG>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  return launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(kThreads), smem, s, tm, a);
}

}  // namespace

cudaError_t planes_to_tiles_tc(const void* in, int P, int64_t br, int64_t bc, const float* coef,
                               void* out, int64_t ldo, cudaStream_t s, int64_t plane_rows) {
  static const int on = probe_env("STL_DEC_TC", 1);
  if (!on || P < 1 || P > 32 || bc < kT || bc % 64 || ldo % 8 ||
      (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  const int Pb = P <= 16 ? 16 : (P + 7) / 8 * 8;
  CUtensorMap tm{};
  if (plane_rows < br) plane_rows = br;
  if (!plane_box_tmap(&tm, in, 2, P, Pb, br, bc, kT, plane_rows)) return cudaErrorNotSupported;
  TcArgs a{};
  a.out = static_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.coef = coef;
  a.P = P;
  a.Pb = Pb;
  a.bc = bc;
  a.upr = (bc + kT - 1) / kT;
  a.nunits = br * a.upr;
  static const int eg = probe_env("STL_DEC_TC_EG", 2);
  if (Pb <= 16) return eg == 1 ? launch_tc<1, 1>(tm, a, s) : launch_tc<1, 2>(tm, a, s);
  return eg == 1 ? launch_tc<2, 1>(tm, a, s) : launch_tc<2, 2>(tm, a, s);
}

// bf16 matrix (4 br x 4 bc, leading dim ldm) -> P <= 32 bf16 planes (P x plane_rows x bc).
cudaError_t tiles_to_planes_tc(const void* m, int64_t ldm, int64_t br, int64_t bc,
                               const float* coef, int P, void* out, cudaStream_t s,
                               int64_t plane_rows) {
  static const int on = probe_env("STL_ENC_TC", 1);
  if (!on || P < 1 || P > 32 || bc < kT || bc % 64 || ldm % 8 ||
      (reinterpret_cast<uintptr_t>(m) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  CUtensorMap tm{};
  if (plane_rows < br) plane_rows = br;
  if (!plane_box_tmap(&tm, out, 2, P, P, br, bc, kT, plane_rows)) return cudaErrorNotSupported;
  TcEncArgs a{};
  a.mat = static_cast<const __nv_bfloat16*>(m);
  a.ldm = ldm;
  a.coef = coef;
  a.P = P;
  a.bc = bc;
  a.upr = (bc + kT - 1) / kT;
  a.nunits = br * a.upr;
  static const int eg = probe_env("STL_ENC_TC_EG", 2);
  switch ((P + 7) / 8) {
    case 1: return eg == 1 ? launch_enc_tc<1, 1>(tm, a, s) : launch_enc_tc<1, 2>(tm, a, s);
    case 2: return eg == 1 ? launch_enc_tc<2, 1>(tm, a, s) : launch_enc_tc<2, 2>(tm, a, s);
    case 3: return eg == 1 ? launch_enc_tc<3, 1>(tm, a, s) : launch_enc_tc<3, 2>(tm, a, s);
    default: return eg == 1 ? launch_enc_tc<4, 1>(tm, a, s) : launch_enc_tc<4, 2>(tm, a, s);
  }
}

}  // namespace stl
