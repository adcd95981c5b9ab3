// stl_stream_tc.cu — the t = 4 tile transforms on the 5th-generation tensor cores (tcgen05 +
// TMEM): the default bf16 path for r <= 32 and tile columns >= 512 (K10-K13).
//
//   k_decode_tc  tile(I, J)[c] = sum_p Z[p][I][J] D[p][c]        decode_tiles (snf_operator.py:88-96)
//   k_encode_tc  planes[p][I][J] = sum_c E[p][c] tile(I, J)[c]   encode_tiles (snf_operator.py:80-85)
//   k_red_tc     the decode plus g_ex = sum Z (x) X on mma.sync warps (toy_network.py:104-105)
//   k_remix_tc   out[p] = sum_q (e_x d^T)[p][q] Z[q]             stl_fused_step (snf_operator.py:175-188)
//
// The same HBM streams as stl_stream.cu's k_stream: a unit is a 512-tile segment of one tile
// row, its bf16 planes land in shared memory as one 4-D TMA box (64 tiles x Pb planes x 8
// chunks, 128-byte swizzle), its 4 matrix rows as 1-D bulk copies, outputs leave by TMA / bulk
// stores. What changes is who does the change of basis: instead of 16 consumer warps running
// mma.sync fragments, one thread issues UMMAs straight on the landed data. Decode:
//   D[tile m][n] = sum_p A[m][p] B[p][n],  A = the plane box read as an MN-major (tile-major)
//   SW128 operand (64-tile atoms Pb * 128 bytes apart, 8-plane groups 1024 bytes apart),
//   B = [D_hi | D_lo] (K-major, 32 columns: the decoder rows split into bf16 hi + lo),
// M = 128 tiles per MMA, N = 32, K = 16 planes per step, fp32 accumulation in TMEM — and the
// epilogue warps read the accumulators back (tcgen05.ld), add the hi and lo columns, round to
// bf16 and stage the output rows for the bulk stores (the encode's operand scheme is described
// at k_encode_tc). The tensor pipe does the arithmetic the SM's issue slots did before, which
// matters inside the forward pipeline: after the slice GEMM the SMs clock lower and the
// mma.sync decode's consumers set its pace.
// Warp roles: 0 = TMA producer, 1 = MMA issuer (and TMEM owner), 2..9 = two epilogue groups on
// alternate units (k_red_tc: + 10..17 reduction warps; k_remix_tc: 2..17, 8 per group).
#include <cstdio>
#include <mutex>
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

// Unit schedule: each CTA takes its first S units round robin (u = blockIdx.x + it * grid, the
// SMs stream adjacent DRAM pages in lock step), the rest from an atomic counter, so SMs that the
// memory system serves faster take more of the tail (dyn0 = S * grid; dyn0 >= nunits: static).
// The producer publishes each unit index in a 16-entry ring (one mbarrier per entry) that the
// MMA issuer and the epilogue read; kNoUnit ends the loop (written twice, once per epilogue
// group's parity). Readers trail the producer by at most nstages + 3 < 16 units.
constexpr uint32_t kNoUnit = 0xFFFFFFFFu;
constexpr int kRing = 16;
constexpr uint32_t kBarBytes = (2 * kMaxSt + 4 + kRing) * 8 + 16 + kRing * 4;

__device__ __forceinline__ uint32_t next_unit(uint32_t it, uint32_t nunits, uint32_t dyn0,
                                              unsigned* cnt) {
  uint32_t u = blockIdx.x + it * gridDim.x;
  if (u >= dyn0) u = dyn0 < nunits ? dyn0 + atomicAdd(cnt, 1u) : kNoUnit;
  return u < nunits ? u : kNoUnit;
}
__device__ __forceinline__ void sched_done(unsigned* cnt, uint32_t dyn0, uint32_t nunits) {
  // the last CTA out resets the counter pair for the slot's next launch
  if (dyn0 < nunits && atomicAdd(cnt + 1, 1u) == gridDim.x - 1) {
    atomicExch(cnt, 0u);
    atomicExch(cnt + 1, 0u);
  }
}

// first tile row and column of unit u: a 512-tile segment of one row, or (R > 1) R whole rows
__device__ __forceinline__ void unit_coord(uint32_t u, uint32_t upr, uint32_t R, uint32_t& I,
                                           uint32_t& J0) {
  if (R > 1) {
    I = u * R;
    J0 = 0;
  } else {
    I = u / upr;
    J0 = (u - I * upr) * 512u;
  }
}

struct TcArgs {
  __nv_bfloat16* out;
  int64_t ldo;
  const float* coef;  // D: P x 16
  int P, Pb;
  int64_t bc, upr, nunits;
  uint32_t nstages, nbuf;
  uint32_t br, R;   // tile rows; R > 1: a unit is R whole tile rows (narrow matrices)
  unsigned* sched;  // counter pair of this launch's slot
  uint32_t dyn0;
  Trace trace;      // probe build: launch span
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
template <int KS, int EG, int EPW = kEpi>
__global__ void __launch_bounds__(32 * (2 + EPW), 1)
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
  uint64_t* rbar = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rbar + kRing);
  volatile uint32_t* ring = tslot + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nunits = static_cast<uint32_t>(a.nunits), upr = static_cast<uint32_t>(a.upr);
  constexpr int kGW = EPW / EG;  // warps per epilogue group

  if (threadIdx.x == 0) {
    trace_mark(a.trace, false);
    trace_cta(a.trace, 0);
    for (uint32_t i = 0; i < nst; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kGW);
    }
    for (int i = 0; i < kRing; ++i) ptx::mbar_init(&rbar[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tm_in);
  if (warp == 1) ptx::tmem_alloc(tslot, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch_dependents();
  griddep_wait();
  if (threadIdx.x == 0) trace_cta(a.trace, 1);  // the planes of this launch are complete (PDL)
  // The UMMA B operand, after griddep_wait (the coefficients may come from the previous
  // launch) and off the producer's path: the first loads are in flight while it is built;
  // the MMA issuer meets the other non-producer warps at a named barrier before its first MMA.
  if (warp != 0) {
    // B = [D_hi | D_lo]: row n < 16 holds the hi halves of decoder column n, row 16 + n the lo
    // halves; K runs along the 128-byte row (16 elements per step), 16-byte chunks XOR-swizzled
    // by (n & 7).
    for (int i = threadIdx.x - 32; i < 32 * 64; i += 32 * (2 + EPW) - 32) {
      const int n = i >> 6, k = i & 63, c = n & 15, st = k >> 4;
      const int pl = (st == 0 ? 0 : Pb - 16) + (k & 15);
      const float d = st < KS && pl < a.P && pl >= 16 * st ? a.coef[pl * 16 + c] : 0.f;
      const __nv_bfloat16 hi = __float2bfloat16_rn(d);
      const __nv_bfloat16 v = n < 16 ? hi : __float2bfloat16_rn(d - __bfloat162float(hi));
      const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
      *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
    }
    ptx::fence_proxy_async_smem();  // generic-proxy B writes -> the UMMAs (async proxy)
    asm volatile("bar.sync 5, %0;" ::"n"(32 * (2 + EPW) - 32) : "memory");
  }

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      for (uint32_t it = 0;; ++it) {
        const uint32_t u = next_unit(it, nunits, a.dyn0, a.sched);
        ring[it % kRing] = u;
        ptx::mbar_arrive(&rbar[it % kRing]);
        if (u == kNoUnit) {
          ring[(it + 1) % kRing] = u;
          ptx::mbar_arrive(&rbar[(it + 1) % kRing]);
          break;
        }
        const uint32_t st = it % nst, ph = (it / nst) & 1;
        uint32_t I, J0;
      unit_coord(u, upr, a.R, I, J0);
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
      for (uint32_t it = 0;; ++it) {
        ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
        if (ring[it % kRing] == kNoUnit) break;
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
    for (uint32_t it = grp, k = 0;; it += EG, ++k) {
      ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
      const uint32_t u = ring[it % kRing];
      if (u == kNoUnit) break;
      const uint32_t buf = it & 1, bph = (it >> 1) & 1;
      const uint32_t ob0 = s_out + (grp * nbuf + k % nbuf) * kOutBytes;
      uint32_t I, J0;
      unit_coord(u, upr, a.R, I, J0);
      ptx::mbar_wait(&tfull[buf], bph);
      ptx::tc_fence_after();
      if (it == 0 && issuer) trace_cta(a.trace, 2);
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
        if (a.R > 1) {  // R whole tile rows: row r of the unit at staging offset r * bc * 8
          const uint32_t nrows = min(a.R, a.br - I), rb = static_cast<uint32_t>(a.bc) * 8;
          for (uint32_t rr = 0; rr < nrows; ++rr)
#pragma unroll
            for (int r = 0; r < 4; ++r)
              bulk_s2g(a.out + (4 * static_cast<int64_t>(I + rr) + r) * a.ldo,
                       sbase + ob0 + r * kOS + rr * rb, rb);
        } else {
          const uint32_t Tw = min(static_cast<uint32_t>(a.bc) - J0, static_cast<uint32_t>(kT));
#pragma unroll
          for (int r = 0; r < 4; ++r)
            bulk_s2g(a.out + (4 * static_cast<int64_t>(I) + r) * a.ldo + 4 * static_cast<int64_t>(J0),
                     sbase + ob0 + r * kOS, Tw * 8);
        }
        ptx::bulk_commit();
      }
    }
    if (issuer) ptx::bulk_wait_all();
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sched_done(a.sched, a.dyn0, nunits);
  if (threadIdx.x == 0) {
    trace_cta(a.trace, 3);
    trace_mark(a.trace, true);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

// Counter pairs for the dynamic tail (one pool per device, slots round robin over launches: a
// slot comes back after 256 launches, long after its launch finished and reset it).
constexpr int kSchedSlots = 256;
// Host threads may launch concurrently (one mutex around the pool and the slot counter); a
// first call inside a stream capture cannot allocate and falls back to the mma.sync kernels.
std::mutex g_sched_mu;
template <typename A>
bool set_schedule(A& a, uint32_t grid) {
  static unsigned* pools[64] = {};
  static uint32_t next[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  {
    std::lock_guard<std::mutex> lock(g_sched_mu);
    if (!pools[dev]) {
      unsigned* p = nullptr;
      if (cudaMalloc(&p, 2 * kSchedSlots * sizeof(unsigned)) != cudaSuccess) return false;
      if (cudaMemset(p, 0, 2 * kSchedSlots * sizeof(unsigned)) != cudaSuccess) {
        cudaFree(p);
        return false;
      }
      pools[dev] = p;
    }
    a.sched = pools[dev] + 2 * (next[dev]++ % kSchedSlots);
  }
  // trailing rounds taken dynamically: a third of them (measured: 8192^3 with 55 rounds per CTA
  // best at 12-24 dynamic rounds, config 2 with 28 at 8-12; all-dynamic loses the lock-step
  // DRAM locality: profiles/r02_tc_dyn_ab.log). Probe STL_TC_DYN: 0 = static, -1 = all dynamic.
  const uint32_t rounds = static_cast<uint32_t>((a.nunits + grid - 1) / grid);
  static const int dyn_env = probe_env("STL_TC_DYN", -2);
  const int dyn = dyn_env != -2 ? dyn_env : static_cast<int>(rounds / 3 > 2 ? rounds / 3 : 2);
  const uint32_t srounds = dyn < 0 ? 1u : (static_cast<uint32_t>(dyn) >= rounds ? 1u : rounds - dyn);
  a.dyn0 = dyn == 0 ? static_cast<uint32_t>(a.nunits) : srounds * grid;
  return true;
}

template <int KS, int EG, int EPW = kEpi>
cudaError_t launch_tc(const CUtensorMap& tm, TcArgs a, cudaStream_t s) {
  const uint32_t kStage = static_cast<uint32_t>(a.Pb) * kT * 2;
  const uint32_t budget = 227 * 1024 - 1024 - kBBytes - kBarBytes;
  static const int nb_env = probe_env("STL_DEC_TC_NBUF", 0);
  static const int st_env = probe_env("STL_DEC_TC_STAGES", 0);
  a.nbuf = nb_env >= 2 && nb_env <= 6 ? nb_env : (EG == 2 ? 3 : 4);
  if (EG * a.nbuf * kOutBytes + 2 * kStage > budget) return cudaErrorNotSupported;
  uint32_t ns = (budget - EG * a.nbuf * kOutBytes) / kStage;
  a.nstages = ns > kMaxSt ? kMaxSt : ns;
  if (st_env >= 2 && static_cast<uint32_t>(st_env) < a.nstages) a.nstages = st_env;
  const uint32_t smem = a.nstages * kStage + EG * a.nbuf * kOutBytes + kBBytes + kBarBytes + 1024;
  auto k = k_decode_tc<KS, EG, EPW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  if (!set_schedule(a, static_cast<uint32_t>(grid))) return cudaErrorNotSupported;
  a.trace = trace_next();
  return launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(32 * (2 + EPW)), smem, s, tm, a);
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
  uint32_t br, R;   // tile rows; R > 1: a unit is R whole tile rows (narrow matrices)
  unsigned* sched;
  uint32_t dyn0;
  Trace trace;
};

// G = 8-plane groups (N = 32 G); EG epilogue groups as in the decode.
template <int G, int EG, int EPW = kEpi>
__global__ void __launch_bounds__(32 * (2 + EPW), 1)
    k_encode_tc(const __grid_constant__ CUtensorMap tm_out, TcEncArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  constexpr int N = 32 * G;
  constexpr uint32_t kStage = 4 * kERow;
  constexpr uint32_t kB = N * 128;
  constexpr int kGW = EPW / EG;
  constexpr int kEMB = 2;  // M-blocks (128 tile pairs) per unit
  const uint32_t nst = a.nstages, nbuf = a.nbuf, ob_bytes = a.out_bytes;
  const uint32_t s_out = nst * kStage;
  const uint32_t s_b = s_out + EG * nbuf * ob_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + s_b + kB);
  uint64_t* empty = full + kMaxSt;
  uint64_t* tfull = empty + kMaxSt;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rbar + kRing);
  volatile uint32_t* ring = tslot + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = a.P;
  const uint32_t nunits = static_cast<uint32_t>(a.nunits), upr = static_cast<uint32_t>(a.upr);
  const uint32_t bc = static_cast<uint32_t>(a.bc);

  if (threadIdx.x == 0) {
    trace_mark(a.trace, false);
    trace_cta(a.trace, 0);
    for (uint32_t i = 0; i < nst; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kGW);
    }
    for (int i = 0; i < kRing; ++i) ptx::mbar_init(&rbar[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tm_out);
  if (warp == 1) ptx::tmem_alloc(tslot, kTmemColsEnc<G>());
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch_dependents();
  griddep_wait();
  if (threadIdx.x == 0) trace_cta(a.trace, 1);
  // The UMMA B operand, after griddep_wait (the coefficients may come from the previous
  // launch) and off the producer's path: the first loads are in flight while it is built;
  // the MMA issuer meets the other non-producer warps at a named barrier before its first MMA.
  if (warp != 0) {
    for (int i = threadIdx.x - 32; i < N * 32; i += 32 * (2 + EPW) - 32) {
      const int n = i >> 5, k = i & 31;
      const int g = n >> 5, par = (n >> 4) & 1, hl = (n >> 3) & 1, p = 8 * g + (n & 7);
      const int ka = k >> 3, kpar = (k >> 2) & 1, kb = k & 3;
      const float e = kpar == par && p < P ? a.coef[p * 16 + 4 * ka + kb] : 0.f;
      const __nv_bfloat16 hi = __float2bfloat16_rn(e);
      const __nv_bfloat16 v = hl == 0 ? hi : __float2bfloat16_rn(e - __bfloat162float(hi));
      const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
      *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
    }
    for (int i = threadIdx.x - 32; i < N * 32; i += 32 * (2 + EPW) - 32) {  // K 32..63 of each B row: zero
      const int n = i >> 5, k = 32 + (i & 31);
      const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
      *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = __float2bfloat16_rn(0.f);
    }
    ptx::fence_proxy_async_smem();  // generic-proxy B writes -> the UMMAs (async proxy)
    asm volatile("bar.sync 5, %0;" ::"n"(32 * (2 + EPW) - 32) : "memory");
  }

  if (warp == 0) {
    // ---------------------------------------------------------------- producer: 4 matrix rows
    for (uint32_t it = 0;; ++it) {
      uint32_t u = 0;
      if (lane == 0) {
        u = next_unit(it, nunits, a.dyn0, a.sched);
        ring[it % kRing] = u;
        ptx::mbar_arrive(&rbar[it % kRing]);
        if (u == kNoUnit) {
          ring[(it + 1) % kRing] = u;
          ptx::mbar_arrive(&rbar[(it + 1) % kRing]);
        }
      }
      u = __shfl_sync(0xFFFFFFFFu, u, 0);
      if (u == kNoUnit) break;
      const uint32_t st = it % nst, ph = (it / nst) & 1;
      uint32_t I, J0;
      unit_coord(u, upr, a.R, I, J0);
      ptx::mbar_wait(&empty[st], ph ^ 1);
      if (a.R > 1) {
        // R whole tile rows: lane 4 rr + r copies matrix row 4 (I + rr) + r after row rr - 1's
        const uint32_t nrows = min(a.R, a.br - I);
        if (lane == 0) ptx::mbar_arrive_expect_tx(&full[st], nrows * 4 * bc * 8);
        __syncwarp();
        const uint32_t rr = lane >> 2, r = lane & 3;
        if (rr < nrows)
          bulk_g2s(sbase + st * kStage + r * kERow + rr * bc * 8,
                   a.mat + (4 * static_cast<int64_t>(I + rr) + r) * a.ldm, bc * 8, &full[st]);
      } else {
        const uint32_t Tw = min(bc - J0, static_cast<uint32_t>(kT));
        if (lane == 0) ptx::mbar_arrive_expect_tx(&full[st], 4 * Tw * 8);
        __syncwarp();
        if (lane < 4)
          bulk_g2s(sbase + st * kStage + lane * kERow,
                   a.mat + (4 * static_cast<int64_t>(I) + lane) * a.ldm + 4 * static_cast<int64_t>(J0),
                   Tw * 8, &full[st]);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N, false, false);
      for (uint32_t it = 0;; ++it) {
        ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
        if (ring[it % kRing] == kNoUnit) break;
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
    for (uint32_t it = grp, k = 0;; it += EG, ++k) {
      ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
      const uint32_t u = ring[it % kRing];
      if (u == kNoUnit) break;
      const uint32_t buf = it & 1, bph = (it >> 1) & 1;
      const uint32_t ob0 = s_out + (grp * nbuf + k % nbuf) * ob_bytes;
      uint32_t I, J0;
      unit_coord(u, upr, a.R, I, J0);
      ptx::mbar_wait(&tfull[buf], bph);
      ptx::tc_fence_after();
      if (it == 0 && issuer) trace_cta(a.trace, 2);
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
  if (threadIdx.x == 0) sched_done(a.sched, a.dyn0, nunits);
  if (threadIdx.x == 0) {
    trace_cta(a.trace, 3);
    trace_mark(a.trace, true);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemColsEnc<G>());
  }
}

template <int G, int EG, int EPW = kEpi>
cudaError_t launch_enc_tc(const CUtensorMap& tm, TcEncArgs a, cudaStream_t s) {
  constexpr uint32_t kStage = 4 * kERow;
  constexpr uint32_t kB = 32 * G * 128;
  a.out_bytes = (static_cast<uint32_t>(a.P) * kT * 2 + 1023) / 1024 * 1024;
  const uint32_t budget = 227 * 1024 - 1024 - kB - kBarBytes;
  static const int nb_env = probe_env("STL_ENC_TC_NBUF", 0);
  static const int st_env = probe_env("STL_ENC_TC_STAGES", 0);
  a.nbuf = nb_env >= 2 && nb_env <= 6 ? nb_env : 2;
  if (EG * a.nbuf * a.out_bytes + 2 * kStage > budget) return cudaErrorNotSupported;
  const uint32_t ns = (budget - EG * a.nbuf * a.out_bytes) / kStage;
  a.nstages = ns > kMaxSt ? kMaxSt : ns;
  if (st_env >= 2 && static_cast<uint32_t>(st_env) < a.nstages) a.nstages = st_env;
  const uint32_t smem = a.nstages * kStage + EG * a.nbuf * a.out_bytes + kB + kBarBytes + 1024;
  auto k = k_encode_tc<G, EG, EPW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  if (!set_schedule(a, static_cast<uint32_t>(grid))) return cudaErrorNotSupported;
  a.trace = trace_next();
  return launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(32 * (2 + EPW)), smem, s, tm, a);
}

// ------------------------------------------------------------------ fused reductions
// The backward's two transforms with a reduction riding on the same stream:
//   ENC (encode_gy + g_d, toy_network.py:100-101): planes = encode(rows), E = coef
//   DEC (decode_gu + g_ex, toy_network.py:104-105): rows = decode(Z), D = coef
//   both: R[p][c] += sum over tiles j of Z[p][j] rows[j][c]   (Z: P bf16 planes, rows: bf16)
// The change of basis runs on tcgen05 exactly as in k_encode_tc / k_decode_tc; the reduction
// needs Z and the rows transposed against each other (the tile values interleave along the
// matrix rows), so eight more warps run it on mma.sync m16n8k16 from the same landed stage —
// the fragment scheme of k_stream's reductions (stl_stream.cu) — and each stage is released by
// the UMMA commit plus those eight warps. The unit schedule stays static (round robin) so the
// per-warp fragments, their fixed-order sum and the per-CTA partials (summed by sum_partials in
// a fixed order) are bit-reproducible.
// Warps: 0 producer, 1 MMA, 2..9 epilogue (two groups), 10..17 reduction.
constexpr int kRedW = 8;
constexpr int kThreadsRed = 32 * (2 + kEpi + kRedW);
constexpr uint32_t kRowPadR = 64;

struct TcRedArgs {
  const __nv_bfloat16* rows;   // ENC: the matrix encoded; DEC: the reduction's matrix
  int64_t ldr;
  __nv_bfloat16* out;          // DEC: output matrix (ENC planes leave through tm_out)
  int64_t ldo;
  const float* coef;           // ENC: E, DEC: D (P x 16)
  float* red_partial;          // [grid][P * 16]
  int P, Pb;                   // Pb: planes per chunk of the Z box
  int64_t bc, upr, nunits;
  uint32_t nstages, nbuf, out_bytes, stage_bytes, rows_off;
  Trace trace;
  unsigned* sched;   // dynamic tail: item counter (pair) of this launch's slot
  uint32_t dyn0;     // first dynamically scheduled unit (>= nunits: all static)
  uint32_t kitem;    // units per dynamic work item
  uint32_t nitems;   // dynamic work items
};
constexpr uint32_t kNoItem = 0x7FFFFFFFu;
constexpr uint32_t kBarBytesR = kBarBytes + kRing * 4;  // + the ring's work-item entries

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// byte offset of (plane p, tile t) in a 128B-swizzled bf16 plane box with Pb planes per chunk
__device__ __forceinline__ uint32_t zbox_off(int Pb, int p, int t) {
  const uint32_t row = static_cast<uint32_t>((t >> 6) * Pb + p);
  const uint32_t byte = static_cast<uint32_t>((t & 63) * 2);
  return row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
}

// TU = tiles per unit (256 / 512); NK = ENC: 8-plane output groups G, DEC: K-steps KS;
// MT = 16-plane groups of the reduction (ceil(P / 16)).
template <bool ENC, int TU, int NK, int MT>
__global__ void __launch_bounds__(kThreadsRed, 1)
    k_red_tc(const __grid_constant__ CUtensorMap tm_z, const __grid_constant__ CUtensorMap tm_out,
             TcRedArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  constexpr uint32_t RS = TU * 8 + kRowPadR;                // padded matrix row
  constexpr int N = ENC ? 32 * NK : 32;                     // UMMA N
  constexpr int kUMB = ENC ? TU / 256 : TU / 128;           // UMMA M-blocks per unit
  constexpr uint32_t kB = ENC ? N * 128 : kBBytes;
  constexpr uint32_t kTcols = (2 * kUMB * N <= 256) ? 256u : 512u;
  constexpr int kGW = kEpi / 2;
  const int Pb = a.Pb, P = a.P;
  const uint32_t nst = a.nstages, nbuf = a.nbuf, ob_bytes = a.out_bytes, SB = a.stage_bytes;
  const uint32_t s_out = nst * SB;
  const uint32_t s_b = s_out + 2 * nbuf * ob_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + s_b + kB);
  uint64_t* empty = full + kMaxSt;
  uint64_t* tfull = empty + kMaxSt;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rbar + kRing);
  volatile uint32_t* ring = tslot + 4;
  volatile uint32_t* ritem = ring + kRing;  // work item | last-unit flag, or kNoItem
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nunits = static_cast<uint32_t>(a.nunits), upr = static_cast<uint32_t>(a.upr);
  const uint32_t bc = static_cast<uint32_t>(a.bc);

  if (threadIdx.x == 0) {
    trace_mark(a.trace, false);
    trace_cta(a.trace, 0);
    for (uint32_t i = 0; i < nst; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1 + kRedW);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kGW);
    }
    for (int i = 0; i < kRing; ++i) ptx::mbar_init(&rbar[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_z);
    if constexpr (ENC) ptx::prefetch_tmap(&tm_out);
  }
  if (warp == 1) ptx::tmem_alloc(tslot, kTcols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch_dependents();
  griddep_wait();
  if (threadIdx.x == 0) trace_cta(a.trace, 1);
  // The UMMA B operand, after griddep_wait (the coefficients may come from the previous
  // launch) and off the producer's path: the first loads are in flight while it is built;
  // the MMA issuer meets the other non-producer warps at a named barrier before its first MMA.
  if (warp != 0) {
    // the UMMA B operand (as in k_encode_tc / k_decode_tc)
    if constexpr (ENC) {
      for (int i = threadIdx.x - 32; i < N * 64; i += kThreadsRed - 32) {
        const int n = i >> 6, k = i & 63;
        const int g = n >> 5, par = (n >> 4) & 1, hl = (n >> 3) & 1, p = 8 * g + (n & 7);
        const int ka = k >> 3, kpar = (k >> 2) & 1, kb = k & 3;
        const float e = k < 32 && kpar == par && p < P ? a.coef[p * 16 + 4 * ka + kb] : 0.f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(e);
        const __nv_bfloat16 v = hl == 0 ? hi : __float2bfloat16_rn(e - __bfloat162float(hi));
        const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
        *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
      }
    } else {
      for (int i = threadIdx.x - 32; i < 32 * 64; i += kThreadsRed - 32) {
        const int n = i >> 6, k = i & 63, c = n & 15, st = k >> 4;
        const int pl = (st == 0 ? 0 : Pb - 16) + (k & 15);
        const float d = st < NK && pl < P && pl >= 16 * st ? a.coef[pl * 16 + c] : 0.f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(d);
        const __nv_bfloat16 v = n < 16 ? hi : __float2bfloat16_rn(d - __bfloat162float(hi));
        const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
        *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
      }
    }
    ptx::fence_proxy_async_smem();  // generic-proxy B writes -> the UMMAs (async proxy)
    asm volatile("bar.sync 5, %0;" ::"n"(kThreadsRed - 32) : "memory");
  }

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    // static rounds, then work items of kitem consecutive units from the counter
    uint32_t sk = 0, item = 0, jj = a.kitem;
    bool dyn = false;
    for (uint32_t it = 0;; ++it) {
      uint32_t u = kNoUnit;
      if (lane == 0) {
        uint32_t info = kNoItem;
        if (!dyn) {
          u = blockIdx.x + sk * gridDim.x;
          if (u < a.dyn0 && u < nunits) ++sk;
          else dyn = true;
        }
        if (dyn) {
          if (jj == a.kitem) {
            item = a.nitems ? atomicAdd(a.sched, 1u) : kNoItem;
            jj = 0;
          }
          u = item < a.nitems ? a.dyn0 + item * a.kitem + jj : kNoUnit;
          if (u >= nunits) u = kNoUnit;
          if (u != kNoUnit) {
            const bool last = jj + 1 == a.kitem || u + 1 == nunits;
            info = item | (last ? 0x80000000u : 0u);
            ++jj;
          }
        }
        ring[it % kRing] = u;
        ritem[it % kRing] = info;
        ptx::mbar_arrive(&rbar[it % kRing]);
        if (u == kNoUnit) {
          ring[(it + 1) % kRing] = u;
          ritem[(it + 1) % kRing] = kNoItem;
          ptx::mbar_arrive(&rbar[(it + 1) % kRing]);
        }
      }
      u = __shfl_sync(0xFFFFFFFFu, u, 0);
      if (u == kNoUnit) break;
      const uint32_t st = it % nst, ph = (it / nst) & 1;
      const uint32_t I = u / upr, J0 = (u - I * upr) * TU;
      const uint32_t Tw = min(bc - J0, static_cast<uint32_t>(TU));
      ptx::mbar_wait(&empty[st], ph ^ 1);
      const uint32_t sz = sbase + st * SB;
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(Pb) * TU * 2 + 4 * Tw * 8);
        tma_load_4d(&tm_z, &full[st], sz, 0, 0, static_cast<int>(J0 / 64), static_cast<int>(I));
      }
      __syncwarp();
      if (lane < 4)
        bulk_g2s(sz + a.rows_off + lane * RS,
                 a.rows + (4 * static_cast<int64_t>(I) + lane) * a.ldr + 4 * static_cast<int64_t>(J0),
                 Tw * 8, &full[st]);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N, !ENC, false);
      for (uint32_t it = 0;; ++it) {
        ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
        if (ring[it % kRing] == kNoUnit) break;
        const uint32_t st = it % nst, ph = (it / nst) & 1;
        const uint32_t buf = it & 1, bph = (it >> 1) & 1;
        ptx::mbar_wait(&tempty[buf], bph ^ 1);
        ptx::mbar_wait(&full[st], ph);
        ptx::tc_fence_after();
        const uint32_t s0 = sbase + st * SB;
#pragma unroll
        for (int mb = 0; mb < kUMB; ++mb)
#pragma unroll
          for (int ks = 0; ks < (ENC ? 2 : NK); ++ks) {
            uint64_t ad;
            if constexpr (ENC) {
              ad = smem_desc_plain(s0 + a.rows_off + 2 * ks * RS + mb * 2048, RS, 128);
            } else {
              const uint32_t off = ks == 0 ? 0u : static_cast<uint32_t>(Pb - 16);
              ad = ptx::smem_desc_sw128(s0 + (2 * mb * Pb + off) * 128, Pb * 128, 1024);
            }
            const uint64_t bd = ptx::smem_desc_sw128(sbase + s_b + ks * 32, 16, 1024);
            ptx::mma_bf16_ss(tmem + buf * (kUMB * N) + mb * N, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
        ptx::mma_commit(&empty[st]);
        ptx::mma_commit(&tfull[buf]);
      }
    }
  } else if (warp < 2 + kEpi) {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 2;
    const int grp = ew / kGW, gw = ew % kGW;
    const uint32_t quarter = warp & 3;
    const bool issuer = gw == 0 && lane == 0;
    for (uint32_t it = grp, k = 0;; it += 2, ++k) {
      ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
      const uint32_t u = ring[it % kRing];
      if (u == kNoUnit) break;
      const uint32_t buf = it & 1, bph = (it >> 1) & 1;
      const uint32_t ob0 = s_out + (grp * nbuf + k % nbuf) * ob_bytes;
      const uint32_t I = u / upr, J0 = (u - I * upr) * TU;
      ptx::mbar_wait(&tfull[buf], bph);
      ptx::tc_fence_after();
      if (it == 0 && issuer) trace_cta(a.trace, 2);
      if constexpr (ENC) {
#pragma unroll 1
        for (int mb = 0; mb < kUMB; ++mb) {
          const uint32_t chunk = 4 * mb + quarter;
#pragma unroll
          for (int g0 = 0; g0 < NK; g0 += 2) {
            float v[2][32];
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (g0 + h < NK)
                tmem_ld_x32(tmem + ((quarter * 32) << 16) + buf * (kUMB * N) + mb * N + 32 * (g0 + h), v[h]);
            ptx::tmem_ld_wait();
            if (mb == kUMB - 1 && g0 + 2 >= NK) {
              ptx::tc_fence_before();
              __syncwarp();
              if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int pp = 0; pp < 8; ++pp) {
                const int p = 8 * (g0 + h) + pp;
                if (g0 + h < NK && p < P) {
                  const uint32_t row = chunk * P + p;
                  const uint32_t byte = 4 * lane;
                  const uint32_t off = row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
                  *reinterpret_cast<uint32_t*>(smem + ob0 + off) =
                      pack_bf16(v[h][pp] + v[h][8 + pp], v[h][16 + pp] + v[h][24 + pp]);
                }
              }
          }
        }
      } else {
        constexpr int kMBW = kUMB * 4 / kGW;  // M-blocks per warp (all of the unit's)
        static_assert(kMBW % 2 == 0, "M-blocks per warp");
        constexpr uint32_t OS = TU * 8;
#pragma unroll
        for (int j = 0; j < kMBW; j += 2) {
          float v[2][32];
#pragma unroll
          for (int h = 0; h < 2; ++h)
            tmem_ld_x32(tmem + ((quarter * 32) << 16) + buf * (kUMB * 32) + (j + h) * 32, v[h]);
          ptx::tmem_ld_wait();
          if (j == kMBW - 2) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t m = (j + h) * 128 + quarter * 32 + lane;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const uint32_t w0 = pack_bf16(v[h][4 * r] + v[h][16 + 4 * r], v[h][4 * r + 1] + v[h][17 + 4 * r]);
              const uint32_t w1 = pack_bf16(v[h][4 * r + 2] + v[h][18 + 4 * r], v[h][4 * r + 3] + v[h][19 + 4 * r]);
              *reinterpret_cast<uint2*>(smem + ob0 + r * OS + m * 8) = make_uint2(w0, w1);
            }
          }
        }
      }
      ptx::fence_proxy_async_smem();
      if (issuer) bulk_wait_read_n(nbuf - 2);
      epi_bar(grp, 32 * kGW);
      if (issuer) {
        if constexpr (ENC) {
          tma_store_4d(&tm_out, sbase + ob0, 0, 0, static_cast<int>(J0 / 64), static_cast<int>(I));
        } else {
          const uint32_t Tw = min(bc - J0, static_cast<uint32_t>(TU));
#pragma unroll
          for (int r = 0; r < 4; ++r)
            bulk_s2g(a.out + (4 * static_cast<int64_t>(I) + r) * a.ldo + 4 * static_cast<int64_t>(J0),
                     sbase + ob0 + r * (TU * 8), Tw * 8);
        }
        ptx::bulk_commit();
      }
    }
    if (issuer) ptx::bulk_wait_all();
  } else {
    // ---------------------------------------------------------------- reduction (mma.sync)
    // warp wr takes the unit's 16-tile k-steps wr, wr + 8, ...: A = Z (rows = planes g / g + 8
    // of each 16-plane group, k = tiles 2q, 2q + 1 | + 8), B = rows (n = c = 8 nt + g: matrix row
    // c >> 2, element c & 3 of tiles 2q, 2q + 1 | + 8; 16-bit loads, distinct words)
    const int wr = warp - 2 - kEpi;
    const int g = lane >> 2, q = lane & 3;
    constexpr int kKS = TU / (16 * kRedW);
    float R[MT][2][4];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int k = 0; k < 4; ++k) R[m][n][k] = 0.f;
    uint32_t rb[2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int c = 8 * nt + g;
      rb[nt] = (c >> 2) * RS + 16 * q + 2 * (c & 3);
    }
    bool ok[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      ok[mt][0] = 16 * mt + g < P;
      ok[mt][1] = 16 * mt + g + 8 < P;
    }
    // per-warp fragments -> a dedicated smem region -> fixed-order sum over the warps -> one
    // partial: this CTA's static units (slot blockIdx.x), then one per dynamic work item (slot
    // grid + item), so every partial covers a fixed set of units whichever CTA ran it
    const int n = P * 16;
    float* s_red = reinterpret_cast<float*>(smem + s_b + kB + kBarBytesR);
    auto flush = [&](uint32_t slot) {
      float* mine = s_red + wr * n;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int c = 8 * nt + 2 * q, p0 = 16 * mt + g, p1 = p0 + 8;
          if (p0 < P) {
            mine[p0 * 16 + c] = R[mt][nt][0];
            mine[p0 * 16 + c + 1] = R[mt][nt][1];
          }
          if (p1 < P) {
            mine[p1 * 16 + c] = R[mt][nt][2];
            mine[p1 * 16 + c + 1] = R[mt][nt][3];
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) R[mt][nt][k] = 0.f;
        }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * kRedW) : "memory");
      for (int o = wr * 32 + lane; o < n; o += 32 * kRedW) {
        float sum = s_red[o];
#pragma unroll
        for (int w = 1; w < kRedW; ++w) sum += s_red[w * n + o];
        a.red_partial[static_cast<int64_t>(slot) * n + o] = sum;
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * kRedW) : "memory");
    };
    bool static_done = false;
    for (uint32_t it = 0;; ++it) {
      ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
      const uint32_t u = ring[it % kRing];
      const uint32_t info = ritem[it % kRing];
      if (u == kNoUnit) break;
      if (info != kNoItem && !static_done) {
        flush(blockIdx.x);
        static_done = true;
      }
      const uint32_t st = it % nst, ph = (it / nst) & 1;
      const uint32_t J0 = (u - (u / upr) * upr) * TU;
      const int Tw = static_cast<int>(min(bc - J0, static_cast<uint32_t>(TU)));
      ptx::mbar_wait(&full[st], ph);
      const uint32_t so = st * SB;
#pragma unroll
      for (int k = 0; k < kKS; ++k) {
        const int t0 = 16 * (wr + kRedW * k);
        if (t0 < Tw) {
          uint32_t b[2][2];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const uint8_t* base = smem + so + a.rows_off + rb[nt] + t0 * 8;
            const uint32_t x0 = *reinterpret_cast<const uint16_t*>(base);
            const uint32_t x1 = *reinterpret_cast<const uint16_t*>(base + 8);
            const uint32_t x8 = *reinterpret_cast<const uint16_t*>(base + 64);
            const uint32_t x9 = *reinterpret_cast<const uint16_t*>(base + 72);
            b[nt][0] = x0 | (x1 << 16);
            b[nt][1] = x8 | (x9 << 16);
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int p0 = 16 * mt + g;
            const uint32_t z0 = so + zbox_off(Pb, p0, t0 + 2 * q);
            const uint32_t z2 = so + zbox_off(Pb, p0, t0 + 2 * q + 8);
            const uint32_t a0 = ok[mt][0] ? *reinterpret_cast<const uint32_t*>(smem + z0) : 0u;
            const uint32_t a2 = ok[mt][0] ? *reinterpret_cast<const uint32_t*>(smem + z2) : 0u;
            const uint32_t a1 = ok[mt][1] ? *reinterpret_cast<const uint32_t*>(smem + z0 + 1024) : 0u;
            const uint32_t a3 = ok[mt][1] ? *reinterpret_cast<const uint32_t*>(smem + z2 + 1024) : 0u;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) mma16816(R[mt][nt], a0, a1, a2, a3, b[nt][0], b[nt][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[st]);
      if (info != kNoItem && (info >> 31)) flush(gridDim.x + (info & 0x7FFFFFFFu));
    }
    if (!static_done) flush(blockIdx.x);
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sched_done(a.sched, a.dyn0, nunits);
  if (threadIdx.x == 0) {
    trace_cta(a.trace, 3);
    trace_mark(a.trace, true);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTcols);
  }
}

template <bool ENC, int TU, int NK, int MT>
cudaError_t launch_red_tc(const CUtensorMap& tz, const CUtensorMap& to, TcRedArgs a, float* red_out,
                          cudaStream_t s) {
  constexpr int N = ENC ? 32 * NK : 32;
  constexpr uint32_t kB = ENC ? N * 128 : kBBytes;
  const uint32_t zbytes = (static_cast<uint32_t>(a.Pb) * TU * 2 + 1023) / 1024 * 1024;
  a.rows_off = zbytes;
  a.stage_bytes = (zbytes + 4 * (TU * 8 + kRowPadR) + 1023) / 1024 * 1024;
  a.out_bytes = ENC ? (static_cast<uint32_t>(a.P) * TU * 2 + 1023) / 1024 * 1024 : 4 * TU * 8;
  const uint32_t red_bytes = kRedW * a.P * 16 * 4;  // the per-warp partials
  const uint32_t budget = 227 * 1024 - 1024 - kB - kBarBytesR - red_bytes;
  static const int nb_env = probe_env("STL_RED_TC_NBUF", 0);
  a.nbuf = nb_env >= 2 && nb_env <= 4 ? nb_env : 2;
  if (2 * a.nbuf * a.out_bytes + 2 * a.stage_bytes > budget) return cudaErrorNotSupported;
  const uint32_t ns = (budget - 2 * a.nbuf * a.out_bytes) / a.stage_bytes;
  a.nstages = ns > kMaxSt ? kMaxSt : ns;
  const uint32_t smem =
      a.nstages * a.stage_bytes + 2 * a.nbuf * a.out_bytes + kB + kBarBytesR + red_bytes + 1024;
  auto k = k_red_tc<ENC, TU, NK, MT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  // Probe STL_RED_DYN=1: a dynamic tail (the last third of the rounds as work items of >= 4
  // units, at most kRedBlocks - grid of them, each with its own partial so the sum stays
  // bit-reproducible). Measured slower at config 2 (decode_gu + g_ex 53.8 -> 59.7 us: the
  // per-item partial flushes; profiles/r02_red_dyn_ab.log), so the product runs static.
  if (!set_schedule(a, static_cast<uint32_t>(grid))) return cudaErrorNotSupported;
  static const int red_dyn = probe_env("STL_RED_DYN", 0);
  a.kitem = 4;
  a.nitems = 0;
  if (!red_dyn || a.dyn0 >= a.nunits) {
    a.dyn0 = static_cast<uint32_t>(a.nunits);
  } else {
    const uint32_t ndyn = static_cast<uint32_t>(a.nunits) - a.dyn0;
    const uint32_t cap = static_cast<uint32_t>(kRedBlocks - grid);
    if (ndyn > a.kitem * cap) a.kitem = (ndyn + cap - 1) / cap;
    a.nitems = (ndyn + a.kitem - 1) / a.kitem;
  }
  a.trace = trace_next();
  e = launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(kThreadsRed), smem, s, tz, to, a);
  if (e != cudaSuccess) return e;
  return sum_partials(a.red_partial, static_cast<int>(grid + a.nitems), a.P * 16, red_out, s);
}

// ------------------------------------------------------------------ remix (fused chain)
//   out[p][I][J] = sum_q C[p][q] Z[q][I][J],  C = e_x d^T     (snf_operator.py:175-188)
// K11's operand scheme with the plane box on both sides: A = the landed input box (MN-major),
// B[q][n] = C split into bf16 hi + lo, n = 16 g + 8 hl + pp (output plane p = 8 g + pp), so a
// 32x32b.x16 read-back holds a group's hi and lo columns; the epilogue writes the output planes
// into a swizzled box for one TMA store. C is formed in the kernel prologue.
// GW = epilogue warps per group: 4 (each warp all 4 M-blocks of its TMEM lane quarter) or 8
// (two warps per quarter, 2 M-blocks each).
template <int KS, int G, int GW>
__global__ void __launch_bounds__(32 * (2 + 2 * GW), 1)
    k_remix_tc(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
               TcEncArgs a, const float* __restrict__ e_x, const float* __restrict__ dcoef) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  constexpr int N = 16 * G;
  constexpr uint32_t kB = N * 128 < 1024 ? 1024 : N * 128;
  constexpr uint32_t kTc = 2 * kMB * N <= 256 ? 256u : 512u;
  constexpr int kGW = GW;
  constexpr int kThr = 32 * (2 + 2 * GW);
  const int P = a.P;
  const int Pb = P <= 16 ? 16 : (P + 7) / 8 * 8;
  const uint32_t kStage = static_cast<uint32_t>(Pb) * kT * 2;
  const uint32_t nst = a.nstages, nbuf = a.nbuf, ob_bytes = a.out_bytes;
  const uint32_t s_out = nst * kStage;
  const uint32_t s_b = s_out + 2 * nbuf * ob_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + s_b + kB);
  uint64_t* empty = full + kMaxSt;
  uint64_t* tfull = empty + kMaxSt;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rbar + kRing);
  volatile uint32_t* ring = tslot + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nunits = static_cast<uint32_t>(a.nunits), upr = static_cast<uint32_t>(a.upr);

  if (threadIdx.x == 0) {
    trace_mark(a.trace, false);
    trace_cta(a.trace, 0);
    for (uint32_t i = 0; i < nst; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kGW);
    }
    for (int i = 0; i < kRing; ++i) ptx::mbar_init(&rbar[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tm_in);
    ptx::prefetch_tmap(&tm_out);
  }
  if (warp == 1) ptx::tmem_alloc(tslot, kTc);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch_dependents();
  griddep_wait();
  if (threadIdx.x == 0) trace_cta(a.trace, 1);
  // The UMMA B operand, after griddep_wait (the coefficients may come from the previous
  // launch) and off the producer's path: the first loads are in flight while it is built;
  // the MMA issuer meets the other non-producer warps at a named barrier before its first MMA.
  if (warp != 0) {
    for (int i = threadIdx.x - 32; i < N * 64; i += kThr - 32) {
      const int n = i >> 6, k = i & 63, st = k >> 4;
      const int g = n >> 4, hl = (n >> 3) & 1, p = 8 * g + (n & 7);
      const int q = (st == 0 ? 0 : Pb - 16) + (k & 15);
      float c = 0.f;
      if (st < KS && p < P && q < P && q >= 16 * st) {
  #pragma unroll
        for (int kk = 0; kk < 16; ++kk) c = fmaf(e_x[p * 16 + kk], dcoef[q * 16 + kk], c);
      }
      const __nv_bfloat16 hi = __float2bfloat16_rn(c);
      const __nv_bfloat16 v = hl == 0 ? hi : __float2bfloat16_rn(c - __bfloat162float(hi));
      const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
      *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
    }
    ptx::fence_proxy_async_smem();  // generic-proxy B writes -> the UMMAs (async proxy)
    asm volatile("bar.sync 5, %0;" ::"n"(kThr - 32) : "memory");
  }

  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t it = 0;; ++it) {
        const uint32_t u = next_unit(it, nunits, a.dyn0, a.sched);
        ring[it % kRing] = u;
        ptx::mbar_arrive(&rbar[it % kRing]);
        if (u == kNoUnit) {
          ring[(it + 1) % kRing] = u;
          ptx::mbar_arrive(&rbar[(it + 1) % kRing]);
          break;
        }
        const uint32_t st = it % nst, ph = (it / nst) & 1;
        const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
        ptx::mbar_wait(&empty[st], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[st], kStage);
        tma_load_4d(&tm_in, &full[st], sbase + st * kStage, 0, 0, static_cast<int>(J0 / 64),
                    static_cast<int>(I));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N, true, false);
      for (uint32_t it = 0;; ++it) {
        ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
        if (ring[it % kRing] == kNoUnit) break;
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
            const uint32_t off = ks == 0 ? 0u : static_cast<uint32_t>(Pb - 16);
            const uint64_t ad = ptx::smem_desc_sw128(a0 + (2 * mb * Pb + off) * 128, Pb * 128, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(sbase + s_b + ks * 32, 16, 1024);
            ptx::mma_bf16_ss(tmem + buf * (kMB * N) + mb * N, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
        ptx::mma_commit(&empty[st]);
        ptx::mma_commit(&tfull[buf]);
      }
    }
  } else {
    const int ew = warp - 2;
    const int grp = ew / kGW, gw = ew % kGW;
    const uint32_t quarter = warp & 3;
    const bool issuer = gw == 0 && lane == 0;
    for (uint32_t it = grp, k = 0;; it += 2, ++k) {
      ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
      const uint32_t u = ring[it % kRing];
      if (u == kNoUnit) break;
      const uint32_t buf = it & 1, bph = (it >> 1) & 1;
      const uint32_t ob0 = s_out + (grp * nbuf + k % nbuf) * ob_bytes;
      const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
      ptx::mbar_wait(&tfull[buf], bph);
      ptx::tc_fence_after();
      if (it == 0 && issuer) trace_cta(a.trace, 2);
      constexpr int kMBW = kMB * 4 / kGW;  // M-blocks per warp
      const int mb0 = (gw >> 2) * kMBW;
#pragma unroll 1
      for (int mb = mb0; mb < mb0 + kMBW; ++mb) {
        const uint32_t m = mb * 128 + quarter * 32 + lane;  // tile of the unit
        const uint32_t chunk = m >> 6, byte = (m & 63) * 2;
#pragma unroll
        for (int g0 = 0; g0 < G; g0 += 2) {
          float v[2][16];
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (g0 + h < G) {
              uint32_t (&uu)[16] = reinterpret_cast<uint32_t(&)[16]>(v[h]);
              ptx::tmem_ld_32x32b_x16(tmem + ((quarter * 32) << 16) + buf * (kMB * N) + mb * N + 16 * (g0 + h), uu);
            }
          ptx::tmem_ld_wait();
          if (mb == mb0 + kMBW - 1 && g0 + 2 >= G) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int pp = 0; pp < 8; ++pp) {
              const int p = 8 * (g0 + h) + pp;
              if (g0 + h < G && p < P) {
                const uint32_t row = chunk * P + p;
                const uint32_t off = row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
                *reinterpret_cast<__nv_bfloat16*>(smem + ob0 + off) = __float2bfloat16_rn(v[h][pp] + v[h][8 + pp]);
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
  if (threadIdx.x == 0) sched_done(a.sched, a.dyn0, nunits);
  if (threadIdx.x == 0) {
    trace_cta(a.trace, 3);
    trace_mark(a.trace, true);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTc);
  }
}

// 8 epilogue warps per group (8192^2 remix 95.6 -> 93.5 us, profiles/r02_remix_gw_ab.log);
// probe STL_REMIX_TC_GW=4: 4
template <int KS, int G, int GW = 8>
cudaError_t launch_remix_tc(const CUtensorMap& ti, const CUtensorMap& to, TcEncArgs a,
                            const float* e_x, const float* d, cudaStream_t s) {
#ifdef STL_PROBES
  if constexpr (GW == 8)
    if (probe_env("STL_REMIX_TC_GW", 8) == 4) return launch_remix_tc<KS, G, 4>(ti, to, a, e_x, d, s);
#endif
  constexpr int N = 16 * G;
  constexpr uint32_t kB = N * 128 < 1024 ? 1024 : N * 128;
  const int Pb = a.P <= 16 ? 16 : (a.P + 7) / 8 * 8;
  const uint32_t kStage = static_cast<uint32_t>(Pb) * kT * 2;
  a.out_bytes = (static_cast<uint32_t>(a.P) * kT * 2 + 1023) / 1024 * 1024;
  const uint32_t budget = 227 * 1024 - 1024 - kB - kBarBytes;
  static const int nb_env = probe_env("STL_REMIX_TC_NBUF", 0);
  a.nbuf = nb_env >= 2 && nb_env <= 4 ? nb_env : 2;
  if (2 * a.nbuf * a.out_bytes + 2 * kStage > budget) return cudaErrorNotSupported;
  const uint32_t ns = (budget - 2 * a.nbuf * a.out_bytes) / kStage;
  a.nstages = ns > kMaxSt ? kMaxSt : ns;
  const uint32_t smem = a.nstages * kStage + 2 * a.nbuf * a.out_bytes + kB + kBarBytes + 1024;
  auto k = k_remix_tc<KS, G, GW>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  if (!set_schedule(a, static_cast<uint32_t>(grid))) return cudaErrorNotSupported;
  a.trace = trace_next();
  return launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(32 * (2 + 2 * GW)), smem, s, ti, to, a,
                    e_x, d);
}

// ------------------------------------------------------------------ t = 2 (configs[2])
// The decode for 2x2 tiles (c = 2a + b: matrix row 2I + a, column 2J + b).
// Decode (k_decode2_tc): A = the plane box exactly as in k_decode_tc, B = [D_hi | D_lo | 0]
// (N = 16: 4 + 4 columns and 8 zero ones, the smallest N an M = 128 UMMA takes); the epilogue
// packs a tile's two values of each of its 2 matrix rows into one bf16x2 word.
// (An encode twin — tile quads as the K-major operand, one K-step per unit — measured even to
// slower than the register-streaming t = 2 encode and was removed: profiles/r02_t2_tc_ab.log.)
constexpr uint32_t kOS2 = kT * 4;         // t = 2 output staging row: 512 tiles x 2 bf16
constexpr uint32_t kBBytes2 = 16 * 128;   // decode B: 16 rows

template <int KS>
__global__ void __launch_bounds__(kThreads, 1)
    k_decode2_tc(const __grid_constant__ CUtensorMap tm_in, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  const int Pb = a.Pb;
  const uint32_t kStage = static_cast<uint32_t>(Pb) * kT * 2;
  const uint32_t nst = a.nstages, nbuf = a.nbuf;
  constexpr uint32_t kOut2 = 2 * kOS2;
  constexpr int kGW = kEpi / 2;
  const uint32_t s_out = nst * kStage;
  const uint32_t s_b = s_out + 2 * nbuf * kOut2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + s_b + kBBytes2);
  uint64_t* empty = full + kMaxSt;
  uint64_t* tfull = empty + kMaxSt;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rbar + kRing);
  volatile uint32_t* ring = tslot + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nunits = static_cast<uint32_t>(a.nunits), upr = static_cast<uint32_t>(a.upr);

  if (threadIdx.x == 0) {
    trace_mark(a.trace, false);
    for (uint32_t i = 0; i < nst; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tfull[i], 1);
      ptx::mbar_init(&tempty[i], kGW);
    }
    for (int i = 0; i < kRing; ++i) ptx::mbar_init(&rbar[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tm_in);
  if (warp == 1) ptx::tmem_alloc(tslot, 128);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_launch_dependents();
  griddep_wait();
  if (warp != 0) {  // B after griddep_wait, off the producer's path (as in k_decode_tc)
    for (int i = threadIdx.x - 32; i < 16 * 64; i += kThreads - 32) {
      const int n = i >> 6, k = i & 63, c = n & 3, st = k >> 4;
      const int pl = (st == 0 ? 0 : Pb - 16) + (k & 15);
      const float d = n < 8 && st < KS && pl < a.P && pl >= 16 * st ? a.coef[pl * 4 + c] : 0.f;
      const __nv_bfloat16 hi = __float2bfloat16_rn(d);
      const __nv_bfloat16 v = n < 4 ? hi : __float2bfloat16_rn(d - __bfloat162float(hi));
      const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + ((k * 2) & 15);
      *reinterpret_cast<__nv_bfloat16*>(smem + s_b + off) = v;
    }
    ptx::fence_proxy_async_smem();
    asm volatile("bar.sync 5, %0;" ::"n"(kThreads - 32) : "memory");
  }

  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t it = 0;; ++it) {
        const uint32_t u = next_unit(it, nunits, a.dyn0, a.sched);
        ring[it % kRing] = u;
        ptx::mbar_arrive(&rbar[it % kRing]);
        if (u == kNoUnit) {
          ring[(it + 1) % kRing] = u;
          ptx::mbar_arrive(&rbar[(it + 1) % kRing]);
          break;
        }
        const uint32_t st = it % nst, ph = (it / nst) & 1;
        const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
        ptx::mbar_wait(&empty[st], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[st], kStage);
        tma_load_4d(&tm_in, &full[st], sbase + st * kStage, 0, 0, static_cast<int>(J0 / 64),
                    static_cast<int>(I));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, 16, true, false);
      for (uint32_t it = 0;; ++it) {
        ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
        if (ring[it % kRing] == kNoUnit) break;
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
            const uint32_t off = ks == 0 ? 0u : static_cast<uint32_t>(Pb - 16);
            const uint64_t ad = ptx::smem_desc_sw128(a0 + (2 * mb * Pb + off) * 128, Pb * 128, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(sbase + s_b + ks * 32, 16, 1024);
            ptx::mma_bf16_ss(tmem + buf * (kMB * 16) + mb * 16, ad, bd, idesc, ks > 0 ? 1u : 0u);
          }
        ptx::mma_commit(&empty[st]);
        ptx::mma_commit(&tfull[buf]);
      }
    }
  } else {
    const int ew = warp - 2;
    const int grp = ew / kGW, gw = ew % kGW;
    const uint32_t quarter = warp & 3;
    const bool issuer = gw == 0 && lane == 0;
    for (uint32_t it = grp, k = 0;; it += 2, ++k) {
      ptx::mbar_wait(&rbar[it % kRing], (it / kRing) & 1);
      const uint32_t u = ring[it % kRing];
      if (u == kNoUnit) break;
      const uint32_t buf = it & 1, bph = (it >> 1) & 1;
      const uint32_t ob0 = s_out + (grp * nbuf + k % nbuf) * kOut2;
      const uint32_t I = u / upr, J0 = (u - I * upr) * kT;
      ptx::mbar_wait(&tfull[buf], bph);
      ptx::tc_fence_after();
      uint32_t v[kMB][16];
#pragma unroll
      for (int mb = 0; mb < kMB; ++mb)
        ptx::tmem_ld_32x32b_x16(tmem + ((quarter * 32) << 16) + buf * (kMB * 16) + mb * 16, v[mb]);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);
#pragma unroll
      for (int mb = 0; mb < kMB; ++mb) {
        const uint32_t m = mb * 128 + quarter * 32 + lane;
        float y[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) y[c] = __uint_as_float(v[mb][c]) + __uint_as_float(v[mb][4 + c]);
#pragma unroll
        for (int r = 0; r < 2; ++r)
          *reinterpret_cast<uint32_t*>(smem + ob0 + r * kOS2 + m * 4) = pack_bf16(y[2 * r], y[2 * r + 1]);
      }
      ptx::fence_proxy_async_smem();
      if (issuer) bulk_wait_read_n(nbuf - 2 > 1 ? 1 : nbuf - 2);
      epi_bar(grp, 32 * kGW);
      if (issuer) {
        const uint32_t Tw = min(static_cast<uint32_t>(a.bc) - J0, static_cast<uint32_t>(kT));
#pragma unroll
        for (int r = 0; r < 2; ++r)
          bulk_s2g(a.out + (2 * static_cast<int64_t>(I) + r) * a.ldo + 2 * static_cast<int64_t>(J0),
                   sbase + ob0 + r * kOS2, Tw * 4);
        ptx::bulk_commit();
      }
    }
    if (issuer) ptx::bulk_wait_all();
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) sched_done(a.sched, a.dyn0, nunits);
  if (threadIdx.x == 0) trace_mark(a.trace, true);
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 128);
  }
}

template <int KS>
cudaError_t launch_dec2_tc(const CUtensorMap& tm, TcArgs a, cudaStream_t s) {
  const uint32_t kStage = static_cast<uint32_t>(a.Pb) * kT * 2;
  constexpr uint32_t kOut2 = 2 * kOS2;
  const uint32_t budget = 227 * 1024 - 1024 - kBBytes2 - kBarBytes;
  a.nbuf = 3;
  const uint32_t ns = (budget - 2 * a.nbuf * kOut2) / kStage;
  if (ns < 2) return cudaErrorNotSupported;
  a.nstages = ns > kMaxSt ? kMaxSt : ns;
  const uint32_t smem = a.nstages * kStage + 2 * a.nbuf * kOut2 + kBBytes2 + kBarBytes + 1024;
  auto k = k_decode2_tc<KS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  if (!set_schedule(a, static_cast<uint32_t>(grid))) return cudaErrorNotSupported;
  a.trace = trace_next();
  return launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(kThreads), smem, s, tm, a);
}

}  // namespace

cudaError_t planes_to_tiles_tc(const void* in, int P, int64_t br, int64_t bc, const float* coef,
                               void* out, int64_t ldo, cudaStream_t s, int64_t plane_rows) {
  static const int on = probe_env("STL_DEC_TC", 1);
  // narrow matrices (bc < 512, bc | 512): units of R = 512 / bc whole tile rows
  const int R = bc < kT && bc >= 64 && kT % bc == 0 ? static_cast<int>(kT / bc) : 1;
  if (!on || P < 1 || P > 32 || (bc < kT && R == 1) || bc % 64 || ldo % 8 ||
      (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  const int Pb = P <= 16 ? 16 : (P + 7) / 8 * 8;
  CUtensorMap tm{};
  if (plane_rows < br) plane_rows = br;
  if (R > 1 && plane_rows != br) return cudaErrorNotSupported;
  if (!plane_box_tmap(&tm, in, 2, P, Pb, br, bc, kT, plane_rows, R)) return cudaErrorNotSupported;
  TcArgs a{};
  a.br = static_cast<uint32_t>(br);
  a.R = static_cast<uint32_t>(R);
  a.out = static_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.coef = coef;
  a.P = P;
  a.Pb = Pb;
  a.bc = bc;
  a.upr = R > 1 ? 1 : (bc + kT - 1) / kT;
  a.nunits = R > 1 ? (br + R - 1) / R : br * a.upr;
#ifdef STL_PROBES
  if (probe_env("STL_DEC_TC_EG", 2) == 1)  // probe: one 8-warp epilogue group
    return Pb <= 16 ? launch_tc<1, 1>(tm, a, s) : launch_tc<2, 1>(tm, a, s);
#endif
  return Pb <= 16 ? launch_tc<1, 2>(tm, a, s) : launch_tc<2, 2>(tm, a, s);
}

// bf16 matrix (4 br x 4 bc, leading dim ldm) -> P <= 32 bf16 planes (P x plane_rows x bc).
cudaError_t tiles_to_planes_tc(const void* m, int64_t ldm, int64_t br, int64_t bc,
                               const float* coef, int P, void* out, cudaStream_t s,
                               int64_t plane_rows) {
  static const int on = probe_env("STL_ENC_TC", 1);
  const int R = bc < kT && bc >= 64 && kT % bc == 0 ? static_cast<int>(kT / bc) : 1;
  if (!on || P < 1 || P > 32 || (bc < kT && R == 1) || bc % 64 || ldm % 8 ||
      (reinterpret_cast<uintptr_t>(m) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  CUtensorMap tm{};
  if (plane_rows < br) plane_rows = br;
  if (R > 1 && plane_rows != br) return cudaErrorNotSupported;
  if (!plane_box_tmap(&tm, out, 2, P, P, br, bc, kT, plane_rows, R)) return cudaErrorNotSupported;
  TcEncArgs a{};
  a.br = static_cast<uint32_t>(br);
  a.R = static_cast<uint32_t>(R);
  a.mat = static_cast<const __nv_bfloat16*>(m);
  a.ldm = ldm;
  a.coef = coef;
  a.P = P;
  a.bc = bc;
  a.upr = R > 1 ? 1 : (bc + kT - 1) / kT;
  a.nunits = R > 1 ? (br + R - 1) / R : br * a.upr;
#ifdef STL_PROBES
  if (probe_env("STL_ENC_TC_EG", 2) == 1) {  // probe: one 8-warp epilogue group
    switch ((P + 7) / 8) {
      case 1: return launch_enc_tc<1, 1>(tm, a, s);
      case 2: return launch_enc_tc<2, 1>(tm, a, s);
      case 3: return launch_enc_tc<3, 1>(tm, a, s);
      default: return launch_enc_tc<4, 1>(tm, a, s);
    }
  }
#endif
  switch ((P + 7) / 8) {
    case 1: return launch_enc_tc<1, 2>(tm, a, s);
    case 2: return launch_enc_tc<2, 2>(tm, a, s);
    case 3: return launch_enc_tc<3, 2>(tm, a, s);
    default: return launch_enc_tc<4, 2>(tm, a, s);
  }
}

// The backward's fused transforms on tcgen05 + mma.sync (k_red_tc): bf16 rows, bf16 Z planes,
// P <= 32. enc: planes_out = encode(rows) (tiles_to_planes_stream with reduction planes);
// dec: rows_out = decode(Z) (planes_to_tiles_stream with a reduction matrix).
cudaError_t red_transform_tc(bool enc, const void* rows, int64_t ldr, const void* z, int P,
                             int64_t br, int64_t bc, const float* coef, void* out, int64_t ldo,
                             float* red_out, float* red_ws, cudaStream_t s, int64_t plane_rows) {
  // default: the decode-reduction only (g_x + g_ex 52 -> 49 us at config 2); the encode-
  // reduction on tcgen05 measured even with the mma.sync one (profiles/r02_red_tc_ab.log), so it
  // stays there (probe STL_RED_TC=1: both, 0: neither)
  static const int on = probe_env("STL_RED_TC", 2);
  static const int tu_env = probe_env("STL_RED_TC_T", 0);
  const int TU = tu_env ? tu_env : (enc ? 256 : 512);
  if (on == 2 && enc) return cudaErrorNotSupported;  // probe: decode-reduction only
  if (!on || P < 1 || P > 32 || bc < TU || bc % 64 || ldr % 8 || (!enc && ldo % 8) ||
      (reinterpret_cast<uintptr_t>(rows) & 15) || (reinterpret_cast<uintptr_t>(z) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15) || !red_out || !red_ws || (TU != 256 && TU != 512))
    return cudaErrorNotSupported;
  if (plane_rows < br) plane_rows = br;
  const int Pb = enc ? (P + 7) / 8 * 8 : (P <= 16 ? 16 : (P + 7) / 8 * 8);
  CUtensorMap tz{}, to{};
  if (!plane_box_tmap(&tz, z, 2, P, Pb, br, bc, TU, plane_rows)) return cudaErrorNotSupported;
  if (enc && !plane_box_tmap(&to, out, 2, P, P, br, bc, TU, plane_rows)) return cudaErrorNotSupported;
  TcRedArgs a{};
  a.rows = static_cast<const __nv_bfloat16*>(rows);
  a.ldr = ldr;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.coef = coef;
  a.red_partial = red_ws;
  a.P = P;
  a.Pb = Pb;
  a.bc = bc;
  a.upr = (bc + TU - 1) / TU;
  a.nunits = br * a.upr;
  const int MT = (P + 15) / 16;
#ifdef STL_PROBES
  if (enc) {  // probe STL_RED_TC=1: the encode + g_d reduction on this kernel
    const int G = (P + 7) / 8;
#define STL_RED_ENC(TUV)                                                                          \
  switch (G) {                                                                                    \
    case 1: return launch_red_tc<true, TUV, 1, 1>(tz, to, a, red_out, s);                         \
    case 2: return launch_red_tc<true, TUV, 2, 1>(tz, to, a, red_out, s);                         \
    case 3: return launch_red_tc<true, TUV, 3, 2>(tz, to, a, red_out, s);                         \
    default: return launch_red_tc<true, TUV, 4, 2>(tz, to, a, red_out, s);                        \
  }
    if (TU == 256) { STL_RED_ENC(256) }
    STL_RED_ENC(512)
#undef STL_RED_ENC
  }
  if (TU == 256)  // probe STL_RED_TC_T=256
    return Pb <= 16 ? launch_red_tc<false, 256, 1, 1>(tz, to, a, red_out, s)
                    : launch_red_tc<false, 256, 2, 2>(tz, to, a, red_out, s);
#else
  if (enc || TU != 512) return cudaErrorNotSupported;
#endif
  const int KS = Pb <= 16 ? 1 : 2;
  return KS == 1 ? launch_red_tc<false, 512, 1, 1>(tz, to, a, red_out, s)
                 : (MT == 1 ? launch_red_tc<false, 512, 2, 1>(tz, to, a, red_out, s)
                            : launch_red_tc<false, 512, 2, 2>(tz, to, a, red_out, s));
}

// The fused-chain remix on tcgen05 (k_remix_tc): P <= 32 bf16 planes -> P bf16 planes,
// out[p] = sum_q (e_x d^T)[p][q] in[q]; cudaErrorNotSupported -> the mma.sync streaming remix.
cudaError_t planes_to_planes_tc(const void* in, int P, int64_t br, int64_t bc, const float* e_x,
                                const float* d, void* out, cudaStream_t s) {
  static const int on = probe_env("STL_REMIX_TC", 1);
  if (!on || P < 1 || P > 32 || bc < kT || bc % 64 || (reinterpret_cast<uintptr_t>(in) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  const int Pb = P <= 16 ? 16 : (P + 7) / 8 * 8;
  CUtensorMap ti{}, to{};
  if (!plane_box_tmap(&ti, in, 2, P, Pb, br, bc, kT, br)) return cudaErrorNotSupported;
  if (!plane_box_tmap(&to, out, 2, P, P, br, bc, kT, br)) return cudaErrorNotSupported;
  TcEncArgs a{};
  a.P = P;
  a.bc = bc;
  a.upr = (bc + kT - 1) / kT;
  a.nunits = br * a.upr;
  const int KS = Pb <= 16 ? 1 : 2;
  switch ((P + 7) / 8) {
    case 1: return launch_remix_tc<1, 1>(ti, to, a, e_x, d, s);
    case 2: return launch_remix_tc<1, 2>(ti, to, a, e_x, d, s);
    case 3: return launch_remix_tc<2, 3>(ti, to, a, e_x, d, s);
    default: return KS == 1 ? cudaErrorNotSupported : launch_remix_tc<2, 4>(ti, to, a, e_x, d, s);
  }
}

// t = 2 decode on tcgen05 (k_decode2_tc): P <= 32 bf16 planes -> bf16 matrix, tile columns
// >= 512 and % 64; cudaErrorNotSupported -> the register-streaming t = 2 decode.
cudaError_t planes_to_tiles2_tc(const void* in, int P, int64_t br, int64_t bc, const float* coef,
                                void* out, int64_t ldo, cudaStream_t s) {
  static const int on = probe_env("STL_T2_TC", 1);
  if (!on || P < 1 || P > 32 || bc < kT || bc % 64 || ldo % 8 ||
      (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return cudaErrorNotSupported;
  const int Pb = P <= 16 ? 16 : (P + 7) / 8 * 8;
  CUtensorMap tm{};
  if (!plane_box_tmap(&tm, in, 2, P, Pb, br, bc, kT, br)) return cudaErrorNotSupported;
  TcArgs a{};
  a.out = static_cast<__nv_bfloat16*>(out);
  a.ldo = ldo;
  a.coef = coef;
  a.P = P;
  a.Pb = Pb;
  a.bc = bc;
  a.upr = (bc + kT - 1) / kT;
  a.nunits = br * a.upr;
  a.br = static_cast<uint32_t>(br);
  a.R = 1;
  return Pb <= 16 ? launch_dec2_tc<1>(tm, a, s) : launch_dec2_tc<2>(tm, a, s);
}

}  // namespace stl
