// stl_stream.cu — HBM-streaming t = 4 tile transforms (the production bf16 path).
//
// The four per-layer tile transforms of the STL step, each one pass over HBM:
//   kEnc    : planes[p][I][J] = sum_c E[p][c] tile(I, J)[c]          encode_tiles (snf_operator.py:80-85)
//   kEncRed : kEnc, plus  R[p][c] += sum_tiles Z[p][tile] tile[c]     g_enc and g_d of _layer_backward
//                                                                     (toy_network.py:100-101)
//   kDec    : tile(I, J)[c] = sum_p Z[p][I][J] D[p][c]                decode_tiles (snf_operator.py:88-96)
//   kDecRed : kDec, plus  R[p][c] += sum_tiles Z[p][tile] X[tile][c]  g_x and g_ex (toy_network.py:104-105)
//   kRemix  : out[p][I][J] = sum_q C[p][q] Z[q][I][J], C = e_x d^T       the fused-chain step's
//             composite (snf_operator.py:175-188, Algorithm 2): planes in, planes out
// Tiles follow the reference layout contract (dense_core.py:98-108): element c = 4a + b of
// tile (I, J) is m[4I + a, 4J + b].
//
// B200 structure: one persistent CTA per SM = 1 producer warp + 8 consumer warps. A unit is a
// row segment of up to 256 tiles (tile row I, tiles J0 .. J0+255): its 4 matrix rows are 4
// contiguous 2 KB runs and each of its plane segments is one contiguous run, so the producer
// moves a unit with cp.async.bulk (1-D bulk copies, completion on an mbarrier) into a
// multi-stage shared-memory ring with padded rows (bank-conflict-free fragment loads). The
// consumers run the per-tile change of basis on the tensor cores (mma.sync m16n8k16, bf16 in,
// fp32 accumulate; fp32 operands split into bf16 hi + lo so products keep ~16 mantissa bits),
// stage the output unit in shared memory and one thread writes it back with bulk stores.
// Loads, math and stores of different units overlap; every byte is read and written once.
// Reductions accumulate in MMA fragments per warp, are summed over warps in a fixed order and
// over CTAs by a fixed-order tree (deterministic).
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include "sm100_ptx.cuh"
#include "stl_internal.h"

namespace stl {
namespace {

enum Mode { kEnc = 0, kEncRed = 1, kDec = 2, kDecRed = 3, kRemix = 4 };

// CW = consumer warps per CTA (template; 16). A measured negative result: an 8-warp, 56 KB
// "lite" configuration meant to share each SM with a slice-GEMM CTA (overlapping the g_x/g_ex
// decode with the g_w GEMM on two streams) ran 137 us alone and the pair 215 us vs 165 us
// sequential, so the backward stays sequential.
// Consumer groups taking alternate units: two 8-warp groups (two units' math in flight hides
// latency; with bf16 slice products the fused reductions gain from it too: 1-2%).
constexpr int kMaxStages = 16;
constexpr uint32_t kRowPad = 64;            // matrix rows: 16-word bank shift per row

template <int MODE> constexpr bool has_rows() { return MODE != kDec && MODE != kRemix; }
template <int MODE> constexpr bool has_planes_in() { return MODE != kEnc; }
template <int MODE> constexpr bool is_enc() { return MODE == kEnc || MODE == kEncRed; }
template <int MODE> constexpr bool has_red() { return MODE == kEncRed || MODE == kDecRed; }
// the unit's output is a plane box (TMA store) rather than 4 matrix rows
template <int MODE> constexpr bool out_planes() { return is_enc<MODE>() || MODE == kRemix; }
template <int MODE, int CW> constexpr int groups_of() { return CW < 16 ? 1 : 2; }

// Plane element types: float, __nv_bfloat16, or F24 (kF24 of stl_internal.h: a 16-bit high
// plane set + an 8-bit low plane set, moved as two boxes).
struct F24 {};
template <typename ZT> constexpr bool is_f24() { return std::is_same<ZT, F24>::value; }
template <typename ZT> constexpr int zhi() { return is_f24<ZT>() ? 2 : static_cast<int>(sizeof(ZT)); }

struct Layout {
  uint32_t pl_bytes;     // plane box of a stage (TMA, 128B-swizzled, 1024-aligned)
  uint32_t pl_lo;        // F24: offset of the 8-bit low box inside the plane region
  uint32_t row_stride, rows_bytes;  // padded matrix rows of a stage
  uint32_t stage_bytes;
  uint32_t out_stride, out_bytes;   // one output staging buffer
  uint32_t nbuf;                    // output staging buffers per consumer group (2..4)
  uint32_t red_bytes;
  uint32_t nstages;
  uint32_t total;                   // dynamic smem incl. barriers and alignment slack
};

__host__ __device__ inline uint32_t rup(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }


// bf16 plane segments moved as one 1-D bulk copy per plane into / out of plain shared-memory
// rows padded by 16 bytes (bank-conflict-free fragment accesses, see the offsets below) instead
// of one 4-D TMA box with 128-byte box rows. Measured per mode (profiles/r02_bulk_planes_ab.log):
// the fused-chain remix's output 105 -> 96 us at 8192^2; but the encode's output 58 -> 72 us,
// the decode's input 55 -> 85 us and the backward's fused reductions ~2x slower — so only the
// remix output uses it (the others keep the TMA boxes; STL_BULK_IN / STL_BULK_OUT: probes).
template <int MODE> inline bool bulk_planes_out() {
  static const bool on = probe_env("STL_BULK_OUT", MODE == kRemix ? 1 : 0) != 0;
  return on;
}
template <int MODE> inline bool bulk_planes_in() {
  static const bool on = probe_env("STL_BULK_IN", 0) != 0;
  return on;
}
template <int kT> constexpr uint32_t bulk_plane_stride() { return kT * 2 + 16; }
template <int MODE, typename ZT> constexpr bool bulk_in_capable() {
  return has_planes_in<MODE>() && std::is_same<ZT, __nv_bfloat16>::value;
}

template <int MODE, typename ZT, int kT, int CW>
inline Layout make_layout(int P, int Pb, uint32_t budget) {
  // Pb >= P: planes of the input box (the TMA zero-fills planes P..Pb-1, so the consumers'
  // plane loops need no bounds checks)
  Layout L{};
  L.pl_lo = is_f24<ZT>() ? rup(Pb * kT * 2, 1024) : 0;
  L.pl_bytes = has_planes_in<MODE>() ? rup(Pb * kT * zhi<ZT>(), 1024) + (is_f24<ZT>() ? rup(Pb * kT, 1024) : 0) : 0;
  if (bulk_in_capable<MODE, ZT>() && bulk_planes_in<MODE>())
    L.pl_bytes = rup(Pb * bulk_plane_stride<kT>(), 1024);
  L.row_stride = kT * 4 * 2 + kRowPad;
  L.rows_bytes = has_rows<MODE>() ? 4 * L.row_stride : 0;
  L.stage_bytes = rup(L.pl_bytes + L.rows_bytes, 1024);
  if (out_planes<MODE>()) {
    L.out_stride = 0;  // swizzled plane box
    L.out_bytes = rup((MODE == kRemix ? Pb : P) * kT * 2, 1024);
    if (bulk_planes_out<MODE>())  // plain planes, 16-byte padded (1-D bulk stores)
      L.out_bytes = rup(Pb * bulk_plane_stride<kT>(), 1024);
  } else {
    L.out_stride = kT * 4 * 2 + kRowPad;
    L.out_bytes = rup(4 * L.out_stride, 1024);
  }
  L.red_bytes = 0;  // the final per-warp reduction partials reuse the (drained) stage ring
  static const uint32_t max_st = probe_env("STL_STREAM_STAGES", 8);
  // Output staging buffers per consumer group: 3 for the plain encode / decode when that still
  // leaves two input stages per group (the store of unit i-1 may still be draining while unit i
  // is staged: 8192^3 encode 63 -> 58 us, decode 60 -> 56 us), else 2. The fused reductions
  // keep 2 (a third buffer costs them input stages: decode_gu+g_ex 49 -> 65 us).
  static const int nbuf_env = probe_env("STL_STREAM_NBUF", 0);
  L.nbuf = 2;
  if (nbuf_env >= 2 && nbuf_env <= 4) {
    L.nbuf = nbuf_env;
  } else if (!has_red<MODE>()) {
    const uint32_t f3 = 3 * groups_of<MODE, CW>() * L.out_bytes;
    if (budget > f3 && (budget - f3) / L.stage_bytes >= 2u * groups_of<MODE, CW>()) L.nbuf = 3;
  }
  const uint32_t fixed = L.nbuf * groups_of<MODE, CW>() * L.out_bytes + L.red_bytes;
  uint32_t ns = (budget - fixed) / L.stage_bytes;
  if (ns > max_st) ns = max_st;
  L.nstages = ns > kMaxStages ? kMaxStages : (ns < 2 ? 2 : ns);
  L.total = L.nstages * L.stage_bytes + fixed + 2 * kMaxStages * 8 + kMaxStages * 4 + 1024;  // + barriers, stage tags, align
  return L;
}

struct StreamArgs {
  const __nv_bfloat16* mat;  // ENC*: input matrix; DEC_RED: reduction matrix X
  int64_t ldm;
  void* out;                 // DEC*: output matrix (ENC* planes go out through tm_out)
  int64_t ldo;
  const float* coef;         // P x 16 (encoder rows for ENC*, decoder rows for DEC*; REMIX: e_x)
  const float* coef2;        // REMIX: d (P x 16); the composite C = e_x d^T is formed in-kernel
  float* red_partial;        // [gridDim.x][P * 16]
  int P;
  int Pb;                    // planes in the (zero-padded) input plane box
  int64_t br, bc;
  int64_t upr;               // units per tile row (1 when R > 1)
  int R;                     // tile rows per unit: kT / bc for narrow matrices (bc | kT), else 1
  int64_t nunits;
  int64_t prow;              // tile rows between planes (>= br: a row band of taller planes)
  int stg;                   // 1: consumers write outputs with st.global (else TMA/bulk stores)
  int nocompute;             // probe: skip the math (pure data movement)
  int contig;                // probe (with nocompute): each unit's planes as ONE contiguous
                             // block (a unit-blocked plane layout), one bulk copy
  int hilo;                  // REMIX: coefficients as bf16 hi + lo (1) or hi only (0)

  int bulk_in;               // bf16 input planes: 1-D bulk copies into plain padded rows
  const uint8_t* planes_in;  // the input planes (bulk path)
  Trace trace;               // probe: launch span
  int bulk_out;              // plane outputs: plain padded staging rows, 1-D bulk stores
  unsigned long long* dbg;   // probe: per-CTA phase timers [grid][4] (ns), or null
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(ptx::smem_u32(bar))
      : "memory");
}
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
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, uint32_t src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// The stage tags are a flag protocol (one writer, spinning readers) done with shared-memory
// atomics — formally race-free, and racecheck-clean — by one lane per warp (the warp then
// reconverges), so a unit costs each consumer warp one atomic when the tag is already set.
__device__ __forceinline__ void tag_store(volatile uint32_t* p, uint32_t v) {
  atomicExch(const_cast<uint32_t*>(p), v);
}
__device__ __forceinline__ void tag_wait(volatile uint32_t* p, uint32_t v, int lane) {
  if (lane == 0)
    while (atomicAdd(const_cast<uint32_t*>(p), 0u) != v) {
    }
  __syncwarp();
}
template <int NT>
__device__ __forceinline__ void cbar() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}
// barrier of one consumer group of NT threads (ids 2, 3)
template <int NT>
__device__ __forceinline__ void gbar(int grp) {
  asm volatile("bar.sync %0, %1;" ::"r"(2 + grp), "n"(NT) : "memory");
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// fp32 pair -> bf16 hi pair + bf16 lo pair (x = hi + lo to ~2^-16 relative)
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  const float2 hf = __bfloat1622float2(h);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = pack2(x0 - hf.x, x1 - hf.y);
}
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                    uint32_t a3, uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// m16n8k8 bf16 (half a k16 step): a0 = (row g, k 2q..2q+1), a1 = row g+8; b0 = (k 2q..2q+1, col g)
__device__ __forceinline__ void mma_k8(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(b0));
}
// fp32 -> tf32 operand, rounded to nearest (ties away) by adding half an ulp of the 10-bit
// mantissa; the tensor core ignores the low 13 bits. (Finite inputs.)
__device__ __forceinline__ uint32_t tf32_rna(float x) { return __float_as_uint(x) + 0x1000u; }
// D += A . B, m16n8k8, tf32 operands (fp32 registers), fp32 accumulate.
//   A: a0 = (row g, k q), a1 = (g+8, q), a2 = (g, q+4), a3 = (g+8, q+4); B: b0 = (k q, col g),
//   b1 = (q+4, g); C as m16n8k16.
__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// F24 pair: high halves of two elements (one 32-bit word) + their low bytes (one 16-bit word)
// (lo2 is zero-extended from 16 bits, so its byte 2 supplies the zero low byte: one PRMT each)
__device__ __forceinline__ float2 f24x2(uint32_t hi2, uint32_t lo2) {
  return make_float2(__uint_as_float(__byte_perm(lo2, hi2, 0x5402)),
                     __uint_as_float(__byte_perm(lo2, hi2, 0x7612)));
}
// two bf16 from (lo16 of a, lo16 of b) -> packed pair
__device__ __forceinline__ uint32_t pair16(uint32_t a, uint32_t b) { return a | (b << 16); }

// A unit's planes in shared memory as the TMA box {W, P, T/W} lands them with 128-byte swizzle:
// 128-byte rows indexed (chunk * P + p), chunk = t / W, W = 128 / sizeof(Z) tiles per row; the
// 16-byte chunk index inside a row is XORed with (row & 7).
template <int ZSZ>
__device__ __forceinline__ uint32_t pl_addr(uint32_t base, int P, int p, int t) {
  constexpr int W = 128 / ZSZ;
  const uint32_t row = static_cast<uint32_t>((t / W) * P + p);
  const uint32_t byte = static_cast<uint32_t>((t % W) * ZSZ);
  return base + row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15));
}

// Swizzled plane-box offset of (plane p, tile t). Adding (16 ks + 8 h) planes to p adds
// (16 ks + 8 h) * 128 bytes and leaves the XOR term unchanged, so per-thread offsets are computed
// once for p < 8 and the plane-group steps become immediates.
template <int ZSZ>
__device__ __forceinline__ uint32_t pl_off(int P, int p, int t) {
  return pl_addr<ZSZ>(0u, P, p, t);
}

// Work split of a kT-tile unit over the C = kGWarps warps of the consumer group that owns it:
//   ENC n-tiles (8 tiles):  warp w -> n-tiles w + C k, k < kT / (8 C)
//   DEC m-tiles (16 tiles): warp w -> m-tiles w + C k, k < kT / (16 C)
//   RED k-steps (16 tiles): warp w -> k-steps w + C k, k < kT / (16 C)

// ------------------------------------------------------------------ the kernel
// MT = number of 16-plane groups (ceil(P / 16)), a template so every plane loop unrolls.
// NTR (kRemix only): output n-tiles = ceil(P / 8); the output staging holds Pb = 8 NTR planes
// per chunk (the TMA store clips planes >= P), so every fragment store is unconditional.
template <int MODE, typename ZT, int MT, int kT, int CW, int NTR = 0>
__global__ void __launch_bounds__(32 * CW + 32, 1)
    k_stream(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_in2,
             const __grid_constant__ CUtensorMap tm_out,
             StreamArgs args, Layout L) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-aligned base kept as shared-array arithmetic so plain C++ loads compile to LDS and the
  // compiler may schedule them; offsets below are relative to `smem`, `sbase` is its address.
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = ptx::smem_u32(smem);
  auto lds32 = [smem](uint32_t o) { return *reinterpret_cast<const uint32_t*>(smem + o); };
  auto lds16 = [smem](uint32_t o) -> uint32_t { return *reinterpret_cast<const uint16_t*>(smem + o); };
  auto lds64f = [smem](uint32_t o) { return *reinterpret_cast<const float2*>(smem + o); };
  auto sts32 = [smem](uint32_t o, uint32_t v) { *reinterpret_cast<uint32_t*>(smem + o) = v; };
  const uint32_t s_stages = 0;
  const uint32_t s_out = s_stages + L.nstages * L.stage_bytes;
  float* s_red = reinterpret_cast<float*>(smem);  // after the unit loop only
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.nstages * L.stage_bytes +
                                               L.nbuf * groups_of<MODE, CW>() * L.out_bytes + L.red_bytes);
  constexpr int kCWarps = CW;
  constexpr int kCThreads = 32 * CW;
  constexpr int kGroups = groups_of<MODE, CW>();
  constexpr int kGWarps = kCWarps / kGroups;  // warps per group
  constexpr int kGThreads = 32 * kGWarps;
  uint64_t* empty = full + kMaxStages;
  // stage tags: the unit a stage is being filled with, written by the producer once it owns the
  // stage. With two consumer groups and an odd stage count a stage alternates between the
  // groups, so a fast group can reach a stage's next use while the other group's fill of it is
  // still in flight; the full barrier's parity alone would alias that to an older, completed
  // phase. Consumers first wait for the tag, then for the barrier phase.
  volatile uint32_t* stage_tag = reinterpret_cast<volatile uint32_t*>(empty + kMaxStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
#ifdef STL_PROBES
  const bool hilo = args.hilo != 0;  // probe: bf16 hi coefficients only
#else
  constexpr bool hilo = true;  // the product build never drops the lo coefficient halves
#endif
  const int P = args.P, Pb = args.Pb;
  constexpr int ZSZ = zhi<ZT>();         // bytes of the (high) plane element
  constexpr bool kZ24 = is_f24<ZT>();
  const uint32_t nunits = static_cast<uint32_t>(args.nunits);
  const uint32_t upr = static_cast<uint32_t>(args.upr);
  const int urows = args.R;  // tile rows per unit
  const uint32_t br = static_cast<uint32_t>(args.br);
  const uint32_t bc = static_cast<uint32_t>(args.bc);

  if (threadIdx.x == 0) {
    trace_mark(args.trace, false);
    trace_cta(args.trace, 0);
    for (uint32_t s = 0; s < L.nstages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], kGWarps);
      tag_store(stage_tag + s, 0xFFFFFFFFu);
    }
    ptx::fence_mbar_init();
  }
  griddep_launch_dependents();
  // e_x / d (remix) and every input may be the previous launch's output (PDL)
  if constexpr (MODE == kRemix) griddep_wait();
  if constexpr (MODE == kRemix) {
    // the fused-step composite C = e_x d^T (P x P, fp32) into the (not yet used) output staging;
    // the consumers read their B fragments from it (a named barrier after the fragment setup
    // keeps the staging untouched until every consumer has them)
    float* sC = reinterpret_cast<float*>(smem + s_out);
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
      const int pp = i / P, qq = i - (i / P) * P;
      float v = 0.f;
  #pragma unroll
      for (int kk = 0; kk < 16; ++kk) v = fmaf(args.coef[pp * 16 + kk], args.coef2[qq * 16 + kk], v);
      sC[i] = v;
    }
  }
  if (warp == kCWarps && lane == 0) {
    if constexpr (has_planes_in<MODE>()) ptx::prefetch_tmap(&tm_in);
    if constexpr (kZ24) ptx::prefetch_tmap(&tm_in2);
    if constexpr (out_planes<MODE>()) ptx::prefetch_tmap(&tm_out);
  }
  __syncthreads();
  if constexpr (MODE != kRemix) griddep_wait();  // inputs of this launch are complete (PDL)
  if (threadIdx.x == 0) trace_cta(args.trace, 1);

  if (warp == kCWarps) {
    // ---------------------------------------------------------------- producer
    // lane 0: the plane box (one 4-D TMA op); lanes 0..3: matrix row a (1-D bulk copy into a
    // padded row).
    uint32_t it = 0;
    for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
      const uint32_t stage = it % L.nstages;
      const uint32_t phase = (it / L.nstages) & 1;
      // a unit: tiles J0 .. J0 + kT - 1 of tile row I, or (R > 1) all bc tiles of the R tile
      // rows I .. I + urows - 1 — the same smem layout (tile t of the unit at the same offsets)
      const uint32_t I = urows > 1 ? u * urows : u / upr;
      const uint32_t J0 = urows > 1 ? 0u : (u - I * upr) * kT;
      const uint32_t nrows = urows > 1 ? min(static_cast<uint32_t>(urows), br - I) : 1u;
      const uint32_t Tw = urows > 1 ? nrows * bc : min(bc - J0, static_cast<uint32_t>(kT));
      ptx::mbar_wait(&empty[stage], phase ^ 1);
      if (lane == 0) tag_store(stage_tag + stage, it);  // before the expect_tx arrive (release) below
      const uint32_t rows_b = has_rows<MODE>() ? Tw * 8 : 0;
      const uint32_t st = s_stages + stage * L.stage_bytes;
      const bool bin = bulk_in_capable<MODE, ZT>() && args.bulk_in;
      if (lane == 0) {
        ptx::mbar_arrive_expect_tx(&full[stage],
                                   4 * rows_b + (!has_planes_in<MODE>() ? 0u
                                                 : bin ? P * Tw * 2
                                                       : Pb * kT * (ZSZ + (kZ24 ? 1 : 0))));
        if constexpr (has_planes_in<MODE>())
          if (!bin)
            tma_load_4d(&tm_in, &full[stage], sbase + st, 0, 0, static_cast<int>(J0 / (128 / ZSZ)),
                        static_cast<int>(I));
        if constexpr (kZ24)
          tma_load_4d(&tm_in2, &full[stage], sbase + st + L.pl_lo, 0, 0, static_cast<int>(J0 / 128),
                      static_cast<int>(I));
      }
      if constexpr (bulk_in_capable<MODE, ZT>()) {
        if (bin) {
          // one bulk copy per plane: the unit's Tw tiles (contiguous also for R > 1)
          __syncwarp();  // the expect_tx above precedes the copies' complete_tx
          if (args.contig) {
            if (lane == 0)
              bulk_g2s(sbase + st, args.planes_in + 2 * static_cast<int64_t>(u) * P * kT, P * Tw * 2,
                       &full[stage]);
          } else {
            for (int p = lane; p < P; p += 32)
              bulk_g2s(sbase + st + p * bulk_plane_stride<kT>(),
                       args.planes_in + 2 * ((static_cast<int64_t>(p) * args.prow + I) * bc + J0),
                       Tw * 2, &full[stage]);
          }
        }
      }
      if constexpr (has_rows<MODE>()) {
        if (urows > 1) {
          // lane = 4 r + a: matrix row a of the unit's tile row r, appended after row r - 1's
          const uint32_t r = lane >> 2, a = lane & 3;
          if (r < nrows)
            bulk_g2s(sbase + st + L.pl_bytes + a * L.row_stride + r * bc * 8,
                     args.mat + (4 * static_cast<int64_t>(I + r) + a) * args.ldm, bc * 8,
                     &full[stage]);
        } else if (lane < 4) {
          bulk_g2s(sbase + st + L.pl_bytes + lane * L.row_stride,
                   args.mat + (4 * static_cast<int64_t>(I) + lane) * args.ldm + 4 * J0, rows_b,
                   &full[stage]);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int ctid = threadIdx.x;
  constexpr uint32_t RS = kT * 4 * 2 + kRowPad;  // == L.row_stride (compile-time: folds into offsets)
  constexpr int kNK = kT / (8 * kGWarps);    // ENC n-tile rounds per warp
  constexpr int kMK = kT / (16 * kGWarps);   // DEC m-tile / RED k-step rounds per warp
  const int grp = warp / kGWarps, wl = warp % kGWarps;  // group, warp within the group
  const int gtid = wl * 32 + lane;
  static_assert(kNK >= 1 && kMK >= 1, "unit too small for the warp count");
  // Coefficient fragments, split hi + lo.
  //  ENC (A = E, M = p, K = c): a0 = E[16m+g][2q, 2q+1], a1 = E[16m+g+8][..], a2/a3: c + 8.
  //  DEC (B = D, K = p, N = c): b0 = (D[16ks+2q][c], D[16ks+2q+1][c]), b1: planes + 8.
  //  REMIX: the same with B = C^T (coef = C^T, row stride P; N = output plane, kNT n-tiles).
  constexpr int kNT = MODE == kRemix ? NTR : 2;     // DEC n-tiles (16 tile values / P planes)
  static_assert(MODE != kRemix || (NTR >= 1 && NTR <= 2 * MT), "remix n-tiles");
  const int CS = MODE == kRemix ? P : 16;            // coefficient row stride
  const int NC = MODE == kRemix ? P : 16;            // valid output columns (zero past them)
  // B coefficient (k = input plane / tile value pa, n = output column c): DEC: D[pa][c];
  // REMIX: C^T[pa][c] = C[c][pa], C = e_x d^T formed at kernel start (no separate launch
  // between the previous slice GEMM and this one)
  auto bcoef = [&](int pa, int c) -> float {
    if constexpr (MODE == kRemix) {
      return reinterpret_cast<const float*>(smem + s_out)[c * P + pa];
    } else {
      return args.coef[pa * CS + c];
    }
  };
  uint32_t fh[MT][is_enc<MODE>() ? 4 : 2 * kNT], fl[MT][is_enc<MODE>() ? 4 : 2 * kNT];
  if constexpr (is_enc<MODE>()) {
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int p = 16 * m + g + 8 * (i & 1), c = 2 * q + 8 * (i >> 1);
        const float e0 = p < P ? args.coef[p * 16 + c] : 0.f;
        const float e1 = p < P ? args.coef[p * 16 + c + 1] : 0.f;
        split2(e0, e1, fh[m][i], fl[m][i]);
      }
  } else {
#pragma unroll
    for (int ks = 0; ks < MT; ++ks)
#pragma unroll
      for (int i = 0; i < 2 * kNT; ++i) {  // i = nt * 2 + h
        const int nt = i >> 1, h = i & 1, c = 8 * nt + g;
        const int pa = 16 * ks + 2 * q + 8 * h, pb = pa + 1;
        const float d0 = pa < P && c < NC ? bcoef(pa, c) : 0.f;
        const float d1 = pb < P && c < NC ? bcoef(pb, c) : 0.f;
        split2(d0, d1, fh[ks][i], fl[ks][i]);
      }
  }
  // Per-thread shared-memory offsets (see the work split above).
  // ENC: B loads at rows + xoff + 512k (+2 RS); C stores at buf + soff[k] + (16m + 8h) * 128.
  const uint32_t xoff = (q >> 1) * RS + 64 * wl + 8 * g + 4 * (q & 1);
  uint32_t soff[kNK];
  // plane steps of the input / output plane regions: 128-byte swizzled box rows, or plain rows
  // of bulk_plane_stride bytes (16-byte pad: word offset 4 per plane -> the fragment accesses
  // below hit 32 distinct banks)
  const bool bin = bulk_in_capable<MODE, ZT>() && args.bulk_in, bout = args.bulk_out != 0;
  constexpr uint32_t PS = bulk_plane_stride<kT>();
  const uint32_t PSi = bin ? PS : 128u, PSo = bout ? PS : 128u;
#pragma unroll
  for (int k = 0; k < kNK; ++k)
    soff[k] = !is_enc<MODE>() ? 0u
              : bout ? g * PS + (8 * (wl + kGWarps * k) + 2 * q) * 2
                     : pl_off<2>(P, g, 8 * (wl + kGWarps * k) + 2 * q);
  // Stores/loads of planes >= P exist only in the last 16-plane group.
  const bool lastp0 = 16 * (MT - 1) + g < P, lastp1 = 16 * (MT - 1) + g + 8 < P;
  const bool okb1 = 16 * (MT - 1) + g + 8 < Pb;  // row inside the (8-padded) input box
  // RED: B loads at rows + rb[nt] + 1024k; A loads at planes + ra0/ra2[k] + (16mt + 8h) * 128.
  uint32_t rb[2], ra0[kMK], ra2[kMK], ra0l[kMK], ra2l[kMK];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int c = 8 * nt + g;
    rb[nt] = (c >> 2) * RS + 128 * wl + 16 * q + 2 * (c & 3);
  }
#pragma unroll
  for (int k = 0; k < kMK; ++k) {
    const int t = 16 * (wl + kGWarps * k) + 2 * q;
    ra0[k] = !has_red<MODE>() ? 0u : bin ? g * PS + t * 2 : pl_off<ZSZ>(Pb, g, t);
    ra2[k] = !has_red<MODE>() ? 0u : bin ? g * PS + (t + 8) * 2 : pl_off<ZSZ>(Pb, g, t + 8);
    ra0l[k] = kZ24 ? L.pl_lo + pl_off<1>(Pb, g, t) : 0u;   // F24 low bytes: same rule, W = 128
    ra2l[k] = kZ24 ? L.pl_lo + pl_off<1>(Pb, g, t + 8) : 0u;
  }
  // DEC: A loads at planes + da[k][j] + (16ks + 8h) * 128 (planes 2q + j + 16ks + 8h at tiles
  // t0, t0 + 1, t0 = 16 (warp + 8k) + 2g); C stores at buf + ooff + 1024k + 2nt RS (+8).
  uint32_t da[kMK][2], dal[kMK][2];
#pragma unroll
  for (int k = 0; k < kMK; ++k)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      da[k][j] = is_enc<MODE>() ? 0u
                 : bin ? (2 * q + j) * PS + (16 * (wl + kGWarps * k) + 2 * g) * 2
                       : pl_off<ZSZ>(Pb, 2 * q + j, 16 * (wl + kGWarps * k) + 2 * g);
      dal[k][j] = kZ24 ? L.pl_lo + pl_off<1>(Pb, 2 * q + j, 16 * (wl + kGWarps * k) + 2 * g) : 0u;
    }
  const uint32_t ooff = (q >> 1) * RS + 128 * wl + 16 * g + 4 * (q & 1);
  bool dok[4];  // last plane group: planes 16(MT-1) + 2q + {0, 1, 8, 9} < P
#pragma unroll
  for (int j = 0; j < 4; ++j) dok[j] = 16 * (MT - 1) + 2 * q + (j & 1) + 8 * (j >> 1) < P;

  // fp32 / F24 planes use single-pass TF32 MMAs (operands rounded to nearest tf32, ~2^-12):
  // DEC B = D with k = q <-> plane 8s + 2q, k = q + 4 <-> plane 8s + 2q + 1 (the planes a
  // thread loads, see below): bt[s][nt][0] = D[8s+2q][8nt+g], bt[s][nt][1] = D[8s+2q+1][8nt+g].
  constexpr bool kTf32 = ZSZ == 4 || kZ24;
  // bf16-plane decode and remix on single-pass TF32 m16n8k8 MMAs over exactly the Pb planes (no
  // PRMT regrouping; coefficients rounded to tf32, 2^-11): 8192^3 decode 62.5 -> 59.1 us, the
  // remix -5 us (profiles/r02_dec_tf32_ab.log). Compile-time per mode: the g_x decode-reduction
  // keeps bf16 hi + lo (no gain there, and both fragment sets live at once spilled registers).
  constexpr bool kTf32Dec = (MODE == kDec || MODE == kRemix) && ZSZ == 2 && !kZ24;
  constexpr int KS8 = 2 * MT;
  uint32_t bt[KS8][kNT][2];
#pragma unroll
  for (int s8 = 0; s8 < KS8; ++s8)
#pragma unroll
    for (int nt = 0; nt < kNT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int pl = 8 * s8 + 2 * q + h, c = 8 * nt + g;
        bt[s8][nt][h] = (!is_enc<MODE>() && (kTf32 || kTf32Dec) && pl < P && c < NC)
                            ? tf32_rna(bcoef(pl, c)) : 0u;
      }
  // REMIX: C stores at buf + ro[k][h] + 1024 nt (output plane 8nt + 2q + h, tiles t0, t0 + 1)
  uint32_t ro[kMK][2];
#pragma unroll
  for (int k = 0; k < kMK; ++k)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      ro[k][h] = MODE != kRemix ? 0u
                 : bout ? (2 * q + h) * PS + (16 * (wl + kGWarps * k) + 2 * g) * 2
                        : pl_off<2>(Pb, 2 * q + h, 16 * (wl + kGWarps * k) + 2 * g);
  const uint32_t ro_nt = 8 * PSo;

  float R[2][2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int k = 0; k < 4; ++k) R[a][b][k] = 0.f;

  if constexpr (MODE == kRemix) cbar<kCThreads>();  // composite fragments read: staging free
  uint64_t dbg_c0 = 0, dbg_t0 = 0;
  if (args.dbg && ctid == 0) {
    dbg_c0 = clock64();
    dbg_t0 = ptx::globaltimer_ns();
  }
  // group grp takes this CTA's units it = grp, grp + 2, ... (stage it % nstages)
  for (uint32_t u = blockIdx.x + grp * gridDim.x, it = grp; u < nunits;
       u += kGroups * gridDim.x, it += kGroups) {
    const uint32_t stage = it % L.nstages;
    const uint32_t phase = (it / L.nstages) & 1;
    const uint32_t I = urows > 1 ? u * urows : u / upr;
    const uint32_t J0 = urows > 1 ? 0u : (u - I * upr) * kT;
    const uint32_t nrows = urows > 1 ? min(static_cast<uint32_t>(urows), br - I) : 1u;
    const int Tw = static_cast<int>(urows > 1 ? nrows * bc : min(bc - J0, static_cast<uint32_t>(kT)));
    const uint32_t buf = s_out + (grp * L.nbuf + (it / kGroups) % L.nbuf) * L.out_bytes;
    const uint32_t planes = s_stages + stage * L.stage_bytes;
    const uint32_t rows = planes + L.pl_bytes;
    const uint64_t t_w0 = args.dbg ? ptx::globaltimer_ns() : 0;
    tag_wait(stage_tag + stage, it, lane);
    ptx::mbar_wait(&full[stage], phase);
    if (it == 0 && ctid == 0) trace_cta(args.trace, 2);
    const uint64_t t_w1 = args.dbg ? ptx::globaltimer_ns() : 0;

    // The unit's math. Full units (Tw == kT) take a copy with compile-time bounds so the
    // compiler can interleave the warp's independent m-tiles / k-steps.
    auto unit_math = [&](auto full_tag) {
      constexpr bool kFull = decltype(full_tag)::value;
      if constexpr (is_enc<MODE>()) {
        // C^T[p][tile] = E . X^T per 8-tile n-tile. B: b0 = X[tile][c 2q, 2q+1] (row q>>1),
        // b1 = row 2 + (q>>1). Banks: 16 (q>>1) + 2g + (q&1) -> conflict-free. C: plane 16m+g
        // (c0, c1) / 16m+g+8 (c2, c3), tiles 8nt+2q, +1, into the swizzled plane box: the 8 planes
        // g land in 8 different 16-byte chunks -> conflict-free.
        const int nnt = kFull ? kT / 8 : (Tw >> 3);
  #pragma unroll
        for (int k = 0; k < kNK; ++k) {
          if (kFull || wl + kGWarps * k < nnt) {
            const uint32_t xb = rows + xoff + 64 * kGWarps * k;
            const uint32_t b0 = lds32(xb), b1 = lds32(xb + 2 * RS);
  #pragma unroll
            for (int m = 0; m < MT; ++m) {
              float c[4] = {0.f, 0.f, 0.f, 0.f};
              mma(c, fh[m][0], fh[m][1], fh[m][2], fh[m][3], b0, b1);
              if (hilo) mma(c, fl[m][0], fl[m][1], fl[m][2], fl[m][3], b0, b1);
              const uint32_t o = buf + soff[k] + 16 * m * PSo;
              if (m < MT - 1 || lastp0) sts32(o, pack2(c[0], c[1]));
              if (m < MT - 1 || lastp1) sts32(o + 8 * PSo, pack2(c[2], c[3]));
            }
          }
        }
      } else {
        // C[tile][c] = Z^T . D per 16-tile m-tile; rows g / g+8 <-> tiles 2g / 2g+1 so each
        // plane load is one 8-byte (fp32) or 4-byte (bf16) access; with the swizzle XOR a
        // half-warp's loads hit 32 distinct banks.
        const int nmt = kFull ? kT / 16 : (Tw >> 4);
  #pragma unroll
        for (int k = 0; k < kMK; ++k) {
          if (kFull || wl + kGWarps * k < nmt) {
            float acc[kNT][4];
  #pragma unroll
            for (int nt = 0; nt < kNT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
            if constexpr (kTf32) {
              // m16n8k8 tf32 per 8 planes: rows g / g+8 = tiles t0 / t0+1, k = q / q+4 = planes
              // 8s+2q / 8s+2q+1: a0 a1 = Z[8s+2q][t0, t0+1] (one 8-byte or F24 load), a2 a3 =
              // Z[8s+2q+1][t0, t0+1].
  #pragma unroll
              for (int s8 = 0; s8 < KS8; ++s8) {
                if (8 * s8 >= Pb) break;  // warp-uniform; planes P..Pb-1 are zero in the box
                float2 v[2];
  #pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const uint32_t ad = planes + da[k][h] + 8 * s8 * 128;
                  if constexpr (kZ24) v[h] = f24x2(lds32(ad), lds16(planes + dal[k][h] + 8 * s8 * 128));
                  else v[h] = lds64f(ad);
                }
                const uint32_t a0 = tf32_rna(v[0].x), a1 = tf32_rna(v[0].y);
                const uint32_t a2 = tf32_rna(v[1].x), a3 = tf32_rna(v[1].y);
  #pragma unroll
                for (int nt = 0; nt < kNT; ++nt)
                  mma_tf32(acc[nt], a0, a1, a2, a3, bt[s8][nt][0], bt[s8][nt][1]);
              }
            } else {
            if constexpr (kTf32Dec) {
              {
                // bf16 planes through m16n8k8 TF32 (as the fp32-plane path): one 4-byte load
                // holds plane 8s + 2q (+1) at tiles t0, t0 + 1; bf16 -> tf32 is exact (<< 16)
  #pragma unroll
                for (int s8 = 0; s8 < KS8; ++s8) {
                  if (8 * s8 >= Pb) break;  // warp-uniform; planes P..Pb-1 are zero in the box
                  const uint32_t w0 = lds32(planes + da[k][0] + 8 * s8 * PSi);
                  const uint32_t w1 = lds32(planes + da[k][1] + 8 * s8 * PSi);
                  const uint32_t a0 = w0 << 16, a1 = w0 & 0xFFFF0000u;
                  const uint32_t a2 = w1 << 16, a3 = w1 & 0xFFFF0000u;
  #pragma unroll
                  for (int nt = 0; nt < kNT; ++nt)
                    mma_tf32(acc[nt], a0, a1, a2, a3, bt[s8][nt][0], bt[s8][nt][1]);
                }
              }
            } else {
  #pragma unroll
            for (int ks = 0; ks < MT; ++ks) {
              if constexpr (ZSZ == 2 && !kZ24) {
                // bf16 planes: each 4-byte load holds one plane at tiles (t0, t0 + 1); the A
                // fragments pair two planes at one tile, so regroup the halves with PRMT
                uint32_t w[4];
  #pragma unroll
                for (int j = 0; j < 4; ++j)
                  w[j] = (ks < MT - 1 || dok[j])
                             ? lds32(planes + da[k][j & 1] + (16 * ks + 8 * (j >> 1)) * PSi)
                             : 0u;
                const uint32_t a0 = __byte_perm(w[0], w[1], 0x5410), a1 = __byte_perm(w[0], w[1], 0x7632);
                const uint32_t a2 = __byte_perm(w[2], w[3], 0x5410), a3 = __byte_perm(w[2], w[3], 0x7632);
                if (MODE == kRemix && ks == MT - 1 && P <= 16 * (MT - 1) + 8) {
                  // REMIX: the last plane group holds <= 8 planes: a k8 step (the mma.sync pipe
                  // bounds the remix: r = 24 needs 1.5 k16-steps, not 2)
  #pragma unroll
                  for (int nt = 0; nt < kNT; ++nt) {
                    mma_k8(acc[nt], a0, a1, fh[ks][2 * nt]);
                    if (hilo) mma_k8(acc[nt], a0, a1, fl[ks][2 * nt]);
                  }
                  continue;
                }
  #pragma unroll
                for (int nt = 0; nt < kNT; ++nt) {
                  mma(acc[nt], a0, a1, a2, a3, fh[ks][2 * nt], fh[ks][2 * nt + 1]);
                  if (hilo)
                    mma(acc[nt], a0, a1, a2, a3, fl[ks][2 * nt], fl[ks][2 * nt + 1]);
                }
                continue;
              }
              float v[4][2];  // planes 16ks + 2q + {0, 1, 8, 9} at tiles t0, t0 + 1
  #pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint32_t ad = planes + da[k][j & 1] + (16 * ks + 8 * (j >> 1)) * 128;
                if (ks < MT - 1 || dok[j]) {
                  if constexpr (kZ24) {
                    const float2 f = f24x2(lds32(ad), lds16(planes + dal[k][j & 1] + (16 * ks + 8 * (j >> 1)) * 128));
                    v[j][0] = f.x;
                    v[j][1] = f.y;
                  } else if constexpr (ZSZ == 4) {
                    const float2 f = lds64f(ad);
                    v[j][0] = f.x;
                    v[j][1] = f.y;
                  } else {
                    const uint32_t w = lds32(ad);
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w));
                    v[j][0] = f.x;
                    v[j][1] = f.y;
                  }
                } else {
                  v[j][0] = v[j][1] = 0.f;
                }
              }
              // a0 = (row g = tile t0: planes 2q, 2q+1), a1 = row g+8 = tile t0+1, a2/a3: +8
              if constexpr (ZSZ == 4 || kZ24) {
                uint32_t h0, l0, h1, l1, h2, l2, h3, l3;
                split2(v[0][0], v[1][0], h0, l0);
                split2(v[0][1], v[1][1], h1, l1);
                split2(v[2][0], v[3][0], h2, l2);
                split2(v[2][1], v[3][1], h3, l3);
  #pragma unroll
                for (int nt = 0; nt < kNT; ++nt) {
                  const uint32_t bh0 = fh[ks][2 * nt], bh1 = fh[ks][2 * nt + 1];
                  mma(acc[nt], h0, h1, h2, h3, bh0, bh1);
                  mma(acc[nt], l0, l1, l2, l3, bh0, bh1);
                  mma(acc[nt], h0, h1, h2, h3, fl[ks][2 * nt], fl[ks][2 * nt + 1]);
                }
              } else {
                const uint32_t a0 = pack2(v[0][0], v[1][0]), a1 = pack2(v[0][1], v[1][1]);
                const uint32_t a2 = pack2(v[2][0], v[3][0]), a3 = pack2(v[2][1], v[3][1]);
  #pragma unroll
                for (int nt = 0; nt < kNT; ++nt) {
                  mma(acc[nt], a0, a1, a2, a3, fh[ks][2 * nt], fh[ks][2 * nt + 1]);
                  mma(acc[nt], a0, a1, a2, a3, fl[ks][2 * nt], fl[ks][2 * nt + 1]);
                }
              }
            }
            }  // !kTf32Dec
            }  // bf16 planes
            if constexpr (MODE == kRemix) {
              // acc[nt][0] / [2] -> output plane 8nt + 2q at tiles t0 / t0 + 1, [1] / [3] -> plane
              // 8nt + 2q + 1: one 4-byte store per plane into the swizzled plane box
  #pragma unroll
              for (int nt = 0; nt < kNT; ++nt) {
                sts32(buf + ro[k][0] + ro_nt * nt, pack2(acc[nt][0], acc[nt][2]));
                sts32(buf + ro[k][1] + ro_nt * nt, pack2(acc[nt][1], acc[nt][3]));
              }
            } else {
            // acc[nt][0,1] -> tile t0, c = 8nt + 2q (+1): row a = 2nt + (q>>1), col b = 2(q&1).
  #pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const uint32_t o = buf + ooff + 128 * kGWarps * k + 2 * nt * RS;
              sts32(o, pack2(acc[nt][0], acc[nt][1]));
              sts32(o + 8, pack2(acc[nt][2], acc[nt][3]));
            }
            }
          }
        }
      }
      if constexpr (has_red<MODE>()) {
        // R[p][c] += sum over 16-tile k-steps of Z[p][tile] X[tile][c] (A = Z: M = p; B = X: N = c).
        // B: b0 = (X[t0+2q][c], X[t0+2q+1][c]), b1 = tiles + 8, c = 8nt + g, 16-bit loads
        // (words 16 (c>>2) + 4q + ((c&3)>>1): distinct). A: Z[p][t0+2q, +1] / [t0+2q+8, +9].
        const int nks = kFull ? kT / 16 : (Tw >> 4);
  #pragma unroll
        for (int k = 0; k < kMK; ++k) {
          if (kFull || wl + kGWarps * k < nks) {
            uint32_t b[2][2], bx[2][2][2];
  #pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const uint32_t base = rows + rb[nt] + 128 * kGWarps * k;
              const uint32_t x0 = lds16(base), x1 = lds16(base + 8), x8 = lds16(base + 64),
                             x9 = lds16(base + 72);
              b[nt][0] = pair16(x0, x1);
              b[nt][1] = pair16(x8, x9);
              bx[nt][0][0] = x0 << 16;
              bx[nt][0][1] = x1 << 16;
              bx[nt][1][0] = x8 << 16;
              bx[nt][1][1] = x9 << 16;
            }
  #pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const bool ok0 = mt < MT - 1 || lastp0, ok1 = mt < MT - 1 || lastp1;
              const uint32_t z0 = planes + ra0[k] + 16 * mt * PSi, z2 = planes + ra2[k] + 16 * mt * PSi;
              if constexpr (kTf32) {
                // two m16n8k8 tf32 steps (tiles t0..t0+7, t0+8..t0+15): rows g / g+8 = planes,
                // k = q / q+4 = tiles 2q / 2q+1 of the step; B = X as fp32 (bf16 << 16, exact).
  #pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                  const uint32_t za = hh ? z2 : z0;
                  // planes 16mt+g (< Pb) and 16mt+g+8 (may pass Pb in the last group: load a
                  // valid row, select zero)
                  const bool in1 = mt < MT - 1 || okb1;
                  const uint32_t d1 = in1 ? 1024u : 0u;
                  float2 v0, v1;
                  if constexpr (kZ24) {
                    const uint32_t la = planes + (hh ? ra2l[k] : ra0l[k]) + 16 * mt * 128;
                    v0 = f24x2(lds32(za), lds16(la));
                    v1 = f24x2(lds32(za + d1), lds16(la + d1));
                  } else {
                    v0 = lds64f(za);
                    v1 = lds64f(za + d1);
                  }
                  if (!in1) v1 = make_float2(0.f, 0.f);
                  const uint32_t a0 = tf32_rna(v0.x), a1 = tf32_rna(v1.x);
                  const uint32_t a2 = tf32_rna(v0.y), a3 = tf32_rna(v1.y);
  #pragma unroll
                  for (int nt = 0; nt < 2; ++nt)
                    mma_tf32(R[mt][nt], a0, a1, a2, a3, bx[nt][hh][0], bx[nt][hh][1]);
                }
              } else if constexpr (ZSZ == 2 && !kZ24) {
                const uint32_t a0 = ok0 ? lds32(z0) : 0u, a2 = ok0 ? lds32(z2) : 0u;
                const uint32_t a1 = ok1 ? lds32(z0 + 8 * PSi) : 0u, a3 = ok1 ? lds32(z2 + 8 * PSi) : 0u;
  #pragma unroll
                for (int nt = 0; nt < 2; ++nt) mma(R[mt][nt], a0, a1, a2, a3, b[nt][0], b[nt][1]);
              } else {
                const float2 zero = make_float2(0.f, 0.f);
                float2 v0, v1, v2, v3;
                if constexpr (kZ24) {
                  const uint32_t l0 = planes + ra0l[k] + 16 * mt * 128, l2 = planes + ra2l[k] + 16 * mt * 128;
                  v0 = ok0 ? f24x2(lds32(z0), lds16(l0)) : zero;
                  v2 = ok0 ? f24x2(lds32(z2), lds16(l2)) : zero;
                  v1 = ok1 ? f24x2(lds32(z0 + 1024), lds16(l0 + 1024)) : zero;
                  v3 = ok1 ? f24x2(lds32(z2 + 1024), lds16(l2 + 1024)) : zero;
                } else {
                  v0 = ok0 ? lds64f(z0) : zero;
                  v2 = ok0 ? lds64f(z2) : zero;
                  v1 = ok1 ? lds64f(z0 + 1024) : zero;
                  v3 = ok1 ? lds64f(z2 + 1024) : zero;
                }
                uint32_t h0, l0, h1, l1, h2, l2, h3, l3;
                split2(v0.x, v0.y, h0, l0);
                split2(v1.x, v1.y, h1, l1);
                split2(v2.x, v2.y, h2, l2);
                split2(v3.x, v3.y, h3, l3);
  #pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                  mma(R[mt][nt], h0, h1, h2, h3, b[nt][0], b[nt][1]);
                  mma(R[mt][nt], l0, l1, l2, l3, b[nt][0], b[nt][1]);
                }
              }
            }
          }
        }
      }
    };
    if (args.nocompute) {
    } else if (Tw == kT) {
      unit_math(std::true_type{});
    } else {
      unit_math(std::false_type{});
    }

    __syncwarp();
    if (args.dbg && ctid == 0) {
      const uint64_t t_c = ptx::globaltimer_ns();
      args.dbg[4 * blockIdx.x + 0] += t_w1 - t_w0;  // waiting for data
      args.dbg[4 * blockIdx.x + 1] += t_c - t_w1;   // math (warp 0's share)
    }
    if (lane == 0) ptx::mbar_arrive(&empty[stage]);
    if (args.stg) {
      // Consumers copy the staged unit to global memory with 16-byte stores (coalesced rows).
      gbar<kGThreads>(grp);
      if constexpr (out_planes<MODE>()) {
        __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(args.out) + static_cast<int64_t>(I) * bc + J0;
        const int64_t ntiles = args.br * args.bc;
        const int pieces = P * (Tw >> 3);  // 16-byte pieces: (p, chunk k, c16)
        for (int i = gtid; i < pieces; i += kGThreads) {
          const int p = i / (Tw >> 3), rest = i - p * (Tw >> 3), k = rest >> 3, c16 = rest & 7;
          const uint32_t row = static_cast<uint32_t>(k * P + p);
          const uint4 v = *reinterpret_cast<const uint4*>(smem + buf + row * 128 + ((c16 ^ (row & 7)) << 4));
          *reinterpret_cast<uint4*>(ob + p * ntiles + 64 * k + 8 * c16) = v;
        }
      } else {
        __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(args.out) + (4 * static_cast<int64_t>(I)) * args.ldo + 4 * J0;
        const int per_row = Tw >> 1;  // 16-byte pieces per output row
        for (int i = gtid; i < 4 * per_row; i += kGThreads) {
          const int a = i / per_row, c = i - a * per_row;
          const uint4 v = *reinterpret_cast<const uint4*>(smem + buf + a * L.out_stride + 16 * c);
          *reinterpret_cast<uint4*>(ob + a * args.ldo + 8 * c) = v;
        }
      }
      continue;
    }
    ptx::fence_proxy_async_smem();
    // The stores of the previous unit (other buffer) must have finished reading it before the
    // barrier: the next unit writes that buffer. One barrier per unit.
    // With nbuf buffers the one written next was last stored nbuf - 1 units ago: allow the
    // nbuf - 2 younger stores to stay in flight.
    if (wl == 0) {
      if (L.nbuf == 2) ptx::bulk_wait_read<0>();
      else if (L.nbuf == 3) ptx::bulk_wait_read<1>();
      else ptx::bulk_wait_read<2>();
    }
    gbar<kGThreads>(grp);
    // the group's warp 0 issues the unit's stores: the plane box (one 4-D TMA op, clipped at
    // the matrix edge) or the 4 output rows (1-D bulk copies).
    if (wl == 0) {
      if constexpr (out_planes<MODE>()) {
        if (bout) {
          // one bulk store per plane: the unit's Tw tiles of tile row I (contiguous also for
          // R > 1: whole tile rows)
          if (args.contig) {
            if (lane == 0)
              bulk_s2g(static_cast<__nv_bfloat16*>(args.out) + static_cast<int64_t>(u) * P * kT,
                       sbase + buf, static_cast<uint32_t>(P * Tw * 2));
          } else {
            for (int p = lane; p < P; p += 32)
              bulk_s2g(static_cast<__nv_bfloat16*>(args.out) +
                           (static_cast<int64_t>(p) * args.prow + I) * bc + J0,
                       sbase + buf + p * PS, static_cast<uint32_t>(Tw) * 2);
          }
        } else if (lane == 0) {
          tma_store_4d(&tm_out, sbase + buf, 0, 0, static_cast<int>(J0 / 64), static_cast<int>(I));
        }
      } else {
        __nv_bfloat16* o =
            static_cast<__nv_bfloat16*>(args.out) + (4 * static_cast<int64_t>(I)) * args.ldo + 4 * J0;
        if (urows > 1) {
          const uint32_t r = lane >> 2, a = lane & 3;
          if (r < nrows)
            bulk_s2g(o + (4 * r + a) * args.ldo, sbase + buf + a * L.out_stride + r * bc * 8, bc * 8);
        } else if (lane < 4) {
          bulk_s2g(o + lane * args.ldo, sbase + buf + lane * L.out_stride, Tw * 8);
        }
      }
      ptx::bulk_commit();
    }
  }
  if (wl == 0) ptx::bulk_wait_all();
  if (wl == 0 && lane == 0) trace_mark(args.trace, true);
  if (ctid == 0) trace_cta(args.trace, 3);
  if (args.dbg && ctid == 0) {  // probe: SM clock over the unit loop (cycles / ns)
    args.dbg[4 * blockIdx.x + 2] = clock64() - dbg_c0;
    args.dbg[4 * blockIdx.x + 3] = ptx::globaltimer_ns() - dbg_t0;
  }

  if constexpr (has_red<MODE>()) {
    // per-warp fragments -> smem (the stage ring, once every warp is done with it) ->
    // fixed-order sum over warps -> this CTA's partial
    cbar<kCThreads>();
    float* mine = s_red + warp * P * 16;
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
      }
    cbar<kCThreads>();
    const int n = P * 16;
    for (int o = ctid; o < n; o += kCThreads) {
      float s = s_red[o];
#pragma unroll
      for (int w = 1; w < kCWarps; ++w) s += s_red[w * n + o];
      args.red_partial[static_cast<int64_t>(blockIdx.x) * n + o] = s;
    }
  }
}

// 4-D plane map (W tiles, P planes, bc/W chunks, br rows) with box {W, P, kT/W, 1}, 128B swizzle.
bool plane_tmap(CUtensorMap* m, const void* base, int zsz, int P, int Pb, int64_t br, int64_t bc,
                int kT, int R, int64_t prow) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  if (!fn) return false;
  const uint64_t W = 128 / zsz;
  cuuint64_t dims[4] = {W, static_cast<cuuint64_t>(P), static_cast<cuuint64_t>(bc / W),
                        static_cast<cuuint64_t>(br)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(prow * bc * zsz), 128,
                           static_cast<cuuint64_t>(bc * zsz)};
  // one unit: kT / W chunks of one tile row, or (R > 1) all bc / W chunks of R tile rows
  cuuint32_t box[4] = {static_cast<cuuint32_t>(W), static_cast<cuuint32_t>(Pb),
                       static_cast<cuuint32_t>((R > 1 ? bc : kT) / W), static_cast<cuuint32_t>(R)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, zsz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                  : zsz == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8,
                  4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    static bool warned = false;
    if (!warned) fprintf(stderr, "[stl_b200] plane tensor map rejected (CUresult %d); using the "
                                 "register transforms\n", static_cast<int>(r));
    warned = true;
  }
  return r == CUDA_SUCCESS;
}

template <int MODE, typename ZT, int MT, int kT, int CW, int NTR = 0>
cudaError_t launch_mt(StreamArgs a, const void* planes_in, void* planes_out, float* red_out,
                      cudaStream_t s, uint32_t budget) {
  a.Pb = ((a.P + 7) / 8) * 8;
  const Layout L = make_layout<MODE, ZT, kT, CW>(a.P, a.Pb, budget);
  static const int stg = probe_env("STL_STREAM_STG", 0);
  static const int multirow = probe_env("STL_STREAM_MULTIROW", 1);
  // narrow matrices (bc < kT, bc | kT): a unit spans R = kT / bc whole tile rows (R <= 8: one
  // producer lane per matrix row), so units stay full instead of bc / kT full
  const int R = (multirow && !stg && a.bc < kT && kT % a.bc == 0 && kT / a.bc <= 8 &&
                 (!is_f24<ZT>() || a.bc % 128 == 0))
                    ? static_cast<int>(kT / a.bc)
                    : 1;
  a.R = R;
  CUtensorMap tin{}, tin2{}, tout{};
  if (a.prow < a.br) a.prow = a.br;
  if (a.prow != a.br && (stg || R > 1)) return cudaErrorNotSupported;  // band: TMA, 1-row units
  if (has_planes_in<MODE>() &&
      !plane_tmap(&tin, planes_in, zhi<ZT>(), a.P, a.Pb, a.br, a.bc, kT, R, a.prow))
    return cudaErrorNotSupported;
  if (is_f24<ZT>() &&
      !plane_tmap(&tin2, static_cast<const uint8_t*>(planes_in) + 2 * a.P * a.prow * a.bc, 1, a.P,
                  a.Pb, a.br, a.bc, kT, R, a.prow))
    return cudaErrorNotSupported;
  if (out_planes<MODE>() &&
      !plane_tmap(&tout, planes_out, 2, a.P, MODE == kRemix ? a.Pb : a.P, a.br, a.bc, kT, R, a.prow))
    return cudaErrorNotSupported;
  auto k = k_stream<MODE, ZT, MT, kT, CW, NTR>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(L.total));
  if (e != cudaSuccess) return e;
  if (probe_env("STL_SMEM_MAX_CARVEOUT", 0))
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  a.stg = stg;
  // probe: 1 = every mode skips its math; a bit mask 2 / 4 / 8 / 16 selects the modes (<< MODE)
  static const int noc_env = probe_env("STL_STREAM_NOCOMPUTE", 0);
  const int noc = noc_env == 1 ? 1 : ((noc_env >> (MODE + 1)) & 1);
  a.nocompute = noc;
  static const int contig = probe_env("STL_PROBE_CONTIG", 0);
  a.contig = contig && noc;
  static const int hilo = probe_env("STL_HILO", 1);  // probe 0: bf16 hi coefficients only
  a.hilo = hilo;
  a.trace = trace_next();
  a.bulk_in = bulk_in_capable<MODE, ZT>() && bulk_planes_in<MODE>();
  a.planes_in = static_cast<const uint8_t*>(planes_in);
  a.bulk_out = out_planes<MODE>() && bulk_planes_out<MODE>() && !stg;
  static const int dbg_on = probe_env("STL_STREAM_DEBUG", 0);
  static unsigned long long* dbg = nullptr;
  if (dbg_on && !dbg) cudaMalloc(&dbg, 4 * 1024 * sizeof(unsigned long long));
  if (dbg_on) cudaMemsetAsync(dbg, 0, 4 * 1024 * sizeof(unsigned long long), s);
  a.dbg = dbg_on ? dbg : nullptr;
  a.upr = R > 1 ? 1 : (a.bc + kT - 1) / kT;  // kT: this launch's unit
  a.nunits = R > 1 ? (a.br + R - 1) / R : a.br * a.upr;
  int64_t grid = sm_count();
  if (grid > a.nunits) grid = a.nunits;
  if (grid < 1) return cudaSuccess;
  const uint64_t t0 = 0;
  (void)t0;
  e = launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(32 * CW + 32), L.total, s, tin, tin2,
                 tout, a, L);
  if (e != cudaSuccess) return e;
  if (a.dbg) {
    unsigned long long h[4 * 1024];
    cudaMemcpyAsync(h, a.dbg, sizeof(unsigned long long) * 4 * grid, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double w = 0, c = 0, cyc = 0, ns = 0;
    for (int i = 0; i < grid; ++i) { w += h[4 * i]; c += h[4 * i + 1]; cyc += h[4 * i + 2]; ns += h[4 * i + 3]; }
    fprintf(stderr, "[stream dbg] mode=%d T=%d units/cta=%.1f stages=%u  avg us: wait=%.1f math=%.1f "
            "loop=%.1f  sm_mhz=%.0f\n",
            MODE, kT, double(a.nunits) / grid, L.nstages, w / grid / 1e3, c / grid / 1e3,
            ns / grid / 1e3, ns > 0 ? 1e3 * cyc / ns : 0.0);
  }
  if constexpr (has_red<MODE>()) return sum_partials(a.red_partial, static_cast<int>(grid), a.P * 16, red_out, s);
  return cudaSuccess;
}

// 512-tile units whenever two pipeline stages per consumer group fit (measured: longer bulk
// segments beat deeper pipelines; the g_x / g_ex decode-reduction even with 3 stages: 47.7 vs
// 55.9 us at config 2, while the g_enc / g_d encode-reduction is faster with 256), else 256.
template <int MODE, typename ZT, int MT, int NTR = 0>
cudaError_t launch_t(StreamArgs a, const void* planes_in, void* planes_out, float* red_out,
                     cudaStream_t s) {
  static const int force_t = probe_env("STL_STREAM_T", 0);
  static const uint32_t budget = probe_env("STL_STREAM_SMEM_KB", 212) * 1024;
  const int pb = ((a.P + 7) / 8) * 8;
  const Layout L512 = make_layout<MODE, ZT, 512, 16>(a.P, pb, budget);
  const bool use512 = force_t ? force_t == 512
                              : (L512.nstages >= (MODE == kDecRed ? 3u : 2u * groups_of<MODE, 16>()) &&
                                 L512.total <= 227 * 1024 && a.bc >= 512);
#ifdef STL_PROBES
  // probe: an 8-consumer-warp CTA (288 threads) that fits beside a slice-GEMM CTA
  if constexpr (!has_red<MODE>() && MODE != kRemix && std::is_same<ZT, __nv_bfloat16>::value)
    if (probe_env("STL_STREAM_CW", 16) == 8)
      return launch_mt<MODE, ZT, MT, 256, 8>(a, planes_in, planes_out, red_out, s, budget);
#endif
  if (use512) return launch_mt<MODE, ZT, MT, 512, 16, NTR>(a, planes_in, planes_out, red_out, s, budget);
  return launch_mt<MODE, ZT, MT, 256, 16, NTR>(a, planes_in, planes_out, red_out, s, budget);
}

template <int MODE, typename ZT>
cudaError_t launch(StreamArgs a, const void* planes_in, void* planes_out, float* red_out,
                   cudaStream_t s) {
  if constexpr (MODE == kRemix) {
    switch ((a.P + 7) / 8) {  // n-tiles of the output planes
      case 1: return launch_t<MODE, ZT, 1, 1>(a, planes_in, planes_out, red_out, s);
      case 2: return launch_t<MODE, ZT, 1, 2>(a, planes_in, planes_out, red_out, s);
      case 3: return launch_t<MODE, ZT, 2, 3>(a, planes_in, planes_out, red_out, s);
      case 4: return launch_t<MODE, ZT, 2, 4>(a, planes_in, planes_out, red_out, s);
      default: return cudaErrorNotSupported;
    }
  } else {
  switch ((a.P + 15) / 16) {
    case 1: return launch_t<MODE, ZT, 1>(a, planes_in, planes_out, red_out, s);
    case 2: return launch_t<MODE, ZT, 2>(a, planes_in, planes_out, red_out, s);
    case 3: if constexpr (!has_red<MODE>() && MODE != kRemix) return launch_t<MODE, ZT, 3>(a, planes_in, planes_out, red_out, s);
            return cudaErrorNotSupported;
    case 4: if constexpr (!has_red<MODE>() && MODE != kRemix) return launch_t<MODE, ZT, 4>(a, planes_in, planes_out, red_out, s);
            return cudaErrorNotSupported;
    default: return cudaErrorNotSupported;
  }
  }
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// encode (+ g_d-style reduction): bf16 matrix -> bf16 planes; red planes bf16 or fp32.
cudaError_t tiles_to_planes_stream(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                                   const float* coef, int P, void* out, int odt, const void* rp,
                                   int rdt, float* ro, float* rw, cudaStream_t s,
                                   int64_t plane_rows) {
  if (mdt != kBF16 || odt != kBF16 || bc % 64 || ldm % 8 || P < 1 || P > 64 ||
      !al16(m) || !al16(out))
    return cudaErrorNotSupported;
  if (rp && (P > 32 || !al16(rp) || !ro || !rw || (rdt == kF24 && bc % 128)))
    return cudaErrorNotSupported;
  if (!rp) {  // the tensor-core (tcgen05) encode, when it takes the shape
    const cudaError_t e = tiles_to_planes_tc(m, ldm, br, bc, coef, P, out, s, plane_rows);
    if (e != cudaErrorNotSupported) return e;
  } else if (rdt == kBF16) {  // tcgen05 encode + mma.sync reduction
    const cudaError_t e =
        red_transform_tc(true, m, ldm, rp, P, br, bc, coef, out, 0, ro, rw, s, plane_rows);
    if (e != cudaErrorNotSupported) return e;
  }
  StreamArgs a{};
  a.mat = static_cast<const __nv_bfloat16*>(m);
  a.ldm = ldm;
  a.out = out;
  a.coef = coef;
  a.red_partial = rw;
  a.P = P;
  a.br = br;
  a.bc = bc;
  a.prow = plane_rows;
  if (!rp) return launch<kEnc, __nv_bfloat16>(a, nullptr, out, nullptr, s);
  if (rdt == kBF16) return launch<kEncRed, __nv_bfloat16>(a, rp, out, ro, s);
  if (rdt == kF24) return launch<kEncRed, F24>(a, rp, out, ro, s);
  return launch<kEncRed, float>(a, rp, out, ro, s);
}

bool plane_box_tmap(CUtensorMap* m, const void* base, int zsz, int P, int Pb, int64_t br,
                    int64_t bc, int kT, int64_t prow, int R) {
  return plane_tmap(m, base, zsz, P, Pb, br, bc, kT, R, prow);
}

// decode (+ g_ex-style reduction): fp32 or bf16 planes -> bf16 matrix; red matrix bf16.
cudaError_t planes_to_tiles_stream(const void* in, int idt, int Q, int64_t br, int64_t bc,
                                   const float* coef, void* out, int odt, int64_t ldo,
                                   const void* rm, int rdt, int64_t ldr, float* ro, float* rw,
                                   cudaStream_t s, int64_t plane_rows) {
  if (odt != kBF16 || bc % 64 || ldo % 8 || Q < 1 || Q > 64 || !al16(in) ||
      !al16(out))
    return cudaErrorNotSupported;
  if (rm && (rdt != kBF16 || Q > 32 || ldr % 8 || !al16(rm) || !ro || !rw))
    return cudaErrorNotSupported;
  if (idt == kF24 && bc % 128) return cudaErrorNotSupported;
  if (!rm && idt == kBF16) {  // the tensor-core (tcgen05) decode, when it takes the shape
    const cudaError_t e = planes_to_tiles_tc(in, Q, br, bc, coef, out, ldo, s, plane_rows);
    if (e != cudaErrorNotSupported) return e;
  } else if (rm && idt == kBF16) {  // tcgen05 decode + mma.sync reduction
    const cudaError_t e =
        red_transform_tc(false, rm, ldr, in, Q, br, bc, coef, out, ldo, ro, rw, s, plane_rows);
    if (e != cudaErrorNotSupported) return e;
  }
  StreamArgs a{};
  a.mat = static_cast<const __nv_bfloat16*>(rm);
  a.ldm = ldr;
  a.out = out;
  a.ldo = ldo;
  a.coef = coef;
  a.red_partial = rw;
  a.P = Q;
  a.br = br;
  a.bc = bc;
  a.prow = plane_rows;
  if (rm) {
    if (idt == kF32) return launch<kDecRed, float>(a, in, nullptr, ro, s);
    if (idt == kF24) return launch<kDecRed, F24>(a, in, nullptr, ro, s);
    return launch<kDecRed, __nv_bfloat16>(a, in, nullptr, ro, s);
  }
  if (idt == kF32) return launch<kDec, float>(a, in, nullptr, nullptr, s);
  if (idt == kF24) return launch<kDec, F24>(a, in, nullptr, nullptr, s);
  return launch<kDec, __nv_bfloat16>(a, in, nullptr, nullptr, s);
}

// the fused-chain remix: r bf16 or fp32 planes -> r bf16 planes, out[p] = sum_q C[p][q] in[q] with
// C = e_x d^T formed in-kernel (e_x, d: r x 16). r <= 32.
cudaError_t planes_to_planes_stream(const void* in, int idt, int P, int64_t br, int64_t bc,
                                    const float* e_x, const float* d, void* out, cudaStream_t s) {
  if ((idt != kBF16 && idt != kF32) || bc % 64 || P < 1 || P > 32 || !al16(in) || !al16(out))
    return cudaErrorNotSupported;
  if (idt == kBF16) {  // the tcgen05 remix, when it takes the shape
    const cudaError_t e = planes_to_planes_tc(in, P, br, bc, e_x, d, out, s);
    if (e != cudaErrorNotSupported) return e;
  }
  StreamArgs a{};
  a.out = out;
  a.coef = e_x;
  a.coef2 = d;
  a.P = P;
  a.br = br;
  a.bc = bc;
  a.prow = br;
  if (idt == kF32) return launch<kRemix, float>(a, in, out, nullptr, s);
  return launch<kRemix, __nv_bfloat16>(a, in, out, nullptr, s);
}

}  // namespace stl
