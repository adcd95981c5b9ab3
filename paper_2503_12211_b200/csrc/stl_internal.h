// stl_internal.h — shared declarations between the STL CUDA translation units.
#pragma once
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace stl {

// Programmatic dependent launch: the hot-path kernels (streaming transforms, CTA-pair GEMM,
// partial sums) are launched with cudaLaunchAttributeProgrammaticStreamSerialization and call
// griddep_wait() before touching global memory, so each one's CTAs can be scheduled and run
// their prologue (barrier init, TMEM alloc, descriptor prefetch) while the previous kernel
// drains. STL_PDL=0 disables the attribute.
bool pdl_enabled();
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Probe build only (-DSTL_PROBES, STL_TRACE=1): every hot-path launch takes a trace slot and its
// CTAs record [first entry, last exit] globaltimer spans there (scripts/trace_fwd.py reads them
// back with stl_trace_read): where a pipeline's time goes between and inside kernels.
struct Trace {
  unsigned long long* buf;  // 2 per slot, or null
  int slot;
  unsigned long long* cta;  // per-CTA event stamps [kTraceCtaSlots][gridDim][4], or null
};
constexpr int kTraceCtaSlots = 64;
#ifdef STL_PROBES
Trace trace_next();
__device__ __forceinline__ void trace_mark(const Trace& t, bool end) {
  if (!t.buf) return;
  unsigned long long now;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
  if (end) atomicMax(t.buf + 2 * t.slot + 1, now);
  else atomicMin(t.buf + 2 * t.slot, now);
}
// per-CTA stamp e (0 entry, 1 after griddep_wait, 2 first unit's data, 3 loop end)
__device__ __forceinline__ void trace_cta(const Trace& t, int e) {
  if (!t.cta || t.slot >= kTraceCtaSlots) return;
  unsigned long long now;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
  t.cta[(static_cast<size_t>(t.slot) * gridDim.x + blockIdx.x) * 4 + e] = now;
}
#else
inline Trace trace_next() { return Trace{nullptr, 0, nullptr}; }
__device__ __forceinline__ void trace_mark(const Trace&, bool) {}
__device__ __forceinline__ void trace_cta(const Trace&, int) {}
#endif

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// kF24: an fp32 quantity rounded to 24 bits (RNE) and stored as two plane sets — the high
// 16 bits of every element (2 bytes each) followed by the next 8 bits (1 byte each) — so a
// tensor of n elements occupies 3n bytes; value = as_float(hi << 16 | lo << 8), ~2^-16 relative.
// Used for the bf16 path's fp32 slice products (forward cache y_enc, backward g_u).
enum Dtype : int { kF32 = 0, kBF16 = 1, kF24 = 2 };

// Measurement probes (the STL_* environment switches used by scripts/ for A/B runs: stage
// counts, store-less mainloops, disabled tile shapes, ...) exist only in the probe build of the
// library (libstl_b200_probe.so, compiled with -DSTL_PROBES). The product library never reads
// the environment: probe_env returns the default there.
inline int probe_env(const char* name, int dflt) {
#ifdef STL_PROBES
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

inline size_t dtype_size(int dt) { return dt == kBF16 ? 2 : (dt == kF24 ? 3 : 4); }

// Operand layouts of one slice-GEMM batch C_p = A_p · B_p (p = 0..r-1), all slices contiguous.
//   A: 0 = (r, M, K) K-contiguous ("K-major"),  1 = (r, K, M) M-contiguous ("MN-major")
//   B: 0 = (r, N, K) K-contiguous ("K-major"),  1 = (r, K, N) N-contiguous ("MN-major")
//   C: (r, M, N) N-contiguous, fp32 or bf16.
struct SliceGemmProblem {
  const void* a;
  int a_layout;
  const void* b;
  int b_layout;
  void* c;
  int c_dtype;
  int ab_dtype;
  int r;
  int64_t M, N, K;
  void* c2 = nullptr;  // optional bf16 copy of C (tcgen05 path only)
  // Rows between consecutive slices of A (K-major) and C; 0 = M. A row band of taller planes:
  // a, c point at the band's first row, M = band rows, m_stride = rows of the whole planes.
  int64_t m_stride = 0;
};

int sm_count();

// 3-D bf16 tensor map over `slices` contiguous (outer x inner) matrices, 128B swizzle.
// slice_bytes: bytes between slices (0 = inner * outer * 2).
bool make_bf16_tmap(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t slices, uint32_t box_inner, uint32_t box_outer,
                    uint64_t slice_bytes = 0);

cudaError_t cast_f32_to_bf16(const float* in, void* out, int64_t n, cudaStream_t s);


// tcgen05 path (bf16 operands, aligned shapes). Returns cudaError_t-like code, 0 = ok.
cudaError_t slice_gemm_tc(const SliceGemmProblem& pb, cudaStream_t s);
bool slice_gemm_tc_supported(const SliceGemmProblem& pb);
// Two problems with the same r in one persistent CTA-pair launch (problem 0's tiles first);
// cudaErrorNotSupported when the pair (kinds, alignment) is not covered -> launch separately.
bool slice_gemm_tc_group_supported(const SliceGemmProblem& p0, const SliceGemmProblem& p1);
cudaError_t slice_gemm_tc_group(const SliceGemmProblem& p0, const SliceGemmProblem& p1,
                                cudaStream_t s);
// F24 output (c_dtype = kF24) is produced by the CTA-pair kernel only.
bool slice_gemm_f24_supported(const SliceGemmProblem& pb);
// out[p] = sum_s partial[p * S + s] over (r * S) fp32 slices of mn elements (split-K).
cudaError_t slice_gemm_sum_splits(const float* partial, int r, int S, int64_t mn, float* out,
                                  cudaStream_t s);
// SIMT path (fp32 or bf16 operands, any shape).
cudaError_t slice_gemm_simt(const SliceGemmProblem& pb, cudaStream_t s);

// Tile <-> plane transforms (see stl_transform.cu).
// red_planes (optional) are P planes (br, bc) of red_dtype.
cudaError_t tiles_to_planes(const void* m, int m_dtype, int64_t ldm, int64_t br, int64_t bc,
                            int t, const float* coef, int P, void* out, int out_dtype,
                            const void* red_planes, int red_dtype, float* red_out,
                            float* red_ws, cudaStream_t s);
cudaError_t planes_to_tiles(const void* in, int in_dtype, int Q, int64_t br, int64_t bc, int t,
                            const float* coef, void* out, int out_dtype, int64_t ldo,
                            const void* red_m, int red_dtype, int64_t ldr, float* red_out,
                            float* red_ws, cudaStream_t s);
cudaError_t planes_to_planes(const void* in, int in_dtype, int Q, int64_t ntiles,
                             const float* coef, int P, void* out, int out_dtype, cudaStream_t s);
// t = 4 vectorised fast paths (stl_transform4.cu); cudaErrorNotSupported -> use generic.
cudaError_t tiles_to_planes4(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                             const float* coef, int P, void* out, int odt, const void* rp,
                             int rdt, float* ro, float* rw, cudaStream_t s);
cudaError_t planes_to_tiles4(const void* in, int idt, int Q, int64_t br, int64_t bc,
                             const float* coef, void* out, int odt, int64_t ldo, const void* rm,
                             int rdt, int64_t ldr, float* ro, float* rw, cudaStream_t s);
// Tensor-core (mma.sync) t = 4 encode (stl_transform_mma.cu): the fallback for shapes the
// streaming encode declines (tile columns not a multiple of 64, e.g. T2T-ViT's 144).
cudaError_t tiles_to_planes_mma(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                                const float* coef, int P, void* out, int odt, const void* rp,
                                int rdt, float* ro, float* rw, cudaStream_t s);
// HBM-streaming bulk-async t = 4 transforms (stl_stream.cu), tried first for t = 4;
// cudaErrorNotSupported -> the kernels above. The only readers of F24 planes.
// plane_rows: tile rows of the whole planes when (m / out, in / out) address a row band of
// them (0 = br).
cudaError_t tiles_to_planes_stream(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                                   const float* coef, int P, void* out, int odt, const void* rp,
                                   int rdt, float* ro, float* rw, cudaStream_t s,
                                   int64_t plane_rows = 0);
cudaError_t planes_to_tiles_stream(const void* in, int idt, int Q, int64_t br, int64_t bc,
                                   const float* coef, void* out, int odt, int64_t ldo,
                                   const void* rm, int rdt, int64_t ldr, float* ro, float* rw,
                                   cudaStream_t s, int64_t plane_rows = 0);
// Register-streaming t = 2 transforms (stl_transform2.cu), tried first for t = 2 without a
// fused reduction: bf16 matrix, bf16 (encode) / bf16 or fp32 (decode) planes, bc % 4 == 0.
cudaError_t tiles_to_planes2(const void* m, int mdt, int64_t ldm, int64_t br, int64_t bc,
                             const float* coef, int P, void* out, int odt, cudaStream_t s);
cudaError_t planes_to_tiles2(const void* in, int idt, int Q, int64_t br, int64_t bc,
                             const float* coef, void* out, int odt, int64_t ldo, cudaStream_t s);
// 4-D plane-box tensor map of the streaming transforms (stl_stream.cu): box {128 / zsz tiles,
// Pb planes, kT * zsz / 128 chunks, 1 tile row}, 128-byte swizzle; prow >= br tile rows per plane.
// R > 1 (narrow matrices, R * bc = kT): a box of R whole tile rows {W, Pb, bc / W, R}.
bool plane_box_tmap(CUtensorMap* m, const void* base, int zsz, int P, int Pb, int64_t br,
                    int64_t bc, int kT, int64_t prow, int R = 1);
// t = 4 decode on tcgen05 (stl_stream_tc.cu): P <= 32 bf16 planes -> bf16 matrix;
// cudaErrorNotSupported -> the mma.sync streaming decode.
cudaError_t planes_to_tiles_tc(const void* in, int P, int64_t br, int64_t bc, const float* coef,
                               void* out, int64_t ldo, cudaStream_t s, int64_t plane_rows);
// t = 4 encode on tcgen05 (stl_stream_tc.cu): bf16 matrix -> P <= 32 bf16 planes;
// cudaErrorNotSupported -> the mma.sync streaming encode.
cudaError_t tiles_to_planes_tc(const void* m, int64_t ldm, int64_t br, int64_t bc,
                               const float* coef, int P, void* out, cudaStream_t s,
                               int64_t plane_rows);
// The backward's fused transforms on tcgen05 + mma.sync (stl_stream_tc.cu): enc: planes = encode
// (rows), R = Z . rows (tiles_to_planes_stream with bf16 reduction planes); dec: rows = decode(Z),
// R = Z . rows (planes_to_tiles_stream with a bf16 reduction matrix). cudaErrorNotSupported ->
// the mma.sync streaming kernels.
cudaError_t red_transform_tc(bool enc, const void* rows, int64_t ldr, const void* z, int P,
                             int64_t br, int64_t bc, const float* coef, void* out, int64_t ldo,
                             float* red_out, float* red_ws, cudaStream_t s, int64_t plane_rows);
// The fused-chain remix on tcgen05 (stl_stream_tc.cu): P <= 32 bf16 planes -> bf16 planes;
// cudaErrorNotSupported -> the mma.sync streaming remix.
cudaError_t planes_to_planes_tc(const void* in, int P, int64_t br, int64_t bc, const float* e_x,
                                const float* d, void* out, cudaStream_t s);
// t = 2 decode on tcgen05 (stl_stream_tc.cu): P <= 32 bf16 planes -> bf16 matrix, tile columns
// >= 512; cudaErrorNotSupported -> the register-streaming t = 2 decode (stl_transform2.cu).
cudaError_t planes_to_tiles2_tc(const void* in, int P, int64_t br, int64_t bc, const float* coef,
                                void* out, int64_t ldo, cudaStream_t s);
// Fused-chain remix (stl_stream.cu kRemix): P <= 32 bf16 / fp32 planes -> bf16 planes,
// out[p] = sum_q C[p][q] in[q], C = e_x d^T formed in-kernel; tile columns % 64 == 0.
cudaError_t planes_to_planes_stream(const void* in, int idt, int P, int64_t br, int64_t bc,
                                    const float* e_x, const float* d, void* out, cudaStream_t s);
// out[o] = sum_b partial[b * n + o], deterministic fixed-order tree.
cudaError_t sum_partials(const float* partial, int nblocks, int n, float* out, cudaStream_t s);
cudaError_t compose_coefs(const float* a, const float* b, int r, int tt, float* out,
                          cudaStream_t s);

// Token-row plumbing for T % t == 1 activations (stl_tokens.cu): pad to Tp = T - 1 + t rows
// (bf16, zero rows/columns), its backward, the learnable fold of the last t rows (+ bias) and
// its backward (d bias, d fold as N + t fixed-order sums). C, Cp, N multiples of 8.
constexpr int kFoldMaxT = 8;
cudaError_t token_pad(const void* x, int dtype_in, int64_t B, int64_t T, int64_t C, void* out,
                      int64_t Tp, int64_t Cp, cudaStream_t s);
cudaError_t token_unpad(const void* g, int64_t B, int64_t Tp, int64_t Cp, void* out,
                        int dtype_out, int64_t T, int64_t C, cudaStream_t s);
cudaError_t token_fold(const void* y, int64_t B, int64_t Tp, int64_t N, int t, const float* fold,
                       const float* bias, void* out, int64_t T, cudaStream_t s);
int64_t token_fold_ws_floats(int64_t B, int64_t T, int64_t N, int t);
cudaError_t token_fold_backward(const void* gout, const void* y, int64_t B, int64_t Tp,
                                int64_t N, int t, const float* fold, int64_t T, void* g_y,
                                float* g_bias_fold, float* ws, cudaStream_t s);

constexpr int kMaxRank = 64;          // upper bound on r handled by the transform kernels
constexpr int kRedBlocks = 1024;      // max partial-sum blocks for the r x t^2 reductions
inline size_t red_ws_floats(int r, int t) { return size_t(kRedBlocks) * r * t * t; }

}  // namespace stl
