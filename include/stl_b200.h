/*
 * stl_b200.h — C ABI of the B200-native Strassen-Tile (STL) operator.
 *
 * The reference (arXiv 2503.12211, /root/reference/pkg/src/strassen_tile) is a pure-Python
 * numpy package with no FFI; its operator API is the flat Python namespace. Each entry point
 * below replaces one reference function on the hot path, cited as file:line. The Python
 * mirror (paper_2503_12211_b200/) binds these through ctypes.
 *
 * Conventions
 *  - All pointers are DEVICE pointers except where noted; `stream` is a cudaStream_t (NULL =
 *    legacy default stream). Calls are stream-ordered and never synchronise the host.
 *  - dtype: STL_F32 or STL_BF16. Matrices are row-major with a leading dimension in elements.
 *  - "planes": the GPU-native encoded layout. An encoded tensor with tile grid (R, C) and rank
 *    r is stored slice-major as r contiguous row-major (R x C) planes: element (I, J, p) at
 *    p*R*C + I*C + J. The reference stores the same numbers fiber-contiguous as (R, C, r)
 *    (snf_operator.py:194-196); convert with a (2, 0, 1) permutation.
 *  - Pre-encoded weights ("w_enc", StlLayer.weights toy_network.py:45-71, reference layout
 *    (K/t, N/t, r)) are stored as planes of the TRANSPOSED tile grid: (r, N/t, K/t), i.e. the
 *    reference tensor permuted (2, 1, 0). Each plane is then the K-major B operand of a
 *    tensor-core slice GEMM.
 *  - Encoders/decoder (SnfTriple e_x, e_w, d; snf_operator.py:45-70) are fp32 (r, t*t) row-major
 *    device arrays; d is applied transposed exactly as in the reference (snf_operator.py:18).
 *  - Every function returns STL_OK (0) or an error code; stl_last_error() describes the last
 *    failure on the calling thread. Error classes mirror the reference: STL_ERR_SHAPE <->
 *    ShapeError (dense_core.py:30-31), STL_ERR_VALUE <-> ValueError, STL_ERR_INDEX <->
 *    IndexError (snf_operator.py:102-103).
 */
#ifndef STL_B200_H
#define STL_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define STL_API __attribute__((visibility("default")))
#else
#define STL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* STL_F24 is never a user-facing input/output dtype: it names the bf16 path's intermediate
 * format for fp32 slice products (the y_enc cache), fp32 rounded to 24 bits and stored as a
 * 16-bit high plane set followed by an 8-bit low plane set (3 bytes per element). */
enum stl_dtype { STL_F32 = 0, STL_BF16 = 1, STL_F24 = 2 };

enum stl_status {
  STL_OK = 0,
  STL_ERR_SHAPE = 1,
  STL_ERR_VALUE = 2,
  STL_ERR_INDEX = 3,
  STL_ERR_CUDA = 4,
  STL_ERR_UNSUPPORTED = 5
};

/* Slice-GEMM operand layouts. */
enum stl_layout { STL_K_MAJOR = 0, STL_MN_MAJOR = 1 };

/* Library version string, e.g. "stl_b200 0.1 sm_100a". Host-only. */
STL_API const char* stl_version(void);
/* Message describing the last non-OK status returned on this thread. Host-only. */
STL_API const char* stl_last_error(void);
/* Largest rank r accepted by the transform kernels. */
STL_API int stl_max_rank(void);
/* Floats of scratch needed by the fused r x t^2 reductions of stl_backward. */
STL_API int64_t stl_reduce_workspace_floats(int r, int t);

/*
 * encode_tiles (snf_operator.py:80-85):  out[I, J, p] = sum_c encoder[p, c] * vec_tile(m, I, J)[c]
 * m: (rows, cols) with leading dim ld_m; out: planes (r, rows/t, cols/t) of dtype_out.
 */
STL_API int stl_encode(const void* m, int dtype_in, int64_t rows, int64_t cols, int64_t ld_m,
               const float* encoder, int t, int r, void* out, int dtype_out, void* stream);

/*
 * decode_tiles (snf_operator.py:88-96):  out tile (I, J) = unvec(decoder^T @ enc[I, J, :])
 * enc: planes (r, block_rows, block_cols); out: (block_rows*t, block_cols*t), leading dim ld_out.
 */
STL_API int stl_decode(const void* enc, int dtype_in, int64_t block_rows, int64_t block_cols, int r,
               const float* decoder, int t, void* out, int dtype_out, int64_t ld_out,
               void* stream);

/*
 * _slice_products (snf_operator.py:107-116):  C_p = A_p @ B_p for p = 0..r-1.
 * A: a_layout STL_K_MAJOR -> planes (r, M, K); STL_MN_MAJOR -> planes (r, K, M).
 * B: b_layout STL_K_MAJOR -> planes (r, N, K); STL_MN_MAJOR -> planes (r, K, N).
 * C: planes (r, M, N) of dtype_c (STL_F32 keeps the slice accumulators exact in fp32;
 *    STL_F24 — bf16 operands, M > 128, N % 16 == 0, 16-byte aligned — writes them rounded to
 *    24 bits as 3*r*M*N bytes: the high 16 bits of every element, then the next 8 bits).
 * dtype_ab = STL_BF16 runs the tcgen05/TMEM tensor-core kernel (when the contiguous dims are
 * multiples of 8); STL_F32 runs the fp32 FFMA kernel (TF32 would miss the 1e-5 fp32 bar).
 */
STL_API int stl_slice_gemm(const void* a, int a_layout, const void* b, int b_layout, void* c,
                   int dtype_c, int dtype_ab, int r, int64_t M, int64_t N, int64_t K,
                   void* stream);

/*
 * Slice-product storage format (the forward's y_enc cache and scratch, the backward's g_u): an
 * explicit argument of the _ex entry points, never process state.
 *   STL_PROD_AUTO: per shape. On the bf16 t = 4 tensor-core path (M/t > 128, K/t % 8 == 0):
 *     bf16 planes for r <= 32 (N/t % 64 == 0); for r in (32, 64] fp32-class products — STL_F24
 *     planes in a cache-less forward (N/t % 128 == 0), fp32 products with a bf16 cache copy in
 *     training. Otherwise fp32 products (a cache in the compute dtype).
 *   STL_BF16 / STL_F24 / STL_F32: force one (STL_ERR_VALUE when the shape cannot use it).
 */
#define STL_PROD_AUTO (-1)
/* Format of the y_enc cache a training forward writes: STL_F32 (fp32 dtype), STL_BF16 or
 * STL_F24; -1 with stl_last_error set when `prod` is unavailable for the shape. */
STL_API int stl_cache_format(int64_t M, int64_t K, int64_t N, int t, int r, int dtype, int prod);
/* Bytes of that cache (r, M/t, N/t) planes: 4, 2 or 3 bytes per element. stl_cache_bytes is the
 * STL_PROD_AUTO case. */
STL_API int64_t stl_cache_bytes_ex(int64_t M, int64_t K, int64_t N, int t, int r, int dtype,
                                   int prod);
STL_API int64_t stl_cache_bytes(int64_t M, int64_t K, int64_t N, int t, int r, int dtype);

/*
 * stl_batched (snf_operator.py:156-172) / stl_layer_forward + _layer_forward_cached
 * (toy_network.py:74-92):  y = decode(slice_products(encode(x, e_x), w_enc), d).
 *   x: (M, K) ld_x, dtype;  w_enc: planes (r, N/t, K/t) of dtype;  y: (M, N) ld_y, dtype.
 *   x_enc_ws: planes (r, M/t, K/t) of dtype (also the cache `u`);
 *   y_enc_cache: NULL, or stl_cache_bytes_ex(..., prod) bytes receiving the slice products in
 *                the format stl_cache_format(..., prod) reports (the cache `y_enc` for
 *                stl_backward_ex, which takes that format back as an argument);
 *   scratch: device workspace of at least stl_forward_scratch_bytes(...) bytes.
 *   M, K, N must be multiples of t (ShapeError otherwise, as the reference).
 * encode -> slice GEMM (tcgen05, bf16 / F24 / fp32 products) -> decode. stl_forward is
 * stl_forward_ex with prod = STL_PROD_AUTO.
 */
STL_API int64_t stl_forward_scratch_bytes(int64_t M, int64_t K, int64_t N, int t, int r,
                                          int dtype);
STL_API int stl_forward_ex(const void* x, int64_t M, int64_t K, int64_t ld_x, const void* w_enc,
                           int64_t N, const float* e_x, const float* d, int t, int r, int dtype,
                           void* y, int64_t ld_y, void* x_enc_ws, void* y_enc_cache, void* scratch,
                           int64_t scratch_bytes, int prod, void* stream);
STL_API int stl_forward(const void* x, int64_t M, int64_t K, int64_t ld_x, const void* w_enc, int64_t N,
                const float* e_x, const float* d, int t, int r, int dtype, void* y, int64_t ld_y,
                void* x_enc_ws, void* y_enc_cache, void* scratch, int64_t scratch_bytes,
                void* stream);

/*
 * _layer_backward (toy_network.py:95-106), all seven formulas:
 *   g_d  = sum_{I,J} y_enc[I,J,p] gvy[I,J,c]      -> g_d  fp32 (r, t*t)
 *   g_enc = gvy @ d^T                              -> g_enc_ws planes (r, M/t, N/t) dtype
 *   g_w  = sum_I u[I,L,p] g_enc[I,J,p]             -> g_w  fp32 planes (r, N/t, K/t)
 *   g_u  = sum_J W[L,J,p] g_enc[I,J,p]             -> g_u_ws (r, M/t, K/t): fp32 planes, or the
 *                                                     products format `gu_prod` (bf16 / F24, in
 *                                                     the first 2-3 bytes per element)
 *   g_ex = sum_{I,L} g_u[I,L,p] vx[I,L,c]          -> g_ex fp32 (r, t*t)
 *   g_x  = untile(g_u @ e_x)                       -> g_x (M, K) ld_gx, dtype
 * Inputs: gy (M, N) ld_gy; x (M, K) ld_x (the layer input, vx); w_enc as in stl_forward;
 * x_enc (= u) and y_enc from the forward cache, y_enc_format = the format the forward wrote it
 * in (stl_cache_format; a format this shape's forward cannot write -> STL_ERR_VALUE).
 * gu_prod: STL_PROD_AUTO (the cache's format family: F24 cache -> F24 g_u where the shape
 * allows, else the AUTO rule) or a forced format. red_ws: stl_reduce_workspace_floats floats.
 * Any of g_ex, g_d, g_w, g_x may be NULL to skip that gradient, except that g_ex is fused with
 * g_x (g_ex without g_x -> STL_ERR_VALUE). gw_ready: a cudaEvent_t or NULL; when given it is
 * recorded on `stream` as soon as g_w is final (before the g_x / g_ex decode), so a
 * data-parallel caller can all-reduce g_w on another stream while the decode runs.
 * stl_backward = stl_backward_ex with the AUTO cache format, gu_prod = STL_PROD_AUTO and no
 * event.
 */
STL_API int stl_backward_ex(const void* gy, int64_t ld_gy, const void* x, int64_t ld_x,
                            const void* w_enc, const float* e_x, const float* d,
                            const void* x_enc, const void* y_enc, int y_enc_format, int64_t M,
                            int64_t K, int64_t N, int t, int r, int dtype, float* g_ex, float* g_d,
                            float* g_w, void* g_x, int64_t ld_gx, void* g_enc_ws, float* g_u_ws,
                            float* red_ws, int gu_prod, void* gw_ready, void* stream);
STL_API int stl_backward(const void* gy, int64_t ld_gy, const void* x, int64_t ld_x, const void* w_enc,
                 const float* e_x, const float* d, const void* x_enc, const void* y_enc,
                 int64_t M, int64_t K, int64_t N, int t, int r, int dtype, float* g_ex,
                 float* g_d, float* g_w, void* g_x, int64_t ld_gx, void* g_enc_ws,
                 float* g_u_ws, float* red_ws, void* stream);

/*
 * stl_fused_step (snf_operator.py:175-188, Algorithm 2):
 *   out = slice_products(x_prev @ (e_x d^T)^T, w_enc), staying in encoded space.
 *   x_prev: fp32 planes (r, BR, BK); w_enc: planes (r, BN, BK) of dtype;
 *   out: fp32 planes (r, BR, BN); mixed_ws: planes (r, BR, BK) of dtype; comp_ws: r*r floats.
 */
STL_API int stl_fused_step(const float* x_prev, int64_t block_rows, int64_t block_k, const void* w_enc,
                   int64_t block_n, const float* e_x, const float* d, int t, int r, int dtype,
                   float* out, void* mixed_ws, float* comp_ws, void* stream);
/*
 * stl_fused_step_ex: the same step with the encoded activations' formats explicit, so a bf16
 * chain stays in 2-byte planes end to end: x_prev_dtype / out_dtype = STL_F32 or STL_BF16
 * (STL_BF16 requires dtype == STL_BF16). The bf16 path remixes with the streaming tensor-core
 * kernel (r <= 32, BK % 64 == 0): one HBM pass over the r planes in and out.
 */
STL_API int stl_fused_step_ex(const void* x_prev, int x_prev_dtype, int64_t block_rows,
                              int64_t block_k, const void* w_enc, int64_t block_n,
                              const float* e_x, const float* d, int t, int r, int dtype, void* out,
                              int out_dtype, void* mixed_ws, float* comp_ws, void* stream);

/*
 * Token-row plumbing for STL layers over (B, T, features) activations with T % t == 1 (the
 * T2T-ViT-7 model's 197 tokens; no counterpart in the reference package,
 * SPEC.md:8). The layer runs on Tp = T - 1 + t rows per sample (t - 1 null rows appended) and
 * the last t output rows of each sample are folded into one with t learnable coefficients.
 * One HBM pass each; activations bf16 row-major, features multiples of 8, 16-byte aligned.
 *   stl_token_pad:   out (B, Tp, Cp) bf16 = x (B, T, C) of dtype_in, zero rows / columns.
 *   stl_token_unpad: out (B, T, C) of dtype_out = g (B, Tp, Cp)[:, :T, :C].
 *   stl_token_fold:  out (B, T, N) = y rows < T-1, row T-1 = sum_i fold[i] y[T-1+i]; + bias
 *                    (bias: N fp32 or NULL; fold: t fp32, device pointers).
 *   stl_token_fold_backward: g_y (B, Tp, N) from g_out (B, T, N) and y; g_bias_fold receives N
 *                    bias gradients then t fold gradients (fixed-order sums; ws of
 *                    stl_token_fold_ws_floats floats).
 */
STL_API int stl_token_pad(const void* x, int dtype_in, int64_t B, int64_t T, int64_t C, void* out,
                          int64_t Tp, int64_t Cp, void* stream);
STL_API int stl_token_unpad(const void* g, int64_t B, int64_t Tp, int64_t Cp, void* out,
                            int dtype_out, int64_t T, int64_t C, void* stream);
STL_API int stl_token_fold(const void* y, int64_t B, int64_t Tp, int64_t N, int t, const float* fold,
                           const float* bias, void* out, int64_t T, void* stream);
STL_API int64_t stl_token_fold_ws_floats(int64_t B, int64_t T, int64_t N, int t);
STL_API int stl_token_fold_backward(const void* g_out, const void* y, int64_t B, int64_t Tp,
                                    int64_t N, int t, const float* fold, int64_t T, void* g_y,
                                    float* g_bias_fold, float* ws, int64_t ws_floats,
                                    void* stream);

/*
 * Launch profiler (no reference counterpart; B200 measurement aid). While enabled, every
 * kernel launch the library issues is bracketed by CUDA events on its own stream, so a caller
 * can attribute device time to kernels inside a timed region without a profiler attached.
 *   stl_profile_enable(1) ... work ... synchronise ... stl_profile_count / stl_profile_get.
 * stl_profile_get fills the kernel name (static string), elapsed milliseconds and the number
 * of kernel launches in that record (1, or 2 for transform+reduction pairs). Host-only.
 */
STL_API int stl_profile_enable(int on);
STL_API int stl_profile_reset(void);
STL_API int stl_profile_count(void);
STL_API int stl_profile_get(int index, const char** name, float* ms, int* launches);

#ifdef __cplusplus
}
#endif

#endif /* STL_B200_H */
