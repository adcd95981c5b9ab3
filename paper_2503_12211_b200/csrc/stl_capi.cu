// stl_capi.cu — extern "C" entry points (include/stl_b200.h): argument validation with the
// reference's error classes, then stream-ordered launches of the STL kernels.
#include <cstdio>
#include <cstdarg>
#include <mutex>
#include <string>
#include <vector>
#include "../../include/stl_b200.h"
#include "stl_internal.h"

namespace {
thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(STL_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return STL_OK;
}

bool valid_dtype(int dt) { return dt == STL_F32 || dt == STL_BF16; }

int check_tr(int t, int r) {
  if (t < 1 || r < 1) return fail(STL_ERR_SHAPE, "need t >= 1 and r >= 1, got t=%d, r=%d", t, r);
  if (!(t == 1 || t == 2 || t == 4 || t == 8))
    return fail(STL_ERR_UNSUPPORTED, "tile size t=%d not supported (1, 2, 4, 8)", t);
  if (r > stl::kMaxRank)
    return fail(STL_ERR_UNSUPPORTED, "rank r=%d exceeds the supported maximum %d", r,
                stl::kMaxRank);
  return STL_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------ launch profiler
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
  int launches;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_pool;
size_t g_pool_used = 0;

// Brackets the launches issued in its scope with events on `s` while profiling is enabled.
struct Prof {
  int idx = -1;
  cudaStream_t s;
  Prof(const char* name, cudaStream_t st, int launches = 1) : s(st) {
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (g_pool_used == g_pool.size()) {
      cudaEvent_t a, b;
      if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return;
      g_pool.emplace_back(a, b);
    }
    auto ev = g_pool[g_pool_used++];
    cudaEventRecord(ev.first, s);
    g_prof.push_back({name, ev.first, ev.second, launches});
    idx = static_cast<int>(g_prof.size()) - 1;
  }
  ~Prof() {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_prof[idx].b, s);
  }
};

int run_gemm(const void* a, int al, const void* b, int bl, void* c, int cdt, int abdt, int r,
             int64_t M, int64_t N, int64_t K, cudaStream_t s, void* c2 = nullptr,
             bool* c2_done = nullptr) {
  if (M == 0 || N == 0 || r == 0) return STL_OK;
  if (K == 0) {
    return check_cuda(cudaMemsetAsync(c, 0, stl::dtype_size(cdt) * r * M * N, s), "memset");
  }  // (F24 zero = all-zero bytes)
  stl::SliceGemmProblem pb{a, al, b, bl, c, cdt, abdt, r, M, N, K};
  if (cdt == stl::kF24 && !stl::slice_gemm_f24_supported(pb))
    return fail(STL_ERR_VALUE, "F24 slice products need 16-byte aligned operands");
  const bool tc = stl::slice_gemm_tc_supported(pb);
  if (tc && c2) {
    pb.c2 = c2;
    if (c2_done) *c2_done = true;
  }
  Prof prof(tc ? "slice_gemm_tcgen05" : "slice_gemm_simt", s);
  cudaError_t e = tc ? stl::slice_gemm_tc(pb, s) : stl::slice_gemm_simt(pb, s);
  return check_cuda(e, "slice_gemm launch");
}
}  // namespace

extern "C" {

const char* stl_version(void) { return "stl_b200 0.1 sm_100a"; }
const char* stl_last_error(void) { return g_last_error.c_str(); }
int stl_max_rank(void) { return stl::kMaxRank; }
int64_t stl_reduce_workspace_floats(int r, int t) {
  return static_cast<int64_t>(stl::red_ws_floats(r, t));
}

int stl_encode(const void* m, int dtype_in, int64_t rows, int64_t cols, int64_t ld_m,
               const float* encoder, int t, int r, void* out, int dtype_out, void* stream) {
  if (int st = check_tr(t, r)) return st;
  if (!valid_dtype(dtype_in) || !valid_dtype(dtype_out))
    return fail(STL_ERR_VALUE, "invalid dtype");
  if (rows < 0 || cols < 0 || rows % t || cols % t)
    return fail(STL_ERR_SHAPE, "tile size %d does not divide shape (%lld, %lld)", t,
                (long long)rows, (long long)cols);
  if (ld_m < cols) return fail(STL_ERR_SHAPE, "leading dimension %lld < cols %lld",
                               (long long)ld_m, (long long)cols);
  return check_cuda(stl::tiles_to_planes(m, dtype_in, ld_m, rows / t, cols / t, t, encoder, r,
                                         out, dtype_out, nullptr, STL_F32, nullptr, nullptr,
                                         as_stream(stream)),
                    "encode");
}

int stl_decode(const void* enc, int dtype_in, int64_t block_rows, int64_t block_cols, int r,
               const float* decoder, int t, void* out, int dtype_out, int64_t ld_out,
               void* stream) {
  if (int st = check_tr(t, r)) return st;
  if (!valid_dtype(dtype_in) || !valid_dtype(dtype_out))
    return fail(STL_ERR_VALUE, "invalid dtype");
  if (block_rows < 0 || block_cols < 0) return fail(STL_ERR_SHAPE, "negative block grid");
  if (ld_out < block_cols * t) return fail(STL_ERR_SHAPE, "leading dimension too small");
  return check_cuda(stl::planes_to_tiles(enc, dtype_in, r, block_rows, block_cols, t, decoder,
                                         out, dtype_out, ld_out, nullptr, STL_F32, 0, nullptr,
                                         nullptr, as_stream(stream)),
                    "decode");
}

int stl_slice_gemm(const void* a, int a_layout, const void* b, int b_layout, void* c,
                   int dtype_c, int dtype_ab, int r, int64_t M, int64_t N, int64_t K,
                   void* stream) {
  if ((!valid_dtype(dtype_c) && dtype_c != STL_F24) || !valid_dtype(dtype_ab))
    return fail(STL_ERR_VALUE, "invalid dtype");
  if (dtype_c == STL_F24 && dtype_ab != STL_BF16)
    return fail(STL_ERR_UNSUPPORTED, "F24 slice products need bf16 operands");
  if (r < 0 || M < 0 || N < 0 || K < 0) return fail(STL_ERR_SHAPE, "negative extent");
  if ((a_layout != 0 && a_layout != 1) || (b_layout != 0 && b_layout != 1))
    return fail(STL_ERR_VALUE, "invalid operand layout");
  return run_gemm(a, a_layout, b, b_layout, c, dtype_c, dtype_ab, r, M, N, K, as_stream(stream));
}

namespace {
// Storage format of the slice products (forward y_enc, backward g_u) — an explicit argument of
// every call (STL_PROD_AUTO or a forced format), never process state, so stl_forward /
// stl_backward are pure and re-entrant and the cache's format travels with the cache.
// AUTO on the bf16 t = 4 path: bf16 planes (2 B/element; they feed bf16-output decodes and
// r x t^2 reductions: measured rel. error of y at 8192^3 2.9e-3 vs 2.4e-3 with fp32-class
// products, bar 1e-2) for r <= 32; above r = 32 (the Strassen x Strassen rank 49, where bf16
// products reach 9.6e-3) fp32-class products: F24 in a cache-less forward, fp32 products with a
// bf16 cache copy in training (the backward's fused reductions read bf16 or F24 at r <= 32).
// Returns the products' format (STL_BF16, STL_F24, or -1 = fp32 products), or -2 when `prod`
// forces a format the shape cannot use.
constexpr int kFp32Products = -1, kBadFormat = -2;
bool bf16_tc_path(int64_t rows, int64_t kt, int t, int dtype) {
  return dtype == STL_BF16 && t == 4 && rows > 128 && kt % 8 == 0;
}
int product_format(int64_t rows, int64_t cols, int64_t kt, int t, int r, int dtype, int prod,
                   bool inference) {
  const bool tc = bf16_tc_path(rows, kt, t, dtype);
  // t = 2 (configs[2]; FLOP-losing by construction, so a cache-less forward only): bf16
  // products halve the r/4 x |Y| plane traffic the decode streams
  const bool tc2 = dtype == STL_BF16 && t == 2 && rows > 128 && kt % 8 == 0 && cols % 4 == 0;
  switch (prod) {
    case STL_PROD_AUTO:
      if (tc2 && inference && r <= 32) return STL_BF16;
      if (!tc) return kFp32Products;
      if (r > 32) return inference && r <= 64 && cols % 128 == 0 ? stl::kF24 : kFp32Products;
      return cols % 64 == 0 ? STL_BF16 : kFp32Products;
    case STL_F32:
      return kFp32Products;
    case STL_BF16:
      if (tc2 && inference) return STL_BF16;
      return tc && cols % 64 == 0 && (inference || r <= 32) ? STL_BF16 : kBadFormat;
    case STL_F24:
      return tc && cols % 128 == 0 && r <= (inference ? 64 : 32) ? stl::kF24 : kBadFormat;
    default:
      return kBadFormat;
  }
}
// The y_enc cache of a training forward: the products' format, or the compute dtype when the
// products are fp32 (a bf16 copy on the bf16 path).
int cache_format(int64_t rows, int64_t cols, int64_t kt, int t, int r, int dtype, int prod) {
  const int pf = product_format(rows, cols, kt, t, r, dtype, prod, false);
  return pf == kFp32Products ? dtype : pf;
}
int bad_format(int prod) {
  return fail(STL_ERR_VALUE, "slice-product format %d is not available for this shape / dtype "
              "(bf16 needs t = 4, r <= 32, N/t %% 64 == 0; F24 needs N/t %% 128 == 0)", prod);
}
// Split-K factor for a tensor-core slice GEMM (M x N per slice, contraction K) whose output
// tiles cannot fill the GPU: S divides K, K / S >= 512; 1 = no split. Used for g_w, whose
// partials (r * S * M * N fp32) fit the g_u workspace (r * K * N fp32) when S * M <= K.
int split_k_factor(int64_t M, int64_t N, int64_t K, int r, int dtype) {
  if (dtype != STL_BF16 || M % 8 || N % 8 || (M * N) % 4) return 1;
  const bool one_cta = M <= 128;  // 1-CTA tiles (128 x BN) vs CTA pairs (256 x BN)
  const int64_t bn = N <= 128 ? 128 : 256;
  const int64_t tiles = static_cast<int64_t>(r) * ((M + (one_cta ? 127 : 255)) / (one_cta ? 128 : 256)) *
                        ((N + bn - 1) / bn);
  const int64_t slots = one_cta ? stl::sm_count() : stl::sm_count() / 2;
  int64_t want = slots / (tiles > 0 ? tiles : 1);
  if (want > 16) want = 16;
  for (int64_t S = want; S > 1; --S)
    if (K % S == 0 && K / S >= 512 && S * M <= K) return static_cast<int>(S);
  return 1;
}
}  // namespace

int stl_cache_format(int64_t M, int64_t K, int64_t N, int t, int r, int dtype, int prod) {
  if (t < 1 || r < 1 || M < 0 || K < 0 || N < 0) return fail(STL_ERR_SHAPE, "invalid shape"), -1;
  if (!valid_dtype(dtype)) return fail(STL_ERR_VALUE, "invalid dtype"), -1;
  const int f = cache_format(M / t, N / t, K / t, t, r, dtype, prod);
  if (f == kBadFormat) return bad_format(prod), -1;
  return f;
}

int64_t stl_cache_bytes_ex(int64_t M, int64_t K, int64_t N, int t, int r, int dtype, int prod) {
  if (t < 1 || r < 1 || M < 0 || K < 0 || N < 0 || !valid_dtype(dtype)) return 0;
  const int f = cache_format(M / t, N / t, K / t, t, r, dtype, prod);
  if (f == kBadFormat) return 0;
  return static_cast<int64_t>(r) * (M / t) * (N / t) * static_cast<int64_t>(stl::dtype_size(f));
}

int64_t stl_cache_bytes(int64_t M, int64_t K, int64_t N, int t, int r, int dtype) {
  return stl_cache_bytes_ex(M, K, N, t, r, dtype, STL_PROD_AUTO);
}

int64_t stl_forward_scratch_bytes(int64_t M, int64_t K, int64_t N, int t, int r, int dtype) {
  if (t < 1 || r < 1 || M < 0 || K < 0 || N < 0) return 0;
  return static_cast<int64_t>(r) * (M / t) * (N / t) * 4;
}

int stl_forward_ex(const void* x, int64_t M, int64_t K, int64_t ld_x, const void* w_enc, int64_t N,
                   const float* e_x, const float* d, int t, int r, int dtype, void* y,
                   int64_t ld_y, void* x_enc_ws, void* y_enc_cache, void* scratch,
                   int64_t scratch_bytes, int prod, void* stream) {
  if (int st = check_tr(t, r)) return st;
  if (!valid_dtype(dtype)) return fail(STL_ERR_VALUE, "invalid dtype");
  if (M < 0 || K < 0 || N < 0) return fail(STL_ERR_SHAPE, "negative extent");
  if (M % t) return fail(STL_ERR_SHAPE, "batch %lld not divisible by tile size %d", (long long)M, t);
  if (K % t || N % t)
    return fail(STL_ERR_SHAPE, "tile size %d does not divide K=%lld / N=%lld", t, (long long)K,
                (long long)N);
  if (ld_x < K || ld_y < N) return fail(STL_ERR_SHAPE, "leading dimension too small");
  cudaStream_t s = as_stream(stream);
  const int64_t bi = M / t, bk = K / t, bj = N / t;
  const int pfmt = product_format(bi, bj, bk, t, r, dtype, prod, y_enc_cache == nullptr);
  if (pfmt == kBadFormat) return bad_format(prod);
  if (M == 0 || N == 0) return STL_OK;
  int st;
  {
    Prof prof("encode_x", s);
    st = check_cuda(stl::tiles_to_planes(x, dtype, ld_x, bi, bk, t, e_x, r, x_enc_ws, dtype,
                                         nullptr, STL_F32, nullptr, nullptr, s),
                    "forward encode");
  }
  if (st) return st;
  if (pfmt >= 0) {
    // slice products (bf16 or F24) straight into the cache (or scratch), decoded from there
    void* prod_buf = y_enc_cache ? y_enc_cache : scratch;
    const int64_t need = static_cast<int64_t>(stl::dtype_size(pfmt)) * r * bi * bj;
    if (!y_enc_cache && scratch_bytes < need)
      return fail(STL_ERR_VALUE, "scratch too small: %lld < %lld bytes", (long long)scratch_bytes,
                  (long long)need);
    st = run_gemm(x_enc_ws, STL_K_MAJOR, w_enc, STL_K_MAJOR, prod_buf, pfmt, dtype, r, bi, bj, bk,
                  s);
    if (st) return st;
    Prof prof("decode_y", s);
    return check_cuda(stl::planes_to_tiles(prod_buf, pfmt, r, bi, bj, t, d, y, dtype, ld_y,
                                           nullptr, STL_F32, 0, nullptr, nullptr, s),
                      "forward decode");
  }
  float* yenc = nullptr;
  if (dtype == STL_F32 && y_enc_cache) {
    yenc = static_cast<float*>(y_enc_cache);
  } else {
    const int64_t need = static_cast<int64_t>(r) * bi * bj * 4;
    if (scratch_bytes < need)
      return fail(STL_ERR_VALUE, "scratch too small: %lld < %lld bytes", (long long)scratch_bytes,
                  (long long)need);
    yenc = static_cast<float*>(scratch);
  }
  bool cache_done = false;
  st = run_gemm(x_enc_ws, STL_K_MAJOR, w_enc, STL_K_MAJOR, yenc, STL_F32, dtype, r, bi, bj, bk, s,
                (y_enc_cache && dtype == STL_BF16) ? y_enc_cache : nullptr, &cache_done);
  if (st) return st;
  {
    Prof prof("decode_y", s);
    st = check_cuda(stl::planes_to_tiles(yenc, STL_F32, r, bi, bj, t, d, y, dtype, ld_y, nullptr,
                                         STL_F32, 0, nullptr, nullptr, s),
                    "forward decode");
  }
  if (st) return st;
  if (y_enc_cache && dtype == STL_BF16 && !cache_done) {
    Prof prof("cache_cast", s);
    st = check_cuda(stl::cast_f32_to_bf16(yenc, y_enc_cache, static_cast<int64_t>(r) * bi * bj, s),
                    "cache cast");
  }
  return st;
}

int stl_forward(const void* x, int64_t M, int64_t K, int64_t ld_x, const void* w_enc, int64_t N,
                const float* e_x, const float* d, int t, int r, int dtype, void* y, int64_t ld_y,
                void* x_enc_ws, void* y_enc_cache, void* scratch, int64_t scratch_bytes,
                void* stream) {
  return stl_forward_ex(x, M, K, ld_x, w_enc, N, e_x, d, t, r, dtype, y, ld_y, x_enc_ws,
                        y_enc_cache, scratch, scratch_bytes, STL_PROD_AUTO, stream);
}

int stl_backward_ex(const void* gy, int64_t ld_gy, const void* x, int64_t ld_x, const void* w_enc,
                    const float* e_x, const float* d, const void* x_enc, const void* y_enc,
                    int y_enc_format, int64_t M, int64_t K, int64_t N, int t, int r, int dtype,
                    float* g_ex, float* g_d, float* g_w, void* g_x, int64_t ld_gx, void* g_enc_ws,
                    float* g_u_ws, float* red_ws, int gu_prod, void* gw_ready, void* stream) {
  if (int st = check_tr(t, r)) return st;
  if (!valid_dtype(dtype)) return fail(STL_ERR_VALUE, "invalid dtype");
  if (M < 0 || K < 0 || N < 0 || M % t || K % t || N % t)
    return fail(STL_ERR_SHAPE, "tile size %d does not divide (M, K, N) = (%lld, %lld, %lld)", t,
                (long long)M, (long long)K, (long long)N);
  if ((g_d || g_ex) && !red_ws) return fail(STL_ERR_VALUE, "reduction workspace required");
  if (g_ex && !g_x) return fail(STL_ERR_VALUE, "g_ex needs the g_x output (it is fused with it)");
  cudaStream_t s = as_stream(stream);
  const int64_t bi = M / t, bk = K / t, bj = N / t;
  // The cache format is the caller's record of what the forward wrote; it must be one this
  // shape's forward can write (any forced format), else the bytes would be misread.
  bool fmt_ok = y_enc_format == dtype;  // fp32 products (fp32 mode) or the bf16 copy
  if (y_enc_format == stl::kF24 || (y_enc_format == STL_BF16 && dtype == STL_BF16))
    fmt_ok = fmt_ok || product_format(bi, bj, bk, t, r, dtype, y_enc_format, false) == y_enc_format;
  if (!fmt_ok)
    return fail(STL_ERR_VALUE, "y_enc cache format %d cannot come from a forward of this shape "
                "and dtype", y_enc_format);
  // g_u products: the cache's format family by default (F24 cache -> F24 g_u when the shape
  // allows it), else as requested.
  int gu_fmt;
  if (gu_prod == STL_PROD_AUTO && y_enc_format == stl::kF24) {
    gu_fmt = product_format(bi, bk, bj, t, r, dtype, stl::kF24, false);
    if (gu_fmt == kBadFormat) gu_fmt = kFp32Products;
  } else {
    gu_fmt = product_format(bi, bk, bj, t, r, dtype, gu_prod, false);
    if (gu_fmt == kBadFormat) return bad_format(gu_prod);
  }
  const int gu_dt = gu_fmt >= 0 ? gu_fmt : STL_F32;
  // gvy -> g_enc (planes), fused with g_d = sum y_enc (x) gvy.
  int st;
  {
    Prof prof(g_d ? "encode_gy+g_d" : "encode_gy", s, g_d ? 2 : 1);
    st = check_cuda(stl::tiles_to_planes(gy, dtype, ld_gy, bi, bj, t, d, r, g_enc_ws, dtype,
                                         g_d ? y_enc : nullptr, y_enc_format, g_d, red_ws, s),
                    "backward encode(gy)");
  }
  if (st) return st;
  // g_w^T_p (N/t x K/t) = g_enc_p^T (N/t x M/t) . u_p (M/t x K/t): both operands MN-major.
  // g_u_p (M/t x K/t) = g_enc_p (M/t x N/t) . W_p (N/t x K/t): B is N-major. Stored in gu_dt
  // (bf16 / F24 on the bf16 path: 2 or 3 of the 4 bytes of g_u_ws used).
  bool gw_done = false, gu_done = false;
  if (g_w && g_x && bi > 0 && bk > 0 && bj > 0 && r > 0) {
    // both slice-GEMMs in one persistent launch (g_w first: its K = M/t is the longer one)
    stl::SliceGemmProblem pw{g_enc_ws, STL_MN_MAJOR, x_enc, STL_MN_MAJOR, g_w, STL_F32, dtype,
                             r, bj, bk, bi};
    stl::SliceGemmProblem pu{g_enc_ws, STL_K_MAJOR, w_enc, STL_MN_MAJOR, g_u_ws, gu_dt, dtype,
                             r, bi, bk, bj};
    if (stl::slice_gemm_tc_group_supported(pw, pu)) {
      Prof prof("slice_gemm_tcgen05", s);
      st = check_cuda(stl::slice_gemm_tc_group(pw, pu, s), "grouped slice_gemm launch");
      if (st) return st;
      gw_done = gu_done = true;
    }
  }
  if (g_w && !gw_done) {
    // Few output tiles (narrow layers: M = N/t and N = K/t small, a long K = M/t): split the
    // contraction over S consecutive row blocks — (r, bi, .) operands are exactly
    // (r * S, bi / S, .) ones — into g_u_ws (free until the g_u GEMM) and sum the S partials
    // in fixed order.
    const int S = g_u_ws ? split_k_factor(bj, bk, bi, r, dtype) : 1;
    if (S > 1) {
      st = run_gemm(g_enc_ws, STL_MN_MAJOR, x_enc, STL_MN_MAJOR, g_u_ws, STL_F32, dtype, r * S,
                    bj, bk, bi / S, s);
      if (st) return st;
      Prof prof("sum_splits", s);
      st = check_cuda(stl::slice_gemm_sum_splits(g_u_ws, r, S, bj * bk, g_w, s), "split-K sum");
    } else {
      st = run_gemm(g_enc_ws, STL_MN_MAJOR, x_enc, STL_MN_MAJOR, g_w, STL_F32, dtype, r, bj, bk,
                    bi, s);
    }
    if (st) return st;
  }
  // g_w is final here (the g_x / g_ex decode does not touch it): let the caller start its
  // data-parallel all-reduce on another stream while the decode runs.
  if (g_w && gw_ready) {
    st = check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(gw_ready), s), "g_w event");
    if (st) return st;
  }
  if (g_x) {
    if (!gu_done) {
      st = run_gemm(g_enc_ws, STL_K_MAJOR, w_enc, STL_MN_MAJOR, g_u_ws, gu_dt, dtype, r, bi, bk,
                    bj, s);
      if (st) return st;
    }
    Prof prof(g_ex ? "decode_gu+g_ex" : "decode_gu", s, g_ex ? 2 : 1);
    st = check_cuda(stl::planes_to_tiles(g_u_ws, gu_dt, r, bi, bk, t, e_x, g_x, dtype, ld_gx,
                                         g_ex ? x : nullptr, dtype, ld_x, g_ex, red_ws, s),
                    "backward decode(g_u)");
    if (st) return st;
  }
  return STL_OK;
}

int stl_backward(const void* gy, int64_t ld_gy, const void* x, int64_t ld_x, const void* w_enc,
                 const float* e_x, const float* d, const void* x_enc, const void* y_enc,
                 int64_t M, int64_t K, int64_t N, int t, int r, int dtype, float* g_ex,
                 float* g_d, float* g_w, void* g_x, int64_t ld_gx, void* g_enc_ws,
                 float* g_u_ws, float* red_ws, void* stream) {
  if (int st = check_tr(t, r)) return st;
  if (!valid_dtype(dtype)) return fail(STL_ERR_VALUE, "invalid dtype");
  const int fmt = t > 0 ? cache_format(M / t, N / t, K / t, t, r, dtype, STL_PROD_AUTO) : dtype;
  return stl_backward_ex(gy, ld_gy, x, ld_x, w_enc, e_x, d, x_enc, y_enc, fmt, M, K, N, t, r, dtype,
                         g_ex, g_d, g_w, g_x, ld_gx, g_enc_ws, g_u_ws, red_ws, STL_PROD_AUTO,
                         nullptr, stream);
}

namespace {
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
}  // namespace

int stl_token_pad(const void* x, int dtype_in, int64_t B, int64_t T, int64_t C, void* out,
                  int64_t Tp, int64_t Cp, void* stream) {
  if (!valid_dtype(dtype_in)) return fail(STL_ERR_VALUE, "invalid dtype");
  if (B < 0 || T < 0 || C < 0 || Tp < T || Cp < C)
    return fail(STL_ERR_SHAPE, "pad (%lld, %lld, %lld) -> (%lld, %lld) shrinks", (long long)B,
                (long long)T, (long long)C, (long long)Tp, (long long)Cp);
  if (C % 8 || Cp % 8 || !al16(x) || !al16(out))
    return fail(STL_ERR_UNSUPPORTED, "token pad needs feature counts %% 8 == 0, aligned buffers");
  Prof prof("token_pad", as_stream(stream));
  return check_cuda(stl::token_pad(x, dtype_in, B, T, C, out, Tp, Cp, as_stream(stream)),
                    "token pad");
}

int stl_token_unpad(const void* g, int64_t B, int64_t Tp, int64_t Cp, void* out, int dtype_out,
                    int64_t T, int64_t C, void* stream) {
  if (!valid_dtype(dtype_out)) return fail(STL_ERR_VALUE, "invalid dtype");
  if (B < 0 || T < 0 || C < 0 || Tp < T || Cp < C)
    return fail(STL_ERR_SHAPE, "unpad target larger than the source");
  if (C % 8 || Cp % 8 || !al16(g) || !al16(out))
    return fail(STL_ERR_UNSUPPORTED, "token unpad needs feature counts %% 8 == 0, aligned buffers");
  Prof prof("token_unpad", as_stream(stream));
  return check_cuda(stl::token_unpad(g, B, Tp, Cp, out, dtype_out, T, C, as_stream(stream)),
                    "token unpad");
}

int stl_token_fold(const void* y, int64_t B, int64_t Tp, int64_t N, int t, const float* fold,
                   const float* bias, void* out, int64_t T, void* stream) {
  if (B < 0 || N < 0 || T < 1 || t < 1 || t > stl::kFoldMaxT || Tp != T - 1 + t)
    return fail(STL_ERR_SHAPE, "fold needs Tp = T - 1 + t (T=%lld, Tp=%lld, t=%d)", (long long)T,
                (long long)Tp, t);
  if (N % 8 || !al16(y) || !al16(out) || !al16(bias))
    return fail(STL_ERR_UNSUPPORTED, "token fold needs N %% 8 == 0, aligned buffers");
  Prof prof("token_fold", as_stream(stream));
  return check_cuda(stl::token_fold(y, B, Tp, N, t, fold, bias, out, T, as_stream(stream)),
                    "token fold");
}

int64_t stl_token_fold_ws_floats(int64_t B, int64_t T, int64_t N, int t) {
  return stl::token_fold_ws_floats(B, T, N, t);
}

int stl_token_fold_backward(const void* g_out, const void* y, int64_t B, int64_t Tp, int64_t N,
                            int t, const float* fold, int64_t T, void* g_y, float* g_bias_fold,
                            float* ws, int64_t ws_floats, void* stream) {
  if (B < 0 || N < 0 || T < 1 || t < 1 || t > stl::kFoldMaxT || Tp != T - 1 + t)
    return fail(STL_ERR_SHAPE, "fold needs Tp = T - 1 + t (T=%lld, Tp=%lld, t=%d)", (long long)T,
                (long long)Tp, t);
  if (N % 8 || N > 8 * 1024 || !al16(g_out) || !al16(y) || !al16(g_y) || !al16(ws))
    return fail(STL_ERR_UNSUPPORTED, "token fold backward needs N %% 8 == 0 (<= 8192), aligned buffers");
  if (ws_floats < stl::token_fold_ws_floats(B, T, N, t))
    return fail(STL_ERR_VALUE, "fold workspace too small");
  Prof prof("token_fold_backward", as_stream(stream), 2);
  return check_cuda(stl::token_fold_backward(g_out, y, B, Tp, N, t, fold, T, g_y, g_bias_fold, ws,
                                             as_stream(stream)),
                    "token fold backward");
}

int stl_fused_step_ex(const void* x_prev, int x_prev_dtype, int64_t block_rows, int64_t block_k,
                      const void* w_enc, int64_t block_n, const float* e_x, const float* d, int t,
                      int r, int dtype, void* out, int out_dtype, void* mixed_ws, float* comp_ws,
                      void* stream) {
  if (int st = check_tr(t, r)) return st;
  if (!valid_dtype(dtype) || !valid_dtype(x_prev_dtype) || !valid_dtype(out_dtype))
    return fail(STL_ERR_VALUE, "invalid dtype");
  if ((x_prev_dtype == STL_BF16 || out_dtype == STL_BF16) && dtype != STL_BF16)
    return fail(STL_ERR_VALUE, "bf16 encoded activations need bf16 weights");
  if (block_rows < 0 || block_k < 0 || block_n < 0) return fail(STL_ERR_SHAPE, "negative extent");
  cudaStream_t s = as_stream(stream);
  int st;
  // bf16 chain: the streaming tensor-core remix forms the composite e_x d^T itself (planes in,
  // planes out, one HBM pass, no extra launch between the two slice GEMMs); else the composite
  // kernel + the generic remix
  cudaError_t e = cudaErrorNotSupported;
  if (dtype == STL_BF16 && t == 4 && r <= 32 && block_k % 64 == 0) {  // composite of 16-wide rows
    Prof prof("remix", s);
    e = stl::planes_to_planes_stream(x_prev, x_prev_dtype, r, block_rows, block_k, e_x, d,
                                     mixed_ws, s);
  }
  if (e == cudaErrorNotSupported) {
    {
      Prof prof("compose", s);
      st = check_cuda(stl::compose_coefs(e_x, d, r, t * t, comp_ws, s), "compose");
    }
    if (st) return st;
    Prof prof("remix", s);
    e = stl::planes_to_planes(x_prev, x_prev_dtype, r, block_rows * block_k, comp_ws, r, mixed_ws,
                              dtype, s);
  }
  st = check_cuda(e, "fused-step remix");
  if (st) return st;
  return run_gemm(mixed_ws, STL_K_MAJOR, w_enc, STL_K_MAJOR, out, out_dtype, dtype, r, block_rows,
                  block_n, block_k, s);
}

int stl_fused_step(const float* x_prev, int64_t block_rows, int64_t block_k, const void* w_enc,
                   int64_t block_n, const float* e_x, const float* d, int t, int r, int dtype,
                   float* out, void* mixed_ws, float* comp_ws, void* stream) {
  return stl_fused_step_ex(x_prev, STL_F32, block_rows, block_k, w_enc, block_n, e_x, d, t, r,
                           dtype, out, STL_F32, mixed_ws, comp_ws, stream);
}

int stl_profile_enable(int on) {
  g_prof_on = on != 0;
  return STL_OK;
}

int stl_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.clear();
  g_pool_used = 0;
  return STL_OK;
}

int stl_profile_count(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  return static_cast<int>(g_prof.size());
}

int stl_profile_get(int index, const char** name, float* ms, int* launches) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (index < 0 || index >= static_cast<int>(g_prof.size()))
    return fail(STL_ERR_INDEX, "profile record %d out of range", index);
  const ProfRec& rec = g_prof[index];
  if (name) *name = rec.name;
  if (launches) *launches = rec.launches;
  if (ms) {
    float v = 0.f;
    if (int st = check_cuda(cudaEventElapsedTime(&v, rec.a, rec.b), "profile elapsed")) return st;
    *ms = v;
  }
  return STL_OK;
}

}  // extern "C"
