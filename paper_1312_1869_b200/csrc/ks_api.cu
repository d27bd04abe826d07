// ks_api.cu -- C-ABI entry points (include/ks.h) for the sketch and the solve.
// The TSQR entry points live in ks_tsqr.cu.  No C++ exception crosses this boundary.
#include "ks_common.cuh"
#include "ks_internal.h"

#include <cmath>
#include <string>

#include <atomic>

namespace ks {
static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};
void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace ks

extern "C" uint64_t ks_launch_count(void) { return ks::g_launches.load(); }

using namespace ks;

static cudaStream_t S(ks_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

static ks_status check_rows(const ks_sketch_desc* desc, int64_t rb, int64_t re) {
  if (rb < 0 || re < rb || re > desc->n) return fail(KS_ERR_INVALID_ARGUMENT, "need 0 <= row_begin <= row_end <= n");
  return KS_OK;
}

#define KS_GUARD_BEGIN try {
#define KS_GUARD_END                                                         \
  }                                                                          \
  catch (const std::exception& e) { return fail(KS_ERR_CUDA, e.what()); }    \
  catch (...) { return fail(KS_ERR_CUDA, "unknown C++ exception"); }

extern "C" const char* ks_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* ks_version(void) { return "ks-b200 0.1.0 (sm_100a)"; }

extern "C" ks_status ks_sketch_workspace_size(const ks_sketch_desc* desc, size_t* bytes) {
  KS_GUARD_BEGIN
  KS_TRY(sketch_validate(desc));
  if (!bytes) return fail(KS_ERR_INVALID_ARGUMENT, "bytes is NULL");
  *bytes = sketch_layout(*desc).bytes;
  return KS_OK;
  KS_GUARD_END
}

extern "C" ks_status ks_sketch(const ks_sketch_desc* desc, const float* pts, int64_t rb, int64_t re, float* Y,
                               void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  KS_TRY(sketch_validate(desc));
  KS_TRY(check_rows(desc, rb, re));
  if (!pts || !ws || (re > rb && !Y)) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if ((reinterpret_cast<uintptr_t>(Y) & 15) != 0) return fail(KS_ERR_INVALID_ARGUMENT, "Y must be 16-byte aligned");
  const SketchLayout L = sketch_layout(*desc);
  if (ws_bytes < L.bytes) return fail(KS_ERR_OOM, "sketch workspace too small: need " + std::to_string(L.bytes));
  char* w = static_cast<char*>(ws);
  KS_TRY(sketch_prepare(*desc, L, pts, w, S(stream), true));
  return sketch_run(*desc, L, rb, re, Y, w, S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_sketch_stored(const ks_sketch_desc* desc, const float* K, int64_t ldk, int64_t rb, int64_t re,
                                      float* Y, void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  if (!desc) return fail(KS_ERR_INVALID_ARGUMENT, "desc is NULL");
  if (desc->kernel != KS_KERNEL_STORED) return fail(KS_ERR_INVALID_ARGUMENT, "ks_sketch_stored needs KS_KERNEL_STORED");
  KS_TRY(sketch_validate(desc));
  KS_TRY(check_rows(desc, rb, re));
  if (!K || !ws || (re > rb && !Y)) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if ((reinterpret_cast<uintptr_t>(Y) & 15) != 0) return fail(KS_ERR_INVALID_ARGUMENT, "Y must be 16-byte aligned");
  if (ldk < desc->n || (ldk & 3) != 0 || (reinterpret_cast<uintptr_t>(K) & 15) != 0)
    return fail(KS_ERR_INVALID_ARGUMENT, "need ldk >= n, ldk % 4 == 0 and a 16-byte aligned K");
  const SketchLayout L = sketch_layout(*desc);
  if (ws_bytes < L.bytes) return fail(KS_ERR_OOM, "sketch workspace too small: need " + std::to_string(L.bytes));
  char* w = static_cast<char*>(ws);
  KS_TRY(sketch_prepare(*desc, L, nullptr, w, S(stream), true));
  const StoredK sk{K, ldk};
  return sketch_run(*desc, L, rb, re, Y, w, S(stream), &sk);
  KS_GUARD_END
}

extern "C" ks_status ks_omega_export(const ks_sketch_desc* desc, int8_t* signs, int32_t* sel, uint16_t* gauss,
                                     void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  KS_TRY(sketch_validate(desc));
  if (!ws) return fail(KS_ERR_INVALID_ARGUMENT, "workspace is NULL");
  const SketchLayout L = sketch_layout(*desc);
  if (ws_bytes < L.bytes) return fail(KS_ERR_OOM, "sketch workspace too small: need " + std::to_string(L.bytes));
  char* w = static_cast<char*>(ws);
  KS_TRY(sketch_prepare(*desc, L, nullptr, w, S(stream), false));
  return omega_export_run(*desc, L, signs, sel, gauss, w, S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_omega_apply(const ks_sketch_desc* desc, const float* Z, int32_t m, int64_t rb, int64_t re,
                                    float* X, void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  KS_TRY(sketch_validate(desc));
  KS_TRY(check_rows(desc, rb, re));
  if (m < 1 || m > 64) return fail(KS_ERR_UNSUPPORTED, "need 1 <= m <= 64");
  if (!Z || !ws || (re > rb && !X)) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  const SketchLayout L = sketch_layout(*desc);
  if (ws_bytes < L.bytes) return fail(KS_ERR_OOM, "sketch workspace too small: need " + std::to_string(L.bytes));
  char* w = static_cast<char*>(ws);
  KS_TRY(sketch_prepare(*desc, L, nullptr, w, S(stream), false));
  return omega_apply_run(*desc, L, Z, m, rb, re, X, w, S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_apply_qt_workspace_size(int64_t rows, int32_t d, int32_t m, size_t* bytes) {
  if (!bytes || rows < 1 || d < 1 || m < 1) return fail(KS_ERR_INVALID_ARGUMENT, "invalid argument");
  if (m > 64) return fail(KS_ERR_UNSUPPORTED, "need m <= 64");
  return apply_qt_ws(rows, d, m, bytes);
}

extern "C" ks_status ks_apply_qt(const float* Q, int64_t rows, int32_t d, const float* X, int32_t m, float* C,
                                 void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  size_t need = 0;
  KS_TRY(ks_apply_qt_workspace_size(rows, d, m, &need));
  if (!Q || !X || !C || !ws) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (ws_bytes < need) return fail(KS_ERR_OOM, "apply_qt workspace too small: need " + std::to_string(need));
  return apply_qt_run(Q, rows, d, X, m, C, ws, S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_apply_q(const float* Q, int64_t rows, int32_t d, const float* C, int32_t m, float* X,
                                ks_stream_t stream) {
  KS_GUARD_BEGIN
  if (!Q || !C || !X || rows < 1 || d < 1 || m < 1) return fail(KS_ERR_INVALID_ARGUMENT, "invalid argument");
  if (m > 64) return fail(KS_ERR_UNSUPPORTED, "need m <= 64");
  return apply_q_run(Q, rows, d, C, m, X, S(stream));
  KS_GUARD_END
}

// ------------------------------------------------------------------ NEXT-4
extern "C" ks_status ks_cond_diag_workspace_size(int64_t rows, int32_t d, size_t* bytes) {
  if (!bytes || rows < 1 || d < 1 || d > 1024) return fail(KS_ERR_INVALID_ARGUMENT, "need rows >= 1, 1 <= d <= 1024");
  return cond_diag_ws(rows, d, bytes);
}

static ks_status cond_check(const float* Y, int64_t rows, int32_t d, const float* R, const void* out, void* ws,
                            size_t ws_bytes) {
  size_t need = 0;
  KS_TRY(ks_cond_diag_workspace_size(rows, d, &need));
  if (!Y || !R || !out || !ws) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (ws_bytes < need) return fail(KS_ERR_OOM, "cond workspace too small: need " + std::to_string(need));
  return KS_OK;
}

extern "C" ks_status ks_cond_diag(const float* Y, int64_t rows, int32_t d, const float* R, float* out, void* ws,
                                  size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  KS_TRY(cond_check(Y, rows, d, R, out, ws, ws_bytes));
  return cond_diag_run(Y, rows, d, R, out, static_cast<char*>(ws), S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_cond_gram(const float* Y, int64_t rows, int32_t d, const float* R, float* G, void* ws,
                                  size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  KS_TRY(cond_check(Y, rows, d, R, G, ws, ws_bytes));
  return cond_gram_run(Y, rows, d, R, G, static_cast<char*>(ws), S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_cond_from_gram(const float* G, int32_t d, float* out, void* ws, size_t ws_bytes,
                                       ks_stream_t stream) {
  KS_GUARD_BEGIN
  if (!G || !out || !ws || d < 1 || d > 1024) return fail(KS_ERR_INVALID_ARGUMENT, "invalid argument");
  if (ws_bytes < cond_from_gram_ws(d))
    return fail(KS_ERR_OOM, "cond workspace too small: need " + std::to_string(cond_from_gram_ws(d)));
  return cond_from_gram_run(G, d, out, static_cast<float*>(ws), S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_gp_workspace_size(int64_t rows, int32_t r, int32_t q, size_t* bytes) {
  if (!bytes || rows < 1 || r < 1 || q < 1) return fail(KS_ERR_INVALID_ARGUMENT, "need rows, r, q >= 1");
  return gp_ws(rows, r, q, bytes);
}

extern "C" ks_status ks_gp_woodbury_solve(const float* U, int64_t rows, int32_t r, const float* lam, float sigma2,
                                          const float* B, int32_t q, float* X, void* ws, size_t ws_bytes,
                                          ks_stream_t stream) {
  KS_GUARD_BEGIN
  size_t need = 0;
  KS_TRY(ks_gp_workspace_size(rows, r, q, &need));
  if (!U || !lam || !B || !X || !ws) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (!(sigma2 > 0.f) || !std::isfinite(sigma2)) return fail(KS_ERR_INVALID_ARGUMENT, "sigma2 must be > 0");
  if (X == B) return fail(KS_ERR_INVALID_ARGUMENT, "X may not alias B");
  if (ws_bytes < need) return fail(KS_ERR_OOM, "gp workspace too small: need " + std::to_string(need));
  return gp_woodbury_run(U, rows, r, lam, sigma2, B, q, X, static_cast<char*>(ws), S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_gp_loglik(const float* U, int64_t rows, int32_t r, const float* lam, float sigma2,
                                  const float* y, double* out, void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  size_t need = 0;
  KS_TRY(ks_gp_workspace_size(rows, r, 1, &need));
  if (!U || !lam || !y || !out || !ws) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (!(sigma2 > 0.f) || !std::isfinite(sigma2)) return fail(KS_ERR_INVALID_ARGUMENT, "sigma2 must be > 0");
  if (ws_bytes < need) return fail(KS_ERR_OOM, "gp workspace too small: need " + std::to_string(need));
  return gp_loglik_run(U, rows, r, lam, sigma2, y, out, static_cast<char*>(ws), S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_trsolve(const float* R, const float* C, int32_t d, int32_t m, float tau, float* Z,
                                int32_t* k_dev, ks_stream_t stream) {
  KS_GUARD_BEGIN
  if (!R || !C || !Z || d < 1 || m < 1) return fail(KS_ERR_INVALID_ARGUMENT, "invalid argument");
  if (d > 512 || m > 64) return fail(KS_ERR_UNSUPPORTED, "need d <= 512, m <= 64");
  if (!(tau >= 0.f) || !std::isfinite(tau)) return fail(KS_ERR_INVALID_ARGUMENT, "tau must be >= 0");
  if (tau == 0.f && !k_dev) return fail(KS_ERR_INVALID_ARGUMENT, "strict solve (tau == 0) needs k_dev");
  KS_TRY(trsolve_run(R, C, d, m, tau, Z, k_dev, S(stream)));
  if (tau == 0.f) {
    int32_t k = 0;
    KS_CUDA_TRY(cudaMemcpyAsync(&k, k_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, S(stream)));
    KS_CUDA_TRY(cudaStreamSynchronize(S(stream)));
    if (k < 0)
      return fail(KS_ERR_SINGULAR, "singular R: |r_jj| <= 1e-12 max|r_ii| at index " + std::to_string(-k - 1));
  }
  return KS_OK;
  KS_GUARD_END
}

// ---------------------------------------------------------------- NEXT-4: Nystrom core + core likelihood
extern "C" ks_status ks_nystrom_workspace_size(const ks_sketch_desc* desc, size_t* bytes) {
  KS_GUARD_BEGIN
  if (!desc || !bytes) return fail(KS_ERR_INVALID_ARGUMENT, "NULL argument");
  ks_sketch_desc D = *desc;
  D.omega = KS_OMEGA_DHT;
  KS_TRY(sketch_validate(&D));
  return nystrom_ws(D, bytes);
  KS_GUARD_END
}

extern "C" ks_status ks_nystrom_core(const ks_sketch_desc* desc, const float* pts, const float* Q, float* W, float* B,
                                     void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  if (!desc) return fail(KS_ERR_INVALID_ARGUMENT, "desc is NULL");
  ks_sketch_desc D = *desc;
  D.omega = KS_OMEGA_DHT;   // (Omega is the given Q; the desc's omega field is ignored)
  if (D.kernel == KS_KERNEL_STORED) return fail(KS_ERR_UNSUPPORTED, "ks_nystrom_core evaluates K from points");
  KS_TRY(sketch_validate(&D));
  if (!pts || !Q || !W || !B || !ws) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(W)) & 15) != 0)
    return fail(KS_ERR_INVALID_ARGUMENT, "Q and W must be 16-byte aligned");
  size_t need = 0;
  KS_TRY(nystrom_ws(D, &need));
  if (ws_bytes < need) return fail(KS_ERR_OOM, "nystrom workspace too small: need " + std::to_string(need));
  return nystrom_run(D, pts, Q, W, B, static_cast<char*>(ws), S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_gp_core_workspace_size(int64_t rows, int32_t d, int32_t q, size_t* bytes) {
  KS_GUARD_BEGIN
  if (!bytes || rows < 1 || d < 1 || q < 1) return fail(KS_ERR_INVALID_ARGUMENT, "invalid argument");
  return gp_core_ws(rows, d, q, bytes);
  KS_GUARD_END
}

static ks_status core_check(const float* Q, int64_t rows, int32_t d, const float* B, float s2, const float* X,
                            int32_t q, size_t ws_bytes, const void* ws) {
  if (!Q || !B || !X || !ws || rows < 1 || d < 1 || q < 1) return fail(KS_ERR_INVALID_ARGUMENT, "invalid argument");
  if (d > 256 || q > 64) return fail(KS_ERR_UNSUPPORTED, "need d <= 256, q <= 64");
  if (!(s2 > 0.f) || !std::isfinite(s2)) return fail(KS_ERR_INVALID_ARGUMENT, "sigma2 must be > 0");
  size_t need = 0;
  KS_TRY(gp_core_ws(rows, d, q, &need));
  if (ws_bytes < need) return fail(KS_ERR_OOM, "gp core workspace too small: need " + std::to_string(need));
  return KS_OK;
}

extern "C" ks_status ks_gp_loglik_core(const float* Q, int64_t rows, int32_t d, const float* B, float sigma2,
                                       const float* y, double* out, void* ws, size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  KS_TRY(core_check(Q, rows, d, B, sigma2, y, 1, ws_bytes, ws));
  if (!out) return fail(KS_ERR_INVALID_ARGUMENT, "out is NULL");
  return gp_loglik_core_run(Q, rows, d, B, sigma2, y, out, static_cast<char*>(ws), S(stream));
  KS_GUARD_END
}

extern "C" ks_status ks_gp_woodbury_core(const float* Q, int64_t rows, int32_t d, const float* B, float sigma2,
                                         const float* X, int32_t q, float* Z, void* ws, size_t ws_bytes,
                                         ks_stream_t stream) {
  KS_GUARD_BEGIN
  KS_TRY(core_check(Q, rows, d, B, sigma2, X, q, ws_bytes, ws));
  if (!Z || Z == X) return fail(KS_ERR_INVALID_ARGUMENT, "Z is NULL or aliases X");
  return gp_woodbury_core_run(Q, rows, d, B, sigma2, X, q, Z, static_cast<char*>(ws), S(stream));
  KS_GUARD_END
}

// ---------------------------------------------------------------- one-shot
namespace {
struct LowrankLayout {
  size_t off_sk, off_Y, off_Q, off_R, off_C, off_qt, off_tsqr, bytes;
};
ks_status lowrank_layout(const ks_sketch_desc* desc, int32_t m, int32_t blocks, LowrankLayout& L) {
  KS_TRY(sketch_validate(desc));
  if (m < 1 || m > 64) return fail(KS_ERR_UNSUPPORTED, "need 1 <= m <= 64");
  const int64_t n = desc->n;
  const int d = desc->d;
  size_t tsqr = 0, qt = 0;
  KS_TRY(ks_tsqr_workspace_size(n, d, blocks, &tsqr));
  KS_TRY(apply_qt_ws(n, d, m, &qt));
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  L.off_sk = take(sketch_layout(*desc).bytes);
  L.off_Y = take(sizeof(float) * (size_t)n * d);
  L.off_Q = take(sizeof(float) * (size_t)n * d);
  L.off_R = take(sizeof(float) * (size_t)d * d);
  L.off_C = take(sizeof(float) * (size_t)d * m);
  L.off_qt = take(qt);
  L.off_tsqr = take(tsqr);
  L.bytes = off;
  return KS_OK;
}
}  // namespace

extern "C" ks_status ks_lowrank_workspace_size(const ks_sketch_desc* desc, int32_t m, int32_t blocks, size_t* bytes) {
  KS_GUARD_BEGIN
  if (!bytes) return fail(KS_ERR_INVALID_ARGUMENT, "bytes is NULL");
  LowrankLayout L;
  KS_TRY(lowrank_layout(desc, m, blocks, L));
  *bytes = L.bytes;
  return KS_OK;
  KS_GUARD_END
}

extern "C" ks_status ks_lowrank_solve(const ks_sketch_desc* desc, const float* pts, const float* A, int32_t m,
                                      int32_t blocks, float tau, float* X, float* Z, int32_t* k_dev, void* ws,
                                      size_t ws_bytes, ks_stream_t stream) {
  KS_GUARD_BEGIN
  LowrankLayout L;
  KS_TRY(lowrank_layout(desc, m, blocks, L));
  if (!pts || !A || !X || !Z || !ws) return fail(KS_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (!(tau >= 0.f) || !std::isfinite(tau)) return fail(KS_ERR_INVALID_ARGUMENT, "tau must be >= 0");
  if (!k_dev) return fail(KS_ERR_INVALID_ARGUMENT, "k_dev is NULL (the truncation rank is the caller's signal)");
  if (ws_bytes < L.bytes) return fail(KS_ERR_OOM, "lowrank workspace too small: need " + std::to_string(L.bytes));
  char* w = static_cast<char*>(ws);
  const int64_t n = desc->n;
  const int d = desc->d;
  size_t sk = sketch_layout(*desc).bytes, tsqr = 0, qt = 0;
  ks_tsqr_workspace_size(n, d, blocks, &tsqr);
  apply_qt_ws(n, d, m, &qt);
  float* Y = reinterpret_cast<float*>(w + L.off_Y);
  float* Q = reinterpret_cast<float*>(w + L.off_Q);
  float* R = reinterpret_cast<float*>(w + L.off_R);
  float* C = reinterpret_cast<float*>(w + L.off_C);
  KS_TRY(ks_sketch(desc, pts, 0, n, Y, w + L.off_sk, sk, stream));
  ks_tsqr_handle h = nullptr;
  KS_TRY(tsqr_create_on_stream(n, d, blocks, w + L.off_tsqr, tsqr, &h, S(stream)));
  tsqr_set_graphs(h, false);   // one-shot plan: capturing a graph would not pay off
  ks_status s = ks_tsqr(h, Y, Q, R, stream);
  ks_tsqr_destroy(h);
  KS_TRY(s);
  KS_TRY(ks_apply_qt(Q, n, d, A, m, C, w + L.off_qt, qt, stream));
  KS_TRY(ks_trsolve(R, C, d, m, tau, Z, k_dev, stream));
  return omega_apply_run(*desc, sketch_layout(*desc), Z, m, 0, n, X, w + L.off_sk, S(stream));
  KS_GUARD_END
}
