// ks_internal.h -- host-side internals shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <mutex>
#include <string>

#include "../../include/ks.h"

namespace ks {

void set_error(const std::string& msg);

// Status helper: records a message and returns the code.
inline ks_status fail(ks_status code, const std::string& msg) { set_error(msg); return code; }

#define KS_CUDA_TRY(expr)                                                                    \
  do {                                                                                       \
    cudaError_t e__ = (expr);                                                                \
    if (e__ != cudaSuccess)                                                                  \
      return ::ks::fail(KS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e__));   \
  } while (0)

void count_launch();
void add_launches(uint64_t n);   // kernels of a replayed CUDA graph

// After every <<<...>>> launch: count it (ks_launch_count) and check the launch error.
#define KS_LAUNCH_CHECK()                \
  do {                                   \
    ::ks::count_launch();                \
    KS_CUDA_TRY(cudaGetLastError());     \
  } while (0)

// Per-device state: every cached answer / one-time setup is keyed by the CURRENT device (a process may
// drive several GPUs, from several host threads).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

// Streaming multiprocessors of the current device (persistent-grid sizing), cached per device.
inline int num_sms() {
  static std::atomic<int> cache[kMaxDevices];
  const int dev = current_device();
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

// One-time per-device setup (e.g. cudaFuncSetAttribute, which is per device): runs f() once for each
// device it is called on; thread-safe (a failed f() is retried on the next call).
struct PerDeviceOnce {
  std::atomic<bool> done[kMaxDevices];
  std::mutex mu;
  template <class F>
  ks_status run(F&& f) {
    const int dev = current_device();
    if (done[dev].load(std::memory_order_acquire)) return KS_OK;
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev].load(std::memory_order_relaxed)) return KS_OK;
    const ks_status s = f();
    if (s == KS_OK) done[dev].store(true, std::memory_order_release);
    return s;
  }
};

#define KS_TRY(expr)                     \
  do {                                   \
    ks_status s__ = (expr);              \
    if (s__ != KS_OK) return s__;        \
  } while (0)

// ---------------------------------------------------------------- sketch side
constexpr int kSrhtB = 512;         // SRHT chunk length (columns of K per transform block)
constexpr int kSrhtRows = 8;        // rows of Y per sketch CTA (128 threads, 4 CTAs per SM)
constexpr int kGaussBM = 128;       // rows per tcgen05 tile
constexpr int kGaussBK = 64;        // reduction (j) block per pipeline stage

struct SketchLayout {
  int64_t N;          // 2^ceil(log2 n)
  int64_t ncols_pad;  // packed-point count (multiple of the chunk length)
  int A;              // number of kSrhtB-chunks covering [0, n) (Omega-apply)
  int tpo;            // SRHT sketch: outputs per thread in the gather phase
  int d_pad;          // SRHT sketch: output slots, 64 * tpo (slot -> output by the perm table)
  size_t off_pk, off_tab, off_sel, off_bucket_ofs, off_bucket_idx, off_bitmap, off_gauss, off_perm, off_sgn, off_ybuf, bytes;
};

ks_status sketch_validate(const ks_sketch_desc* desc);
// Gaussian path: K is generated pre-multiplied by S = 2^floor(log2(2^14 / (sigma2 + nugget))) so that
// its fp16 hi/lo split stays in fp16's normal range (max S*K = 2^14); Y is divided by S at the end.
double gauss_scale(const ks_sketch_desc& desc);
SketchLayout sketch_layout(const ks_sketch_desc& desc);
// Fill the workspace with this desc's randomness (packed points need pts).
ks_status sketch_prepare(const ks_sketch_desc& desc, const SketchLayout& L, const float* pts, char* ws,
                         cudaStream_t st, bool need_points);
// A stored K (NEXT-2): row-major fp32, K[i][j] at K[i * ldk + j].
struct StoredK {
  const float* K;
  int64_t ldk;
};
ks_status sketch_run(const ks_sketch_desc& desc, const SketchLayout& L, int64_t row_begin, int64_t row_end,
                     float* Y, char* ws, cudaStream_t st, const StoredK* sk = nullptr);
ks_status omega_apply_run(const ks_sketch_desc& desc, const SketchLayout& L, const float* Z, int m,
                          int64_t row_begin, int64_t row_end, float* X, char* ws, cudaStream_t st);
ks_status omega_export_run(const ks_sketch_desc& desc, const SketchLayout& L, int8_t* signs, int32_t* sel,
                           uint16_t* gauss, char* ws, cudaStream_t st);
ks_status gauss_sketch_run(const ks_sketch_desc& desc, const SketchLayout& L, int64_t row_begin,
                           int64_t row_end, float* Y, char* ws, cudaStream_t st, const StoredK* sk);

// NEXT-4: W = K Om for a dense given Om (n x d, row-major), workspace dense_apply_ws(desc)
ks_status dense_apply_run(const ks_sketch_desc& D, const float* pts, const float* Om, float* W, char* ws,
                          cudaStream_t st);
size_t dense_apply_ws(const ks_sketch_desc& D);

// ---------------------------------------------------------------- TSQR
// Plans replay their launch sequence as a cached CUDA graph; one-shot plans switch that off.
void tsqr_set_graphs(ks_tsqr_handle h, bool on);
// ks_tsqr_create with the plan metadata uploaded stream-ordered on st (one-shot plans).
ks_status tsqr_create_on_stream(int64_t rows, int32_t d, int32_t blocks, void* ws, size_t ws_bytes,
                                ks_tsqr_handle* out, cudaStream_t st, int32_t topology = KS_TSQR_TREE);

// ---------------------------------------------------------------- solve side
// NEXT-4 (ks_gp.cu)
ks_status cond_diag_ws(int64_t rows, int d, size_t* bytes);
ks_status cond_gram_run(const float* Y, int64_t rows, int d, const float* R, float* G, char* ws, cudaStream_t st);
ks_status cond_from_gram_run(const float* G, int d, float* out, float* V, cudaStream_t st);
size_t cond_from_gram_ws(int d);
ks_status cond_diag_run(const float* Y, int64_t rows, int d, const float* R, float* out, char* ws, cudaStream_t st);
ks_status gp_ws(int64_t rows, int r, int q, size_t* bytes);
ks_status gp_woodbury_run(const float* U, int64_t rows, int r, const float* lam, float s2, const float* B, int q,
                          float* X, char* ws, cudaStream_t st);
ks_status gp_loglik_run(const float* U, int64_t rows, int r, const float* lam, float s2, const float* y, double* out,
                        char* ws, cudaStream_t st);
ks_status nystrom_ws(const ks_sketch_desc& D, size_t* bytes);
ks_status nystrom_run(const ks_sketch_desc& D, const float* pts, const float* Q, float* W, float* B, char* ws,
                      cudaStream_t st);
ks_status gp_core_ws(int64_t rows, int d, int q, size_t* bytes);
ks_status gp_loglik_core_run(const float* Q, int64_t rows, int d, const float* B, float s2, const float* y, double* out,
                             char* ws, cudaStream_t st);
ks_status gp_woodbury_core_run(const float* Q, int64_t rows, int d, const float* B, float s2, const float* X, int q,
                               float* Z, char* ws, cudaStream_t st);
ks_status apply_qt_ws(int64_t rows, int d, int m, size_t* bytes);
ks_status apply_qt_run(const float* Q, int64_t rows, int d, const float* X, int m, float* C, void* ws,
                       cudaStream_t st);
// X = Q C, or X = alpha B + beta Q C when B != nullptr (any m).
ks_status apply_q_run(const float* Q, int64_t rows, int d, const float* C, int m, float* X, cudaStream_t st,
                      const float* B = nullptr, float alpha = 0.f, float beta = 1.f);
ks_status trsolve_run(const float* R, const float* C, int d, int m, float tau, float* Z, int32_t* k,
                      cudaStream_t st);

}  // namespace ks
