// ks_gp.cu -- NEXT-4: what the low-rank factorisation is for ("evaluating a Gaussian type
// likelihood") and Theorem 5's stability diagnostic.
//
//   Theorem 5 diagnostic   c(K-hat R^{-1}) (reading L19: K-hat = K Omega = Y, the garbled c(K R_k^{-1}) of
//                          :364), X = Y R^{-1} (== Q-hat in exact arithmetic):
//                            k_rtrsm       X = Y R^{-1}, 32 rows per CTA, forward substitution over columns
//                            apply_qt_run  G = X^T X (deterministic split-K Gram)
//                            k_cond_lanczos the extreme eigenvalues of G - I (Lanczos, full
//                                          reorthogonalisation): cond = sqrt(l_max / l_min),
//                                          eps = ||G - I||_2, the Theorem's "(1 + eps) / (1 - eps)" form.
//   GP likelihood          zero-mean Gaussian with covariance U diag(lam) U^T + sigma2 I (U orthonormal,
//                          n x r), through the Woodbury identity and the determinant lemma:
//                            X  = (B - U diag(lam / (lam + sigma2)) U^T B) / sigma2
//                            ll = -1/2 [n log 2 pi + sum log(lam + sigma2) + (n - r) log sigma2 + y^T X(y)]
#include "ks_common.cuh"
#include "ks_internal.h"

#include <cmath>

namespace ks {

// Rt = R^T (square, d x d): column j of R becomes a contiguous row for k_rtrsm.
__global__ void k_transpose_sq(const float* __restrict__ R, int d, float* __restrict__ Rt) {
  __shared__ float t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8)
    if (by + i < d && bx + threadIdx.x < d) t[i][threadIdx.x] = R[(int64_t)(by + i) * d + bx + threadIdx.x];
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8)
    if (bx + i < d && by + threadIdx.x < d) Rt[(int64_t)(bx + i) * d + by + threadIdx.x] = t[threadIdx.x][i];
}

// X = Y R^{-1} (R upper triangular): row i solves x R = y by forward substitution over the columns,
// x_j = (y_j - sum_{l<j} x_l R_lj) / R_jj.  A CTA holds 32 rows in shared memory (leading dimension
// ld = 8 mod 32: the 4 rows of a warp hit distinct banks); 8 lanes per row split the dot product.
__global__ void __launch_bounds__(256) k_rtrsm(const float* __restrict__ Y, int64_t rows, int d, int ld,
                                               const float* __restrict__ Rt, float* __restrict__ X) {
  extern __shared__ float xs[];   // [32][ld]
  const int tid = threadIdx.x, r = tid >> 3, t8 = tid & 7;
  const int64_t row0 = (int64_t)blockIdx.x * 32;
  for (int p = tid; p < 32 * d; p += 256) {
    const int rr = p / d, j = p - rr * d;
    xs[rr * ld + j] = row0 + rr < rows ? Y[(row0 + rr) * d + j] : 0.f;
  }
  __syncthreads();
  float* xr = xs + r * ld;
  for (int j = 0; j < d; ++j) {
    const float* rc = Rt + (int64_t)j * d;   // R[0..d)[j]
    float s = 0.f;
    for (int l = t8; l < j; l += 8) s = fmaf(xr[l], __ldg(rc + l), s);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (t8 == 0) xr[j] = (xr[j] - s) / __ldg(rc + j);
    __syncwarp();
  }
  __syncthreads();
  for (int p = tid; p < 32 * d; p += 256) {
    const int rr = p / d, j = p - rr * d;
    if (row0 + rr < rows) X[(row0 + rr) * d + j] = xs[rr * ld + j];
  }
}

// The extreme eigenvalues of E = G - I (d <= 1024) by Lanczos with full reorthogonalisation (classical
// Gram-Schmidt, twice), K = min(d, 256) steps in one CTA; the basis lives in the workspace (K x d).  The
// extremes of the tridiagonal T_K (Sturm-count bisection, thread 0) converge first (Kaniel-Paige), also
// for the clustered spectra of a nearly orthonormal X.
constexpr int kLanczos = 256;
KS_DEVINL float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

// number of eigenvalues of the symmetric tridiagonal (a[0..k), b[1..k)) below x (Sturm sequence)
KS_DEVINL int sturm_count(const double* a, const double* b, int k, double x) {
  int c = 0;
  double q = 1.0;
  for (int i = 0; i < k; ++i) {
    q = a[i] - x - (i ? b[i] * b[i] / q : 0.0);
    if (q == 0.0) q = -1e-300;
    if (q < 0.0) ++c;
  }
  return c;
}

// out[0] = cond = sqrt(l_max / l_min) of G, out[1] = eps = ||G - I||_2, out[2] = l_min, out[3] = l_max.
__global__ void __launch_bounds__(1024) k_cond_lanczos(const float* __restrict__ G, int d, float* __restrict__ V,
                                                       float* __restrict__ out) {
  extern __shared__ float ls[];   // w[d], c[kLanczos]
  __shared__ float red[32];
  __shared__ double al[kLanczos], be[kLanczos];
  __shared__ int kdone;
  float* w = ls;
  float* cf = ls + d;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int K = min(d, kLanczos);
  // v_0: deterministic start, normalised
  float nn = 0.f;
  for (int i = tid; i < d; i += blockDim.x) {
    const float x = 1.f + 0.5f * __sinf(0.7f * (float)i + 0.3f);
    V[i] = x;
    nn = fmaf(x, x, nn);
  }
  nn = block_sum(nn, red);
  for (int i = tid; i < d; i += blockDim.x) V[i] *= rsqrtf(nn);
  if (tid == 0) kdone = K;
  __syncthreads();
  for (int k = 0; k < K; ++k) {
    const float* vk = V + (int64_t)k * d;
    for (int i = wid; i < d; i += nw) {   // w = (G - I) v_k
      const float* g = G + (int64_t)i * d;
      float sacc = 0.f;
      for (int j = lane; j < d; j += 32) sacc = fmaf(__ldg(g + j), vk[j], sacc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
      if (lane == 0) w[i] = sacc - vk[i];
    }
    __syncthreads();
    float a = 0.f;
    for (int i = tid; i < d; i += blockDim.x) a = fmaf(w[i], vk[i], a);
    a = block_sum(a, red);
    if (tid == 0) al[k] = a;
    for (int pass = 0; pass < 2; ++pass) {   // w -= V_{0..k} (V_{0..k}^T w), twice
      for (int m = wid; m <= k; m += nw) {
        const float* vm = V + (int64_t)m * d;
        float sacc = 0.f;
        for (int j = lane; j < d; j += 32) sacc = fmaf(vm[j], w[j], sacc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (lane == 0) cf[m] = sacc;
      }
      __syncthreads();
      for (int i = tid; i < d; i += blockDim.x) {
        float x = w[i];
        for (int m = 0; m <= k; ++m) x = fmaf(-cf[m], V[(int64_t)m * d + i], x);
        w[i] = x;
      }
      __syncthreads();
    }
    float bb = 0.f;
    for (int i = tid; i < d; i += blockDim.x) bb = fmaf(w[i], w[i], bb);
    bb = block_sum(bb, red);
    const float bnorm = sqrtf(bb);
    if (k + 1 < K) {
      if (tid == 0) be[k + 1] = bnorm;
      if (!(bnorm > 1e-30f)) {   // invariant subspace: T_{k+1} holds the spectrum seen from v_0
        if (tid == 0) kdone = k + 1;
        break;
      }
      float* vn = V + (int64_t)(k + 1) * d;
      for (int i = tid; i < d; i += blockDim.x) vn[i] = w[i] / bnorm;
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    const int k = kdone;
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < k; ++i) {   // Gershgorin interval of T_k
      const double r = (i ? fabs(be[i]) : 0.0) + (i + 1 < k ? fabs(be[i + 1]) : 0.0);
      lo = fmin(lo, al[i] - r);
      hi = fmax(hi, al[i] + r);
    }
    double a0 = lo, a1 = hi, b0 = lo, b1 = hi;
    for (int it = 0; it < 100; ++it) {   // smallest: count(x) >= 1 ; largest: count(x) >= k
      const double m0 = 0.5 * (a0 + a1), m1 = 0.5 * (b0 + b1);
      if (sturm_count(al, be, k, m0) >= 1) a1 = m0; else a0 = m0;
      if (sturm_count(al, be, k, m1) >= k) b1 = m1; else b0 = m1;
    }
    const double emin = 0.5 * (a0 + a1), emax = 0.5 * (b0 + b1);
    out[0] = (float)sqrt((1.0 + emax) / (1.0 + emin));
    out[1] = (float)fmax(fabs(emin), fabs(emax));
    out[2] = (float)(1.0 + emin);
    out[3] = (float)(1.0 + emax);
  }
}

struct CondLayout {
  size_t off_rt, off_x, off_g, off_qt, off_v, bytes;
};
static CondLayout cond_layout(int64_t rows, int d) {
  CondLayout L{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  L.off_rt = take(sizeof(float) * (size_t)d * d);
  L.off_x = take(sizeof(float) * (size_t)rows * d);
  L.off_g = take(sizeof(float) * (size_t)d * d);
  size_t qt = 0;
  apply_qt_ws(rows, d, d, &qt);
  L.off_qt = take(qt);
  L.off_v = take(sizeof(float) * (size_t)kLanczos * d);
  L.bytes = off;
  return L;
}

ks_status cond_diag_ws(int64_t rows, int d, size_t* bytes) {
  *bytes = cond_layout(rows, d).bytes;
  return KS_OK;
}

ks_status cond_gram_run(const float* Y, int64_t rows, int d, const float* R, float* G, char* ws, cudaStream_t st) {
  const CondLayout L = cond_layout(rows, d);
  float* Rt = reinterpret_cast<float*>(ws + L.off_rt);
  float* X = reinterpret_cast<float*>(ws + L.off_x);
  k_transpose_sq<<<dim3((unsigned)((d + 31) / 32), (unsigned)((d + 31) / 32)), dim3(32, 8), 0, st>>>(R, d, Rt);
  KS_LAUNCH_CHECK();
  const int ld = d + ((8 - d % 32) % 32 + 32) % 32;
  const int smem = 32 * ld * (int)sizeof(float);
  KS_CUDA_TRY(cudaFuncSetAttribute(k_rtrsm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_rtrsm<<<(unsigned)((rows + 31) / 32), 256, smem, st>>>(Y, rows, d, ld, Rt, X);
  KS_LAUNCH_CHECK();
  return apply_qt_run(X, rows, d, X, d, G, ws + L.off_qt, st);
}

size_t cond_from_gram_ws(int d) { return sizeof(float) * (size_t)kLanczos * d; }

ks_status cond_from_gram_run(const float* G, int d, float* out, float* V, cudaStream_t st) {
  const int smem = (d + kLanczos) * (int)sizeof(float);
  k_cond_lanczos<<<1, 1024, smem, st>>>(G, d, V, out);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

ks_status cond_diag_run(const float* Y, int64_t rows, int d, const float* R, float* out, char* ws, cudaStream_t st) {
  const CondLayout L = cond_layout(rows, d);
  float* G = reinterpret_cast<float*>(ws + L.off_g);
  KS_TRY(cond_gram_run(Y, rows, d, R, G, ws, st));
  return cond_from_gram_run(G, d, out, reinterpret_cast<float*>(ws + L.off_v), st);
}

// ------------------------------------------------------------------ GP likelihood (Woodbury)
// C'[a][c] = lam_a / (lam_a + sigma2) * C[a][c]
__global__ void k_woodbury_weights(float* __restrict__ C, const float* __restrict__ lam, int r, int q, float s2) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= r * q) return;
  const float l = lam[p / q];
  C[p] *= l / (l + s2);
}

// Per-block fp64 partial sums of y . x; the last block (ticket) adds them in block order (deterministic)
// and writes out = {loglik, y^T Sigma^{-1} y, log det Sigma}.
__global__ void __launch_bounds__(256) k_loglik(const float* __restrict__ y, const float* __restrict__ x, int64_t n,
                                                const float* __restrict__ lam, int r, float s2,
                                                double* __restrict__ part, unsigned* __restrict__ ticket,
                                                double* __restrict__ out) {
  __shared__ double red[8];
  __shared__ bool last;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    s = fma((double)y[i], (double)x[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < 8; ++w) b += red[w];
    part[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double quad = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) quad += ((volatile double*)part)[b];
  double ld = (double)(n - r) * log((double)s2);
  for (int a = 0; a < r; ++a) ld += log((double)lam[a] + (double)s2);
  out[0] = -0.5 * ((double)n * log(2.0 * 3.14159265358979323846) + ld + quad);
  out[1] = quad;
  out[2] = ld;
  *ticket = 0u;
}

struct GpLayout {
  size_t off_c, off_qt, off_x, off_part, off_ticket, bytes;
};
static constexpr int kLlBlocks = 296;
static GpLayout gp_layout(int64_t rows, int r, int q) {
  GpLayout L{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  L.off_c = take(sizeof(float) * (size_t)r * q);
  size_t qt = 0;
  apply_qt_ws(rows, r, q, &qt);
  L.off_qt = take(qt);
  L.off_x = take(sizeof(float) * (size_t)rows);
  L.off_part = take(sizeof(double) * kLlBlocks);
  L.off_ticket = take(sizeof(unsigned));
  L.bytes = off;
  return L;
}

ks_status gp_ws(int64_t rows, int r, int q, size_t* bytes) {
  *bytes = gp_layout(rows, r, q).bytes;
  return KS_OK;
}

ks_status gp_woodbury_run(const float* U, int64_t rows, int r, const float* lam, float s2, const float* B, int q,
                          float* X, char* ws, cudaStream_t st) {
  const GpLayout L = gp_layout(rows, r, q);
  float* C = reinterpret_cast<float*>(ws + L.off_c);
  KS_TRY(apply_qt_run(U, rows, r, B, q, C, ws + L.off_qt, st));   // C = U^T B
  k_woodbury_weights<<<(unsigned)((r * q + 255) / 256), 256, 0, st>>>(C, lam, r, q, s2);
  KS_LAUNCH_CHECK();
  return apply_q_run(U, rows, r, C, q, X, st, B, 1.f / s2, -1.f / s2);   // X = (B - U C') / s2
}

ks_status gp_loglik_run(const float* U, int64_t rows, int r, const float* lam, float s2, const float* y, double* out,
                        char* ws, cudaStream_t st) {
  const GpLayout L = gp_layout(rows, r, 1);
  float* x = reinterpret_cast<float*>(ws + L.off_x);
  KS_TRY(gp_woodbury_run(U, rows, r, lam, s2, y, 1, x, ws, st));
  unsigned* ticket = reinterpret_cast<unsigned*>(ws + L.off_ticket);
  KS_CUDA_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
  k_loglik<<<kLlBlocks, 256, 0, st>>>(y, x, rows, lam, r, s2, reinterpret_cast<double*>(ws + L.off_part), ticket,
                                      out);
  KS_LAUNCH_CHECK();
  return KS_OK;
}


// ------------------------------------------------------------------ NEXT-4: the Nystrom core and its likelihood
// K ~ Q B Q^T with B = Q^T K Q (PAPER.md:25's "approximate spectral decompositions", HM11 Alg. 5.3): W = K Q
// is a second fused pass over K on the tensor cores (dense_apply_run), B = Q^T W by the deterministic split-K
// Q^T-apply, then symmetrised.
__global__ void k_symmetrize(float* __restrict__ B, int d) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= d * d) return;
  const int i = p / d, j = p - i * d;
  if (j <= i) return;
  const float v = 0.5f * (B[i * d + j] + B[j * d + i]);
  B[i * d + j] = v;
  B[j * d + i] = v;
}

struct NysLayout {
  size_t off_dense, off_qt, bytes;
};
static NysLayout nys_layout(const ks_sketch_desc& D) {
  NysLayout L{};
  size_t off = 0, qt = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  L.off_dense = take(dense_apply_ws(D));
  apply_qt_ws(D.n, D.d, D.d, &qt);
  L.off_qt = take(qt);
  L.bytes = off;
  return L;
}

ks_status nystrom_ws(const ks_sketch_desc& D, size_t* bytes) {
  *bytes = nys_layout(D).bytes;
  return KS_OK;
}

ks_status nystrom_run(const ks_sketch_desc& D, const float* pts, const float* Q, float* W, float* B, char* ws,
                      cudaStream_t st) {
  const NysLayout L = nys_layout(D);
  KS_TRY(dense_apply_run(D, pts, Q, W, ws + L.off_dense, st));
  KS_TRY(apply_qt_run(Q, D.n, D.d, W, D.d, B, ws + L.off_qt, st));
  k_symmetrize<<<(unsigned)((D.d * D.d + 255) / 256), 256, 0, st>>>(B, D.d);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

// One CTA (1024 threads), fp64: L L^T = B + s2 I by right-looking Cholesky in the workspace A (d x d, the
// lower triangle; L2-resident, column j broadcast through shared memory), then Z = (B + s2 I)^{-1} C for the
// q columns of C at once (forward / backward substitution, the right-hand sides in shared memory), and
//   out[0] = log det (B + s2 I) = 2 sum log l_jj,  out[1 + c] = C[:, c]^T C[:, c],  out[1 + q + c] = C[:, c]^T Z[:, c].
constexpr int kCholThreads = 1024;
constexpr int kCoreMaxD = 256, kCoreMaxQ = 64;
constexpr int kCoreSmem = (kCoreMaxD * kCoreMaxQ + kCoreMaxD + 64) * 8;
__global__ void __launch_bounds__(kCholThreads, 1)
k_core_chol_solve(const float* __restrict__ B, int d, float s2, double* __restrict__ A, const float* __restrict__ Cm,
                  int q, float* __restrict__ Z, double* __restrict__ out) {
  extern __shared__ double csm[];
  double* rs = csm;                       // [d][q] right-hand sides -> solutions
  double* col = rs + kCoreMaxD * kCoreMaxQ;
  double* red = col + kCoreMaxD;          // [64]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int p = tid; p < d * d; p += kCholThreads) {
    const int i = p / d, k = p - i * d;
    if (k <= i) A[p] = (double)B[p] + (i == k ? (double)s2 : 0.0);
  }
  __syncthreads();
  double logdet = 0.0;   // (thread 0)
  for (int j = 0; j < d; ++j) {
    if (tid == 0) {
      const double l = sqrt(A[j * d + j]);
      A[j * d + j] = l;
      col[j] = l;
      logdet += 2.0 * log(l);
    }
    __syncthreads();
    const double lj = col[j];
    for (int i = j + 1 + tid; i < d; i += kCholThreads) {
      const double v = A[i * d + j] / lj;
      A[i * d + j] = v;
      col[i] = v;
    }
    __syncthreads();
    for (int i = j + 1 + warp; i < d; i += kCholThreads / 32) {   // trailing update, row i by one warp
      const double ci = col[i];
      for (int k = j + 1 + lane; k <= i; k += 32) A[i * d + k] = fma(-ci, col[k], A[i * d + k]);
    }
    __syncthreads();
  }
  if (tid == 0) out[0] = logdet;
  for (int p = tid; p < d * q; p += kCholThreads) rs[p] = (double)Cm[p];
  __syncthreads();
  for (int j = 0; j < d; ++j) {   // forward: u_j = r_j / l_jj, then r_i -= l_ij u_j (i > j)
    const double ljj = A[j * d + j];
    for (int c = tid; c < q; c += kCholThreads) rs[j * q + c] /= ljj;
    __syncthreads();
    for (int p = tid; p < (d - j - 1) * q; p += kCholThreads) {
      const int i = j + 1 + p / q, c = p % q;
      rs[i * q + c] = fma(-A[i * d + j], rs[j * q + c], rs[i * q + c]);
    }
    __syncthreads();
  }
  for (int j = d - 1; j >= 0; --j) {   // backward: z_j = r_j / l_jj, then r_k -= l_jk z_j (k < j)
    const double ljj = A[j * d + j];
    for (int c = tid; c < q; c += kCholThreads) rs[j * q + c] /= ljj;
    __syncthreads();
    for (int p = tid; p < j * q; p += kCholThreads) {
      const int k = p / q, c = p % q;
      rs[k * q + c] = fma(-A[j * d + k], rs[j * q + c], rs[k * q + c]);
    }
    __syncthreads();
  }
  for (int p = tid; p < d * q; p += kCholThreads) Z[p] = (float)rs[p];
  // c^T c and c^T z per column, fixed-order block sums (warp shuffles, then the 32 warp sums)
  for (int c = 0; c < q; ++c) {
    for (int w = 0; w < 2; ++w) {
      double v = 0.0;
      for (int i = tid; i < d; i += kCholThreads) {
        const double ci = (double)Cm[i * q + c];
        v = fma(ci, w == 0 ? ci : rs[i * q + c], v);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[warp] = v;
      __syncthreads();
      if (tid < 32) {
        double u = red[tid];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
        if (tid == 0) out[1 + w * q + c] = u;
      }
      __syncthreads();
    }
  }
}

// u = z - c / s2 (fp32, d x q) for the core Woodbury solve X = B / s2 + Q u
__global__ void k_core_u(const float* __restrict__ Z, const float* __restrict__ C, int n, float s2,
                         float* __restrict__ U) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) U[p] = Z[p] - C[p] / s2;
}

// y^T y in fp64 over fixed blocks, then out = {loglik, quad, logdet} from the core sums
__global__ void __launch_bounds__(256) k_core_loglik(const float* __restrict__ y, int64_t n, int d, float s2,
                                                     const double* __restrict__ core, double* __restrict__ part,
                                                     unsigned* __restrict__ ticket, double* __restrict__ out) {
  __shared__ double red[8];
  __shared__ bool last;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)gridDim.x * 256)
    s = fma((double)y[i], (double)y[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < 8; ++w) b += red[w];
    part[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double yy = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) yy += ((volatile double*)part)[b];
  const double quad = (yy - core[1]) / (double)s2 + core[2];
  const double ld = core[0] + (double)(n - d) * log((double)s2);
  out[0] = -0.5 * ((double)n * log(2.0 * 3.14159265358979323846) + ld + quad);
  out[1] = quad;
  out[2] = ld;
  *ticket = 0u;
}

struct CoreLayout {
  size_t off_c, off_z, off_u, off_core, off_a, off_qt, off_part, off_ticket, bytes;
};
static CoreLayout core_layout(int64_t rows, int d, int q) {
  CoreLayout L{};
  size_t off = 0, qt = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  L.off_c = take(sizeof(float) * (size_t)d * q);
  L.off_z = take(sizeof(float) * (size_t)d * q);
  L.off_u = take(sizeof(float) * (size_t)d * q);
  L.off_core = take(sizeof(double) * (1 + 2 * (size_t)q));
  L.off_a = take(sizeof(double) * (size_t)d * d);
  apply_qt_ws(rows, d, q, &qt);
  L.off_qt = take(qt);
  L.off_part = take(sizeof(double) * kLlBlocks);
  L.off_ticket = take(sizeof(unsigned));
  L.bytes = off;
  return L;
}

ks_status gp_core_ws(int64_t rows, int d, int q, size_t* bytes) {
  *bytes = core_layout(rows, d, q).bytes;
  return KS_OK;
}

static ks_status core_solve(const float* Q, int64_t rows, int d, const float* B, float s2, const float* X, int q,
                            char* ws, cudaStream_t st, const CoreLayout& L) {
  if (d > kCoreMaxD) return fail(KS_ERR_UNSUPPORTED, "core solve supports d <= 256");
  if (q > kCoreMaxQ) return fail(KS_ERR_UNSUPPORTED, "core solve supports q <= 64");
  float* C = reinterpret_cast<float*>(ws + L.off_c);
  KS_TRY(apply_qt_run(Q, rows, d, X, q, C, ws + L.off_qt, st));   // C = Q^T X
  static PerDeviceOnce attr;
  KS_TRY(attr.run([] {
    KS_CUDA_TRY(cudaFuncSetAttribute(k_core_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, kCoreSmem));
    return KS_OK;
  }));
  k_core_chol_solve<<<1, kCholThreads, kCoreSmem, st>>>(B, d, s2, reinterpret_cast<double*>(ws + L.off_a), C, q,
                                                        reinterpret_cast<float*>(ws + L.off_z),
                                                        reinterpret_cast<double*>(ws + L.off_core));
  KS_LAUNCH_CHECK();
  return KS_OK;
}

ks_status gp_loglik_core_run(const float* Q, int64_t rows, int d, const float* B, float s2, const float* y, double* out,
                             char* ws, cudaStream_t st) {
  const CoreLayout L = core_layout(rows, d, 1);
  KS_TRY(core_solve(Q, rows, d, B, s2, y, 1, ws, st, L));
  unsigned* ticket = reinterpret_cast<unsigned*>(ws + L.off_ticket);
  KS_CUDA_TRY(cudaMemsetAsync(ticket, 0, sizeof(unsigned), st));
  k_core_loglik<<<kLlBlocks, 256, 0, st>>>(y, rows, d, s2, reinterpret_cast<const double*>(ws + L.off_core),
                                           reinterpret_cast<double*>(ws + L.off_part), ticket, out);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

ks_status gp_woodbury_core_run(const float* Q, int64_t rows, int d, const float* B, float s2, const float* X, int q,
                               float* Z, char* ws, cudaStream_t st) {
  const CoreLayout L = core_layout(rows, d, q);
  KS_TRY(core_solve(Q, rows, d, B, s2, X, q, ws, st, L));
  float* U = reinterpret_cast<float*>(ws + L.off_u);
  k_core_u<<<(unsigned)((d * q + 255) / 256), 256, 0, st>>>(reinterpret_cast<const float*>(ws + L.off_z),
                                                          reinterpret_cast<const float*>(ws + L.off_c), d * q, s2, U);
  KS_LAUNCH_CHECK();
  return apply_q_run(Q, rows, d, U, q, Z, st, X, 1.f / s2, 1.f);   // Z = X / s2 + Q u
}

}  // namespace ks
