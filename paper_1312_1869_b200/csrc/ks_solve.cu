// ks_solve.cu -- the low-rank solve after TSQR (readings L11, L14).
//
//   C = Q^T A          k_qtx_partial + k_qtx_reduce (deterministic split-K over row chunks)
//   Z = R^{-1} C       k_trsolve: truncated back substitution, fp64, one CTA
//   X = Omega Z        ks_sketch.cu (omega_apply_run)
#include "ks_common.cuh"
#include "ks_internal.h"

namespace ks {

constexpr int kQtRows = 1024;  // rows per partial chunk

// Partial C_chunk[dt*64 .. +64, 0 .. m) = Q[rows of chunk]^T X[rows of chunk].
__global__ void __launch_bounds__(256) k_qtx_partial(const float* __restrict__ Q, int64_t rows, int d,
                                                     const float* __restrict__ X, int m, float* __restrict__ part) {
  __shared__ float Qs[32][64 + 4];
  __shared__ float Xs[32][64 + 4];
  const int chunk = blockIdx.x, dt = blockIdx.y;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t r0 = (int64_t)chunk * kQtRows;
  const int64_t r1 = min(rows, r0 + kQtRows);
  float acc[4][4] = {};
  for (int64_t rs = r0; rs < r1; rs += 32) {
    for (int p = tid; p < 32 * 64; p += 256) {
      const int rr = p >> 6, cc = p & 63;
      const int64_t r = rs + rr;
      const int dc = dt * 64 + cc;
      Qs[rr][cc] = (r < r1 && dc < d) ? Q[r * d + dc] : 0.f;
      Xs[rr][cc] = (r < r1 && cc < m) ? X[r * m + cc] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < 32; ++rr) {
      const float4 q = *reinterpret_cast<const float4*>(&Qs[rr][4 * ty]);
      const float4 x = *reinterpret_cast<const float4*>(&Xs[rr][4 * tx]);
      const float qa[4] = {q.x, q.y, q.z, q.w}, xa[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = fmaf(qa[a], xa[c], acc[a][c]);
    }
    __syncthreads();
  }
  float* P = part + (int64_t)chunk * d * m;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int dr = dt * 64 + 4 * ty + a, mc = 4 * tx + c;
      if (dr < d && mc < m) P[dr * m + mc] = acc[a][c];
    }
}

__global__ void k_qtx_reduce(const float* __restrict__ part, int nchunks, int dm, float* __restrict__ C) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= dm) return;
  float s = 0.f;
  for (int c = 0; c < nchunks; ++c) s += part[(int64_t)c * dm + p];
  C[p] = s;
}

// X (rows x m) = Q (rows x d) C (d x m)
__global__ void __launch_bounds__(256) k_qc(const float* __restrict__ Q, int64_t rows, int d,
                                            const float* __restrict__ C, int m, float* __restrict__ X) {
  __shared__ float Qs[32][33];
  __shared__ float Cs[32][64 + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  float acc[2][4] = {};
  for (int k0 = 0; k0 < d; k0 += 32) {
    for (int p = tid; p < 32 * 32; p += 256) {
      const int rr = p >> 5, kk = p & 31;
      Qs[rr][kk] = (r0 + rr < rows && k0 + kk < d) ? Q[(r0 + rr) * d + k0 + kk] : 0.f;
    }
    for (int p = tid; p < 32 * 64; p += 256) {
      const int kk = p >> 6, cc = p & 63;
      Cs[kk][cc] = (k0 + kk < d && cc < m) ? C[(k0 + kk) * m + cc] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = fmaf(Qs[2 * ty + a][kk], Cs[kk][4 * tx + c], acc[a][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t r = r0 + 2 * ty + a;
      const int mc = 4 * tx + c;
      if (r < rows && mc < m) X[r * m + mc] = acc[a][c];
    }
}

// Truncated back substitution in fp64 (one CTA of 1024 threads).
//   k = largest prefix with |r_jj| >= tau max|r_ii| (tau > 0), or k = d (tau == 0; a diagonal
//   <= 1e-12 max|r_ii| is reported as -(index+1) in *kout).
// Thread t owns column col = t % m and rows j = slot + nslots*q of C (in registers, fp64).
constexpr int kTrQ = 32;
__global__ void __launch_bounds__(1024) k_trsolve(const float* __restrict__ R, const float* __restrict__ C, int d,
                                                  int m, float tau, float* __restrict__ Z, int32_t* __restrict__ kout) {
  __shared__ double zrow[2][64];
  __shared__ int s_k;
  const int tid = threadIdx.x;
  if (tid < 32) {
    double mx = 0.0;
    for (int i = tid; i < d; i += 32) mx = fmax(mx, fabs((double)R[(int64_t)i * d + i]));
    for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (tid == 0) {
      int k = 0;
      if (tau > 0.f) {
        while (k < d) {
          const double r = fabs((double)R[(int64_t)k * d + k]);
          if (!(r >= (double)tau * mx) || r == 0.0) break;
          ++k;
        }
      } else {
        k = d;
        for (int i = 0; i < d; ++i)
          if (fabs((double)R[(int64_t)i * d + i]) <= 1e-12 * mx) { k = -(i + 1); break; }
      }
      s_k = k;
      if (kout) *kout = k;
    }
  }
  __syncthreads();
  const int k = s_k;
  const int nslots = 1024 / m;
  const int col = tid % m, slot = tid / m;
  const bool active = slot < nslots;
  for (int p = tid; p < d * m; p += 1024) Z[p] = 0.f;   // rows >= k stay 0
  __syncthreads();
  if (k <= 0) return;
  double c[kTrQ];
#pragma unroll
  for (int q = 0; q < kTrQ; ++q) {
    const int j = slot + nslots * q;
    c[q] = (active && j < k) ? (double)C[(int64_t)j * m + col] : 0.0;
  }
  for (int i = k - 1; i >= 0; --i) {
    const int par = i & 1;
    if (active && (i % nslots) == slot) {
      double ci = 0.0;
#pragma unroll
      for (int q = 0; q < kTrQ; ++q)
        if (slot + nslots * q == i) ci = c[q];
      const double z = ci / (double)R[(int64_t)i * d + i];
      zrow[par][col] = z;
      Z[(int64_t)i * m + col] = (float)z;
    }
    __syncthreads();
    if (active) {
      const double z = zrow[par][col];
#pragma unroll
      for (int q = 0; q < kTrQ; ++q) {
        const int j = slot + nslots * q;
        if (j < i) c[q] = fma(-(double)R[(int64_t)j * d + i], z, c[q]);
      }
    }
  }
}

ks_status apply_qt_ws(int64_t rows, int d, int m, size_t* bytes) {
  const int64_t nchunks = (rows + kQtRows - 1) / kQtRows;
  *bytes = sizeof(float) * (size_t)nchunks * d * m;
  return KS_OK;
}

ks_status apply_qt_run(const float* Q, int64_t rows, int d, const float* X, int m, float* C, void* ws, cudaStream_t st) {
  const int64_t nchunks = (rows + kQtRows - 1) / kQtRows;
  float* part = static_cast<float*>(ws);
  dim3 grid((unsigned)nchunks, (unsigned)((d + 63) / 64));
  k_qtx_partial<<<grid, 256, 0, st>>>(Q, rows, d, X, m, part);
  KS_LAUNCH_CHECK();
  k_qtx_reduce<<<(d * m + 255) / 256, 256, 0, st>>>(part, (int)nchunks, d * m, C);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

ks_status apply_q_run(const float* Q, int64_t rows, int d, const float* C, int m, float* X, cudaStream_t st) {
  k_qc<<<(unsigned)((rows + 31) / 32), 256, 0, st>>>(Q, rows, d, C, m, X);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

ks_status trsolve_run(const float* R, const float* C, int d, int m, float tau, float* Z, int32_t* k, cudaStream_t st) {
  k_trsolve<<<1, 1024, 0, st>>>(R, C, d, m, tau, Z, k);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

}  // namespace ks
