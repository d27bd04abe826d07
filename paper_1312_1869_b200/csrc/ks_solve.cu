// ks_solve.cu -- the low-rank solve after TSQR (readings L11, L14).
//
//   C = Q^T A          k_qtx_partial + k_qtx_reduce (deterministic split-K over row chunks)
//   Z = R^{-1} C       k_trsolve: truncated back substitution, fp64, blocked, one CTA per 4 columns
//   X = Omega Z        ks_sketch.cu (omega_apply_run)
#include "ks_common.cuh"
#include "ks_internal.h"

#include <algorithm>

namespace ks {

constexpr int kQtRows = 1024;  // rows per partial chunk

// Partial C_chunk[dt*64 .. +64, 0 .. m) = Q[rows of chunk]^T X[rows of chunk].
__global__ void __launch_bounds__(256) k_qtx_partial(const float* __restrict__ Q, int64_t rows, int d,
                                                     const float* __restrict__ X, int m, float* __restrict__ part,
                                                     int64_t chunk_rows) {
  __shared__ float Qs[32][64 + 4];
  __shared__ float Xs[32][64 + 4];
  const int chunk = blockIdx.x, dt = blockIdx.y, mt = blockIdx.z;   // 64 x 64 tile (dt, mt) of C
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t r0 = (int64_t)chunk * chunk_rows;
  const int64_t r1 = min(rows, r0 + chunk_rows);
  float acc[4][4] = {};
  for (int64_t rs = r0; rs < r1; rs += 32) {
    for (int p = tid; p < 32 * 64; p += 256) {
      const int rr = p >> 6, cc = p & 63;
      const int64_t r = rs + rr;
      const int dc = dt * 64 + cc;
      Qs[rr][cc] = (r < r1 && dc < d) ? Q[r * d + dc] : 0.f;
      Xs[rr][cc] = (r < r1 && mt * 64 + cc < m) ? X[r * m + mt * 64 + cc] : 0.f;
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
      const int dr = dt * 64 + 4 * ty + a, mc = mt * 64 + 4 * tx + c;
      if (dr < d && mc < m) P[dr * m + mc] = acc[a][c];
    }
}

// Fast path (d % 4 == 0, m % 4 == 0): a CTA owns a 256 x MT tile of C over a chunk of rows.  32-row slabs
// of Q (32 x 256) and X (32 x MT) are double buffered in shared memory by cp.async (zero-filled outside
// the matrix); thread (tx, ty) accumulates an 8 x (MT/8) micro-tile with packed f32x2 FMAs, the
// broadcast operands read as LDS.128 (Q: 4 distinct 32-B rows per warp, X: 8 distinct) -- 2 FMA per byte
// of shared memory read.
KS_DEVINL void qt_cp16(void* sdst, const void* gsrc, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(ok ? 16 : 0)
               : "memory");
}
template <int MT>
__global__ void __launch_bounds__(256, 2) k_qtx_fast(const float* __restrict__ Q, int64_t rows, int d,
                                                    const float* __restrict__ X, int m, float* __restrict__ part,
                                                    int64_t chunk_rows) {
  constexpr int MU = MT / 8;               // m columns per thread
  extern __shared__ __align__(16) float qsm[];
  float* Qs = qsm;                         // [2][32][256]
  float* Xs = qsm + 2 * 32 * 256;          // [2][32][MT]
  const int chunk = blockIdx.x, d0 = 256 * blockIdx.y, m0 = MT * blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = lane & 7, ty = 4 * warp + (lane >> 3);
  const int64_t r0 = (int64_t)chunk * chunk_rows;
  const int64_t r1 = min(rows, r0 + chunk_rows);
  auto issue = [&](int64_t rs, int b) {
    float* qb = Qs + b * (32 * 256);
#pragma unroll
    for (int i = 0; i < 8; ++i) {   // 32 rows x 64 chunks of 16 B
      const int p = tid + 256 * i, rr = p >> 6, c4 = 4 * (p & 63);
      const bool ok = rs + rr < r1 && d0 + c4 < d;
      qt_cp16(qb + rr * 256 + c4, ok ? Q + (rs + rr) * d + d0 + c4 : Q, ok);
    }
    float* xb = Xs + b * (32 * MT);
    for (int p = tid; p < 32 * (MT / 4); p += 256) {
      const int rr = p / (MT / 4), c4 = 4 * (p % (MT / 4));
      const bool ok = rs + rr < r1 && m0 + c4 < m;
      qt_cp16(xb + rr * MT + c4, ok ? X + (rs + rr) * m + m0 + c4 : X, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  f2_t acc[8][MU / 2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < MU / 2; ++c) acc[a][c] = 0ull;
  if (r0 < r1) issue(r0, 0);
  int b = 0;
  for (int64_t rs = r0; rs < r1; rs += 32, b ^= 1) {
    if (rs + 32 < r1) issue(rs + 32, b ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const float* qb = Qs + b * (32 * 256) + 8 * ty;
    const float* xb = Xs + b * (32 * MT) + MU * tx;
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      const float4 qa = *reinterpret_cast<const float4*>(qb + rr * 256);
      const float4 qc = *reinterpret_cast<const float4*>(qb + rr * 256 + 4);
      const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qc.x, qc.y, qc.z, qc.w};
      f2_t xv[MU / 2];
#pragma unroll
      for (int c4 = 0; c4 < MU / 4; ++c4) {
        const float4 x = *reinterpret_cast<const float4*>(xb + rr * MT + 4 * c4);
        xv[2 * c4] = f2(x.x, x.y);
        xv[2 * c4 + 1] = f2(x.z, x.w);
      }
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < MU / 2; ++c) acc[a][c] = f2fma(f2s(qv[a]), xv[c], acc[a][c]);
    }
    __syncthreads();   // buffer b is refilled by the next-but-one issue
  }
  float* P = part + (int64_t)chunk * d * m;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int dr = d0 + 8 * ty + a;
    if (dr >= d) continue;
#pragma unroll
    for (int c = 0; c < MU / 2; ++c) {
      const int mc = m0 + MU * tx + 2 * c;
      if (mc < m) P[(int64_t)dr * m + mc] = f2lo(acc[a][c]);
      if (mc + 1 < m) P[(int64_t)dr * m + mc + 1] = f2hi(acc[a][c]);
    }
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
// (general form: X = alpha B + beta Q C when B != nullptr; 64-column tiles of C / X by blockIdx.y)
__global__ void __launch_bounds__(256) k_qc(const float* __restrict__ Q, int64_t rows, int d,
                                            const float* __restrict__ C, int m, float* __restrict__ X,
                                            const float* __restrict__ B = nullptr, float alpha = 0.f,
                                            float beta = 1.f) {
  __shared__ float Qs[32][33];
  __shared__ float Cs[32][64 + 4];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int m0 = 64 * blockIdx.y;
  float acc[2][4] = {};
  for (int k0 = 0; k0 < d; k0 += 32) {
    for (int p = tid; p < 32 * 32; p += 256) {
      const int rr = p >> 5, kk = p & 31;
      Qs[rr][kk] = (r0 + rr < rows && k0 + kk < d) ? Q[(r0 + rr) * d + k0 + kk] : 0.f;
    }
    for (int p = tid; p < 32 * 64; p += 256) {
      const int kk = p >> 6, cc = p & 63;
      Cs[kk][cc] = (k0 + kk < d && m0 + cc < m) ? C[(k0 + kk) * m + m0 + cc] : 0.f;
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
      const int mc = m0 + 4 * tx + c;
      if (r < rows && mc < m) X[r * m + mc] = B ? fmaf(alpha, B[r * m + mc], beta * acc[a][c]) : acc[a][c];
    }
}

// Truncated back substitution in fp64 ("backward substitution"; readings L11, L14).
//   k = largest prefix with |r_jj| >= tau max|r_ii| (tau > 0), or k = d (tau == 0; a diagonal
//   <= 1e-12 max|r_ii| is reported as -(index+1) in *kout).
// Blocked right-looking: CTA b owns columns [kTrMC*b, kTrMC*b + kTrMC) of C (fp64 in shared memory).
// For each 32-row block of R from the bottom: warp 0 solves the 32 x 32 diagonal block (lane = row, its
// R segment and 1/r_ll in registers), the block's column panel R[0:b0, b0:b0+32) is staged in shared
// memory by coalesced row reads, and every thread subtracts R[j, block] z[block] from its rows j < b0.
// Every CTA computes k itself.
constexpr int kTrMC = 4;
constexpr int kTrMaxD = 1024;
constexpr int kTrSmem = kTrMaxD * kTrMC * 8 + kTrMaxD * 33 * 4;   // C block (fp64) + R column panel
__global__ void __launch_bounds__(256) k_trsolve(const float* __restrict__ R, const float* __restrict__ C, int d,
                                                 int m, float tau, float* __restrict__ Z, int32_t* __restrict__ kout) {
  extern __shared__ __align__(16) double trs[];
  double (*cs)[kTrMC] = reinterpret_cast<double (*)[kTrMC]>(trs);              // [kTrMaxD][kTrMC]
  float* Rp = reinterpret_cast<float*>(trs + kTrMaxD * kTrMC);                  // [kTrMaxD][33]
  __shared__ double zb[32][kTrMC];
  __shared__ float red[8];
  __shared__ int redi[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = blockIdx.x * kTrMC;
  const int nc = min(kTrMC, m - col0);
  // ---- k (parallel max of |r_ii|, then the first failing index)
  float mx = 0.f;
  for (int i = tid; i < d; i += 256) mx = fmaxf(mx, fabsf(R[(int64_t)i * d + i]));
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int g = 1; g < 8; ++g) mx = fmaxf(mx, red[g]);
  int first = d;
  for (int i = tid; i < d; i += 256) {
    const double r = fabs((double)R[(int64_t)i * d + i]);
    const bool bad = tau > 0.f ? (!(r >= (double)tau * (double)mx) || r == 0.0) : (r <= 1e-12 * (double)mx);
    if (bad && i < first) first = i;
  }
  for (int o = 16; o >= 1; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  if (lane == 0) redi[warp] = first;
  __syncthreads();
  first = redi[0];
  for (int g = 1; g < 8; ++g) first = min(first, redi[g]);
  const int k = tau > 0.f ? first : (first < d ? -(first + 1) : d);
  if (blockIdx.x == 0 && tid == 0 && kout) *kout = k;
  for (int p = tid; p < d * nc; p += 256) {
    const int j = p / nc, c = p - j * nc;
    Z[(int64_t)j * m + col0 + c] = 0.f;   // rows >= k stay 0
  }
  if (k <= 0) return;
  for (int p = tid; p < k * kTrMC; p += 256) {
    const int j = p / kTrMC, c = p - j * kTrMC;
    cs[j][c] = c < nc ? (double)C[(int64_t)j * m + col0 + c] : 0.0;
  }
  __syncthreads();
  for (int b0 = ((k - 1) / 32) * 32; b0 >= 0; b0 -= 32) {
    const int bw = min(32, k - b0);
    // stage R[0:b0, b0:b0+bw) (coalesced: a warp reads 32 consecutive floats of a row)
    for (int j = warp; j < b0; j += 8) Rp[j * 33 + lane] = lane < bw ? R[(int64_t)j * d + b0 + lane] : 0.f;
    if (warp == 0) {
      // lane l = row b0 + l: its R segment R[b0+l][b0 .. b0+bw) in registers
      double rr[32];
      const float* Rr = R + (int64_t)(b0 + min(lane, bw - 1)) * d + b0;
#pragma unroll
      for (int q = 0; q < 32; ++q) rr[q] = (q < bw && lane < bw) ? (double)Rr[q] : 0.0;
      double inv = 1.0;
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q == lane) inv = lane < bw ? 1.0 / rr[q] : 0.0;
      double c[kTrMC];
#pragma unroll
      for (int cc = 0; cc < kTrMC; ++cc) c[cc] = lane < bw ? cs[b0 + lane][cc] : 0.0;
#pragma unroll
      for (int q = 31; q >= 0; --q) {
        if (q < bw) {
#pragma unroll
          for (int cc = 0; cc < kTrMC; ++cc) {
            const double zq = __shfl_sync(0xffffffffu, c[cc] * inv, q);   // lane q's value is z_q
            if (lane == q) c[cc] = zq;
            else if (lane < q) c[cc] = fma(-rr[q], zq, c[cc]);
          }
        }
      }
      if (lane < bw) {
#pragma unroll
        for (int cc = 0; cc < kTrMC; ++cc) {
          zb[lane][cc] = c[cc];
          if (cc < nc) Z[(int64_t)(b0 + lane) * m + col0 + cc] = (float)c[cc];
        }
      }
    }
    __syncthreads();
    for (int j = tid; j < b0; j += 256) {
      double acc[kTrMC];
#pragma unroll
      for (int cc = 0; cc < kTrMC; ++cc) acc[cc] = cs[j][cc];
      for (int q = 0; q < bw; ++q) {
        const double r = (double)Rp[j * 33 + q];
#pragma unroll
        for (int cc = 0; cc < kTrMC; ++cc) acc[cc] = fma(-r, zb[q][cc], acc[cc]);
      }
#pragma unroll
      for (int cc = 0; cc < kTrMC; ++cc) cs[j][cc] = acc[cc];
    }
    __syncthreads();
  }
}

// Rows per partial chunk: kQtRows, doubled while the chunks' (d x m) partials would exceed 64 MiB.
static int64_t qt_chunk_rows(int64_t rows, int d, int m) {
  int64_t c = kQtRows;
  while (((rows + c - 1) / c) * (int64_t)d * m * 4 > (int64_t(64) << 20)) c *= 2;
  return c;
}

ks_status apply_qt_ws(int64_t rows, int d, int m, size_t* bytes) {
  const int64_t cr = qt_chunk_rows(rows, d, m), nchunks = (rows + cr - 1) / cr;
  *bytes = sizeof(float) * (size_t)nchunks * d * m;
  return KS_OK;
}

ks_status apply_qt_run(const float* Q, int64_t rows, int d, const float* X, int m, float* C, void* ws, cudaStream_t st) {
  const int64_t cr = qt_chunk_rows(rows, d, m), nchunks = (rows + cr - 1) / cr;
  float* part = static_cast<float*>(ws);
  const bool fast = (d & 3) == 0 && (m & 3) == 0 && (reinterpret_cast<uintptr_t>(Q) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  if (fast) {
    // ~2 CTAs per SM: chunks of >= cr rows (fewer partials than the workspace holds), multiples of 32
    const int mt = m <= 32 ? 32 : 64;
    const int64_t tiles = (int64_t)((d + 255) / 256) * ((m + mt - 1) / mt);
    int64_t fc = (rows * tiles + 2 * num_sms() - 1) / (2 * num_sms());
    fc = std::max<int64_t>(cr, (fc + 31) / 32 * 32);
    const int64_t nc = (rows + fc - 1) / fc;
    dim3 grid((unsigned)nc, (unsigned)((d + 255) / 256), (unsigned)((m + mt - 1) / mt));
    const int smem = (int)sizeof(float) * 2 * 32 * (256 + mt);
    if (mt == 32) {
      KS_CUDA_TRY(cudaFuncSetAttribute(k_qtx_fast<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_qtx_fast<32><<<grid, 256, smem, st>>>(Q, rows, d, X, m, part, fc);
    } else {
      KS_CUDA_TRY(cudaFuncSetAttribute(k_qtx_fast<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      k_qtx_fast<64><<<grid, 256, smem, st>>>(Q, rows, d, X, m, part, fc);
    }
    KS_LAUNCH_CHECK();
    k_qtx_reduce<<<(d * m + 255) / 256, 256, 0, st>>>(part, (int)nc, d * m, C);
    KS_LAUNCH_CHECK();
    return KS_OK;
  }
  dim3 grid((unsigned)nchunks, (unsigned)((d + 63) / 64), (unsigned)((m + 63) / 64));
  k_qtx_partial<<<grid, 256, 0, st>>>(Q, rows, d, X, m, part, cr);
  KS_LAUNCH_CHECK();
  k_qtx_reduce<<<(d * m + 255) / 256, 256, 0, st>>>(part, (int)nchunks, d * m, C);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

ks_status apply_q_run(const float* Q, int64_t rows, int d, const float* C, int m, float* X, cudaStream_t st,
                      const float* B, float alpha, float beta) {
  k_qc<<<dim3((unsigned)((rows + 31) / 32), (unsigned)((m + 63) / 64)), 256, 0, st>>>(Q, rows, d, C, m, X, B, alpha,
                                                                                     beta);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

ks_status trsolve_run(const float* R, const float* C, int d, int m, float tau, float* Z, int32_t* k, cudaStream_t st) {
  if (d > kTrMaxD) return fail(KS_ERR_UNSUPPORTED, "trsolve supports d <= 1024");
  static PerDeviceOnce attr;
  KS_TRY(attr.run([] {
    KS_CUDA_TRY(cudaFuncSetAttribute(k_trsolve, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrSmem));
    return KS_OK;
  }));
  k_trsolve<<<(unsigned)((m + kTrMC - 1) / kTrMC), 256, kTrSmem, st>>>(R, C, d, m, tau, Z, k);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

}  // namespace ks
