// ks_sketch.cu -- sketch randomness and the fused SRHT sketch kernel (sm_100a).
//
//   Y[i, t] = (1/sqrt N) * sum_j K[i,j] s_j H_N[j, S_t]          (Def. 1)
//
// with K[i,j] generated in registers from the points (never stored) and H_N the
// natural-order Walsh-Hadamard matrix.  The transform is the
// Kronecker split H_N = H_A (x) H_B, B = 512:
//
//   j = c*B + l,  S_t = a_t*B + m_t:
//   Y[i, t] = (1/sqrt N) sum_c (-1)^popc(c & a_t) * FWHT_B(s o K[i, cB : cB+B])[m_t]
//
// i.e. every chunk of B columns is transformed completely (log2 B butterfly
// levels, 4 in registers + 5 after one shared-memory transpose) and the d
// selected outputs are gathered with the chunk's sign -- N (log2 B + d/B)
// adds per row, the "n log d" of PAPER.md:19, instead of N log2 N.
#include "ks_common.cuh"
#include "ks_internal.h"

#include <algorithm>
#include <cmath>

namespace ks {

// ===================================================================== layout
SketchLayout sketch_layout(const ks_sketch_desc& desc) {
  SketchLayout L{};
  L.N = next_pow2(desc.n);
  if (desc.omega == KS_OMEGA_SRHT) {
    L.A = (int)((desc.n + kSrhtB - 1) / kSrhtB);
    L.ncols_pad = (int64_t)L.A * kSrhtB;
    int tpg = 2;
    while (32 * tpg < desc.d) tpg *= 2;
    L.tpg = tpg;
    L.d_pad = 32 * tpg;
  } else {
    L.A = 0;
    L.ncols_pad = (desc.n + kGaussBK - 1) / kGaussBK * kGaussBK;
    if (L.ncols_pad < kGaussBM) L.ncols_pad = kGaussBM;
    L.tpg = 0;
    L.d_pad = desc.d;
  }
  // Row points are read from the same packed array; rows beyond n never occur.
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  L.off_pk = take(sizeof(float4) * (size_t)L.ncols_pad);
  L.off_tab = take(sizeof(uint32_t) * 512);
  L.off_sel = take(sizeof(int32_t) * (size_t)(desc.d > 0 ? desc.d : 1));
  L.off_bucket_ofs = take(sizeof(int32_t) * (kSrhtB + 1));
  L.off_bucket_idx = take(sizeof(int32_t) * 512);
  L.off_bitmap = take(sizeof(uint32_t) * (size_t)((L.N + 31) / 32));
  L.off_gauss = take(desc.omega == KS_OMEGA_GAUSS ? sizeof(__half) * (size_t)desc.d * (size_t)L.ncols_pad : 0);
  L.bytes = off;
  return L;
}

ks_status sketch_validate(const ks_sketch_desc* desc) {
  if (!desc) return fail(KS_ERR_INVALID_ARGUMENT, "desc is NULL");
  const ks_sketch_desc& D = *desc;
  if (D.n < 1) return fail(KS_ERR_INVALID_ARGUMENT, "n must be >= 1");
  if (D.n > (int64_t(1) << 30)) return fail(KS_ERR_UNSUPPORTED, "n > 2^30 not supported");
  if (D.dim < 1 || D.dim > 3) return fail(KS_ERR_INVALID_ARGUMENT, "dim must be 1, 2 or 3");
  if (D.kernel != KS_KERNEL_SQEXP && D.kernel != KS_KERNEL_MATERN32)
    return fail(KS_ERR_INVALID_ARGUMENT, "unknown kernel kind");
  if (!(D.sigma2 > 0.0f) || !std::isfinite(D.sigma2)) return fail(KS_ERR_INVALID_ARGUMENT, "sigma2 must be > 0");
  if (!(D.ell > 0.0f) || !std::isfinite(D.ell)) return fail(KS_ERR_INVALID_ARGUMENT, "ell must be > 0");
  if (!(D.nugget >= 0.0f) || !std::isfinite(D.nugget)) return fail(KS_ERR_INVALID_ARGUMENT, "nugget must be >= 0");
  const int64_t N = next_pow2(D.n);
  if (D.d < 1 || D.d > N) return fail(KS_ERR_INVALID_ARGUMENT, "need 1 <= d <= N");
  if (D.omega == KS_OMEGA_SRHT) {
    if (D.d > 512) return fail(KS_ERR_UNSUPPORTED, "SRHT path supports d <= 512");
  } else if (D.omega == KS_OMEGA_GAUSS) {
    if (D.d > D.n) return fail(KS_ERR_INVALID_ARGUMENT, "Gaussian sketch needs d <= n");
    if (D.d % 16 != 0 || D.d < 16 || D.d > 256)
      return fail(KS_ERR_UNSUPPORTED, "Gaussian tcgen05 path needs d % 16 == 0 and 16 <= d <= 256");
  } else {
    return fail(KS_ERR_INVALID_ARGUMENT, "unknown omega kind");
  }
  return KS_OK;
}

// ============================================================ randomness kernels
// Packed point j: (scaled coords, amplitude).  SE: coords * sqrt(log2(e) / (2 ell^2)) so that
// exp(-r^2/(2 ell^2)) = 2^(-r'^2).  Matern-3/2: coords * sqrt(3)/ell so that r' = sqrt(3) r/ell.
// amplitude = s_j * sigma2 (SRHT; the Rademacher sign folded in) or S * sigma2 (Gaussian, gauss_scale);
// padded columns j >= n get amplitude 0 (zero padding, reading L3).
__global__ void k_pack_points(const float* __restrict__ pts, int64_t n, int dim, int64_t ncols_pad, float scale,
                              float sigma2, uint64_t seed, int srht, float4* __restrict__ pk) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols_pad) return;
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
  if (j < n) {
    p.x = pts[j] * scale;
    if (dim > 1) p.y = pts[n + j] * scale;
    if (dim > 2) p.z = pts[2 * n + j] * scale;
    p.w = srht ? rademacher(seed, j) * sigma2 : sigma2;
  }
  pk[j] = p;
}

// Selection S: the first d distinct values of (philox(seed, 2, t).x & (N-1)), t = 0, 1, ...
// (uniform without replacement, reading L4), sorted ascending.  One CTA of 1024 threads;
// also writes the SRHT gather table and the (m_t)-bucket CSR used by the Omega-apply.
__global__ void __launch_bounds__(1024) k_selection(uint64_t seed, int64_t N, int d, int d_pad,
                                                    uint32_t* __restrict__ bitmap, int32_t* __restrict__ sel,
                                                    uint32_t* __restrict__ tab, int32_t* __restrict__ bofs,
                                                    int32_t* __restrict__ bidx) {
  __shared__ uint32_t cand[1024];
  __shared__ int warp_sums[32];
  __shared__ int s_count;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t nwords = (N + 31) / 32;
  for (int64_t w = tid; w < nwords; w += 1024) bitmap[w] = 0u;
  if (tid == 0) s_count = 0;
  __syncthreads();
  for (uint64_t base = 0; s_count < d; base += 1024) {
    const uint32_t c = philox(seed, kStreamSelect, base + (uint64_t)tid).x & (uint32_t)(N - 1);
    cand[tid] = c;
    __syncthreads();
    bool isnew = !((bitmap[c >> 5] >> (c & 31)) & 1u);
    for (int q = 0; q < tid && isnew; ++q) isnew = cand[q] != c;
    // block exclusive scan of isnew
    const unsigned ball = __ballot_sync(0xffffffffu, isnew);
    const int in_warp = __popc(ball & ((1u << lane) - 1u));
    if (lane == 0) warp_sums[wid] = __popc(ball);
    __syncthreads();
    if (wid == 0) {
      int v = warp_sums[lane];
      for (int o = 1; o < 32; o <<= 1) { int u = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v += u; }
      warp_sums[lane] = v;  // inclusive
    }
    __syncthreads();
    const int excl = (wid ? warp_sums[wid - 1] : 0) + in_warp;
    const int total = warp_sums[31];
    const int remaining = d - s_count;
    if (isnew && excl < remaining) atomicOr(&bitmap[c >> 5], 1u << (c & 31));
    __syncthreads();
    if (tid == 0) s_count += total < remaining ? total : remaining;
    __syncthreads();
  }
  // Sorted enumeration of the bitmap: contiguous word ranges per thread, block scan of counts.
  const int64_t per = (nwords + 1023) / 1024;
  const int64_t w0 = (int64_t)tid * per, w1 = (w0 + per < nwords) ? w0 + per : nwords;
  int cnt = 0;
  for (int64_t w = w0; w < w1; ++w) cnt += __popc(bitmap[w]);
  int v = cnt;
  for (int o = 1; o < 32; o <<= 1) { int u = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v += u; }
  if (lane == 31) warp_sums[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int x = warp_sums[lane];
    for (int o = 1; o < 32; o <<= 1) { int u = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += u; }
    warp_sums[lane] = x;
  }
  __syncthreads();
  int pos = (wid ? warp_sums[wid - 1] : 0) + v - cnt;
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t bits = bitmap[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      sel[pos++] = (int32_t)(w * 32 + b);
    }
  }
  __syncthreads();
  // SRHT gather table: (m_t | a_t << 16), padded entries inert.
  for (int t = tid; t < d_pad; t += 1024) {
    uint32_t e = 0u;
    if (t < d) {
      const uint32_t s = (uint32_t)sel[t];
      e = (s & (kSrhtB - 1)) | ((s / kSrhtB) << 16);
    }
    tab[t] = e;
  }
  // CSR of t by m_t (deterministic, ascending t within a bucket) for the Omega-apply.
  if (tid == 0) {
    for (int b = 0; b <= kSrhtB; ++b) bofs[b] = 0;
    for (int t = 0; t < d; ++t) bofs[(sel[t] & (kSrhtB - 1)) + 1]++;
    for (int b = 0; b < kSrhtB; ++b) bofs[b + 1] += bofs[b];
    for (int t = 0; t < d; ++t) {
      const int b = sel[t] & (kSrhtB - 1);
      int p = bofs[b];
      while (bidx[p] != -1 && p < bofs[b + 1]) ++p;  // first free slot (slots pre-marked -1 below)
      bidx[p] = t;
    }
  }
}

__global__ void k_fill_i32(int32_t* p, int n, int32_t v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// Gaussian Omega^T (d x ncols_pad, fp16): Omega_jt = fp16_RN(z), z = Box-Muller(philox(seed, 3, j*d + t))
// (reading L6); the 1/sqrt(d) is applied in the sketch epilogue.  Columns j >= n are zero.
__global__ void k_gauss_omega(uint64_t seed, int64_t n, int d, int64_t ncols_pad, __half* __restrict__ omT) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (j >= ncols_pad) return;
  __half h = __float2half_rn(0.0f);
  if (j < n) h = __double2half(box_muller(philox(seed, kStreamGauss, (uint64_t)j * (uint64_t)d + (uint64_t)t)));
  omT[(int64_t)t * ncols_pad + j] = h;
}

double gauss_scale(const ks_sketch_desc& D) {
  const double kmax = (double)D.sigma2 + (double)D.nugget;
  int e = (int)std::floor(std::log2(16384.0 / kmax));
  e = std::max(-60, std::min(60, e));
  return std::ldexp(1.0, e);
}

static float coord_scale(const ks_sketch_desc& D) {
  if (D.kernel == KS_KERNEL_SQEXP) return (float)std::sqrt(1.4426950408889634 / (2.0 * (double)D.ell * (double)D.ell));
  return (float)(std::sqrt(3.0) / (double)D.ell);
}

ks_status sketch_prepare(const ks_sketch_desc& D, const SketchLayout& L, const float* pts, char* ws,
                         cudaStream_t st, bool need_points) {
  const int srht = D.omega == KS_OMEGA_SRHT;
  if (need_points) {
    const int64_t nb = (L.ncols_pad + 255) / 256;
    const float amp = srht ? D.sigma2 : (float)(D.sigma2 * gauss_scale(D));
    k_pack_points<<<(unsigned)nb, 256, 0, st>>>(pts, D.n, D.dim, L.ncols_pad, coord_scale(D), amp, D.seed,
                                                 srht, reinterpret_cast<float4*>(ws + L.off_pk));
    KS_LAUNCH_CHECK();
  }
  if (srht) {
    k_fill_i32<<<2, 256, 0, st>>>(reinterpret_cast<int32_t*>(ws + L.off_bucket_idx), 512, -1);
    KS_LAUNCH_CHECK();
    k_selection<<<1, 1024, 0, st>>>(D.seed, L.N, D.d, L.d_pad, reinterpret_cast<uint32_t*>(ws + L.off_bitmap),
                                    reinterpret_cast<int32_t*>(ws + L.off_sel),
                                    reinterpret_cast<uint32_t*>(ws + L.off_tab),
                                    reinterpret_cast<int32_t*>(ws + L.off_bucket_ofs),
                                    reinterpret_cast<int32_t*>(ws + L.off_bucket_idx));
    KS_LAUNCH_CHECK();
  } else {
    dim3 grid((unsigned)((L.ncols_pad + 255) / 256), (unsigned)D.d);
    k_gauss_omega<<<grid, 256, 0, st>>>(D.seed, D.n, D.d, L.ncols_pad, reinterpret_cast<__half*>(ws + L.off_gauss));
    KS_LAUNCH_CHECK();
  }
  return KS_OK;
}

// ============================================================ fused SRHT kernel
// One CTA = 16 rows of Y (256 threads, 2-3 CTAs per SM); loops over the column chunks c of K.
// The tile W is double buffered, so a chunk needs 2 barriers (after phase A, after phase B).
// Shared tile W: column l (0..511) of the chunk holds its 16 row values at
// A(l, r) = l*16 + (l >> 5)*16 + r (the (l >> 5) pad makes phase B conflict-free).
//   phase A : thread (rg = t&7, cg = t>>3) evaluates K*s for rows 2rg, 2rg+1 and columns
//             l = cg + 32q, q < 16, butterflies over l bits 5-8 in registers, stores W.
//   phase B : thread (rp = t&15, g = t>>4) loads row rp at l = 32g + b, b < 32, butterflies
//             over l bits 0-4, stores back.  W now holds FWHT_B of the chunk (natural order).
//   phase C : thread (rq = t&3, og = t>>2) accumulates its TPO = TPG/2 outputs for rows
//             4rq..4rq+3: acc[k] += (-1)^popc(c & a_t) * W[m_t][4rq .. 4rq+3].
KS_DEVINL int srht_w(int l, int r) { return l * 16 + (l >> 5) * 16 + r; }
constexpr int kSrhtSmemFloats = kSrhtB * 16 + (kSrhtB / 32) * 16;   // 33 KB per buffer

template <int DIM, int KIND, int TPG>
__global__ void __launch_bounds__(256, TPG <= 8 ? 3 : 2)
k_sketch_srht(const float4* __restrict__ pk, const uint32_t* __restrict__ tab, int64_t row_begin, int64_t row_end,
              int A, int d, float out_scale, float nugget, float* __restrict__ Y) {
  constexpr int TPO = TPG / 2;
  extern __shared__ __align__(16) float Wbuf[];   // [2][kSrhtSmemFloats], double buffered: chunk c uses half c & 1
  const int t = threadIdx.x;
  const int rg = t & 7, cg = t >> 3;
  const int rp = t & 15, g = t >> 4;
  const int rq = t & 3, og = t >> 2;
  const int64_t row0 = row_begin + (int64_t)blockIdx.x * kSrhtRows;
  const int oA = cg * 16 + 2 * rg;         // + 528 q           (= srht_w(cg + 32 q, 2 rg))
  const int oB = 528 * g + rp;             // + 16 b            (= srht_w(32 g + b, rp))

  float xi[2][3];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    int64_t i = row0 + 2 * rg + rr;
    if (i >= row_end) i = row_end - 1;
    const float4 p = pk[i];
    xi[rr][0] = p.x; xi[rr][1] = p.y; xi[rr][2] = p.z;
  }
  int wofs[TPO];
  uint32_t ahi[TPO];
#pragma unroll
  for (int k = 0; k < TPO; ++k) {
    const uint32_t e = tab[og * TPO + k];
    wofs[k] = srht_w((int)(e & 0xFFFFu), 4 * rq);
    ahi[k] = e >> 16;
  }
  float acc[TPO][4];
#pragma unroll
  for (int k = 0; k < TPO; ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.f;

  for (int c = 0; c < A; ++c) {
    float* W = Wbuf + (c & 1) * kSrhtSmemFloats;
    float* wA = W + oA;
    float* wB = W + oB;
    // ---------------- phase A (writes the other buffer than chunk c-1's phase C reads: no barrier before it)
    {
      const float4* pc = pk + (int64_t)c * kSrhtB + cg;
      float v[2][16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float4 p = __ldg(pc + 32 * q);
        v[0][q] = cov_signed<DIM, KIND>(xi[0], p);
        v[1][q] = cov_signed<DIM, KIND>(xi[1], p);
      }
#pragma unroll
      for (int h = 1; h < 16; h <<= 1)
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (!(q & h)) {
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
              const float x = v[rr][q], y = v[rr][q + h];
              v[rr][q] = x + y;
              v[rr][q + h] = x - y;
            }
          }
#pragma unroll
      for (int q = 0; q < 16; ++q) *reinterpret_cast<float2*>(wA + 528 * q) = make_float2(v[0][q], v[1][q]);
    }
    __syncthreads();
    // ---------------- phase B
    {
      float u[32];
#pragma unroll
      for (int b = 0; b < 32; ++b) u[b] = wB[16 * b];
#pragma unroll
      for (int h = 1; h < 32; h <<= 1)
#pragma unroll
        for (int b = 0; b < 32; ++b)
          if (!(b & h)) {
            const float x = u[b], y = u[b + h];
            u[b] = x + y;
            u[b + h] = x - y;
          }
#pragma unroll
      for (int b = 0; b < 32; ++b) wB[16 * b] = u[b];
    }
    __syncthreads();
    // ---------------- phase C
#pragma unroll
    for (int k = 0; k < TPO; ++k) {
      const float sg = __int_as_float(0x3f800000u | ((__popc((uint32_t)c & ahi[k]) & 1u) << 31));
      const float4 w = *reinterpret_cast<const float4*>(W + wofs[k]);
      acc[k][0] = fmaf(sg, w.x, acc[k][0]);
      acc[k][1] = fmaf(sg, w.y, acc[k][1]);
      acc[k][2] = fmaf(sg, w.z, acc[k][2]);
      acc[k][3] = fmaf(sg, w.w, acc[k][3]);
    }
  }
  // ---------------- epilogue: scale, nugget (by index, reading L9), store.
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int64_t i = row0 + 4 * rq + rr;
    if (i >= row_end) continue;
    const float si = pk[i].w > 0.f ? 1.f : -1.f;
    float* yrow = Y + (i - row_begin) * (int64_t)d;
#pragma unroll
    for (int k = 0; k < TPO; ++k) {
      const int tt = og * TPO + k;
      if (tt < d) {
        const uint32_t e = tab[tt];
        const uint32_t S = (e & 0xFFFFu) + (e >> 16) * (uint32_t)kSrhtB;
        const float h = (__popcll((unsigned long long)i & (unsigned long long)S) & 1) ? -1.f : 1.f;
        yrow[tt] = fmaf(nugget * si, h * out_scale, acc[k][rr] * out_scale);
      }
    }
  }
}

template <int DIM, int KIND, int TPG>
static ks_status launch_srht(const SketchLayout& L, const ks_sketch_desc& D, int64_t rb, int64_t re, float* Y,
                             char* ws, cudaStream_t st) {
  auto kern = k_sketch_srht<DIM, KIND, TPG>;
  const int smem = 2 * kSrhtSmemFloats * (int)sizeof(float);
  KS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const unsigned grid = (unsigned)((re - rb + kSrhtRows - 1) / kSrhtRows);
  kern<<<grid, 256, smem, st>>>(reinterpret_cast<const float4*>(ws + L.off_pk),
                                reinterpret_cast<const uint32_t*>(ws + L.off_tab), rb, re, L.A, D.d,
                                (float)(1.0 / std::sqrt((double)L.N)), D.nugget, Y);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

template <int DIM, int KIND>
static ks_status dispatch_tpg(const SketchLayout& L, const ks_sketch_desc& D, int64_t rb, int64_t re, float* Y,
                              char* ws, cudaStream_t st) {
  switch (L.tpg) {
    case 2: return launch_srht<DIM, KIND, 2>(L, D, rb, re, Y, ws, st);
    case 4: return launch_srht<DIM, KIND, 4>(L, D, rb, re, Y, ws, st);
    case 8: return launch_srht<DIM, KIND, 8>(L, D, rb, re, Y, ws, st);
    case 16: return launch_srht<DIM, KIND, 16>(L, D, rb, re, Y, ws, st);
  }
  return fail(KS_ERR_UNSUPPORTED, "unsupported SRHT output width");
}

ks_status sketch_run(const ks_sketch_desc& D, const SketchLayout& L, int64_t rb, int64_t re, float* Y, char* ws,
                     cudaStream_t st) {
  if (re <= rb) return KS_OK;
  if (D.omega == KS_OMEGA_GAUSS) return gauss_sketch_run(D, L, rb, re, Y, ws, st);
  const bool se = D.kernel == KS_KERNEL_SQEXP;
  switch (D.dim) {
    case 1: return se ? dispatch_tpg<1, KS_KERNEL_SQEXP>(L, D, rb, re, Y, ws, st)
                      : dispatch_tpg<1, KS_KERNEL_MATERN32>(L, D, rb, re, Y, ws, st);
    case 2: return se ? dispatch_tpg<2, KS_KERNEL_SQEXP>(L, D, rb, re, Y, ws, st)
                      : dispatch_tpg<2, KS_KERNEL_MATERN32>(L, D, rb, re, Y, ws, st);
    case 3: return se ? dispatch_tpg<3, KS_KERNEL_SQEXP>(L, D, rb, re, Y, ws, st)
                      : dispatch_tpg<3, KS_KERNEL_MATERN32>(L, D, rb, re, Y, ws, st);
  }
  return fail(KS_ERR_INVALID_ARGUMENT, "dim");
}

// ============================================================ Omega-apply
// SRHT: X[j, col] = s_j / sqrt(N) * (H_N scatter_S(Z[:, col]))[j]  (Omega Z with Omega^T = (1/sqrt N) H[S,:] D_s).
// Per chunk c (rows j = cB + l):  u[m] = sum_{t: m_t = m} (-1)^popc(c & a_t) Z[t, col];  X = s o FWHT_B(u).
__global__ void __launch_bounds__(256) k_omega_apply_srht(const float* __restrict__ Z, int m, int d,
                                                          const uint32_t* __restrict__ tab,
                                                          const int32_t* __restrict__ bofs,
                                                          const int32_t* __restrict__ bidx, uint64_t seed,
                                                          int64_t n, int64_t row_begin, int64_t row_end,
                                                          int c_first, float scale, float* __restrict__ X) {
  extern __shared__ float u[];  // [kSrhtB][m + 1]
  const int ld = m + 1;
  const int c = c_first + blockIdx.x;
  const int tid = threadIdx.x;
  for (int p = tid; p < kSrhtB * m; p += 256) {
    const int l = p / m, col = p - l * m;
    float acc = 0.f;
    for (int q = bofs[l]; q < bofs[l + 1]; ++q) {
      const int tt = bidx[q];
      const uint32_t a = tab[tt] >> 16;
      const float v = Z[tt * m + col];
      acc += (__popc((uint32_t)c & a) & 1) ? -v : v;
    }
    u[l * ld + col] = acc;
  }
  __syncthreads();
  for (int h = 1; h < kSrhtB; h <<= 1) {
    for (int p = tid; p < (kSrhtB / 2) * m; p += 256) {
      const int b = p / m, col = p - b * m;
      const int l = ((b / h) * 2 * h) + (b % h);
      const float x = u[l * ld + col], y = u[(l + h) * ld + col];
      u[l * ld + col] = x + y;
      u[(l + h) * ld + col] = x - y;
    }
    __syncthreads();
  }
  for (int l = tid; l < kSrhtB; l += 256) {
    const int64_t j = (int64_t)c * kSrhtB + l;
    if (j < row_begin || j >= row_end || j >= n) continue;
    const float s = rademacher(seed, j) * scale;
    float* xr = X + (j - row_begin) * (int64_t)m;
    for (int col = 0; col < m; ++col) xr[col] = s * u[l * ld + col];
  }
}

// Gaussian: X[j, :] = (1/sqrt d) sum_t Omega[j, t] Z[t, :].
__global__ void __launch_bounds__(256) k_omega_apply_gauss(const __half* __restrict__ omT, int64_t ldo,
                                                           const float* __restrict__ Z, int m, int d,
                                                           int64_t row_begin, int64_t row_end, float scale,
                                                           float* __restrict__ X) {
  extern __shared__ float zs[];  // d x m
  for (int p = threadIdx.x; p < d * m; p += blockDim.x) zs[p] = Z[p];
  __syncthreads();
  const int64_t j = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= row_end) return;
  float* xr = X + (j - row_begin) * (int64_t)m;
  for (int c0 = 0; c0 < m; c0 += 8) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < d; ++t) {
      const float o = __half2float(omT[(int64_t)t * ldo + j]);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + q < m) acc[q] = fmaf(o, zs[t * m + c0 + q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (c0 + q < m) xr[c0 + q] = acc[q] * scale;
  }
}

ks_status omega_apply_run(const ks_sketch_desc& D, const SketchLayout& L, const float* Z, int m, int64_t rb,
                          int64_t re, float* X, char* ws, cudaStream_t st) {
  if (re <= rb) return KS_OK;
  if (D.omega == KS_OMEGA_SRHT) {
    const int c0 = (int)(rb / kSrhtB), c1 = (int)((re - 1) / kSrhtB);
    const int smem = kSrhtB * (m + 1) * (int)sizeof(float);
    KS_CUDA_TRY(cudaFuncSetAttribute(k_omega_apply_srht, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_omega_apply_srht<<<(unsigned)(c1 - c0 + 1), 256, smem, st>>>(
        Z, m, D.d, reinterpret_cast<const uint32_t*>(ws + L.off_tab),
        reinterpret_cast<const int32_t*>(ws + L.off_bucket_ofs), reinterpret_cast<const int32_t*>(ws + L.off_bucket_idx),
        D.seed, D.n, rb, re, c0, (float)(1.0 / std::sqrt((double)L.N)), X);
    KS_LAUNCH_CHECK();
  } else {
    const int smem = D.d * m * (int)sizeof(float);
    KS_CUDA_TRY(cudaFuncSetAttribute(k_omega_apply_gauss, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const unsigned grid = (unsigned)((re - rb + 255) / 256);
    k_omega_apply_gauss<<<grid, 256, smem, st>>>(reinterpret_cast<const __half*>(ws + L.off_gauss), L.ncols_pad, Z,
                                                  m, D.d, rb, re, (float)(1.0 / std::sqrt((double)D.d)), X);
    KS_LAUNCH_CHECK();
  }
  return KS_OK;
}

// ============================================================ export (tests)
__global__ void k_export_signs(uint64_t seed, int64_t N, int8_t* __restrict__ s) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) s[j] = (int8_t)(rademacher(seed, j) > 0.f ? 1 : -1);
}
__global__ void k_export_gauss(const __half* __restrict__ omT, int64_t ldo, int64_t n, int d, uint16_t* __restrict__ g) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n * d) return;
  const int64_t j = p / d;
  const int t = (int)(p - j * d);
  g[p] = __half_as_ushort(omT[(int64_t)t * ldo + j]);
}

ks_status omega_export_run(const ks_sketch_desc& D, const SketchLayout& L, int8_t* signs, int32_t* sel,
                           uint16_t* gauss, char* ws, cudaStream_t st) {
  if (signs) {
    k_export_signs<<<(unsigned)((L.N + 255) / 256), 256, 0, st>>>(D.seed, L.N, signs);
    KS_LAUNCH_CHECK();
  }
  if (sel) {
    if (D.omega != KS_OMEGA_SRHT) return fail(KS_ERR_INVALID_ARGUMENT, "selection exists only for SRHT");
    KS_CUDA_TRY(cudaMemcpyAsync(sel, ws + L.off_sel, sizeof(int32_t) * (size_t)D.d, cudaMemcpyDeviceToDevice, st));
  }
  if (gauss) {
    if (D.omega != KS_OMEGA_GAUSS) return fail(KS_ERR_INVALID_ARGUMENT, "Gaussian Omega exists only for GAUSS");
    const int64_t tot = D.n * (int64_t)D.d;
    k_export_gauss<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(reinterpret_cast<const __half*>(ws + L.off_gauss),
                                                                   L.ncols_pad, D.n, D.d, gauss);
    KS_LAUNCH_CHECK();
  }
  return KS_OK;
}

}  // namespace ks
