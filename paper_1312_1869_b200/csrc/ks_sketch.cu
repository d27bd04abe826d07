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
// i.e. every chunk of B columns is transformed (log2 B butterfly levels: 4 in
// registers, 5 after one shared-memory exchange) and the d selected outputs are
// gathered with the chunk's sign --
// N (log2 B + d/B) adds per row, the "n log d" of PAPER.md:19, instead of N log2 N.
// All arithmetic on row PAIRS uses Blackwell's packed f32x2 instructions
// (FADD2/FMUL2/FFMA2): the FP32 pipe does the same lane-ops, but each instruction
// issues once for two rows, so the kernel is bound by the FP32 pipe, not by issue.
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
    int tpo = 1;
    while (64 * tpo < desc.d) tpo *= 2;   // 64 output groups in the gather phase
    L.tpo = tpo;
    L.d_pad = 64 * tpo;
  } else {   // GAUSS, DHT, DCT: the tensor-core contraction
    L.A = 0;
    L.ncols_pad = (desc.n + kGaussBK - 1) / kGaussBK * kGaussBK;
    if (L.ncols_pad < kGaussBM) L.ncols_pad = kGaussBM;
    L.tpo = 0;
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
  const int om_planes = desc.omega == KS_OMEGA_GAUSS ? 1 : (desc.omega == KS_OMEGA_SRHT ? 0 : 2);   // trig: hi + lo
  L.off_gauss = take(sizeof(__half) * (size_t)om_planes * (size_t)desc.d * (size_t)L.ncols_pad);
  L.off_perm = take(desc.omega == KS_OMEGA_SRHT ? sizeof(int32_t) * (size_t)L.d_pad : 0);
  L.off_sgn = take(desc.omega == KS_OMEGA_SRHT ? sizeof(float) * (size_t)L.A * (size_t)L.d_pad : 0);
  // Gaussian split-K: the second half's partial Y (rows x d)
  L.off_ybuf = take(desc.omega != KS_OMEGA_SRHT ? sizeof(float) * (size_t)desc.n * (size_t)desc.d : 0);
  L.bytes = off;
  return L;
}

ks_status sketch_validate(const ks_sketch_desc* desc) {
  if (!desc) return fail(KS_ERR_INVALID_ARGUMENT, "desc is NULL");
  const ks_sketch_desc& D = *desc;
  if (D.n < 1) return fail(KS_ERR_INVALID_ARGUMENT, "n must be >= 1");
  if (D.n > (int64_t(1) << 30)) return fail(KS_ERR_UNSUPPORTED, "n > 2^30 not supported");
  const bool stored = D.kernel == KS_KERNEL_STORED;
  if (!stored && (D.dim < 1 || D.dim > 3)) return fail(KS_ERR_INVALID_ARGUMENT, "dim must be 1, 2 or 3");
  if (D.kernel != KS_KERNEL_SQEXP && D.kernel != KS_KERNEL_MATERN32 && !stored)
    return fail(KS_ERR_INVALID_ARGUMENT, "unknown kernel kind");
  if (!(D.sigma2 > 0.0f) || !std::isfinite(D.sigma2)) return fail(KS_ERR_INVALID_ARGUMENT, "sigma2 must be > 0");
  if (!stored && (!(D.ell > 0.0f) || !std::isfinite(D.ell))) return fail(KS_ERR_INVALID_ARGUMENT, "ell must be > 0");
  if (!(D.nugget >= 0.0f) || !std::isfinite(D.nugget)) return fail(KS_ERR_INVALID_ARGUMENT, "nugget must be >= 0");
  const int64_t N = next_pow2(D.n);
  if (D.d < 1 || D.d > N) return fail(KS_ERR_INVALID_ARGUMENT, "need 1 <= d <= N");
  if (D.omega == KS_OMEGA_SRHT) {
    if (D.d > 512) return fail(KS_ERR_UNSUPPORTED, "SRHT path supports d <= 512");
  } else if (D.omega == KS_OMEGA_GAUSS || D.omega == KS_OMEGA_DHT || D.omega == KS_OMEGA_DCT) {
    if (D.d > D.n) return fail(KS_ERR_INVALID_ARGUMENT, "Gaussian / Hartley / cosine sketch needs d <= n");
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
    if (pts) {   // (a stored K has no points: amplitudes only)
      p.x = pts[j] * scale;
      if (dim > 1) p.y = pts[n + j] * scale;
      if (dim > 2) p.z = pts[2 * n + j] * scale;
    }
    p.w = srht ? rademacher(seed, j) * sigma2 : sigma2;
  }
  pk[j] = p;
}

// Exclusive block scan of a 0/1 flag over 1024 threads: returns the rank, *total = number of flags.
KS_DEVINL int block_rank(bool flag, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  __syncthreads();   // wsum reuse
  if (lane == 0) wsum[wid] = __popc(b);
  __syncthreads();
  if (wid == 0) {
    int v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v += u; }
    wsum[lane] = v;   // inclusive
  }
  __syncthreads();
  *total = wsum[31];
  return (wid ? wsum[wid - 1] : 0) + __popc(b & ((1u << lane) - 1u));
}

// Selection S (reading L4): the first d distinct values of (philox(seed, 2, t).x & (N-1)), t = 0, 1, ...,
// sorted ascending.  Warp 0 scans the stream 32 draws at a time (__match_any_sync finds duplicates inside
// the round, a bitmap of N bits -- in shared memory when N <= 2^20 -- the earlier ones), then all 1024
// threads enumerate the bitmap in order.  Also builds, for the sketch and the Omega-apply:
//   tab[t]  = m_t | a_t << 16 (kSrhtB-chunks),
//   bofs/bidx = CSR of t by bucket m_t, ascending t inside a bucket,
//   perm[s] = the gather slot permutation of the sketch (bank-conflict-free bins, see the perm section).
constexpr int64_t kSelSmemBits = int64_t(1) << 20;
__global__ void __launch_bounds__(1024) k_selection(uint64_t seed, int64_t N, int64_t range, int d, int d_pad, int tpo,
                                                    uint32_t* __restrict__ gbitmap, int32_t* __restrict__ sel,
                                                    uint32_t* __restrict__ tab, int32_t* __restrict__ bofs,
                                                    int32_t* __restrict__ bidx, int32_t* __restrict__ perm) {
  extern __shared__ uint32_t sbits[];   // N/32 words when N <= 2^20
  __shared__ int s_sel[512];
  __shared__ int s_lst[4][512];         // outputs of each class, ascending t
  __shared__ int s_left[512];
  __shared__ int s_over[512];
  __shared__ int s_moved[512];
  __shared__ int s_hist[kSrhtB + 1];
  __shared__ int s_fill[kSrhtB];
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool in_smem = N <= kSelSmemBits;
  uint32_t* bitmap = in_smem ? sbits : gbitmap;
  const int64_t nwords = (N + 31) / 32;
  for (int64_t w = tid; w < nwords; w += 1024) bitmap[w] = 0u;
  __syncthreads();
  if (wid == 0) {
    int count = 0;
    for (uint64_t base = 0; count < d; base += 32) {
      const uint32_t c = philox(seed, kStreamSelect, base + (uint64_t)lane).x & (uint32_t)(N - 1);
      const unsigned same = __match_any_sync(0xffffffffu, c);
      const uint32_t word = in_smem ? bitmap[c >> 5] : __ldcg(bitmap + (c >> 5));
      const bool keep = (__ffs(same) - 1) == lane && !((word >> (c & 31)) & 1u) && (int64_t)c < range;
      const unsigned ball = __ballot_sync(0xffffffffu, keep);
      const int pos = count + __popc(ball & ((1u << lane) - 1u));
      if (keep && pos < d) atomicOr(bitmap + (c >> 5), 1u << (c & 31));
      count = min(d, count + __popc(ball));
      __syncwarp();
    }
  }
  __syncthreads();
  // sorted enumeration: contiguous word ranges per thread, block scan of the counts
  const int64_t per = (nwords + 1023) / 1024;
  const int64_t w0 = (int64_t)tid * per, w1 = (w0 + per < nwords) ? w0 + per : nwords;
  int cnt = 0;
  for (int64_t w = w0; w < w1; ++w) cnt += __popc(in_smem ? bitmap[w] : __ldcg(bitmap + w));
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v += u; }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int x = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += u; }
    wsum[lane] = x;
  }
  __syncthreads();
  int pos = (wid ? wsum[wid - 1] : 0) + v - cnt;
  for (int64_t w = w0; w < w1; ++w) {
    uint32_t bits = in_smem ? bitmap[w] : __ldcg(bitmap + w);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      s_sel[pos] = (int32_t)(w * 32 + b);
      sel[pos] = (int32_t)(w * 32 + b);
      ++pos;
    }
  }
  for (int b = tid; b <= kSrhtB; b += 1024) s_hist[b] = 0;
  if (tid < kSrhtB) s_fill[tid] = 0;
  __syncthreads();
  // ---- tab and the bucket CSR (counting sort by m_t, then each bucket sorted by t)
  const bool act = tid < d;
  const int st = act ? s_sel[tid] : 0;
  const int m = st & (kSrhtB - 1);
  if (act) {
    tab[tid] = (uint32_t)m | ((uint32_t)(st / kSrhtB) << 16);
    atomicAdd(&s_hist[m + 1], 1);
  }
  __syncthreads();
  if (wid == 0) {   // exclusive offsets: s_hist[b] = first slot of bucket b (16 buckets per lane)
    int loc[16], acc = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) { acc += s_hist[16 * lane + q + 1]; loc[q] = acc; }
    int x = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int u = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += u; }
    const int base = x - acc;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 16; ++q) s_hist[16 * lane + q + 1] = base + loc[q];
  }
  __syncthreads();
  for (int b = tid; b <= kSrhtB; b += 1024) bofs[b] = s_hist[b];
  if (act) s_left[s_hist[m] + atomicAdd(&s_fill[m], 1)] = tid;
  __syncthreads();
  if (tid < kSrhtB) {   // insertion sort of each (tiny) bucket by t
    const int b0 = s_hist[tid], b1 = s_hist[tid + 1];
    for (int i = b0 + 1; i < b1; ++i) {
      const int x = s_left[i];
      int j = i - 1;
      while (j >= b0 && s_left[j] > x) { s_left[j + 1] = s_left[j]; --j; }
      s_left[j + 1] = x;
    }
  }
  __syncthreads();
  if (act) bidx[tid] = s_left[tid];
  if (tpo == 0) return;   // Hartley / cosine: no SRHT gather permutation
  // ---- perm.  Slot s = og*tpo + k is read by quarter-warp lanes of column og & 3 at bin (og >> 2)*tpo + k;
  // a bin's four columns are conflict-free when their outputs sit in distinct 8-bank classes
  // cls(m) = (m + (m >> 5)) & 3, or share one m (a broadcast).  Column c takes class c's outputs; a class
  // with more than G = d_pad/4 outputs moves e_c = n_c - G of them as pairs of equal m: one bin holds
  // both halves of a pair (its own column and a spare column of an under-full class), which frees one
  // slot of column c.  Outputs left over (too few pairs) fill the remaining empty slots in order.
  const int G = d_pad / 4;
  const int h = (m + (m >> 5)) & 3;
  int ncls[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) (void)block_rank(act && h == c, wsum, &ncls[c]);
  int e[4], sp[4], Eb[5], Sb[5];
  Eb[0] = Sb[0] = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    e[c] = max(0, ncls[c] - G);
    sp[c] = max(0, G - ncls[c]);
    Eb[c + 1] = Eb[c] + e[c];
    Sb[c + 1] = Sb[c] + sp[c];
  }
  const int E = min(Eb[4], G);
  for (int i = tid; i < 4 * 512; i += 1024) (&s_lst[0][0])[i] = -1;
  if (tid < 512) s_moved[tid] = 0;
  // pair leaders, in bucket order (equal m adjacent): positions 0, 2, 4, ... of a bucket with a successor
  bool lead = false;
  int lt = 0, lp = 0, lc = 0;
  if (tid < d) {
    lt = s_left[tid];
    const int lm = s_sel[lt] & (kSrhtB - 1);
    lead = ((tid - s_hist[lm]) & 1) == 0 && tid + 1 < s_hist[lm + 1];
    lp = lead ? s_left[tid + 1] : 0;
    lc = (lm + (lm >> 5)) & 3;
  }
  int pr = 0, le = 0, lEb = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {   // (the first barrier publishes the initialisation above)
    int tot;
    const int r = block_rank(lead && lc == c, wsum, &tot);
    if (lc == c) { pr = r; le = e[c]; lEb = Eb[c]; }
  }
  if (lead && pr < le && lEb + pr < G) {
    const int mv = lEb + pr;
    int u = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) u = (Sb[c] <= mv && mv < Sb[c + 1]) ? c : u;
    s_lst[lc][mv] = lt;
    s_lst[u][mv] = lp;
    s_moved[lt] = 1;
    s_moved[lp] = 1;
  }
  __syncthreads();
  // the other outputs of class h in ascending t, into column h's bins outside its reserved range [lo, hi)
  const bool rem = act && !s_moved[tid];
  int rr = 0, lo = 0, hi = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    int tot;
    const int r = block_rank(rem && h == c, wsum, &tot);
    if (h == c) {
      rr = r;
      if (e[c] > 0) { lo = min(Eb[c], G); hi = min(Eb[c] + e[c], G); }
      else if (sp[c] > 0) { lo = min(Sb[c], E); hi = min(Sb[c] + sp[c], E); }
    }
  }
  const int bin = rr < lo ? rr : rr + (hi - lo);
  const bool ovf = rem && bin >= G;
  if (rem && !ovf) s_lst[h][bin] = tid;
  int novf = 0;
  const int orank = block_rank(ovf, wsum, &novf);   // (its barriers publish s_lst)
  if (ovf) s_over[orank] = tid;
  const bool sact = tid < d_pad;
  const int og = tid / tpo, kk = tid - og * tpo, want = og & 3, mi = (og >> 2) * tpo + kk;
  const int sv = sact ? s_lst[want][mi] : -1;
  const bool empty = sact && sv < 0;
  int nemp = 0;
  const int erank = block_rank(empty, wsum, &nemp);   // (its barriers publish s_over)
  if (sact) perm[tid] = empty ? (erank < novf ? s_over[erank] : -1) : sv;
}

// Chunk signs of the sketch's gather, one byte per (chunk c, output group og): bit k set iff
// (-1)^popc(c & a_t) = -1 for slot s = og*TPO + k, t = perm[s], a_t = S_t / B (empty slots: bit clear; their
// accumulators are never stored).  A warp of the sketch reads its 16 groups' bytes as one 16-B sector.
__global__ void k_srht_signs(const int32_t* __restrict__ sel, const int32_t* __restrict__ perm, int d_pad, int tpo,
                             int A, uint8_t* __restrict__ sgnb) {
  const int ng = d_pad / tpo;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)A * ng) return;
  const int c = (int)(p / ng), og = (int)(p - (int64_t)c * ng);
  uint32_t bits = 0;
  for (int k = 0; k < tpo; ++k) {
    const int t = perm[og * tpo + k];
    if (t >= 0 && (__popc((uint32_t)c & ((uint32_t)sel[t] / (uint32_t)kSrhtB)) & 1)) bits |= 1u << k;
  }
  sgnb[p] = (uint8_t)bits;
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

// NEXT-1: structured Omega^T (d x ncols_pad) = (D_s T[:, S])^T * sqrt(n) in fp16 hi + lo, T the orthonormal
// discrete Hartley (kind DHT: cas(2 pi j k / n) / sqrt n) or cosine DCT-II (sqrt(2/n) eps_k cos(pi (2j+1) k / 2n))
// transform; the sqrt(n) scale keeps the entries O(1) so that lo = fp16(v - hi) stays a normal number for
// typical entries (|v - hi - lo| <~ 2^-22 |v|).  The angle's integer part is reduced exactly, then fp64
// sincospi.  Columns j >= n are zero.
__global__ void k_trig_omega(uint64_t seed, int64_t n, int d, int64_t ncols_pad, int kind,
                             const int32_t* __restrict__ sel, __half* __restrict__ hi, __half* __restrict__ lo) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  if (j >= ncols_pad) return;
  __half h = __float2half_rn(0.f), l = __float2half_rn(0.f);
  if (j < n) {
    const int64_t k = sel[t];
    double v;
    if (kind == KS_OMEGA_DHT) {
      double sn, cs;
      sincospi(2.0 * (double)((j * k) % n) / (double)n, &sn, &cs);
      v = cs + sn;
    } else {
      v = (k == 0 ? 1.0 : 1.4142135623730951) * cospi((double)(((2 * j + 1) * k) % (4 * n)) / (2.0 * (double)n));
    }
    v *= (double)rademacher(seed, j);
    h = __double2half(v);
    l = __double2half(v - (double)__half2float(h));
  }
  hi[(int64_t)t * ncols_pad + j] = h;
  lo[(int64_t)t * ncols_pad + j] = l;
}

double gauss_scale(const ks_sketch_desc& D) {
  const double kmax = (double)D.sigma2 + (double)D.nugget;
  int e = (int)std::floor(std::log2(16384.0 / kmax));
  e = std::max(-60, std::min(60, e));
  return std::ldexp(1.0, e);
}

static float coord_scale(const ks_sketch_desc& D) {
  if (D.kernel == KS_KERNEL_STORED) return 1.f;
  if (D.kernel == KS_KERNEL_SQEXP) return (float)std::sqrt(1.4426950408889634 / (2.0 * (double)D.ell * (double)D.ell));
  return (float)(std::sqrt(3.0) / (double)D.ell);
}

ks_status sketch_prepare(const ks_sketch_desc& D, const SketchLayout& L, const float* pts, char* ws,
                         cudaStream_t st, bool need_points) {
  const int srht = D.omega == KS_OMEGA_SRHT;
  if (need_points) {
    const int64_t nb = (L.ncols_pad + 255) / 256;
    // a stored K carries its own scale: amplitude s_j (SRHT) or S (tensor-core path)
    const float sig = D.kernel == KS_KERNEL_STORED ? 1.f : D.sigma2;
    const float amp = srht ? sig : (float)(sig * gauss_scale(D));
    k_pack_points<<<(unsigned)nb, 256, 0, st>>>(pts, D.n, D.dim, L.ncols_pad, coord_scale(D), amp, D.seed,
                                                 srht, reinterpret_cast<float4*>(ws + L.off_pk));
    KS_LAUNCH_CHECK();
  }
  static PerDeviceOnce attr;
  KS_TRY(attr.run([] {
    KS_CUDA_TRY(cudaFuncSetAttribute(k_selection, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSelSmemBits / 8)));
    return KS_OK;
  }));
  const int sel_smem = L.N <= kSelSmemBits ? (int)((L.N + 31) / 32 * 4) : 0;
  if (srht) {
    k_selection<<<1, 1024, sel_smem, st>>>(D.seed, L.N, L.N, D.d, L.d_pad, L.tpo,
                                           reinterpret_cast<uint32_t*>(ws + L.off_bitmap),
                                           reinterpret_cast<int32_t*>(ws + L.off_sel),
                                           reinterpret_cast<uint32_t*>(ws + L.off_tab),
                                           reinterpret_cast<int32_t*>(ws + L.off_bucket_ofs),
                                           reinterpret_cast<int32_t*>(ws + L.off_bucket_idx),
                                           reinterpret_cast<int32_t*>(ws + L.off_perm));
    KS_LAUNCH_CHECK();
    const int64_t ns = (int64_t)L.A * (L.d_pad / L.tpo);
    k_srht_signs<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(reinterpret_cast<const int32_t*>(ws + L.off_sel),
                                                               reinterpret_cast<const int32_t*>(ws + L.off_perm),
                                                               L.d_pad, L.tpo, L.A,
                                                               reinterpret_cast<uint8_t*>(ws + L.off_sgn));
    KS_LAUNCH_CHECK();
  } else if (D.omega == KS_OMEGA_GAUSS) {
    dim3 grid((unsigned)((L.ncols_pad + 255) / 256), (unsigned)D.d);
    k_gauss_omega<<<grid, 256, 0, st>>>(D.seed, D.n, D.d, L.ncols_pad, reinterpret_cast<__half*>(ws + L.off_gauss));
    KS_LAUNCH_CHECK();
  } else {   // Hartley / cosine: S from [0, n) by rejection, then Omega^T (hi, lo)
    k_selection<<<1, 1024, sel_smem, st>>>(D.seed, L.N, D.n, D.d, 0, 0, reinterpret_cast<uint32_t*>(ws + L.off_bitmap),
                                           reinterpret_cast<int32_t*>(ws + L.off_sel),
                                           reinterpret_cast<uint32_t*>(ws + L.off_tab),
                                           reinterpret_cast<int32_t*>(ws + L.off_bucket_ofs),
                                           reinterpret_cast<int32_t*>(ws + L.off_bucket_idx), nullptr);
    KS_LAUNCH_CHECK();
    __half* hi = reinterpret_cast<__half*>(ws + L.off_gauss);
    dim3 grid((unsigned)((L.ncols_pad + 255) / 256), (unsigned)D.d);
    k_trig_omega<<<grid, 256, 0, st>>>(D.seed, D.n, D.d, L.ncols_pad, D.omega,
                                       reinterpret_cast<const int32_t*>(ws + L.off_sel), hi,
                                       hi + (size_t)D.d * L.ncols_pad);
    KS_LAUNCH_CHECK();
  }
  return KS_OK;
}

// ============================================================ NEXT-4: K times a dense given matrix
// W = K Om for a caller-given dense Om (n x d fp32, row-major -- e.g. the sketch's Q, the second pass over K
// of the Nystrom core B = Q^T K Q): the tensor-core contraction of the Hartley / cosine path (NB = 2: Om
// as fp16 hi + lo planes, x sqrt(n) like the trig planes) with the planes transposed from Om in 32 x 32
// tiles (coalesced reads and writes).
__global__ void k_dense_omega(const float* __restrict__ Om, int64_t n, int d, int64_t ncols_pad, float scale,
                              __half* __restrict__ hi, __half* __restrict__ lo) {
  __shared__ float tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int t0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {   // rows j0 + r, columns t0 + threadIdx.x of Om
    const int64_t j = j0 + r;
    const int t = t0 + threadIdx.x;
    tile[r][threadIdx.x] = (j < n && t < d) ? Om[j * d + t] * scale : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {   // plane row t0 + r, columns j0 + threadIdx.x
    const int t = t0 + r;
    const int64_t j = j0 + threadIdx.x;
    if (t < d && j < ncols_pad) {
      const float v = tile[threadIdx.x][r];
      const __half h = __float2half_rn(v);
      hi[(int64_t)t * ncols_pad + j] = h;
      lo[(int64_t)t * ncols_pad + j] = __float2half_rn(v - __half2float(h));
    }
  }
}

ks_status dense_apply_run(const ks_sketch_desc& D0, const float* pts, const float* Om, float* W, char* ws,
                          cudaStream_t st) {
  ks_sketch_desc D = D0;
  D.omega = KS_OMEGA_DHT;   // the layout / launch of the two-plane tensor-core path
  const SketchLayout L = sketch_layout(D);
  const int64_t nb = (L.ncols_pad + 255) / 256;
  k_pack_points<<<(unsigned)nb, 256, 0, st>>>(pts, D.n, D.dim, L.ncols_pad, coord_scale(D),
                                               (float)(D.sigma2 * gauss_scale(D)), D.seed, 0,
                                               reinterpret_cast<float4*>(ws + L.off_pk));
  KS_LAUNCH_CHECK();
  __half* hi = reinterpret_cast<__half*>(ws + L.off_gauss);
  k_dense_omega<<<dim3((unsigned)((L.ncols_pad + 31) / 32), (unsigned)((D.d + 31) / 32)), dim3(32, 8), 0, st>>>(
      Om, D.n, D.d, L.ncols_pad, (float)std::sqrt((double)D.n), hi, hi + (size_t)D.d * L.ncols_pad);
  KS_LAUNCH_CHECK();
  return gauss_sketch_run(D, L, 0, D.n, W, ws, st, nullptr);
}

size_t dense_apply_ws(const ks_sketch_desc& D0) {
  ks_sketch_desc D = D0;
  D.omega = KS_OMEGA_DHT;
  return sketch_layout(D).bytes;
}

// ============================================================ fused SRHT kernel
// One CTA = 8 rows of Y (128 threads, 4 CTAs per SM, whose phases interleave); loops over the column
// chunks c of K.  The tile W is double buffered, so a chunk needs 2 barriers (after phase A, after B).
// Shared tile W: column l (0..511) of the chunk holds its 8 row values at
// A(l, r) = l*8 + (l >> 5)*8 + r (the (l >> 5) pad makes phase B conflict-free).
//   phase A : thread (rg = t&3, cg = t>>2) evaluates K*s for the row pair 2rg, 2rg+1 (packed f32x2)
//             at columns l = cg + 32q, q < 16, butterflies over l bits 5-8 in registers (the first level
//             with the amplitudes folded into FFMAs), stores W.
//   phase B : thread (rp = t&7, g = t>>3) loads row rp at l = 32g + b, b < 32, into register pairs
//             (b, b+16), butterflies over l bits 0-3 (packed) and bit 4, stores back.  W now holds
//             FWHT_B of the chunk (natural order).
//   phase C : thread (rq = t&1, og = t>>1) accumulates its TPO gather slots s = og*TPO + k (output
//             t = perm[s]) for rows 4rq..4rq+3: acc += sgn[c][s] * W[m_t][4rq .. 4rq+3] (packed).
// Packed f32x2 arithmetic issues once per row pair: the FP32 pipe does the same lane-ops, but the
// kernel is no longer bound by issue slots.  The chunk's packed points are staged in shared memory
// by cp.async one chunk ahead.
constexpr int kSrhtThreads = 128;
KS_DEVINL int srht_w(int l, int r) { return l * 8 + (l >> 5) * 8 + r; }
constexpr int kSrhtSmemFloats = kSrhtB * 8 + (kSrhtB / 32) * 8;   // 16.5 KB per buffer
constexpr int kSrhtSmemBytes = 2 * kSrhtSmemFloats * 4 + 2 * kSrhtB * 16;   // + 2 x 8 KB point tiles

KS_DEVINL void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
KS_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
KS_DEVINL void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Stored K: this thread's 32 values of a chunk (rows i0, i1 packed; columns jb + 32 q), zero beyond n.
KS_DEVINL void load_k32(f2_t (&kv)[16], const float* kr0, const float* kr1, int64_t jb, int64_t ncols) {
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int64_t j = jb + 32 * q;
    kv[q] = j < ncols ? f2(__ldg(kr0 + j), __ldg(kr1 + j)) : 0ull;
  }
}

template <int DIM, int KIND, int TPO>
__global__ void __launch_bounds__(kSrhtThreads, 4)
k_sketch_srht(const float4* __restrict__ pk, const int32_t* __restrict__ sel, const int32_t* __restrict__ perm,
              const uint8_t* __restrict__ sgnb, int64_t row_begin, int64_t row_end, int A, int d, int d_pad,
              float out_scale, float nugget, float* __restrict__ Y, const float* __restrict__ Kst, int64_t ldk,
              int64_t ncols) {
  extern __shared__ __align__(16) float Wbuf[];   // [2][kSrhtSmemFloats], chunk c uses half c & 1
  float4* Pbuf = reinterpret_cast<float4*>(Wbuf + 2 * kSrhtSmemFloats);   // [2][kSrhtB] packed points
  const int t = threadIdx.x;
  const int rg = t & 3, cg = t >> 2;
  const int rp = t & 7, g = t >> 3;
  const int rq = t & 1, og = t >> 1;
  const int64_t row0 = row_begin + (int64_t)blockIdx.x * kSrhtRows;
  const int oA = srht_w(cg, 2 * rg);       // + 264 q   (= srht_w(cg + 32 q, 2 rg))
  const int oB = 264 * g + rp;             // + 8 b     (= srht_w(32 g + b, rp))

  f2_t xi2[3];
  const float *kr0 = nullptr, *kr1 = nullptr;   // stored K (NEXT-2): this thread's two rows
  {
    int64_t i0 = row0 + 2 * rg, i1 = i0 + 1;
    if (i0 >= row_end) i0 = row_end - 1;
    if (i1 >= row_end) i1 = row_end - 1;
    const float4 a = pk[i0], b = pk[i1];
    xi2[0] = f2(a.x, b.x); xi2[1] = f2(a.y, b.y); xi2[2] = f2(a.z, b.z);
    if (KIND == KS_KERNEL_STORED) { kr0 = Kst + (i0 - row_begin) * ldk; kr1 = Kst + (i1 - row_begin) * ldk; }
  }
  int wofs[TPO];
#pragma unroll
  for (int k = 0; k < TPO; ++k) {
    const int tt = perm[og * TPO + k];
    wofs[k] = srht_w(tt >= 0 ? (sel[tt] & (kSrhtB - 1)) : 0, 4 * rq);
  }
  f2_t kpre[KIND == KS_KERNEL_STORED ? 16 : 1];
  if constexpr (KIND == KS_KERNEL_STORED) load_k32(kpre, kr0, kr1, cg, ncols);
  f2_t acc[TPO][2];
#pragma unroll
  for (int k = 0; k < TPO; ++k) acc[k][0] = acc[k][1] = 0ull;
  // chunk 0's points
#pragma unroll
  for (int q = 0; q < kSrhtB / kSrhtThreads; ++q) cp_async16(Pbuf + t + kSrhtThreads * q, pk + t + kSrhtThreads * q);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  for (int c = 0; c < A; ++c) {
    float* W = Wbuf + (c & 1) * kSrhtSmemFloats;
    if (c + 1 < A) {   // chunk c+1's points into the other tile (its last reader, phase A of c-1, is done)
      float4* pn = Pbuf + ((c + 1) & 1) * kSrhtB;
      const float4* src = pk + (int64_t)(c + 1) * kSrhtB;
#pragma unroll
      for (int q = 0; q < kSrhtB / kSrhtThreads; ++q) cp_async16(pn + t + kSrhtThreads * q, src + t + kSrhtThreads * q);
      cp_async_commit();
    }
    // ---------------- phase A (writes the other buffer than chunk c-1's phase C reads: no barrier before it)
    {
      const float4* pc = Pbuf + (c & 1) * kSrhtB + cg;
      f2_t v[16];
      if constexpr (KIND == KS_KERNEL_STORED) {   // K streamed from HBM: this chunk's values were loaded
#pragma unroll                                 // (in flight) during the previous chunk's phases B and C
        for (int q = 0; q < 16; ++q) v[q] = kpre[q];
#pragma unroll
        for (int q = 0; q < 16; q += 2) {   // level h = 1 with the signs a_j = s_j folded in
          const float4 p0 = pc[32 * q], p1 = pc[32 * (q + 1)];
          const f2_t m0 = f2mul(v[q], f2s(p0.w)), k1 = v[q + 1];
          v[q] = f2fma(k1, f2s(p1.w), m0);
          v[q + 1] = f2fma(k1, f2s(-p1.w), m0);
        }
      } else {
#pragma unroll
      for (int q = 0; q < 16; q += 2) {   // level h = 1 with the amplitudes a_j = s_j sigma^2 folded in
        const float4 p0 = pc[32 * q], p1 = pc[32 * (q + 1)];
        const f2_t k0 = cov_kappa2<DIM, KIND>(xi2, p0), k1 = cov_kappa2<DIM, KIND>(xi2, p1);
        const f2_t m0 = f2mul(k0, f2s(p0.w));
        v[q] = f2fma(k1, f2s(p1.w), m0);
        v[q + 1] = f2fma(k1, f2s(-p1.w), m0);
      }
      }
#pragma unroll
      for (int h = 2; h < 16; h <<= 1)
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (!(q & h)) {
            const f2_t x = v[q], y = v[q + h];
            v[q] = f2add(x, y);
            v[q + h] = f2sub(x, y);
          }
#pragma unroll
      for (int q = 0; q < 16; ++q) *reinterpret_cast<f2_t*>(W + oA + 264 * q) = v[q];
      if constexpr (KIND == KS_KERNEL_STORED)
        if (c + 1 < A) load_k32(kpre, kr0, kr1, (int64_t)(c + 1) * kSrhtB + cg, ncols);
    }
    __syncthreads();
    // ---------------- phase B: pairs (b, b+16) packed for l bits 0-3, then bit 4 inside the pairs
    // (measured: a row-pair form -- 64 threads, LDS.64 / STS.64, all five levels in registers -- halves the
    // shared-memory instructions but is slower, c4 51.6 -> 55.3 ms, c5 811 -> 881 ms: half the warps idle)
    {
      float* wB = W + oB;
      f2_t u[16];
#pragma unroll
      for (int b = 0; b < 16; ++b) u[b] = f2(wB[8 * b], wB[8 * (b + 16)]);
#pragma unroll
      for (int h = 1; h < 16; h <<= 1)
#pragma unroll
        for (int b = 0; b < 16; ++b)
          if (!(b & h)) {
            const f2_t x = u[b], y = u[b + h];
            u[b] = f2add(x, y);
            u[b + h] = f2sub(x, y);
          }
#pragma unroll
      for (int b = 0; b < 16; ++b) {
        const float x = f2lo(u[b]), y = f2hi(u[b]);
        wB[8 * b] = x + y;
        wB[8 * (b + 16)] = x - y;
      }
    }
    cp_async_wait_all();   // chunk c+1's points visible to all threads after the barrier
    __syncthreads();
    // ---------------- phase C (the chunk's sign bits: one byte per output group, 64 bytes per chunk)
    float sg[TPO];
    {
      const uint32_t sb = __ldg(sgnb + (int64_t)c * (d_pad / TPO) + og);
#pragma unroll
      for (int k = 0; k < TPO; ++k) sg[k] = __uint_as_float(((sb << (31 - k)) & 0x80000000u) | 0x3f800000u);
    }
#pragma unroll
    for (int k = 0; k < TPO; ++k) {
      const ulonglong2 w = *reinterpret_cast<const ulonglong2*>(W + wofs[k]);
      acc[k][0] = f2fma(f2s(sg[k]), w.x, acc[k][0]);
      acc[k][1] = f2fma(f2s(sg[k]), w.y, acc[k][1]);
    }
  }
  // ---------------- epilogue: scale, nugget (by index, reading L9), store.
#pragma unroll
  for (int k = 0; k < TPO; ++k) {
    const int tt = perm[og * TPO + k];
    if (tt < 0) continue;
    const uint32_t S = (uint32_t)sel[tt];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int64_t i = row0 + 4 * rq + rr;
      if (i >= row_end) continue;
      const float si = pk[i].w > 0.f ? 1.f : -1.f;
      const float h = (__popcll((unsigned long long)i & (unsigned long long)S) & 1) ? -1.f : 1.f;
      const f2_t a2 = acc[k][rr >> 1];
      const float a = (rr & 1) ? f2hi(a2) : f2lo(a2);
      Y[(i - row_begin) * (int64_t)d + tt] = fmaf(nugget * si, h * out_scale, a * out_scale);
    }
  }
}

template <int DIM, int KIND, int TPO>
static ks_status launch_srht(const SketchLayout& L, const ks_sketch_desc& D, int64_t rb, int64_t re, float* Y,
                             char* ws, cudaStream_t st, const StoredK* sk) {
  auto kern = k_sketch_srht<DIM, KIND, TPO>;
  const int smem = kSrhtSmemBytes;
  KS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const unsigned grid = (unsigned)((re - rb + kSrhtRows - 1) / kSrhtRows);
  kern<<<grid, kSrhtThreads, smem, st>>>(reinterpret_cast<const float4*>(ws + L.off_pk),
                                reinterpret_cast<const int32_t*>(ws + L.off_sel),
                                reinterpret_cast<const int32_t*>(ws + L.off_perm),
                                reinterpret_cast<const uint8_t*>(ws + L.off_sgn), rb, re, L.A, D.d, L.d_pad,
                                (float)(1.0 / std::sqrt((double)L.N)), D.nugget, Y, sk ? sk->K : nullptr,
                                sk ? sk->ldk : 0, D.n);
  KS_LAUNCH_CHECK();
  return KS_OK;
}

template <int DIM, int KIND>
static ks_status dispatch_tpo(const SketchLayout& L, const ks_sketch_desc& D, int64_t rb, int64_t re, float* Y,
                              char* ws, cudaStream_t st, const StoredK* sk = nullptr) {
  switch (L.tpo) {
    case 1: return launch_srht<DIM, KIND, 1>(L, D, rb, re, Y, ws, st, sk);
    case 2: return launch_srht<DIM, KIND, 2>(L, D, rb, re, Y, ws, st, sk);
    case 4: return launch_srht<DIM, KIND, 4>(L, D, rb, re, Y, ws, st, sk);
    case 8: return launch_srht<DIM, KIND, 8>(L, D, rb, re, Y, ws, st, sk);
  }
  return fail(KS_ERR_UNSUPPORTED, "unsupported SRHT output width");
}

ks_status sketch_run(const ks_sketch_desc& D, const SketchLayout& L, int64_t rb, int64_t re, float* Y, char* ws,
                     cudaStream_t st, const StoredK* sk) {
  if (re <= rb) return KS_OK;
  if (D.omega != KS_OMEGA_SRHT) return gauss_sketch_run(D, L, rb, re, Y, ws, st, sk);   // Gaussian, Hartley, cosine
  if (sk) return dispatch_tpo<1, KS_KERNEL_STORED>(L, D, rb, re, Y, ws, st, sk);
  const bool se = D.kernel == KS_KERNEL_SQEXP;
  switch (D.dim) {
    case 1: return se ? dispatch_tpo<1, KS_KERNEL_SQEXP>(L, D, rb, re, Y, ws, st)
                      : dispatch_tpo<1, KS_KERNEL_MATERN32>(L, D, rb, re, Y, ws, st);
    case 2: return se ? dispatch_tpo<2, KS_KERNEL_SQEXP>(L, D, rb, re, Y, ws, st)
                      : dispatch_tpo<2, KS_KERNEL_MATERN32>(L, D, rb, re, Y, ws, st);
    case 3: return se ? dispatch_tpo<3, KS_KERNEL_SQEXP>(L, D, rb, re, Y, ws, st)
                      : dispatch_tpo<3, KS_KERNEL_MATERN32>(L, D, rb, re, Y, ws, st);
  }
  return fail(KS_ERR_INVALID_ARGUMENT, "dim");
}

// ============================================================ Omega-apply
// SRHT: X[j, col] = s_j / sqrt(N) * (H_N scatter_S(Z[:, col]))[j]  (Omega Z with Omega^T = (1/sqrt N) H[S,:] D_s).
// Per chunk c (rows j = cB + l):  u[m] = sum_{t: m_t = m} (-1)^popc(c & a_t) Z[t, col];  X = s o FWHT_B(u).
// CTA = (chunk c, 32-column tile of Z): the bucket CSR and the chunk signs of the d outputs are staged in
// shared memory, u = scatter(Z) (a warp per bucket row, lanes along the columns), FWHT_512 as three radix-8
// passes in shared memory, then coalesced row writes of s_j u / sqrt N.
constexpr int kOaCols = 32;
__global__ void __launch_bounds__(256) k_omega_apply_srht(const float* __restrict__ Z, int m, int d,
                                                          const uint32_t* __restrict__ tab,
                                                          const int32_t* __restrict__ bofs,
                                                          const int32_t* __restrict__ bidx, uint64_t seed,
                                                          int64_t n, int64_t row_begin, int64_t row_end,
                                                          int c_first, float scale, float* __restrict__ X) {
  constexpr int ld = kOaCols + 1;
  extern __shared__ float u[];          // [kSrhtB][ld]
  __shared__ int s_bofs[kSrhtB + 1];
  __shared__ int s_bidx[512];
  __shared__ float s_sgn[512];          // (-1)^popc(c & a_t), by output t
  __shared__ float srow[kSrhtB];        // s_j / sqrt N of this chunk's rows
  const int c = c_first + blockIdx.x;
  const int col0 = kOaCols * blockIdx.y, ncol = min(kOaCols, m - col0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int l = tid; l <= kSrhtB; l += 256) s_bofs[l] = bofs[l];
  for (int t = tid; t < d; t += 256) {
    s_bidx[t] = bidx[t];
    s_sgn[t] = (__popc((uint32_t)c & (tab[t] >> 16)) & 1) ? -1.f : 1.f;
  }
  for (int l = tid; l < kSrhtB; l += 256) {
    const int64_t j = (int64_t)c * kSrhtB + l;
    srow[l] = (j < n) ? rademacher(seed, j) * scale : 0.f;
  }
  __syncthreads();
  // ---- scatter: u[l][col] = sum over the outputs t of bucket l of sgn_t Z[t][col]
  for (int l = warp; l < kSrhtB; l += 8) {
    float acc = 0.f;
    if (lane < ncol) {
      for (int q = s_bofs[l]; q < s_bofs[l + 1]; ++q) {
        const int tt = s_bidx[q];
        acc = fmaf(s_sgn[tt], Z[(int64_t)tt * m + col0 + lane], acc);
      }
    }
    u[l * ld + lane] = acc;
  }
  __syncthreads();
  // ---- FWHT_512: three radix-8 passes (strides 1, 8, 64); item = (group g of 8, column)
#pragma unroll 1
  for (int h = 1; h < kSrhtB; h *= 8) {
    for (int it = tid; it < 64 * kOaCols; it += 256) {
      const int g = it >> 5, col = it & 31;
      const int base = (g / h) * 8 * h + (g % h);
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = u[(base + k * h) * ld + col];
#pragma unroll
      for (int hh = 1; hh < 8; hh <<= 1)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (!(k & hh)) {
            const float x = v[k], y = v[k + hh];
            v[k] = x + y;
            v[k + hh] = x - y;
          }
#pragma unroll
      for (int k = 0; k < 8; ++k) u[(base + k * h) * ld + col] = v[k];
    }
    __syncthreads();
  }
  // ---- X rows of this chunk: a warp per row, lanes along the columns (coalesced row writes)
  for (int l = warp; l < kSrhtB; l += 8) {
    const int64_t j = (int64_t)c * kSrhtB + l;
    if (j < row_begin || j >= row_end || j >= n || lane >= ncol) continue;
    X[(j - row_begin) * (int64_t)m + col0 + lane] = srow[l] * u[l * ld + lane];
  }
}

// Gaussian: X[j, :] = (1/sqrt d) sum_t Omega[j, t] Z[t, :].  Thread = row j, up to 32 columns per pass in
// registers (one read of Omega^T per pass, coalesced across the rows of a warp), the t loop unrolled by 8 so
// eight Omega loads are in flight together; Z broadcast from shared memory.
__global__ void __launch_bounds__(256) k_omega_apply_gauss(const __half* __restrict__ omT, const __half* __restrict__ omT_lo,
                                                           int64_t ldo, const float* __restrict__ Z, int m, int d,
                                                           int64_t row_begin, int64_t row_end, float scale,
                                                           float* __restrict__ X) {
  extern __shared__ float zs[];  // d x m
  for (int p = threadIdx.x; p < d * m; p += blockDim.x) zs[p] = Z[p];
  __syncthreads();
  const int64_t j = row_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= row_end) return;
  float* xr = X + (j - row_begin) * (int64_t)m;
  for (int c0 = 0; c0 < m; c0 += 32) {
    const int nc = min(32, m - c0);
    float acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = 0.f;
    for (int t0 = 0; t0 < d; t0 += 8) {
      float o[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u;
        o[u] = 0.f;
        if (t < d) {
          o[u] = __half2float(omT[(int64_t)t * ldo + j]);
          if (omT_lo) o[u] += __half2float(omT_lo[(int64_t)t * ldo + j]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u;
        if (t < d) {
          const float* zr = zs + t * m + c0;
          if ((m & 3) == 0) {   // 16-B aligned rows of Z: LDS.128 broadcasts
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4)
              if (4 * q4 < nc) {
                const float4 z = *reinterpret_cast<const float4*>(zr + 4 * q4);
                acc[4 * q4 + 0] = fmaf(o[u], z.x, acc[4 * q4 + 0]);
                acc[4 * q4 + 1] = fmaf(o[u], z.y, acc[4 * q4 + 1]);
                acc[4 * q4 + 2] = fmaf(o[u], z.z, acc[4 * q4 + 2]);
                acc[4 * q4 + 3] = fmaf(o[u], z.w, acc[4 * q4 + 3]);
              }
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (q < nc) acc[q] = fmaf(o[u], zr[q], acc[q]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (q < nc) xr[c0 + q] = acc[q] * scale;
  }
}

ks_status omega_apply_run(const ks_sketch_desc& D, const SketchLayout& L, const float* Z, int m, int64_t rb,
                          int64_t re, float* X, char* ws, cudaStream_t st) {
  if (re <= rb) return KS_OK;
  if (D.omega == KS_OMEGA_SRHT) {
    const int c0 = (int)(rb / kSrhtB), c1 = (int)((re - 1) / kSrhtB);
    const int smem = kSrhtB * (kOaCols + 1) * (int)sizeof(float);
    KS_CUDA_TRY(cudaFuncSetAttribute(k_omega_apply_srht, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_omega_apply_srht<<<dim3((unsigned)(c1 - c0 + 1), (unsigned)((m + kOaCols - 1) / kOaCols)), 256, smem, st>>>(
        Z, m, D.d, reinterpret_cast<const uint32_t*>(ws + L.off_tab),
        reinterpret_cast<const int32_t*>(ws + L.off_bucket_ofs), reinterpret_cast<const int32_t*>(ws + L.off_bucket_idx),
        D.seed, D.n, rb, re, c0, (float)(1.0 / std::sqrt((double)L.N)), X);
    KS_LAUNCH_CHECK();
  } else {
    const int smem = D.d * m * (int)sizeof(float);
    KS_CUDA_TRY(cudaFuncSetAttribute(k_omega_apply_gauss, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const unsigned grid = (unsigned)((re - rb + 255) / 256);
    const __half* hi = reinterpret_cast<const __half*>(ws + L.off_gauss);
    const bool trig = D.omega != KS_OMEGA_GAUSS;   // Hartley / cosine: hi + lo, scaled by sqrt(n)
    k_omega_apply_gauss<<<grid, 256, smem, st>>>(hi, trig ? hi + (size_t)D.d * L.ncols_pad : nullptr, L.ncols_pad, Z,
                                                  m, D.d, rb, re,
                                                  (float)(1.0 / std::sqrt((double)(trig ? D.n : D.d))), X);
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
    if (D.omega == KS_OMEGA_GAUSS) return fail(KS_ERR_INVALID_ARGUMENT, "no selection for the Gaussian Omega");
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
