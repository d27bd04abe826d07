// ks_gauss.cu -- Gaussian-Omega sketch on the 5th-generation tensor cores (sm_100a).
//
//   Y = K Omega,  Omega_jt = fp16(z_jt) / sqrt(d)       (reading L6)
//
// "The product B Omega involves O(n^2 d) flops": a true dense
// contraction, so it runs on tcgen05.  K is never stored: producer warps
// evaluate a 128 x 64 tile of S*K in registers (S = gauss_scale, a power of two
// keeping the split in fp16's normal range), split it S*K = K_hi + K_lo (K_hi =
// S*K truncated to 10 fraction bits, exact in fp16; K_lo = fp16_RN(S*K - K_hi))
// and write both halves into shared memory in the UMMA K-major SWIZZLE_128B
// layout.  Omega^T tiles (d x 64 fp16) arrive by TMA.  One elected thread issues
//     acc += K_hi Omega ;  acc += K_lo Omega        (M=128, N=d, K=16 per MMA)
// into ONE fp32 TMEM accumulator.  Omega's fp16 values are exact tensor-core
// operands, so the operand error is the <= 2^-21 relative split error of K.
// The tensor core's fp32 accumulation is not round-to-nearest (its error grows
// linearly with the number of MMAs accumulated: tools/gauss_precision.py), so
// the column loop is cut into segments whose partial sums are folded by dedicated warps into a running
// sum kept in the other half of TMEM, with fp32 round-to-nearest adds.
//
#include "ks_common.cuh"
#include "ks_internal.h"
#include "ks_tc.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

namespace ks {

constexpr int kGaussSegKb = 16;   // 1024 columns of K per TMEM accumulation segment
#ifndef KS_GAUSS_DRAINERS
#define KS_GAUSS_DRAINERS 4   // drainer warps per CTA (4 or 8); 8 measured slower: c3 sketch 3.544 vs 3.492 ms
#endif
constexpr int kGDrainWarps = KS_GAUSS_DRAINERS;
#ifndef KS_GAUSS_DRAIN_U
#define KS_GAUSS_DRAIN_U 2   // 16-column TMEM loads in flight per drainer step
#endif
constexpr int kDrainU = KS_GAUSS_DRAIN_U;
#ifndef KS_GAUSS_PRODUCERS
#define KS_GAUSS_PRODUCERS 8   // K-tile producer warps per CTA (8: 4 rows per thread; 16: 2 rows per thread)
#endif
constexpr int kGProdWarps = KS_GAUSS_PRODUCERS;
constexpr int kGRowsPT = 128 / (4 * kGProdWarps);   // rows per producer thread (8 column groups of 8)
static_assert(kGRowsPT == 2 || kGRowsPT == 4, "8 or 16 producer warps");
constexpr int kGThreads = 128 + 32 * kGProdWarps + 32 * kGDrainWarps;
constexpr int kATileBytes = kGaussBM * kGaussBK * 2;  // 16 KB per fp16 half

KS_DEVINL uint32_t pack_half2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// fp32 -> (hi, lo) fp16 pair: hi = x truncated to 10 fraction bits (exact in fp16 for the normal range),
// lo = fp16_RN(x - hi) (x - hi is exact in fp32), so |x - hi - lo| <= 2^-21 |x|.
// One producer thread's share of a stage: rows 4rq..4rq+3 (two packed row pairs) x columns j0..j0+7 of
// S*K, split hi/lo and stored in the UMMA K-major SW128 layout.  The covariance and the lo = x - hi
// subtraction run on packed f32x2 row pairs (one issue slot per two rows).
template <int DIM, int KIND>
KS_DEVINL void produce_tile(const f2_t (&xi2)[kGRowsPT / 2][3], const int64_t (&irow)[kGRowsPT], const float4 (&pts)[8],
                            int64_t j0, bool diag, float nugget, uint8_t* a_hi, uint8_t* a_lo, int rq, int cq) {
#pragma unroll
  for (int pr = 0; pr < kGRowsPT / 2; ++pr) {
    f2_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = cov_signed2<DIM, KIND>(xi2[pr], pts[q]);
    if (diag) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float a = f2lo(v[q]), b = f2hi(v[q]);
        if (j0 + q == irow[2 * pr]) a += nugget;       // nugget by index (reading L9)
        if (j0 + q == irow[2 * pr + 1]) b += nugget;
        v[q] = f2(a, b);
      }
    }
    uint32_t hi[2][4], lo[2][4];
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      const f2_t h0 = f2(__uint_as_float(__float_as_uint(f2lo(v[q])) & 0xFFFFE000u),
                         __uint_as_float(__float_as_uint(f2hi(v[q])) & 0xFFFFE000u));
      const f2_t h1 = f2(__uint_as_float(__float_as_uint(f2lo(v[q + 1])) & 0xFFFFE000u),
                         __uint_as_float(__float_as_uint(f2hi(v[q + 1])) & 0xFFFFE000u));
      const f2_t l0 = f2sub(v[q], h0), l1 = f2sub(v[q + 1], h1);   // exact in fp32
      hi[0][q >> 1] = pack_half2(f2lo(h0), f2lo(h1));
      hi[1][q >> 1] = pack_half2(f2hi(h0), f2hi(h1));
      lo[0][q >> 1] = pack_half2(f2lo(l0), f2lo(l1));
      lo[1][q >> 1] = pack_half2(f2hi(l0), f2hi(l1));
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = kGRowsPT * rq + 2 * pr + h;
      const uint32_t off = (uint32_t)r * 128u + ((uint32_t)(cq ^ (r & 7)) << 4);
      sts128(smem_u32(a_hi + off), hi[h][0], hi[h][1], hi[h][2], hi[h][3]);   // st.shared: the tile pointers
      sts128(smem_u32(a_lo + off), lo[h][0], lo[h][1], lo[h][2], lo[h][3]);   // are generic (aligned base)
    }
  }
}

// Stored K (NEXT-2): the same tile from K in HBM, v = K[i][j] * a_j (a_j = S), no evaluation.  The loads
// of the next stage are issued right after this stage's tile is stored (load_tile_stored), so they are in
// flight while the producer waits on the ring barriers.
KS_DEVINL void load_tile_stored(const float* __restrict__ Kst, int64_t ldk, int64_t ncols, const int64_t (&irow)[kGRowsPT],
                                int64_t row_last, int64_t j0, float (&kv)[kGRowsPT][8]) {
#pragma unroll
  for (int r = 0; r < kGRowsPT; ++r) {
    const float* kr = Kst + (irow[r] <= row_last ? irow[r] : row_last) * ldk + j0;
    if (j0 + 8 <= ncols) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(kr)), b = __ldg(reinterpret_cast<const float4*>(kr + 4));
      kv[r][0] = a.x; kv[r][1] = a.y; kv[r][2] = a.z; kv[r][3] = a.w;
      kv[r][4] = b.x; kv[r][5] = b.y; kv[r][6] = b.z; kv[r][7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) kv[r][q] = j0 + q < ncols ? __ldg(kr + q) : 0.f;
    }
  }
}
KS_DEVINL void produce_tile_stored(const float (&kv)[kGRowsPT][8], const int64_t (&irow)[kGRowsPT], const float4 (&pts)[8],
                                   int64_t j0, bool diag, float nugget, uint8_t* a_hi, uint8_t* a_lo, int rq, int cq) {
#pragma unroll
  for (int pr = 0; pr < kGRowsPT / 2; ++pr) {
    f2_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = f2mul(f2(kv[2 * pr][q], kv[2 * pr + 1][q]), f2s(pts[q].w));
    if (diag) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float a = f2lo(v[q]), b = f2hi(v[q]);
        if (j0 + q == irow[2 * pr]) a += nugget;
        if (j0 + q == irow[2 * pr + 1]) b += nugget;
        v[q] = f2(a, b);
      }
    }
    uint32_t hi[2][4], lo[2][4];
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      const f2_t h0 = f2(__uint_as_float(__float_as_uint(f2lo(v[q])) & 0xFFFFE000u),
                         __uint_as_float(__float_as_uint(f2hi(v[q])) & 0xFFFFE000u));
      const f2_t h1 = f2(__uint_as_float(__float_as_uint(f2lo(v[q + 1])) & 0xFFFFE000u),
                         __uint_as_float(__float_as_uint(f2hi(v[q + 1])) & 0xFFFFE000u));
      const f2_t l0 = f2sub(v[q], h0), l1 = f2sub(v[q + 1], h1);
      hi[0][q >> 1] = pack_half2(f2lo(h0), f2lo(h1));
      hi[1][q >> 1] = pack_half2(f2hi(h0), f2hi(h1));
      lo[0][q >> 1] = pack_half2(f2lo(l0), f2lo(l1));
      lo[1][q >> 1] = pack_half2(f2hi(l0), f2hi(l1));
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = kGRowsPT * rq + 2 * pr + h;
      const uint32_t off = (uint32_t)r * 128u + ((uint32_t)(cq ^ (r & 7)) << 4);
      sts128(smem_u32(a_hi + off), hi[h][0], hi[h][1], hi[h][2], hi[h][3]);
      sts128(smem_u32(a_lo + off), lo[h][0], lo[h][1], lo[h][2], lo[h][3]);
    }
  }
}

// Drainer step over 16 U columns of this warp's 32 TMEM lanes: running sum (columns DN + c) += segment
// accumulator (columns c), fp32 round-to-nearest; the last segment scales and stores the row of Y.  All
// loads of the step are in flight together (one tcgen05.wait::ld), so a segment boundary -- where the MMA
// waits for the drain -- costs one TMEM round trip per 16 U columns instead of two per 16.
template <int U>
KS_DEVINL void drain_cols(uint32_t tl, int DN, int c0, bool first, bool last, bool ok, float* yr, float out_scale) {
  uint32_t a[U][16], b[U][16];
#pragma unroll
  for (int u = 0; u < U; ++u) tmem_ld16_issue(tl + (uint32_t)(c0 + 16 * u), a[u]);
  if (!first) {
#pragma unroll
    for (int u = 0; u < U; ++u) tmem_ld16_issue(tl + (uint32_t)(DN + c0 + 16 * u), b[u]);
  }
  tmem_wait_ld();
#pragma unroll
  for (int u = 0; u < U; ++u) {
    tmem_pin16(a[u]);
    float v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(a[u][q]);
    if (!first) {
      tmem_pin16(b[u]);
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] += __uint_as_float(b[u][q]);
    }
    if (last) {
      if (ok) {
        float4* dst = reinterpret_cast<float4*>(yr + c0 + 16 * u);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          dst[q] = make_float4(v[4 * q] * out_scale, v[4 * q + 1] * out_scale, v[4 * q + 2] * out_scale,
                               v[4 * q + 3] * out_scale);
      }
    } else {
      tmem_st16(tl + (uint32_t)(DN + c0 + 16 * u), v);
    }
  }
}

// ------------------------------------------------------------------ 2-CTA kernel (cta_group::2)
// A CTA pair (cluster of 2, same TPC) computes a 256-row tile with M = 256 MMAs issued by the leader:
// each CTA supplies its own 128 rows of K (A operand, produced in its smem) and HALF of Omega^T
// (B operand, N/2 = d/2 rows by TMA); the accumulator rows live in each CTA's own TMEM.  This halves
// the shared-memory operand traffic per SM of the 1-CTA kernel (which is smem-bandwidth bound).
// Barriers: the MMA waits on the LEADER's full[s] (producers of both CTAs arrive remotely; both TMAs
// complete_tx on it) and acce[b] (drainers of both CTAs arrive); its commits multicast to both CTAs'
// empty[s] / accf[b].
constexpr int kG2Stages = 4;
constexpr int kPtsStages = 8;                       // ring of the stages' packed points (1 KB each)
constexpr int kPtsBytes = kGaussBK * 16;

KS_DEVINL uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
KS_DEVINL uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
KS_DEVINL void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-D tensor copy global -> own shared memory, completing on an mbarrier of this CTA.
KS_DEVINL void tma_load_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
KS_DEVINL float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
KS_DEVINL void tma_load_2d_2cta(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
KS_DEVINL void umma_f16_2cta(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
KS_DEVINL void umma_commit_2cta(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

// NB = 1: Gaussian Omega (one fp16 plane); NB = 2: Hartley / cosine Omega as fp16 hi + lo planes (NEXT-1),
// a third MMA per K step (K_hi Omega_lo) and 3 pipeline stages (the B tiles double).
template <int DIM, int KIND, int NB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGThreads, 1)
k_sketch_gauss2(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmP,
                const float4* __restrict__ pk, int64_t row_begin,
                int64_t row_end, int nkb_all, int seg_kb, int DN, float nugget, float out_scale,
                float* __restrict__ Y0, float* __restrict__ Y1, int dbg, const float* __restrict__ Kst, int64_t ldk,
                int64_t ncols) {
  // split-K: blockIdx.y selects the half of the column blocks (Y0 gets the first half's partial sum,
  // Y1 the second's; k_add_halves adds them) so that the row tiles fill a whole number of waves.
  const int kh = blockIdx.y, nkb_a = gridDim.y > 1 ? nkb_all / 2 : nkb_all;
  const int kb0 = kh * nkb_a, nkb = kh ? nkb_all - nkb_a : nkb_a;
  float* __restrict__ Y = kh ? Y1 : Y0;
  constexpr int NST = NB == 1 ? kG2Stages : 3;
  const int kBHalfBytes = (DN / 2) * kGaussBK * 2;
  const int kBStage = NB * kBHalfBytes;
  const uint32_t kTmemCols = (2 * DN <= 32) ? 32 : (2 * DN <= 64) ? 64 : (2 * DN <= 128) ? 128 : (2 * DN <= 256) ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_hi = smem;
  uint8_t* a_lo = smem + NST * kATileBytes;
  uint8_t* b_t = a_lo + NST * kATileBytes;
  // [kPtsStages][8 groups][8 points]: TMA SWIZZLE_128B stores point 8g + q of a stage at 16-B chunk q ^ g of
  // its 128-B row g, so the 8 lanes reading 8 different groups at the same q hit 8 different bank groups.
  float4* pring = reinterpret_cast<float4*>(b_t + NST * kBStage);
  uint64_t* bars = reinterpret_cast<uint64_t*>(pring + kPtsStages * kGaussBK);
  // full[S], empty[S], accf[2], acce[2], pfull[PS], pempty[PS], lfull[S]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NST + 4 + 2 * kPtsStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int64_t row0 = row_begin + (int64_t)(blockIdx.x >> 1) * 256 + 128 * (int64_t)rank;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + NST);
  const uint32_t accf0 = smem_u32(bars + 2 * NST), acce0 = smem_u32(bars + 2 * NST + 2);
  const uint32_t pfull0 = smem_u32(bars + 2 * NST + 4), pempty0 = pfull0 + 8 * kPtsStages;
  const uint32_t lfull0 = pempty0 + 8 * kPtsStages;
  const uint32_t full0_L = mapa_u32(full0, 0), acce0_L = mapa_u32(acce0, 0);   // the leader's barriers
  const int nseg = (nkb + seg_kb - 1) / seg_kb;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full0 + 8 * s, kGProdWarps + 1 + 1);   // leader's producer warps + the peer's relay + expect_tx
      mbar_init(lfull0 + 8 * s, kGProdWarps);           // peer: its producer warps (relayed to the leader)
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, 2 * kGDrainWarps);   // the drain warps of both CTAs
    }
    for (int s = 0; s < kPtsStages; ++s) {
      mbar_init(pfull0 + 8 * s, 1);
      mbar_init(pempty0 + 8 * s, kGProdWarps);   // the producer warps of this CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmP)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA: this CTA's half of the Omega^T tile (DN/2 x 64)
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % NST;
        const uint32_t ph = (kb / NST) & 1;
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        if (dbg & 4) {   // timing study only (wrong results): bit 2 skips the Omega tile loads
          if (rank == 0) mbar_arrive(full0 + 8 * s);
          continue;
        }
        if (rank == 0) mbar_arrive_tx(full0 + 8 * s, 2 * kBStage);
        tma_load_2d_2cta(smem_u32(b_t + s * kBStage), &tmB, (kb0 + kb) * kGaussBK, (int)rank * (DN / 2),
                         full0_L + 8 * s);
        if (NB == 2)   // the lo plane: rows DN .. 2 DN of the stacked Omega^T
          tma_load_2d_2cta(smem_u32(b_t + s * kBStage + kBHalfBytes), &tmB, (kb0 + kb) * kGaussBK,
                           DN + (int)rank * (DN / 2), full0_L + 8 * s);
      }
    }
  } else if (warp == 3) {
    // ---------------- peer relay: the peer's A tiles are written by generic stores and read by the leader's
    // MMA; a release at CLUSTER scope is needed for that (a CTA-scope arrive is not enough).  One thread
    // collects the 8 producer warps on a local barrier and issues one cluster-scope arrive per stage.
    if (rank == 1 && lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % NST;
        mbar_wait(lfull0 + 8 * s, (kb / NST) & 1);
#ifdef KS_GAUSS_RELAY_RELAXED   // timing study only: no cluster-scope release (unsafe with real tiles)
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(full0_L + 8 * s) : "memory");
#else
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(full0_L + 8 * s) : "memory");
#endif
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {  // ---------------- points loader: the stage's 64 packed points, kPtsStages ahead
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kPtsStages;
        const uint32_t ph = (kb / kPtsStages) & 1;
        mbar_wait(pempty0 + 8 * s, ph ^ 1);
        mbar_arrive_tx(pfull0 + 8 * s, kPtsBytes);
        tma_load_2d(smem_u32(pring + s * kGaussBK), &tmP, 0, (kb0 + kb) * (kGaussBK / 8), pfull0 + 8 * s);
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {  // ---------------- MMA issuer (leader only)
      const uint32_t idesc = (1u << 4) | ((uint32_t)(DN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      for (int g = 0; g < nseg; ++g) {
        mbar_wait(acce0, (g & 1) ^ 1);   // the drainers have folded segment g-1 into the running sum
        tc_fence_after();
        const uint32_t dtm = tmem;
        const int kb1 = min(nkb, (g + 1) * seg_kb);
        for (int kb = g * seg_kb; kb < kb1; ++kb) {
          const int s = kb % NST;
          const uint32_t ph = (kb / NST) & 1;
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint64_t dh = umma_desc_sw128(smem_u32(a_hi + s * kATileBytes));
          const uint64_t dl = umma_desc_sw128(smem_u32(a_lo + s * kATileBytes));
          const uint64_t db = umma_desc_sw128(smem_u32(b_t + s * kBStage));
          const uint64_t dbl = umma_desc_sw128(smem_u32(b_t + s * kBStage + kBHalfBytes));
#pragma unroll
          for (int kk = 0; kk < kGaussBK / 16; ++kk) {
            if (!(dbg & 1)) {   // timing studies only (KS_GAUSS_DEBUG): bit 0 skips the MMAs
              umma_f16_2cta(dtm, dh + 2 * kk, db + 2 * kk, idesc, (kb != g * seg_kb || kk != 0) ? 1u : 0u);
              umma_f16_2cta(dtm, dl + 2 * kk, db + 2 * kk, idesc, 1u);
              if (NB == 2) umma_f16_2cta(dtm, dh + 2 * kk, dbl + 2 * kk, idesc, 1u);
            }
          }
          umma_commit_2cta(empty0 + 8 * s);
        }
        umma_commit_2cta(accf0);
      }
    }
  } else if (warp >= 4 && warp < 4 + kGProdWarps) {
    // ---------------- K-tile producers: thread p -> rows kGRowsPT rq .. + kGRowsPT - 1, columns 8cq..8cq+7
    const int p = threadIdx.x - 128;
    const int rq = p >> 3, cq = p & 7;
    f2_t xi2[kGRowsPT / 2][3];
    int64_t irow[kGRowsPT];
#pragma unroll
    for (int pr = 0; pr < kGRowsPT / 2; ++pr) {
      float4 q[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int64_t i = row0 + kGRowsPT * rq + 2 * pr + h;
        irow[2 * pr + h] = i;
        if (i >= row_end) i = row_end - 1;
        q[h] = pk[i];
      }
      xi2[pr][0] = f2(q[0].x, q[1].x); xi2[pr][1] = f2(q[0].y, q[1].y); xi2[pr][2] = f2(q[0].z, q[1].z);
    }
    const float* Kb = Kst - row_begin * ldk;   // (stored K: row i at Kb + i * ldk)
    float kv[kGRowsPT][8];
    if constexpr (KIND == KS_KERNEL_STORED) load_tile_stored(Kb, ldk, ncols, irow, row_end - 1, (int64_t)kb0 * kGaussBK + 8 * cq, kv);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % NST;
      const uint32_t ph = (kb / NST) & 1;
      const int64_t j0 = (int64_t)(kb0 + kb) * kGaussBK + 8 * cq;
      const int ps = kb % kPtsStages;
      mbar_wait(pfull0 + 8 * ps, (kb / kPtsStages) & 1);
      float4 pts[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) pts[q] = lds128(smem_u32(pring + ps * kGaussBK + 8 * cq + (q ^ cq)));
#ifdef KS_GAUSS_EARLY_PEMPTY   // (study only: releases the slot while the LDS may still be in flight)
      __syncwarp();
      if (lane == 0) mbar_arrive(pempty0 + 8 * ps);
#endif
      mbar_wait(empty0 + 8 * s, ph ^ 1);
      const bool diag = (j0 + 8 > row0 + kGRowsPT * rq) && (j0 < row0 + kGRowsPT * rq + kGRowsPT);
      if constexpr (KIND == KS_KERNEL_STORED) {
        produce_tile_stored(kv, irow, pts, j0, diag, nugget, a_hi + s * kATileBytes, a_lo + s * kATileBytes, rq, cq);
        if (kb + 1 < nkb) load_tile_stored(Kb, ldk, ncols, irow, row_end - 1, j0 + kGaussBK, kv);
      } else if (!(dbg & 2))   // bit 1 skips the producers' arithmetic
        produce_tile<DIM, KIND>(xi2, irow, pts, j0, diag, nugget, a_hi + s * kATileBytes, a_lo + s * kATileBytes, rq, cq);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(rank == 0 ? full0 + 8 * s : lfull0 + 8 * s);
#ifndef KS_GAUSS_EARLY_PEMPTY
        // the points slot is released only once its values have been consumed (the tile above used them),
        // so no shared load of the slot can still be in flight when the loader's TMA refills it
        mbar_arrive(pempty0 + 8 * ps);
#endif
      }
    }
  } else if (warp >= 4 + kGProdWarps) {
    // ---------------- drainers: running sum (TMEM columns [DN, 2 DN)) += segment accumulator (columns
    // [0, DN)), added in fp32 round-to-nearest on the CUDA cores; the last segment is scaled and stored.
    // (with 8 drain warps, two per lane quarter, each folds half of the columns: the MMA waits for the drain)
    const int quarter = warp & 3, dpart = (warp - 4 - kGProdWarps) >> 2, nparts = kGDrainWarps / 4;
    const int row = 32 * quarter + lane;
    const int64_t i = row0 + row;
    const bool ok = i < row_end;
    float* yr = Y + (i - row_begin) * (int64_t)DN;
    const uint32_t tl = tmem + ((uint32_t)(32 * quarter) << 16);
    const int cb = 16 * ((DN / 16) * dpart / nparts), ce = 16 * ((DN / 16) * (dpart + 1) / nparts);   // 16-col units
    for (int g = 0; g < nseg; ++g) {
      mbar_wait(accf0, g & 1);
      tc_fence_after();
      const bool first = g == 0, last = g == nseg - 1;
      int c0 = cb;
      for (; c0 + 16 * kDrainU <= ce; c0 += 16 * kDrainU) drain_cols<kDrainU>(tl, DN, c0, first, last, ok, yr, out_scale);
      for (; c0 < ce; c0 += 16) drain_cols<1>(tl, DN, c0, first, last, ok, yr, out_scale);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {   // once per segment: cluster-scope release (this CTA's TMEM accesses -> the leader's MMA)
        if (rank == 0) mbar_arrive(acce0);
        else asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(acce0_L) : "memory");
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// Y0 += Y1 (the two split-K partial sums; d % 16 == 0 so rows x d is a multiple of 4).
__global__ void k_add_halves(float4* __restrict__ Y0, const float4* __restrict__ Y1, int64_t n4) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n4; p += (int64_t)gridDim.x * blockDim.x) {
    float4 a = Y0[p];
    const float4 b = Y1[p];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    Y0[p] = a;
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Stages per accumulation segment (bounds the tensor core's fp32 accumulation
// run to 8 * seg_kb MMAs).  KS_GAUSS_SEG overrides it for the precision study (tools/gauss_precision.py).
static int gauss_seg_kb() {
  static int v = [] {
    const char* e = getenv("KS_GAUSS_SEG");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? x : kGaussSegKb;
  }();
  return v;
}

template <int DIM, int KIND, int NB>
static ks_status launch_gauss(const ks_sketch_desc& D, const SketchLayout& L, int64_t rb, int64_t re, float* Y,
                              char* ws, cudaStream_t st, const StoredK* sk) {
  auto encode = get_encode();
  if (!encode) return fail(KS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int DN = D.d;
  cuuint64_t dims[2] = {(cuuint64_t)L.ncols_pad, (cuuint64_t)(NB * DN)};   // NB = 2: hi plane over lo plane
  cuuint64_t strides[1] = {(cuuint64_t)L.ncols_pad * 2};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap tm2;   // half-width boxes (DN/2 rows of Omega^T) for the CTA pair
  cuuint32_t box2[2] = {(cuuint32_t)kGaussBK, (cuuint32_t)(DN / 2)};
  CUresult r = encode(&tm2, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ws + L.off_gauss, dims, strides, box2, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  CUtensorMap tmP;   // packed points as rows of 8 float4 (128 B), 8-row boxes, SWIZZLE_128B
  cuuint64_t pdims[2] = {32, (cuuint64_t)(L.ncols_pad / 8)};
  cuuint64_t pstrides[1] = {128};
  cuuint32_t pbox[2] = {32, (cuuint32_t)(kGaussBK / 8)};
  r = encode(&tmP, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ws + L.off_pk, pdims, pstrides, pbox, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KS_ERR_CUDA, "cuTensorMapEncodeTiled (points) failed: " + std::to_string((int)r));
  const int nkb = (int)(L.ncols_pad / kGaussBK);
  const double S = gauss_scale(D);
  // Gaussian: Omega = fp16 / sqrt(d); Hartley / cosine: the planes hold Omega * sqrt(n)
  const float nug = (float)(S * D.nugget),
              osc = (float)(1.0 / (S * std::sqrt((double)(NB == 1 ? D.d : D.n))));
  const float4* pk = reinterpret_cast<const float4*>(ws + L.off_pk);
  constexpr int NST = NB == 1 ? kG2Stages : 3;
  const int smem = 1024 + NST * (2 * kATileBytes + NB * (DN / 2) * kGaussBK * 2) + kPtsStages * kPtsBytes + 512;
  // split the column blocks in two when the row tiles leave a partial last wave (one CTA pair per 2 SMs)
  const int pair_slots = num_sms() / 2;
  const int64_t pairs = (re - rb + 255) / 256;
  const int ksplit = (nkb >= 2 && pairs % pair_slots != 0 && pairs < 16 * pair_slots) ? 2 : 1;
  float* Y1 = reinterpret_cast<float*>(ws + L.off_ybuf);
  auto kern = k_sketch_gauss2<DIM, KIND, NB>;
  KS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const dim3 grid(2u * (unsigned)pairs, (unsigned)ksplit);
  static const int dbg = [] { const char* e = getenv("KS_GAUSS_DEBUG"); return e ? atoi(e) : 0; }();
  // NB = 2 issues 3 MMAs per K step: 11 stages per segment keep the non-RN accumulation run as for NB = 1
  const int seg = NB == 1 ? gauss_seg_kb() : std::max(1, gauss_seg_kb() * 2 / 3);
  kern<<<grid, kGThreads, smem, st>>>(tm2, tmP, pk, rb, re, nkb, seg, DN, nug, osc, Y, Y1, dbg, sk ? sk->K : nullptr,
                                      sk ? sk->ldk : 0, D.n);
  KS_LAUNCH_CHECK();
  if (ksplit == 2) {
    const int64_t tot = (re - rb) * (int64_t)DN;
    k_add_halves<<<(unsigned)std::min<int64_t>((tot / 4 + 255) / 256, (int64_t)num_sms() * 16), 256, 0, st>>>(
        reinterpret_cast<float4*>(Y), reinterpret_cast<const float4*>(Y1), tot / 4);
    KS_LAUNCH_CHECK();
  }
  return KS_OK;
}

template <int DIM, int KIND>
static ks_status launch_gauss_nb(const ks_sketch_desc& D, const SketchLayout& L, int64_t rb, int64_t re, float* Y,
                                 char* ws, cudaStream_t st, const StoredK* sk = nullptr) {
  return D.omega == KS_OMEGA_GAUSS ? launch_gauss<DIM, KIND, 1>(D, L, rb, re, Y, ws, st, sk)
                                   : launch_gauss<DIM, KIND, 2>(D, L, rb, re, Y, ws, st, sk);
}

ks_status gauss_sketch_run(const ks_sketch_desc& D, const SketchLayout& L, int64_t rb, int64_t re, float* Y,
                           char* ws, cudaStream_t st, const StoredK* sk) {
  if (sk) return launch_gauss_nb<1, KS_KERNEL_STORED>(D, L, rb, re, Y, ws, st, sk);
  const bool se = D.kernel == KS_KERNEL_SQEXP;
  switch (D.dim) {
    case 1: return se ? launch_gauss_nb<1, KS_KERNEL_SQEXP>(D, L, rb, re, Y, ws, st)
                      : launch_gauss_nb<1, KS_KERNEL_MATERN32>(D, L, rb, re, Y, ws, st);
    case 2: return se ? launch_gauss_nb<2, KS_KERNEL_SQEXP>(D, L, rb, re, Y, ws, st)
                      : launch_gauss_nb<2, KS_KERNEL_MATERN32>(D, L, rb, re, Y, ws, st);
    case 3: return se ? launch_gauss_nb<3, KS_KERNEL_SQEXP>(D, L, rb, re, Y, ws, st)
                      : launch_gauss_nb<3, KS_KERNEL_MATERN32>(D, L, rb, re, Y, ws, st);
  }
  return fail(KS_ERR_INVALID_ARGUMENT, "dim");
}

}  // namespace ks
