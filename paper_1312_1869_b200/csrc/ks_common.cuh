// ks_common.cuh -- shared device helpers of the CUDA path (sm_100a only).
// Nothing here is shared with oracle/: the generator below is this library's
// own implementation of the DESIGN.md "RNG" definition.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/ks.h"

#define KS_DEVINL __device__ __forceinline__

namespace ks {

constexpr uint32_t kStreamSigns = 1;
constexpr uint32_t kStreamSelect = 2;
constexpr uint32_t kStreamGauss = 3;

// Philox4x32-10, key (lo32(seed), hi32(seed)), counter (lo32(idx), hi32(idx), stream, 0).
KS_DEVINL uint4 philox(uint64_t seed, uint32_t stream, uint64_t idx) {
  uint32_t c0 = (uint32_t)idx, c1 = (uint32_t)(idx >> 32), c2 = stream, c3 = 0u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;   // the bump after the last round is unused
  }
  return make_uint4(c0, c1, c2, c3);
}

// Rademacher sign s_j = 1 - 2*bit(j & 127) of philox(seed, 1, j >> 7).
KS_DEVINL float rademacher(uint64_t seed, int64_t j) {
  const uint4 w = philox(seed, kStreamSigns, (uint64_t)j >> 7);
  const int b = (int)(j & 127);
  const uint32_t word = (b < 64) ? ((b < 32) ? w.x : w.y) : ((b < 96) ? w.z : w.w);
  return ((word >> (b & 31)) & 1u) ? -1.0f : 1.0f;
}

KS_DEVINL double u53(uint32_t a, uint32_t b) {
  const double v = (double)((((uint64_t)(a >> 5)) << 26) + (uint64_t)(b >> 6));
  return (v + 0.5) * 0x1p-53;
}

// z ~ N(0,1) by fp64 Box-Muller from one Philox block.
KS_DEVINL double box_muller(uint4 w) {
  return sqrt(-2.0 * log(u53(w.x, w.y))) * cos(6.283185307179586 * u53(w.z, w.w));
}

KS_DEVINL int ilog2(int64_t x) { int l = 0; while ((int64_t(1) << l) < x) ++l; return l; }

KS_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------- covariance
KS_DEVINL float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
KS_DEVINL float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// K[i,j] * s_j from the packed (scaled) coordinates: SE 2^(-r'^2); Matern-3/2 (1 + z) e^-z, z = r'.
template <int DIM, int KIND>
KS_DEVINL float cov_signed(const float (&xi)[3], const float4 p) {
  const float dx = xi[0] - p.x;
  float r2 = dx * dx;
  if (DIM > 1) { const float dy = xi[1] - p.y; r2 = fmaf(dy, dy, r2); }
  if (DIM > 2) { const float dz = xi[2] - p.z; r2 = fmaf(dz, dz, r2); }
  if (KIND == KS_KERNEL_SQEXP) {
    return p.w * ex2_approx(-r2);
  } else {
    const float z = sqrt_approx(r2);
    const float e = ex2_approx(-1.4426950408889634f * z);
    return fmaf(p.w, z, p.w) * e;
  }
}

// ---------------------------------------------------------------- packed f32x2 (sm_100)
// A pair of fp32 values in one 64-bit register pair; FADD2/FMUL2/FFMA2 process both halves with one
// issue slot (round to nearest, like the scalar ops).  A scalar operand is broadcast with f2s(); ptxas
// folds it into the instruction's .F32 operand modifier (no MOV).
typedef unsigned long long f2_t;
KS_DEVINL f2_t f2(float lo, float hi) { f2_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
KS_DEVINL f2_t f2s(float a) { return f2(a, a); }
KS_DEVINL float f2lo(f2_t r) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a; }
KS_DEVINL float f2hi(f2_t r) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return b; }
KS_DEVINL f2_t f2add(f2_t a, f2_t b) { f2_t r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
KS_DEVINL f2_t f2sub(f2_t a, f2_t b) { f2_t r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
KS_DEVINL f2_t f2mul(f2_t a, f2_t b) { f2_t r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
KS_DEVINL f2_t f2fma(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// kappa(r_i0j) and kappa(r_i1j) without the amplitude (SE 2^(-r'^2); Matern-3/2 (1 + z) e^-z): the caller
// folds the amplitude p.w into its first butterfly level.
template <int DIM, int KIND>
KS_DEVINL f2_t cov_kappa2(const f2_t (&xi2)[3], const float4 p) {
  const f2_t dx = f2sub(xi2[0], f2s(p.x));
  f2_t r2 = f2mul(dx, dx);
  if (DIM > 1) { const f2_t dy = f2sub(xi2[1], f2s(p.y)); r2 = f2fma(dy, dy, r2); }
  if (DIM > 2) { const f2_t dz = f2sub(xi2[2], f2s(p.z)); r2 = f2fma(dz, dz, r2); }
  if (KIND == KS_KERNEL_SQEXP) {
    return f2(ex2_approx(-f2lo(r2)), ex2_approx(-f2hi(r2)));
  } else {
    const f2_t z = f2(sqrt_approx(f2lo(r2)), sqrt_approx(f2hi(r2)));
    const f2_t tz = f2mul(z, f2s(-1.4426950408889634f));
    const f2_t e = f2(ex2_approx(f2lo(tz)), ex2_approx(f2hi(tz)));
    return f2fma(z, e, e);
  }
}

// K[i0,j] s_j and K[i1,j] s_j for a row pair (packed coordinates xi2[c] = (x_i0c, x_i1c)) and one
// packed point p = (scaled coords, amplitude); same arithmetic as cov_signed, per half.
template <int DIM, int KIND>
KS_DEVINL f2_t cov_signed2(const f2_t (&xi2)[3], const float4 p) {
  const f2_t dx = f2sub(xi2[0], f2s(p.x));
  f2_t r2 = f2mul(dx, dx);
  if (DIM > 1) { const f2_t dy = f2sub(xi2[1], f2s(p.y)); r2 = f2fma(dy, dy, r2); }
  if (DIM > 2) { const f2_t dz = f2sub(xi2[2], f2s(p.z)); r2 = f2fma(dz, dz, r2); }
  if (KIND == KS_KERNEL_SQEXP) {
    const f2_t e = f2(ex2_approx(-f2lo(r2)), ex2_approx(-f2hi(r2)));
    return f2mul(e, f2s(p.w));
  } else {
    const f2_t z = f2(sqrt_approx(f2lo(r2)), sqrt_approx(f2hi(r2)));
    const f2_t tz = f2mul(z, f2s(-1.4426950408889634f));
    const f2_t e = f2(ex2_approx(f2lo(tz)), ex2_approx(f2hi(tz)));
    return f2mul(f2fma(z, f2s(p.w), f2s(p.w)), e);
  }
}

}  // namespace ks

// ----------------------------------------------------------------- host side
namespace ks {
inline int64_t next_pow2(int64_t n) { int64_t p = 1; while (p < n) p <<= 1; return p; }
inline int log2_exact(int64_t p) { int l = 0; while ((int64_t(1) << l) < p) ++l; return l; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace ks
