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

}  // namespace ks

// ----------------------------------------------------------------- host side
namespace ks {
inline int64_t next_pow2(int64_t n) { int64_t p = 1; while (p < n) p <<= 1; return p; }
inline int log2_exact(int64_t p) { int l = 0; while ((int64_t(1) << l) < p) ++l; return l; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace ks
