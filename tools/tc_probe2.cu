// Probe 2: MN-major SW128 operands of tcgen05.mma, f16 (control) and tf32, one MMA of M=128, N=64,
// against a CPU reference.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o /tmp/tcp2 tools/tc_probe2.cu && /tmp/tcp2
// SW128 atoms: a 128-B line holds 128 B of the contiguous (MN or K) dimension; 8 lines per 1024-B atom;
// 16-B chunk j of line r sits at chunk j ^ (r & 7).
//   MN-major: line = one K index, 8 K per atom (SBO = stride of the next 8 K), next MN chunk at LBO.
//   K-major : line = one MN index (128 B of K), 8 MN per atom (SBO = next 8 MN rows), LBO unused (16).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>
#include <cuda_fp16.h>
#include "../paper_1312_1869_b200/csrc/ks_tc.cuh"
using namespace ks;

// byte offset of element (mn, k) of an operand with esz-byte elements
__host__ __device__ inline uint32_t off_mn(int mn, int k, int esz, uint32_t lbo, uint32_t sbo) {
  const int per = 128 / esz;   // elements of MN per line
  const int e = mn % per, line = k % 8;
  const uint32_t b = (e * esz);
  return (mn / per) * lbo + (k / 8) * sbo + line * 128 + ((((b >> 4) ^ line) & 7) << 4) + (b & 15);
}
// SWIZZLE_128B_BASE32B MN-major (tf32): 128-B lines of 32 MN elements, one per K; 32-B granule g of line r
// at g ^ (r & 3); groups of 4 K lines at SBO, MN chunks of 32 at LBO.
__host__ __device__ inline uint32_t off_mn32(int mn, int k, uint32_t lbo, uint32_t sbo) {
  const int e = mn % 32, line = k % 4;
  const uint32_t b = e * 4;
  return (mn / 32) * lbo + (k / 4) * sbo + line * 128 + ((((b >> 5) ^ line) & 3) << 5) + (b & 31);
}
__host__ __device__ inline uint32_t off_k(int mn, int k, int esz, uint32_t sbo) {
  const int line = mn % 8;
  const uint32_t b = k * esz;   // K < 128 B
  return (mn / 8) * sbo + line * 128 + ((((b >> 4) ^ line) & 7) << 4) + (b & 15);
}

__global__ void probe(const float* Ag, const float* Bg, float* D, int mode, uint32_t lboA, uint32_t sboA,
                      uint32_t lboB, uint32_t sboB, int amn, int bmn) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bufA = sm;            // 32 KB
  uint8_t* bufB = sm + 32768;    // 16 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 49152);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool f16 = mode == 0;
  const int K = f16 ? 16 : 8, esz = f16 ? 2 : 4;
  for (int p = tid; p < 32768 / 4; p += blockDim.x) reinterpret_cast<uint32_t*>(bufA)[p] = 0x7fc00000u;   // NaN fill
  for (int p = tid; p < 16384 / 4; p += blockDim.x) reinterpret_cast<uint32_t*>(bufB)[p] = 0x7fc00000u;
  if (tid == 0) { mbar_init(smem_u32(bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(64u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  for (int p = tid; p < 128 * K; p += blockDim.x) {   // A[m][k]
    const int m = p / K, k = p % K;
    const uint32_t o = amn == 2 ? off_mn32(m, k, lboA, sboA) : amn ? off_mn(m, k, esz, lboA, sboA) : off_k(m, k, esz, sboA);
    if (f16) *reinterpret_cast<__half*>(bufA + o) = __float2half(Ag[p]);
    else *reinterpret_cast<float*>(bufA + o) = Ag[p];
  }
  for (int p = tid; p < 64 * K; p += blockDim.x) {    // B[n][k]
    const int n = p / K, k = p % K;
    const uint32_t o = bmn == 2 ? off_mn32(n, k, lboB, sboB) : bmn ? off_mn(n, k, esz, lboB, sboB) : off_k(n, k, esz, sboB);
    if (f16) *reinterpret_cast<__half*>(bufB + o) = __float2half(Bg[p]);
    else *reinterpret_cast<float*>(bufB + o) = Bg[p];
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t fmt = f16 ? 0u : 2u;
    const uint32_t id = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(amn != 0) << 15) | ((uint32_t)(bmn != 0) << 16) |
                        ((64u >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t da = umma_desc(smem_u32(bufA), lboA, sboA), db = umma_desc(smem_u32(bufB), lboB, sboB);
    if (amn == 2) da = (da & ~(7ull << 61)) | (1ull << 61);   // SWIZZLE_128B_BASE32B
    if (bmn == 2) db = (db & ~(7ull << 61)) | (1ull << 61);
    if (f16)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(id));
    else
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(id));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
  }
  mbar_wait(smem_u32(bar), 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 64; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
    for (int q = 0; q < 16; ++q) D[(32 * warp + lane) * 64 + c0 + q] = v[q];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64u));
  }
}

static float tf32r(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  srand(7);
  std::vector<float> A(128 * 16), B(64 * 16), D(128 * 64);
  for (auto& x : A) x = tf32r((rand() % 2001 - 1000) / 512.f);
  for (auto& x : B) x = tf32r((rand() % 2001 - 1000) / 512.f);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 52000);
  struct Case { int mode, amn, bmn; uint32_t la, sa, lb, sb; const char* what; };
  // f16: MN-major line = 64 halfs; A (M=128) = 2 MN chunks.  tf32: line = 32 floats; A = 4 chunks, B (N=64) = 2.
  std::vector<Case> cs = {
      {0, 0, 0, 16, 1024, 16, 1024, "f16 K-major A,B (control)"},
      {0, 1, 0, 8192, 1024, 16, 1024, "f16 MN-major A lbo=8192 sbo=1024"},
      {0, 1, 0, 1024, 8192, 16, 1024, "f16 MN-major A lbo=1024 sbo=8192"},
      {0, 0, 1, 16, 1024, 8192, 1024, "f16 MN-major B lbo=8192 sbo=1024"},
      {0, 0, 1, 16, 1024, 1024, 8192, "f16 MN-major B lbo=1024 sbo=8192"},
      {0, 1, 1, 8192, 1024, 8192, 1024, "f16 MN-major A,B lbo=8192 sbo=1024"},
      {1, 0, 0, 16, 1024, 16, 1024, "tf32 K-major A,B (control)"},
      {1, 1, 0, 4096, 1024, 16, 1024, "tf32 MN-major A lbo=4096 sbo=1024"},
      {1, 1, 0, 1024, 4096, 16, 1024, "tf32 MN-major A lbo=1024 sbo=4096"},
      {1, 0, 1, 16, 1024, 4096, 1024, "tf32 MN-major B lbo=4096 sbo=1024"},
      {1, 0, 1, 16, 1024, 1024, 4096, "tf32 MN-major B lbo=1024 sbo=4096"},
      {1, 1, 1, 4096, 1024, 4096, 1024, "tf32 MN-major A,B lbo=4096 sbo=1024"},
      {1, 2, 0, 1024, 512, 16, 1024, "tf32 MN32B A lbo=1024 sbo=512"},
      {1, 2, 0, 512, 1024, 16, 1024, "tf32 MN32B A lbo=512 sbo=1024"},
      {1, 2, 0, 4096, 512, 16, 1024, "tf32 MN32B A lbo=4096 sbo=512"},
      {1, 2, 0, 512, 4096, 16, 1024, "tf32 MN32B A lbo=512 sbo=4096"},
      {1, 0, 2, 16, 1024, 1024, 512, "tf32 MN32B B lbo=1024 sbo=512"},
      {1, 0, 2, 16, 1024, 512, 1024, "tf32 MN32B B lbo=512 sbo=1024"},
      {1, 2, 2, 1024, 512, 1024, 512, "tf32 MN32B A,B lbo=1024 sbo=512"},
      {1, 2, 2, 2048, 1024, 2048, 1024, "tf32 MN32B A,B lbo=2048 sbo=1024"},
  };
  for (auto& c : cs) {
    const int K = c.mode == 0 ? 16 : 8;
    std::vector<float> a(128 * K), b(64 * K);
    for (int m = 0; m < 128; ++m) for (int k = 0; k < K; ++k) a[m * K + k] = A[m * 16 + k];
    for (int n = 0; n < 64; ++n) for (int k = 0; k < K; ++k) b[n * K + k] = B[n * 16 + k];
    cudaMemcpy(dA, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, 52000>>>(dA, dB, dD, c.mode, c.la, c.sa, c.lb, c.sb, c.amn, c.bmn);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    int nan = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)a[m * K + k] * b[n * K + k];
        const double g = D[m * 64 + n];
        if (g != g) { ++nan; continue; }
        err = fmax(err, fabs(g - r)); nrm = fmax(nrm, fabs(r));
      }
    printf("%-42s max|err| %.3e (max|ref| %.3e) nan %d  D0 %g %s\n", c.what, err, nrm, nan, D[0],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
