// Probe 3: how kind::tf32 reads fp32 operand bits (truncate vs round).  D = A * B with B = e_0 (exact 1.0):
// D[m][0] = A[m][0] as the tensor core sees it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o /tmp/tcp3 tools/tc_probe3.cu && /tmp/tcp3
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1312_1869_b200/csrc/ks_tc.cuh"
using namespace ks;
__global__ void probe(const float* Ag, float* D) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t *bufA = sm, *bufB = sm + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) { mbar_init(smem_u32(bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(32u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // K-major SW128, K = 8 fp32 (32 B) per row: A 128 rows, B 32 rows (N = 32)
  for (int p = tid; p < 128 * 8; p += blockDim.x) {
    const int m = p / 8, k = p % 8;
    const uint32_t o = (m / 8) * 1024 + (m % 8) * 128 + ((((k >> 2) ^ m) & 7) << 4) + (k & 3) * 4;
    *reinterpret_cast<float*>(bufA + o) = Ag[p];
  }
  for (int p = tid; p < 32 * 8; p += blockDim.x) {
    const int n = p / 8, k = p % 8;
    const uint32_t o = (n / 8) * 1024 + (n % 8) * 128 + ((((k >> 2) ^ n) & 7) << 4) + (k & 3) * 4;
    *reinterpret_cast<float*>(bufB + o) = (n == 0 && k == 0) ? 1.f : 0.f;
  }
  fence_proxy_async(); tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem), "l"(umma_desc(smem_u32(bufA), 16, 1024)), "l"(umma_desc(smem_u32(bufB), 16, 1024)), "r"(id));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
  }
  mbar_wait(smem_u32(bar), 0);
  tc_fence_after();
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16), v);
  D[32 * warp + lane] = v[0];
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32u)); }
}
int main() {
  std::vector<float> A(128 * 8, 0.f);
  // row m: A[m][0] = 1 + f * 2^-10 with f in {0.25, 0.5 (tie), 0.75, ...} and negatives
  const float fr[8] = {0.25f, 0.5f, 0.75f, 0.49f, 0.51f, 1.5f, 0.125f, 0.875f};
  for (int m = 0; m < 128; ++m) {
    const float f = fr[m % 8];
    const float sgn = (m / 8) % 2 ? -1.f : 1.f;
    A[m * 8] = sgn * (1.f + f * 0x1p-10f);
  }
  float *dA, *dD; cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dD, 128 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  probe<<<1, 128, 40000>>>(dA, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> D(128); cudaMemcpy(D.data(), dD, 128 * 4, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  for (int m = 0; m < 16; ++m) {
    const float a = A[m * 8];
    uint32_t u; memcpy(&u, &a, 4);
    uint32_t tr = u & 0xFFFFE000u; float t; memcpy(&t, &tr, 4);
    printf("a = %.10f  (1 + %.4f ulp_tf32)  tc sees %.10f  trunc %.10f  -> %s\n", a, fr[m % 8], D[m], t,
           D[m] == t ? "truncate" : "other");
  }
  return 0;
}
