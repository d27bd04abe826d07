// Probe 4: a TMA load with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B lands a row-major fp32 tile in the
// SWIZZLE_128B_BASE32B MN-major operand layout of tcgen05 kind::tf32 (G3), so the landed X chunk can be the
// A operand (A = X^T, M = columns, K = rows) without a conversion pass.
//   (1) the byte position of every element after the TMA load vs the BASE32B formula (granule ^ (k & 3),
//       4-line groups at SBO = 512, 32-column chunks at LBO = 4096);
//   (2) D (128 x 32) = X^T V with A from the TMA-landed tile (MN-major, BASE32B) and B = V^T K-major SW128,
//       K = 32 (4 MMAs of K = 8, start address + 1024 B per step), vs a CPU reference on tf32-truncated X.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o /tmp/tcp4 tools/tc_probe4.cu -lcuda && /tmp/tcp4
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <vector>
#include "../paper_1312_1869_b200/csrc/ks_tc.cuh"
using namespace ks;

__device__ __forceinline__ void tload(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(bar) : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap tm, const float* Vg, float* dump, float* D, uint32_t lbo,
                      uint32_t sbo, uint32_t kstep) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t *bufA = sm, *bufB = sm + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 4096);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(smem_u32(bar), 1);
    mbar_init(smem_u32(bar + 1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(32u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B = V^T, K-major SW128: row n (reflector), K = 32 rows of V (128 B per row)
  for (int p = tid; p < 32 * 32; p += blockDim.x) {
    const int n = p / 32, kk = p % 32;
    const uint32_t o = n * 128 + ((((kk >> 2) ^ n) & 7) << 4) + (kk & 3) * 4;
    *reinterpret_cast<float*>(bufB + o) = Vg[kk * 32 + n];
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_arrive_tx(smem_u32(bar), 16384u);
    for (int cg = 0; cg < 4; ++cg) tload(smem_u32(bufA) + 4096u * cg, &tm, 32 * cg, 0, smem_u32(bar));
  }
  mbar_wait(smem_u32(bar), 0);
  for (int p = tid; p < 4096; p += blockDim.x) dump[p] = reinterpret_cast<float*>(bufA)[p];
  const uint32_t tmem = *slot;
  if (tid == 0) {
    tc_fence_after();
    // D f32, A / B tf32, A MN-major (bit 15), B K-major, N = 32, M = 128
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    for (int k8 = 0; k8 < 4; ++k8) {
      uint64_t da = umma_desc(smem_u32(bufA) + kstep * k8, lbo, sbo);
      da = (da & ~(7ull << 61)) | (1ull << 61);   // SWIZZLE_128B_BASE32B
      const uint64_t db = umma_desc_sw128(smem_u32(bufB) + 32 * k8);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(id), "r"(k8));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar + 1)) : "memory");
  }
  mbar_wait(smem_u32(bar + 1), 0);
  tc_fence_after();
  if (warp < 4)
    for (int c0 = 0; c0 < 32; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      for (int q = 0; q < 16; ++q) D[(32 * warp + lane) * 32 + c0 + q] = v[q];
    }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32u));
  }
}

static float tf32t(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }
// BASE32B MN-major position (bytes) of element (mn, k)
static uint32_t off_mn32(int mn, int k, uint32_t lbo, uint32_t sbo) {
  const int e = mn % 32, line = k % 4;
  const uint32_t b = e * 4;
  return (mn / 32) * lbo + (k / 4) * sbo + line * 128 + ((((b >> 5) ^ line) & 3) << 5) + (b & 31);
}

int main() {
  const int R = 32, C = 128;
  std::vector<float> X(R * C), V(32 * 32), dump(4096), D(128 * 32);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) X[r * C + c] = (float)(r * C + c);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  float *dX, *dV, *dd, *dD;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dV, V.size() * 4); cudaMalloc(&dd, 4096 * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, str[1] = {(cuuint64_t)C * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode ATOM_32B: %d\n", (int)cr);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 24000);
  // (1) layout
  probe<<<1, 128, 24000>>>(tm, dV, dd, dD, 4096, 512, 1024);
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  cudaMemcpy(dump.data(), dd, 4096 * 4, cudaMemcpyDeviceToHost);
  int ok = 0, bad = 0;
  for (int p = 0; p < 4096; ++p) {
    const int v = (int)dump[p], r = v / C, c = v % C;
    if (off_mn32(c, r, 4096, 512) == (uint32_t)p * 4) ++ok;
    else if (bad++ < 8) printf("  pos %d holds (r %d, c %d), formula %u\n", p * 4, r, c, off_mn32(c, r, 4096, 512));
  }
  printf("layout: %d / 4096 elements where the BASE32B formula puts them\n", ok);
  // (2) MMA from the TMA-landed tile
  srand(3);
  for (auto& x : X) x = (rand() % 20001 - 10000) / 1024.f;
  for (auto& x : V) x = tf32t((rand() % 2001 - 1000) / 512.f);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice);
  for (uint32_t ks : {1024u, 512u}) {
    for (uint32_t sbo : {512u, 1024u}) {
      cudaMemset(dD, 0, D.size() * 4);
      probe<<<1, 128, 24000>>>(tm, dV, dd, dD, 4096, sbo, ks);
      e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, nrm = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32; ++n) {
          double r = 0;
          for (int k = 0; k < 32; ++k) r += (double)tf32t(X[k * C + m]) * V[k * 32 + n];
          err = fmax(err, fabs(D[m * 32 + n] - r));
          nrm = fmax(nrm, fabs(r));
        }
      printf("MMA A=TMA tile (MN-major BASE32B, lbo 4096, sbo %u, k-step %u B): max|err| %.3e (max|ref| %.3e) %s\n", sbo, ks,
             err, nrm, cudaGetErrorString(e));
    }
  }
  return 0;
}
