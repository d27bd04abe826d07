// Probe of the tcgen05 kind::tf32 operand layouts used by k_panel_apply_tc (MN-major SW128 A and B,
// K-major SW128 A), against a CPU reference.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o /tmp/tcp tools/tc_probe.cu && /tmp/tcp
// Test 1: D (128 x 32) = A^T B with A = X (32 rows x 128 cols, MN-major: 4 slabs of 32 cols x 32 rows),
//         B = V (32 rows x 32, MN-major), K = 32 (4 MMAs of K = 8).
// Test 2: D (128 x 128) = V W with A = V (128 rows x 32, K-major), B = W (32 x 128, MN-major slabs).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cstring>
#include <cuda_fp16.h>
#include "../paper_1312_1869_b200/csrc/ks_tc.cuh"

using namespace ks;

KS_DEVINL void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc));
}
KS_DEVINL void commit1(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// mode: 0 = test 1, 1 = test 2.  lboA/sboA/lboB/sboB: descriptor byte offsets.
__global__ void probe(const float* X, const float* V, const float* Wm, float* D, int mode, int lboA, int sboA, int lboB,
                      int sboB) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bufA = sm;            // 16 KB
  uint8_t* bufB = sm + 16384;    // 16 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) { mbar_init(smem_u32(bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(256u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // stage operands (SW128: 16-B chunk q of a 128-B row r at chunk q ^ (r & 7))
  if (mode == 0) {
    for (int p = tid; p < 32 * 128; p += blockDim.x) {   // X[s][c]: slab c/32, row s
      const int s = p / 128, c = p % 128, sl = c / 32, cc = c % 32;
      const uint32_t off = sl * 4096 + s * 128 + ((((cc >> 2) ^ s) & 7) << 4) + (cc & 3) * 4;
      *reinterpret_cast<float*>(bufA + off) = X[p];
    }
    for (int p = tid; p < 32 * 32; p += blockDim.x) {    // V[s][a]
      const int s = p / 32, a = p % 32;
      const uint32_t off = s * 128 + ((((a >> 2) ^ s) & 7) << 4) + (a & 3) * 4;
      *reinterpret_cast<float*>(bufB + off) = V[p];
    }
  } else if (mode == 2) {   // control: f16, both K-major, rows of 32 halfs = 64 B (SW128 atoms hold 64 halfs)
    for (int p = tid; p < 128 * 64; p += blockDim.x) {   // A[m][k] (k < 64 halfs per 128-B row)
      const int m = p / 64, kk = p % 64;
      const uint32_t off = m * 128 + ((((kk >> 3) ^ m) & 7) << 4) + (kk & 7) * 2;
      *reinterpret_cast<__half*>(bufA + off) = __float2half(kk < 32 ? X[(kk) * 128 + m] : 0.f);
    }
    for (int p = tid; p < 32 * 64; p += blockDim.x) {    // B[n][k]
      const int n = p / 64, kk = p % 64;
      const uint32_t off = n * 128 + ((((kk >> 3) ^ n) & 7) << 4) + (kk & 7) * 2;
      *reinterpret_cast<__half*>(bufB + off) = __float2half(kk < 32 ? V[kk * 32 + n] : 0.f);
    }
  } else if (mode == 3) {
    for (int p = tid; p < 128 * 32; p += blockDim.x) {   // A = V[s][a] K-major
      const int s = p / 32, a = p % 32;
      const uint32_t off = s * 128 + ((((a >> 2) ^ s) & 7) << 4) + (a & 3) * 4;
      *reinterpret_cast<float*>(bufA + off) = V[p];
    }
    for (int p = tid; p < 32 * 128; p += blockDim.x) {   // B[n = c][k = a] = W[a][c], K-major rows of 32
      const int a = p / 128, c = p % 128;
      const uint32_t off = c * 128 + ((((a >> 2) ^ c) & 7) << 4) + (a & 3) * 4;
      *reinterpret_cast<float*>(bufB + off) = Wm[p];
    }
  } else {
    for (int p = tid; p < 128 * 32; p += blockDim.x) {   // V[s][a], 128 rows
      const int s = p / 32, a = p % 32;
      const uint32_t off = s * 128 + ((((a >> 2) ^ s) & 7) << 4) + (a & 3) * 4;
      *reinterpret_cast<float*>(bufA + off) = V[p];
    }
    for (int p = tid; p < 32 * 128; p += blockDim.x) {   // W[a][c]: slab c/32, row a
      const int a = p / 128, c = p % 128, sl = c / 32, cc = c % 32;
      const uint32_t off = sl * 4096 + a * 128 + ((((cc >> 2) ^ a) & 7) << 4) + (cc & 3) * 4;
      *reinterpret_cast<float*>(bufB + off) = Wm[p];
    }
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (tid == 0) {
    const uint32_t a0 = smem_u32(bufA), b0 = smem_u32(bufB);
    if (mode == 0) {
      const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
      for (int ks = 0; ks < 4; ++ks)
        mma_tf32(tmem, umma_desc(a0 + 1024 * ks, lboA, sboA), umma_desc(b0 + 1024 * ks, lboB, sboB), id, ks > 0);
    } else if (mode == 2) {
      const uint32_t id = (1u << 4) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(umma_desc(a0, 16, 1024)),
                   "l"(umma_desc(b0, 16, 1024)), "r"(id));
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(umma_desc(a0 + 32, 16, 1024)),
                   "l"(umma_desc(b0 + 32, 16, 1024)), "r"(id));
    } else if (mode == 3) {
      const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      for (int ks = 0; ks < 4; ++ks)
        mma_tf32(tmem, umma_desc(a0 + 32 * ks, 16, 1024), umma_desc(b0 + 32 * ks, 16, 1024), id, ks > 0);
    } else {
      const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      for (int ks = 0; ks < 4; ++ks)
        mma_tf32(tmem, umma_desc(a0 + 32 * ks, lboA, sboA), umma_desc(b0 + 1024 * ks, lboB, sboB), id, ks > 0);
    }
    commit1(smem_u32(bar));
  }
  mbar_wait(smem_u32(bar), 0);
  tc_fence_after();
  if (warp < 4) {
    const int ncol = (mode == 1 || mode == 3) ? 128 : 32;
    for (int c0 = 0; c0 < ncol; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      for (int q = 0; q < 16; ++q) D[(32 * warp + lane) * ncol + c0 + q] = v[q];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
  }
}

static float tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  srand(1);
  std::vector<float> X(32 * 128), V(128 * 32), W(32 * 128);
  for (auto& x : X) x = tf32((rand() % 2001 - 1000) / 500.f);
  for (auto& x : V) x = tf32((rand() % 2001 - 1000) / 500.f);
  for (auto& x : W) x = tf32((rand() % 2001 - 1000) / 500.f);
  float *dX, *dV, *dW, *dD;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dV, V.size() * 4); cudaMalloc(&dW, W.size() * 4); cudaMalloc(&dD, 128 * 128 * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  // reference
  std::vector<double> R1(128 * 32), R2(128 * 128);
  for (int c = 0; c < 128; ++c)
    for (int a = 0; a < 32; ++a) { double s = 0; for (int k = 0; k < 32; ++k) s += (double)X[k * 128 + c] * V[k * 32 + a]; R1[c * 32 + a] = s; }
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 128; ++c) { double s = 0; for (int k = 0; k < 32; ++k) s += (double)V[r * 32 + k] * W[k * 128 + c]; R2[r * 128 + c] = s; }
  std::vector<float> D(128 * 128);
  int cand[][4] = {{4096, 1024, 16, 1024}, {1024, 4096, 1024, 16}, {4096, 1024, 1024, 16}, {1024, 4096, 16, 1024},
                   {4096, 1024, 128, 1024}, {16, 1024, 16, 1024}};
  {
    cudaMemset(dD, 0, 128 * 128 * 4);
    probe<<<1, 128, 40000>>>(dX, dV, dW, dD, 2, 16, 1024, 16, 1024);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int i = 0; i < 128 * 32; ++i) { err = fmax(err, fabs(D[i] - R1[i])); nrm = fmax(nrm, fabs(R1[i])); }
    printf("control f16 K-major: max|err| %.3e (max|ref| %.3e) D[0..3] %g %g %g %g ref %g %g %s\n", err, nrm, D[0], D[1], D[2],
           D[3], R1[0], R1[1], e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  {
    cudaMemset(dD, 0, 128 * 128 * 4);
    probe<<<1, 128, 40000>>>(dX, dV, dW, dD, 3, 16, 1024, 16, 1024);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int i = 0; i < 128 * 128; ++i) { err = fmax(err, fabs(D[i] - R2[i])); nrm = fmax(nrm, fabs(R2[i])); }
    printf("tf32 both K-major: max|err| %.3e (max|ref| %.3e) D[0..3] %g %g %g %g ref %g %g %s\n", err, nrm, D[0], D[1], D[2],
           D[3], R2[0], R2[1], e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  for (int mode = 0; mode < 2; ++mode) {
    for (auto& c : cand) {
      int la = c[0], sa = c[1], lb = c[2], sb = c[3];
      if (mode == 1) { la = c[2]; sa = c[3]; lb = c[0]; sb = c[1]; }   // A K-major, B MN-major
      cudaMemset(dD, 0, 128 * 128 * 4);
      probe<<<1, 128, 40000>>>(dX, dV, dW, dD, mode, la, sa, lb, sb);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, 128 * 128 * 4, cudaMemcpyDeviceToHost);
      double err = 0, nrm = 0;
      const int n = mode == 0 ? 128 * 32 : 128 * 128;
      for (int i = 0; i < n; ++i) {
        const double r = mode == 0 ? R1[i] : R2[i];
        err = fmax(err, fabs(D[i] - r)); nrm = fmax(nrm, fabs(r));
      }
      printf("mode %d  lboA %5d sboA %5d lboB %5d sboB %5d  -> max|err| %.3e (max|ref| %.3e) D %g %g %g ref %g %g %g %s\n", mode,
             la, sa, lb, sb, err, nrm, D[0], D[1], D[2], mode == 0 ? R1[0] : R2[0], mode == 0 ? R1[1] : R2[1],
             mode == 0 ? R1[2] : R2[2], e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
