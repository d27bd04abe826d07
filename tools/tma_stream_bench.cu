// TMA streaming ceiling for the TSQR leaf-apply access pattern (study tool, not product):
// a rows x cols fp32 matrix (row stride cols) is read and written back in place by (512-row leaf, BC-column
// tile) items, 32-row x 32-column SWIZZLE_128B boxes, a DEPTH-deep ring of 32-row chunks per CTA, one CTA
// per SM, persistent over a balanced share of the items.  Reports GB/s (read + write bytes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_stream_bench.cu -o /tmp/tmab -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void bar_tx(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void tload(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint32_t b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(b) : "memory");
}
__device__ __forceinline__ void tstore(const CUtensorMap* tm, int c0, int c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"((uint64_t)tm), "r"(c0), "r"(c1), "r"(src) : "memory");
}

template <int BC, int DEPTH>
__global__ void __launch_bounds__(128, 1) k_stream(const __grid_constant__ CUtensorMap tm, int rows, int cols, int store) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~uintptr_t(1023));
  uint64_t* bars = (uint64_t*)(sm + DEPTH * 32 * BC * 4);
  constexpr int NB = BC / 32;
  const int leaves = rows / 512, ntl = cols / BC;
  const long total = (long)leaves * ntl;
  const long i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < DEPTH; ++i) bar_init(su32(bars + i), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t ph = 0;
  const long nch = (i1 - i0) * 16;   // 16 chunks of 32 rows per item
  auto issue = [&](long q) {
    const long it = i0 + q / 16;
    const int c = (int)(q % 16);
    const int leaf = (int)(it / ntl), t = (int)(it % ntl);
    const int s = (int)(q % DEPTH);
    const uint32_t dst = su32(sm) + (uint32_t)s * 32 * BC * 4;
    bar_tx(su32(bars + s), 32 * BC * 4);
    for (int b = 0; b < NB; ++b) tload(dst + 4096u * b, &tm, t * BC + 32 * b, leaf * 512 + 32 * c, su32(bars + s));
  };
  for (long q = 0; q < DEPTH - 1 && q < nch; ++q) issue(q);
  for (long q = 0; q < nch; ++q) {
    if (q + DEPTH - 1 < nch) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // slot (q-1) % DEPTH stored
      issue(q + DEPTH - 1);
    }
    const int s = (int)(q % DEPTH);
    bar_wait(su32(bars + s), (uint32_t)((q / DEPTH) & 1));
    if (store) {
      const long it = i0 + q / 16;
      const int c = (int)(q % 16);
      const int leaf = (int)(it / ntl), t = (int)(it % ntl);
      const uint32_t src = su32(sm) + (uint32_t)s * 32 * BC * 4;
      for (int b = 0; b < NB; ++b) tstore(&tm, t * BC + 32 * b, leaf * 512 + 32 * c, src + 4096u * b);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const int rows = 262144, cols = argc > 1 ? atoi(argv[1]) : 512;
  float* X;
  cudaMalloc(&X, (size_t)rows * cols * 4);
  cudaMemset(X, 0, (size_t)rows * cols * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, int depth, int bc, int store, const char* name) {
    const int smem = depth * 32 * bc * 4 + 1024 + 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a);
      kern<<<sms, 128, smem>>>(tm, rows, cols, store);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)rows * cols * 4 * (store ? 2 : 1);
      if (r == 2) printf("%-28s %8.3f ms  %7.0f GB/s  (%s)\n", name, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(k_stream<128, 4>, 4, 128, 1, "BC128 depth4 r+w");
  run(k_stream<128, 8>, 8, 128, 1, "BC128 depth8 r+w");
  run(k_stream<128, 12>, 12, 128, 1, "BC128 depth12 r+w");
  run(k_stream<128, 4>, 4, 128, 0, "BC128 depth4 read");
  run(k_stream<128, 8>, 8, 128, 0, "BC128 depth8 read");
  run(k_stream<32, 16>, 16, 32, 1, "BC32 depth16 r+w");
  run(k_stream<256, 4>, 4, 256, 1, "BC256 depth4 r+w");
  run(k_stream<256, 6>, 6, 256, 1, "BC256 depth6 r+w");
  float* Y;
  cudaMalloc(&Y, (size_t)rows * cols * 4);
  cudaEventRecord(a);
  cudaMemcpy(Y, X, (size_t)rows * cols * 4, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %8.3f ms  %7.0f GB/s\n", "cudaMemcpy D2D", ms, 2.0 * rows * cols * 4 / ms / 1e6);
  return 0;
}
