// FFMA2 (fma.rn.f32x2) operand-form microbenchmark: lane-FMA/clk/SM for the packed forms the TSQR apply and
// the SRHT gather use.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/uf tools/ubench_ffma2.cu && /tmp/uf
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
constexpr int C = 16, IT = 2048;
template <int V>
__global__ void __launch_bounds__(256) k(float* out, float s0) {
  u64 acc[C], x[C];
  float s[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { acc[c] = pk(c, threadIdx.x); x[c] = pk(s0 + c, s0 - c); s[c] = s0 * c; }
  const u64 x0 = x[0], sb0 = pk(s[1], s[1]);
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (V == 0) acc[c] = fma2(pk(s[c], s[c]), x[c], acc[c]);             // bcast scalar, pair, acc: all distinct
      if (V == 1) acc[c] = fma2(sb0, x[c], acc[c]);                        // shared bcast operand
      if (V == 2) acc[c] = fma2(pk(s[c], s[c]), x0, acc[c]);               // shared pair operand
      if (V == 3) acc[c] = fma2(x[(c + 1) % C], x[c], acc[c]);             // three distinct pairs
      if (V == 4) acc[c] = fma2(pk(s[c >> 1], s[c >> 1]), x[c], acc[c]);  // bcast shared by consecutive pairs
      if (V == 5) acc[c] = fma2(pk(s[c], s[c]), x[c >> 1], acc[c]);       // pair shared by consecutive pairs
    }
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(acc[c])); r += a + b; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int V>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  const int blocks = sms * 8;
  k<V><<<blocks, 256>>>(out, 1.0001f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<V><<<blocks, 256>>>(out, 1.0001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double lanes = 2.0 * C * IT * (double)blocks * 256;   // lane-FMAs
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-44s %8.3f ms  %8.1f G lane-FMA/s  %6.1f lane-FMA/clk/SM (at %d MHz)\n", name, ms, lanes / ms / 1e6,
         lanes / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  cudaFree(out);
}
int main() {
  run<0>("FFMA2 bcast(s_c), x_c, acc_c (distinct)");
  run<1>("FFMA2 bcast(s) shared, x_c, acc_c");
  run<2>("FFMA2 bcast(s_c), x shared, acc_c");
  run<3>("FFMA2 x_{c+1}, x_c, acc_c (3 pairs)");
  run<4>("FFMA2 bcast(s_{c/2}) shared by 2, x_c, acc_c");
  run<5>("FFMA2 bcast(s_c), x_{c/2} shared by 2, acc_c");
  return 0;
}
