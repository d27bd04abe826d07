// Microbenchmark of the B200 ALU pipes the sketch kernels lean on (ops / clock / SM).
// Build + run on the GPU box:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_alu.cu && /tmp/ub
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

template <int OP>
__global__ void kern(float* out, float s0, float s1, long long* clk) {
  float a[kChains], b[kChains];
  unsigned u[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    a[c] = s0 + threadIdx.x * 1e-3f + c;
    b[c] = s1 + c * 1e-4f;
    u[c] = threadIdx.x * 7u + c;
  }
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (OP == 0) a[c] = a[c] + b[c];                                  // FADD reg-reg
      if (OP == 1) a[c] = a[c] * b[c];                                  // FMUL reg-reg
      if (OP == 2) a[c] = fmaf(a[c], b[c], b[(c + 1) % kChains]);      // FFMA 3 regs
      if (OP == 3) a[c] = fmaf(a[c], 1.00001f, 0.5f);                   // FFMA imm
      if (OP == 4) {                                                    // MUFU.EX2
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[c]));
        a[c] = y;
      }
      if (OP == 5) {                                                    // F2FP pack (cvt.rn.f16x2.f32)
        __half2 h = __floats2half2_rn(a[c], b[c]);
        u[c] ^= *reinterpret_cast<unsigned*>(&h);
        a[c] = __uint_as_float(u[c] | 0x3f800000u);
      }
      if (OP == 6) u[c] = (u[c] & 0xFFFFE000u) ^ (u[c] >> 3);          // LOP3 + SHF
      if (OP == 7) a[c] = a[c] - b[c] * b[c];                           // FFMA with shared operand
      if (OP == 8 && (c & 1) == 0) {                                    // FADD2 (packed f32x2)
        unsigned long long x, y;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[c]), "f"(a[c + 1]));
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b[c]), "f"(b[c + 1]));
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a[c]), "=f"(a[c + 1]) : "l"(x));
      }
      if (OP == 9 && (c & 1) == 0) {                                    // FFMA2 (packed f32x2)
        unsigned long long x, y, z;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[c]), "f"(a[c + 1]));
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b[c]), "f"(b[c + 1]));
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(z) : "f"(b[(c + 2) % kChains]), "f"(b[(c + 3) % kChains]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(y), "l"(z));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(a[c]), "=f"(a[c + 1]) : "l"(x));
      }
      if (OP == 10) a[c] = a[c] + b[(c + 1) % kChains] * 0.f + a[c] * 1e-7f; // mixed FFMA/FADD
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += a[c] + __uint_as_float(u[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int OP>
void run(const char* name, int opsPerIter) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* clk;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  cudaMalloc(&clk, sizeof(long long));
  const int threads = 1024, blocks = sms * 2;
  kern<OP><<<blocks, threads>>>(out, 1.0f, 0.999f, clk);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(out, 1.0f, 0.999f, clk);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c = 0;
  cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  const double ops = (double)blocks * threads * kIters * kChains * opsPerIter;
  // per-SM per-clock from the in-kernel clock of block 0 (2 blocks per SM resident together)
  const double per_sm_clk = (double)threads * 2 * kIters * kChains * opsPerIter / (double)c;
  printf("%-28s %8.3f ms  %10.1f Gop/s  %6.1f op/clk/SM (clock64)\n", name, ms, ops / ms / 1e6, per_sm_clk);
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run<0>("FADD r,r", 1);
  run<1>("FMUL r,r", 1);
  run<2>("FFMA r,r,r", 1);
  run<3>("FFMA r,imm,imm", 1);
  run<4>("MUFU.EX2", 1);
  run<5>("F2FP.PACK (+LOP)", 1);
  run<6>("LOP3+SHF (2 ops)", 2);
  run<7>("FFMA r,r,r (shared b)", 1);
  run<8>("FADD2 f32x2 (2 flop-lanes)", 1);
  run<9>("FFMA2 f32x2 (2 flop-lanes)", 1);
  return 0;
}
