// Pipe-throughput microbenchmarks for the roofline of the summation kernel
// ("measure MUFU.EX2, FFMA and FFMA2 throughput and the in-kernel
// clock on the box").  Each thread runs 8 independent dependency chains of the
// instruction under test; the grid fills every SM.  Prints per-SM per-clock
// rates (from clock64 in the kernel) and per-second rates (CUDA events).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void ex2_kernel(float* out, long long* cyc, float seed) {
  float v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = seed * (q + 1) * 1e-3f - 0.5f * threadIdx.x * 1e-6f;
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[q]));
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += v[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void ffma2_kernel(float* out, long long* cyc, float seed) {
  unsigned long long v[8];
  const float2 m = make_float2(0.999f, 0.999f), a = make_float2(1e-3f, 1e-3f);
  unsigned long long M, A;
  asm("mov.b64 %0, {%1,%2};" : "=l"(M) : "f"(m.x), "f"(m.y));
  asm("mov.b64 %0, {%1,%2};" : "=l"(A) : "f"(a.x), "f"(a.y));
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float x = seed + q, y = seed - q;
    asm("mov.b64 %0, {%1,%2};" : "=l"(v[q]) : "f"(x), "f"(y));
  }
  long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[q]) : "l"(M), "l"(A));
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float x, y;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(v[q]));
    s += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <class K>
void run(const char* name, K kernel, double ops_per_thread_iter, int sms) {
  const int threads = 512, blocks = sms * 4;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * threads * blocks);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  kernel<<<blocks, threads>>>(out, cyc, 1.0f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kernel<<<blocks, threads>>>(out, cyc, 1.0f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (int i = 0; i < blocks; ++i) cmax = h[i] > cmax ? h[i] : cmax;
  const double ops = ops_per_thread_iter * kIters * (double)threads * blocks;
  // 4 resident blocks of 512 threads per SM run concurrently: per-SM clock rate
  const double per_sm_clk = ops / sms / cmax;
  printf("{\"op\": \"%s\", \"per_sm_per_clk\": %.2f, \"per_s\": %.4e, \"ms\": %.3f, \"cycles\": %.0f, "
         "\"clock_ghz\": %.3f}\n",
         name, per_sm_clk, ops / (ms * 1e-3), ms, cmax, cmax / (ms * 1e-3) / 1e9);
  delete[] h;
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  run("mufu_ex2 (lane-ops)", ex2_kernel, 8.0, p.multiProcessorCount);
  run("ffma2 (fp32 FMA lane-ops, 2 per FFMA2)", ffma2_kernel, 16.0, p.multiProcessorCount);
  return 0;
}
