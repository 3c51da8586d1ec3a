// Probe: MUFU.EX2 and FFMA2 throughput per SM on this B200 (warps per SMSP = blockDim/128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_probe.cu -o tools/mufu_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, long long* clk) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0fBA800000;" : "+f"(a[i]));
      // packed forms: one instruction, two results (reported per instruction)
      if (OP == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(*reinterpret_cast<uint32_t*>(&a[i])));
      if (OP == 3) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(*reinterpret_cast<uint32_t*>(&a[i])));
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}

// dependent-chain latency of one warp: 0 = FMNMX (2-input), 1 = FMNMX3, 2 = FFMA2, 3 = MUFU.EX2
template <int OP>
__global__ void lat(float* out, int iters, long long* clk) {
  float x = threadIdx.x * 1e-3f, a = -1.f, b = -2.f;
  uint64_t x2 = 0x3f8000003f800000ull;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) asm volatile("max.f32 %0, %0, %1;" : "+f"(x) : "f"(a));
      if (OP == 1) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(a), "f"(b));
      if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x2));
      if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) clk[0] = t1 - t0;
  if (x == 12345.f || x2 == 7) out[0] = x;
}

template <int OP>
void run_lat(const char* name) {
  float* o; long long* clk; cudaMalloc(&o, 4); cudaMalloc(&clk, 8);
  lat<OP><<<1, 32>>>(o, 16, clk);
  cudaDeviceSynchronize();
  lat<OP><<<1, 32>>>(o, 1024, clk);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  printf("{\"op\": \"%s\", \"dependent_latency_clk\": %.2f}\n", name, double(c) / (1024.0 * 16));
  fflush(stdout);
  cudaFree(o); cudaFree(clk);
}

template <int OP>
void run(const char* name, int threads) {
  float* o; long long* clk; cudaMalloc(&o, 4); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  k<OP><<<148, threads>>>(o, 16, clk);
  cudaDeviceSynchronize();
  k<OP><<<148, threads>>>(o, iters, clk);
  cudaDeviceSynchronize();
  long long c[148]; cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  double ops = double(threads) * iters * 8;
  printf("{\"op\": \"%s\", \"threads_per_sm\": %d, \"ops_per_clk_per_sm\": %.2f}\n", name, threads, ops / double(c[0]));
  fflush(stdout);
  cudaFree(o); cudaFree(clk);
}

int main() {
  for (int t : {128, 256, 512}) run<0>("MUFU.EX2", t);
  for (int t : {128, 256, 512}) run<1>("FFMA", t);
  for (int t : {128, 256, 512}) run<2>("MUFU.EX2 bf16x2 (instructions)", t);
  for (int t : {128, 256, 512}) run<3>("MUFU.EX2 f16x2 (instructions)", t);
  run_lat<0>("FMNMX (max.f32, 2 inputs)");
  run_lat<1>("FMNMX3 (max.f32, 3 inputs)");
  run_lat<2>("FFMA2 (fma.rn.f32x2)");
  run_lat<3>("MUFU.EX2");
  return 0;
}
