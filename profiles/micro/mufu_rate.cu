// B200 issue-rate microbenchmark: MUFU.EX2 (fp32) vs FFMA2 per SM per clock (clock64 bracketed).
#include <cstdio>
#include <cstdint>
__global__ void k_ex2(float* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ffma2(float* out, int iters, long long* cyc) {
  unsigned long long a[8];
  for (int i = 0; i < 8; ++i) { float x = 0.5f + threadIdx.x * 1e-3f + i; a[i] = (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(x) << 32); }
  unsigned long long m; { float x = 0.999f; m = (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(x) << 32); }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a[i]) : "l"(m));
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += __uint_as_float((unsigned)a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    k_ex2<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_ex2<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 8;
    printf("ex2   threads %4d: %.2f ops/clk/SM\n", threads, ops / h[0]);
    k_ffma2<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_ffma2<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("ffma2 threads %4d: %.2f instr/clk/SM (x2 flops lanes)\n", threads, ops / h[0]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
