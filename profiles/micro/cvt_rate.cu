// B200 issue-rate microbenchmark for the softmax's pack step: cvt.rn.bf16x2.f32 (F2FP) alone, with
// MUFU.EX2 interleaved (does F2FP share the SFU's 16/clk/SM?), and PRMT (byte permute: the pack by
// truncation) per SM per clock (clock64 bracketed, 148 CTAs).
#include <cstdio>
#include <cstdint>
__global__ void k_cvt(unsigned* out, int iters, long long* cyc) {
  float a[8];
  unsigned u[8];
  for (int i = 0; i < 8; ++i) { a[i] = 0.001f * (threadIdx.x + i); u[i] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i])));
    }
  long long t1 = clock64();
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
// per iteration: 8 ex2 + 4 cvt (one cvt per pair of exps, as in the softmax)
__global__ void k_ex2_cvt(unsigned* out, int iters, long long* cyc) {
  float a[8];
  unsigned u[4];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) u[i] = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[2 * i]), "f"(a[2 * i + 1] + __uint_as_float(u[i])));
  }
  long long t1 = clock64();
  unsigned s = 0; for (int i = 0; i < 4; ++i) s += u[i];
  for (int i = 0; i < 8; ++i) s += __float_as_uint(a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ex2_only(unsigned* out, int iters, long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  long long t1 = clock64();
  unsigned s = 0;
  for (int i = 0; i < 8; ++i) s += __float_as_uint(a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_prmt(unsigned* out, int iters, long long* cyc) {
  unsigned u[8];
  for (int i = 0; i < 8; ++i) u[i] = threadIdx.x * 77u + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(u[i]) : "r"(u[(i + 1) & 7]));
  long long t1 = clock64();
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2_h2(unsigned* out, int iters, long long* cyc) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0xB800B800u + threadIdx.x + i;  // about -0.5 in f16
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  long long t1 = clock64();
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void k_ex2_bf2(unsigned* out, int iters, long long* cyc) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0xBF00BF00u + threadIdx.x + i;  // about -0.5 in bf16
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  long long t1 = clock64();
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  unsigned* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  const int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    double n = (double)threads * iters * 8;
    k_cvt<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_cvt<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cvt.bf16x2     threads %4d: %.2f instr/clk/SM\n", threads, n / h[0]);
    k_ex2_only<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_ex2_only<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double c_ex = (double)h[0];
    printf("ex2            threads %4d: %.2f ops/clk/SM\n", threads, n / h[0]);
    k_ex2_cvt<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_ex2_cvt<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("ex2 + cvt/2    threads %4d: %.2f ex2/clk/SM (time x%.2f of ex2 alone)\n", threads, n / h[0], h[0] / c_ex);
    k_prmt<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_prmt<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("prmt           threads %4d: %.2f instr/clk/SM\n", threads, n / h[0]);
    k_ex2_h2<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_ex2_h2<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("ex2.f16x2      threads %4d: %.2f instr/clk/SM (x2 exps)\n", threads, n / h[0]);
    k_ex2_bf2<<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    k_ex2_bf2<<<148, threads>>>(out, iters, cyc); cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("ex2.bf16x2     threads %4d: %.2f instr/clk/SM (x2 exps)\n", threads, n / h[0]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
