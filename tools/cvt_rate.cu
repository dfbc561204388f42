// Throughput of cvt.rn.f32.f64 (F2F.F32.F64) against FP64 add and FP32 FMA on one SM: 512 threads, 16 independent values
// per thread (the FFT kernel's FP32 applies convert their FP64 operand on load).
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void __launch_bounds__(512, 1) k(const double* in, float* out, long long* cyc, int mode) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = in[threadIdx.x * 16 + i];
  float acc[16];
  for (int i = 0; i < 16; ++i) acc[i] = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 256; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (mode == 0) acc[i] += (float)x[i];              // cvt + FADD
      else if (mode == 1) x[i] = x[i] + 1.0;             // DADD
      else acc[i] = fmaf(acc[i], 1.0001f, 0.5f);         // FFMA
      if (mode == 0) x[i] = __longlong_as_double(__double_as_longlong(x[i]) ^ (long long)it);  // defeat hoisting
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[mode] = t1 - t0;
  float s = 0.f;
  for (int i = 0; i < 16; ++i) s += acc[i] + (float)x[i];
  out[threadIdx.x] = s;
}
int main() {
  double* in; float* out; long long* cyc;
  cudaMalloc(&in, 512 * 16 * 8); cudaMemset(in, 0, 512 * 16 * 8);
  cudaMalloc(&out, 512 * 4); cudaMalloc(&cyc, 3 * 8);
  for (int m = 0; m < 3; ++m) { k<<<1, 512>>>(in, out, cyc, m); k<<<1, 512>>>(in, out, cyc, m); }
  cudaDeviceSynchronize();
  long long h[3]; cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  const double n = 512.0 * 16 * 256;
  printf("cvt.f32.f64 (+FADD, +LOP): %.2f thread-ops/clk/SM; DADD: %.2f; FFMA: %.2f\n", n / h[0], n / h[1], n / h[2]);
  return 0;
}
