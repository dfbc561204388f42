// DMMA throughput under different operand patterns (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
__device__ __forceinline__ void mma(double (&c)[4], double a0, double a1, double b0) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b0));
}
// MODE 0: shared a,b regs. MODE 1: distinct regs per mma (WR=2 x NF=4 tile, like the kernel), no loads.
// MODE 2: like 1 but operands loaded from shared memory each k-step (kernel-like).
template <int MODE, int WR, int NF>
__global__ void k(double* out, double seed) {
  __shared__ double sm[6144];
  for (int i = threadIdx.x; i < 6144; i += blockDim.x) sm[i] = seed * i;
  __syncthreads();
  double c[WR][NF][4];
  for (int i = 0; i < WR; i++) for (int j = 0; j < NF; j++) for (int e = 0; e < 4; e++) c[i][j][e] = 0;
  double a[WR][2], b[NF];
  for (int i = 0; i < WR; i++) { a[i][0] = seed + i; a[i][1] = seed - i; }
  for (int j = 0; j < NF; j++) b[j] = seed * j;
  const int lane = threadIdx.x & 31;
  const double* As = sm + (lane >> 2) * 132 + (lane & 3);
  const double* Bs = sm + 5000 + (lane >> 2) - (lane & 3) + 64;
  for (int it = 0; it < ITERS; it++) {
    if (MODE == 2) {
      const int k0 = (it & 15) * 4;
#pragma unroll
      for (int i = 0; i < WR; i++) { a[i][0] = As[16 * i * 132 + k0]; a[i][1] = As[(16 * i + 8) * 132 + k0]; }
#pragma unroll
      for (int j = 0; j < NF; j++) b[j] = Bs[8 * j - k0];
    }
#pragma unroll
    for (int i = 0; i < WR; i++)
#pragma unroll
      for (int j = 0; j < NF; j++) {
        if (MODE == 0) mma(c[i][j], a[0][0], a[0][1], b[0]);
        else mma(c[i][j], a[i][0], a[i][1], b[j]);
      }
  }
  double s = 0;
  for (int i = 0; i < WR; i++) for (int j = 0; j < NF; j++) for (int e = 0; e < 4; e++) s += c[i][j][e];
  if (s == 1.2345) out[threadIdx.x] = s;
}
template <int MODE, int WR, int NF>
double run(int blocks, int threads) {
  double* d; cudaMalloc(&d, 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE, WR, NF><<<blocks, threads>>>(d, 1.0);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) k<MODE, WR, NF><<<blocks, threads>>>(d, 1.0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 5.0 * blocks * (threads / 32) * (double)ITERS * WR * NF * 2.0 * 16 * 8 * 4;
  cudaFree(d);
  return flops / (ms * 1e-3) / 1e12;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {8, 16}) {
    int t = 32 * w;
    printf("warps %2d | same-regs 2x4: %.2f | distinct 2x4: %.2f  1x4: %.2f  1x2: %.2f | smem 2x4: %.2f  1x4: %.2f  1x2: %.2f TF/s\n", w,
           run<0, 2, 4>(sms, t), run<1, 2, 4>(sms, t), run<1, 1, 4>(sms, t), run<1, 1, 2>(sms, t),
           run<2, 2, 4>(sms, t), run<2, 1, 4>(sms, t), run<2, 1, 2>(sms, t));
  }
  return 0;
}
