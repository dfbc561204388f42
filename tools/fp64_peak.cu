// Microbenchmark: FP64 throughput of DMMA shapes and DFMA on sm_100a.
// Used once to pick the MMA shape and to measure the FP64 roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
template <int SHAPE>
__global__ void dmma_kernel(double* out, double seed) {
  double a[8], b[4], c[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = seed + i + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; i++) b[i] = seed * i;
#pragma unroll
  for (int j = 0; j < 8; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) c[j][i] = 0.0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (SHAPE == 4) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 8) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else if (SHAPE == 16) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      } else if (SHAPE == 1) {  // m8n8k4
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      } else {  // DFMA: 4 independent chains per j
#pragma unroll
        for (int i = 0; i < 4; i++) c[j][i] = fma(a[i], b[i & 3], c[j][i]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int SHAPE>
double run(int blocks, int threads) {
  double* d; cudaMalloc(&d, 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_kernel<SHAPE><<<blocks, threads>>>(d, 1.0);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) dmma_kernel<SHAPE><<<blocks, threads>>>(d, 1.0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flop_per_instr = SHAPE == 4 ? 2.0*16*8*4 : SHAPE == 8 ? 2.0*16*8*8 : SHAPE == 16 ? 2.0*16*8*16 : SHAPE == 1 ? 2.0*8*8*4 : 2.0*4*32;
  double flops = 5.0 * blocks * (threads / 32) * (double)ITERS * 8 * flop_per_instr;
  cudaFree(d);
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int w : {4, 8, 16}) {
    int t = 32 * w;
    printf("warps/blk %2d: m8n8k4 %.2f  m16n8k4 %.2f  m16n8k8 %.2f  m16n8k16 %.2f  DFMA %.2f TFLOP/s\n", w,
           run<1>(sms * 2, t), run<4>(sms * 2, t), run<8>(sms * 2, t), run<16>(sms * 2, t), run<0>(sms * 2, t));
  }
  return 0;
}
