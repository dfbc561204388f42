// Microbenchmark: legacy mma.sync throughput of the low-precision shapes on sm_100a (BF16 / FP16 / TF32
// inputs, FP32 accumulation) next to FP64 DMMA -- sizing data for the mixed-precision preconditioner.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
template <int KIND>
__global__ void mma_kernel(float* out, float seed) {
  unsigned a[4], b[2];
  float c[8][4];
#pragma unroll
  for (int i = 0; i < 4; i++) a[i] = __float_as_uint(seed + i + threadIdx.x);
#pragma unroll
  for (int i = 0; i < 2; i++) b[i] = __float_as_uint(seed * i);
#pragma unroll
  for (int j = 0; j < 8; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) c[j][i] = 0.f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (KIND == 0) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 1) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else {  // FFMA
#pragma unroll
        for (int i = 0; i < 4; i++) c[j][i] = fmaf(__uint_as_float(a[i]), __uint_as_float(b[i & 1]), c[j][i]);
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++)
#pragma unroll
    for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

template <int KIND>
double run(int blocks, int threads) {
  float* d;
  cudaMalloc(&d, 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_kernel<KIND><<<blocks, threads>>>(d, 1.0f);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) mma_kernel<KIND><<<blocks, threads>>>(d, 1.0f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flop_per_instr = KIND == 0 || KIND == 1 ? 2.0 * 16 * 8 * 16 : KIND == 2 ? 2.0 * 16 * 8 * 8 : 2.0 * 4 * 32;
  double flops = 5.0 * blocks * (threads / 32) * (double)ITERS * 8 * flop_per_instr;
  cudaFree(d);
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int w : {4, 8, 16}) {
    int t = 32 * w;
    printf("warps/blk %2d: bf16 m16n8k16 %.1f  f16 m16n8k16 %.1f  tf32 m16n8k8 %.1f  FFMA %.1f TFLOP/s\n", w,
           run<0>(sms * 2, t), run<1>(sms * 2, t), run<2>(sms * 2, t), run<3>(sms * 2, t));
  }
  return 0;
}
