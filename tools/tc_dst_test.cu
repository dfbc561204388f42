// Stand-alone check of the tcgen05 DST stage used by the FFT chain kernel's preconditioner (rm_tc.cuh):
// D[k][n] = sum_i S[k][i] X[n][i], S the orthonormal DST-I matrix of order 255 (padded to 256) in FP16, X a strip of
// 32 rows, FP32 accumulation in TMEM.  Compares with a double-precision reference on the host.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_1805_06688_b200/csrc tools/tc_dst_test.cu -o tools/tc_dst_test
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "rm_tc.cuh"

using namespace rm::tc;

// variant with S resident in tensor memory (A operand from TMEM): no shared-memory copy of S at all
__global__ void __launch_bounds__(512, 1) dst_stage_ts_kernel(const __half* s_rowmajor, const float* x, float* out,
                                                              int reps, long long* cyc, int issuers) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __half* sB = reinterpret_cast<__half*>(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + B_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bars[1], issuers == 4 ? 4 : 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, TMEM_COLS_RESIDENT);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  load_matrix_tmem(tmem, s_rowmajor, warp, lane);
  tc_fence_before();
  __syncthreads();
  unsigned ph_mma = 0;
  for (int rep = 0; rep < reps; ++rep) {
    long long t0 = clock64();
    for (int e = tid; e < 32 * 256; e += 512) {
      const int n = e >> 8, i = e & 255;
      sB[b_index(n, i)] = __float2half_rn(x[e]);
    }
    fence_async_smem();
    long long t1 = clock64();
    tc_fence_before();
    __syncthreads();
    long long t2 = clock64();
    if (issuers == 4) {
      if ((warp & 3) == 0 && lane == 0) {
        tc_fence_after();
        issue_dst_mma_ts_part(sB, tmem, warp >> 2);
        tc_commit(&bars[1]);
      }
    } else if (tid == 0) {
      tc_fence_after();
      issue_dst_mma_ts(sB, tmem);
      tc_commit(&bars[1]);
    }
    mbar_wait(&bars[1], ph_mma);
    ph_mma ^= 1;
    tc_fence_after();
    long long t3 = clock64();
    float v[16];
    const int q = warp & 3, t = (warp >> 2) & 1, h = warp >> 3;
    if (issuers == 4) {
      float w[16];
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(TMEM_D_COL + 32 * (2 * t) + 16 * h), v);
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(TMEM_D_COL + 32 * (2 * t + 1) + 16 * h), w);
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] += w[c];
    } else {
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(TMEM_D_COL + 32 * t + 16 * h), v);
    }
    const int k = 128 * t + 32 * q + lane;
    float4* o4 = reinterpret_cast<float4*>(out + k * 32 + 16 * h);
#pragma unroll
    for (int c = 0; c < 4; ++c) o4[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    tc_fence_before();
    __syncthreads();
    long long t4 = clock64();
    if (tid == 0 && blockIdx.x == 0) {
      cyc[rep * 4 + 0] = t1 - t0;
      cyc[rep * 4 + 1] = t2 - t1;
      cyc[rep * 4 + 2] = t3 - t2;
      cyc[rep * 4 + 3] = t4 - t3;
    }
  }
  if (warp == 0) tmem_free(tmem, TMEM_COLS_RESIDENT);
}

__global__ void __launch_bounds__(512, 1) dst_stage_kernel(const __half* s_canon, const float* x, float* out, int reps,
                                                           long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __half* sA = reinterpret_cast<__half*>(smem);                    // 128 KB
  __half* sB = reinterpret_cast<__half*>(smem + A_BYTES);          // 16 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + A_BYTES + B_BYTES);  // [0] TMA, [1] MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  unsigned ph_tma = 0, ph_mma = 0;
  for (int rep = 0; rep < reps; ++rep) {
    long long t0 = clock64();
    if (tid == 0) load_matrix_async(sA, s_canon, &bars[0]);
    // B operand: rows n = 0..31 of x (FP32 [32][256]) -> FP16 canonical K-major
    for (int e = tid; e < 32 * 256; e += 512) {
      const int n = e >> 8, i = e & 255;
      sB[b_index(n, i)] = __float2half_rn(x[e]);
    }
    fence_async_smem();
    long long t1 = clock64();
    mbar_wait(&bars[0], ph_tma);
    ph_tma ^= 1;
    __syncthreads();
    long long t2 = clock64();
    if (tid == 0) {
      tc_fence_after();
      issue_dst_mma(sA, sB, tmem);
      tc_commit(&bars[1]);
    }
    mbar_wait(&bars[1], ph_mma);
    ph_mma ^= 1;
    tc_fence_after();
    long long t3 = clock64();
    float v[16];
    const int q = warp & 3, t = (warp >> 2) & 1, h = warp >> 3;
    tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * t + 16 * h), v);
    const int k = 128 * t + 32 * q + lane;
#pragma unroll
    for (int c = 0; c < 16; ++c) out[k * 32 + 16 * h + c] = v[c];
    tc_fence_before();
    __syncthreads();
    long long t4 = clock64();
    if (tid == 0 && blockIdx.x == 0) {
      cyc[rep * 4 + 0] = t1 - t0;
      cyc[rep * 4 + 1] = t2 - t1;
      cyc[rep * 4 + 2] = t3 - t2;
      cyc[rep * 4 + 3] = t4 - t3;
    }
  }
  if (warp == 0) tmem_free(tmem, TMEM_COLS);
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 3;
  std::vector<__half> s(256 * 256), srm(256 * 256);
  std::vector<double> sd(256 * 256, 0.0);
  const double c = sqrt(2.0 / 256.0);
  for (int k = 0; k < 256; ++k)
    for (int i = 0; i < 256; ++i) {
      const double v = (k < 255 && i < 255) ? c * sin(M_PI * (k + 1) * (i + 1) / 256.0) : 0.0;
      sd[k * 256 + i] = v;
      s[a_index(k, i)] = __float2half_rn((float)v);
      srm[k * 256 + i] = __float2half_rn((float)v);
    }
  std::vector<float> x(32 * 256);
  srand(1);
  for (auto& v : x) v = (float)rand() / RAND_MAX - 0.5f;
  __half* d_s;
  float *d_x, *d_o;
  cudaMalloc(&d_s, s.size() * 2);
  cudaMalloc(&d_x, x.size() * 4);
  cudaMalloc(&d_o, 256 * 32 * 4);
  cudaMemcpy(d_s, s.data(), s.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(d_x, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  const int smem = A_BYTES + B_BYTES + 64;
  cudaFuncSetAttribute(dst_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* d_c;
  cudaMalloc(&d_c, reps * 4 * 8);
  const int grid = argc > 2 ? atoi(argv[2]) : 1;
  const bool ts = argc > 3 && atoi(argv[3]);
  if (ts) {
    cudaMemcpy(d_s, srm.data(), srm.size() * 2, cudaMemcpyHostToDevice);
    dst_stage_ts_kernel<<<grid, 512, B_BYTES + 64>>>(d_s, d_x, d_o, reps, d_c, argc > 4 ? atoi(argv[4]) : 1);
  } else {
    dst_stage_kernel<<<grid, 512, smem>>>(d_s, d_x, d_o, reps, d_c);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> o(256 * 32);
  cudaMemcpy(o.data(), d_o, o.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0.0, maxref = 0.0;
  for (int k = 0; k < 256; ++k)
    for (int n = 0; n < 32; ++n) {
      double r = 0.0;
      for (int i = 0; i < 256; ++i) r += sd[k * 256 + i] * (double)x[n * 256 + i];
      maxerr = fmax(maxerr, fabs(r - (double)o[k * 32 + n]));
      maxref = fmax(maxref, fabs(r));
    }
  std::vector<long long> cy(reps * 4);
  cudaMemcpy(cy.data(), d_c, reps * 4 * 8, cudaMemcpyDeviceToHost);
  for (int r = 0; r < reps; ++r)
    printf("rep %d (grid %d): convert B %lld, wait S copy %lld, MMA issue->done %lld, ld+store %lld cycles\n", r, grid,
           cy[r * 4], cy[r * 4 + 1], cy[r * 4 + 2], cy[r * 4 + 3]);
  printf("max |ref| %.4f  max err %.3e (FP16 operands: expect ~1e-3)\n", maxref, maxerr);
  return maxerr < 5e-3 * maxref ? 0 : 2;
}
