// FFT chain kernel for the 255^2 grids (BASELINE config 3): the same chain / (P)CG / MGRIT-epilogue
// semantics as the large-grid DMMA kernel (rm_big.cu), with every operator evaluated in FP64 through
// 512-point FFTs instead of dense Toeplitz contractions.
//
// Why: the block-Toeplitz step operator M + s(Kx Ax + Ky Ay) (reference assembly.py:100-115, 155-161)
// is a sum of six 2-level Toeplitz terms -- along x, g_t(i - k) acting on rows j, j+1, j-1 (t = 0, 1, 2);
// along y, g_t(j - l) acting on columns i, i+1, i-1 (t = 3, 4, 5) -- plus the 7-point P1 mass.  A
// Toeplitz block of order n <= 255 is a circular convolution of length L = 512 >= 2n - 1, so one apply
// costs O(n^2 log n) instead of the 8 n^3 FLOPs of the dense contraction (16.6 MF vs 133 MF at 255^2),
// at FP64 rounding (measured ~2e-16 relative against the dense reference operator).  The tau
// preconditioner's orthonormal DST-I of order 255 is the odd extension of a 512-point FFT, so both halves
// of a PCG iteration run on one FFT primitive.  SURVEY.md §8(f)3 ("FFT Toeplitz matvec").
//
// Layout.  A chain (one F-interval, or one C-point solve) is owned by G = 8 CTAs (cooperative launch,
// global-memory group barrier, one CTA per SM): CTA r owns grid rows [32 r, 32 r + 32) ("owner" phases:
// thread (warp w, lane t) holds rows 32 r + w and 32 r + w + 16 at columns t + 32 m, m < 8) and, for the
// y-direction passes, columns [32 r, 32 r + 32) (data staged through shared memory).  Two real rows
// (columns) are transformed as one complex sequence (re, im), 16 + 2 halo pairs per pass, each by one
// warp; the 18 spectra stay in shared memory for the 3-row (3-column) coupling of the Toeplitz terms.
// Per-chain vectors live in an L2-resident scratch in natural [256][256] order: PV (operand: p, the step
// input, x for true residuals; read across CTAs), W (y-pass output), SR (row-DST output), X, R, B.
//
// 512-point FFT of one warp, N = 16 x 32: thread t holds x[t + 32 m] (m < 16); a register radix-16 DFT
// over m, twiddles W512^{t q}, a transpose through shared memory, a register radix-16 DFT over the even
// or odd half of t, and a radix-2 step between lane pairs (shuffles).  The spectrum X[q + 16 (r + 16 v)]
// ends in thread 2 q + v, register r ("k-layout"); the inverse runs the same stages backwards, so a
// forward/inverse pair needs no reordering.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <vector>

#include "riesz_mgrit_b200.h"
#include "rm_device.cuh"
#include "rm_kernels.h"

namespace rm {
namespace fft {

constexpr int NP = 256;               // padded order (n = 255)
constexpr int L = 512;                // transform length
constexpr int G = 8;                  // CTAs per chain
constexpr int RS = NP / G;            // rows (columns) per CTA
constexpr int H = RS / 2;             // packing partner offset
constexpr int THREADS = 512;
constexpr int WARPS = 16;
constexpr int NSLOT = H + 2;          // packed pairs incl. the +-1 halo
constexpr int SLOT = 548;             // double2 per slot: >= 16 x 34 transpose scratch
constexpr int TS = 34;                // transpose row stride (conflict-free 16-byte accesses)
constexpr int NVEC = 6;               // per-chain vectors
constexpr size_t VEC = (size_t)NP * NP;
constexpr size_t SMEM = sizeof(double2) * ((size_t)NSLOT * SLOT + L + 16 + 6 * L) + sizeof(double) * (4 * 32) + 64;
static_assert(SMEM <= 227 * 1024, "shared memory budget");

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 shfl_xor2(double2 a, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m));
}

// DFT of length 4: forward kernel W4 = -i, inverse +i
template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  if (!INV) {
    a1 = make_double2(d02.x + d13.y, d02.y - d13.x);
    a3 = make_double2(d02.x - d13.y, d02.y + d13.x);
  } else {
    a1 = make_double2(d02.x - d13.y, d02.y + d13.x);
    a3 = make_double2(d02.x + d13.y, d02.y - d13.x);
  }
}

// y *= W16^{e} (forward) or W16^{-e} (inverse), e in {1, 2, 3, 4, 6, 9}
template <bool INV, int E>
__device__ __forceinline__ void tw16(double2& y) {
  constexpr double C1 = 0.92387953251128674, S1 = 0.38268343236508978, R2 = 0.70710678118654752;
  if constexpr (E == 4) {
    y = INV ? make_double2(-y.y, y.x) : make_double2(y.y, -y.x);
  } else {
    constexpr double c = E == 1 ? C1 : E == 2 ? R2 : E == 3 ? S1 : E == 6 ? -R2 : -C1;
    constexpr double sn = E == 1 ? S1 : E == 2 ? R2 : E == 3 ? C1 : E == 6 ? R2 : -S1;  // sin(2 pi E / 16)
    const double2 w = make_double2(c, INV ? sn : -sn);
    y = cmul(y, w);
  }
}

// in place: a[k] = sum_n a[n] W16^{+-nk}
template <bool INV>
__device__ __forceinline__ void dft16(double2 (&a)[16]) {
  // n = 4 n1 + n2, k = k1 + 4 k2
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(a[n2], a[4 + n2], a[8 + n2], a[12 + n2]);
  // a[4 k1 + n2] = Y[n2][k1]; twiddle W16^{n2 k1}
  tw16<INV, 1>(a[4 + 1]);
  tw16<INV, 2>(a[4 + 2]);
  tw16<INV, 3>(a[4 + 3]);
  tw16<INV, 2>(a[8 + 1]);
  tw16<INV, 4>(a[8 + 2]);
  tw16<INV, 6>(a[8 + 3]);
  tw16<INV, 3>(a[12 + 1]);
  tw16<INV, 6>(a[12 + 2]);
  tw16<INV, 9>(a[12 + 3]);
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(a[4 * k1], a[4 * k1 + 1], a[4 * k1 + 2], a[4 * k1 + 3]);
  // a[4 k1 + k2] = X[k1 + 4 k2] -> a[k]
  double2 t[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) t[k] = a[4 * (k & 3) + (k >> 2)];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = t[k];
}

// forward 512-point FFT of one warp.  in: a[m] = x[lane + 32 m]; out: a[r] = X[q + 16 (r + 16 v)] with
// q = lane >> 1, v = lane & 1.  `scr` (>= 16 x TS double2) is clobbered.
__device__ __forceinline__ void fft512_fwd(double2 (&a)[16], double2* scr, const double2* tw2, const double2* tw32,
                                           int lane) {
  dft16<false>(a);
#pragma unroll
  for (int q = 1; q < 16; ++q) a[q] = cmul(a[q], tw2[q * 32 + lane]);  // W512^{lane q}
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 16; ++q) scr[q * TS + lane] = a[q];
  __syncwarp();
  const int q2 = lane >> 1, v = lane & 1;
#pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = scr[q2 * TS + 2 * u + v];
  dft16<false>(a);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double2 o = shfl_xor2(a[r], 1);
    const double2 a0 = v ? o : a[r], a1 = v ? a[r] : o;
    const double2 t = cmul(a1, tw32[r]);
    a[r] = v ? csub(a0, t) : cadd(a0, t);
  }
}

// unnormalised inverse (x 512) of fft512_fwd: in k-layout, out a[m] = 512 x[lane + 32 m]
__device__ __forceinline__ void fft512_inv(double2 (&a)[16], double2* scr, const double2* tw2, const double2* tw32,
                                           int lane) {
  const int q2 = lane >> 1, v = lane & 1;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double2 o = shfl_xor2(a[r], 1);
    const double2 y0 = v ? o : a[r], y1 = v ? a[r] : o;
    a[r] = v ? cmulc(csub(y0, y1), tw32[r]) : cadd(y0, y1);
  }
  dft16<true>(a);
  __syncwarp();
#pragma unroll
  for (int u = 0; u < 16; ++u) scr[q2 * TS + 2 * u + v] = a[u];
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = scr[q * TS + lane];
#pragma unroll
  for (int q = 1; q < 16; ++q) a[q] = cmulc(a[q], tw2[q * 32 + lane]);
  dft16<true>(a);
}

__device__ __forceinline__ int klay(int lane, int r) { return (lane >> 1) + 16 * (r + 16 * (lane & 1)); }

// orthonormal DST-I (order 255) of a packed pair, forward-FFT form.  in: a[m] = (x_a, x_b)[lane + 32 m],
// m < 8 (index 255 must be 0); out: k-layout w[k] = ((S x_a)[k-1], (S x_b)[k-1]) for 1 <= k <= 255 (and the
// odd mirror w[512 - k] = -w[k]).  `slot` is clobbered.
__device__ __forceinline__ void dst_fwd(double2 (&a)[16], double2* slot, const double2* tw2, const double2* tw32,
                                        int lane, double half_c) {
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 8; ++m) slot[lane + 32 * m] = a[m];
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int n = lane + 32 * m;
    if (m < 8) {
      a[m] = n >= 1 ? slot[n - 1] : make_double2(0.0, 0.0);
    } else {
      const double2 t = slot[(511 - n) & 511];
      a[m] = n >= 257 ? make_double2(-t.x, -t.y) : make_double2(0.0, 0.0);
    }
  }
  fft512_fwd(a, slot, tw2, tw32, lane);
  // (S x)[k-1] = c D[k], X = FFT(ext) = -2 i D  ->  w = (c/2) i X
#pragma unroll
  for (int r = 0; r < 16; ++r) a[r] = make_double2(-half_c * a[r].y, half_c * a[r].x);
}

// orthonormal DST-I from k-layout odd-symmetric input w (w[0] = w[256] = 0, w[512-k] = -w[k]), inverse-FFT
// form.  out: a[m] = ((S w_a), (S w_b))[lane + 32 m], m < 8 (index 255 -> 0).  `slot` is clobbered.
__device__ __forceinline__ void dst_inv(double2 (&a)[16], double2* slot, const double2* tw2, const double2* tw32,
                                        int lane, double half_c) {
  fft512_inv(a, slot, tw2, tw32, lane);
  // I = sum_k w[k] e^{+2 pi i k n / L} = 2 i D(w)[n]  ->  (S w)[n-1] = c D[n] = (c/2)(-i) I[n]
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 8; ++m) slot[lane + 32 * m] = a[m];
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int i = lane + 32 * m;
    const double2 t = slot[(i + 1) & 511];
    a[m] = i + 1 <= 255 ? make_double2(half_c * t.y, -half_c * t.x) : make_double2(0.0, 0.0);
  }
}

// fast 1/d (d > 0, preconditioner scaling: ~1e-14 relative, deterministic)
__device__ __forceinline__ double rcp_fast(double d) {
  const double y = (double)__frcp_rn((float)d);
  const double e = fma(-d, y, 1.0);
  return fma(y, e, y) + y * e * e;
}

struct Sync {
  unsigned* gbar;
  double* gred;  // [2 buffers][4 values][G]
  int* sched;
  unsigned epoch;
};

__device__ __forceinline__ void gsync(Sync& sy) {
  __syncthreads();
  if (threadIdx.x == 0) {
    sy.epoch += 1;
    __threadfence();
    atomicAdd(sy.gbar, 1u);
    const unsigned target = sy.epoch * (unsigned)G;
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sy.gbar) : "memory");
      if (v >= target) break;
      __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// deterministic group sum of NV per-thread partials: warp butterfly -> warps in order -> CTAs in rank order
template <int NV>
__device__ __forceinline__ void greduce(double (&part)[NV], double* wred, Sync& sy, int& buf, int rank, int warp,
                                        int lane, double (&out)[NV]) {
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const double x = warp_allsum(part[v]);
    if (lane == 0) wred[v * 32 + warp] = x;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double x = warp_allsum(lane < WARPS ? wred[v * 32 + lane] : 0.0);
      if (lane == 0) sy.gred[(buf * 4 + v) * G + rank] = x;
    }
  }
  gsync(sy);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < G; ++q) x += __ldcg(sy.gred + (buf * 4 + v) * G + q);
    out[v] = x;
  }
  buf ^= 1;
}

}  // namespace fft

#define RM_OWN_FOR _Pragma("unroll") for (int p = 0; p < 2; ++p) _Pragma("unroll") for (int m = 0; m < 8; ++m)

template <bool PRE>
__global__ void __launch_bounds__(fft::THREADS, 1) chain_fft_kernel(const ChainArgs P) {
  using namespace fft;
  extern __shared__ __align__(16) double2 sm2[];
  double2* slots = sm2;                  // NSLOT x SLOT
  double2* tw2 = slots + NSLOT * SLOT;   // tw2[q * 32 + t] = W512^{q t}
  double2* tw32 = tw2 + L;               // W32^r = W512^{16 r}
  double2* sym = tw32 + 16;              // 6 stiffness spectra in k-layout
  double* wred = reinterpret_cast<double*>(sym + 6 * L);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = blockIdx.x % G;
  const int R0 = RS * rank, C0 = RS * rank;
  const int cid = blockIdx.x / G;

  Sync sy;
  sy.gbar = P.gbar + (size_t)cid * 32;
  sy.gred = P.gbuf + (size_t)cid * 1024;
  sy.sched = reinterpret_cast<int*>(sy.gred + 8 * G);
  sy.epoch = 0;

  for (int i = tid; i < L; i += THREADS) {
    const int q = i >> 5, t = i & 31;
    double sn, cs;
    sincospi(-2.0 * (double)(q * t) / (double)L, &sn, &cs);
    tw2[i] = make_double2(cs, sn);
  }
  if (tid < 16) {
    double sn, cs;
    sincospi(-2.0 * (double)(16 * tid) / (double)L, &sn, &cs);
    tw32[tid] = make_double2(cs, sn);
  }
  for (int i = tid; i < 6 * L; i += THREADS) sym[i] = P.fsym[i];

  const rm_sweep& W_ = P.sw;
  const int nx = P.nx, ny = P.ny;
  const double cm = P.cm;
  const int64_t max_iter = W_.max_iter > 0 ? W_.max_iter : 10 * (int64_t)nx * ny;
  const bool need_in = W_.explicit_rhs || W_.x0_mode == 1;
  const double half_c = 0.5 * sqrt(2.0 / (double)(nx + 1));
  const double inv_l = 1.0 / (double)L;

  double* base = P.fscratch + (size_t)cid * NVEC * VEC;
  double* PV = base;            // operand (read across CTAs)
  double* WV = base + VEC;      // y-pass output
  double* SR = base + 2 * VEC;  // row-DST output
  double* XV = base + 3 * VEC;  // iterate (owner rows)
  double* RV = base + 4 * VEC;  // residual
  double* BV = base + 5 * VEC;  // right-hand side
  // zero this chain slot's vectors once (padding row / column 255 is never written afterwards)
  for (size_t i = (size_t)rank * THREADS + tid; i < NVEC * VEC; i += (size_t)G * THREADS) base[i] = 0.0;
  int buf = 0;
  gsync(sy);

  auto own_j = [&](int p) { return R0 + warp + H * p; };
  auto own_i = [&](int m) { return lane + 32 * m; };
  auto valid = [&](int j, int i) { return j < ny && i < nx; };
  auto pv = [&](int j, int i) -> double { return (j >= 0 && i >= 0) ? __ldcg(PV + j * NP + i) : 0.0; };
  auto mass_pv = [&](int j, int i) -> double {
    double s = 6.0 * pv(j, i);
    s += pv(j, i - 1);
    s += pv(j, i + 1);
    s += pv(j + 1, i);
    s += pv(j + 1, i + 1);
    s += pv(j - 1, i);
    s += pv(j - 1, i - 1);
    return cm * s;
  };

  // ---- y-direction pass of the stiffness apply: WV[:, own columns] = (1/L) sum_t IFFT(S_t FFT(PV col +- 0/1))
  auto col_pass_apply = [&]() {
    // stage columns C0-1 .. C0+32 into slots s = 0..17 (pair (C0+s-1, C0+s+15)), natural row order
    for (int idx = tid; idx < NP * 34; idx += THREADS) {
      const int j = idx / 34, o = idx % 34 - 1, c = C0 + o;
      const double v = (c >= 0 && c < NP) ? __ldcg(PV + j * NP + c) : 0.0;
      if (o <= 16) slots[(o + 1) * SLOT + j].x = v;
      if (o >= 15) slots[(o - 15) * SLOT + j].y = v;
    }
    for (int idx = tid; idx < NSLOT * (L - NP); idx += THREADS)
      slots[(idx / (L - NP)) * SLOT + NP + idx % (L - NP)] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int s = warp; s < NSLOT; s += WARPS) {
      double2 a[16];
      double2* sl = slots + s * SLOT;
#pragma unroll
      for (int m = 0; m < 16; ++m) a[m] = sl[lane + 32 * m];
      fft512_fwd(a, sl, tw2, tw32, lane);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 16; ++r) sl[r * 32 + lane] = a[r];
    }
    __syncthreads();
    double2 a[16];
    {
      const double2* s0 = slots + (warp + 1) * SLOT;  // columns i
      const double2* sp = s0 + SLOT;                  // columns i + 1
      const double2* sm = s0 - SLOT;                  // columns i - 1
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int e = r * 32 + lane;
        double2 y = cmul(sym[3 * L + e], s0[e]);
        y = cadd(y, cmul(sym[4 * L + e], sp[e]));
        a[r] = cadd(y, cmul(sym[5 * L + e], sm[e]));
      }
    }
    __syncthreads();
    {
      double2* sl = slots + (warp + 1) * SLOT;
      fft512_inv(a, sl, tw2, tw32, lane);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 8; ++m) sl[lane + 32 * m] = cscale(a[m], inv_l);
    }
    __syncthreads();
    for (int idx = tid; idx < NP * RS; idx += THREADS) {
      const int j = idx / RS, o = idx % RS;
      const double2 t = slots[(o < H ? o + 1 : o - H + 1) * SLOT + j];
      WV[j * NP + C0 + o] = o < H ? t.x : t.y;
    }
  };

  // ---- x-direction pass for the owner rows: acc = (1/L) sum_t IFFT(S_t FFT(PV rows j + 0/+1/-1))
  auto row_pass_apply = [&](double (&acc)[2][8]) {
    for (int s = warp; s < NSLOT; s += WARPS) {
      const int ja = R0 + s - 1, jb = R0 + s - 1 + H;
      double2 a[16];
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        const int i = lane + 32 * m;
        a[m] = make_double2(m < 8 && ja >= 0 && ja < NP ? __ldcg(PV + ja * NP + i) : 0.0,
                            m < 8 && jb < NP ? __ldcg(PV + jb * NP + i) : 0.0);
      }
      double2* sl = slots + s * SLOT;
      fft512_fwd(a, sl, tw2, tw32, lane);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 16; ++r) sl[r * 32 + lane] = a[r];
    }
    __syncthreads();
    double2 a[16];
    {
      const double2* s0 = slots + (warp + 1) * SLOT;
      const double2* sp = s0 + SLOT;
      const double2* sm = s0 - SLOT;
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int e = r * 32 + lane;
        double2 y = cmul(sym[0 * L + e], s0[e]);
        y = cadd(y, cmul(sym[1 * L + e], sp[e]));
        a[r] = cadd(y, cmul(sym[2 * L + e], sm[e]));
      }
    }
    __syncthreads();
    fft512_inv(a, slots + (warp + 1) * SLOT, tw2, tw32, lane);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      acc[0][m] = a[m].x * inv_l;
      acc[1][m] = a[m].y * inv_l;
    }
  };

  // acc = (M + sg K) PV for the owner rows (PV complete and visible; one group barrier inside)
  auto apply_pv = [&](double (&acc)[2][8], double sg) {
    col_pass_apply();
    gsync(sy);
    row_pass_apply(acc);
    RM_OWN_FOR {
      const int j = own_j(p), i = own_i(m);
      acc[p][m] = valid(j, i) ? mass_pv(j, i) + sg * (acc[p][m] + __ldcg(WV + j * NP + i)) : 0.0;
    }
  };

  // z = P(s)^-1 r = (Sy x Sx) diag(1/d(s)) (Sy x Sx) r for the owner rows (two group barriers)
  auto precond = [&](const double (&r)[2][8], double (&z)[2][8], double s) {
    {  // SR[own rows] = Sx r (x-frequency along the row)
      double2 a[16];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = make_double2(r[0][m], r[1][m]);
      double2* sl = slots + warp * SLOT;
      dst_fwd(a, sl, tw2, tw32, lane, half_c);
      if ((lane & 1) == 0) {
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
          const int k = klay(lane, rr);
          if (k >= 1 && k <= 255) {
            SR[own_j(0) * NP + k - 1] = a[rr].x;
            SR[own_j(1) * NP + k - 1] = a[rr].y;
          }
        }
      }
    }
    gsync(sy);
    {  // column pass: WV[:, own columns] = Sy diag(1/d) Sy SR
      for (int idx = tid; idx < NP * RS; idx += THREADS) {
        const int j = idx / RS, o = idx % RS;
        const double v = __ldcg(SR + j * NP + C0 + o);
        if (o < H)
          slots[(o + 1) * SLOT + j].x = v;
        else
          slots[(o - H + 1) * SLOT + j].y = v;
      }
      __syncthreads();
      double2* sl = slots + (warp + 1) * SLOT;
      double2 a[16];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = sl[lane + 32 * m];
      dst_fwd(a, sl, tw2, tw32, lane, half_c);
      const int ca = C0 + warp, cb = C0 + warp + H;  // x-frequencies of the pair
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        const int k = klay(lane, rr);
        const int kk = k <= 256 ? k : 512 - k;
        double2 w = make_double2(0.0, 0.0);
        if (kk >= 1 && kk <= 255) {
          const double da = ca < nx ? __ldg(P.dmT + ca * nx + kk - 1) + s * __ldg(P.dkT + ca * nx + kk - 1) : 1.0;
          const double db = cb < nx ? __ldg(P.dmT + cb * nx + kk - 1) + s * __ldg(P.dkT + cb * nx + kk - 1) : 1.0;
          w = make_double2(a[rr].x * rcp_fast(da), a[rr].y * rcp_fast(db));
        }
        a[rr] = w;
      }
      dst_inv(a, sl, tw2, tw32, lane, half_c);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 8; ++m) sl[lane + 32 * m] = a[m];
      __syncthreads();
      for (int idx = tid; idx < NP * RS; idx += THREADS) {
        const int j = idx / RS, o = idx % RS;
        const double2 t = slots[(o < H ? o + 1 : o - H + 1) * SLOT + j];
        WV[j * NP + C0 + o] = o < H ? t.x : t.y;
      }
    }
    gsync(sy);
    {  // z[own rows] = Sx WV[own rows]
      double2 a[16];
      const int ja = own_j(0), jb = own_j(1);
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        const int k = klay(lane, rr);
        double2 w = make_double2(0.0, 0.0);
        if (k >= 1 && k <= 255)
          w = make_double2(__ldcg(WV + ja * NP + k - 1), __ldcg(WV + jb * NP + k - 1));
        else if (k >= 257)
          w = make_double2(-__ldcg(WV + ja * NP + 511 - k), -__ldcg(WV + jb * NP + 511 - k));
        a[rr] = w;
      }
      dst_inv(a, slots + warp * SLOT, tw2, tw32, lane, half_c);
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        z[0][m] = valid(ja, own_i(m)) ? a[m].x : 0.0;
        z[1][m] = valid(jb, own_i(m)) ? a[m].y : 0.0;
      }
    }
  };

  auto put_pv = [&](const double (&v)[2][8]) {
    RM_OWN_FOR { PV[own_j(p) * NP + own_i(m)] = v[p][m]; }
  };

  for (;;) {
    if (rank == 0 && tid == 0) sy.sched[0] = atomicAdd(P.chain_counter, 1);
    gsync(sy);
    const int chain = __ldcg(sy.sched);
    gsync(sy);
    if (chain >= W_.nchains) break;
    const int n0 = W_.first + chain * W_.cstride;
    const int n1 = min(n0 + W_.clen - 1, W_.nmax);
    bool in_tile = false;
    bool chain_ok = false;
    double s_prev = 0.0;
    for (int n = n0; n <= n1; ++n) {
      const double s = 0.5 * W_.d_dt[n - 1];
      const double fs = W_.d_f ? (W_.d_fscale ? W_.d_fscale[n] : 1.0) : 0.0;
      const double* Fn = W_.d_f ? W_.d_f + (int64_t)n * W_.f_stride : nullptr;
      const bool rhs_free = need_in && W_.explicit_rhs && in_tile && chain_ok && W_.d_hg != nullptr &&
                            W_.d_gadd != nullptr && W_.d_sub == nullptr;
      const bool rhs_ain = need_in && W_.explicit_rhs && !in_tile && n >= 2 && W_.d_ain != nullptr &&
                           W_.d_hg != nullptr && !rhs_free;
      int64_t nmv = 0, npc = 0;
      double acc[2][8];
      RM_OWN_FOR { acc[p][m] = 0.0; }
      if (need_in && !in_tile) {
        const double* src = W_.d_src + (int64_t)(n - 1) * W_.src_stride;
        RM_OWN_FOR {
          const int j = own_j(p), i = own_i(m);
          PV[j * NP + i] = valid(j, i) ? __ldcg(src + j * nx + i) : 0.0;
        }
        gsync(sy);
      }
      if (rhs_free) {
        const double* Hn = W_.d_hg + (int64_t)(n - 1) * W_.hg_stride;
        const double q = s / s_prev;
        RM_OWN_FOR {
          const int j = own_j(p), i = own_i(m);
          if (valid(j, i)) {
            const int e = j * NP + i;
            acc[p][m] = (1.0 + q) * mass_pv(j, i) - q * (__ldcg(BV + e) - __ldcg(RV + e) + __ldcg(Hn + j * nx + i));
          }
        }
      } else if (rhs_ain) {
        const double* An = W_.d_ain + (int64_t)(n - 1) * W_.ain_stride;
        const double* Hn = W_.d_hg + (int64_t)(n - 1) * W_.hg_stride;
        const double q = s / (0.5 * W_.d_dt[n - 2]);
        RM_OWN_FOR {
          const int j = own_j(p), i = own_i(m);
          if (valid(j, i)) {
            const int gi = j * nx + i;
            acc[p][m] = (1.0 + q) * mass_pv(j, i) - q * (__ldcg(An + gi) + __ldcg(Hn + gi));
          }
        }
      } else if (need_in) {
        apply_pv(acc, -s);  // (M - s K) v
        nmv = 1;
      }
      s_prev = s;
      chain_ok = false;

      // right-hand side, initial iterate and residual
      double part[2] = {0.0, 0.0};
      RM_OWN_FOR {
        const int j = own_j(p), i = own_i(m);
        const int e = j * NP + i;
        double b = 0.0, x = 0.0, r = 0.0;
        if (valid(j, i)) {
          const double am = acc[p][m];
          if (W_.explicit_rhs) b = am;
          if (Fn) {
            const double f = fs * __ldcg(Fn + j * nx + i);
            b = W_.explicit_rhs ? f + b : f;
          }
          if (W_.x0_mode == 1) {
            x = __ldcg(PV + e);
            r = b - (2.0 * mass_pv(j, i) - am);  // (M + s K) v = 2 M v - (M - s K) v
          } else {
            r = b;
          }
        }
        BV[e] = b;
        XV[e] = x;
        RV[e] = r;
        part[0] += b * b;
        part[1] += r * r;
      }
      if (W_.x0_mode == 2 || W_.x0_mode == 4) {
        // given initial iterate (x0_mode 2, stepper.py:203) / apply probe (x0_mode 4: out = (M + s K) b)
        gsync(sy);  // every CTA done reading PV
        const double* x0 = W_.x0_mode == 2 ? W_.d_x0 + (int64_t)n * W_.x0_stride : Fn;
        const double sc = W_.x0_mode == 2 ? 1.0 : fs;
        RM_OWN_FOR {
          const int j = own_j(p), i = own_i(m);
          PV[j * NP + i] = valid(j, i) ? sc * __ldcg(x0 + j * nx + i) : 0.0;
        }
        gsync(sy);
        apply_pv(acc, s);
        ++nmv;
        part[1] = 0.0;
        RM_OWN_FOR {
          const int j = own_j(p), i = own_i(m);
          const int e = j * NP + i;
          if (W_.x0_mode == 4) {
            XV[e] = acc[p][m];
          } else {
            const double r = valid(j, i) ? __ldcg(BV + e) - acc[p][m] : 0.0;
            XV[e] = valid(j, i) ? __ldcg(PV + e) : 0.0;
            RV[e] = r;
            part[1] += r * r;
          }
        }
      }
      double tot[2];
      greduce<2>(part, wred, sy, buf, rank, warp, lane, tot);
      const double bnorm = sqrt(tot[0]);
      const double target = bnorm > 0.0 ? W_.rel_tol * bnorm : W_.rel_tol;
      if (W_.d_guess && W_.x0_mode < 3 && sqrt(tot[1]) > target) {
        const double* gu = W_.d_guess + (int64_t)n * W_.guess_stride;
        const double* Gr = W_.d_gadd ? W_.d_gadd + (int64_t)n * W_.gadd_stride : nullptr;
        const double* Ax0 = W_.d_gax ? W_.d_gax + (int64_t)n * W_.gax_stride : nullptr;
        double ag[2][8];
        if (!Ax0) {
          gsync(sy);  // every CTA done reading PV
          RM_OWN_FOR {
            const int j = own_j(p), i = own_i(m);
            double v = 0.0;
            if (valid(j, i)) {
              const int gi = j * nx + i;
              v = Gr ? __ldcg(gu + gi) - __ldcg(Gr + gi) : __ldcg(gu + gi);
            }
            PV[j * NP + i] = v;
          }
          gsync(sy);
          apply_pv(ag, s);
          ++nmv;
        }
        double pg[1] = {0.0};
        RM_OWN_FOR {
          const int j = own_j(p), i = own_i(m);
          double r = 0.0;
          if (valid(j, i)) r = __ldcg(BV + j * NP + i) - (Ax0 ? __ldcg(Ax0 + j * nx + i) : ag[p][m]);
          ag[p][m] = r;
          pg[0] += r * r;
        }
        double rg[1];
        greduce<1>(pg, wred, sy, buf, rank, warp, lane, rg);
        if (rg[0] < tot[1]) {
          tot[1] = rg[0];
          RM_OWN_FOR {
            const int j = own_j(p), i = own_i(m);
            const int e = j * NP + i;
            double x0 = 0.0;
            if (valid(j, i)) {
              const int gi = j * nx + i;
              x0 = Ax0 ? (Gr ? __ldcg(gu + gi) - __ldcg(Gr + gi) : __ldcg(gu + gi)) : __ldcg(PV + e);
            }
            XV[e] = x0;
            RV[e] = ag[p][m];
          }
        }
      }
      double res = sqrt(tot[1]);
      double rz = tot[1];
      int64_t its = 0;
      int fail = 0;
      bool done = res <= target || W_.x0_mode == 4;
      if (W_.x0_mode == 3) {
        // preconditioner probe: x = P^-1 b
        if constexpr (PRE) {
          double r0[2][8], z[2][8];
          RM_OWN_FOR { r0[p][m] = __ldcg(RV + own_j(p) * NP + own_i(m)); }
          precond(r0, z, s);
          ++npc;
          RM_OWN_FOR { XV[own_j(p) * NP + own_i(m)] = z[p][m]; }
        }
        done = true;
      }

      // p = z (PRE) or r into PV, after every CTA finished reading PV
      auto start_direction = [&]() {
        double r0[2][8], z[2][8];
        RM_OWN_FOR { r0[p][m] = __ldcg(RV + own_j(p) * NP + own_i(m)); }
        double pr[1] = {0.0};
        if constexpr (PRE) {
          precond(r0, z, s);
          ++npc;
          RM_OWN_FOR { pr[0] += r0[p][m] * z[p][m]; }
        } else {
          RM_OWN_FOR {
            z[p][m] = r0[p][m];
            pr[0] += r0[p][m] * r0[p][m];
          }
        }
        double o[1];
        greduce<1>(pr, wred, sy, buf, rank, warp, lane, o);  // also: every CTA is past its PV reads
        rz = o[0];
        put_pv(z);
        gsync(sy);
      };
      if (!done) start_direction();

      for (int64_t k = 1; !done; ++k) {
        if (k > max_iter) {
          fail = RM_CG_BUDGET;
          its = max_iter;
          break;
        }
        double ap[2][8];
        apply_pv(ap, s);
        ++nmv;
        double p1[1] = {0.0};
        RM_OWN_FOR { p1[0] += __ldcg(PV + own_j(p) * NP + own_i(m)) * ap[p][m]; }
        double pap[1];
        greduce<1>(p1, wred, sy, buf, rank, warp, lane, pap);
        if (!isfinite(pap[0]) || pap[0] <= 0.0) {
          fail = RM_CG_BREAKDOWN;
          its = k;
          break;
        }
        const double alpha = rz / pap[0];
        double rn[2][8];
        RM_OWN_FOR {
          const int e = own_j(p) * NP + own_i(m);
          XV[e] = __ldcg(XV + e) + alpha * __ldcg(PV + e);
          rn[p][m] = __ldcg(RV + e) - alpha * ap[p][m];
          RV[e] = rn[p][m];
        }
        double red2[2];
        double z[2][8];
        {
          double part2[2] = {0.0, 0.0};
          if constexpr (PRE) {
            precond(rn, z, s);
            ++npc;
            RM_OWN_FOR {
              part2[0] += rn[p][m] * rn[p][m];
              part2[1] += rn[p][m] * z[p][m];
            }
          } else {
            RM_OWN_FOR {
              z[p][m] = rn[p][m];
              part2[0] += rn[p][m] * rn[p][m];
            }
            part2[1] = part2[0];
          }
          greduce<2>(part2, wred, sy, buf, rank, warp, lane, red2);
        }
        res = sqrt(red2[0]);
        if (!isfinite(res)) {
          fail = RM_CG_NONFINITE;
          its = k;
          break;
        }
        if (res <= target) {
          // acceptance on the true residual (krylov.py:71-83); every CTA is past its PV reads
          double xv[2][8];
          RM_OWN_FOR { xv[p][m] = __ldcg(XV + own_j(p) * NP + own_i(m)); }
          put_pv(xv);
          gsync(sy);
          double ax[2][8];
          apply_pv(ax, s);
          ++nmv;
          double pt[1] = {0.0};
          RM_OWN_FOR {
            const int j = own_j(p), i = own_i(m);
            const double rt = valid(j, i) ? __ldcg(BV + j * NP + i) - ax[p][m] : 0.0;
            ax[p][m] = rt;
            pt[0] += rt * rt;
          }
          double tt[1];
          greduce<1>(pt, wred, sy, buf, rank, warp, lane, tt);
          const double true_res = sqrt(tt[0]);
          RM_OWN_FOR { RV[own_j(p) * NP + own_i(m)] = ax[p][m]; }
          if (true_res <= fmax(target, 10.0 * res)) {
            its = k;
            done = true;
            break;
          }
          res = true_res;  // recurrence drifted: restart from the true residual
          if (res <= target) {
            its = k;
            done = true;
            break;
          }
          start_direction();
          continue;
        }
        const double beta = red2[1] / rz;
        rz = red2[1];
        // p = z + beta p (every CTA finished reading PV: the reductions above were group barriers)
        RM_OWN_FOR {
          const int e = own_j(p) * NP + own_i(m);
          PV[e] = z[p][m] + beta * __ldcg(PV + e);
        }
        gsync(sy);
      }

      chain_ok = done && !fail && W_.x0_mode < 3;
      if (rank == 0 && tid == 0) {
        atomicAdd(W_.d_counters, 1ull);
        atomicAdd(W_.d_counters + 1, (unsigned long long)its);
        atomicAdd(W_.d_counters + 2, (unsigned long long)nmv);
        atomicAdd(W_.d_counters + 3, (unsigned long long)npc);
      }
      if (fail) {
        if (rank == 0 && tid == 0 && atomicCAS(P.fail, 0, fail) == 0) {
          P.fail_info[0] = (double)n;
          P.fail_info[1] = (double)its;
          P.fail_info[2] = res;
        }
        gsync(sy);
        break;
      }
      // ---------------- MGRIT epilogue: y = [G_n +] x [- S_n] ----------------
      const bool next_in_tile = n < n1 && need_in;
      const int oi = n / W_.out_div;
      const double* Gn = W_.d_gadd ? W_.d_gadd + (int64_t)n * W_.gadd_stride : nullptr;
      const double* Sn = W_.d_sub ? W_.d_sub + (int64_t)n * W_.sub_stride : nullptr;
      double* On = W_.d_out ? W_.d_out + (int64_t)oi * W_.out_stride : nullptr;
      double* Kn = W_.d_keep ? W_.d_keep + (int64_t)oi * W_.keep_stride : nullptr;
      double* An = W_.d_ax ? W_.d_ax + (int64_t)oi * W_.ax_stride : nullptr;
      gsync(sy);  // every CTA done reading PV before it is overwritten with y
      double py[1] = {0.0};
      RM_OWN_FOR {
        const int j = own_j(p), i = own_i(m);
        if (valid(j, i)) {
          const int gi = j * nx + i, e = j * NP + i;
          double y = __ldcg(XV + e);
          if (An) An[gi] = __ldcg(BV + e) - __ldcg(RV + e);  // A x = b - r (true residual)
          if (Gn) y = __ldcg(Gn + gi) + y;
          if (Kn) Kn[gi] = y;
          if (Sn) y = y - __ldcg(Sn + gi);
          if (On) On[gi] = y;
          if (next_in_tile) PV[e] = y;
          py[0] += y * y;
        }
      }
      if (W_.d_norms) {
        double yy[1];
        greduce<1>(py, wred, sy, buf, rank, warp, lane, yy);
        if (rank == 0 && tid == 0) W_.d_norms[oi] = yy[0];
      }
      in_tile = next_in_tile;
      gsync(sy);
    }
  }
}

#undef RM_OWN_FOR

// Host: spectra of the six stiffness tables (entry d + np of table t, |d| < n used) in k-layout order:
// out[2 (t L + r 32 + lane) + {0, 1}] = S_t[k], k = (lane >> 1) + 16 (r + 16 (lane & 1)).
void fft_symbols(const double* tab, int np, int gl, double* out) {
  const int L = fft::L, n = np - 1;
  std::vector<double> cs(L), sn(L);
  for (int i = 0; i < L; ++i) {
    cs[i] = cos(2.0 * M_PI * i / L);
    sn[i] = sin(2.0 * M_PI * i / L);
  }
  for (int t = 0; t < 6; ++t)
    for (int r = 0; r < 16; ++r)
      for (int lane = 0; lane < 32; ++lane) {
        const int k = (lane >> 1) + 16 * (r + 16 * (lane & 1));
        double re = 0.0, im = 0.0;
        for (int d = -(n - 1); d <= n - 1; ++d) {
          const double v = tab[t * gl + d + np];
          if (v == 0.0) continue;
          const int idx = (((d * k) % L) + L) % L;
          re += v * cs[idx];
          im -= v * sn[idx];
        }
        const size_t e = (size_t)t * L + r * 32 + lane;
        out[2 * e] = re;
        out[2 * e + 1] = im;
      }
}

bool fft_supported(int np, int nx, int ny) { return np == fft::NP && nx == fft::NP - 1 && ny == fft::NP - 1; }

int fft_group() { return fft::G; }

size_t fft_scratch_doubles_per_chain() { return fft::NVEC * fft::VEC; }

static cudaError_t fft_prepare(const void* kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft::SMEM);
}

cudaError_t fft_max_chains(int* out) {
  auto kern = chain_fft_kernel<true>;
  cudaError_t err = fft_prepare((const void*)kern);
  if (err != cudaSuccess) return err;
  int per_sm = 0, dev = 0, sms = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fft::THREADS, fft::SMEM);
  if (err != cudaSuccess) return err;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  *out = per_sm * sms / fft::G;
  return cudaSuccess;
}

cudaError_t launch_fft(const ChainArgs& a, int max_chains, cudaStream_t st) {
  auto kern = a.sw.precond ? chain_fft_kernel<true> : chain_fft_kernel<false>;
  cudaError_t err = fft_prepare((const void*)kern);
  if (err != cudaSuccess) return err;
  if (!a.gbar || !a.gbuf || !a.fscratch || !a.fsym) return cudaErrorInvalidValue;
  int nch = max_chains < a.sw.nchains ? max_chains : a.sw.nchains;
  if (nch < 1) nch = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch * fft::G);
  cfg.blockDim = dim3(fft::THREADS);
  cfg.dynamicSmemBytes = fft::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // the G CTAs of a chain are co-resident (group barrier)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace rm
