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
#include "rm_tc.cuh"

#ifndef RM_STAGE_NB
#define RM_STAGE_NB 3  // column-staging loads in flight per thread and batch (x2 values)
#endif
#ifndef RM_CNT_T
#define RM_CNT_T int64_t  // per-solve iteration / apply counters
#endif
#ifndef RM_POLL_RELAXED
#define RM_POLL_RELAXED 0  // group barrier: relaxed polls + one acquire fence (1) or acquire polls (0)
#endif
#ifndef RM_STORE_NB
#define RM_STORE_NB 4  // column-store batch
#endif

namespace rm {
namespace fft {

constexpr int NP = 256;               // padded order (n = 255)
constexpr int L = 512;                // transform length
constexpr int G = 8;                  // CTAs per chain
constexpr int RS = NP / G;            // rows (columns) per CTA
constexpr int H = RS / 2;             // packing partner offset
constexpr int THREADS = 512;
constexpr int WARPS = 16;
constexpr int NOWN = 2;               // owner rows per thread (one packed pair per warp)
constexpr int PPW = NOWN / 2;          // packed pairs per warp
constexpr int NSLOT = H + 2;          // packed pairs incl. the +-1 halo
constexpr int SLOT = 545;             // double2 per slot: >= 16 x 34 transpose scratch; = 1 mod 8 (16-byte
                                      // accesses to consecutive slots hit distinct bank groups)
constexpr int TS = 34;                // transpose row stride (conflict-free 16-byte accesses)
constexpr int NVEC = 6;               // per-chain vectors
constexpr size_t VEC = (size_t)NP * NP;
constexpr size_t DIV = (size_t)H * 16 * 32 * 2;  // per-CTA 1/d(s) cache (doubles)
constexpr int SLOTF = 1089;            // float2 per slot in the FP32 (preconditioner) passes: odd -> conflict-free
static_assert(SLOTF * 8 <= SLOT * 16, "FP32 slots overlay the FP64 ones");
constexpr size_t SMEM_FFT = sizeof(double2) * ((size_t)NSLOT * SLOT + L + 16 + 3 * L) + sizeof(double) * (4 * 32) +
                            sizeof(float2) * (L + 16);
// tensor-core preconditioner (PRE == 2, rm_tc.cuh): the strip operand, the mbarriers and the tensor-memory base
// address follow the FFT tables (the DST matrix itself lives in tensor memory)
constexpr size_t OFF_TCB = (SMEM_FFT + 127) / 128 * 128;
constexpr size_t OFF_TCBAR = OFF_TCB + tc::B_BYTES;
// two more spectrum slots: the row pass's halo pairs are transformed during the column pass's halo round
constexpr size_t OFF_XSLOT = OFF_TCBAR + 64;
constexpr size_t SMEM = OFF_XSLOT + 2 * sizeof(double2) * SLOT;
static_assert(SMEM <= 227 * 1024, "shared memory budget");

// complex arithmetic on double2 / float2 (the preconditioner's DSTs run in FP32, see precond)
template <class V>
struct Cx;
template <>
struct Cx<double2> {
  using R = double;
  static __device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }
  static __device__ __forceinline__ double ffma(double a, double b, double c) { return fma(a, b, c); }
};
template <>
struct Cx<float2> {
  using R = float;
  static __device__ __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
  static __device__ __forceinline__ float ffma(float a, float b, float c) { return fmaf(a, b, c); }
};

template <class V>
__device__ __forceinline__ V cadd(V a, V b) { return Cx<V>::mk(a.x + b.x, a.y + b.y); }
template <class V>
__device__ __forceinline__ V csub(V a, V b) { return Cx<V>::mk(a.x - b.x, a.y - b.y); }
template <class V>
__device__ __forceinline__ V cmul(V a, V b) {
  return Cx<V>::mk(Cx<V>::ffma(a.x, b.x, -a.y * b.y), Cx<V>::ffma(a.x, b.y, a.y * b.x));
}
template <class V>
__device__ __forceinline__ V cmulc(V a, V b) {  // a * conj(b)
  return Cx<V>::mk(Cx<V>::ffma(a.x, b.x, a.y * b.y), Cx<V>::ffma(a.y, b.x, -a.x * b.y));
}
template <class V>
__device__ __forceinline__ V cscale(V a, typename Cx<V>::R s) { return Cx<V>::mk(a.x * s, a.y * s); }
template <class V>
__device__ __forceinline__ V shfl_xor2(V a, int m) {
  return Cx<V>::mk(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m));
}

// DFT of length 4: forward kernel W4 = -i, inverse +i
template <bool INV, class V>
__device__ __forceinline__ void dft4(V& a0, V& a1, V& a2, V& a3) {
  const V s02 = cadd(a0, a2), d02 = csub(a0, a2), s13 = cadd(a1, a3), d13 = csub(a1, a3);
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  if (!INV) {
    a1 = Cx<V>::mk(d02.x + d13.y, d02.y - d13.x);
    a3 = Cx<V>::mk(d02.x - d13.y, d02.y + d13.x);
  } else {
    a1 = Cx<V>::mk(d02.x - d13.y, d02.y + d13.x);
    a3 = Cx<V>::mk(d02.x + d13.y, d02.y - d13.x);
  }
}

// y *= W16^{e} (forward) or W16^{-e} (inverse), e in {1, 2, 3, 4, 6, 9}
template <bool INV, int E, class V>
__device__ __forceinline__ void tw16(V& y) {
  using R = typename Cx<V>::R;
  constexpr double C1 = 0.92387953251128674, S1 = 0.38268343236508978, R2 = 0.70710678118654752;
  if constexpr (E == 4) {
    y = INV ? Cx<V>::mk(-y.y, y.x) : Cx<V>::mk(y.y, -y.x);
  } else {
    constexpr double c = E == 1 ? C1 : E == 2 ? R2 : E == 3 ? S1 : E == 6 ? -R2 : -C1;
    constexpr double sn = E == 1 ? S1 : E == 2 ? R2 : E == 3 ? C1 : E == 6 ? R2 : -S1;  // sin(2 pi E / 16)
    const V w = Cx<V>::mk((R)c, (R)(INV ? sn : -sn));
    y = cmul(y, w);
  }
}

// in place: a[k] = sum_n a[n] W16^{+-nk}
template <bool INV, class V>
__device__ __forceinline__ void dft16(V (&a)[16]) {
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
  V t[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) t[k] = a[4 * (k & 3) + (k >> 2)];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = t[k];
}

// stage-1 twiddles W512^{lane q}, q = 1..15, from six table entries (q = a + 4 b: W^{lane a} W^{4 lane b});
// CONJ: their conjugates (inverse transform)
template <bool CONJ, class V>
__device__ __forceinline__ void twiddle_stage1(V (&a)[16], const V* tw2, int lane) {
  V wa[4], wb[4];
#pragma unroll
  for (int k = 1; k < 4; ++k) {
    wa[k] = tw2[k * 32 + lane];
    wb[k] = tw2[4 * k * 32 + lane];
  }
#pragma unroll
  for (int q = 1; q < 16; ++q) {
    const int qa = q & 3, qb = q >> 2;
    const V w = qa == 0 ? wb[qb] : (qb == 0 ? wa[qa] : cmul(wa[qa], wb[qb]));
    a[q] = CONJ ? cmulc(a[q], w) : cmul(a[q], w);
  }
}

// forward 512-point FFT of one warp.  in: a[m] = x[lane + 32 m]; out: a[r] = X[q + 16 (r + 16 v)] with
// q = lane >> 1, v = lane & 1.  `scr` (>= 16 x TS elements) is clobbered.
template <class V>
__device__ __forceinline__ void fft512_fwd(V (&a)[16], V* scr, const V* tw2, const V* tw32, int lane) {
  dft16<false>(a);
  twiddle_stage1<false>(a, tw2, lane);  // W512^{lane q}
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
    const V o = shfl_xor2(a[r], 1);
    const V a0 = v ? o : a[r], a1 = v ? a[r] : o;
    const V t = cmul(a1, tw32[r]);
    a[r] = v ? csub(a0, t) : cadd(a0, t);
  }
}

// unnormalised inverse (x 512) of fft512_fwd: in k-layout, out a[m] = 512 x[lane + 32 m]
template <class V>
__device__ __forceinline__ void fft512_inv(V (&a)[16], V* scr, const V* tw2, const V* tw32, int lane) {
  const int q2 = lane >> 1, v = lane & 1;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const V o = shfl_xor2(a[r], 1);
    const V y0 = v ? o : a[r], y1 = v ? a[r] : o;
    a[r] = v ? cmulc(csub(y0, y1), tw32[r]) : cadd(y0, y1);
  }
  dft16<true>(a);
  __syncwarp();
#pragma unroll
  for (int u = 0; u < 16; ++u) scr[q2 * TS + 2 * u + v] = a[u];
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = scr[q * TS + lane];
  twiddle_stage1<true>(a, tw2, lane);
  dft16<true>(a);
}

__device__ __forceinline__ int klay(int lane, int r) { return (lane >> 1) + 16 * (r + 16 * (lane & 1)); }

// orthonormal DST-I (order 255) of a packed pair, forward-FFT form.  in: a[m] = (x_a, x_b)[lane + 32 m],
// m < 8 (index 255 must be 0); out: k-layout w[k] = ((S x_a)[k-1], (S x_b)[k-1]) for 1 <= k <= 255 (and the
// odd mirror w[512 - k] = -w[k]).  `slot` is clobbered.
template <class V>
__device__ __forceinline__ void dst_fwd(V (&a)[16], V* slot, const V* tw2, const V* tw32, int lane,
                                        typename Cx<V>::R half_c) {
  using R = typename Cx<V>::R;
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 8; ++m) slot[lane + 32 * m] = a[m];
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int n = lane + 32 * m;
    if (m < 8) {
      a[m] = n >= 1 ? slot[n - 1] : Cx<V>::mk(R(0), R(0));
    } else {
      const V t = slot[(511 - n) & 511];
      a[m] = n >= 257 ? Cx<V>::mk(-t.x, -t.y) : Cx<V>::mk(R(0), R(0));
    }
  }
  fft512_fwd(a, slot, tw2, tw32, lane);
  // (S x)[k-1] = c D[k], X = FFT(ext) = -2 i D  ->  w = (c/2) i X
#pragma unroll
  for (int r = 0; r < 16; ++r) a[r] = Cx<V>::mk(-half_c * a[r].y, half_c * a[r].x);
}

// orthonormal DST-I from k-layout odd-symmetric input w (w[0] = w[256] = 0, w[512-k] = -w[k]), inverse-FFT
// form.  out: a[m] = ((S w_a), (S w_b))[lane + 32 m], m < 8 (index 255 -> 0).  `slot` is clobbered.
template <class V>
__device__ __forceinline__ void dst_inv(V (&a)[16], V* slot, const V* tw2, const V* tw32, int lane,
                                        typename Cx<V>::R half_c) {
  using R = typename Cx<V>::R;
  fft512_inv(a, slot, tw2, tw32, lane);
  // I = sum_k w[k] e^{+2 pi i k n / L} = 2 i D(w)[n]  ->  (S w)[n-1] = c D[n] = (c/2)(-i) I[n]
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 8; ++m) slot[lane + 32 * m] = a[m];
  __syncwarp();
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int i = lane + 32 * m;
    const V t = slot[(i + 1) & 511];
    a[m] = i + 1 <= 255 ? Cx<V>::mk(half_c * t.y, -half_c * t.x) : Cx<V>::mk(R(0), R(0));
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
    // release-add: the CTA's writes (ordered before by the CTA barrier) become visible with the arrival
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(sy.gbar) : "memory");
    const unsigned target = sy.epoch * (unsigned)G;
#if RM_POLL_RELAXED
    // relaxed polls, one acquire fence after the last: an acquire load costs an L1 invalidation (CCTL.IVALL) per poll
    for (;;) {
      unsigned v;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sy.gbar) : "memory");
      if (v >= target) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#else
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sy.gbar) : "memory");
      if (v >= target) break;
    }
#endif
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
  // every warp sums the G tile partials with the same butterfly: identical in all CTAs
  double g[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) g[v] = lane < G ? __ldcg(sy.gred + (buf * 4 + v) * G + lane) : 0.0;  // (loads first)
#pragma unroll
  for (int v = 0; v < NV; ++v) out[v] = warp_allsum(g[v]);
  buf ^= 1;
}


// ---- per-CTA context and the kernel's building blocks (all force-inlined: the owner vectors stay in
// registers across them) ------------------------------------------------------------------------------
#ifdef RM_TIMING
// phase timing of CTA 0 (debug builds only): cycles per phase slot, tools/fft_phase_timing.py
#define FT_MARK(c) (c).t_mark = clock64()
#define FT(c, slot)                                                            \
  do {                                                                         \
    const long long t_now_ = clock64();                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) (c).P->timing[slot] += t_now_ - (c).t_mark; \
    (c).t_mark = t_now_;                                                       \
  } while (0)
#else
#define FT_MARK(c)
#define FT(c, slot)
#endif
#if defined(RM_TIMING) && defined(RM_TIMING_FINE)
// sub-phase slots of the two apply passes (replace the coarse slots: -DRM_TIMING,RM_TIMING_FINE)
#undef FT
#define FT(c, slot)
#define FTF(c, slot)                                                           \
  do {                                                                         \
    const long long t_now_ = clock64();                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) (c).P->timing[slot] += t_now_ - (c).t_mark; \
    (c).t_mark = t_now_;                                                       \
  } while (0)
#else
#define FTF(c, slot)
#endif
#if defined(RM_TIMING) && defined(RM_TIMING_SOLVE)
// solve-level slots (replace the others: -DRM_TIMING,RM_TIMING_SOLVE): 0 step prologue (right-hand side, initial
// residual, second guess), 1 first direction, 2 PCG iterations, 3 acceptance (true residual), 4 epilogue
#undef FT
#define FT(c, slot)
#undef FTF
#define FTF(c, slot)
#define ST_MARK(c) (c).s_mark = clock64()
#define ST(c, slot)                                                            \
  do {                                                                         \
    const long long t_now_ = clock64();                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) (c).P->timing[slot] += t_now_ - (c).s_mark; \
    (c).s_mark = t_now_;                                                       \
  } while (0)
#else
#define ST_MARK(c)
#define ST(c, slot)
#endif

struct Ctx {
#ifdef RM_TIMING
  long long t_mark;
  long long s_mark;
#endif
  double* base;        // this chain's vectors
  const ChainArgs* P;
  int rank;
  double di_s;         // s of the cached DI (NaN: none)
  Sync sy;
  int buf;
  // tensor-core preconditioner state (PRE == 2; uniform over the CTA)
  uint32_t tmem;        // tensor-memory base (512 columns: the DST matrix in [0, 256), accumulator from 256)
  unsigned ph_mma;      // phase of the MMA-completion mbarrier
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ int lane() const { return threadIdx.x & 31; }
  __device__ __forceinline__ int warp() const { return threadIdx.x >> 5; }
  __device__ __forceinline__ int R0() const { return RS * rank; }
  __device__ __forceinline__ int C0() const { return RS * rank; }
  __device__ __forceinline__ double* PV() const { return base; }            // operand (read across CTAs)
  __device__ __forceinline__ double* WV() const { return base + VEC; }      // y-pass output
  __device__ __forceinline__ double* SR() const { return base + 2 * VEC; }  // row-DST output
  __device__ __forceinline__ double* XV() const { return base + 3 * VEC; }  // iterate (owner rows)
  __device__ __forceinline__ double* RV() const { return base + 4 * VEC; }  // residual
  __device__ __forceinline__ double* BV() const { return base + 5 * VEC; }  // right-hand side
  __device__ __forceinline__ float* SRf() const { return reinterpret_cast<float*>(SR()); }  // FP32 row-DST output
  __device__ __forceinline__ float* WVf() const { return reinterpret_cast<float*>(WV()); }  // FP32 column-DST output
  // this CTA's 1/d(s) of its column pairs, k-layout [pair][r][lane]
  __device__ __forceinline__ float2* DI() const {
    return reinterpret_cast<float2*>(base + NVEC * VEC + (size_t)rank * DIV);
  }
};

__device__ __forceinline__ double2* smem2() {
  extern __shared__ __align__(128) double2 fft_smem[];
  return fft_smem;
}
__device__ __forceinline__ double2* SLOTS() { return smem2(); }
__device__ __forceinline__ double2* XSLOT(int which) {  // row-pass halo spectra: 0 = pair (R0-1, R0+15), 1 = (R0+16, R0+32)
  return reinterpret_cast<double2*>(reinterpret_cast<unsigned char*>(smem2()) + OFF_XSLOT) + which * SLOT;
}
__device__ __forceinline__ const double2* TW2() { return smem2() + NSLOT * SLOT; }
__device__ __forceinline__ const double2* TW32() { return smem2() + NSLOT * SLOT + L; }
// stiffness spectra (k-layout): per direction d (0 = x, 1 = y) the diagonal block's (real: T1 is symmetric)
// and the off-diagonal block's; the third (transposed block) is its conjugate (rm_fft_symbols checks both)
__device__ __forceinline__ const double* SYMR(int d) {
  return reinterpret_cast<const double*>(smem2() + NSLOT * SLOT + L + 16) + d * L;
}
__device__ __forceinline__ const double2* SYMC(int d) { return smem2() + NSLOT * SLOT + L + 16 + L + d * L; }
__device__ __forceinline__ double* WRED() { return reinterpret_cast<double*>(smem2() + NSLOT * SLOT + L + 16 + 3 * L); }
// FP32 twiddles (tw2f[q * 32 + t] = W512^{q t}, tw32f[r] = W32^r) and the FP32 view of the slots
__device__ __forceinline__ const float2* TW2F() { return reinterpret_cast<const float2*>(WRED() + 4 * 32); }
__device__ __forceinline__ const float2* TW32F() { return TW2F() + L; }
__device__ __forceinline__ float2* SLOTSF() { return reinterpret_cast<float2*>(smem2()); }
constexpr int NX = NP - 1;  // the kernel serves n = 255 grids only (fft_supported)
constexpr double HALF_C = 0.044194173824159220;  // sqrt(2 / 256) / 2
constexpr float HALF_CF = 0.0441941738f;

#define RM_OWN_FOR _Pragma("unroll") for (int p = 0; p < NOWN; ++p) _Pragma("unroll") for (int m = 0; m < 8; ++m)

// owner rows of thread (warp w, lane t): pairs q = w + WARPS (p >> 1), component p & 1 -> row R0 + q + H (p & 1)
__device__ __forceinline__ int own_j(const Ctx& c, int p) { return c.R0() + c.warp() + WARPS * (p >> 1) + H * (p & 1); }
__device__ __forceinline__ int own_i(const Ctx& c, int m) { return c.lane() + 32 * m; }
__device__ __forceinline__ int own_e(const Ctx& c, int p, int m) { return own_j(c, p) * NP + own_i(c, m); }
__device__ __forceinline__ bool own_valid(const Ctx& c, int p, int m) { return own_j(c, p) < NX && own_i(c, m) < NX; }

template <int NV>
__device__ __forceinline__ void creduce(Ctx& c, double (&part)[NV], double (&out)[NV]) {
  greduce<NV>(part, WRED(), c.sy, c.buf, c.rank, c.warp(), c.lane(), out);
}

// M v of the owner rows from PV (7-point P1 mass; per step, not per iteration)
__device__ __forceinline__ void mass_own(const Ctx& c, double (&out)[NOWN][8]) {
#pragma unroll
  for (int p = 0; p < NOWN; ++p) {
#pragma unroll
    for (int m0 = 0; m0 < 8; m0 += 4) {  // (four elements' 28 loads in flight, then the arithmetic)
      double up[4], upr[4], ce[4], r[4], l[4], dn[4], dnl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int m = m0 + u;
        const int j = own_j(c, p), i = own_i(c, m);
        const double* q = c.PV() + j * NP + i;
        const bool ok = own_valid(c, p, m);
        up[u] = ok ? __ldcg(q + NP) : 0.0;
        upr[u] = ok ? __ldcg(q + NP + 1) : 0.0;
        ce[u] = ok ? __ldcg(q) : 0.0;
        r[u] = ok ? __ldcg(q + 1) : 0.0;
        l[u] = (ok && i > 0) ? __ldcg(q - 1) : 0.0;
        dn[u] = (ok && j > 0) ? __ldcg(q - NP) : 0.0;
        dnl[u] = (ok && j > 0 && i > 0) ? __ldcg(q - NP - 1) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        out[p][m0 + u] = own_valid(c, p, m0 + u)
                             ? c.P->cm * (6.0 * ce[u] + l[u] + r[u] + up[u] + upr[u] + dn[u] + dnl[u])
                             : 0.0;
    }
  }
}

// slot geometry and twiddle tables of the two precisions the apply passes run in: FP64 (double2: the operator as the
// algorithm defines it) and FP32 (float2: in-iteration applies once the residual is small, see the PCG loop)
template <class V>
struct Sl;
template <>
struct Sl<double2> {
  static constexpr int STRIDE = SLOT;
  static __device__ __forceinline__ double2* base() { return SLOTS(); }
  static __device__ __forceinline__ double2* xslot(int w) { return XSLOT(w); }
  static __device__ __forceinline__ const double2* tw2() { return TW2(); }
  static __device__ __forceinline__ const double2* tw32() { return TW32(); }
};
// FP32 applies: slots of 545 float2 (spectrum 512, transpose scratch 16 x 34) fill half of the FP64 slot region; FP32
// copies of the stiffness symbols follow them (converted at the start of every FP32 column pass: the FP64 passes and
// the preconditioner's staging overwrite the region in between)
constexpr int SLOT32 = 545;
constexpr size_t OFF_SYMF = ((size_t)NSLOT * SLOT32 * sizeof(float2) + 127) / 128 * 128;
static_assert(OFF_SYMF + 6 * L * sizeof(float) <= (size_t)NSLOT * SLOT * sizeof(double2), "FP32 symbols fit behind the slots");
__device__ __forceinline__ float* SYMF() {
  return reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(smem2()) + OFF_SYMF);
}
template <class V>
struct Sym;
template <>
struct Sym<double2> {
  static __device__ __forceinline__ double re(int d, int e) { return SYMR(d)[e]; }
  static __device__ __forceinline__ double2 cx(int d, int e) { return SYMC(d)[e]; }
};
template <>
struct Sym<float2> {
  static __device__ __forceinline__ float re(int d, int e) { return SYMF()[d * L + e]; }
  static __device__ __forceinline__ float2 cx(int d, int e) {
    return reinterpret_cast<const float2*>(SYMF() + 2 * L)[d * L + e];
  }
};
template <>
struct Sl<float2> {
  static constexpr int STRIDE = SLOT32;
  static __device__ __forceinline__ float2* base() { return SLOTSF(); }
  static __device__ __forceinline__ float2* xslot(int w) { return reinterpret_cast<float2*>(XSLOT(0)) + w * SLOT32; }
  static __device__ __forceinline__ const float2* tw2() { return TW2F(); }
  static __device__ __forceinline__ const float2* tw32() { return TW32F(); }
};

// forward FFT of the warp's own pair (slot warp + 1): the spectrum is stored for the neighbours and stays in
// registers for the combination; LOAD(s, a) fills a[0..8) with the pair of slot s (a[8..16) = 0: zero padding
// known at compile time, so the first radix stage is pruned)
template <class V, class LOAD>
__device__ __forceinline__ void own_forward(Ctx& c, V (&a)[16], LOAD load) {
  using R = typename Cx<V>::R;
  const int s = c.warp() + 1;
  load(s, a);
#pragma unroll
  for (int m = 8; m < 16; ++m) a[m] = Cx<V>::mk(R(0), R(0));
  V* sl = Sl<V>::base() + s * Sl<V>::STRIDE;
  fft512_fwd(a, sl, Sl<V>::tw2(), Sl<V>::tw32(), c.lane());
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) sl[r * 32 + c.lane()] = a[r];
}

// the row pass's pair of slot s (rows R0 + s - 1 and R0 + s - 1 + H) from PV
template <class V>
__device__ __forceinline__ void load_row_pair(const Ctx& c, int s, V (&x)[16]) {
  using R = typename Cx<V>::R;
  const int ja = c.R0() + s - 1, jb = c.R0() + s - 1 + H;
  const double* ra = c.PV() + ja * NP + c.lane();
  const double* rb = c.PV() + jb * NP + c.lane();
  const bool va = ja >= 0, vb = jb < NP;
  double da[8], db[8];  // (raw loads first, then the conversion)
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    da[m] = va ? __ldcg(ra + 32 * m) : 0.0;
    db[m] = vb ? __ldcg(rb + 32 * m) : 0.0;
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) x[m] = Cx<V>::mk((R)da[m], (R)db[m]);
}

// The halo round of an apply: the two halo pairs of the column pass (warps 0 and WARPS-1: slots 0 and NSLOT-1,
// staged columns) and, at the same time, the two halo pairs of the ROW pass (warps 1 and WARPS-2: rows R0-1 / R0+32
// with their partners, straight from PV, into the extra slots), so that the row pass needs no halo round of its own.
template <class V>
__device__ __forceinline__ void halo_forward(Ctx& c, V (&a)[16]) {
  using R = typename Cx<V>::R;
  const int w = c.warp();
  if (w < 2 || w >= WARPS - 2) {
    const bool row = (w == 1 || w == WARPS - 2);
    const bool hi = w >= WARPS - 2;
    const int s = hi ? NSLOT - 1 : 0;
    V* sl = row ? Sl<V>::xslot(hi) : Sl<V>::base() + s * Sl<V>::STRIDE;
    if (row) {
      load_row_pair(c, s, a);
    } else {
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = sl[c.lane() + 32 * m];
      __syncwarp();  // (the slot doubles as the transform's transpose scratch)
    }
#pragma unroll
    for (int m = 8; m < 16; ++m) a[m] = Cx<V>::mk(R(0), R(0));
    fft512_fwd(a, sl, Sl<V>::tw2(), Sl<V>::tw32(), c.lane());
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) sl[r * 32 + c.lane()] = a[r];
  }
}

// y-direction pass of the stiffness: WV[:, own columns] = (1/L) sum_t IFFT(S_t FFT(PV columns i + 0/+1/-1)).
// DOT: also returns this thread's share of sum PV .* WV over the own columns (the y-part of p.Ap, summed by
// the column owners so that the group reduction of p.Ap is the barrier that publishes WV)
template <bool DOT, class V>
__device__ __forceinline__ double col_pass_apply(Ctx& c) {
  using R = typename Cx<V>::R;
  constexpr int ST = Sl<V>::STRIDE;
  static_assert(PPW == 1 && (NP * NSLOT) % THREADS == 0 && (NP * H) % THREADS == 0, "pass geometry");
  V* slots = Sl<V>::base();
  if constexpr (sizeof(R) == 4) {  // FP32 copies of the symbols (visible after the staging barrier)
    const double* sym = SYMR(0);
#pragma unroll
    for (int k = 0; k < 6 * L / THREADS; ++k) SYMF()[c.tid() + k * THREADS] = (float)sym[c.tid() + k * THREADS];
  }
  FTF(c, 10);
  {  // stage columns C0-1 .. C0+32: slot s = (column C0+s-1, column C0+s+15), natural row order; the loads of a
     // batch are issued before its first store
    constexpr int NIT = NP * NSLOT / THREADS, NB = RM_STAGE_NB;
    static_assert(NIT % NB == 0, "staging batches");
#pragma unroll 1
    for (int it0 = 0; it0 < NIT; it0 += NB) {
      double va[NB], vb[NB];  // (raw loads first: a conversion between two loads would serialise their round trips)
#pragma unroll
      for (int it = 0; it < NB; ++it) {
        const int idx = c.tid() + (it0 + it) * THREADS;
        const int j = idx / NSLOT, s = idx - j * NSLOT;
        const int ca = c.C0() + s - 1, cb = c.C0() + s + H - 1;
        const double* row = c.PV() + j * NP;
        va[it] = ca >= 0 ? __ldcg(row + ca) : 0.0;
        vb[it] = cb < NP ? __ldcg(row + cb) : 0.0;
      }
#pragma unroll
      for (int it = 0; it < NB; ++it) {
        const int idx = c.tid() + (it0 + it) * THREADS;
        const int j = idx / NSLOT, s = idx - j * NSLOT;
        slots[s * ST + j] = Cx<V>::mk((R)va[it], (R)vb[it]);
      }
    }
  }
  FTF(c, 11);
  __syncthreads();
  FTF(c, 0);
  V a[16];  // own pair q = warp
  halo_forward(c, a);
  own_forward(c, a, [&](int s, V (&x)[16]) {
    const V* sl = slots + s * ST;
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = sl[c.lane() + 32 * m];
    __syncwarp();  // (the slot doubles as the transform's transpose scratch)
  });
  __syncthreads();
  FTF(c, 1);
  {
    const V* s0 = slots + (c.warp() + 1) * ST;  // columns i
    const V* sp = s0 + ST;                      // columns i + 1
    const V* sm = s0 - ST;                      // columns i - 1
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int e = r * 32 + c.lane();
      const R s0v = Sym<V>::re(1, e);
      const V s1v = Sym<V>::cx(1, e);
      V y = cscale(a[r], s0v);
      y = cadd(y, cmul(s1v, sp[e]));
      a[r] = cadd(y, cmulc(sm[e], s1v));
    }
  }
  __syncthreads();
  FTF(c, 2);
  {
    V* sl = slots + (c.warp() + 1) * ST;
    fft512_inv(a, sl, Sl<V>::tw2(), Sl<V>::tw32(), c.lane());
    __syncwarp();
    constexpr R inv_l = R(1.0 / (double)L);
#pragma unroll
    for (int m = 0; m < 8; ++m) sl[c.lane() + 32 * m] = cscale(a[m], inv_l);
  }
  __syncthreads();
  FTF(c, 3);
  // store the 32 own columns, one row per half-warp step
  double dot = 0.0;
  {
    constexpr int NIT = NP * H / THREADS, NB = RM_STORE_NB;
    static_assert(NIT % NB == 0, "store batches");
#pragma unroll 1
    for (int it0 = 0; it0 < NIT; it0 += NB) {
      double2 pv[NB];
      if constexpr (DOT) {
#pragma unroll
        for (int it = 0; it < NB; ++it) {
          const int idx = c.tid() + (it0 + it) * THREADS;
          const int j = idx / H, q = idx % H;
          const double* row = c.PV() + j * NP + c.C0() + q;
          pv[it] = make_double2(__ldcg(row), __ldcg(row + H));
        }
      }
#pragma unroll
      for (int it = 0; it < NB; ++it) {
        const int idx = c.tid() + (it0 + it) * THREADS;
        const int j = idx / H, q = idx % H;
        const V t = slots[(q + 1) * ST + j];
        const double tx = (double)t.x, ty = (double)t.y;
        c.WV()[j * NP + c.C0() + q] = tx;
        c.WV()[j * NP + c.C0() + q + H] = ty;
        if constexpr (DOT) dot = fma(pv[it].x, tx, fma(pv[it].y, ty, dot));
      }
    }
  }
  FTF(c, 4);
  return dot;
}

// x-direction pass for the owner rows with the P1 mass folded in: acc = (1/L) sum_t IFFT((sg S_t + cm M_t) FFT(PV
// rows j + 0/+1/-1)); the mass blocks tridiag(1,6,1), (1 at d = 0,-1), (1 at d = 0,+1) have the spectra
// 6 + 2 cos(theta), 1 + e^{i theta}, 1 + e^{-i theta}, theta = 2 pi k / L (rm_device.cuh build_step_tables)
template <class V>
__device__ __forceinline__ void row_pass_apply(Ctx& c, double (&acc)[NOWN][8], double sg) {
  using R = typename Cx<V>::R;
  constexpr int ST = Sl<V>::STRIDE;
  V* slots = Sl<V>::base();
  V a[16];  // own pair q = warp (the halo pairs' spectra come from the column pass's halo round)
  own_forward(c, a, [&](int s, V (&x)[16]) { load_row_pair(c, s, x); });
  __syncthreads();
  FTF(c, 6);
  {
    const V w0 = Sl<V>::tw2()[32 + (c.lane() >> 1)];   // W512^{q}
    const R sgn = (c.lane() & 1) ? R(-1) : R(1);        // W512^{256 v}
    const R cm = (R)c.P->cm, sgr = (R)sg;
    const V* s0 = slots + (c.warp() + 1) * ST;
    const V* sp = c.warp() == WARPS - 1 ? Sl<V>::xslot(1) : s0 + ST;
    const V* sm = c.warp() == 0 ? Sl<V>::xslot(0) : s0 - ST;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int e = r * 32 + c.lane();
      const V w = cscale(cmul(w0, Sl<V>::tw32()[r]), sgn);  // e^{-i theta_k}
      // c0 real (symmetric T1, tridiag(1,6,1)), c2 = conj(c1) (transposed block)
      const R s0v = Sym<V>::re(0, e);
      const V s1d = Sym<V>::cx(0, e);
      const R c0 = Cx<V>::ffma(sgr, s0v, cm * (R(6) + R(2) * w.x));
      const V c1 = Cx<V>::mk(Cx<V>::ffma(sgr, s1d.x, cm * (R(1) + w.x)), Cx<V>::ffma(sgr, s1d.y, -cm * w.y));
      V y = cscale(a[r], c0);
      y = cadd(y, cmul(c1, sp[e]));
      a[r] = cadd(y, cmulc(sm[e], c1));
    }
  }
  __syncthreads();
  FTF(c, 7);
  constexpr R inv_l = R(1.0 / (double)L);
  fft512_inv(a, slots + (c.warp() + 1) * ST, Sl<V>::tw2(), Sl<V>::tw32(), c.lane());
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    acc[0][m] = (double)(a[m].x * inv_l);
    acc[1][m] = (double)(a[m].y * inv_l);
  }
  FTF(c, 8);
}

// acc = (M + sg K) PV for the owner rows (PV complete and visible; one group barrier inside)
__device__ __forceinline__ void apply_pv(Ctx& c, double (&acc)[NOWN][8], double sg) {
  FT_MARK(c);
  col_pass_apply<false, double2>(c);
  FT(c, 0);
  gsync(c.sy);
  FT(c, 1);
  FTF(c, 5);
  row_pass_apply<double2>(c, acc, sg);
  double wv[NOWN][8];
  RM_OWN_FOR { wv[p][m] = __ldcg(c.WV() + own_e(c, p, m)); }
  RM_OWN_FOR { acc[p][m] = own_valid(c, p, m) ? fma(sg, wv[p][m], acc[p][m]) : 0.0; }
  FT(c, 2);
  FTF(c, 9);
}

// The PCG loop's apply: acc = (M + sg K) PV for the owner rows and the group's p.Ap = PV . acc.  The column
// owners sum the y-part's share of the dot product inside the column pass, so ONE group reduction delivers
// p.Ap and is the barrier that publishes WV to the row owners.
// V = float2: the same apply through FP32 FFTs (operand converted on load, output and dot product in FP64); the PCG loop
// uses it once the residual is small enough for an FP32-accurate A p (see there).
template <int PRE, class V>
__device__ __forceinline__ double apply_pv_dot(Ctx& c, double (&acc)[NOWN][8], double sg) {
  FT_MARK(c);
  const double dcol = col_pass_apply<true, V>(c);
  FT(c, 0);
  FTF(c, 5);
  row_pass_apply<V>(c, acc, sg);
  double part[1] = {sg * dcol};
  {
    double pv[NOWN][8];
    RM_OWN_FOR { pv[p][m] = __ldcg(c.PV() + own_e(c, p, m)); }  // zero outside the grid
    RM_OWN_FOR { part[0] = fma(pv[p][m], acc[p][m], part[0]); }
  }
  FT(c, 2);
  double pap[1];
  creduce<1>(c, part, pap);
  FT(c, 3);
  double wv[NOWN][8];
  RM_OWN_FOR { wv[p][m] = __ldcg(c.WV() + own_e(c, p, m)); }
  RM_OWN_FOR { acc[p][m] = own_valid(c, p, m) ? fma(sg, wv[p][m], acc[p][m]) : 0.0; }
  FTF(c, 9);
  return pap[0];
}

// refresh this CTA's 1/d(s) cache when s changed (once per sweep on uniform levels)
__device__ __forceinline__ void dinv_refresh(Ctx& c, double s) {
  if (s == c.di_s) return;
  c.di_s = s;
#pragma unroll 1
  for (int h = 0; h < PPW; ++h) {
    const int q = c.warp() + WARPS * h;
    const int ca = c.C0() + q, cb = c.C0() + q + H;  // x-frequencies of the column pair
#pragma unroll 4
    for (int r = 0; r < 16; ++r) {
      const int k = klay(c.lane(), r);
      const int kk = k <= 256 ? k : 512 - k;
      float2 w = make_float2(0.f, 0.f);
      if (kk >= 1 && kk <= 255) {
        const int a = kk - 1;
        if (ca < NX) w.x = (float)(1.0 / (__ldg(c.P->dmT + ca * NX + a) + s * __ldg(c.P->dkT + ca * NX + a)));
        if (cb < NX) w.y = (float)(1.0 / (__ldg(c.P->dmT + cb * NX + a) + s * __ldg(c.P->dkT + cb * NX + a)));
      }
      c.DI()[(q * 16 + r) * 32 + c.lane()] = w;
    }
  }
}

// z = P(s)^-1 r = (Sy x Sx) diag(1/d(s)) (Sy x Sx) r for the owner rows, in two halves around ONE group reduction.
// The DST stages run as FP32 FFTs (FP32 intermediates SR / WV, FP32 1/d): P^-1 only steers the iteration --
// every stop is decided on the FP64 true residual -- and FP32 keeps it within ~1e-7 of the FP64 operator.
//
// precond_front: row DSTs of r, group barrier, column DST -> 1/d(s) -> column DST into WV.  The column owners hold
// the full 2-D sine spectrum rhat = S r at that point, so r.z = r^T P^-1 r = sum rhat^2 / d is summed there
// (FP64 accumulation of the FP32 spectrum); the group reduction that publishes WV to the row owners delivers
// red = {sum of part0 over the group (the caller's r.r share), r.z}.
__device__ __forceinline__ void precond_front(Ctx& c, const double (&r)[NOWN][8], double s, double part0,
                                              double (&red)[2]) {
  static_assert(PPW == 1, "one packed pair per warp");
  float2* slots = SLOTSF();
  FT_MARK(c);
  dinv_refresh(c, s);
  {  // SR[own rows] = Sx r (x-frequency along the row), pair q = warp
    float2 a[16];
#pragma unroll
    for (int m = 0; m < 8; ++m) a[m] = make_float2((float)r[0][m], (float)r[1][m]);
    dst_fwd(a, slots + c.warp() * SLOTF, TW2F(), TW32F(), c.lane(), HALF_CF);
    if ((c.lane() & 1) == 0) {
      float* sa = c.SRf() + own_j(c, 0) * NP - 1;
      float* sb = c.SRf() + own_j(c, 1) * NP - 1;
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        const int k = klay(c.lane(), rr);
        if (k >= 1) {
          sa[k] = a[rr].x;
          sb[k] = a[rr].y;
        }
      }
    }
  }
  FT(c, 5);
  gsync(c.sy);
  FT(c, 6);
  double rz = 0.0;
  {  // column pass: WV[:, own columns] = Sy diag(1/d) Sy SR
    constexpr int NIT = NP * H / THREADS;
    {
      float2 v[NIT];
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const int idx = c.tid() + it * THREADS;
        const int j = idx / H, q = idx % H;
        const float* row = c.SRf() + j * NP + c.C0();
        v[it] = make_float2(__ldcg(row + q), __ldcg(row + q + H));
      }
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const int idx = c.tid() + it * THREADS;
        const int j = idx / H, q = idx % H;
        slots[(q + 1) * SLOTF + j] = v[it];
      }
    }
    __syncthreads();
    {
      const int q = c.warp();
      float2* sl = slots + (q + 1) * SLOTF;
      float2 a[16];
#pragma unroll
      for (int m = 0; m < 8; ++m) a[m] = sl[c.lane() + 32 * m];
      dst_fwd(a, sl, TW2F(), TW32F(), c.lane(), HALF_CF);
      const float2* di = c.DI() + q * 16 * 32 + c.lane();
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) {
        const float2 d = __ldcg(di + rr * 32);
        const float2 t = make_float2(a[rr].x * d.x, a[rr].y * d.y);
        rz = fma((double)a[rr].x, (double)t.x, fma((double)a[rr].y, (double)t.y, rz));
        a[rr] = t;
      }
      dst_inv(a, sl, TW2F(), TW32F(), c.lane(), HALF_CF);
      __syncwarp();
#pragma unroll
      for (int m = 0; m < 8; ++m) sl[c.lane() + 32 * m] = a[m];
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int idx = c.tid() + it * THREADS;
      const int j = idx / H, q = idx % H;
      const float2 t = slots[(q + 1) * SLOTF + j];
      c.WVf()[j * NP + c.C0() + q] = t.x;
      c.WVf()[j * NP + c.C0() + q + H] = t.y;
    }
  }
  FT(c, 7);
  // the k-layout spectrum carries every frequency twice (k and its odd mirror L - k, same 1/d)
  double part[2] = {part0, 0.5 * rz};
  creduce<2>(c, part, red);
  FT(c, 8);
}

// precond_back: z[own rows] = Sx WV[own rows] (after precond_front's reduction)
__device__ __forceinline__ void precond_back(Ctx& c, double (&z)[NOWN][8]) {
  float2* slots = SLOTSF();
  FT_MARK(c);
  float2 a[16];
  const float* wa = c.WVf() + own_j(c, 0) * NP;
  const float* wb = c.WVf() + own_j(c, 1) * NP;
#pragma unroll
  for (int rr = 0; rr < 16; ++rr) {
    const int k = klay(c.lane(), rr);
    float2 w = make_float2(0.f, 0.f);
    if (k >= 1 && k <= 255)
      w = make_float2(__ldcg(wa + k - 1), __ldcg(wb + k - 1));
    else if (k >= 257)
      w = make_float2(-__ldcg(wa + 511 - k), -__ldcg(wb + 511 - k));
    a[rr] = w;
  }
  dst_inv(a, slots + c.warp() * SLOTF, TW2F(), TW32F(), c.lane(), HALF_CF);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    z[0][m] = own_valid(c, 0, m) ? (double)a[m].x : 0.0;
    z[1][m] = own_valid(c, 1, m) ? (double)a[m].y : 0.0;
  }
  FT(c, 9);
}

// ---- tensor-core tau preconditioner (PRE == 2) -------------------------------------------------------------
// The four sine-transform stages as tcgen05 GEMMs (rm_tc.cuh): per CTA D[256][32] = S[256][256] X^T, S the FP16
// DST-I matrix RESIDENT IN TENSOR MEMORY for the whole kernel (loaded once per launch), X a 32-row strip converted
// to FP16 in shared memory, FP32 accumulation in tensor memory.  Intermediates cross the group in FP16,
// transposed so that the next stage's strip operand is contiguous along its contraction index: SRh[kx][j]
// (x-frequency major), WVh[j][kx].
// Scaling: r is scaled by a power of two that maps the previous residual norm into [256, 512) -- the orthonormal
// transforms preserve the 2-norm, so no entry exceeds it; conversions saturate instead of overflowing should the
// norm grow more than 128-fold in one step -- and 1/d(s) is normalised by its upper bound 1/(min dm + s min dk).
__device__ __forceinline__ __half* TC_B() {
  return reinterpret_cast<__half*>(reinterpret_cast<unsigned char*>(smem2()) + OFF_TCB);
}
__device__ __forceinline__ uint64_t* TC_BARS() {
  return reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(smem2()) + OFF_TCBAR);
}
__device__ __forceinline__ uint32_t* TC_TMEM_SLOT() { return reinterpret_cast<uint32_t*>(TC_BARS() + 2); }
__device__ __forceinline__ __half* SRh(const Ctx& c) { return reinterpret_cast<__half*>(c.SR()); }
__device__ __forceinline__ __half* WVh(const Ctx& c) { return reinterpret_cast<__half*>(c.WV()); }
__device__ __forceinline__ float* DItc(const Ctx& c) { return reinterpret_cast<float*>(c.DI()); }

__device__ __forceinline__ unsigned short f2h_sat(float x) {
  unsigned short h;
  asm("cvt.rn.satfinite.f16.f32 %0, %1;" : "=h"(h) : "f"(x));
  return h;
}

// the strip operand is written: run the stage's 32 MMAs and wait for the accumulator
__device__ __forceinline__ void tc_stage_mma(Ctx& c) {
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  if ((c.warp() & 3) == 0 && c.lane() == 0) {  // four issuers: M tile x K half each (rm_tc.cuh)
    tc::tc_fence_after();
    tc::issue_dst_mma_ts_part(TC_B(), c.tmem, c.warp() >> 2);
    tc::tc_commit(TC_BARS() + 1);
  }
  tc::mbar_wait(TC_BARS() + 1, c.ph_mma);
  c.ph_mma ^= 1;
  tc::tc_fence_after();
}

// this warp's share of the accumulator: rows (lanes) 128 t + 32 q + lane, strip columns 16 h .. 16 h + 15
__device__ __forceinline__ void tc_read(const Ctx& c, float (&v)[16], int& row, int& col0) {
  const int q = c.warp() & 3, t = (c.warp() >> 2) & 1, h = c.warp() >> 3;
  float w[16];  // the two K halves were accumulated separately
  tc::tmem_ld16(c.tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(tc::TMEM_D_COL + tc::NB * (2 * t) + 16 * h), v);
  tc::tmem_ld16(c.tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(tc::TMEM_D_COL + tc::NB * (2 * t + 1) + 16 * h), w);
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] += w[e];
  row = 128 * t + 32 * q + c.lane();
  col0 = 16 * h;
}

__device__ __forceinline__ void tc_store16h(__half* dst, const float (&v)[16]) {
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = (uint32_t)f2h_sat(v[2 * i]) | ((uint32_t)f2h_sat(v[2 * i + 1]) << 16);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
  d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// strip operand = 32 consecutive rows of a [256][256] FP16 array (each row contiguous along the contraction index)
__device__ __forceinline__ void tc_load_strip(const Ctx& c, const __half* rows) {
  uint4 val[2];
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int ch = c.tid() + it * THREADS;  // 16-byte chunk: row n, contraction indices 8 jc .. 8 jc + 7
    const int n = ch >> 5, jc = ch & 31;
    val[it] = __ldcg(reinterpret_cast<const uint4*>(rows + n * NP + jc * 8));
  }
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int ch = c.tid() + it * THREADS;
    const int n = ch >> 5, jc = ch & 31;
    *reinterpret_cast<uint4*>(TC_B() + tc::b_index(n, jc * 8)) = val[it];
  }
}

// (1 / d(s)) / bound for this CTA's x-frequencies, [y-frequency l][32 x-frequencies], FP32
__device__ __forceinline__ void dinv_refresh_tc(Ctx& c, double s) {
  if (s == c.di_s) return;
  c.di_s = s;
  const double num = c.P->lp_dmin + s * c.P->lp_kmin;
  for (int idx = c.tid(); idx < NP * tc::NB; idx += THREADS) {
    const int kk = idx >> 8, l = idx & 255;
    const int ca = c.C0() + kk;
    float w = 0.f;
    if (l < NX && ca < NX) w = (float)(num / (__ldg(c.P->dmT + ca * NX + l) + s * __ldg(c.P->dkT + ca * NX + l)));
    DItc(c)[l * tc::NB + kk] = w;
  }
  __syncthreads();  // (read back below by other threads of this CTA; global memory, CTA scope)
}

// red = {group sum of part0, r.z}; nrm: a recent 2-norm of r (sets the power-of-two scaling)
__device__ __forceinline__ void precond_front_tc(Ctx& c, const double (&r)[NOWN][8], double s, double nrm, double part0,
                                                 double (&red)[2]) {
  FT_MARK(c);
  dinv_refresh_tc(c, s);
  const double sc1 = (nrm > 0.0 && isfinite(nrm)) ? scalbn(1.0, 8 - ilogb(nrm)) : 1.0;
  {  // stage 1: SRh[kx][own rows] = Sx r
#pragma unroll
    for (int p = 0; p < NOWN; ++p)
#pragma unroll
      for (int m = 0; m < 8; ++m)
        reinterpret_cast<unsigned short*>(TC_B())[tc::b_index(c.warp() + H * p, c.lane() + 32 * m)] =
            f2h_sat((float)(r[p][m] * sc1));
    tc_stage_mma(c);
    float v[16];
    int k, j0;
    tc_read(c, v, k, j0);
    tc_store16h(SRh(c) + k * NP + c.R0() + j0, v);
  }
  FT(c, 5);
  gsync(c.sy);
  FT(c, 6);
  double rz = 0.0;
  {  // stage 2: Sy along the rows of SRh (own x-frequencies), 1/d, stage 3: Sy again, WVh[j][own x-frequencies]
    tc_load_strip(c, SRh(c) + c.C0() * NP);
    tc_stage_mma(c);
    float v[16];
    int l, k0;
    tc_read(c, v, l, k0);
    const float4* di = reinterpret_cast<const float4*>(DItc(c) + l * tc::NB + k0);
    float4 dq[4];
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4) dq[g4] = __ldcg(di + g4);  // (all loads before the first use)
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4) {
      const float4 d = dq[g4];
      const float dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float t = v[4 * g4 + e] * dd[e];
        rz = fma((double)v[4 * g4 + e], (double)t, rz);
        v[4 * g4 + e] = t;
      }
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) reinterpret_cast<unsigned short*>(TC_B())[tc::b_index(k0 + e, l)] = f2h_sat(v[e]);
    tc_stage_mma(c);
    int j;
    tc_read(c, v, j, k0);
    tc_store16h(WVh(c) + j * NP + c.C0() + k0, v);
  }
  FT(c, 7);
  const double bound = 1.0 / (c.P->lp_dmin + s * c.P->lp_kmin);
  double part[2] = {part0, rz * bound / (sc1 * sc1)};
  creduce<2>(c, part, red);
  FT(c, 8);
}

// z[own rows] = Sx WVh[own rows], unscaled
__device__ __forceinline__ void precond_back_tc(Ctx& c, double (&z)[NOWN][8], double s, double nrm) {
  FT_MARK(c);
  const double sc1 = (nrm > 0.0 && isfinite(nrm)) ? scalbn(1.0, 8 - ilogb(nrm)) : 1.0;
  const double unscale = 1.0 / ((c.P->lp_dmin + s * c.P->lp_kmin) * sc1);
  tc_load_strip(c, WVh(c) + c.R0() * NP);
  tc_stage_mma(c);
  float v[16];
  int i, n0;
  tc_read(c, v, i, n0);
  float* zs = reinterpret_cast<float*>(smem2());  // [32 strip rows][256] in the (idle) FFT slots
#pragma unroll
  for (int e = 0; e < 16; ++e) zs[(n0 + e) * NP + i] = v[e];
  __syncthreads();
#pragma unroll
  for (int p = 0; p < NOWN; ++p)
#pragma unroll
    for (int m = 0; m < 8; ++m)
      z[p][m] = own_valid(c, p, m) ? (double)zs[(c.warp() + H * p) * NP + c.lane() + 32 * m] * unscale : 0.0;
  FT(c, 9);
}


__device__ __forceinline__ void put_pv(Ctx& c, const double (&v)[NOWN][8]) {
  RM_OWN_FOR { c.PV()[own_e(c, p, m)] = v[p][m]; }
}

// p = z (PRE) or r into PV (every CTA is past its PV reads: the reduction of r.z is a group barrier); returns r.z
template <int PRE>
__device__ __forceinline__ double start_direction(Ctx& c, double s, double nrm, RM_CNT_T& npc) {
  double r0[NOWN][8], z[NOWN][8];
  RM_OWN_FOR { r0[p][m] = __ldcg(c.RV() + own_e(c, p, m)); }
  double rz;
  if constexpr (PRE == 2) {
    double red[2];
    precond_front_tc(c, r0, s, nrm, 0.0, red);
    ++npc;
    rz = red[1];
    precond_back_tc(c, z, s, nrm);
  } else if constexpr (PRE == 1) {
    double red[2];
    precond_front(c, r0, s, 0.0, red);
    ++npc;
    rz = red[1];
    precond_back(c, z);
  } else {
    double pr[1] = {0.0}, o[1];
    RM_OWN_FOR {
      z[p][m] = r0[p][m];
      pr[0] += r0[p][m] * r0[p][m];
    }
    creduce<1>(c, pr, o);
    rz = o[0];
  }
  put_pv(c, z);
  gsync(c.sy);
  return rz;
}

}  // namespace fft

template <int PRE>  // 0: plain CG, 1: tau preconditioner by FP32 FFTs, 2: tau preconditioner on the tensor cores
__global__ void __launch_bounds__(fft::THREADS, 1) chain_fft_kernel(const __grid_constant__ ChainArgs P) {
  using namespace fft;
  Ctx c;
  c.P = &P;
  c.rank = blockIdx.x % G;
  const int cid = blockIdx.x / G;
  const int tid = threadIdx.x;
  c.sy.gbar = P.gbar + (size_t)cid * 32;
  c.sy.gred = P.gbuf + (size_t)cid * 1024;
  c.sy.sched = reinterpret_cast<int*>(c.sy.gred + 8 * G);
  c.sy.epoch = 0;
  c.buf = 0;
  c.tmem = 0;
  c.ph_mma = 0;
  if constexpr (PRE == 2) {
    if (tid == 0) {
      tc::mbar_init(TC_BARS() + 1, 4);  // four MMA issuers commit to it
      tc::fence_mbar_init();
    }
    if (tid < 32) tc::tmem_alloc(TC_TMEM_SLOT(), tc::TMEM_COLS_RESIDENT);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    c.tmem = *TC_TMEM_SLOT();
    // the DST matrix moves into tensor memory once per launch and stays there
    tc::load_matrix_tmem(c.tmem, reinterpret_cast<const __half*>(P.dstc), tid >> 5, tid & 31);
    tc::tc_fence_before();
    __syncthreads();
  }
  {
    double2* tw2 = const_cast<double2*>(TW2());    // tw2[q * 32 + t] = W512^{q t}
    double2* tw32 = const_cast<double2*>(TW32());  // W32^r = W512^{16 r}
    double* sym = const_cast<double*>(SYMR(0));    // stiffness spectra (2 x 512 real, 2 x 512 complex)
    for (int i = tid; i < L; i += THREADS) {
      const int q = i >> 5, t = i & 31;
      double sn, cs;
      sincospi(-2.0 * (double)(q * t) / (double)L, &sn, &cs);
      tw2[i] = make_double2(cs, sn);
      const_cast<float2*>(TW2F())[i] = make_float2((float)cs, (float)sn);
    }
    if (tid < 16) {
      double sn, cs;
      sincospi(-2.0 * (double)(16 * tid) / (double)L, &sn, &cs);
      tw32[tid] = make_double2(cs, sn);
      const_cast<float2*>(TW32F())[tid] = make_float2((float)cs, (float)sn);
    }
    for (int i = tid; i < 6 * L; i += THREADS) sym[i] = P.fsym[i];  // 6 L doubles
  }
  const rm_sweep& W_ = P.sw;
  constexpr int nx = NX;
  c.di_s = __longlong_as_double(0x7ff8000000000000ll);  // NaN: nothing cached
  const RM_CNT_T max_iter =
      (RM_CNT_T)(W_.max_iter > 0 ? (W_.max_iter < 2000000000 ? W_.max_iter : 2000000000) : 10 * (int64_t)NX * NX);
  const bool need_in = W_.explicit_rhs || W_.x0_mode == 1;
  const bool lowp_ok = W_.lp_matvec != 0 && P.lp_thr > 0.0;
  // G row scale (compressed G, rm_sweep.d_gscale): rows of d_gadd / d_hg are d_gscale[n] times the stored row
  auto gsc = [&](int k) -> double { return W_.d_gscale ? W_.d_gscale[k] : 1.0; };
  c.base = P.fscratch + (size_t)cid * (NVEC * VEC + G * DIV);
  // zero this chain slot's vectors once (padding row / column 255 is never written afterwards)
  for (size_t i = (size_t)c.rank * THREADS + tid; i < NVEC * VEC; i += (size_t)G * THREADS) c.base[i] = 0.0;
  gsync(c.sy);

  for (;;) {
    if (c.rank == 0 && tid == 0) c.sy.sched[0] = atomicAdd(P.chain_counter, 1);
    gsync(c.sy);
    const int chain = __ldcg(c.sy.sched);
    gsync(c.sy);
    if (chain >= W_.nchains) break;
    const int n0 = W_.first + chain * W_.cstride;
    const int n1 = min(n0 + W_.clen - 1, W_.nmax);
    bool in_tile = false;
    bool chain_ok = false;
    double s_prev = 0.0;
    for (int n = n0; n <= n1; ++n) {
      ST_MARK(c);
      const double s = 0.5 * W_.d_dt[n - 1];
      const double fs = W_.d_f ? (W_.d_fscale ? W_.d_fscale[n] : 1.0) : 0.0;
      const double* Fn = W_.d_f ? W_.d_f + (int64_t)n * W_.f_stride : nullptr;
      const bool rhs_free = need_in && W_.explicit_rhs && in_tile && chain_ok && W_.d_hg != nullptr &&
                            W_.d_gadd != nullptr && W_.d_sub == nullptr;
      const bool rhs_ain = need_in && W_.explicit_rhs && !in_tile && n >= 2 && W_.d_ain != nullptr &&
                           W_.d_hg != nullptr && !rhs_free;
      RM_CNT_T nmv = 0, npc = 0, nmv32 = 0;
      double acc[NOWN][8];
      RM_OWN_FOR { acc[p][m] = 0.0; }
      if (need_in && !in_tile) {
        const double* src = W_.d_src + (int64_t)(n - 1) * W_.src_stride;
        double v[NOWN][8];
        RM_OWN_FOR { v[p][m] = own_valid(c, p, m) ? __ldcg(src + own_j(c, p) * nx + own_i(c, m)) : 0.0; }
        put_pv(c, v);
        gsync(c.sy);
      }
      ST(c, 5);
      double mv[NOWN][8];  // M v of the step input (explicit sides without an apply, x0 = v)
      if (rhs_free || rhs_ain) mass_own(c, mv);
      ST(c, 6);
      if (rhs_free) {
        const double* Hn = W_.d_hg + (int64_t)(n - 1) * W_.hg_stride;
        const double q = s / s_prev;
        double bv[NOWN][8], rv[NOWN][8], hv[NOWN][8];
        RM_OWN_FOR {
          const int e = own_e(c, p, m);
          const bool ok = own_valid(c, p, m);
          bv[p][m] = __ldcg(c.BV() + e);
          rv[p][m] = __ldcg(c.RV() + e);
          hv[p][m] = ok ? __ldcg(Hn + own_j(c, p) * nx + own_i(c, m)) : 0.0;  // (raw: arithmetic after the loads)
        }
        const double gs1 = gsc(n - 1);
        RM_OWN_FOR {
          acc[p][m] =
              own_valid(c, p, m) ? (1.0 + q) * mv[p][m] - q * (bv[p][m] - rv[p][m] + gs1 * hv[p][m]) : 0.0;
        }
      } else if (rhs_ain) {
        const double* An = W_.d_ain + (int64_t)(n - 1) * W_.ain_stride;
        const double* Hn = W_.d_hg + (int64_t)(n - 1) * W_.hg_stride;
        const double q = s / (0.5 * W_.d_dt[n - 2]);
        double av[NOWN][8], hv[NOWN][8];
        RM_OWN_FOR {
          const int gi = own_j(c, p) * nx + own_i(c, m);
          const bool ok = own_valid(c, p, m);
          av[p][m] = ok ? __ldcg(An + gi) : 0.0;
          hv[p][m] = ok ? __ldcg(Hn + gi) : 0.0;
        }
        const double gs1 = gsc(n - 1);
        RM_OWN_FOR {
          acc[p][m] = own_valid(c, p, m) ? (1.0 + q) * mv[p][m] - q * (av[p][m] + gs1 * hv[p][m]) : 0.0;
        }
      } else if (need_in) {
        apply_pv(c, acc, -s);  // (M - s K) v
        nmv = 1;
        if (W_.x0_mode == 1) mass_own(c, mv);
      } else if (W_.x0_mode == 1) {
        mass_own(c, mv);
      }
      s_prev = s;
      chain_ok = false;

      // right-hand side, initial iterate and residual
      double part[2] = {0.0, 0.0};
      {
        double fv[NOWN][8], xv[NOWN][8];
        RM_OWN_FOR {
          const bool ok = own_valid(c, p, m);
          fv[p][m] = (Fn && ok) ? __ldcg(Fn + own_j(c, p) * nx + own_i(c, m)) : 0.0;
          xv[p][m] = (W_.x0_mode == 1 && ok) ? __ldcg(c.PV() + own_e(c, p, m)) : 0.0;
        }
        RM_OWN_FOR {
          const int e = own_e(c, p, m);
          double b = 0.0, r = 0.0;
          if (own_valid(c, p, m)) {
            const double am = acc[p][m];
            if (W_.explicit_rhs) b = am;
            if (Fn) b = W_.explicit_rhs ? fs * fv[p][m] + b : fs * fv[p][m];
            // x0 = v: (M + s K) v = 2 M v - (M - s K) v
            r = W_.x0_mode == 1 ? b - (2.0 * mv[p][m] - am) : b;
          }
          c.BV()[e] = b;
          c.XV()[e] = xv[p][m];
          c.RV()[e] = r;
          part[0] += b * b;
          part[1] += r * r;
        }
      }
      if (W_.x0_mode == 2 || W_.x0_mode == 4) {
        // given initial iterate (x0_mode 2, stepper.py:203) / apply probe (x0_mode 4: out = (M + s K) b)
        gsync(c.sy);  // every CTA done reading PV
        const double* x0 = W_.x0_mode == 2 ? W_.d_x0 + (int64_t)n * W_.x0_stride : Fn;
        const double sc = W_.x0_mode == 2 ? 1.0 : fs;
        double v[NOWN][8];
        RM_OWN_FOR { v[p][m] = own_valid(c, p, m) ? __ldcg(x0 + own_j(c, p) * nx + own_i(c, m)) : 0.0; }
        RM_OWN_FOR { v[p][m] = sc * v[p][m]; }
        put_pv(c, v);
        gsync(c.sy);
        apply_pv(c, acc, s);
        ++nmv;
        part[1] = 0.0;
        double bq[NOWN][8];
        RM_OWN_FOR { bq[p][m] = W_.x0_mode == 4 ? 0.0 : __ldcg(c.BV() + own_e(c, p, m)); }
        RM_OWN_FOR {
          const int e = own_e(c, p, m);
          if (W_.x0_mode == 4) {
            c.XV()[e] = acc[p][m];
          } else {
            const double r = own_valid(c, p, m) ? bq[p][m] - acc[p][m] : 0.0;
            c.XV()[e] = v[p][m];
            c.RV()[e] = r;
            part[1] += r * r;
          }
        }
      }
      ST(c, 7);
      double tot[2];
      creduce<2>(c, part, tot);
      ST(c, 8);
      const double bnorm = sqrt(tot[0]);
      const double target = bnorm > 0.0 ? W_.rel_tol * bnorm : W_.rel_tol;
      if (W_.d_guess && W_.x0_mode < 3 && sqrt(tot[1]) > target) {
        const double* gu = W_.d_guess + (int64_t)n * W_.guess_stride;
        const double* Gr = W_.d_gadd ? W_.d_gadd + (int64_t)n * W_.gadd_stride : nullptr;
        const double* Ax0 = W_.d_gax ? W_.d_gax + (int64_t)n * W_.gax_stride : nullptr;
        auto guess_vec = [&](double (&g0)[NOWN][8]) {  // (all loads first, then the arithmetic)
          double gr[NOWN][8];
          RM_OWN_FOR {
            const bool ok = own_valid(c, p, m);
            const int gi = own_j(c, p) * nx + own_i(c, m);
            g0[p][m] = ok ? __ldcg(gu + gi) : 0.0;
            gr[p][m] = (ok && Gr) ? __ldcg(Gr + gi) : 0.0;
          }
          if (Gr) {
            const double gs0 = gsc(n);
            RM_OWN_FOR { g0[p][m] = g0[p][m] - gs0 * gr[p][m]; }
          }
        };
        double ag[NOWN][8];
        if (!Ax0) {
          double g0[NOWN][8];
          guess_vec(g0);
          gsync(c.sy);  // every CTA done reading PV
          put_pv(c, g0);
          gsync(c.sy);
          apply_pv(c, ag, s);
          ++nmv;
        } else {
          RM_OWN_FOR { ag[p][m] = own_valid(c, p, m) ? __ldcg(Ax0 + own_j(c, p) * nx + own_i(c, m)) : 0.0; }
        }
        double pg[1] = {0.0};
        {
          double bq[NOWN][8];
          RM_OWN_FOR { bq[p][m] = __ldcg(c.BV() + own_e(c, p, m)); }
          RM_OWN_FOR {
            const double r = own_valid(c, p, m) ? bq[p][m] - ag[p][m] : 0.0;
            ag[p][m] = r;
            pg[0] += r * r;
          }
        }
        double rg[1];
        creduce<1>(c, pg, rg);
        if (rg[0] < tot[1]) {
          tot[1] = rg[0];
          double g0[NOWN][8];
          if (Ax0)
            guess_vec(g0);
          else
            RM_OWN_FOR { g0[p][m] = __ldcg(c.PV() + own_e(c, p, m)); }
          RM_OWN_FOR {
            const int e = own_e(c, p, m);
            c.XV()[e] = g0[p][m];
            c.RV()[e] = ag[p][m];
          }
        }
      }
      double res = sqrt(tot[1]);
      double rz = tot[1];
      RM_CNT_T its = 0;
      int fail = 0;
      bool done = res <= target || W_.x0_mode == 4;
      if (W_.x0_mode == 3) {
        // preconditioner probe: x = P^-1 b
        if constexpr (PRE) {
          double r0[NOWN][8], z[NOWN][8], red[2];
          RM_OWN_FOR { r0[p][m] = __ldcg(c.RV() + own_e(c, p, m)); }
          if constexpr (PRE == 2) {
            precond_front_tc(c, r0, s, res, 0.0, red);
            precond_back_tc(c, z, s, res);
          } else {
            precond_front(c, r0, s, 0.0, red);
            precond_back(c, z);
          }
          ++npc;
          RM_OWN_FOR { c.XV()[own_e(c, p, m)] = z[p][m]; }
        }
        done = true;
      }
      ST(c, 0);
      if (!done) rz = start_direction<PRE>(c, s, res, npc);
      ST(c, 1);

      // PCG (krylov.py:57-86 with the tau preconditioner); x += alpha p is folded into the next direction
      // update (or the acceptance check), which reads p anyway
      double alpha = 0.0;
      for (RM_CNT_T k = 1; !done; ++k) {
        if (k > max_iter) {
          fail = RM_CG_BUDGET;
          its = max_iter;
          break;
        }
        double ap[NOWN][8];
        // one group reduction: p.Ap, and WV published.  Once the residual has dropped to lp_thr |b| the apply runs
        // through FP32 FFTs (rm_sweep.lp_matvec, precond 2): an apply error eps |A| |p_k| enters the residual gap
        // scaled by the step length, i.e. by |r_k|, so FP32 (eps ~ 3e-7) keeps the gap below the 1e-12 |b| target
        // from |r_k| <= ~1e-6 |b| on (inexact-Krylov relaxation); acceptance stays on the FP64 true residual, with
        // the restart on drift as the safety net.
        double pap;
        if (PRE == 2 && lowp_ok && res <= P.lp_thr * bnorm) {
          pap = apply_pv_dot<PRE, float2>(c, ap, s);
          ++nmv32;
        } else {
          pap = apply_pv_dot<PRE, double2>(c, ap, s);
          ++nmv;
        }
        if (!isfinite(pap) || pap <= 0.0) {
          fail = RM_CG_BREAKDOWN;
          its = k;
          break;
        }
        alpha = rz / pap;
        const double res_prev = res;
        double red2[2];
        {
          double rn[NOWN][8];
          double rr = 0.0;
          {
            double rv[NOWN][8];
            RM_OWN_FOR { rv[p][m] = __ldcg(c.RV() + own_e(c, p, m)); }
            RM_OWN_FOR {
              rn[p][m] = rv[p][m] - alpha * ap[p][m];
              c.RV()[own_e(c, p, m)] = rn[p][m];
              rr += rn[p][m] * rn[p][m];
            }
          }
          if constexpr (PRE == 2) {
            precond_front_tc(c, rn, s, res_prev, rr, red2);  // (res: the previous residual norm sets the FP16 scaling)
            ++npc;
          } else if constexpr (PRE == 1) {
            precond_front(c, rn, s, rr, red2);  // one group reduction: r.r and r.z, and the column DSTs published
            ++npc;
          } else {
            double part1[1] = {rr}, o1[1];
            FT_MARK(c);
            creduce<1>(c, part1, o1);
            FT(c, 10);
            red2[0] = red2[1] = o1[0];
          }
        }
        res = sqrt(red2[0]);
        if (!isfinite(res)) {
          fail = RM_CG_NONFINITE;
          its = k;
          break;
        }
        if (res <= target) {
          ST(c, 2);
          // x += alpha p, then acceptance on the true residual (krylov.py:71-83); every CTA is past its PV
          // reads (the reductions above were group barriers)
          double xv[NOWN][8];
          {
            double xo[NOWN][8], pv[NOWN][8];
            RM_OWN_FOR {
              xo[p][m] = __ldcg(c.XV() + own_e(c, p, m));
              pv[p][m] = __ldcg(c.PV() + own_e(c, p, m));
            }
            RM_OWN_FOR {
              xv[p][m] = xo[p][m] + alpha * pv[p][m];
              c.XV()[own_e(c, p, m)] = xv[p][m];
            }
          }
          put_pv(c, xv);
          gsync(c.sy);
          double ax[NOWN][8];
          apply_pv(c, ax, s);
          ++nmv;
          double pt[1] = {0.0};
          {
            double bv[NOWN][8];
            RM_OWN_FOR { bv[p][m] = __ldcg(c.BV() + own_e(c, p, m)); }
            RM_OWN_FOR {
              const double rt = own_valid(c, p, m) ? bv[p][m] - ax[p][m] : 0.0;
              ax[p][m] = rt;
              pt[0] += rt * rt;
            }
          }
          double tt[1];
          creduce<1>(c, pt, tt);
          const double true_res = sqrt(tt[0]);
          RM_OWN_FOR { c.RV()[own_e(c, p, m)] = ax[p][m]; }
          ST(c, 3);
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
          rz = start_direction<PRE>(c, s, res, npc);
          continue;
        }
        const double beta = red2[1] / rz;
        rz = red2[1];
        double z[NOWN][8];
        if constexpr (PRE == 2) {
          precond_back_tc(c, z, s, res_prev);
        } else if constexpr (PRE == 1) {
          precond_back(c, z);
        } else {
          RM_OWN_FOR { z[p][m] = __ldcg(c.RV() + own_e(c, p, m)); }
        }
        FT_MARK(c);
        // x += alpha p, p = z + beta p (every CTA finished reading PV: the reductions were group barriers)
        {
          double xo[NOWN][8], pv[NOWN][8];
          RM_OWN_FOR {
            xo[p][m] = __ldcg(c.XV() + own_e(c, p, m));
            pv[p][m] = __ldcg(c.PV() + own_e(c, p, m));
          }
          RM_OWN_FOR {
            const int e = own_e(c, p, m);
            c.XV()[e] = xo[p][m] + alpha * pv[p][m];
            c.PV()[e] = z[p][m] + beta * pv[p][m];
          }
        }
        gsync(c.sy);
        FT(c, 11);
      }

      ST(c, 2);
      chain_ok = done && !fail && W_.x0_mode < 3;
      if (c.rank == 0 && tid == 0) {
        atomicAdd(W_.d_counters, 1ull);
        atomicAdd(W_.d_counters + 1, (unsigned long long)its);
        atomicAdd(W_.d_counters + 2, (unsigned long long)nmv);
        atomicAdd(W_.d_counters + 3, (unsigned long long)npc);
        atomicAdd(W_.d_counters + 4, (unsigned long long)nmv32);
      }
      if (fail) {
        if (c.rank == 0 && tid == 0 && atomicCAS(P.fail, 0, fail) == 0) {
          P.fail_info[0] = (double)n;
          P.fail_info[1] = (double)its;
          P.fail_info[2] = res;
        }
        gsync(c.sy);
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
      gsync(c.sy);  // every CTA done reading PV before it is overwritten with y
      double py[1] = {0.0};
      {
        double xv[NOWN][8], gv[NOWN][8], sv[NOWN][8], bv[NOWN][8], rv[NOWN][8];
        const double gsn = Gn ? gsc(n) : 0.0;
        RM_OWN_FOR {
          const bool ok = own_valid(c, p, m);
          const int e = own_e(c, p, m), gi = own_j(c, p) * nx + own_i(c, m);
          xv[p][m] = __ldcg(c.XV() + e);
          gv[p][m] = (Gn && ok) ? __ldcg(Gn + gi) : 0.0;  // (scaled below: arithmetic after the loads)
          sv[p][m] = (Sn && ok) ? __ldcg(Sn + gi) : 0.0;
          bv[p][m] = An ? __ldcg(c.BV() + e) : 0.0;
          rv[p][m] = An ? __ldcg(c.RV() + e) : 0.0;
        }
        RM_OWN_FOR {
          if (own_valid(c, p, m)) {
            const int gi = own_j(c, p) * nx + own_i(c, m);
            double y = xv[p][m];
            if (An) An[gi] = bv[p][m] - rv[p][m];  // A x = b - r (true residual)
            if (Gn) y = gsn * gv[p][m] + y;
            if (Kn) Kn[gi] = y;
            if (Sn) y = y - sv[p][m];
            if (On) On[gi] = y;
            if (next_in_tile) c.PV()[own_e(c, p, m)] = y;
            py[0] += y * y;
          }
        }
      }
      if (W_.d_norms) {
        double yy[1];
        creduce<1>(c, py, yy);
        if (c.rank == 0 && tid == 0) W_.d_norms[oi] = yy[0];
      }
      in_tile = next_in_tile;
      gsync(c.sy);
      ST(c, 4);
    }
  }
  if constexpr (PRE == 2) {
    tc::tc_fence_before();
    __syncthreads();
    if (tid < 32) tc::tmem_free(c.tmem, tc::TMEM_COLS_RESIDENT);
  }
}

#undef RM_OWN_FOR

// Host: spectra of the stiffness tables (entry d + np of table t, |d| < n used) in k-layout order
// (k = (lane >> 1) + 16 (r + 16 (lane & 1)), element e = r 32 + lane): out[0 .. 2L) = the real spectra of tables 0
// (x) and 3 (y), out[2L .. 6L) = the complex spectra of tables 1 and 4.  Returns false unless tables 0 / 3 are
// symmetric (real spectra) and tables 2 / 5 are the reversals of 1 / 4 (conjugate spectra), which the kernel
// relies on (the Riesz generators, reference assembly.py:190-251, have both properties).
bool fft_symbols(const double* tab, int np, int gl, double* out) {
  const int L = fft::L, n = np - 1;
  std::vector<double> cs(L), sn(L);
  for (int i = 0; i < L; ++i) {
    cs[i] = cos(2.0 * M_PI * i / L);
    sn[i] = sin(2.0 * M_PI * i / L);
  }
  for (int d = 1; d < n; ++d)
    for (int t = 0; t < 6; t += 3) {
      if (tab[t * gl + np + d] != tab[t * gl + np - d]) return false;
      if (tab[(t + 2) * gl + np + d] != tab[(t + 1) * gl + np - d] ||
          tab[(t + 2) * gl + np - d] != tab[(t + 1) * gl + np + d])
        return false;
    }
  for (int dir = 0; dir < 2; ++dir)
    for (int which = 0; which < 2; ++which) {
      const int t = 3 * dir + which;
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
          const int e = r * 32 + lane;
          if (which == 0) {
            out[dir * L + e] = re;
          } else {
            out[2 * L + 2 * (dir * L + e)] = re;
            out[2 * L + 2 * (dir * L + e) + 1] = im;
          }
        }
    }
  return true;
}

bool fft_supported(int np, int nx, int ny) { return np == fft::NP && nx == fft::NP - 1 && ny == fft::NP - 1; }

int fft_group() { return fft::G; }

size_t fft_scratch_doubles_per_chain() { return fft::NVEC * fft::VEC + fft::G * fft::DIV; }

static cudaError_t fft_prepare(const void* kern) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft::SMEM);
}

cudaError_t fft_max_chains(int* out) {
  auto kern = chain_fft_kernel<1>;
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
  if (a.sw.precond == 2 && !a.dstc) return cudaErrorInvalidValue;
  auto kern = a.sw.precond == 2 ? chain_fft_kernel<2> : a.sw.precond ? chain_fft_kernel<1> : chain_fft_kernel<0>;
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
