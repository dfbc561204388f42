// B200 kernels of the MGRIT fine-propagator hot path (sm_100a).
//
//  chain_kernel : persistent kernel; each cluster of G CTAs pulls propagation
//                 chains from a work counter and runs, per time step, the
//                 explicit apply, the reference-exact CG solve and the MGRIT
//                 epilogue (add G_n / subtract U_n / squared norm) without
//                 leaving the SM: the iterate, residual and rhs live in a
//                 fragment-native scratch (L2 resident), the search direction
//                 lives in shared memory (broadcast to the cluster over DSMEM).
//  apply_kernel : batched operator apply (CombinedStepOperator.apply / BttbOperator.apply).
//  pcg64_kernel : numpy-bit-exact PCG64 uniform doubles (initial guess).
//  correct_kernel, diff_sqnorm_kernel : small MGRIT helpers.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "riesz_mgrit_b200.h"
#include "rm_device.cuh"
#include "rm_kernels.h"

namespace rm {

#ifdef RM_TIMING
// phase timing of CTA 0 (debug builds only: python -m paper_1805_06688_b200.build --timing)
#define RM_T0() long long t_mark_ = clock64();
#define RM_TM() t_mark_ = clock64()
#define RM_T(slot)                                                     \
  do {                                                                 \
    long long t_now_ = clock64();                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0) P.timing[slot] += t_now_ - t_mark_; \
    t_mark_ = t_now_;                                                  \
  } while (0)
#else
#define RM_T0()
#define RM_TM()
#define RM_T(slot)
#endif

// ----------------------------------------------------------------------------
// chain kernel
// ----------------------------------------------------------------------------

template <class C>
struct Ctx {
  int tid, lane, warp, gq, tig, rank;
  int urow, ucol;  // first unit (row, col) of this warp
  int tm, tn;      // transposed DST stage: unit column (m) and first unit row (n) of this warp
  int tm_fold;           // transposed-stage m unit when the x-direction DST is folded
};

#define RM_FOR_ELEM                                \
  _Pragma("unroll") for (int mr = 0; mr < C::WR; ++mr) \
  _Pragma("unroll") for (int nf = 0; nf < C::NF; ++nf) \
  _Pragma("unroll") for (int e = 0; e < 4; ++e)

template <class C>
__device__ __forceinline__ int elem_row(const Ctx<C>& c, int mr, int e) {
  return prow<C>(c.urow + mr, c.gq + 8 * (e >> 1));
}
template <class C>
__device__ __forceinline__ int elem_col(const Ctx<C>& c, int nf, int e) {
  return 16 * c.ucol + 8 * nf + 2 * c.tig + (e & 1);
}
template <class C>
__device__ __forceinline__ int elem_sidx(const Ctx<C>& c, int mr, int nf, int e) {
  return (((c.urow + mr) * C::UR + c.ucol + (nf >> 1)) * 256) + (((nf & 1) * 4 + e) * 32) + c.lane;
}

// Vt <- a (- b): flattened element order, UN independent loads per array in flight per thread
// (the rows come from HBM or L2; a per-row loop would expose one latency per row)
template <class C, bool SUB>
__device__ __forceinline__ void load_rows(double* Vt, const double* __restrict__ a, const double* __restrict__ b,
                                          int nx, int ny, const Ctx<C>& c, double bs = 1.0) {
  constexpr int UN = SUB ? 4 : 8;
  const int ndof = nx * ny;
  for (int base = c.tid; base < ndof; base += C::THREADS * UN) {
    double va[UN], vb[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int e = base + u * C::THREADS;
      va[u] = e < ndof ? __ldcg(a + e) : 0.0;
      if constexpr (SUB) vb[u] = e < ndof ? __ldcg(b + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int e = base + u * C::THREADS;
      if (e < ndof) {
        const int j = e / nx, i = e - j * nx;
        Vt[vt_idx<C>(j, i)] = SUB ? va[u] - bs * vb[u] : va[u];
      }
    }
  }
}

template <class C>
__device__ __forceinline__ void load_vec(double* Vt, const double* __restrict__ src, int nx, int ny,
                                         const Ctx<C>& c) {
  load_rows<C, false>(Vt, src, nullptr, nx, ny, c);
}

// Vt <- guess - G (G may be null)
template <class C>
__device__ __forceinline__ void load_guess(double* Vt, const double* __restrict__ guess, const double* __restrict__ G,
                                           int nx, int ny, const Ctx<C>& c, double gs) {
  if (G)
    load_rows<C, true>(Vt, guess, G, nx, ny, c, gs);
  else
    load_rows<C, false>(Vt, guess, nullptr, nx, ny, c);
}

// Hint: pull [p, p+bytes) into L2 (TMA bulk prefetch; whole 16-byte granules inside the range only)
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  uintptr_t a = ((uintptr_t)p + 15) & ~(uintptr_t)15;
  const uintptr_t e = ((uintptr_t)p + bytes) & ~(uintptr_t)15;
  while (a < e) {
    const uint32_t sz = (uint32_t)min((uintptr_t)32768, e - a);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(sz) : "memory");
    a += sz;
  }
}

template <class C>
__device__ __forceinline__ void zero_part(double (&p)[C::WR][C::WC]) {
#pragma unroll
  for (int mr = 0; mr < C::WR; ++mr)
#pragma unroll
    for (int uc = 0; uc < C::WC; ++uc) p[mr][uc] = 0.0;
}

template <class C>
__device__ __forceinline__ int elem_xidx(const Ctx<C>& c, int mr, int nf, int e) {
  // x lives in shared memory in fragment-native order (lane-contiguous: conflict free)
  return (((c.warp * C::WR + mr) * C::WC + (nf >> 1)) * 8 + (nf & 1) * 4 + e) * 32 + c.lane;
}

// element (row j, col i) held by (nf, e) of the transposed DST-x stage
template <class C>
__device__ __forceinline__ int elemT_row(const Ctx<C>& c, int nf, int e) {
  return trow<C>(c.tn + (nf >> 1), 8 * (nf & 1) + 2 * c.tig + (e & 1));
}


// Shared state of one chain kernel instance (per CTA).
template <class C>
struct Smem {
  double* Vt;
  double* gens;
  double* red;
  double* xs;
  double* tabx;
  double* taby;
  double* red_peer[C::G];
  double* mx;
  double* mx_peer[C::G];
};

// z = P^{-1} r for the tau preconditioner: T1 = R Sx; T2 = Sy T1 * dinv; T3 = T2 Sx; z = Sy T3.
// The x-direction stages read only this CTA's own rows (transposed mapping), so their inputs are
// written locally without any exchange; only the y-stage inputs (T1, T3) are broadcast.  The DST
// folds are applied on the fly (rm_device.cuh), so the tile is never modified in place: the only
// cluster barrier inside is the one between the passes (every peer has received this CTA's band and
// finished its y-stage before the own rows are overwritten and new bands are pushed).
// Precondition: every CTA finished reading its operand tile and nobody reads this CTA's own rows any
// more.  Result z in acc (normal mapping).
template <class C>
__device__ __forceinline__ void apply_tau(const Ctx<C>& c, const Smem<C>& sm, Bcast<C>& bc,
                                          const double (&r)[C::WR][C::NF][4], double (&acc)[C::WR][C::NF][4],
                                          const double* __restrict__ dinv, int nx, int ny, int Lx, int Ly,
                                          long long* timing) {
  const int kx_end = (nx + 3) & ~3, ky_end = (ny + 3) & ~3;
  double* Vt = sm.Vt;
#ifdef RM_TIMING
  struct {
    long long* timing;
  } P{timing};
#endif
  RM_T0();
#ifdef RM_NO_FOLD
  const bool fold_x = false, fold_y = false;
#else
  const bool fold_x = C::FOLD && nx == C::NP - 1, fold_y = C::FOLD && ny == C::NP - 1;
#endif
  RM_FOR_ELEM {
    const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
    if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = r[mr][nf][e];
  }
  __syncthreads();
  RM_T(8);
  const int tm = fold_x ? c.tm_fold : c.tm;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if constexpr (C::G > C::UR) {
      // two CTAs share each own row (column halves): exchange the halves
      bcast_band<C>(bc, c.rank, c.tid);
    }
    // x-direction (transposed mapping) on the CTA's own rows
    dst_xT<C>(Vt, sm.tabx, Lx, acc, tm, c.tn, c.gq, c.tig, kx_end, fold_x);
    if constexpr (C::G > C::UR)
      group_sync<C::G>();  // the row-sharing peer received our half and finished reading its copy
    else
      __syncthreads();
    RM_T(9);
    RM_FOR_ELEM {
      const int j = elemT_row<C>(c, nf, e), i = fold_alpha<C>(16 * tm + c.gq + 8 * (e >> 1), fold_x) - 1;
      if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = acc[mr][nf][e];
    }
    bcast_band<C>(bc, c.rank, c.tid);
    RM_T(10);
    // y-direction (normal mapping) over all rows
    dst_y<C>(Vt, sm.taby, Ly, acc, c.urow, c.ucol, c.gq, c.tig, ky_end, fold_y);
    RM_T(11);
    if (pass == 1) break;
    // diagonal scaling: the dinv loads are issued before the barrier, which hides their L2 latency
    double dv[C::WR][C::NF][4];
    RM_FOR_ELEM { dv[mr][nf][e] = __ldcg(dinv + elem_sidx<C>(c, mr, nf, e)); }
    group_sync<C::G>();  // every CTA done reading its tile before peers push the next band
    RM_FOR_ELEM {
      const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
      if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = acc[mr][nf][e] * dv[mr][nf][e];
    }
    __syncthreads();
    RM_T(12);
  }
}

// Same preconditioner with the DST contractions on FP16 tensor-core MMAs (rm_device.cuh, Lp): the FP64
// tile region holds the FP16 tile and the DST matrix (bulk-copied from L2 per application).
// z = Sy (Sx-stage (Sy (Sx-stage r s1)) * dinv s2) / (s1 s2), FP32 accumulation, returned as FP64 in acc;
// s1 = 2^(6 - ilogb max|r|) (group maximum), s2 = 2^-ilogb(dbound), dbound >= max 1/d(s).
// A group barrier on entry: peers push FP16 bands into this CTA's tile region, which aliases FP64 rows
// that its threads may still read just before the call; the warp maxima of |r| travel with it.
template <class C>
__device__ __forceinline__ void apply_tau_lp(const Ctx<C>& c, const Smem<C>& sm, Bcast<C>& bc,
                                             const double (&r)[C::WR][C::NF][4], double (&acc)[C::WR][C::NF][4],
                                             const double* __restrict__ dinv, int nx, int ny,
                                             const uint16_t* __restrict__ gs, double dbound, bool restore,
                                             long long* timing) {
  using L = Lp<C>;
  static_assert(C::WR == 1, "DST stages assume one unit row per warp");
  static_assert(C::G * C::WARPS <= 64, "max slots");
  uint16_t* vh = reinterpret_cast<uint16_t*>(sm.Vt);
  const uint32_t vh_s = smem_addr(vh);
  const uint32_t s_s = vh_s + L::TILE_BYTES;  // square grids: one matrix serves both directions
#ifdef RM_TIMING
  struct {
    long long* timing;
  } P{timing};
#endif
  RM_T0();
  double m = 0.0;
#pragma unroll
  for (int nf = 0; nf < C::NF; ++nf)
#pragma unroll
    for (int e = 0; e < 4; ++e) m = fmax(m, fabs(r[0][nf][e]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (c.lane == 0) {
#pragma unroll
    for (int q = 0; q < C::G; ++q) sm.mx_peer[q][c.rank * C::WARPS + c.warp] = m;
  }
  group_sync<C::G>();
  if (c.tid == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bc.mbar2), "r"(L::TILE_BYTES)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s_s),
                 "l"(gs), "r"(L::TILE_BYTES), "r"(bc.mbar2)
                 : "memory");
  }
  double gm = 0.0;
  for (int t = c.lane; t < C::G * C::WARPS; t += 32) gm = fmax(gm, sm.mx[t]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, off));
  const int e1 = gm > 0.0 ? 6 - ilogb(gm) : 0;
  const int e2 = dbound > 0.0 ? -ilogb(dbound) : 0;
  const double s1 = ldexp(1.0, e1), s2 = ldexp(1.0, e2), unscale = ldexp(1.0, -e1 - e2);
  // r s1 -> Vh (own units; zero outside the grid)
#pragma unroll
  for (int nf = 0; nf < C::NF; ++nf)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = elem_row<C>(c, 0, 2 * h), i = elem_col<C>(c, nf, 2 * h);
      const bool in = j < ny;
      const float lo = (in && i < nx) ? (float)(r[0][nf][2 * h] * s1) : 0.f;
      const float hi = (in && i + 1 < nx) ? (float)(r[0][nf][2 * h + 1] * s1) : 0.f;
      *reinterpret_cast<uint32_t*>(vh + j * L::SH + i) = pack_f16x2(lo, hi);
    }
  RM_T(8);
  mbar_wait(bc.mbar2, bc.phase2);
  float a32[C::NF][4];
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if constexpr (C::G > C::UR) {
      // two CTAs share each own row (column halves): exchange the halves
      bcast_issue_tile<C, BcastShapeLp<C>>(bc, vh_s, c.rank, c.tid);
      bcast_wait<C>(bc);
    } else {
      __syncthreads();
    }
    dst_xT_lp<C>(vh_s, s_s, a32, c.tm, c.tn, c.lane);
    if constexpr (C::G > C::UR)
      group_sync<C::G>();  // the row-sharing peer received our half and finished reading its copy
    else
      __syncthreads();
    RM_T(9);
#pragma unroll
    for (int nf = 0; nf < C::NF; ++nf)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = elemT_row<C>(c, nf, e), i = 16 * c.tm + c.gq + 8 * (e >> 1);
        vh[j * L::SH + i] = to_f16(a32[nf][e]);
      }
    bcast_issue_tile<C, BcastShapeLp<C>>(bc, vh_s, c.rank, c.tid);
    bcast_wait<C>(bc);
    RM_T(10);
    dst_y_lp<C>(vh_s, s_s, a32, c.urow, c.ucol, c.lane);
    RM_T(11);
    if (pass == 1) break;
    double dv[C::NF][4];
#pragma unroll
    for (int nf = 0; nf < C::NF; ++nf)
#pragma unroll
      for (int e = 0; e < 4; ++e) dv[nf][e] = __ldcg(dinv + elem_sidx<C>(c, 0, nf, e)) * s2;
    group_sync<C::G>();  // every CTA done reading its tile before peers push the next band
#pragma unroll
    for (int nf = 0; nf < C::NF; ++nf)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = elem_row<C>(c, 0, 2 * h), i = elem_col<C>(c, nf, 2 * h);
        const bool in = j < ny;
        const float lo = (in && i < nx) ? (float)(a32[nf][2 * h] * dv[nf][2 * h]) : 0.f;
        const float hi = (in && i + 1 < nx) ? (float)(a32[nf][2 * h + 1] * dv[nf][2 * h + 1]) : 0.f;
        *reinterpret_cast<uint32_t*>(vh + j * L::SH + i) = pack_f16x2(lo, hi);
      }
    RM_T(12);
  }
#pragma unroll
  for (int nf = 0; nf < C::NF; ++nf)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[0][nf][e] = (double)a32[nf][e] * unscale;
  // restore the zero halo / padding of the FP64 tile rows the FP16 data overwrote (the matvec reads
  // them; the interior is rewritten with the next operand by the caller).  Not needed when the next
  // apply is the split-FP16 one (its caller restores the FP64 halo before any FP64 apply).
  if (!restore) return;
  __syncthreads();
  {
    constexpr int touched = (2 * (int)L::TILE_BYTES + 8 * C::S - 1) / (8 * C::S);
    double* Vt = sm.Vt;
    for (int R = c.tid; R < touched; R += C::THREADS) {
      double* row = Vt + R * C::S;
      if (R == 0 || R > ny) {
        for (int k = 0; k < C::S; ++k) row[k] = 0.0;
      } else {
        row[0] = 0.0;
        row[1] = 0.0;
        for (int k = nx + 2; k < C::S; ++k) row[k] = 0.0;
      }
    }
  }
}

// Zero every non-interior entry of the FP64 operand tile (halo rows / columns and the padding beyond
// nx, ny): the FP64 apply and the mass stencil read them.  Needed after the split-FP16 iteration or the
// FP16 preconditioner reused the tile region.  Touches no interior entry (peers' bands may be arriving).
template <class C>
__device__ __forceinline__ void vt_zero_halo(double* Vt, int nx, int ny, int tid) {
  for (int R = tid; R < C::NP + 2; R += C::THREADS) {
    double* row = Vt + R * C::S;
    if (R == 0 || R > ny) {
      for (int k = 0; k < C::S; ++k) row[k] = 0.0;
    } else {
      row[0] = 0.0;
      row[1] = 0.0;
      for (int k = nx + 2; k < C::S; ++k) row[k] = 0.0;
    }
  }
}

// Zero the halo rows and pad columns of both split-FP16 data tiles (this CTA's copy, all rows).
template <class C>
__device__ __forceinline__ void mx_zero_pads(double* Vt, int tid) {
  using X = Mx<C>;
  constexpr int RB = X::SHD * 2 / 16;  // 16-byte chunks per row
  uint4* base = reinterpret_cast<uint4*>(Vt);
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  constexpr int FULL = 2 * 2 * RB;                    // rows -1 and NP of both tiles
  constexpr int PADS = 2 * C::NP * 3;                 // 3 pad chunks per interior row (cols [-8,0), [NP,NP+16))
  for (int idx = tid; idx < FULL + PADS; idx += C::THREADS) {
    if (idx < FULL) {
      const int t = idx / (2 * RB), rr = (idx / RB) % 2, ch = idx % RB;
      base[t * (X::TILE_BYTES / 16) + (rr ? C::NP + 1 : 0) * RB + ch] = z;
    } else {
      const int k = idx - FULL, t = k / (3 * C::NP), rr = (k / 3) % C::NP + 1, ch = k % 3;
      base[t * (X::TILE_BYTES / 16) + rr * RB + (ch == 0 ? 0 : RB - 3 + ch)] = z;
    }
  }
}

// the split-FP16 data tiles: each CTA's own rows of both tiles (hi, lo) in one exchange
template <class C>
struct BcastShapeMx {
  using B = BcastShapeT<C, 2, Mx<C>::SHD, 1, Mx<C>::COL0>;
  static constexpr int NSEG = 2 * B::NSEG;
  static constexpr uint32_t SEG_BYTES = B::SEG_BYTES;
  static __device__ __forceinline__ uint32_t seg_off(int rank, int t) {
    return B::seg_off(rank, t >> 1) + (t & 1) * Mx<C>::TILE_BYTES;
  }
};

// split-FP16 iteration: residual replacement once the recursive residual fell below this fraction of
// the true residual at the last replacement (the apply is accurate to ~1e-5 for smooth directions)
constexpr double kLpReplace = 1e-5;
// split-FP16 iteration only for steps with s max|K| <= kLpMaxRatio * 6 cm (condition number ~< 20)
constexpr double kLpMaxRatio = 16.0;

template <class C, bool PRE>
__global__ void __launch_bounds__(C::THREADS, 1) chain_kernel(const ChainArgs P) {
  static_assert(C::SMEM <= 227 * 1024, "shared memory budget");
  extern __shared__ __align__(16) double smem[];
  Smem<C> sm;
  sm.Vt = smem;                    // operand tile (p, or the vector being applied)
  sm.gens = sm.Vt + C::VT;         // generator tables
  sm.red = sm.gens + 6 * C::GL;    // reduction buffers
  sm.xs = sm.red + C::RED;         // this CTA's part of the previous search direction (PCG)
  sm.tabx = sm.xs + C::XS;         // DST sine tables
  sm.taby = sm.tabx + C::ST;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sm.taby + C::ST);  // [0] band exchange, [1] DST matrix
  int* sched = reinterpret_cast<int*>(mbar + 2);
  sm.mx = reinterpret_cast<double*>(mbar) + 8;  // [G * WARPS] warp maxima of |r| (low-precision tau)
  double* Vt = sm.Vt;
  double* gens = sm.gens;
  double* red = sm.red;

  Ctx<C> c;
  c.tid = threadIdx.x;
  c.lane = c.tid & 31;
  c.warp = c.tid >> 5;
  c.gq = c.lane >> 2;
  c.tig = c.lane & 3;
  c.rank = 0;
  if constexpr (C::G > 1) c.rank = (int)cgx::this_cluster().block_rank();
  {
    int r0, c0;
    if constexpr (C::G <= C::UR) {
      r0 = c.rank * C::CR;
      c0 = 0;
    } else {
      constexpr int per = C::G / C::UR;
      r0 = c.rank / per;
      c0 = (c.rank % per) * C::CC;
    }
    constexpr int wcols = C::CC / C::WC;
    c.urow = r0 + (c.warp / wcols) * C::WR;
    c.ucol = c0 + (c.warp % wcols) * C::WC;
    // transposed DST stage: m over the CTA's CC unit columns, n over its CR unit rows
    constexpr int tcols = C::CR / C::WC > 0 ? C::CR / C::WC : 1;
    c.tm = c0 + c.warp / tcols;
    c.tn = r0 + (c.warp % tcols) * C::WC;
    c.tm_fold = c.tm;
    if constexpr (C::G > C::UR) {
      // two CTAs share a unit row (column halves): with the fold, output column i = alpha - 1 comes
      // from m = i/2 (i even) or HALF + i/2 (i odd), so take both halves' m units of own columns
      const int w = c.warp / tcols;
      c.tm_fold = w < C::CC / 2 ? c0 / 2 + w : C::UR / 2 + c0 / 2 + (w - C::CC / 2);
    }
  }

  int* sched_peer[C::G];
  if constexpr (C::G == 1) {
    sm.red_peer[0] = red;
    sm.mx_peer[0] = sm.mx;
    sched_peer[0] = sched;
  } else {
    auto cl = cgx::this_cluster();
#pragma unroll
    for (int q = 0; q < C::G; ++q) {
      sm.red_peer[q] = cl.map_shared_rank(red, q);
      sm.mx_peer[q] = cl.map_shared_rank(sm.mx, q);
      sched_peer[q] = cl.map_shared_rank(sched, q);
    }
  }

  const rm_sweep& W = P.sw;
  const int nx = P.nx, ny = P.ny;
  const int ndof = nx * ny;
  const int kx_end = (nx + 3) & ~3, ky_end = (ny + 3) & ~3;
  const int Lx = 2 * (nx + 1), Ly = 2 * (ny + 1);
  const double cm = P.cm;
  const int64_t max_iter = W.max_iter > 0 ? W.max_iter : 10 * (int64_t)ndof;
  const bool need_in = W.explicit_rhs || W.x0_mode == 1;
  // G row scale (compressed G, rm_sweep.d_gscale): rows of d_gadd / d_hg are d_gscale[n] times the stored row
  auto gsc = [&](int k) -> double { return W.d_gscale ? W.d_gscale[k] : 1.0; };

  for (int i = c.tid; i < C::VT; i += C::THREADS) Vt[i] = 0.0;
  if constexpr (PRE) {
    for (int i = c.tid; i < Lx; i += C::THREADS) sm.tabx[tab_idx(i)] = P.tabx[i];
    for (int i = c.tid; i < Ly; i += C::THREADS) sm.taby[tab_idx(i)] = P.taby[i];
  }
  Bcast<C> bc;
  bcast_setup<C>(bc, Vt, mbar, c.tid);
  group_sync<C::G>();

  const int cid = blockIdx.x / C::G;
  double* sb_ = P.scratch + (size_t)cid * 3 * C::NP * C::NP;  // right-hand side b (true-residual checks)
  double* dinv = sb_ + C::NP * C::NP;                         // 1 / d(s) of the tau preconditioner
  // CG iterate x of this CTA's units, fragment-native in the L2-resident scratch: updated with
  // fire-and-forget reductions (one owner thread per element: ordered, deterministic), read back once
  // per solve; its shared-memory slot holds the previous search direction instead (critical path)
  double* xs = dinv + C::NP * C::NP + (size_t)c.rank * C::CU * 256;
  double* pold_ = sm.xs;
  int buf = 0;

  double acc[C::WR][C::NF][4];  // operator output of the current matvec / DST stage
  double rr_[C::WR][C::NF][4];  // CG residual r (register resident)
  // z = P^-1 r into acc: FP16 tensor-core DST stages (precond 2) or FP64 DMMA (precond 1)
  const bool lp_dst = W.precond == 2;
  // split-FP16 search-direction applies inside the PCG iteration (Mx; with the FP16 preconditioner)
  const bool lp_mv = Mx<C>::ENABLED && PRE && lp_dst && W.lp_matvec;
  bool lp_step = false;  // this step runs the split-FP16 iteration (well-conditioned step operators only)
  double lp_dbound = 1.0;  // >= max_i 1/d_i(s) of the current step
  auto tau_apply = [&](const double(&rin)[C::WR][C::NF][4]) {
    if (lp_dst)
      apply_tau_lp<C>(c, sm, bc, rin, acc, dinv, nx, ny, P.dst16, lp_dbound, !lp_step, P.timing);
    else
      apply_tau<C>(c, sm, bc, rin, acc, dinv, nx, ny, Lx, Ly, P.timing);
  };
  // split-FP16 iteration state: power-of-two scales of the data (2^lp_ep, from a bound on max|p|) and of
  // the pair tables (2^lp_et, per step); the tables are rebuilt whenever FP64 data overwrote them
  uint32_t* lp_pt = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(Vt) + Mx<C>::PT_OFF);
  int lp_ep = 0, lp_et = 0;
  double lp_bp = 0.0;
  double lp_rrep = 0.0;  // true residual norm at the solve start / last replacement
  bool lp_true_next = false;  // the next iteration computes the true residual (FP64 apply)
  bool lp_pt_ok = false;
  // p = z [+ beta p_old] (z in acc): FP64 copy in pold_, split-FP16 copy in the data tiles (own units),
  // pads zeroed, pair tables rebuilt if needed, own bands pushed to the peers (waited for in the apply)
  auto lp_set_p = [&](double beta, bool with_old) {
#pragma unroll
    for (int nf = 0; nf < C::NF; ++nf)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = elem_row<C>(c, 0, 2 * h), i = elem_col<C>(c, nf, 2 * h);
        double pv[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int e = 2 * h + u;
          pv[u] = 0.0;
          if (j < ny && i + u < nx) {
            const int xi = elem_xidx<C>(c, 0, nf, e);
            pv[u] = with_old ? acc[0][nf][e] + beta * pold_[xi] : acc[0][nf][e];
            pold_[xi] = pv[u];
          }
        }
        const double sc = ldexp(1.0, lp_ep);
        float h0, l0, h1, l1;
        split_f16(pv[0] * sc, h0, l0);
        split_f16(pv[1] * sc, h1, l1);
        uint32_t* hi = reinterpret_cast<uint32_t*>(reinterpret_cast<uint16_t*>(Vt) + (j + 1) * Mx<C>::SHD +
                                                   Mx<C>::COL0 + i);
        hi[0] = pack_f16x2(h0, h1);
        hi[Mx<C>::TILE / 2] = pack_f16x2(l0, l1);
      }
    mx_zero_pads<C>(Vt, c.tid);
    if (!lp_pt_ok) {
      build_pair_tables<C>(lp_pt, gens, ldexp(1.0, lp_et), c.tid);
      lp_pt_ok = true;
    }
    bcast_issue_tile<C, BcastShapeMx<C>>(bc, smem_addr(Vt), c.rank, c.tid);
  };

  for (;;) {
    if (c.rank == 0 && c.tid == 0) {
      const int ch = atomicAdd(P.chain_counter, 1);
#pragma unroll
      for (int q = 0; q < C::G; ++q) sched_peer[q][0] = ch;
    }
    group_sync<C::G>();
    const int chain = sched[0];
    group_sync<C::G>();
    if (chain >= W.nchains) break;

    const int n0 = W.first + chain * W.cstride;
    const int n1 = min(n0 + W.clen - 1, W.nmax);
    bool in_tile = false;   // previous step left this step's input in Vt
    bool chain_ok = false;  // ... and its accepted true residual in rr_ (apply-free next right-hand side)
    double s_prev = 0.0;
    for (int n = n0; n <= n1; ++n) {
      const double s = 0.5 * W.d_dt[n - 1];
      if (lp_dst) {
        const double dlow = P.lp_dmin + s * P.lp_kmin;
        lp_dbound = dlow > 0.0 ? 1.0 / dlow : 0.0;
      }
      const double fs = W.d_f ? (W.d_fscale ? W.d_fscale[n] : 1.0) : 0.0;
      const double* Fn = W.d_f ? W.d_f + (int64_t)n * W.f_stride : nullptr;
      if (lp_mv) {
        vt_zero_halo<C>(Vt, nx, ny, c.tid);  // the previous solve's FP16 data overwrote the FP64 tile
        lp_et = 13 - ilogb(fabs(s) * P.gen_absmax + 6.0 * cm);  // max |table entry| < 2^14 after scaling
        lp_pt_ok = false;
        // the apply error grows with the step operator's condition number (~ s max|K| / (6 cm)):
        // only well-conditioned steps (the fine levels) iterate in split FP16
        lp_step = fabs(s) * P.gen_absmax <= kLpMaxRatio * 6.0 * cm;
      }

      // ---------------- right-hand side, initial iterate and residual --------------
      // (the previous step ended with a group barrier: nobody reads the tables any more)
      // Inside a chain (the previous step's output y_{n-1} = x + G_{n-1} is in the tile and its true residual
      // r = b - A_{s0} x in rr_) the explicit side needs no apply:
      //   (M - s K) y = (1 + s/s0) M y - (s/s0) (b - r + A_{s0} G_{n-1}),   A_{s0} G_{n-1} = d_hg row n-1
      // (host-precomputed per level; s0 = dt_{n-1}/2).  Exact up to rounding.
      const bool rhs_free = need_in && W.explicit_rhs && in_tile && chain_ok && W.d_hg != nullptr &&
                            W.d_gadd != nullptr && W.d_sub == nullptr;
      // ... and at a chain's first step whose input point n-1 was written by an accepted solve whose A x was
      // stored (d_ain, with d_hg): A_{s0} y = A x + A G of that point
      const bool rhs_ain = need_in && W.explicit_rhs && !in_tile && n >= 2 && W.d_ain != nullptr &&
                           W.d_hg != nullptr;
      if (need_in && !rhs_free) {
        if (!rhs_ain) build_step_tables<C::NP, C::GL, C::THREADS>(gens, P.gens, -s, cm, c.tid);  // M - s K
        if (!in_tile) load_vec<C>(Vt, W.d_src + (int64_t)(n - 1) * W.src_stride, nx, ny, c);
        __syncthreads();
        if (!rhs_ain) matvec<C>(Vt, gens, acc, c.urow, c.ucol, c.gq, c.tig, kx_end, ky_end, true, true, P.merge);
      }
      if (rhs_ain) {
        const double* An = W.d_ain + (int64_t)(n - 1) * W.ain_stride;
        const double* Hn = W.d_hg + (int64_t)(n - 1) * W.hg_stride;
        const double q = s / (0.5 * W.d_dt[n - 2]);
        RM_FOR_ELEM {
          const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
          double am = 0.0;
          if (j < ny && i < nx) {
            const int gi = j * nx + i;
            am = (1.0 + q) * mass_stencil<C>(Vt, j, i, cm) - q * (__ldcg(An + gi) + gsc(n - 1) * __ldcg(Hn + gi));
          }
          acc[mr][nf][e] = am;
        }
      }
      if (rhs_free) {
        __syncthreads();  // the tile's halo (re-zeroed above in the split-FP16 mode) before the mass stencil
        const double* Hn = W.d_hg + (int64_t)(n - 1) * W.hg_stride;
        const double q = s / s_prev;
        RM_FOR_ELEM {
          const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
          double am = 0.0;
          if (j < ny && i < nx) {
            const double ax = sb_[elem_sidx<C>(c, mr, nf, e)] - rr_[mr][nf][e] + gsc(n - 1) * __ldcg(Hn + j * nx + i);
            am = (1.0 + q) * mass_stencil<C>(Vt, j, i, cm) - q * ax;
          }
          acc[mr][nf][e] = am;
        }
      }
      s_prev = s;
      chain_ok = false;  // set again when this step's solve is accepted
      int64_t nmv = need_in && !rhs_free && !rhs_ain ? 1 : 0;
      int64_t nmv16 = 0;  // split-FP16 applies (lp_step)
      int64_t npc = 0;  // preconditioner applications
      double part[2][C::WR][C::WC];
      zero_part<C>(part[0]);
      zero_part<C>(part[1]);
      RM_FOR_ELEM {
        const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
        double b = 0.0, x = 0.0, r = 0.0;
        const int si = elem_sidx<C>(c, mr, nf, e);
        if (j < ny && i < nx) {
          const double am = need_in ? acc[mr][nf][e] : 0.0;  // (M - s K) v
          if (W.explicit_rhs) b = am;
          if (Fn) {
            const double f = fs * __ldcg(Fn + j * nx + i);
            b = W.explicit_rhs ? f + b : f;
          }
          if (W.x0_mode == 1) {
            // x0 = v: (M + s K) v = 2 M v - (M - s K) v
            x = Vt[vt_idx<C>(j, i)];
            r = b - (2.0 * mass_stencil<C>(Vt, j, i, cm) - am);
          } else {
            r = b;  // x0 = 0: r = b - A*0 (krylov.py:47,50)
          }
          if constexpr (PRE) dinv[si] = 1.0 / (__ldg(P.dm + j * nx + i) + s * __ldg(P.dk + j * nx + i));
        }
        sb_[si] = b;
        xs[elem_xidx<C>(c, mr, nf, e)] = x;
        rr_[mr][nf][e] = r;
        part[0][mr][nf >> 1] += b * b;
        part[1][mr][nf >> 1] += r * r;
      }
      __syncthreads();
      build_step_tables<C::NP, C::GL, C::THREADS>(gens, P.gens, s, cm, c.tid);  // M + s K from here on
      __syncthreads();
      if (W.x0_mode == 2) {
        // given initial iterate (spacetime_residual, stepper.py:203)
        load_vec<C>(Vt, W.d_x0 + (int64_t)n * W.x0_stride, nx, ny, c);
        __syncthreads();
        matvec<C>(Vt, gens, acc, c.urow, c.ucol, c.gq, c.tig, kx_end, ky_end, true, true, P.merge);
        ++nmv;
        zero_part<C>(part[1]);
        RM_FOR_ELEM {
          const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
          double x = 0.0, r = 0.0;
          if (j < ny && i < nx) {
            x = Vt[vt_idx<C>(j, i)];
            r = sb_[elem_sidx<C>(c, mr, nf, e)] - acc[mr][nf][e];
          }
          xs[elem_xidx<C>(c, mr, nf, e)] = x;
          rr_[mr][nf][e] = r;
          part[1][mr][nf >> 1] += r * r;
        }
      }
      double tot[2];
      group_reduce<C, 2>(part, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, tot);
      buf ^= 1;
      const double bnorm = sqrt(tot[0]);
      const double target = bnorm > 0.0 ? W.rel_tol * bnorm : W.rel_tol;
      if (W.d_guess && W.x0_mode != 3 && sqrt(tot[1]) > target) {
        // second candidate start x0' = guess_n [- G_n] (the value this solve is about to replace);
        // keep whichever initial residual is smaller (deterministic: both norms are group-reduced)
        const double* Gr = W.d_gadd ? W.d_gadd + (int64_t)n * W.gadd_stride : nullptr;
        const double* Gu = W.d_guess + (int64_t)n * W.guess_stride;
        // A x0' is either applied, or -- when this point was last written by an accepted solve of the same
        // operator whose A x was stored (d_gax) -- read back: no apply
        const double* Ax0 = W.d_gax ? W.d_gax + (int64_t)n * W.gax_stride : nullptr;
        if (!Ax0) {
          load_guess<C>(Vt, Gu, Gr, nx, ny, c, gsc(n));
          __syncthreads();
          matvec<C>(Vt, gens, acc, c.urow, c.ucol, c.gq, c.tig, kx_end, ky_end, true, true, P.merge);
          ++nmv;
        }
        double pg[1][C::WR][C::WC];
        zero_part<C>(pg[0]);
        RM_FOR_ELEM {
          const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
          double r = 0.0;
          if (j < ny && i < nx)
            r = sb_[elem_sidx<C>(c, mr, nf, e)] - (Ax0 ? __ldcg(Ax0 + j * nx + i) : acc[mr][nf][e]);
          acc[mr][nf][e] = r;
          pg[0][mr][nf >> 1] += r * r;
        }
        double rg[1];
        group_reduce<C, 1>(pg, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, rg);
        buf ^= 1;
        if (rg[0] < tot[1]) {
          tot[1] = rg[0];
          RM_FOR_ELEM {
            const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
            double x0 = 0.0;
            if (j < ny && i < nx) {
              if (Ax0)
                x0 = Gr ? __ldcg(Gu + j * nx + i) - gsc(n) * __ldcg(Gr + j * nx + i) : __ldcg(Gu + j * nx + i);
              else
                x0 = Vt[vt_idx<C>(j, i)];
            }
            xs[elem_xidx<C>(c, mr, nf, e)] = x0;
            rr_[mr][nf][e] = acc[mr][nf][e];
          }
        }
      }
      double res = sqrt(tot[1]);
      double rr = tot[1];  // r.r (CG) or r.z (PCG)
      lp_rrep = res;
      lp_true_next = false;
      int64_t its = 0;
      int fail = 0;
      bool done = res <= target;
      if (W.x0_mode == 3) {
        // preconditioner probe: y = P^-1 b, no CG (the host checks it against precond.py)
        if constexpr (PRE) {
          tau_apply(rr_);
          ++npc;
          RM_FOR_ELEM { xs[elem_xidx<C>(c, mr, nf, e)] = acc[mr][nf][e]; }
        }
        done = true;
      }
      if (W.x0_mode == 4) {
        // split-FP16 apply probe: y = (M + s K) b through the in-iteration path (b in the role of p)
        if (lp_mv) {
          RM_FOR_ELEM { acc[mr][nf][e] = rr_[mr][nf][e]; }
          double mb = 0.0, one[1];
          RM_FOR_ELEM { mb = fmax(mb, fabs(acc[mr][nf][e])); }
          double p0[1][C::WR][C::WC];
          zero_part<C>(p0[0]);
          group_reduce_mx<C, 1>(p0, mb, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, one, lp_bp);
          buf ^= 1;
          lp_ep = lp_bp > 0.0 ? 13 - ilogb(lp_bp) : 0;
          lp_set_p(0.0, false);
          bcast_wait<C>(bc);
          float a32[C::NF][4];
          matvec_lp<C>(smem_addr(Vt), lp_pt, a32, c.urow, c.ucol, c.gq, c.tig, c.lane);
          const double inv = ldexp(1.0, -(lp_ep + lp_et));
          RM_FOR_ELEM { xs[elem_xidx<C>(c, mr, nf, e)] = (double)a32[nf][e] * inv; }
          ++nmv16;
          group_sync<C::G>();
        }
        done = true;
      }

      if (!done) {
        if constexpr (PRE) {
          // z = P^-1 r, p = z, rz = r.z
          tau_apply(rr_);
          ++npc;
          double p1[1][C::WR][C::WC];
          zero_part<C>(p1[0]);
          RM_FOR_ELEM { p1[0][mr][nf >> 1] += rr_[mr][nf][e] * acc[mr][nf][e]; }
          double rz[1];
          if (lp_step) {
            double mz = 0.0;
            RM_FOR_ELEM { mz = fmax(mz, fabs(acc[mr][nf][e])); }
            double gz;
            group_reduce_mx<C, 1>(p1, mz, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, rz, gz);
            buf ^= 1;
            rr = rz[0];
            lp_bp = gz;
            lp_ep = gz > 0.0 ? 13 - ilogb(gz) : 0;
            lp_set_p(0.0, false);  // waited for inside the first apply
          } else {
            group_reduce<C, 1>(p1, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, rz);
            buf ^= 1;
            rr = rz[0];
            RM_FOR_ELEM {
              const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
              if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = acc[mr][nf][e];
            }
            bcast_issue<C>(bc, c.rank, c.tid);  // waited for inside the first matvec
          }
        } else {
          // p = r into the operand tile of every CTA of the group
          RM_FOR_ELEM {
            const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
            if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = rr_[mr][nf][e];
          }
          bcast_issue<C>(bc, c.rank, c.tid);  // waited for inside the first matvec
        }
      }
      if (c.tid == 0 && n < n1) {
        // the chain's next-step inputs: L2 resident by the time this solve finishes (each CTA of the
        // group takes a slice of every row)
        const size_t vb = (size_t)ndof * sizeof(double);
        const size_t lo = vb * c.rank / C::G, hi = vb * (c.rank + 1) / C::G;
        auto pf = [&](const double* base, int64_t stride) {
          if (base) prefetch_l2(reinterpret_cast<const char*>(base + (int64_t)(n + 1) * stride) + lo, hi - lo);
        };
        pf(W.d_guess, W.guess_stride);
        pf(W.d_gadd, W.gadd_stride);
        pf(W.d_f, W.f_stride);
        pf(W.d_sub, W.sub_stride);
        pf(W.d_gax, W.gax_stride);
        if (W.d_hg)  // the next step's apply-free right-hand side reads row n
          prefetch_l2(reinterpret_cast<const char*>(W.d_hg + (int64_t)n * W.hg_stride) + lo, hi - lo);
      }
      RM_T0();
      for (int64_t k = 1; !done; ++k) {
        if (k > max_iter) {
          bcast_wait<C>(bc);  // complete the pending exchange (keeps the mbarrier phase in step)
          fail = RM_CG_BUDGET;
          its = max_iter;
          break;
        }
        RM_T(7);
        // Ap and p'Ap; the peers' bands of p arrive during the diagonal x segment (own rows only)
        if (lp_step) {
          bcast_wait<C>(bc);
          float a32[C::NF][4];
          matvec_lp<C>(smem_addr(Vt), lp_pt, a32, c.urow, c.ucol, c.gq, c.tig, c.lane);
          const double inv = ldexp(1.0, -(lp_ep + lp_et));
          RM_FOR_ELEM { acc[mr][nf][e] = (double)a32[nf][e] * inv; }
          ++nmv16;
        } else {
          if constexpr (C::G > C::UR) bcast_wait<C>(bc);  // own rows are shared: nothing to overlap
          matvec<C>(Vt, gens, acc, c.urow, c.ucol, c.gq, c.tig, kx_end, ky_end, true, true, P.merge, [&] {
            if constexpr (C::G <= C::UR) bcast_wait<C>(bc);
          });
          ++nmv;
        }
        RM_T(0);
        double p1[1][C::WR][C::WC];
        zero_part<C>(p1[0]);
        RM_FOR_ELEM {
          const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
          double ap = 0.0;
          if (j < ny && i < nx) {
            ap = acc[mr][nf][e];
            p1[0][mr][nf >> 1] += (lp_step ? pold_[elem_xidx<C>(c, mr, nf, e)] : Vt[vt_idx<C>(j, i)]) * ap;
          }
          acc[mr][nf][e] = ap;
        }
        RM_T(1);
        double pap[1];
        group_reduce<C, 1>(p1, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, pap);
        buf ^= 1;
        RM_T(2);
        if (!isfinite(pap[0]) || pap[0] <= 0.0) {
          fail = RM_CG_BREAKDOWN;
          its = k;
          break;
        }
        const double alpha = rr / pap[0];
        double part2[2][C::WR][C::WC];
        zero_part<C>(part2[0]);
        zero_part<C>(part2[1]);
        const bool true_now = lp_step && lp_true_next;
        RM_FOR_ELEM {
          const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
          if (j < ny && i < nx) {
            const int xi = elem_xidx<C>(c, mr, nf, e);
            const double pv = lp_step ? pold_[xi] : Vt[vt_idx<C>(j, i)];
            atomicAdd(xs + xi, alpha * pv);  // RED: no return value, no latency on the critical path
            const double rn = rr_[mr][nf][e] - alpha * acc[mr][nf][e];
            rr_[mr][nf][e] = rn;
            if (!true_now) part2[0][mr][nf >> 1] += rn * rn;
            // the preconditioner overwrites the operand tile: keep p for the direction update
            if constexpr (PRE)
              if (!lp_step) pold_[xi] = pv;
          }
        }
        if (true_now) {
          // split-FP16 iteration, predicted to cross the target or the replacement threshold: this
          // iteration's residual is the TRUE one, b - A x with the FP64 apply (residual replacement; the
          // search direction recurrence continues), so no preconditioner application is wasted
          vt_zero_halo<C>(Vt, nx, ny, c.tid);
          lp_pt_ok = false;
          RM_FOR_ELEM {
            const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
            if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = xs[elem_xidx<C>(c, mr, nf, e)];
          }
          bcast_band<C>(bc, c.rank, c.tid);
          matvec<C>(Vt, gens, acc, c.urow, c.ucol, c.gq, c.tig, kx_end, ky_end, true, true, P.merge);
          ++nmv;
          RM_FOR_ELEM {
            const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
            double rt = 0.0;
            if (j < ny && i < nx) rt = sb_[elem_sidx<C>(c, mr, nf, e)] - acc[mr][nf][e];
            rr_[mr][nf][e] = rt;
            part2[0][mr][nf >> 1] += rt * rt;
          }
        }
        RM_T(3);
        double red2[2];
        double lp_mz = 0.0;
        if constexpr (PRE) {
          // z = P^-1 r; reduce r.r (convergence test) and r.z together
          tau_apply(rr_);
          ++npc;
          RM_TM();
          RM_FOR_ELEM { part2[1][mr][nf >> 1] += rr_[mr][nf][e] * acc[mr][nf][e]; }
          if (lp_step) {
            double mz = 0.0;
            RM_FOR_ELEM { mz = fmax(mz, fabs(acc[mr][nf][e])); }
            group_reduce_mx<C, 2>(part2, mz, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, red2, lp_mz);
          } else {
            group_reduce<C, 2>(part2, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, red2);
          }
        } else {
          double p0[1][C::WR][C::WC];
#pragma unroll
          for (int mr = 0; mr < C::WR; ++mr)
#pragma unroll
            for (int uc = 0; uc < C::WC; ++uc) p0[0][mr][uc] = part2[0][mr][uc];
          double one[1];
          group_reduce<C, 1>(p0, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, one);
          red2[0] = one[0];
          red2[1] = one[0];
        }
        buf ^= 1;
        RM_T(4);
        double rr_new = red2[0];
        const double res_prev = res;
        res = sqrt(rr_new);
        if (!isfinite(res)) {
          fail = RM_CG_NONFINITE;
          its = k;
          break;
        }
        if (true_now) {
          if (res <= target) {  // the reference criterion on the true residual
            its = k;
            done = true;
            break;
          }
          lp_rrep = res;
      lp_true_next = false;
        }
        if (lp_step) {
          // next residual ~ res * (res / res_prev): make it the true one if it is predicted to cross the
          // target or the replacement threshold
          const double pred = res * fmin(1.0, res / res_prev);
          lp_true_next = pred <= target || pred <= kLpReplace * lp_rrep;
        }
        if (res <= target && !true_now) {
          // acceptance on the true residual (krylov.py:71-83), FP64 apply.  Split-FP16 iteration: also a
          // residual replacement every kLpReplace of contraction (the recursive residual drifts from the
          // true one by ~1e-5 of the residual at the last replacement), the search direction kept.
          if (lp_step) {
            vt_zero_halo<C>(Vt, nx, ny, c.tid);
            lp_pt_ok = false;
          }
          RM_FOR_ELEM {
            const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
            if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = xs[elem_xidx<C>(c, mr, nf, e)];
          }
          bcast_band<C>(bc, c.rank, c.tid);
          matvec<C>(Vt, gens, acc, c.urow, c.ucol, c.gq, c.tig, kx_end, ky_end, true, true, P.merge);
          ++nmv;
          zero_part<C>(p1[0]);
          RM_FOR_ELEM {
            const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
            double rt = 0.0;
            if (j < ny && i < nx)
              rt = sb_[elem_sidx<C>(c, mr, nf, e)] - acc[mr][nf][e];
            acc[mr][nf][e] = rt;
            p1[0][mr][nf >> 1] += rt * rt;
          }
          double tt[1];
          group_reduce<C, 1>(p1, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, tt);
          buf ^= 1;
          const double true_res = sqrt(tt[0]);
          // the reference's acceptance; the split-FP16 iteration accepts only a true residual <= target
          if (true_res <= (lp_step ? target : fmax(target, 10.0 * res))) {
            RM_FOR_ELEM { rr_[mr][nf][e] = acc[mr][nf][e]; }  // r_n = b_n - A x_n for the chain's next rhs
            its = k;
            done = true;
            break;
          }
          // recurrence drifted: restart from the true residual
          res = true_res;
          RM_FOR_ELEM { rr_[mr][nf][e] = acc[mr][nf][e]; }
          if (res <= target) {
            its = k;
            done = true;
            break;
          }
          if constexpr (PRE) {
            tau_apply(rr_);
            ++npc;
            zero_part<C>(p1[0]);
            RM_FOR_ELEM { p1[0][mr][nf >> 1] += rr_[mr][nf][e] * acc[mr][nf][e]; }
            double rz[1];
            if (lp_step) {
              // residual replacement: continue the direction recurrence from the true residual
              double mz = 0.0;
              RM_FOR_ELEM { mz = fmax(mz, fabs(acc[mr][nf][e])); }
              double gz;
              group_reduce_mx<C, 1>(p1, mz, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, rz, gz);
              buf ^= 1;
              const double beta = rz[0] / rr;
              rr = rz[0];
              lp_rrep = true_res;
              lp_bp = gz + fabs(beta) * lp_bp;
              lp_ep = lp_bp > 0.0 ? 13 - ilogb(lp_bp) : 0;
              lp_set_p(beta, true);
              continue;
            }
            group_reduce<C, 1>(p1, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, rz);
            buf ^= 1;
            rr = rz[0];
          } else {
            rr = tt[0];
          }
          RM_FOR_ELEM {
            const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
            if (j < ny && i < nx) Vt[vt_idx<C>(j, i)] = acc[mr][nf][e];
          }
          bcast_issue<C>(bc, c.rank, c.tid);
          continue;
        }
        const double rho_new = red2[1];
        const double beta = rho_new / rr;
        rr = rho_new;
        if (lp_step) {
          // max|p| <= max|z| + beta max|p_old| (all CTAs hold the same bound)
          lp_bp = lp_mz + fabs(beta) * lp_bp;
          lp_ep = lp_bp > 0.0 ? 13 - ilogb(lp_bp) : 0;
          lp_set_p(beta, true);
          RM_T(5);
          RM_T(6);
          continue;
        }
        RM_FOR_ELEM {
          const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
          if (j < ny && i < nx) {
            const int vi = vt_idx<C>(j, i);
            if constexpr (PRE)
              Vt[vi] = acc[mr][nf][e] + beta * pold_[elem_xidx<C>(c, mr, nf, e)];
            else
              Vt[vi] = rr_[mr][nf][e] + beta * Vt[vi];
          }
        }
        RM_T(5);
        bcast_issue<C>(bc, c.rank, c.tid);
        RM_T(6);
      }

      chain_ok = done && !fail && W.x0_mode < 3;
      if (c.rank == 0 && c.tid == 0) {
        atomicAdd(W.d_counters, 1ull);
        atomicAdd(W.d_counters + 1, (unsigned long long)its);
        atomicAdd(W.d_counters + 2, (unsigned long long)nmv);
        atomicAdd(W.d_counters + 3, (unsigned long long)npc);
        if (lp_step) atomicAdd(W.d_counters + 4, (unsigned long long)nmv16);
      }
      if (fail) {
        if (c.rank == 0 && c.tid == 0 && atomicCAS(P.fail, 0, fail) == 0) {
          P.fail_info[0] = (double)n;
          P.fail_info[1] = (double)its;
          P.fail_info[2] = res;
        }
        group_sync<C::G>();
        break;  // abandon the chain (the host raises CgFailure)
      }

      // ---------------- MGRIT epilogue: y = [G_n +] x [- S_n] ----------------
      // every CTA is past its last read of Vt (the final reduction synchronised the group)
      const bool next_in_tile = n < n1 && need_in;
      const int oi = n / W.out_div;
      const double* Gn = W.d_gadd ? W.d_gadd + (int64_t)n * W.gadd_stride : nullptr;
      const double* Sn = W.d_sub ? W.d_sub + (int64_t)n * W.sub_stride : nullptr;
      double* On = W.d_out ? W.d_out + (int64_t)oi * W.out_stride : nullptr;
      double* Kn = W.d_keep ? W.d_keep + (int64_t)oi * W.keep_stride : nullptr;
      double* An = W.d_ax ? W.d_ax + (int64_t)oi * W.ax_stride : nullptr;
      double p1[1][C::WR][C::WC];
      zero_part<C>(p1[0]);
      RM_FOR_ELEM {
        const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
        if (j < ny && i < nx) {
          const int gi = j * nx + i;
          double y = xs[elem_xidx<C>(c, mr, nf, e)];
          if (An) An[gi] = sb_[elem_sidx<C>(c, mr, nf, e)] - rr_[mr][nf][e];  // A x = b - r (true residual)
          if (Gn) y = gsc(n) * __ldcg(Gn + gi) + y;
          if (Kn) Kn[gi] = y;
          if (Sn) y = y - __ldcg(Sn + gi);
          if (On) On[gi] = y;
          if (next_in_tile) Vt[vt_idx<C>(j, i)] = y;
          p1[0][mr][nf >> 1] += y * y;
        }
      }
      if (W.d_norms) {
        double yy[1];
        group_reduce<C, 1>(p1, red, sm.red_peer, buf, c.urow, c.ucol, c.lane, yy);
        buf ^= 1;
        if (c.rank == 0 && c.tid == 0) W.d_norms[oi] = yy[0];
      }
      in_tile = next_in_tile;
      if (next_in_tile) bcast_band<C>(bc, c.rank, c.tid);
      group_sync<C::G>();
    }
  }
}

// ----------------------------------------------------------------------------
// batched apply
// ----------------------------------------------------------------------------

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1) apply_kernel(const ApplyArgs P) {
  extern __shared__ __align__(16) double smem[];
  double* Vt = smem;
  double* gens = Vt + C::VT;
  Ctx<C> c;
  c.tid = threadIdx.x;
  c.lane = c.tid & 31;
  c.warp = c.tid >> 5;
  c.gq = c.lane >> 2;
  c.tig = c.lane & 3;
  c.rank = 0;
  constexpr int wcols = C::CC / C::WC;
  c.urow = (c.warp / wcols) * C::WR;
  c.ucol = (c.warp % wcols) * C::WC;
  const int nx = P.nx, ny = P.ny;
  for (int i = c.tid; i < C::VT; i += C::THREADS) Vt[i] = 0.0;
  for (int i = c.tid; i < 6 * C::GL; i += C::THREADS) gens[i] = P.gens[i];
  __syncthreads();
  const int b = blockIdx.x;
  load_vec<C>(Vt, P.v + (int64_t)b * P.v_stride, nx, ny, c);
  __syncthreads();
  double acc[C::WR][C::NF][4];
  const bool dox = P.which == 0 || P.which == 2;
  const bool doy = P.which == 0 || P.which == 3;
  if (dox || doy)
    matvec<C>(Vt, gens, acc, c.urow, c.ucol, c.gq, c.tig, (nx + 3) & ~3, (ny + 3) & ~3, dox, doy, P.merge);
  double sc = 0.0;
  if (P.which == 0) sc = P.sign * 0.5 * P.dt[b];
  if (P.which == 2) sc = 1.0 / P.kx;
  if (P.which == 3) sc = 1.0 / P.ky;
  double* out = P.out + (int64_t)b * P.out_stride;
  RM_FOR_ELEM {
    const int j = elem_row<C>(c, mr, e), i = elem_col<C>(c, nf, e);
    if (j < ny && i < nx) {
      double y;
      if (P.which == 1)
        y = mass_stencil<C>(Vt, j, i, P.cm);
      else if (P.which == 0)
        y = mass_stencil<C>(Vt, j, i, P.cm) + sc * acc[mr][nf][e];
      else
        y = sc * acc[mr][nf][e];
      out[j * nx + i] = y;
    }
  }
}

// ----------------------------------------------------------------------------
// PCG64 (numpy default_rng bit generator: 128-bit LCG + XSL-RR output)
// ----------------------------------------------------------------------------

typedef unsigned __int128 u128;

__device__ __forceinline__ void lcg_jump(u128 mult, u128 plus, uint64_t delta, u128& am, u128& ap) {
  u128 acc_m = 1, acc_p = 0;
  while (delta) {
    if (delta & 1) {
      acc_m *= mult;
      acc_p = acc_p * mult + plus;
    }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  am = acc_m;
  ap = acc_p;
}

#ifndef RM_CASE_NP  // per-case translation units hold only their chain kernel instantiation
__global__ void pcg64_kernel(PcgArgs P) {
  const u128 MULT = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
  const u128 inc = ((u128)P.inc_hi << 64) | P.inc_lo;
  const u128 s0 = ((u128)P.state_hi << 64) | P.state_lo;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.count) return;
  u128 am, ap;
  // state after (start + t + 1) steps is the one whose output is draw (start + t)
  lcg_jump(MULT, inc, (uint64_t)(P.start + t + 1), am, ap);
  u128 s = am * s0 + ap;
  u128 jm, jp;
  lcg_jump(MULT, inc, (uint64_t)T, jm, jp);
  for (int64_t i = t; i < P.count; i += T) {
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const uint64_t x = hi ^ lo;
    const unsigned rot = (unsigned)(s >> 122);
    const uint64_t o = (x >> rot) | (x << ((64u - rot) & 63u));
    const double d = (double)(o >> 11) * (1.0 / 9007199254740992.0);
    P.out[(i / P.row) * P.out_stride + (i % P.row)] = d;
    s = jm * s + jp;
  }
}

// ----------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------

__global__ void correct_kernel(int ndof, int nc, int m, double* u, int64_t us, const double* uc, int64_t ucs) {
  const int64_t total = (int64_t)(nc + 1) * ndof;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / ndof, i = t % ndof;
    u[k * m * us + i] += uc[k * ucs + i];
  }
}

__global__ void diff_sqnorm_kernel(int64_t n, const double* a, const double* b, double* out) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  s = warp_allsum(s);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    x = warp_allsum(x);
    if (threadIdx.x == 0) out[0] = x;
  }
}

// dot product a . b into out[0]: one CTA, fixed summation order (generic-operator CG, krylov.py:57-66)
__global__ void vec_dot_kernel(int64_t n, const double* a, const double* b, double* out) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i], b[i], s);
  s = warp_allsum(s);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
    x = warp_allsum(x);
    if (threadIdx.x == 0) out[0] = x;
  }
}

// out = alpha x + beta y (out may alias x or y)
__global__ void vec_axpby_kernel(int64_t n, double alpha, const double* x, double beta, const double* y, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = alpha * x[i] + beta * y[i];
}

#endif

// ----------------------------------------------------------------------------
// launch helpers (instantiations)
// ----------------------------------------------------------------------------

template <int NP, int G>
cudaError_t launch_chain_t(const ChainArgs& a, int max_clusters, cudaStream_t st) {
  using C = Cfg<NP, G>;
  auto kern = a.sw.precond ? chain_kernel<C, true> : chain_kernel<C, false>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (err != cudaSuccess) return err;
  if (G > 8) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
  }
  int ncl = max_clusters;
  if (ncl > a.sw.nchains) ncl = a.sw.nchains;
  if (ncl < 1) ncl = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * G);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int NP, int G>
cudaError_t max_clusters_t(int* out) {
  using C = Cfg<NP, G>;
  auto kern = chain_kernel<C, true>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (err != cudaSuccess) return err;
  if (G > 8) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, kern, &cfg);
}

#define RM_CHAIN_CASES(X) \
  X(16, 1)                \
  X(32, 1)                \
  X(32, 2)                \
  X(64, 1)                \
  X(64, 2)                \
  X(64, 4)                \
  X(128, 2)               \
  X(128, 4)               \
  X(128, 8)               \
  X(128, 16)

#ifdef RM_CASE_NP
// build.py compiles this file once per (NP, G) case with -DRM_CASE_NP/-DRM_CASE_G (parallel nvcc jobs)
template cudaError_t launch_chain_t<RM_CASE_NP, RM_CASE_G>(const ChainArgs&, int, cudaStream_t);
template cudaError_t max_clusters_t<RM_CASE_NP, RM_CASE_G>(int*);
#else
#define X(A, B)                                                                              \
  extern template cudaError_t launch_chain_t<A, B>(const ChainArgs&, int, cudaStream_t); \
  extern template cudaError_t max_clusters_t<A, B>(int*);
RM_CHAIN_CASES(X)
#undef X

bool chain_supported(int np, int g) {
#define X(a, b) \
  if (np == a && g == b) return true;
  RM_CHAIN_CASES(X)
#undef X
  return false;
}

cudaError_t launch_chain(int np, int g, const ChainArgs& a, int max_clusters, cudaStream_t st) {
#define X(A, B) \
  if (np == A && g == B) return launch_chain_t<A, B>(a, max_clusters, st);
  RM_CHAIN_CASES(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t chain_max_clusters(int np, int g, int* out) {
#define X(A, B) \
  if (np == A && g == B) return max_clusters_t<A, B>(out);
  RM_CHAIN_CASES(X)
#undef X
  return cudaErrorInvalidValue;
}

size_t chain_smem(int np, int g) {
#define X(A, B) \
  if (np == A && g == B) return Cfg<A, B>::SMEM;
  RM_CHAIN_CASES(X)
#undef X
  return 0;
}

template <int NP>
static cudaError_t launch_apply_t(const ApplyArgs& a, int batch, cudaStream_t st) {
  using C = Cfg<NP, 1>;
  auto kern = apply_kernel<C>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::APPLY_SMEM);
  if (err != cudaSuccess) return err;
  kern<<<batch, C::THREADS, C::APPLY_SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_apply(int np, const ApplyArgs& a, int batch, cudaStream_t st) {
  switch (np) {
    case 16: return launch_apply_t<16>(a, batch, st);
    case 32: return launch_apply_t<32>(a, batch, st);
    case 64: return launch_apply_t<64>(a, batch, st);
    case 128: return launch_apply_t<128>(a, batch, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pcg64(const PcgArgs& a, cudaStream_t st) {
  int64_t threads = 256;
  int64_t blocks = (a.count + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  pcg64_kernel<<<(unsigned)blocks, (unsigned)threads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_correct(int ndof, int nc, int m, double* u, int64_t us, const double* uc, int64_t ucs,
                           cudaStream_t st) {
  const int64_t total = (int64_t)(nc + 1) * ndof;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  correct_kernel<<<(unsigned)blocks, 256, 0, st>>>(ndof, nc, m, u, us, uc, ucs);
  return cudaGetLastError();
}

cudaError_t launch_diff_sqnorm(int64_t n, const double* a, const double* b, double* out, cudaStream_t st) {
  diff_sqnorm_kernel<<<1, 1024, 0, st>>>(n, a, b, out);
  return cudaGetLastError();
}

cudaError_t launch_vec_dot(int64_t n, const double* a, const double* b, double* out, cudaStream_t st) {
  vec_dot_kernel<<<1, 1024, 0, st>>>(n, a, b, out);
  return cudaGetLastError();
}

cudaError_t launch_vec_axpby(int64_t n, double alpha, const double* x, double beta, const double* y, double* out,
                             cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  vec_axpby_kernel<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), threads, 0, st>>>(n, alpha, x, beta, y, out);
  return cudaGetLastError();
}

#endif  // RM_CASE_NP

}  // namespace rm
