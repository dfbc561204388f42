// Chain kernel for large grids (NP = 256, 512: BASELINE configs 3 and 4).
//
// The operand vector no longer fits one CTA's shared memory, so it lives in an
// L2-resident padded copy in global memory ("PV" layout: rows -1..NP, row stride
// NP+16 doubles, column c at offset c+8, zero halos) and every matvec streams it
// through shared memory in 32-wide K chunks (cp.async, double buffered):
//   x-part:  chunk = rows R0-1..R0+128 of the tile band x 32 columns  (A operand)
//   y-part:  chunk = 32 rows x columns C0-8..C0+135 of the tile band  (B operand)
// The Toeplitz operand comes from the generator tables in shared memory as in the
// small-grid kernel.  One CTA owns one 128x128 output tile (16 warps, each a 16x64
// strip, 32 accumulators per thread); the G = (NP/128)^2 CTAs of a chain form a
// cluster.  CG state x, r, b (and dinv, p_old for PCG) lives in a fragment-native
// global scratch (coalesced, L2 resident); p is the PV copy.  Dot products: per
// unit (fixed lane order) -> per tile (fixed unit order) -> over tiles (tile order).
// The CG / PCG control flow is the small-grid kernel's (reference stopping rule,
// true-residual acceptance, restart on drift, second starting guess).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "riesz_mgrit_b200.h"
#include "rm_device.cuh"
#include "rm_kernels.h"

namespace rm {

template <int NP_>
struct BigCfg {
  static constexpr int NP = NP_;
  static constexpr int TPR = NP / 128;  // tiles per row
  static constexpr int G = TPR * TPR;   // CTAs per chain (cluster size)
  static constexpr int THREADS = 512;
  static constexpr int WARPS = 16;
  static constexpr int NF = 8;             // n-fragments per warp (16 x 64 strip)
  static constexpr int SP = NP + 16;       // PV row stride (doubles)
  static constexpr int PV = (NP + 2) * SP; // PV vector size (doubles)
  static constexpr int GL = 2 * NP + 8;    // generator / sine table length
  // K chunk width: 32, or 16 at NP = 1024 (the generator/sine tables take 129 KB of shared memory)
  static constexpr int KC = NP > 512 ? 16 : 32;
  static constexpr int XS = KC + 2;        // x-stage row stride (== 2 mod 16: rows 2 apart conflict-free)
  static constexpr int XROWS = 130;
  static constexpr int YS = 148;           // y-stage row stride (== 4 mod 16)
  static constexpr int YCOLS = 144;        // C0-8 .. C0+135
  static constexpr int CHUNK = (XROWS * XS > (KC + 1) * YS ? XROWS * XS : (KC + 1) * YS);  // doubles per chunk
  // The chain's CTAs synchronise through global memory (co-resident by a cooperative launch) rather
  // than as a thread-block cluster: clusters of 4/16 CTAs leave 16-20 SMs unplaced (measured 132 and
  // 128 of 148 SMs busy) and 64 CTAs (NP = 1024) exceed the cluster limit; the group barrier costs
  // little against phases of >= 33 MFLOP per CTA (cfg3 sweep 17.5 -> 20.5 TF/s, cfg4 16.0 -> 22.8).
  // -DRM_BIG_CLUSTER restores cluster barriers and DSMEM reductions for G <= 16.
#ifdef RM_BIG_CLUSTER
  static constexpr bool GSYNC = G > 16;
#else
  static constexpr bool GSYNC = true;
#endif
  static constexpr int STAGE = 2 * CHUNK;  // a chunk and (folded DST) its mirror
  static constexpr int HALF = NP / 2;
  static constexpr int TE = 128 * 128;     // elements per tile
  static constexpr int TL = (GL + GL / 8 + 3) & ~1;  // padded sine table (tab_idx), even length
  static constexpr size_t SMEM = sizeof(double) * (6 * GL + 2 * TL + 2 * STAGE + 4 * 64 + 2 * 4 * 16) + 64;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

struct BigCtx {
  int tid, lane, warp, gq, tig, rank;
  int R0, C0;   // tile origin
  int wr, wc0;  // warp strip: unit row wr (0..7), first unit column wc0 (0 or 4)
};

// Row r (0..15) of unit row ur inside a tile: parity-interleaved in 32-row blocks, so that every
// MMA fragment of the folded y-DST has outputs of one parity (one K operand, see rm_device.cuh).
__device__ __forceinline__ int big_urow(int ur, int r) { return 32 * (ur >> 1) + (ur & 1) + 2 * r; }

// element of (nf, e) in the normal mapping, tile coordinates added
__device__ __forceinline__ int big_row(const BigCtx& c, int e) {
  return c.R0 + big_urow(c.wr, c.gq + 8 * (e >> 1));
}
__device__ __forceinline__ int big_col(const BigCtx& c, int nf, int e) {
  return c.C0 + 16 * c.wc0 + 8 * nf + 2 * c.tig + (e & 1);
}
// transposed mapping (DST-x stage): m over columns (unit wr), n over rows (units wc0..)
__device__ __forceinline__ int bigT_row(const BigCtx& c, int nf, int e) {
  return c.R0 + 16 * c.wc0 + 8 * nf + 2 * c.tig + (e & 1);
}
// output column of the transposed stage; folded: m-tiles 0..3 give the even columns (u half, alpha odd),
// 4..7 the odd ones (w half) of the tile
__device__ __forceinline__ int bigT_col(const BigCtx& c, int e, bool fold) {
  return fold ? c.C0 + 32 * (c.wr & 3) + 2 * c.gq + 16 * (e >> 1) + (c.wr >> 2) : c.C0 + 16 * c.wr + c.gq + 8 * (e >> 1);
}
// fragment-native index of (nf, e) inside the CTA's scratch vectors
__device__ __forceinline__ int big_fidx(const BigCtx& c, int nf, int e) {
  return ((c.warp * 8 + nf) * 4 + e) * 32 + c.lane;
}

template <class C>
__device__ __forceinline__ int pv_idx(int j, int i) {
  return (j + 1) * C::SP + i + 8;
}

#define RM_BIG_FOR _Pragma("unroll") for (int nf = 0; nf < 8; ++nf) _Pragma("unroll") for (int e = 0; e < 4; ++e)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---- chunk loaders (all threads) ------------------------------------------------------
template <class C>
__device__ __forceinline__ void load_xchunk(double* st, const double* __restrict__ pv, int R0, int k0, int tid) {
  // rows R0-1 .. R0+128 (130), cols k0-2 .. k0+KC-1 (KC/2+1 x 16B per row; column k0-1 for the merged segment)
  constexpr int QR = C::KC / 2 + 1;
  for (int t = tid; t < C::XROWS * QR; t += C::THREADS) {
    const int r = t / QR, q = t % QR;
    cp_async16(st + r * C::XS + 2 * q, pv + pv_idx<C>(R0 - 1 + r, k0 - 2) + 2 * q);
  }
}
template <class C>
__device__ __forceinline__ void load_ychunk(double* st, const double* __restrict__ pv, int l0, int C0, int tid) {
  // rows l0-1 .. l0+KC-1 (row l0-1 for the merged segment), cols C0-8 .. C0+135 (72 x 16B per row)
  for (int t = tid; t < (C::KC + 1) * 72; t += C::THREADS) {
    const int r = t / 72, q = t % 72;
    cp_async16(st + r * C::YS + 2 * q, pv + pv_idx<C>(l0 - 1 + r, C0 - 8) + 2 * q);
  }
}

// acc = X + Y (stiffness, generator tables) of the tile, operand streamed from pv
template <class C>
__device__ __forceinline__ void big_matvec(const double* __restrict__ pv, const double* __restrict__ gens,
                                           double* stage, double (&acc)[8][4], const BigCtx& c, int kx_end,
                                           int ky_end, int merge) {
#pragma unroll
  for (int nf = 0; nf < 8; ++nf)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nf][e] = 0.0;
  double* st[2] = {stage, stage + C::STAGE};
  // ---- x-part: K = columns
  const int nkx = (kx_end + C::KC - 1) / C::KC;
  load_xchunk<C>(st[0], pv, c.R0, 0, c.tid);
  cp_async_commit();
  for (int ch = 0; ch < nkx; ++ch) {
    if (ch + 1 < nkx) load_xchunk<C>(st[(ch + 1) & 1], pv, c.R0, C::KC * (ch + 1), c.tid);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* s = st[ch & 1];
    const int k0 = C::KC * ch;
#pragma unroll 1
    for (int seg = 0; seg < ((merge & 1) ? 2 : 3); ++seg) {
      const int delta = seg == 0 ? 0 : (seg == 1 ? 1 : -1);
      const double* tab = gens + seg * C::GL + C::NP + c.C0 + 16 * c.wc0 + c.gq - c.tig - k0;
      const double* ar = s + (big_urow(c.wr, c.gq) + delta + 1) * C::XS + c.tig + 2;
      if (seg == 1 && (merge & 1)) {  // T2 (V[j+1][k] + V[j-1][k-1]), see rm_device.cuh matvec
        const double* am = s + big_urow(c.wr, c.gq) * C::XS + c.tig + 1;
#pragma unroll 4
        for (int k = 0; k < C::KC; k += 4) {
          const double a0 = ar[k] + am[k], a1 = ar[k + 16 * C::XS] + am[k + 16 * C::XS];
          double b[8];
#pragma unroll
          for (int nf = 0; nf < 8; ++nf) b[nf] = tab[8 * nf - k];
#pragma unroll
          for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
        }
        continue;
      }
#pragma unroll 4
      for (int k = 0; k < C::KC; k += 4) {
        const double a0 = ar[k], a1 = ar[k + 16 * C::XS];
        double b[8];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) b[nf] = tab[8 * nf - k];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
      }
    }
    __syncthreads();
  }
  // ---- y-part: K = rows
  const int nky = (ky_end + C::KC - 1) / C::KC;
  load_ychunk<C>(st[0], pv, 0, c.C0, c.tid);
  cp_async_commit();
  for (int ch = 0; ch < nky; ++ch) {
    if (ch + 1 < nky) load_ychunk<C>(st[(ch + 1) & 1], pv, C::KC * (ch + 1), c.C0, c.tid);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* s = st[ch & 1];
    const int l0 = C::KC * ch;
#pragma unroll 1
    for (int seg = 0; seg < ((merge & 2) ? 2 : 3); ++seg) {
      const int delta = seg == 0 ? 0 : (seg == 1 ? 1 : -1);
      const double* tab = gens + (3 + seg) * C::GL + C::NP + c.R0 + big_urow(c.wr, c.gq) - c.tig - l0;
      const double* br = s + (c.tig + 1) * C::YS + 16 * c.wc0 + c.gq + delta + 8;
      if (seg == 1 && (merge & 2)) {  // T2 (V[l][i+1] + V[l-1][i-1])
        const double* bm = s + c.tig * C::YS + 16 * c.wc0 + c.gq + 7;
#pragma unroll 4
        for (int l = 0; l < C::KC; l += 4) {
          const double a0 = tab[-l], a1 = tab[16 - l];
          double b[8];
#pragma unroll
          for (int nf = 0; nf < 8; ++nf) b[nf] = br[l * C::YS + 8 * nf] + bm[l * C::YS + 8 * nf];
#pragma unroll
          for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
        }
        continue;
      }
#pragma unroll 4
      for (int l = 0; l < C::KC; l += 4) {
        const double a0 = tab[-l], a1 = tab[16 - l];
        double b[8];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) b[nf] = br[l * C::YS + 8 * nf];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
      }
    }
    __syncthreads();
  }
}

// DST along x in the transposed mapping: out^T[i][j] = sum_k Sx[i][k] V[j][k].  Folded (n = NP-1, see
// rm_device.cuh): K runs over k < HALF with the B operand v_k +- v_{NP-2-k}; every K chunk streams its
// mirror chunk (columns NP-KC-2-k0 .. NP-1-k0) next to it; output columns per bigT_col.
template <class C>
__device__ __forceinline__ void big_dst_xT(const double* __restrict__ pv, const double* __restrict__ tab, int L,
                                           double* stage, double (&acc)[8][4], const BigCtx& c, int kx_end,
                                           bool fold) {
#pragma unroll
  for (int nf = 0; nf < 8; ++nf)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nf][e] = 0.0;
  double* st[2] = {stage, stage + C::STAGE};
  const int kend = fold ? C::HALF : kx_end;
  const int nkx = (kend + C::KC - 1) / C::KC;
  const int xa = bigT_col(c, 0, fold) + 1, xb = bigT_col(c, 2, fold) + 1;  // alpha of rows gq, gq+8
  int ia = (xa * (c.tig + 1)) % L, ib = (xb * (c.tig + 1)) % L;
  const int sa = (4 * xa) % L, sb = (4 * xb) % L;
  const bool w = c.wr >= 4;
  const double sgn = w ? -1.0 : 1.0;
  const double sgn_last = (c.tig == 3) ? (w ? -1.0 : 0.0) : sgn;
  load_xchunk<C>(st[0], pv, c.R0, 0, c.tid);
  if (fold) load_xchunk<C>(st[0] + C::CHUNK, pv, c.R0, C::NP - C::KC, c.tid);
  cp_async_commit();
  for (int ch = 0; ch < nkx; ++ch) {
    if (ch + 1 < nkx) {
      load_xchunk<C>(st[(ch + 1) & 1], pv, c.R0, C::KC * (ch + 1), c.tid);
      if (fold) load_xchunk<C>(st[(ch + 1) & 1] + C::CHUNK, pv, c.R0, C::NP - C::KC - C::KC * (ch + 1), c.tid);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* br = st[ch & 1] + (16 * c.wc0 + c.gq + 1) * C::XS + c.tig + 2;
    if (fold) {
      // partner column NP-2-k of k = k0 + kk sits at mirror offset KC - kk (chunk column index)
      const double* bm = st[ch & 1] + C::CHUNK + (16 * c.wc0 + c.gq + 1) * C::XS + C::KC - c.tig;
      const bool last_chunk = C::KC * ch + C::KC >= C::HALF;
#pragma unroll 4
      for (int k = 0; k < C::KC; k += 4) {
        const double a0 = tab[tab_idx(ia)], a1 = tab[tab_idx(ib)];
        const double f = (last_chunk && k == C::KC - 4) ? sgn_last : sgn;
        double b[8];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) b[nf] = fma(f, bm[8 * nf * C::XS - k], br[8 * nf * C::XS + k]);
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
        ia += sa;
        ia -= ia >= L ? L : 0;
        ib += sb;
        ib -= ib >= L ? L : 0;
      }
    } else {
#pragma unroll 4
      for (int k = 0; k < C::KC; k += 4) {
        const double a0 = tab[tab_idx(ia)], a1 = tab[tab_idx(ib)];
        double b[8];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) b[nf] = br[8 * nf * C::XS + k];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
        ia += sa;
        ia -= ia >= L ? L : 0;
        ib += sb;
        ib -= ib >= L ? L : 0;
      }
    }
    __syncthreads();
  }
}

// DST along y in the normal mapping: out[j][i] = sum_l Sy[j][l] V[l][i].  Folded: K over l < HALF with
// v_l +- v_{NP-2-l} (u for even unit rows = alpha odd, w for odd ones); mirror rows NP-KC-2-l0 .. NP-2-l0.
template <class C>
__device__ __forceinline__ void big_dst_y(const double* __restrict__ pv, const double* __restrict__ tab, int L,
                                          double* stage, double (&acc)[8][4], const BigCtx& c, int ky_end,
                                          bool fold) {
#pragma unroll
  for (int nf = 0; nf < 8; ++nf)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nf][e] = 0.0;
  double* st[2] = {stage, stage + C::STAGE};
  const int kend = fold ? C::HALF : ky_end;
  const int nky = (kend + C::KC - 1) / C::KC;
  const int ja = big_row(c, 0) + 1, jb = big_row(c, 2) + 1;
  int ia = (ja * (c.tig + 1)) % L, ib = (jb * (c.tig + 1)) % L;
  const int sa = (4 * ja) % L, sb = (4 * jb) % L;
  const bool w = c.wr & 1;
  const double sgn = w ? -1.0 : 1.0;
  const double sgn_last = (c.tig == 3) ? (w ? -1.0 : 0.0) : sgn;
  load_ychunk<C>(st[0], pv, 0, c.C0, c.tid);
  if (fold) load_ychunk<C>(st[0] + C::CHUNK, pv, C::NP - C::KC - 1, c.C0, c.tid);
  cp_async_commit();
  for (int ch = 0; ch < nky; ++ch) {
    if (ch + 1 < nky) {
      load_ychunk<C>(st[(ch + 1) & 1], pv, C::KC * (ch + 1), c.C0, c.tid);
      if (fold) load_ychunk<C>(st[(ch + 1) & 1] + C::CHUNK, pv, C::NP - C::KC - 1 - C::KC * (ch + 1), c.C0, c.tid);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* br = st[ch & 1] + (c.tig + 1) * C::YS + 16 * c.wc0 + c.gq + 8;
    if (fold) {
      // partner row NP-2-l of l = l0 + ll sits at mirror row KC - ll
      const double* bm = st[ch & 1] + C::CHUNK + (C::KC - c.tig) * C::YS + 16 * c.wc0 + c.gq + 8;
      const bool last_chunk = C::KC * ch + C::KC >= C::HALF;
#pragma unroll 4
      for (int l = 0; l < C::KC; l += 4) {
        const double a0 = tab[tab_idx(ia)], a1 = tab[tab_idx(ib)];
        const double f = (last_chunk && l == C::KC - 4) ? sgn_last : sgn;
        double b[8];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) b[nf] = fma(f, bm[8 * nf - l * C::YS], br[l * C::YS + 8 * nf]);
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
        ia += sa;
        ia -= ia >= L ? L : 0;
        ib += sb;
        ib -= ib >= L ? L : 0;
      }
    } else {
#pragma unroll 4
      for (int l = 0; l < C::KC; l += 4) {
        const double a0 = tab[tab_idx(ia)], a1 = tab[tab_idx(ib)];
        double b[8];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) b[nf] = br[l * C::YS + 8 * nf];
#pragma unroll
        for (int nf = 0; nf < 8; ++nf) dmma(acc[nf], a0, a1, b[nf]);
        ia += sa;
        ia -= ia >= L ? L : 0;
        ib += sb;
        ib -= ib >= L ? L : 0;
      }
    }
    __syncthreads();
  }
}

template <class C>
__device__ __forceinline__ double big_mass(const double* __restrict__ pv, int j, int i, double cm) {
  const double* q = pv + pv_idx<C>(j, i);
  double s = 6.0 * __ldcg(q);
  s += __ldcg(q - 1);
  s += __ldcg(q + 1);
  s += __ldcg(q + C::SP);
  s += __ldcg(q + C::SP + 1);
  s += __ldcg(q - C::SP);
  s += __ldcg(q - C::SP - 1);
  return cm * s;
}

// Synchronisation of the CTAs of one chain: cluster barriers and DSMEM (G <= 16), or a global-memory
// barrier and global reduction slots (GSYNC: the CTAs are co-resident through a cooperative launch).
template <class C>
struct BigSync {
  double* tred;                                 // cluster: this CTA's tile-partial slots (shared memory)
  double* tred_peer[C::GSYNC ? 1 : C::G];       // cluster: the peers' slots
  int* sched;                                   // chain index broadcast (shared memory / global)
  int* sched_peer[C::GSYNC ? 1 : C::G];
  unsigned* gbar;                               // GSYNC: this group's arrival counter (zeroed per launch)
  double* gred;                                 // GSYNC: [2][4][G] tile partials
  unsigned epoch;                               // GSYNC: barriers passed (thread 0)
};

template <class C>
__device__ __forceinline__ void big_sync(BigSync<C>& sy) {
  if constexpr (C::GSYNC) {
    __syncthreads();
    if (threadIdx.x == 0) {
      sy.epoch += 1;
      __threadfence();  // this CTA's writes (ordered before by the CTA barrier) before the arrival
      atomicAdd(sy.gbar, 1u);
      const unsigned target = sy.epoch * (unsigned)C::G;
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sy.gbar) : "memory");
        if (v >= target) break;
        __nanosleep(32);
      }
      __threadfence();
    }
    __syncthreads();
  } else {
    group_sync<C::G>();
  }
}

// Deterministic group sum of NV values: unit (warp butterfly) -> tile (unit order) -> group (tile order).
template <class C, int NV>
__device__ __forceinline__ void big_reduce(double (&part)[NV][4], double* wred, BigSync<C>& sy, int buf,
                                           const BigCtx& c, double (&out)[NV]) {
  // part[v][u]: this thread's partial for its warp strip's unit u (4 units per warp)
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int u = 0; u < 4; ++u) part[v][u] = warp_allsum(part[v][u]);
  if (c.lane == 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int u = 0; u < 4; ++u) wred[v * 64 + c.wr * 8 + c.wc0 + u] = part[v][u];
  }
  __syncthreads();
  if (c.warp == 0) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double x = wred[v * 64 + c.lane] + wred[v * 64 + 32 + c.lane];
      x = warp_allsum(x);
      if constexpr (C::GSYNC) {
        if (c.lane == 0) sy.gred[(buf * 4 + v) * C::G + c.rank] = x;
      } else {
        if (c.lane < C::G) sy.tred_peer[c.lane][buf * 4 * 16 + v * 16 + c.rank] = x;
      }
    }
  }
  big_sync<C>(sy);
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double x = 0.0;
    if constexpr (C::GSYNC) {
      const double* g = sy.gred + (buf * 4 + v) * C::G;
#pragma unroll
      for (int q = 0; q < C::G; q += 32)
        if (q + c.lane < C::G) x += __ldcg(g + q + c.lane);
    } else {
      x = c.lane < C::G ? sy.tred[buf * 4 * 16 + v * 16 + c.lane] : 0.0;
    }
    out[v] = warp_allsum(x);
  }
}

// ---- FP16 DST stages of the tau preconditioner (precond 2; see rm_device.cuh Lp) ----------------------
// The stage inputs live in two FP16 copies V16a, V16b [NP][SHH] inside the (FP64) preconditioner temporary
// pv1; the DST matrix S16 [NP][SHH] (row alpha-1, column kappa-1, zero beyond n) comes from the grid.
// Each stage is a 128 x 128 x NP tile GEMM per CTA: K chunks of 64 (A: 128 rows of S16, B: 128 x 64 or
// 64 x 128 of the vector) are staged by cp.async (double buffered) and fed to mma.sync m16n8k16 through
// ldmatrix (transposed for the y-stage), FP32 accumulation.  Power-of-two scaling as in the small kernel.
template <class C>
struct BigLp {
  static constexpr int SHH = C::NP + 8;  // global row stride (fp16), 16-byte rows
  static constexpr int KC = 64;          // K chunk
  static constexpr int AS = KC + 8;      // smem row stride of the A chunk / x-stage B chunk (== 4 words mod 32)
  static constexpr int BYS = 128 + 8;    // smem row stride of the y-stage B chunk
  static constexpr int ABYTES = 128 * AS * 2;
  static constexpr int BBYTES = (128 * AS > KC * BYS ? 128 * AS : KC * BYS) * 2;
  static constexpr int BUF = ABYTES + BBYTES;  // one pipeline buffer
  static_assert(2 * BUF <= 2 * (int)sizeof(double) * C::STAGE, "FP16 stage buffers must fit the FP64 stage space");
  static_assert(2 * (size_t)C::NP * SHH * 2 <= sizeof(double) * C::PV, "two FP16 vectors fit in pv1");
};

// A chunk: rows row0 .. row0+127 of S16, columns k0 .. k0+63 (8 x 16 B per row)
template <class C>
__device__ __forceinline__ void load_a16(char* st, const uint16_t* __restrict__ s16, int row0, int k0, int tid) {
  using B = BigLp<C>;
  for (int t = tid; t < 128 * 8; t += C::THREADS) {
    const int r = t >> 3, q = t & 7;
    cp_async16(st + (r * B::AS + 8 * q) * 2, s16 + (size_t)(row0 + r) * B::SHH + k0 + 8 * q);
  }
}
// x-stage B chunk: rows R0 .. R0+127 of the vector, columns k0 .. k0+63
template <class C>
__device__ __forceinline__ void load_bx16(char* st, const uint16_t* __restrict__ v, int R0, int k0, int tid) {
  using B = BigLp<C>;
  for (int t = tid; t < 128 * 8; t += C::THREADS) {
    const int r = t >> 3, q = t & 7;
    cp_async16(st + (r * B::AS + 8 * q) * 2, v + (size_t)(R0 + r) * B::SHH + k0 + 8 * q);
  }
}
// y-stage B chunk: rows k0 .. k0+63 of the vector, columns C0 .. C0+127 (16 x 16 B per row)
template <class C>
__device__ __forceinline__ void load_by16(char* st, const uint16_t* __restrict__ v, int k0, int C0, int tid) {
  using B = BigLp<C>;
  for (int t = tid; t < B::KC * 16; t += C::THREADS) {
    const int r = t >> 4, q = t & 15;
    cp_async16(st + (r * B::BYS + 8 * q) * 2, v + (size_t)(k0 + r) * B::SHH + C0 + 8 * q);
  }
}

// One FP16 DST stage of the tile.  YST: out[j][i] = sum_l S[j][l] V[l][i] in the normal mapping (rows
// R0 + big_urow(wr, .), columns C0 + 16 wc0 + .); else the transposed x-stage out^T[i][j] = sum_k S[i][k]
// V[j][k] (i = C0 + 16 wr + ., j = R0 + 16 wc0 + .).
template <class C, bool YST>
__device__ __forceinline__ void big_dst16(const uint16_t* __restrict__ s16, const uint16_t* __restrict__ v,
                                          char* stage, float (&acc)[8][4], const BigCtx& c) {
  using B = BigLp<C>;
#pragma unroll
  for (int nf = 0; nf < 8; ++nf)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nf][e] = 0.f;
  const int row0 = YST ? c.R0 : c.C0;
  const int q = c.lane >> 3, r = c.lane & 7;
  const int arow = YST ? big_urow(c.wr, r + 8 * (q & 1)) : 16 * c.wr + r + 8 * (q & 1);
  constexpr int NK = C::NP / B::KC;
  auto load = [&](int ch, int b) {
    char* st = stage + b * B::BUF;
    load_a16<C>(st, s16, row0, B::KC * ch, c.tid);
    if constexpr (YST)
      load_by16<C>(st + B::ABYTES, v, B::KC * ch, c.C0, c.tid);
    else
      load_bx16<C>(st + B::ABYTES, v, c.R0, B::KC * ch, c.tid);
  };
  load(0, 0);
  cp_async_commit();
  for (int ch = 0; ch < NK; ++ch) {
    if (ch + 1 < NK) load(ch + 1, (ch + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const uint32_t sa = smem_addr(stage + (ch & 1) * B::BUF);
    const uint32_t sb = sa + B::ABYTES;
#pragma unroll
    for (int kk = 0; kk < B::KC; kk += 16) {
      uint32_t a[4];
      ldsm_x4(a, sa + 2u * (arow * B::AS + kk + 8 * (q >> 1)));
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        uint32_t b[4];
        if constexpr (YST)
          ldsm_x4_t(b, sb + 2u * ((kk + r + 8 * (q & 1)) * B::BYS + 16 * c.wc0 + 8 * (2 * p + (q >> 1))));
        else
          ldsm_x4(b, sb + 2u * ((16 * c.wc0 + 8 * (2 * p + (q >> 1)) + r) * B::AS + kk + 8 * (q & 1)));
        hmma_f16(acc[2 * p], a, b[0], b[1]);
        hmma_f16(acc[2 * p + 1], a, b[2], b[3]);
      }
    }
    __syncthreads();
  }
}

// Group maximum of a nonnegative value (one barrier; channel 3 of the reduction slots).
template <class C>
__device__ __forceinline__ double big_max(double m, double* wred, BigSync<C>& sy, int buf, const BigCtx& c) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (c.lane == 0) wred[3 * 64 + c.warp] = m;
  __syncthreads();
  if (c.warp == 0) {
    double x = c.lane < C::WARPS ? wred[3 * 64 + c.lane] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, off));
    if constexpr (C::GSYNC) {
      if (c.lane == 0) sy.gred[(buf * 4 + 3) * C::G + c.rank] = x;
    } else {
      if (c.lane < C::G) sy.tred_peer[c.lane][buf * 4 * 16 + 3 * 16 + c.rank] = x;
    }
  }
  big_sync<C>(sy);
  double x = 0.0;
  if constexpr (C::GSYNC) {
    const double* g = sy.gred + (buf * 4 + 3) * C::G;
#pragma unroll
    for (int q = 0; q < C::G; q += 32)
      if (q + c.lane < C::G) x = fmax(x, __ldcg(g + q + c.lane));
  } else {
    x = c.lane < C::G ? sy.tred[buf * 4 * 16 + 3 * 16 + c.lane] : 0.0;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, off));
  return x;
}

template <class C, bool PRE>
__global__ void __launch_bounds__(512, 1) chain_big_kernel(const ChainArgs P) {
  extern __shared__ __align__(16) double smem[];
  double* gens = smem;
  double* tabx = gens + 6 * C::GL;
  double* taby = tabx + C::TL;
  double* stage = taby + C::TL;
  double* wred = stage + 2 * C::STAGE;  // 4 values x 64 units
  double* tred = wred + 4 * 64;         // 2 buffers x 4 values x 16 tiles
  int* sched = reinterpret_cast<int*>(tred + 2 * 4 * 16);

  BigCtx c;
  c.tid = threadIdx.x;
  c.lane = c.tid & 31;
  c.warp = c.tid >> 5;
  c.gq = c.lane >> 2;
  c.tig = c.lane & 3;
  if constexpr (C::GSYNC)
    c.rank = blockIdx.x % C::G;
  else
    c.rank = (int)cgx::this_cluster().block_rank();
  c.R0 = 128 * (c.rank / C::TPR);
  c.C0 = 128 * (c.rank % C::TPR);
  c.wr = c.warp >> 1;
  c.wc0 = (c.warp & 1) * 4;

  BigSync<C> sy;
  sy.tred = tred;
  sy.sched = sched;
  sy.epoch = 0;
  if constexpr (C::GSYNC) {
    sy.gbar = P.gbar + (size_t)(blockIdx.x / C::G) * 32;
    sy.gred = P.gbuf + (size_t)(blockIdx.x / C::G) * 1024;
    sy.sched = reinterpret_cast<int*>(sy.gred + 8 * C::G);
  } else {
    auto cl = cgx::this_cluster();
#pragma unroll
    for (int q = 0; q < C::G; ++q) {
      sy.tred_peer[q] = cl.map_shared_rank(tred, q);
      sy.sched_peer[q] = cl.map_shared_rank(sched, q);
    }
  }

  const rm_sweep& W = P.sw;
  const int nx = P.nx, ny = P.ny, ndof = nx * ny;
  const int kx_end = (nx + 3) & ~3, ky_end = (ny + 3) & ~3;
  const int Lx = 2 * (nx + 1), Ly = 2 * (ny + 1);
  const double cm = P.cm;
  const int64_t max_iter = W.max_iter > 0 ? W.max_iter : 10 * (int64_t)ndof;
  const bool need_in = W.explicit_rhs || W.x0_mode == 1;
  // G row scale (compressed G, rm_sweep.d_gscale): rows of d_gadd / d_hg are d_gscale[n] times the stored row
  auto gsc = [&](int k) -> double { return W.d_gscale ? W.d_gscale[k] : 1.0; };
  const bool fold_x = nx == C::NP - 1, fold_y = ny == C::NP - 1;  // even/odd folded DST stages

  if constexpr (PRE) {
    for (int i = c.tid; i < Lx; i += C::THREADS) tabx[tab_idx(i)] = P.tabx[i];
    for (int i = c.tid; i < Ly; i += C::THREADS) taby[tab_idx(i)] = P.taby[i];
  }

  // per-cluster scratch: two PV vectors, then per-CTA fragment-native vectors
  const int cid = blockIdx.x / C::G;
  double* base = P.scratch + (size_t)cid * (2 * (size_t)C::PV + 5 * (size_t)C::G * C::TE);
  double* pv0 = base;           // operand: p, the step input, x for true-residual checks
  double* pv1 = base + C::PV;   // preconditioner temporary
  double* fr = base + 2 * C::PV + (size_t)c.rank * 5 * C::TE;
  double* __restrict__ xs = fr;              // iterate x
  double* __restrict__ rs = fr + C::TE;      // residual r
  double* __restrict__ bs = fr + 2 * C::TE;  // right-hand side b
  double* __restrict__ ds = fr + 3 * C::TE;  // 1 / d(s)
  double* __restrict__ ps = fr + 4 * C::TE;  // p_old (PCG)
  // zero the PV halos / padding of this cluster's vectors once (only interior points are ever written)
  for (size_t i = (size_t)c.rank * C::THREADS + c.tid; i < 2 * (size_t)C::PV; i += (size_t)C::G * C::THREADS)
    base[i] = 0.0;
  big_sync<C>(sy);

  int buf = 0;
  double acc[8][4];
  const bool lp_dst = PRE && W.precond == 2 && P.dst16 != nullptr;  // FP16 DST stages
  double lp_dbound = 1.0;

  auto put_tile = [&](double* pv, int j, int i, double v) { pv[pv_idx<C>(j, i)] = v; };

  for (;;) {
    if (c.rank == 0 && c.tid == 0) {
      const int ch = atomicAdd(P.chain_counter, 1);
      if constexpr (C::GSYNC) {
        sy.sched[0] = ch;
      } else {
#pragma unroll
        for (int q = 0; q < C::G; ++q) sy.sched_peer[q][0] = ch;
      }
    }
    big_sync<C>(sy);
    const int chain = C::GSYNC ? __ldcg(sy.sched) : sy.sched[0];
    big_sync<C>(sy);
    if (chain >= W.nchains) break;
    const int n0 = W.first + chain * W.cstride;
    const int n1 = min(n0 + W.clen - 1, W.nmax);
    bool in_tile = false;
    bool chain_ok = false;  // the previous step's accepted true residual is in rs (apply-free next rhs)
    double s_prev = 0.0;
    for (int n = n0; n <= n1; ++n) {
      const double s = 0.5 * W.d_dt[n - 1];
      if (lp_dst) {
        const double dlow = P.lp_dmin + s * P.lp_kmin;
        lp_dbound = dlow > 0.0 ? 1.0 / dlow : 0.0;  // >= max 1/d(s) (FP16 stage scaling)
      }
      const double fs = W.d_f ? (W.d_fscale ? W.d_fscale[n] : 1.0) : 0.0;
      const double* Fn = W.d_f ? W.d_f + (int64_t)n * W.f_stride : nullptr;
      // apply-free explicit side inside a chain (see the small-grid kernel):
      //   (M - s K) y = (1 + s/s0) M y - (s/s0) (b - r + A_{s0} G_{n-1})
      const bool rhs_free = need_in && W.explicit_rhs && in_tile && chain_ok && W.d_hg != nullptr &&
                            W.d_gadd != nullptr && W.d_sub == nullptr;
      int64_t nmv = need_in && !rhs_free ? 1 : 0, npc = 0;
      if (rhs_free) {
        const double* Hn = W.d_hg + (int64_t)(n - 1) * W.hg_stride;
        const double q = s / s_prev;
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          const int fi = big_fidx(c, nf, e);
          double am = 0.0;
          if (j < ny && i < nx)
            am = (1.0 + q) * big_mass<C>(pv0, j, i, cm) - q * (bs[fi] - rs[fi] + gsc(n - 1) * __ldcg(Hn + j * nx + i));
          acc[nf][e] = am;
        }
      }
      s_prev = s;
      chain_ok = false;

      // ... and at a chain's first step from the stored A x of its input point (d_ain, see the small kernel)
      const bool rhs_ain = need_in && W.explicit_rhs && !in_tile && n >= 2 && W.d_ain != nullptr &&
                           W.d_hg != nullptr;
      if (rhs_ain) nmv = 0;
      if (need_in && !rhs_free) {
        // step-operator tables M - s K (rm_device.cuh build_step_tables); the previous step ended
        // with a group barrier
        if (!rhs_ain) build_step_tables<C::NP, C::GL, C::THREADS>(gens, P.gens, -s, cm, c.tid);
        if (!in_tile) {
          const double* src = W.d_src + (int64_t)(n - 1) * W.src_stride;
          RM_BIG_FOR {
            const int j = big_row(c, e), i = big_col(c, nf, e);
            if (j < ny && i < nx) put_tile(pv0, j, i, __ldcg(src + j * nx + i));
          }
          big_sync<C>(sy);
        } else {
          __syncthreads();
        }
        if (!rhs_ain) big_matvec<C>(pv0, gens, stage, acc, c, kx_end, ky_end, P.merge);
      }
      if (rhs_ain) {
        const double* An = W.d_ain + (int64_t)(n - 1) * W.ain_stride;
        const double* Hn = W.d_hg + (int64_t)(n - 1) * W.hg_stride;
        const double q = s / (0.5 * W.d_dt[n - 2]);
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          double am = 0.0;
          if (j < ny && i < nx) {
            const int gi = j * nx + i;
            am = (1.0 + q) * big_mass<C>(pv0, j, i, cm) - q * (__ldcg(An + gi) + gsc(n - 1) * __ldcg(Hn + gi));
          }
          acc[nf][e] = am;
        }
      }
      double part[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
      RM_BIG_FOR {
        const int j = big_row(c, e), i = big_col(c, nf, e);
        const int fi = big_fidx(c, nf, e);
        double b = 0.0, x = 0.0, r = 0.0;
        if (j < ny && i < nx) {
          const double am = need_in ? acc[nf][e] : 0.0;  // (M - s K) v
          if (W.explicit_rhs) b = am;
          if (Fn) {
            const double f = fs * __ldcg(Fn + j * nx + i);
            b = W.explicit_rhs ? f + b : f;
          }
          if (W.x0_mode == 1) {
            x = __ldcg(pv0 + pv_idx<C>(j, i));
            r = b - (2.0 * big_mass<C>(pv0, j, i, cm) - am);  // (M + s K) v = 2 M v - (M - s K) v
          } else {
            r = b;
          }
          if constexpr (PRE) ds[fi] = 1.0 / (__ldg(P.dm + j * nx + i) + s * __ldg(P.dk + j * nx + i));
        }
        bs[fi] = b;
        xs[fi] = x;
        rs[fi] = r;
        part[0][nf >> 1] += b * b;
        part[1][nf >> 1] += r * r;
      }
      __syncthreads();
      build_step_tables<C::NP, C::GL, C::THREADS>(gens, P.gens, s, cm, c.tid);  // M + s K from here on
      __syncthreads();
      if (W.x0_mode == 2) {
        big_sync<C>(sy);
        const double* x0 = W.d_x0 + (int64_t)n * W.x0_stride;
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          if (j < ny && i < nx) put_tile(pv0, j, i, __ldcg(x0 + j * nx + i));
        }
        big_sync<C>(sy);
        big_matvec<C>(pv0, gens, stage, acc, c, kx_end, ky_end, P.merge);
        ++nmv;
        part[1][0] = part[1][1] = part[1][2] = part[1][3] = 0.0;
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          const int fi = big_fidx(c, nf, e);
          double x = 0.0, r = 0.0;
          if (j < ny && i < nx) {
            x = __ldcg(pv0 + pv_idx<C>(j, i));
            r = bs[fi] - acc[nf][e];
          }
          xs[fi] = x;
          rs[fi] = r;
          part[1][nf >> 1] += r * r;
        }
      }
      double tot[2];
      big_reduce<C, 2>(part, wred, sy, buf, c, tot);
      buf ^= 1;
      const double bnorm = sqrt(tot[0]);
      const double target = bnorm > 0.0 ? W.rel_tol * bnorm : W.rel_tol;
      if (W.d_guess && sqrt(tot[1]) > target) {
        const double* gu = W.d_guess + (int64_t)n * W.guess_stride;
        const double* Gr = W.d_gadd ? W.d_gadd + (int64_t)n * W.gadd_stride : nullptr;
        // A x0' applied, or read back from the solve that wrote the point (d_gax, see the small kernel)
        const double* Ax0 = W.d_gax ? W.d_gax + (int64_t)n * W.gax_stride : nullptr;
        if (!Ax0) {
          RM_BIG_FOR {
            const int j = big_row(c, e), i = big_col(c, nf, e);
            if (j < ny && i < nx) {
              const int gi = j * nx + i;
              put_tile(pv0, j, i, Gr ? __ldcg(gu + gi) - gsc(n) * __ldcg(Gr + gi) : __ldcg(gu + gi));
            }
          }
          big_sync<C>(sy);
          big_matvec<C>(pv0, gens, stage, acc, c, kx_end, ky_end, P.merge);
          ++nmv;
        }
        double pg[1][4] = {{0, 0, 0, 0}};
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          double r = 0.0;
          if (j < ny && i < nx)
            r = bs[big_fidx(c, nf, e)] - (Ax0 ? __ldcg(Ax0 + j * nx + i) : acc[nf][e]);
          acc[nf][e] = r;
          pg[0][nf >> 1] += r * r;
        }
        double rg[1];
        big_reduce<C, 1>(pg, wred, sy, buf, c, rg);
        buf ^= 1;
        if (rg[0] < tot[1]) {
          tot[1] = rg[0];
          RM_BIG_FOR {
            const int j = big_row(c, e), i = big_col(c, nf, e);
            const int fi = big_fidx(c, nf, e);
            double x0 = 0.0;
            if (j < ny && i < nx) {
              const int gi = j * nx + i;
              x0 = Ax0 ? (Gr ? __ldcg(gu + gi) - gsc(n) * __ldcg(Gr + gi) : __ldcg(gu + gi)) : __ldcg(pv0 + pv_idx<C>(j, i));
            }
            xs[fi] = x0;
            rs[fi] = acc[nf][e];
          }
        }
      }
      double res = sqrt(tot[1]);
      double rr = tot[1];
      int64_t its = 0;
      int fail = 0;
      bool done = res <= target;

      // z = P^-1 r (PRE) into acc; uses pv1 <- r, pv0 <- T1, pv1 <- T2 * dinv, pv0 <- T3
      auto apply_tau_big = [&]() {
        __syncthreads();
        big_sync<C>(sy);  // every CTA done reading pv0 / pv1
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          if (j < ny && i < nx) put_tile(pv1, j, i, __ldcg(rs + big_fidx(c, nf, e)));
        }
        big_sync<C>(sy);
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          big_dst_xT<C>(pv1, tabx, Lx, stage, acc, c, kx_end, fold_x);
          RM_BIG_FOR {
            const int j = bigT_row(c, nf, e), i = bigT_col(c, e, fold_x);
            if (j < ny && i < nx) put_tile(pv0, j, i, acc[nf][e]);
          }
          big_sync<C>(sy);
          big_dst_y<C>(pv0, taby, Ly, stage, acc, c, ky_end, fold_y);
          if (pass == 1) break;
          RM_BIG_FOR {
            const int j = big_row(c, e), i = big_col(c, nf, e);
            if (j < ny && i < nx) put_tile(pv1, j, i, acc[nf][e] * __ldcg(ds + big_fidx(c, nf, e)));
          }
          big_sync<C>(sy);
        }
        ++npc;
      };
      // FP16 DST stages (precond 2): V16a <- r s1; V16b <- x-stage; V16a <- y-stage * dinv s2; V16b <- x-stage;
      // acc <- y-stage / (s1 s2)
      auto apply_tau_big_lp = [&]() {
        using BL = BigLp<C>;
        uint16_t* v16a = reinterpret_cast<uint16_t*>(pv1);
        uint16_t* v16b = v16a + (size_t)C::NP * BL::SHH;
        char* st16 = reinterpret_cast<char*>(stage);
        __syncthreads();
        double m = 0.0;
        RM_BIG_FOR { m = fmax(m, fabs(__ldcg(rs + big_fidx(c, nf, e)))); }
        // (its group barrier also orders every CTA's last read of pv1 before the writes below)
        const double gm = big_max<C>(m, wred, sy, buf, c);
        const int e1 = gm > 0.0 ? 6 - ilogb(gm) : 0;
        const int e2 = lp_dbound > 0.0 ? -ilogb(lp_dbound) : 0;
        const double s1 = ldexp(1.0, e1), s2 = ldexp(1.0, e2), unscale = ldexp(1.0, -e1 - e2);
#pragma unroll
        for (int nf = 0; nf < 8; ++nf)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = big_row(c, 2 * h), i = big_col(c, nf, 2 * h);
            const bool in = j < ny;
            const float lo = (in && i < nx) ? (float)(__ldcg(rs + big_fidx(c, nf, 2 * h)) * s1) : 0.f;
            const float hi = (in && i + 1 < nx) ? (float)(__ldcg(rs + big_fidx(c, nf, 2 * h + 1)) * s1) : 0.f;
            *reinterpret_cast<uint32_t*>(v16a + (size_t)j * BL::SHH + i) = pack_f16x2(lo, hi);
          }
        big_sync<C>(sy);
        float a32[8][4];
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          big_dst16<C, false>(P.dst16, v16a, st16, a32, c);
          RM_BIG_FOR {
            const int j = c.R0 + 16 * c.wc0 + 8 * nf + 2 * c.tig + (e & 1);
            const int i = c.C0 + 16 * c.wr + c.gq + 8 * (e >> 1);
            v16b[(size_t)j * BL::SHH + i] = to_f16(a32[nf][e]);
          }
          big_sync<C>(sy);
          big_dst16<C, true>(P.dst16, v16b, st16, a32, c);
          if (pass == 1) break;
          // every CTA finished its x-stage reads of V16a before the barrier above
#pragma unroll
          for (int nf = 0; nf < 8; ++nf)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int j = big_row(c, 2 * h), i = big_col(c, nf, 2 * h);
              const bool in = j < ny;
              const float lo =
                  (in && i < nx) ? (float)(a32[nf][2 * h] * (__ldcg(ds + big_fidx(c, nf, 2 * h)) * s2)) : 0.f;
              const float hi =
                  (in && i + 1 < nx) ? (float)(a32[nf][2 * h + 1] * (__ldcg(ds + big_fidx(c, nf, 2 * h + 1)) * s2))
                                     : 0.f;
              *reinterpret_cast<uint32_t*>(v16a + (size_t)j * BL::SHH + i) = pack_f16x2(lo, hi);
            }
          big_sync<C>(sy);
        }
        RM_BIG_FOR { acc[nf][e] = (double)a32[nf][e] * unscale; }
        ++npc;
      };
      auto set_direction_from = [&](bool use_z) {
        // p = z (PRE) or r into pv0 (after every CTA finished reading pv0)
        big_sync<C>(sy);
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          if (j < ny && i < nx) put_tile(pv0, j, i, use_z ? acc[nf][e] : __ldcg(rs + big_fidx(c, nf, e)));
        }
        big_sync<C>(sy);
      };

      if (!done) {
        if constexpr (PRE) {
          if (lp_dst) apply_tau_big_lp(); else apply_tau_big();
          double p1[1][4] = {{0, 0, 0, 0}};
          RM_BIG_FOR { p1[0][nf >> 1] += __ldcg(rs + big_fidx(c, nf, e)) * acc[nf][e]; }
          double rz[1];
          big_reduce<C, 1>(p1, wred, sy, buf, c, rz);
          buf ^= 1;
          rr = rz[0];
          set_direction_from(true);
        } else {
          set_direction_from(false);
        }
      }
      for (int64_t k = 1; !done; ++k) {
        if (k > max_iter) {
          fail = RM_CG_BUDGET;
          its = max_iter;
          break;
        }
        big_matvec<C>(pv0, gens, stage, acc, c, kx_end, ky_end, P.merge);
        ++nmv;
        double p1[1][4] = {{0, 0, 0, 0}};
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          double ap = 0.0;
          if (j < ny && i < nx) {
            ap = acc[nf][e];
            p1[0][nf >> 1] += __ldcg(pv0 + pv_idx<C>(j, i)) * ap;
          }
          acc[nf][e] = ap;
        }
        double pap[1];
        big_reduce<C, 1>(p1, wred, sy, buf, c, pap);
        buf ^= 1;
        if (!isfinite(pap[0]) || pap[0] <= 0.0) {
          fail = RM_CG_BREAKDOWN;
          its = k;
          break;
        }
        const double alpha = rr / pap[0];
        double part2[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // one unit (8 elements) per batch: loads first, then stores
          double pv[8], xv[8], rv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int nf = 2 * u + (q >> 2), e = q & 3;
            const int j = big_row(c, e), i = big_col(c, nf, e);
            const int fi = big_fidx(c, nf, e);
            const bool ok = j < ny && i < nx;
            pv[q] = ok ? __ldcg(pv0 + pv_idx<C>(j, i)) : 0.0;
            xv[q] = __ldcg(xs + fi);
            rv[q] = __ldcg(rs + fi);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int nf = 2 * u + (q >> 2), e = q & 3;
            const int j = big_row(c, e), i = big_col(c, nf, e);
            const int fi = big_fidx(c, nf, e);
            if (j < ny && i < nx) {
              xs[fi] = xv[q] + alpha * pv[q];
              const double rn = rv[q] - alpha * acc[nf][e];
              rs[fi] = rn;
              part2[0][u] += rn * rn;
              if constexpr (PRE) ps[fi] = pv[q];
            }
          }
        }
        double red2[2];
        if constexpr (PRE) {
          if (lp_dst) apply_tau_big_lp(); else apply_tau_big();
          RM_BIG_FOR { part2[1][nf >> 1] += __ldcg(rs + big_fidx(c, nf, e)) * acc[nf][e]; }
          big_reduce<C, 2>(part2, wred, sy, buf, c, red2);
        } else {
          double p0[1][4] = {{part2[0][0], part2[0][1], part2[0][2], part2[0][3]}};
          double one[1];
          big_reduce<C, 1>(p0, wred, sy, buf, c, one);
          red2[0] = red2[1] = one[0];
        }
        buf ^= 1;
        double rr_new = red2[0];
        res = sqrt(rr_new);
        if (!isfinite(res)) {
          fail = RM_CG_NONFINITE;
          its = k;
          break;
        }
        if (res <= target) {
          big_sync<C>(sy);
          RM_BIG_FOR {
            const int j = big_row(c, e), i = big_col(c, nf, e);
            if (j < ny && i < nx) put_tile(pv0, j, i, xs[big_fidx(c, nf, e)]);
          }
          big_sync<C>(sy);
          big_matvec<C>(pv0, gens, stage, acc, c, kx_end, ky_end, P.merge);
          ++nmv;
          double pt[1][4] = {{0, 0, 0, 0}};
          RM_BIG_FOR {
            const int j = big_row(c, e), i = big_col(c, nf, e);
            double rt = 0.0;
            if (j < ny && i < nx) rt = bs[big_fidx(c, nf, e)] - acc[nf][e];
            acc[nf][e] = rt;
            pt[0][nf >> 1] += rt * rt;
          }
          double tt[1];
          big_reduce<C, 1>(pt, wred, sy, buf, c, tt);
          buf ^= 1;
          const double true_res = sqrt(tt[0]);
          if (true_res <= fmax(target, 10.0 * res)) {
            RM_BIG_FOR { rs[big_fidx(c, nf, e)] = acc[nf][e]; }  // r = b - A x for the chain's next rhs
            its = k;
            done = true;
            break;
          }
          res = true_res;
          RM_BIG_FOR { rs[big_fidx(c, nf, e)] = acc[nf][e]; }
          if (res <= target) {
            its = k;
            done = true;
            break;
          }
          if constexpr (PRE) {
            if (lp_dst) apply_tau_big_lp(); else apply_tau_big();
            double p3[1][4] = {{0, 0, 0, 0}};
            RM_BIG_FOR { p3[0][nf >> 1] += __ldcg(rs + big_fidx(c, nf, e)) * acc[nf][e]; }
            double rz[1];
            big_reduce<C, 1>(p3, wred, sy, buf, c, rz);
            buf ^= 1;
            rr = rz[0];
            set_direction_from(true);
          } else {
            rr = tt[0];
            set_direction_from(false);
          }
          continue;
        }
        const double beta = red2[1] / rr;
        rr = red2[1];
        big_sync<C>(sy);  // every CTA done reading pv0 (and the DST stages)
        RM_BIG_FOR {
          const int j = big_row(c, e), i = big_col(c, nf, e);
          if (j < ny && i < nx) {
            const int fi = big_fidx(c, nf, e);
            const double pold = PRE ? __ldcg(ps + fi) : __ldcg(pv0 + pv_idx<C>(j, i));
            const double zi = PRE ? acc[nf][e] : rs[fi];
            put_tile(pv0, j, i, zi + beta * pold);
          }
        }
        big_sync<C>(sy);
      }

      chain_ok = done && !fail;
      if (c.rank == 0 && c.tid == 0) {
        atomicAdd(W.d_counters, 1ull);
        atomicAdd(W.d_counters + 1, (unsigned long long)its);
        atomicAdd(W.d_counters + 2, (unsigned long long)nmv);
        atomicAdd(W.d_counters + 3, (unsigned long long)npc);
      }
      if (fail) {
        if (c.rank == 0 && c.tid == 0 && atomicCAS(P.fail, 0, fail) == 0) {
          P.fail_info[0] = (double)n;
          P.fail_info[1] = (double)its;
          P.fail_info[2] = res;
        }
        big_sync<C>(sy);
        break;
      }
      // ---------------- MGRIT epilogue ----------------
      const bool next_in_tile = n < n1 && need_in;
      const int oi = n / W.out_div;
      const double* Gn = W.d_gadd ? W.d_gadd + (int64_t)n * W.gadd_stride : nullptr;
      const double* Sn = W.d_sub ? W.d_sub + (int64_t)n * W.sub_stride : nullptr;
      double* On = W.d_out ? W.d_out + (int64_t)oi * W.out_stride : nullptr;
      double* Kn = W.d_keep ? W.d_keep + (int64_t)oi * W.keep_stride : nullptr;
      double* An = W.d_ax ? W.d_ax + (int64_t)oi * W.ax_stride : nullptr;
      big_sync<C>(sy);  // every CTA done reading pv0 before it is overwritten with y
      double py[1][4] = {{0, 0, 0, 0}};
      RM_BIG_FOR {
        const int j = big_row(c, e), i = big_col(c, nf, e);
        if (j < ny && i < nx) {
          const int gi = j * nx + i;
          double y = xs[big_fidx(c, nf, e)];
          if (An) An[gi] = bs[big_fidx(c, nf, e)] - rs[big_fidx(c, nf, e)];  // A x = b - r (true residual)
          if (Gn) y = gsc(n) * __ldcg(Gn + gi) + y;
          if (Kn) Kn[gi] = y;
          if (Sn) y = y - __ldcg(Sn + gi);
          if (On) On[gi] = y;
          if (next_in_tile) put_tile(pv0, j, i, y);
          py[0][nf >> 1] += y * y;
        }
      }
      if (W.d_norms) {
        double yy[1];
        big_reduce<C, 1>(py, wred, sy, buf, c, yy);
        buf ^= 1;
        if (c.rank == 0 && c.tid == 0) W.d_norms[oi] = yy[0];
      }
      in_tile = next_in_tile;
      big_sync<C>(sy);
    }
  }
}

// Batched operator apply for large grids (rm_apply_batched; setup and tests, not the hot path):
// one thread per output element, DFMA over the Toeplitz sums, operand read from global memory.
__global__ void apply_big_kernel(const ApplyArgs P, int np) {
  const int nx = P.nx, ny = P.ny;
  const int b = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nx * ny) return;
  const int j = idx / nx, i = idx % nx;
  const double* v = P.v + (int64_t)b * P.v_stride;
  const int GL = 2 * np + 8;
  const double* g = P.gens + np;
  auto V = [&](int jj, int ii) { return (jj < 0 || jj >= ny || ii < 0 || ii >= nx) ? 0.0 : __ldg(v + jj * nx + ii); };
  const bool dox = P.which == 0 || P.which == 2, doy = P.which == 0 || P.which == 3;
  double acc = 0.0;
  if (dox)
    for (int seg = 0; seg < 3; ++seg) {
      const int d = seg == 0 ? 0 : (seg == 1 ? 1 : -1);
      for (int k = 0; k < nx; ++k) acc = fma(g[seg * GL + i - k], V(j + d, k), acc);
    }
  if (doy)
    for (int seg = 0; seg < 3; ++seg) {
      const int d = seg == 0 ? 0 : (seg == 1 ? 1 : -1);
      for (int l = 0; l < ny; ++l) acc = fma(g[(3 + seg) * GL + j - l], V(l, i + d), acc);
    }
  double mass = 6.0 * V(j, i);
  mass += V(j, i - 1);
  mass += V(j, i + 1);
  mass += V(j + 1, i);
  mass += V(j + 1, i + 1);
  mass += V(j - 1, i);
  mass += V(j - 1, i - 1);
  mass *= P.cm;
  double y;
  if (P.which == 1)
    y = mass;
  else if (P.which == 0)
    y = mass + P.sign * 0.5 * P.dt[b] * acc;
  else
    y = (P.which == 2 ? 1.0 / P.kx : 1.0 / P.ky) * acc;
  P.out[(int64_t)b * P.out_stride + idx] = y;
}

cudaError_t launch_apply_big(int np, const ApplyArgs& a, int batch, cudaStream_t st) {
  dim3 grid((a.nx * a.ny + 255) / 256, batch);
  apply_big_kernel<<<grid, 256, 0, st>>>(a, np);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------------------
template <int NP>
static cudaError_t launch_big_t(const ChainArgs& a, int max_clusters, cudaStream_t st) {
  using C = BigCfg<NP>;
  auto kern = a.sw.precond ? chain_big_kernel<C, true> : chain_big_kernel<C, false>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (err != cudaSuccess) return err;
  if (C::G > 8 && !C::GSYNC) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
  }
  int ncl = max_clusters < a.sw.nchains ? max_clusters : a.sw.nchains;
  if (ncl < 1) ncl = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncl * C::G);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if constexpr (C::GSYNC) {
    if (!a.gbar || !a.gbuf) return cudaErrorInvalidValue;
    attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs of a group co-resident (global barrier)
    attr[0].val.cooperative = 1;
  } else {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C::G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int NP>
static cudaError_t max_clusters_big_t(int* out) {
  using C = BigCfg<NP>;
  auto kern = chain_big_kernel<C, true>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (err != cudaSuccess) return err;
  if constexpr (C::GSYNC) {
    int per_sm = 0, dev = 0, sms = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM);
    if (err != cudaSuccess) return err;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    *out = per_sm * sms / C::G;
    return cudaSuccess;
  }
  if (C::G > 8) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C::G);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, kern, &cfg);
}

bool big_supported(int np) { return np == 256 || np == 512 || np == 1024; }

int big_group(int np) { return (np / 128) * (np / 128); }

size_t big_scratch_doubles_per_cluster(int np) {
  const size_t pv = (size_t)(np + 2) * (np + 16);
  return 2 * pv + 5 * (size_t)big_group(np) * 128 * 128;
}

cudaError_t launch_big(int np, const ChainArgs& a, int max_clusters, cudaStream_t st) {
  if (np == 256) return launch_big_t<256>(a, max_clusters, st);
  if (np == 512) return launch_big_t<512>(a, max_clusters, st);
  if (np == 1024) return launch_big_t<1024>(a, max_clusters, st);
  return cudaErrorInvalidValue;
}

cudaError_t big_max_clusters(int np, int* out) {
  if (np == 256) return max_clusters_big_t<256>(out);
  if (np == 512) return max_clusters_big_t<512>(out);
  if (np == 1024) return max_clusters_big_t<1024>(out);
  return cudaErrorInvalidValue;
}

}  // namespace rm
