// Internal kernel-launch interface (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "riesz_mgrit_b200.h"

namespace rm {

struct ChainArgs {
  rm_sweep sw;
  int nx, ny;
  double cm;
  const double* gens;  // 6 generator tables of length 2*NP+8 (device)
  int merge;           // bit 0/1: merged off-diagonal x/y segments (see matvec)
  double* scratch;     // NP*NP doubles per cluster (device): right-hand side b
  int* chain_counter;  // work counter, zeroed before launch
  int* fail;           // first-failure flag
  double* fail_info;   // n, iterations, residual norm
  long long* timing;   // RM_TIMING builds: per-phase cycles of CTA 0
  const double* dm;    // tau preconditioner: d(s) = dm + s*dk, [ny][nx] (device)
  const double* dk;
  const double* tabx;  // sine tables sqrt(2/(n+1)) sin(pi m/(n+1)), m < 2(n+1) (device)
  const double* taby;
  unsigned* gbar;      // large grids beyond the cluster limit: per-group barrier counters (32 words each)
  double* gbuf;        // ... and per-group reduction / broadcast slots (1024 doubles each)
  const uint16_t* dst16; // FP16 DST-I matrix [NP][NP+8] of the low-precision tau stages (precond 2, nx == ny)
  double lp_dmin, lp_kmin; // min over the grid of dm, dk: 1/(lp_dmin + s lp_kmin) bounds max 1/d(s)
  double gen_absmax;       // max |entry| of the six generator tables (split-FP16 table scaling)
  // FFT kernel (rm_fft.cu, 255^2 grids)
  const double* fsym;      // stiffness spectra (rm_fft.cu fft_symbols): 2 x 512 real, 2 x 512 complex, k-layout
  double* fscratch;        // per-chain vectors (fft_scratch_doubles_per_chain each)
  const double* dmT;       // tau diagonals transposed, [nx][ny]
  const double* dkT;
  double lp_thr;           // FFT kernel, lp_matvec: FP32 in-iteration applies once |r| <= lp_thr |b| (0: never)
  const uint16_t* dstc;    // FP16 DST-I matrix, order 256, row-major (tensor-core preconditioner, rm_tc.cuh)
};

struct ApplyArgs {
  int nx, ny, which, sign;
  double cm, kx, ky;
  const double* gens;
  int merge;
  const double* dt;
  const double* v;
  int64_t v_stride;
  double* out;
  int64_t out_stride;
};

struct PcgArgs {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
  int64_t start, count, row;
  double* out;
  int64_t out_stride;
};

bool chain_supported(int np, int g);
cudaError_t launch_chain(int np, int g, const ChainArgs& a, int max_clusters, cudaStream_t st);
cudaError_t chain_max_clusters(int np, int g, int* out);
size_t chain_smem(int np, int g);
cudaError_t launch_apply(int np, const ApplyArgs& a, int batch, cudaStream_t st);
cudaError_t launch_pcg64(const PcgArgs& a, cudaStream_t st);
cudaError_t launch_correct(int ndof, int nc, int m, double* u, int64_t us, const double* uc, int64_t ucs,
                           cudaStream_t st);
bool big_supported(int np);  // 256, 512 (clusters), 1024 (global-memory group barrier)
int big_group(int np);
size_t big_scratch_doubles_per_cluster(int np);
cudaError_t launch_big(int np, const ChainArgs& a, int max_clusters, cudaStream_t st);
cudaError_t big_max_clusters(int np, int* out);
cudaError_t launch_apply_big(int np, const ApplyArgs& a, int batch, cudaStream_t st);
bool fft_supported(int np, int nx, int ny);
int fft_group();
size_t fft_scratch_doubles_per_chain();
cudaError_t fft_max_chains(int* out);
cudaError_t launch_fft(const ChainArgs& a, int max_chains, cudaStream_t st);
bool fft_symbols(const double* tab, int np, int gl, double* out_klayout);
cudaError_t launch_diff_sqnorm(int64_t n, const double* a, const double* b, double* out, cudaStream_t st);
cudaError_t launch_vec_dot(int64_t n, const double* a, const double* b, double* out, cudaStream_t st);
cudaError_t launch_vec_axpby(int64_t n, double alpha, const double* x, double beta, const double* y, double* out,
                             cudaStream_t st);

}  // namespace rm
