// extern "C" boundary of the B200 hot path (declared in include/riesz_mgrit_b200.h).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <vector>

#include "riesz_mgrit_b200.h"
#include "rm_kernels.h"
#include "rm_tc.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return RM_ECUDA;
}

#define RM_CUDA(call, what)                     \
  do {                                          \
    cudaError_t e_ = (call);                    \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

const int kGroups[5] = {1, 2, 4, 8, 16};

int padded_order(int nx, int ny) {
  int n = std::max(nx, ny);
  int np = 16;
  while (np < n) np *= 2;
  return np;
}

}  // namespace

struct rm_grid {
  int nx, ny, np, device;
  int merge = 0;  // bit 0/1: off-diagonal Toeplitz block along x/y has t2(d) = t2(-1-d) (see rm_device.cuh matvec)
  double kx, ky, sx, sy, cm;
  double* d_gens = nullptr;
  double* d_scratch = nullptr;
  int scratch_clusters = 0;
  int* d_counter = nullptr;
  int* d_fail = nullptr;
  double* d_fail_info = nullptr;
  long long* d_timing = nullptr;
  unsigned* d_gbar = nullptr;  // NP = 1024: per-group barrier counters of the global-sync large-grid kernel
  double* d_gbuf = nullptr;    //            and per-group reduction slots
  int big_slots = 0;           // resident chain groups of the large-grid kernel
  double* d_dm = nullptr;  // tau preconditioner (rm_grid_set_tau)
  double* d_dk = nullptr;
  double* d_tab = nullptr;  // sine tables x then y
  uint16_t* d_dst16 = nullptr;  // FP16 DST-I matrix [np][np+8] (chain kernel, precond 2, nx == ny)
  double lp_dmin = 0.0, lp_kmin = 0.0;  // min over the grid of the tau diagonals dm, dk
  double gen_absmax = 0.0;               // max |entry| of the six generator tables
  int max_clusters[5] = {0, 0, 0, 0, 0};
  // FFT kernel (rm_fft.cu): 255^2 grids
  bool fft_ok = false;
  int fft_slots = 0;
  double* d_fsym = nullptr;
  double* d_fscratch = nullptr;
  double* d_dmT = nullptr;
  double* d_dkT = nullptr;
  uint16_t* d_dstc = nullptr;  // FP16 DST-I matrix in the tcgen05 canonical layout (tensor-core preconditioner)
};

extern "C" {

const char* rm_version(void) { return "riesz_mgrit_b200 0.1.0 (sm_100a, FP64 DMMA)"; }

const char* rm_last_error(void) { return g_err.c_str(); }

int rm_max_order(void) { return 1024; }

int rm_grid_create(int nx, int ny, const double* t1x_col, const double* t1x_row, const double* t2x_col,
                   const double* t2x_row, const double* t1y_col, const double* t1y_row, const double* t2y_col,
                   const double* t2y_row, double sx, double sy, double kx, double ky, double mass_scale,
                   rm_grid** out) {
  if (!out) return fail(RM_EINVAL, "rm_grid_create: null output pointer");
  *out = nullptr;
  if (nx < 1 || ny < 1) return fail(RM_EINVAL, "rm_grid_create: need nx, ny >= 1");
  if (!t1x_col || !t1x_row || !t2x_col || !t2x_row || !t1y_col || !t1y_row || !t2y_col || !t2y_row)
    return fail(RM_EINVAL, "rm_grid_create: null generator");
  const int np = padded_order(nx, ny);
  if (np > rm_max_order())
    return fail(RM_EUNSUP, "rm_grid_create: grid order " + std::to_string(std::max(nx, ny)) +
                               " exceeds the supported maximum " + std::to_string(rm_max_order()));
  rm_grid* g = new rm_grid();
  g->nx = nx;
  g->ny = ny;
  g->np = np;
  g->kx = kx;
  g->ky = ky;
  g->sx = sx;
  g->sy = sy;
  g->cm = mass_scale;
  cudaGetDevice(&g->device);
  // generator tables: entry (d + np) of table t, d in [-np, np+8)
  const int GL = 2 * np + 8;
  std::vector<double> tab(6 * GL, 0.0);
  // entry (d) of a Toeplitz block given by first column/row: T[i][k] = t(i - k)
  auto t2 = [](const double* col, const double* row, int d) { return d >= 0 ? col[d] : row[-d]; };
  const double fx = kx * sx, fy = ky * sy;
  for (int d = -np; d < np + 8; ++d) {
    const int idx = d + np;
    if (std::abs(d) < nx) {
      tab[0 * GL + idx] = fx * t2(t1x_col, t1x_row, d);
      tab[1 * GL + idx] = fx * t2(t2x_col, t2x_row, d);
      tab[2 * GL + idx] = fx * t2(t2x_col, t2x_row, -d);
    }
    if (std::abs(d) < ny) {
      tab[3 * GL + idx] = fy * t2(t1y_col, t1y_row, d);
      tab[4 * GL + idx] = fy * t2(t2y_col, t2y_row, d);
      tab[5 * GL + idx] = fy * t2(t2y_col, t2y_row, -d);
    }
  }
  // T2 with first column == first row shifted by one (the Riesz stiffness A2, assembly.py:239-249):
  // the two off-diagonal segments of the matvec merge into one of length n+1 (needs t2(-n) = col[n-1])
  auto shifted_sym = [](const double* col, const double* row, int n) {
    if (n % 4 == 0) return false;
    for (int d = 0; d + 1 < n; ++d)
      if (col[d] != row[d + 1]) return false;
    return true;
  };
  if (shifted_sym(t2x_col, t2x_row, nx)) {
    g->merge |= 1;
    tab[1 * GL + np - nx] = fx * t2x_col[nx - 1];
  }
  if (shifted_sym(t2y_col, t2y_row, ny)) {
    g->merge |= 2;
    tab[4 * GL + np - ny] = fy * t2y_col[ny - 1];
  }
  if (const char* m = getenv("RM_MERGE")) g->merge &= atoi(m);
  std::vector<double> fsym;
  if (rm::fft_supported(np, nx, ny)) {
    fsym.resize(6 * 512);
    if (!rm::fft_symbols(tab.data(), np, GL, fsym.data())) fsym.clear();  // generators without the symmetries
  }
  cudaError_t e;
  int maxc = 1;
  size_t scratch_per_cluster = 3 * (size_t)np * np;
  if (rm::big_supported(np)) {
    int n = 0;
    e = rm::big_max_clusters(np, &n);
    if (e != cudaSuccess || n <= 0) {
      cudaGetLastError();
      delete g;
      return fail(RM_EUNSUP, "rm_grid_create: no resident cluster for the large-grid kernel");
    }
    for (int gi = 0; gi < 5; ++gi) g->max_clusters[gi] = kGroups[gi] == rm::big_group(np) ? n : 0;
    g->big_slots = n;
    maxc = n;
    scratch_per_cluster = rm::big_scratch_doubles_per_cluster(np);
  }
  for (int gi = 0; gi < 5 && !rm::big_supported(np); ++gi) {
    const int G = kGroups[gi];
    if (!rm::chain_supported(np, G)) continue;
    int n = 0;
    e = rm::chain_max_clusters(np, G, &n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    g->max_clusters[gi] = n;
    maxc = std::max(maxc, n);
  }
  g->scratch_clusters = maxc;
  for (double v : tab) g->gen_absmax = std::max(g->gen_absmax, fabs(v));
  if ((e = cudaMalloc(&g->d_gens, sizeof(double) * tab.size())) != cudaSuccess ||
      (e = cudaMemcpy(g->d_gens, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMalloc(&g->d_scratch, sizeof(double) * scratch_per_cluster * maxc)) != cudaSuccess ||
      (e = cudaMalloc(&g->d_counter, sizeof(int))) != cudaSuccess ||
      (e = cudaMalloc(&g->d_fail, sizeof(int))) != cudaSuccess ||
      (e = cudaMemset(g->d_fail, 0, sizeof(int))) != cudaSuccess ||
      (e = cudaMalloc(&g->d_fail_info, 4 * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&g->d_timing, 16 * sizeof(long long))) != cudaSuccess ||
      (e = cudaMemset(g->d_timing, 0, 16 * sizeof(long long))) != cudaSuccess ||
      (rm::big_supported(np) &&
       ((e = cudaMalloc(&g->d_gbar, sizeof(unsigned) * 32 * maxc)) != cudaSuccess ||
        (e = cudaMalloc(&g->d_gbuf, sizeof(double) * 1024 * maxc)) != cudaSuccess))) {
    rm_grid_destroy(g);
    return cuda_fail(e, "rm_grid_create");
  }
  if (!fsym.empty()) {
    int nch = 0;
    e = rm::fft_max_chains(&nch);
    if (e != cudaSuccess || nch <= 0) {
      cudaGetLastError();
    } else {
      nch = std::min(nch, g->big_slots);  // group barrier / reduction slots are shared with the DMMA kernel
      if ((e = cudaMalloc(&g->d_fsym, sizeof(double) * fsym.size())) != cudaSuccess ||
          (e = cudaMemcpy(g->d_fsym, fsym.data(), sizeof(double) * fsym.size(), cudaMemcpyHostToDevice)) !=
              cudaSuccess ||
          (e = cudaMalloc(&g->d_fscratch, sizeof(double) * rm::fft_scratch_doubles_per_chain() * nch)) !=
              cudaSuccess) {
        rm_grid_destroy(g);
        return cuda_fail(e, "rm_grid_create (FFT kernel)");
      }
      g->fft_slots = nch;
      g->fft_ok = true;
    }
  }
  *out = g;
  return RM_OK;
}

int rm_grid_destroy(rm_grid* g) {
  if (!g) return RM_OK;
  cudaFree(g->d_gens);
  cudaFree(g->d_scratch);
  cudaFree(g->d_counter);
  cudaFree(g->d_fail);
  cudaFree(g->d_fail_info);
  cudaFree(g->d_timing);
  cudaFree(g->d_gbar);
  cudaFree(g->d_gbuf);
  cudaFree(g->d_dm);
  cudaFree(g->d_dk);
  cudaFree(g->d_tab);
  cudaFree(g->d_dst16);
  cudaFree(g->d_fsym);
  cudaFree(g->d_fscratch);
  cudaFree(g->d_dmT);
  cudaFree(g->d_dkT);
  cudaFree(g->d_dstc);
  delete g;
  return RM_OK;
}

int rm_grid_flags(const rm_grid* g) {
  if (!g) return -1;
  const bool fft = g->fft_ok && !(getenv("RM_NO_FFT") && atoi(getenv("RM_NO_FFT")));
  return g->merge | (fft ? 4 : 0);
}

int rm_apply_batched(const rm_grid* g, int which, int batch, const double* d_dt, int sign, const double* d_v,
                     int64_t v_stride, double* d_out, int64_t out_stride, void* stream) {
  if (!g) return fail(RM_EINVAL, "rm_apply_batched: null grid");
  if (which < 0 || which > 3) return fail(RM_EINVAL, "rm_apply_batched: which must be 0..3");
  if (which == 0 && sign != 1 && sign != -1) return fail(RM_EINVAL, "sign must be +1 or -1");
  if (batch < 0) return fail(RM_EINVAL, "rm_apply_batched: negative batch");
  if (batch == 0) return RM_OK;
  if (!d_v || !d_out || (which == 0 && !d_dt)) return fail(RM_EINVAL, "rm_apply_batched: null pointer");
  rm::ApplyArgs a;
  a.nx = g->nx;
  a.ny = g->ny;
  a.which = which;
  a.sign = sign;
  a.cm = g->cm;
  a.kx = g->kx;
  a.ky = g->ky;
  a.gens = g->d_gens;
  a.merge = g->merge;
  a.dt = d_dt;
  a.v = d_v;
  a.v_stride = v_stride;
  a.out = d_out;
  a.out_stride = out_stride;
  if (rm::big_supported(g->np))
    RM_CUDA(rm::launch_apply_big(g->np, a, batch, (cudaStream_t)stream), "rm_apply_batched");
  else
    RM_CUDA(rm::launch_apply(g->np, a, batch, (cudaStream_t)stream), "rm_apply_batched");
  return RM_OK;
}

// Relative time of one chain step on a cluster of G CTAs (measured on B200, tools/group_sweep.py,
// cfg2 127^2: G=2 1.29 ms, G=4 0.83, G=8 0.62, G=16 0.97 per PCG step; 16-CTA clusters have 4-warp
// CTAs and 15-peer exchanges).  Lower is faster; 0 = not available.
static double group_step_cost(int np, int G) {
  switch (np) {
    case 128: return G == 2 ? 1.0 : G == 4 ? 0.64 : G == 8 ? 0.48 : G == 16 ? 0.75 : 0.0;
    case 64: return G == 1 ? 1.0 : G == 2 ? 0.62 : G == 4 ? 0.5 : 0.0;
    case 32: return G == 1 ? 1.0 : G == 2 ? 0.75 : 0.0;
    default: return G == 1 ? 1.0 : 0.0;
  }
}

static int choose_group(const rm_grid* g, int nchains) {
  double best = 1e300;
  int best_g = 1;
  for (int gi = 0; gi < 5; ++gi) {
    const int G = kGroups[gi];
    const double cost = group_step_cost(g->np, G);
    if (cost <= 0.0 || !rm::chain_supported(g->np, G) || g->max_clusters[gi] <= 0) continue;
    const int slots = std::min(g->max_clusters[gi], g->scratch_clusters);
    const double est = ceil((double)nchains / slots) * cost;
    if (est < best * 0.999) {
      best = est;
      best_g = G;
    }
  }
  return best_g;
}

int rm_sweep_run(rm_grid* g, const rm_sweep* sw, void* stream) {
  if (!g || !sw) return fail(RM_EINVAL, "rm_sweep_run: null argument");
  if (sw->nchains <= 0) return RM_OK;
  if (!sw->d_dt) return fail(RM_EINVAL, "rm_sweep_run: d_dt is required");
  if (sw->clen < 1 || sw->first < 1 || sw->nmax < sw->first) return fail(RM_EINVAL, "rm_sweep_run: bad chain shape");
  if (sw->out_div < 1) return fail(RM_EINVAL, "rm_sweep_run: out_div must be >= 1");
  if ((sw->explicit_rhs || sw->x0_mode == 1) && !sw->d_src) return fail(RM_EINVAL, "rm_sweep_run: d_src required");
  if (sw->x0_mode < 0 || sw->x0_mode > 4) return fail(RM_EINVAL, "rm_sweep_run: x0_mode must be 0..4");
  const bool use_fft = g->fft_ok && !(getenv("RM_NO_FFT") && atoi(getenv("RM_NO_FFT")));
  if (sw->x0_mode == 4 && !use_fft &&
      (sw->precond != 2 || !sw->lp_matvec || rm::big_supported(g->np) || g->nx != g->ny))
    return fail(RM_EUNSUP, "rm_sweep_run: x0_mode 4 (apply probe) needs the FFT kernel or precond 2 with lp_matvec");
  if (sw->x0_mode == 3 && (!sw->precond || (rm::big_supported(g->np) && !use_fft)))
    return fail(RM_EUNSUP, "rm_sweep_run: x0_mode 3 (preconditioner probe) needs precond > 0 and a grid up to 127^2 "
                           "or the FFT kernel");
  if (sw->x0_mode == 2 && !sw->d_x0) return fail(RM_EINVAL, "rm_sweep_run: d_x0 required for x0_mode 2");
  if (sw->clen > 1 && (!sw->d_out || sw->out_div != 1))
    return fail(RM_EINVAL, "rm_sweep_run: chains longer than one step need d_out with out_div == 1");
  if (!sw->d_counters) return fail(RM_EINVAL, "rm_sweep_run: d_counters is required");
  if (!(sw->rel_tol > 0)) return fail(RM_EINVAL, "relative tolerance must be positive");
  if (sw->precond < 0 || sw->precond > 2) return fail(RM_EINVAL, "rm_sweep_run: precond must be 0, 1 or 2");
  if (sw->precond && !g->d_dm) return fail(RM_EINVAL, "rm_sweep_run: precond needs rm_grid_set_tau first");
  if (use_fft) {
    if (sw->group > 0 && sw->group != rm::fft_group())
      return fail(RM_EUNSUP, "rm_sweep_run: the FFT kernel uses a fixed group size");
    if (sw->precond && !g->d_dmT) return fail(RM_EINVAL, "rm_sweep_run: precond needs rm_grid_set_tau first");
    rm::ChainArgs a = {};
    a.gbar = g->d_gbar;
    a.gbuf = g->d_gbuf;
    a.sw = *sw;
    // lp_matvec (with precond 2): FP32-FFT in-iteration applies once |r| <= lp_thr |b| (RM_FFT_LP_THR, 0 = off)
    a.lp_thr = 1e-6;
    if (const char* t = getenv("RM_FFT_LP_THR")) a.lp_thr = atof(t);
    // precond 1 ('tau64'): DST stages as FP32 FFTs; precond 2 ('tau', 'tau16'): on the tensor cores (FP16
    // operands, FP32 accumulation; RM_FFT_TC=0 falls back to the FFT stages)
    if (a.sw.precond == 2 && (!g->d_dstc || (getenv("RM_FFT_TC") && !atoi(getenv("RM_FFT_TC"))))) a.sw.precond = 1;
    if (a.sw.precond != 2) a.sw.lp_matvec = 0;
    a.dstc = g->d_dstc;
    a.lp_dmin = g->lp_dmin;
    a.lp_kmin = g->lp_kmin;
    a.nx = g->nx;
    a.ny = g->ny;
    a.cm = g->cm;
    a.gens = g->d_gens;
    a.merge = g->merge;
    a.chain_counter = g->d_counter;
    a.fail = g->d_fail;
    a.fail_info = g->d_fail_info;
    a.timing = g->d_timing;
    a.dm = g->d_dm;
    a.dk = g->d_dk;
    a.fsym = g->d_fsym;
    a.fscratch = g->d_fscratch;
    a.dmT = g->d_dmT;
    a.dkT = g->d_dkT;
    cudaStream_t stf = (cudaStream_t)stream;
    RM_CUDA(cudaMemsetAsync(g->d_counter, 0, sizeof(int), stf), "rm_sweep_run: counter reset");
    RM_CUDA(cudaMemsetAsync(g->d_gbar, 0, sizeof(unsigned) * 32 * g->fft_slots, stf), "rm_sweep_run: barriers");
    RM_CUDA(rm::launch_fft(a, g->fft_slots, stf), "rm_sweep_run: launch (FFT kernel)");
    return RM_OK;
  }
  if (rm::big_supported(g->np)) {
    if (sw->group > 0 && sw->group != rm::big_group(g->np))
      return fail(RM_EUNSUP, "rm_sweep_run: the large-grid kernel uses a fixed cluster size");
    rm::ChainArgs a;
    a.gbar = g->d_gbar;
    a.gbuf = g->d_gbuf;
    a.sw = *sw;
    // FP16 DST stages for square grids; the split-FP16 iteration applies are a small-grid feature
    a.dst16 = g->d_dst16;
    if (a.sw.precond == 2 && !g->d_dst16) a.sw.precond = 1;
    a.lp_dmin = g->lp_dmin;
    a.lp_kmin = g->lp_kmin;
    a.gen_absmax = g->gen_absmax;
    a.sw.lp_matvec = 0;
    a.nx = g->nx;
    a.ny = g->ny;
    a.cm = g->cm;
    a.gens = g->d_gens;
  a.merge = g->merge;
    a.scratch = g->d_scratch;
    a.chain_counter = g->d_counter;
    a.fail = g->d_fail;
    a.fail_info = g->d_fail_info;
    a.timing = g->d_timing;
    a.dm = g->d_dm;
    a.dk = g->d_dk;
    a.tabx = g->d_tab;
    a.taby = g->d_tab ? g->d_tab + (2 * g->np + 8) : nullptr;
    cudaStream_t stb = (cudaStream_t)stream;
    RM_CUDA(cudaMemsetAsync(g->d_counter, 0, sizeof(int), stb), "rm_sweep_run: counter reset");
    if (g->d_gbar)
      RM_CUDA(cudaMemsetAsync(g->d_gbar, 0, sizeof(unsigned) * 32 * g->big_slots, stb), "rm_sweep_run: barriers");
    RM_CUDA(rm::launch_big(g->np, a, std::min(g->big_slots, g->scratch_clusters), stb),
            "rm_sweep_run: launch (large grid)");
    return RM_OK;
  }
  int G = sw->group > 0 ? sw->group : choose_group(g, sw->nchains);
  if (!rm::chain_supported(g->np, G))
    return fail(RM_EUNSUP, "rm_sweep_run: group size " + std::to_string(G) + " unsupported for order " +
                               std::to_string(g->np));
  int gi = 0;
  while (kGroups[gi] != G) ++gi;
  int slots = g->max_clusters[gi];
  if (slots <= 0) return fail(RM_EUNSUP, "rm_sweep_run: no resident cluster of size " + std::to_string(G));
  slots = std::min(slots, g->scratch_clusters);
  cudaStream_t st = (cudaStream_t)stream;
  rm::ChainArgs a;
  a.gbar = nullptr;
  a.gbuf = nullptr;
  a.sw = *sw;
  a.dst16 = g->d_dst16;
  a.lp_dmin = g->lp_dmin;
  a.lp_kmin = g->lp_kmin;
  a.gen_absmax = g->gen_absmax;
  if (a.sw.precond == 2 && !g->d_dst16) a.sw.precond = 1;  // nx != ny: DST stages in FP64
  a.nx = g->nx;
  a.ny = g->ny;
  a.cm = g->cm;
  a.gens = g->d_gens;
  a.merge = g->merge;
  a.scratch = g->d_scratch;
  a.chain_counter = g->d_counter;
  a.fail = g->d_fail;
  a.fail_info = g->d_fail_info;
  a.timing = g->d_timing;
  a.dm = g->d_dm;
  a.dk = g->d_dk;
  a.tabx = g->d_tab;
  a.taby = g->d_tab ? g->d_tab + (2 * g->np + 8) : nullptr;
  RM_CUDA(cudaMemsetAsync(g->d_counter, 0, sizeof(int), st), "rm_sweep_run: counter reset");
  RM_CUDA(rm::launch_chain(g->np, G, a, slots, st), "rm_sweep_run: launch");
  return RM_OK;
}

int rm_grid_set_tau(rm_grid* g, const double* dm, const double* dk) {
  if (!g || !dm || !dk) return fail(RM_EINVAL, "rm_grid_set_tau: null argument");
  const size_t n = (size_t)g->nx * g->ny;
  for (size_t i = 0; i < n; ++i)
    if (!(dm[i] > 0.0) || !(dk[i] >= 0.0 || dk[i] < 0.0))
      return fail(RM_EINVAL, "rm_grid_set_tau: the mass diagonal must be positive and finite");
  const int np = g->np, st = 2 * np + 8;
  std::vector<double> tab(2 * (size_t)st, 0.0);
  const int ns[2] = {g->nx, g->ny};
  for (int t = 0; t < 2; ++t) {
    const int nn = ns[t], L = 2 * (nn + 1);
    const double c = sqrt(2.0 / (nn + 1));
    for (int m = 0; m < L; ++m) tab[t * st + m] = c * sin(M_PI * (double)m / (double)(nn + 1));
  }
  cudaError_t e;
  if (!g->d_dm && ((e = cudaMalloc(&g->d_dm, n * sizeof(double))) != cudaSuccess ||
                   (e = cudaMalloc(&g->d_dk, n * sizeof(double))) != cudaSuccess ||
                   (e = cudaMalloc(&g->d_tab, tab.size() * sizeof(double))) != cudaSuccess))
    return cuda_fail(e, "rm_grid_set_tau");
  RM_CUDA(cudaMemcpy(g->d_dm, dm, n * sizeof(double), cudaMemcpyHostToDevice), "rm_grid_set_tau");
  RM_CUDA(cudaMemcpy(g->d_dk, dk, n * sizeof(double), cudaMemcpyHostToDevice), "rm_grid_set_tau");
  RM_CUDA(cudaMemcpy(g->d_tab, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice), "rm_grid_set_tau");
  if (g->fft_ok) {
    std::vector<double> mt(n), kt(n);
    for (int a = 0; a < g->ny; ++a)
      for (int b = 0; b < g->nx; ++b) {
        mt[(size_t)b * g->ny + a] = dm[(size_t)a * g->nx + b];
        kt[(size_t)b * g->ny + a] = dk[(size_t)a * g->nx + b];
      }
    if (!g->d_dmT && ((e = cudaMalloc(&g->d_dmT, n * sizeof(double))) != cudaSuccess ||
                      (e = cudaMalloc(&g->d_dkT, n * sizeof(double))) != cudaSuccess))
      return cuda_fail(e, "rm_grid_set_tau");
    RM_CUDA(cudaMemcpy(g->d_dmT, mt.data(), n * sizeof(double), cudaMemcpyHostToDevice), "rm_grid_set_tau");
    RM_CUDA(cudaMemcpy(g->d_dkT, kt.data(), n * sizeof(double), cudaMemcpyHostToDevice), "rm_grid_set_tau");
    // tensor-core preconditioner: the orthonormal DST-I matrix of order nx (= ny), zero-padded to 256, FP16,
    // row-major (each CTA moves it into tensor memory once per launch)
    std::vector<uint16_t> hc((size_t)rm::tc::NS * rm::tc::NS, 0);
    const int nn = g->nx;
    const double c = sqrt(2.0 / (nn + 1));
    for (int a = 0; a < nn; ++a)
      for (int b = 0; b < nn; ++b) {
        const double v = c * sin(M_PI * (double)((a + 1) * (b + 1) % (2 * (nn + 1))) / (double)(nn + 1));
        hc[(size_t)a * rm::tc::NS + b] = __half_as_ushort(__float2half_rn((float)v));
      }
    if (!g->d_dstc && (e = cudaMalloc(&g->d_dstc, hc.size() * sizeof(uint16_t))) != cudaSuccess)
      return cuda_fail(e, "rm_grid_set_tau");
    RM_CUDA(cudaMemcpy(g->d_dstc, hc.data(), hc.size() * sizeof(uint16_t), cudaMemcpyHostToDevice), "rm_grid_set_tau");
  }
  g->lp_dmin = dm[0];
  g->lp_kmin = dk[0];
  for (size_t i = 1; i < n; ++i) {
    g->lp_dmin = std::min(g->lp_dmin, dm[i]);
    g->lp_kmin = std::min(g->lp_kmin, dk[i]);
  }
  if (g->nx == g->ny) {
    // FP16 DST-I matrix for the low-precision stages: row alpha-1, column kappa-1, zero beyond n
    // (rm_device.cuh Lp); |S| <= sqrt(2/(n+1)) and every nonzero entry is an FP16 normal number
    const int sh = np + 8, nn = g->nx;
    std::vector<uint16_t> h((size_t)np * sh, 0);
    const double c = sqrt(2.0 / (nn + 1));
    for (int a = 0; a < nn; ++a)
      for (int b = 0; b < nn; ++b) {
        const double v = c * sin(M_PI * (double)((a + 1) * (b + 1) % (2 * (nn + 1))) / (double)(nn + 1));
        h[(size_t)a * sh + b] = __half_as_ushort(__float2half_rn((float)v));
      }
    if (!g->d_dst16 && (e = cudaMalloc(&g->d_dst16, h.size() * sizeof(uint16_t))) != cudaSuccess)
      return cuda_fail(e, "rm_grid_set_tau");
    RM_CUDA(cudaMemcpy(g->d_dst16, h.data(), h.size() * sizeof(uint16_t), cudaMemcpyHostToDevice), "rm_grid_set_tau");
  }
  return RM_OK;
}

int rm_fail_info(rm_grid* g, int* code, int* n, int64_t* iterations, double* residual_norm) {
  if (!g) return fail(RM_EINVAL, "rm_fail_info: null grid");
  int flag = 0;
  double info[3] = {0, 0, 0};
  RM_CUDA(cudaMemcpy(&flag, g->d_fail, sizeof(int), cudaMemcpyDeviceToHost), "rm_fail_info");
  if (!flag) return 0;
  RM_CUDA(cudaMemcpy(info, g->d_fail_info, 3 * sizeof(double), cudaMemcpyDeviceToHost), "rm_fail_info");
  if (code) *code = flag;
  if (n) *n = (int)info[0];
  if (iterations) *iterations = (int64_t)info[1];
  if (residual_norm) *residual_norm = info[2];
  return 1;
}

int rm_debug_timing(rm_grid* g, long long* out16) {
  if (!g || !out16) return fail(RM_EINVAL, "rm_debug_timing: bad argument");
  RM_CUDA(cudaMemcpy(out16, g->d_timing, 16 * sizeof(long long), cudaMemcpyDeviceToHost), "rm_debug_timing");
  return RM_OK;
}

int rm_fail_reset(rm_grid* g, void* stream) {
  if (!g) return fail(RM_EINVAL, "rm_fail_reset: null grid");
  RM_CUDA(cudaMemsetAsync(g->d_fail, 0, sizeof(int), (cudaStream_t)stream), "rm_fail_reset");
  return RM_OK;
}

int rm_correct(int ndof, int nc, int m, double* d_u, int64_t u_stride, const double* d_uc, int64_t uc_stride,
               void* stream) {
  if (ndof < 1 || nc < 0 || m < 1 || !d_u || !d_uc) return fail(RM_EINVAL, "rm_correct: bad argument");
  RM_CUDA(rm::launch_correct(ndof, nc, m, d_u, u_stride, d_uc, uc_stride, (cudaStream_t)stream), "rm_correct");
  return RM_OK;
}

int rm_diff_sqnorm(int64_t n, const double* d_a, const double* d_b, double* d_out, void* stream) {
  if (n < 0 || !d_a || !d_b || !d_out) return fail(RM_EINVAL, "rm_diff_sqnorm: bad argument");
  RM_CUDA(rm::launch_diff_sqnorm(n, d_a, d_b, d_out, (cudaStream_t)stream), "rm_diff_sqnorm");
  return RM_OK;
}

int rm_vec_dot(int64_t n, const double* d_a, const double* d_b, double* d_out, void* stream) {
  if (n < 0 || !d_a || !d_b || !d_out) return fail(RM_EINVAL, "rm_vec_dot: bad argument");
  RM_CUDA(rm::launch_vec_dot(n, d_a, d_b, d_out, (cudaStream_t)stream), "rm_vec_dot");
  return RM_OK;
}

int rm_vec_axpby(int64_t n, double alpha, const double* d_x, double beta, const double* d_y, double* d_out,
                 void* stream) {
  if (n < 0 || !d_x || !d_y || !d_out) return fail(RM_EINVAL, "rm_vec_axpby: bad argument");
  RM_CUDA(rm::launch_vec_axpby(n, alpha, d_x, beta, d_y, d_out, (cudaStream_t)stream), "rm_vec_axpby");
  return RM_OK;
}

int rm_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t start,
                     int64_t count, int64_t row, double* d_out, int64_t out_stride, void* stream) {
  if (count < 0 || start < 0 || row < 1 || !d_out) return fail(RM_EINVAL, "rm_pcg64_uniform: bad argument");
  if (count == 0) return RM_OK;
  rm::PcgArgs a{state_hi, state_lo, inc_hi, inc_lo, start, count, row, d_out, out_stride};
  RM_CUDA(rm::launch_pcg64(a, (cudaStream_t)stream), "rm_pcg64_uniform");
  return RM_OK;
}

}  // extern "C"
