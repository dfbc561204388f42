// tcgen05 (5th-generation tensor core) building blocks of the FFT chain kernel's tau preconditioner: the four
// sine-transform stages of P^-1 = (Sy x Sx) D^-1 (Sy x Sx) at order 255 are 256 x 256 x 32 GEMMs per CTA,
//     D[k][n] = sum_i S[k][i] X[n][i],      S = orthonormal DST-I matrix (FP16, symmetric), X = a 32-row strip,
// issued as tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = 32, K = 16; two M tiles, sixteen K steps).  S is the
// A operand and stays RESIDENT IN TENSOR MEMORY for the whole kernel (256 of the CTA's 512 columns: rows on the
// lanes, two halves of K per 32-bit column), the strip is the B operand in shared memory (no-swizzle K-major
// canonical layout, 8 x 16-byte core matrices) and the FP32 accumulator lives in tensor memory, read back with
// tcgen05.ld.  (A shared-memory-A variant with a bulk-copied canonical S is kept for tools/tc_dst_test.cu.)
//
// The preconditioner only steers the PCG iteration (every stop is decided on the FP64 true residual), which is why
// FP16 operands with FP32 accumulation are admissible here and nowhere else in the kernel.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace rm {
namespace tc {

constexpr int NS = 256;                 // padded transform order
constexpr int NB = 32;                  // strip rows (N of the MMA)
constexpr int A_BYTES = NS * NS * 2;    // 131072
constexpr int B_LBO = NB * 16 + 16;     // bytes between successive 8-wide K groups of the strip operand: one
                                        // 16-byte pad per group spreads the groups over the shared-memory banks
constexpr int B_BYTES = (NS / 8) * B_LBO;  // 16896
constexpr int TMEM_COLS = 64;           // two M tiles x 32 FP32 columns (S staged in shared memory)
// S resident in tensor memory (A operand from TMEM): two M tiles x 128 columns (256 halves of K, two per 32-bit
// column) followed by the accumulator; the allocation is the next power of two
constexpr int TMEM_S_COLS = 256;
constexpr int TMEM_D_COL = TMEM_S_COLS;
constexpr int TMEM_COLS_RESIDENT = 512;

// canonical K-major layout without swizzle: 8 rows x 8 halves (16 bytes per row) form one contiguous 128-byte core
// matrix; core matrices of consecutive 8-row groups follow each other (stride byte offset 128), the next 8 values
// of K start after all rows (leading byte offset = rows x 16)
__host__ __device__ constexpr int a_index(int r, int k) {
  return (k >> 3) * (NS * 8) + (r >> 3) * 64 + (r & 7) * 8 + (k & 7);
}
__host__ __device__ constexpr int b_index(int n, int k) {
  return (k >> 3) * (B_LBO / 2) + (n >> 3) * 64 + (n & 7) * 8 + (k & 7);
}

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// spin on the barrier's phase; a barrier that never completes traps instead of hanging the device
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_u32(bar);
  const long long t0 = clock64();
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) break;
    if (clock64() - t0 > 4000000000ll) __trap();
  }
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// one warp allocates (and later frees) the CTA's tensor-memory columns; the base address lands in shared memory
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t addr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(addr), "r"(cols) : "memory");
}

// shared-memory matrix descriptor (version 1, no swizzle): start address, leading / stride byte offsets in 16-byte units
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo_bytes >> 4) << 16) | ((uint64_t)(sbo_bytes >> 4) << 32) |
         (1ull << 46);
}

// instruction descriptor: FP32 accumulator, FP16 A and B, both K-major, M x N
__host__ __device__ constexpr uint32_t instr_desc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)accumulate)
      : "memory");
}

// arrive on the mbarrier once every MMA issued so far by this thread has completed
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// the whole stage: D (tensor memory, columns [0, 32) = rows 0..127 of the product, [32, 64) = rows 128..255) =
// S (sA, canonical) x X^T (sB, canonical); one thread issues
__device__ __forceinline__ void issue_dst_mma(const __half* sA, const __half* sB, uint32_t tmem) {
  constexpr uint32_t idesc = instr_desc_f16(128, NB);
  const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
#pragma unroll
  for (int t = 0; t < 2; ++t) {
#pragma unroll
    for (int ks = 0; ks < NS / 16; ++ks) {
      const uint64_t ad = smem_desc(a0 + t * (128 * 16) + ks * 2 * (NS * 16), NS * 16, 128);
      const uint64_t bd = smem_desc(b0 + ks * 2 * B_LBO, B_LBO, 128);
      mma_f16(tmem + (uint32_t)(NB * t), ad, bd, idesc, ks > 0);
    }
  }
}

// A operand from tensor memory (rows = lanes, K packed two halves per 32-bit column, 8 columns per K = 16 step)
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"((uint32_t)accumulate)
      : "memory");
}

// the whole stage with S resident in tensor memory: D (columns TMEM_D_COL + 32 t) = S (columns 128 t ..) x X^T (sB)
__device__ __forceinline__ void issue_dst_mma_ts(const __half* sB, uint32_t tmem) {
  constexpr uint32_t idesc = instr_desc_f16(128, NB);
  const uint32_t b0 = smem_u32(sB);
#pragma unroll
  for (int t = 0; t < 2; ++t) {
#pragma unroll
    for (int ks = 0; ks < NS / 16; ++ks) {
      const uint64_t bd = smem_desc(b0 + ks * 2 * B_LBO, B_LBO, 128);
      mma_f16_ts(tmem + (uint32_t)(TMEM_D_COL + NB * t), tmem + (uint32_t)(128 * t + 8 * ks), bd, idesc, ks > 0);
    }
  }
}

// The same stage issued by four threads (one per warp quarter group), each one M tile x one half of K into its own
// accumulator: issuer u = 2 t + kh writes columns TMEM_D_COL + 32 u; the reader adds the two K halves.  The MMA of
// a 128 x 32 x 16 tile is shorter than its single-thread issue interval, so the issue is what gets parallelised.
__device__ __forceinline__ void issue_dst_mma_ts_part(const __half* sB, uint32_t tmem, int u) {
  constexpr uint32_t idesc = instr_desc_f16(128, NB);
  const uint32_t b0 = smem_u32(sB);
  const int t = u >> 1, kh = u & 1;
#pragma unroll
  for (int k8 = 0; k8 < NS / 32; ++k8) {
    const int ks = kh * (NS / 32) + k8;
    const uint64_t bd = smem_desc(b0 + ks * 2 * B_LBO, B_LBO, 128);
    mma_f16_ts(tmem + (uint32_t)(TMEM_D_COL + NB * u), tmem + (uint32_t)(128 * t + 8 * ks), bd, idesc, k8 > 0);
  }
}

// 32 lanes x 16 consecutive 32-bit columns from registers into the warp's tensor-memory lane quarter
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// load the row-major FP16 matrix S[256][256] (global) into tensor-memory columns [0, 256) of `tmem`; called by
// all 16 warps of the CTA (warp w: lane quarter w & 3, 64-column part w >> 2), followed by a CTA barrier
__device__ __forceinline__ void load_matrix_tmem(uint32_t tmem, const __half* s_rowmajor, int warp, int lane) {
  const int q = warp & 3, part = warp >> 2;
  const uint32_t* s32 = reinterpret_cast<const uint32_t*>(s_rowmajor);
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int col = 64 * part + 16 * g;          // tensor-memory column = 128 t + (k / 2)
    const int t = col >> 7, cc = col & 127;
    const int row = 128 * t + 32 * q + lane;
    const uint4* src = reinterpret_cast<const uint4*>(s32 + row * 128 + cc);
    uint32_t r[16];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const uint4 x = __ldg(src + v);
      r[4 * v] = x.x;
      r[4 * v + 1] = x.y;
      r[4 * v + 2] = x.z;
      r[4 * v + 3] = x.w;
    }
    tmem_st16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)col, r);
  }
  tmem_wait_st();
}

// 32 lanes x 16 consecutive FP32 columns of the warp's tensor-memory lane quarter
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// bulk async copy of the 128 KB canonical matrix into shared memory; completion on `bar` (one arrival + bytes)
__device__ __forceinline__ void load_matrix_async(__half* sA, const __half* gA, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"((uint32_t)A_BYTES) : "memory");
  constexpr int CH = 32768;
#pragma unroll
  for (int o = 0; o < A_BYTES; o += CH)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sA) + o),
                 "l"(reinterpret_cast<const char*>(gA) + o), "r"((uint32_t)CH), "r"(b)
                 : "memory");
}
#endif  // __CUDACC__

}  // namespace tc
}  // namespace rm
