"""Algorithmic FLOP counts of the hot path's two kernels-within-the-kernel.

Used by bench.py (roofline "achieved") and tools/profile_solve.py.  Counts are the arithmetic the
algorithm as implemented needs, not what the tensor cores execute on zero padding.
"""

from __future__ import annotations


def fmv(nx: int, ny: int, merge: int = 0) -> float:
    """One combined-operator apply (M + s K) v: per direction a diagonal-block Toeplitz product
    along every row, plus the two off-diagonal ones (rows j+-1) -- or, when the off-diagonal block is
    shifted-symmetric (``merge`` bit, rm_grid_flags), one length-(n+1) product of the pre-added
    neighbours.  The P1 mass and the step scale s are folded into the Toeplitz tables once per step
    (rm_device.cuh build_step_tables), so they add no per-apply arithmetic."""
    fx = 2.0 * nx * nx * ny + (2.0 * nx * (nx + 1) * ny + nx * ny if merge & 1 else 2.0 * nx * nx * 2 * (ny - 1))
    fy = 2.0 * ny * ny * nx + (2.0 * ny * (ny + 1) * nx + nx * ny if merge & 2 else 2.0 * ny * ny * 2 * (nx - 1))
    return fx + fy


def fpc(nx: int, ny: int) -> float:
    """One tau-preconditioner application: two even/odd-folded DST-I contractions per direction
    (half the dense count), the folds and the diagonal scaling."""
    return 2.0 * nx * ny * (nx + ny) + 5.0 * nx * ny


def fpc_dense(nx: int, ny: int) -> float:
    """One tau-preconditioner application as the FP16 tensor-core path executes it: four unfolded
    DST-I contractions (rm_device.cuh Lp), 2 n^3 each on an n x n grid, plus the diagonal scaling."""
    return 4.0 * nx * ny * (nx + ny) + nx * ny


def fmv_split16(nx: int, ny: int) -> float:
    """One split-FP16 operator apply inside the PCG iteration (rm_device.cuh Mx) as executed: three
    unmerged Toeplitz segments per direction, each a three-term split product (hi*hi + lo*hi + hi*lo)."""
    return 3.0 * (3 * 2.0 * nx * nx * ny + 3 * 2.0 * ny * ny * nx)


def fft_flops(L: int) -> float:
    """One complex FFT of length L (conventional 5 L log2 L)."""
    import math

    return 5.0 * L * math.log2(L)


def fmv_fft(nx: int, ny: int) -> float:
    """One operator apply by the FFT kernel (csrc/rm_fft.cu), algorithmic: per direction, the rows (columns)
    as ceil(n/2) packed complex pairs, a forward and an inverse L-point FFT each (L = 2(n+1)), the three-term
    symbol combination (3 complex multiplies + 2 adds per point), plus the final scale-and-add."""
    L = 2 * (max(nx, ny) + 1)
    px, py = (ny + 1) // 2, (nx + 1) // 2
    per_pair = 2.0 * fft_flops(L) + 22.0 * L
    return (px + py) * per_pair + 2.0 * nx * ny


def fpc_fft(nx: int, ny: int) -> float:
    """One tau-preconditioner application by the FFT kernel: four DST-I passes (one odd-extended L-point FFT
    per packed pair) and the diagonal scaling."""
    L = 2 * (max(nx, ny) + 1)
    return 2.0 * ((ny + 1) // 2 + (nx + 1) // 2) * fft_flops(L) + 2.0 * nx * ny


def fpc_tc(nx: int, ny: int) -> float:
    """One tau-preconditioner application on the 5th-generation tensor cores as executed (csrc/rm_tc.cuh): four
    DST-I stages, each a dense 256 x 256 GEMM against every row / column of the padded 256 x 256 grid."""
    n = 256 if max(nx, ny) <= 255 else 2 * (max(nx, ny) + 1)
    return 4.0 * 2.0 * n * n * n


# legacy mma.sync m16n8k16 FP16 -> FP32 on B200, measured with tools/lowp_peak.cu (profiles/r01_lowp_peak.txt)
FP16_MMA_SYNC_PEAK_TFLOPS = 555.0
