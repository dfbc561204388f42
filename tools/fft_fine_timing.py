"""Sub-phase cycles of the FFT chain kernel's two apply passes (CTA 0), from a -DRM_TIMING,RM_TIMING_FINE build:

    RM_DEFINES=RM_TIMING_FINE RM_LIB_OUT=/path/lib_fine.so python -c "from paper_1805_06688_b200 import build; build.build(timing=True, force=True)"
    RM_LIB=/path/lib_fine.so python tools/fft_fine_timing.py
"""
import fft_phase_timing as base

base.NAMES = ["col: stage from L2", "col: forward FFTs (18 on 16 warps)", "col: combine", "col: inverse FFTs",
              "col: store WV", "apply: group barrier", "row: load + forward FFTs", "row: combine",
              "row: inverse FFTs", "row: add WV", "col: (FP32) symbol copies", "col: staging loads + stores", "", "", "", ""]

if __name__ == "__main__":
    base.main()
