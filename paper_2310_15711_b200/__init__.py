"""B200-native Hash Chain (HC) exact string matcher (arXiv 2310.15711).

The search runs in hand-written sm_100a CUDA kernels behind the C-ABI of
``include/hc.h`` (``libhc.so``).  ``paper_2310_15711_b200.hc`` is the thin
ctypes binding; ``paper_2310_15711_b200.inputs`` holds the seeded synthetic
inputs.  Submodules are imported explicitly (``from paper_2310_15711_b200
import hc``) so the input generators work without the CUDA library.
"""
