"""paper_1204_3853_b200 -- B200-native (sm_100a, fp64) hot path of Hittinger & Banks,
"Block-Structured Adaptive Mesh Refinement Algorithms for Vlasov Simulation" (arXiv:1204.3853).

The compute path is libvlasov.so (hand-written CUDA, C ABI in include/vlasov.h); this package is
its thin binding (``api``) plus the step orchestration (``solver``).  There is no CPU fallback:
importing ``api`` fails if the library is not built, and compute calls fail without an sm_100
device.
"""
__version__ = "0.1.0"
