"""B200-native SGAD-SLAM hot paths (mapping rasterizer fwd+bwd, GICP tracking).

Drop-in for the reference ``raysplat`` render/track API on CUDA tensors; the
compute runs in libsgad.so (hand-written sm_100a kernels behind a C ABI,
include/sgad.h).  See DESIGN.md.
"""

__version__ = "0.1.0"
