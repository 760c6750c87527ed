"""B200-native data-parallel CNN training step (arXiv 1709.06622 hot path).

Layout:
  csrc/host      traincap:: C++ planner (decisions: Eq 1-6, Lemma 1/2)
  csrc/cuda      sm_100a kernels (tcgen05 implicit-GEMM conv, Winograd, FFT,
                 pools, fused momentum-SGD)
  csrc/runtime   HBM arena + step executor + NCCL parameter-server shards
  lib/           the built libtraincap.so / libtcb.so (in-tree)
"""
__all__ = ["planner"]
