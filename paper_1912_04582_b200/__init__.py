"""B200-native TT-DVM explicit step (arXiv 1912.04582 hot path).

Product package: the CUDA C-ABI library (csrc/, built in-tree as
libttdvm_cuda.so) and its host-side mirror of the reference interface.
"""
