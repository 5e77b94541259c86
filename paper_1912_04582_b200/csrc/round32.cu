// One-warp-CTA build of the exact-Gram rounding kernel (namespace
// ttdvm::g32): the same source as round.cu's ttdvm::g128 kernels.  Every
// CTA barrier is a warp barrier, so the short phases of tiny roundings
// (Gram dimension D <= TTDVM_NARROW_D: f_S, collision and most update sums)
// run without block synchronisation, many outputs in flight per SM.
#define TTDVM_ROUND_NT 32
#define TTDVM_GRAM_ONLY 1
#include "round.cu"
