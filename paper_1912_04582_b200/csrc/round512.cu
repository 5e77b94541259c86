// 512-thread-CTA build of the exact-Gram rounding kernel (namespace
// ttdvm::g512): the same source as round.cu's ttdvm::g128 kernels.  The
// high-rank bins of the step (summed ranks at or above the mode size: T
// route, 44..64 x ~100 operands, ~200 KB of shared memory per output, so one
// CTA per SM) are bound by the latency of their double-double Gram chains;
// sixteen warps per output instead of eight hide twice as much of it.
#define TTDVM_ROUND_NT 512
#define TTDVM_GRAM_ONLY 1
#include "round.cu"
