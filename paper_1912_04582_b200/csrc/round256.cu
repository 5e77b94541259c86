// 256-thread-CTA build of the exact-Gram rounding kernel (namespace
// ttdvm::g256): the same source as round.cu's ttdvm::g128 kernels.  The host
// plan (capi.cu run_round) takes it for the rank bins with larger Gram
// dimensions, where more threads per dense slice product pay off.
#define TTDVM_ROUND_NT 256
#define TTDVM_GRAM_ONLY 1
#include "round.cu"
