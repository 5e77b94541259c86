// Shared device-side types of the TT-DVM CUDA library (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ttdvm {

constexpr int kMaxSets = 12;
constexpr int kMaxTerms = 16;     // summands per rounded output
constexpr int kAccSlots = 64;     // spread slots of the per-launch work counters
constexpr int kRoundThreads = 128;
// rank bins of a rounding launch: upper edges of max(R1, R2) of the summed input
constexpr int kRankBins = 11;
// per-bin maxima written by the bin kernel: R1, R2, staged-slice doubles,
// summands, doubles of the distinct operand tensors (operand cache)
constexpr int kBinWords = 5;
__device__ __constant__ const int kRankEdges[kRankBins] = {4, 8, 12, 16, 24, 32, 48, 64, 96, 128,
                                                           1 << 30};

// A set of packed TT tensors (ttdvm_tt_batch layout) resident in an arena.
struct TSet {
  const int* ranks;        // [2*count]
  const long long* off;    // [count]
  const double* base;
  const double* tscale;    // optional per-tensor scale (e.g. nu of J)
  double uscale;           // uniform scale (e.g. dt for R)
};

// One summand of a rounded output:
//   scale * dscale[dsi] * (fset[fidx] o factor o reflect(set[idx])).
// factor (fac >= 0) indexes a rank-1 face factor u1 (x) u2 (x) u3 in
// RoundArgs::factors (the axis-aligned (xi.n)^{+/-});
// fset >= 0 names a TT Hadamard factor (oblique-normal xi_n and |xi_n|
// estimate, T12/T13) taken from another set; refl (1..3) is the specular-
// ghost index reversal (T9 / T20) of the set[idx] operand; dsi >= 0 picks a
// per-step scale computed on the device (the wall-ghost density n_w, T19).
struct Term {
  int set;
  int idx;
  double scale;
  int fac = -1;
  int refl = 0;
  int fset = -1;
  int fidx = 0;
  int dsi = -1;
};

struct RoundOut {
  int* ranks;                   // [2*nout]
  long long* off;               // [nout]
  double* base;
  unsigned long long* used;     // bump counter (doubles)
  long long capacity;           // doubles
};

// status words written by kernels (device memory, read back by the host)
enum StatusWord {
  kStOverflow = 0,  // an output did not fit its arena
  kStMaxR1 = 1,
  kStMaxR2 = 2,
  kStError = 3,     // 0 ok, else error code (see kErr*)
  kStErrIdx = 4,    // index of the first failing item
  kStAux = 5,       // kernel-specific counter (face factors: imprecise normals)
  kStWords = 8
};
enum ErrCode {
  kErrNone = 0,
  kErrDensity = 1,
  kErrTemperature = 2,
  kErrNonFinite = 3,
  kErrZeroFactor = 4,      // face factor of an all-zero operand
  kErrWallDegenerate = 5,  // wall_ghost: degenerate wall Maxwellian flux
  kErrWallDensity = 6      // wall_ghost: nonpositive balance density
};

struct RoundArgs {
  TSet sets[kMaxSets];
  const long long* term_off;    // [nout+1] CSR into terms
  const Term* terms;
  const double* factors;        // [nfac][n1+n2+n3]
  const double* dscale;         // per-step device scales (Term::dsi)
  const int* olist;             // optional: block b rounds output olist[b] (rank bins)
  int n1, n2, n3;
  int nout;
  double eps;
  int cap;
  RoundOut out;
  int* status;                  // [kStWords]
  double* margins;              // optional [2*nout]
  double* acc;                  // [2 * kAccSlots]: canonical FLOPs, compulsory bytes
  unsigned long long* prof;     // optional [16] per-phase SM cycles (diagnostics)
  // shared-memory plan (doubles), chosen by the host launcher
  int RM1, RM2;                 // bounds on the summed input ranks
  int HMAX;                     // rows of the TSQR block buffer
  int MSMAX;                    // doubles of the staged middle slices
  int JB;                       // slices per barrier phase (exact-Gram kernel)
  int no_dmma;                  // diagnostics (TTDVM_DMMA=0): slice products on the FMA strips
  int OC;                       // doubles of the shared-memory operand cache (0 = off): every
                                // distinct operand tensor of an output is fetched whole by one
                                // cp.async.bulk (TMA) at set-up and read from shared memory after
  // spill plan (working sets above the shared-memory budget: n = 64, large
  // summed ranks): the four largest buffers live in a per-CTA global scratch
  // slice (L1/L2-resident) and the launch is persistent over nblk outputs
  double* gscratch;             // [gridDim.x * gstride] or null
  long long gstride;            // doubles per CTA slice
  int nblk;                     // outputs of this launch (persistent loop bound)
};

}  // namespace ttdvm
