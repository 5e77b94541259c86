// Block-level FP64 linear-algebra helpers shared by the rounding and
// face-factor kernels (one CTA of kRoundThreads threads per problem).
// Everything sits in an anonymous namespace: each translation unit gets its
// own copy (no relocatable device code).
#pragma once

#include <math.h>

#include "ttdvm_device.cuh"

namespace ttdvm {
namespace {

// A translation unit may build the helpers for another CTA width
// (round256.cu sets 256 for the wide rounding kernel).
#ifndef TTDVM_ROUND_NT
#define TTDVM_ROUND_NT 128
#endif
static_assert(TTDVM_ROUND_NT == kRoundThreads || TTDVM_ROUND_NT == 256 || TTDVM_ROUND_NT == 32 ||
                  TTDVM_ROUND_NT == 512,
              "CTA width");
constexpr int NT = TTDVM_ROUND_NT;
constexpr int NW = NT / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int W>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) s += red[w];
  return s;
}

// FP64 reciprocal and reciprocal square root with an FP32 seed and two
// Newton steps in FP64 (23 -> 46 -> 92 bits, i.e. correct to a few ulps):
// the IEEE-exact double div/sqrt sequences sit on the serial critical path
// of every Householder and Jacobi step.  Exponents are split off exactly so
// the FP32 seed never over- or underflows.
__device__ __forceinline__ double fast_rcp(double x) {
  const long long bits = __double_as_longlong(x);
  const int e = (int)((bits >> 52) & 0x7ff) - 1023;
  const double m = __longlong_as_double((bits & ~(0x7ffLL << 52)) | (1023LL << 52));  // [1,2)
  double r = (double)__frcp_rn((float)m);
  r = r * (2.0 - m * r);
  r = r * (2.0 - m * r);
  return r * __longlong_as_double((long long)(1023 - e) << 52);
}

__device__ __forceinline__ double fast_rsqrt(double x) {  // x > 0, normal
  const long long bits = __double_as_longlong(x);
  int e = (int)((bits >> 52) & 0x7ff) - 1023;
  const int odd = e & 1;
  e -= odd;  // even exponent: x = m * 2^e, m in [1, 4)
  const double m = __longlong_as_double((bits & ~(0x7ffLL << 52)) | ((long long)(1023 + odd) << 52));
  double r = (double)rsqrtf((float)m);
  r = r * (1.5 - 0.5 * m * r * r);
  r = r * (1.5 - 0.5 * m * r * r);
  return r * __longlong_as_double((long long)(1023 - e / 2) << 52);
}

// LAPACK dlarfg on (alpha, ||x||^2): H = I - tau v v^T, v = [1; x*scale],
// tau = (beta - alpha)/beta = 1 - alpha/beta, with 1/|beta| from one rsqrt.
__device__ __forceinline__ void larfg(double alpha, double sigma2, double& beta, double& tau,
                                      double& scale) {
  if (sigma2 == 0.0) {
    beta = alpha;
    tau = 0.0;
    scale = 0.0;
    return;
  }
  const double h = alpha * alpha + sigma2;
  const double ri = fast_rsqrt(h);
  const double nrm = h * ri;
  beta = alpha >= 0.0 ? -nrm : nrm;
  const double rb = alpha >= 0.0 ? -ri : ri;  // 1 / beta
  tau = 1.0 - alpha * rb;
  scale = fast_rcp(alpha - beta);
}

// Visit (r, c) in [0, rows) x [0, cols) without integer division: threads
// are split into power-of-two row lanes (r = tid & (rp - 1), rp <= NT) and
// column strides; rows beyond rp wrap in an inner loop.  One code path per
// lambda (instruction-cache footprint matters: the rounding kernel is
// latency-bound and several CTAs per SM run different phases).  No
// barriers or shuffles may be used inside f.
constexpr int LOG_NT = NT == 32 ? 5 : (NT == 64 ? 6 : (NT == 128 ? 7 : (NT == 256 ? 8 : 9)));
template <class Fn>
__device__ __forceinline__ void for2d(int rows, int cols, Fn&& f) {
  if (rows <= 0 || cols <= 0) return;
  int lg = rows <= 1 ? 0 : 32 - __clz(rows - 1);
  lg = lg < LOG_NT ? lg : LOG_NT;
  const int rp = 1 << lg;
  const int r0 = threadIdx.x & (rp - 1);
  if (r0 >= rows) return;
  const int step = NT >> lg;
  for (int c = threadIdx.x >> lg; c < cols; c += step)
#pragma unroll 1
    for (int r = r0; r < rows; r += rp) f(r, c);
}

__device__ __forceinline__ int floor_pow2(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}
// Jacobi stopping rule: stop after a sweep in which every coupling
// gamma^2 / (alpha beta) stayed below TTDVM_JACOBI_BIG2.  By the quadratic
// convergence of cyclic Jacobi the couplings left after that sweep are
// O(TTDVM_JACOBI_BIG2).  The rounding kernels use 1e-10: the left-over
// couplings (~1e-10 relative) perturb the kept singular values by ~1e-20
// and the bases by ~1e-10, far below any rounding tolerance the step uses,
// and about one sweep in 2.4 is saved (config-4 flux phase -3 %, same-box
// A/B in scripts/gpu_ab_jacobi.sh).  facefactor.cu (from_full at 1e-12)
// keeps 1e-18.
#ifndef TTDVM_JACOBI_BIG2
#define TTDVM_JACOBI_BIG2 1e-10
#endif
// One-sided (Hestenes) Jacobi on the columns of X (m x c, ld ldx) with
// tracked squared column norms (one dot product per pair and round; the
// norms are refreshed at every sweep).
// TTDVM_JACOBI_UNROLL: unroll factor of the row loops of a pair (1 in the
// rounding kernels, whose instruction footprint matters; facefactor.cu,
// latency-bound at 8 warps per SM, batches the loads of 4 rows).
#ifndef TTDVM_JACOBI_UNROLL
#define TTDVM_JACOBI_UNROLL 1
#endif
constexpr int kJacobiUnroll = TTDVM_JACOBI_UNROLL;
template <int TPP>
__device__ int jacobi_t(double* X, int ldx, int m, int c, double* nrm) {
  const int cp = c + (c & 1);
  const int npairs = cp / 2;
  const int pi = threadIdx.x / TPP, sub = threadIdx.x % TPP;
  const double tol2 = 1e-30;  // (1e-15)^2, |gamma| > 1e-15 sqrt(alpha beta)
  for (int sweep = 0; sweep < 60; ++sweep) {
    for (int j = threadIdx.x; j < c; j += NT) {
      double s = 0.0;
#pragma unroll 1
      for (int i = 0; i < m; ++i) s += X[i + ldx * j] * X[i + ldx * j];
      nrm[j] = s;
    }
    __syncthreads();
    bool rotated = false;
    bool big = false;  // some rotation in this sweep had |gamma| > 1e-9 sqrt(alpha beta)
    for (int r = 0; r < cp - 1; ++r) {
      for (int base = 0; base < npairs; base += NT / TPP) {
        const int pp = base + pi;
        // round-robin pairs: a = (pp + r - 1) mod (cp - 1) + 1 (pp > 0),
        // b = (cp - 2 - pp + r) mod (cp - 1) + 1; both arguments < 2 (cp - 1)
        int a = pp + r - 1;
        if (a >= cp - 1) a -= cp - 1;
        a = pp == 0 ? 0 : a + 1;
        int b = cp - 2 - pp + r;
        if (b >= cp - 1) b -= cp - 1;
        b += 1;
        const bool live = pp < npairs && a < c && b < c;
        double ga = 0.0;
#if TTDVM_JACOBI_UNROLL > 1
        double* __restrict__ x = X + ldx * (live ? a : 0);  // a != b: distinct columns
        double* __restrict__ y = X + ldx * (live ? b : 0);
#else
        double* x = X + ldx * (live ? a : 0);
        double* y = X + ldx * (live ? b : 0);
#endif
        if (live)
#pragma unroll kJacobiUnroll
          for (int i = sub; i < m; i += TPP) ga += x[i] * y[i];
        ga = group_sum<TPP>(ga);
        if (live && ga != 0.0) {
          const double al = nrm[a], be = nrm[b];
          if (ga * ga > tol2 * al * be) {
            big = big || (ga * ga > TTDVM_JACOBI_BIG2 * al * be);
            // t = sign(d) 2 ga / (|d| + sqrt(d^2 + 4 ga^2)), d = be - al: the
            // angle needs no more than FP32 accuracy (an inexact angle only
            // slows convergence); cs, sn are normalised in FP64 so the
            // rotation stays orthogonal to working precision.
            const double d = be - al;
            const double mag = fmax(fabs(d), 2.0 * fabs(ga));
            const int ex = (int)((__double_as_longlong(mag) >> 52) & 0x7ff) - 1023;
            const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
            const float df = (float)(d * sc), gf = (float)(ga * sc);
            const float tf = copysignf(1.0f, df) * (2.0f * gf) /
                             (fabsf(df) + sqrtf(df * df + 4.0f * gf * gf));
            const double t = (double)tf;
            rotated = rotated || (tf != 0.0f);  // an FP32-underflowed angle is converged
            const double cs = fast_rsqrt(1.0 + t * t), sn = cs * t;
#pragma unroll kJacobiUnroll
            for (int i = sub; i < m; i += TPP) {
              const double xi = x[i], yi = y[i];
              x[i] = cs * xi - sn * yi;
              y[i] = sn * xi + cs * yi;
            }
            if (sub == 0) {
              const double c2 = cs * cs, tg = 2.0 * t * ga, t2 = t * t;
              nrm[a] = c2 * (al - tg + t2 * be);
              nrm[b] = c2 * (be + tg + t2 * al);
            }
          }
        }
      }
      __syncthreads();
    }
    // rotations in this sweep were all below 1e-9 of the column norms: by
    // the quadratic convergence of cyclic Jacobi the remaining couplings
    // are O(1e-18), below the 1e-15 threshold -- no verification sweep
    const int any_rot = __syncthreads_or(rotated ? 1 : 0);
    const int any_big = __syncthreads_or(big ? 1 : 0);
    if (!any_rot || !any_big) return sweep + 1;
  }
  return 60;
}

__device__ __noinline__ int jacobi(double* X, int ldx, int m, int c, double* nrm) {
  const int npairs = (c + 1) / 2;
  const int tpp = min(32, floor_pow2(max(1, NT / max(npairs, 1))));
  switch (tpp) {
    case 32: return jacobi_t<32>(X, ldx, m, c, nrm);
    case 16: return jacobi_t<16>(X, ldx, m, c, nrm);
    case 8: return jacobi_t<8>(X, ldx, m, c, nrm);
    case 4: return jacobi_t<4>(X, ldx, m, c, nrm);
    case 2: return jacobi_t<2>(X, ldx, m, c, nrm);
    default: return jacobi_t<1>(X, ldx, m, c, nrm);
  }
}

// proj/src/tt_tensor.cpp:18-29, plus the decision margin.
__device__ int truncation_rank(const double* sigma, int len, double budget2, int cap,
                               double* margin) {
  int r = len;
  double tail = 0.0;
  double mg = INFINITY;
  while (r > 1) {
    const double s2 = sigma[r - 1] * sigma[r - 1];
    if (tail + s2 > budget2) {
      mg = fmin(mg, (tail + s2 - budget2));
      break;
    }
    tail += s2;
    --r;
  }
  mg = fmin(mg, budget2 - tail);
  if (cap > 0 && r > cap) r = cap;
  if (margin) *margin = budget2 > 0.0 ? mg / budget2 : INFINITY;
  return r;
}

struct SvdWork {
  unsigned long long* prof;  // optional sweep counter
  double* Xs;    // mx x mx
  double* vn;    // mx
  double* sig;   // mx
  double* sraw;  // mx
  int* piv;      // mx
  int* perm;     // mx
  double* sh;
  int ldx;
};
// ---- double-double arithmetic for the exact Gram route -------------------
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

// (hi, lo) += a * b with the product and the sum error kept in lo
__device__ __forceinline__ void dd_fma_acc(double& hi, double& lo, double a, double b) {
  const double p = a * b;
  const double pe = fma(a, b, -p);
  double s, e;
  two_sum(hi, p, s, e);
  hi = s;
  lo += e + pe;
}

__device__ __forceinline__ void dd_norm(double& hi, double& lo) {
  double s, e;
  two_sum(hi, lo, s, e);
  hi = s;
  lo = e;
}

// (a_hi, a_lo) * (b_hi, b_lo) -> (p, pe), unnormalised
__device__ __forceinline__ void dd_mul(double ah, double al, double bh, double bl, double& p,
                                       double& pe) {
  p = ah * bh;
  pe = fma(ah, bh, -p) + (ah * bl + al * bh);
}

// Visit the upper triangle (i <= j) of a d x d matrix: entry e -> (i, j).
__device__ __forceinline__ void tri_index(int e, int d, int& i, int& j) {
  int row = 0, len = d;
  while (e >= len) {
    e -= len;
    ++row;
    --len;
  }
  i = row;
  j = row + e;
}

// Pivoted Cholesky of the symmetric PSD matrix G (d x d, hi/lo planes, ld
// d) in double-double: Pi^T G Pi = R^T R, stopping when the largest
// remaining pivot is <= thresh.  R (k x d, ld ldr, columns in pivoted
// order) is rounded to double; piv[v] = original index of virtual column v.
// Returns the rank k.
__device__ __noinline__ int chol_piv_dd(double* Gh, double* Gl, int d, double thresh, double* R, int ldr,
                           int* piv, double* sh) {
  for (int t = threadIdx.x; t < d; t += NT) piv[t] = t;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int k = 0;
  for (; k < d; ++k) {
    double bv = -1.0;
    int bi = k;
    for (int v = k + lane; v < d; v += 32) {
      const int o = piv[v];
      const double g = Gh[o + d * o];
      if (g > bv) {
        bv = g;
        bi = v;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (!(bv > thresh)) break;  // uniform: every warp found the same maximum
    __syncthreads();            // everyone has read piv
    if (bi != k)  // earlier rows of R follow the column swap (one row per thread)
      for (int r = threadIdx.x; r < k; r += NT) {
        const double a = R[r + ldr * k];
        R[r + ldr * k] = R[r + ldr * bi];
        R[r + ldr * bi] = a;
      }
    if (threadIdx.x == 0) {
      const int q = piv[k];
      piv[k] = piv[bi];
      piv[bi] = q;
      const int o = piv[k];
      const double ah = Gh[o + d * o], al = Gl[o + d * o];
      const double s = sqrt(ah);
      const double p = s * s, pe = fma(s, s, -p);
      const double r = ((ah - p) - pe + al) * (0.5 / s);
      double sh_, sl_;
      two_sum(s, r, sh_, sl_);
      sh[0] = sh_;
      sh[1] = sl_;
      sh[2] = 1.0 / sh_;
    }
    __syncthreads();
    const int pk = piv[k];
    const double rh = sh[0], rl = sh[1], rinv = sh[2];
    // row k: R_kj = G[pk, p_j] / r_kk, kept in G's row pk (dd)
    for (int v = k + 1 + threadIdx.x; v < d; v += NT) {
      const int o = piv[v];
      const double ah = Gh[pk + d * o], al = Gl[pk + d * o];
      const double q1 = ah * rinv;
      double p, pe;
      dd_mul(q1, 0.0, rh, rl, p, pe);
      const double res = ((ah - p) - pe) + al;
      const double q2 = res * rinv;
      double qh, ql;
      two_sum(q1, q2, qh, ql);
      Gh[pk + d * o] = qh;
      Gl[pk + d * o] = ql;
      R[k + ldr * v] = qh + ql;
    }
    if (threadIdx.x == 0) R[k + ldr * k] = rh + rl;
    __syncthreads();
    // trailing update G[p_i, p_j] -= R_ki R_kj, i, j > k
    const int m = d - k - 1;
    for2d(m, m, [&](int a, int b) {
      const int oi = piv[k + 1 + a], oj = piv[k + 1 + b];
      double p, pe;
      dd_mul(Gh[pk + d * oi], Gl[pk + d * oi], Gh[pk + d * oj], Gl[pk + d * oj], p, pe);
      double s, e;
      two_sum(Gh[oi + d * oj], -p, s, e);
      double lo = Gl[oi + d * oj] + e - pe;
      dd_norm(s, lo);
      Gh[oi + d * oj] = s;
      Gl[oi + d * oj] = lo;
    });
    __syncthreads();
  }
  return k;
}

// Singular values and leading left singular vectors of C from the factor R
// (k x m, ld ldr, pivoted columns piv) with C C^T = Pi R^T R Pi^T: Jacobi
// on X = R^T, U_C = Pi * normalised columns of X (svd_left without the QR).
__device__ __noinline__ int svd_from_r(const double* R, int ldr, int k, int m, const int* piv,
                          const SvdWork& w, double budget2, int cap, double* U, int ldu,
                          double* margin_out, int* s_int) {
  for2d(m, k, [&](int i, int r) { w.Xs[i + w.ldx * r] = i >= r ? R[r + ldr * i] : 0.0; });
  __syncthreads();
  const int sweeps = jacobi(w.Xs, w.ldx, m, k, w.vn);
  if (w.prof && threadIdx.x == 0) {
    atomicAdd(&w.prof[12], (unsigned long long)sweeps);
    atomicAdd(&w.prof[13], 1ULL);
    if (sweeps >= 60) atomicAdd(&w.prof[14], 1ULL);
  }
  for (int q = threadIdx.x; q < k; q += NT) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += w.Xs[i + w.ldx * q] * w.Xs[i + w.ldx * q];
    w.sraw[q] = sqrt(s);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < k; q += NT) {
    const double v = w.sraw[q];
    int rank = 0;
    for (int o = 0; o < k; ++o) {
      const double u = w.sraw[o];
      rank += (u > v) || (u == v && o < q);
    }
    w.sig[rank] = v;
    w.perm[rank] = q;
  }
  __syncthreads();
  if (threadIdx.x == 0) *s_int = truncation_rank(w.sig, k, budget2, cap, margin_out);
  __syncthreads();
  const int t = *s_int;
  for2d(m, t, [&](int i, int r) {
    U[piv[i] + ldu * r] = w.Xs[i + w.ldx * w.perm[r]] / w.sig[r];
  });
  __syncthreads();
  return t;
}

// ---- single-warp small-matrix routines ------------------------------------
// The sequential factorizations of a rounding (pivoted Cholesky, one-sided
// Jacobi) on Gram dimensions d <= 32 run on warp 0 alone with warp-level
// synchronisation: each column step costs a few shuffles instead of three
// block barriers, and the other warps of the CTA wait at ONE barrier after
// the call (other CTAs keep the SM busy).  Same arithmetic as the block
// versions, same results.
constexpr unsigned kFull = 0xffffffffu;
#ifndef TTDVM_WARP_MAX_D
#define TTDVM_WARP_MAX_D 16
#endif
constexpr int kWarpMaxD = TTDVM_WARP_MAX_D;  // measured: the block versions win from ~24 up

// chol_piv_dd on warp 0 (d <= 32): lane v holds virtual column v's pivot;
// row k of R is formed by lane v (> k) and broadcast by shuffles for the
// trailing update.  Caller: if (threadIdx.x < 32) k = ...; then a barrier.
__device__ __noinline__ int chol_piv_dd_warp(double* Gh, double* Gl, int d, double thresh,
                                             double* R, int ldr, int* piv) {
  const int lane = threadIdx.x & 31;
  int mp = lane;  // original index of virtual column `lane`
  int k = 0;
  for (; k < d; ++k) {
    double bv = -1.0;
    int bi = k;
    if (lane >= k && lane < d) {
      bv = Gh[mp + d * mp];
      bi = lane;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (!(bv > thresh)) break;  // uniform
    const int pk_old = __shfl_sync(kFull, mp, k);
    const int pk = __shfl_sync(kFull, mp, bi);
    if (lane == k) mp = pk;
    else if (lane == bi) mp = pk_old;
    if (bi != k && lane < k) {  // earlier rows of R follow the column swap
      const double a = R[lane + ldr * k];
      R[lane + ldr * k] = R[lane + ldr * bi];
      R[lane + ldr * bi] = a;
    }
    const double ah = Gh[pk + d * pk], al = Gl[pk + d * pk];
    const double s = sqrt(ah);
    const double p0 = s * s, pe0 = fma(s, s, -p0);
    const double r0 = ((ah - p0) - pe0 + al) * (0.5 / s);
    double rh, rl;
    two_sum(s, r0, rh, rl);
    const double rinv = 1.0 / rh;
    double qh = 0.0, ql = 0.0;
    const bool act = lane > k && lane < d;
    if (act) {
      const double gh = Gh[pk + d * mp], gl = Gl[pk + d * mp];
      const double q1 = gh * rinv;
      double p, pe;
      dd_mul(q1, 0.0, rh, rl, p, pe);
      const double res = ((gh - p) - pe) + gl;
      two_sum(q1, res * rinv, qh, ql);
      R[k + ldr * lane] = qh + ql;
    }
    if (lane == k) R[k + ldr * k] = rh + rl;
    // trailing update G[p_i, p_j] -= R_ki R_kj (i, j > k): lane j, loop over i
    for (int i = k + 1; i < d; ++i) {
      const double hi = __shfl_sync(kFull, qh, i), lo = __shfl_sync(kFull, ql, i);
      const int pi = __shfl_sync(kFull, mp, i);
      if (act) {
        double p, pe;
        dd_mul(hi, lo, qh, ql, p, pe);
        const int e = pi + d * mp;
        double sh_, e_;
        two_sum(Gh[e], -p, sh_, e_);
        double l2 = Gl[e] + e_ - pe;
        dd_norm(sh_, l2);
        Gh[e] = sh_;
        Gl[e] = l2;
      }
    }
    __syncwarp();
  }
  if (lane < d) piv[lane] = mp;
  __syncwarp();
  return k;
}

// jacobi_t on warp 0 (c <= 32 columns): TPP lanes per pair.
template <int TPP>
__device__ int jacobi_warp_t(double* X, int ldx, int m, int c, double* nrm) {
  const int lane = threadIdx.x & 31;
  const int cp = c + (c & 1);
  const int npairs = cp / 2;
  const int pi = lane / TPP, sub = lane % TPP;
  const double tol2 = 1e-30;
  for (int sweep = 0; sweep < 60; ++sweep) {
    for (int j = lane; j < c; j += 32) {
      double s0 = 0.0, s1 = 0.0;
      int i = 0;
#pragma unroll 1
      for (; i + 1 < m; i += 2) {
        s0 += X[i + ldx * j] * X[i + ldx * j];
        s1 += X[i + 1 + ldx * j] * X[i + 1 + ldx * j];
      }
      if (i < m) s0 += X[i + ldx * j] * X[i + ldx * j];
      nrm[j] = s0 + s1;
    }
    __syncwarp();
    bool rotated = false, big = false;
    for (int r = 0; r < cp - 1; ++r) {
      for (int base = 0; base < npairs; base += 32 / TPP) {
        const int pp = base + pi;
        int a = pp + r - 1;
        if (a >= cp - 1) a -= cp - 1;
        a = pp == 0 ? 0 : a + 1;
        int b = cp - 2 - pp + r;
        if (b >= cp - 1) b -= cp - 1;
        b += 1;
        const bool live = pp < npairs && a < c && b < c;
        double ga = 0.0;
        double* x = X + ldx * (live ? a : 0);
        double* y = X + ldx * (live ? b : 0);
        if (live)
#pragma unroll 1
          for (int i = sub; i < m; i += TPP) ga += x[i] * y[i];
        ga = group_sum<TPP>(ga);
        if (live && ga != 0.0) {
          const double al = nrm[a], be = nrm[b];
          if (ga * ga > tol2 * al * be) {
            big = big || (ga * ga > TTDVM_JACOBI_BIG2 * al * be);
            const double dlt = be - al;
            const double mag = fmax(fabs(dlt), 2.0 * fabs(ga));
            const int ex = (int)((__double_as_longlong(mag) >> 52) & 0x7ff) - 1023;
            const double sc = __longlong_as_double((long long)(1023 - ex) << 52);
            const float df = (float)(dlt * sc), gf = (float)(ga * sc);
            const float tf = copysignf(1.0f, df) * (2.0f * gf) /
                             (fabsf(df) + sqrtf(df * df + 4.0f * gf * gf));
            const double t = (double)tf;
            rotated = rotated || (tf != 0.0f);
            const double cs = fast_rsqrt(1.0 + t * t), sn = cs * t;
#pragma unroll 1
            for (int i = sub; i < m; i += TPP) {
              const double xi = x[i], yi = y[i];
              x[i] = cs * xi - sn * yi;
              y[i] = sn * xi + cs * yi;
            }
            if (sub == 0) {
              const double c2 = cs * cs, tg = 2.0 * t * ga, t2 = t * t;
              nrm[a] = c2 * (al - tg + t2 * be);
              nrm[b] = c2 * (be + tg + t2 * al);
            }
          }
        }
      }
      __syncwarp();
    }
    if (!__any_sync(kFull, rotated) || !__any_sync(kFull, big)) return sweep + 1;
  }
  return 60;
}

__device__ __noinline__ int jacobi_warp(double* X, int ldx, int m, int c, double* nrm) {
  const int npairs = (c + 1) / 2;
  const int tpp = min(32, floor_pow2(max(1, 32 / max(npairs, 1))));
  switch (tpp) {
    case 32: return jacobi_warp_t<32>(X, ldx, m, c, nrm);
    case 16: return jacobi_warp_t<16>(X, ldx, m, c, nrm);
    case 8: return jacobi_warp_t<8>(X, ldx, m, c, nrm);
    case 4: return jacobi_warp_t<4>(X, ldx, m, c, nrm);
    case 2: return jacobi_warp_t<2>(X, ldx, m, c, nrm);
    default: return jacobi_warp_t<1>(X, ldx, m, c, nrm);
  }
}

// svd_from_r on warp 0 (k <= 32); t is returned to every lane of warp 0.
__device__ __noinline__ int svd_from_r_warp(const double* R, int ldr, int k, int m, const int* piv,
                                            const SvdWork& w, double budget2, int cap, double* U,
                                            int ldu, double* margin_out) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < m * k; e += 32) {
    const int r = e / m, i = e - r * m;
    w.Xs[i + w.ldx * r] = i >= r ? R[r + ldr * i] : 0.0;
  }
  __syncwarp();
  const int sweeps = jacobi_warp(w.Xs, w.ldx, m, k, w.vn);
  if (w.prof && lane == 0) {
    atomicAdd(&w.prof[12], (unsigned long long)sweeps);
    atomicAdd(&w.prof[13], 1ULL);
    if (sweeps >= 60) atomicAdd(&w.prof[14], 1ULL);
  }
  double v = 0.0;
  if (lane < k) {
    double s0 = 0.0, s1 = 0.0;
    int i = 0;
    for (; i + 1 < m; i += 2) {
      s0 += w.Xs[i + w.ldx * lane] * w.Xs[i + w.ldx * lane];
      s1 += w.Xs[i + 1 + w.ldx * lane] * w.Xs[i + 1 + w.ldx * lane];
    }
    if (i < m) s0 += w.Xs[i + w.ldx * lane] * w.Xs[i + w.ldx * lane];
    v = sqrt(s0 + s1);
  }
  // descending rank of lane's value (ties: lower index first)
  int rank = 0;
  for (int o = 0; o < k; ++o) {
    const double u = __shfl_sync(kFull, v, o);
    rank += (u > v) || (u == v && o < lane);
  }
  if (lane < k) {
    w.sig[rank] = v;
    w.perm[rank] = lane;
  }
  __syncwarp();
  int t = 0;
  if (lane == 0) t = truncation_rank(w.sig, k, budget2, cap, margin_out);
  t = __shfl_sync(kFull, t, 0);
  for (int e = lane; e < m * t; e += 32) {
    const int r = e / m, i = e - r * m;
    U[piv[i] + ldu * r] = w.Xs[i + w.ldx * w.perm[r]] / w.sig[r];
  }
  __syncwarp();
  return t;
}

}  // namespace
}  // namespace ttdvm
