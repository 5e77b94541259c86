// Moments, S-model equilibrium and packing kernels (SURVEY.md §8(a)
// T14-T17), FP64.
#include <math.h>

#include "ttdvm_device.cuh"

namespace ttdvm {

namespace {
constexpr int MT = 128;  // threads per cell

__device__ double msum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < MT / 32; ++w) s += red[w];
  return s;
}
}  // namespace

struct MacroArgs {
  TSet set;
  int count, n;
  const double* nodes;
  const double* weights;
  double gas[6];        // m, R, Pr, mu_ref, t_ref, omega
  double* macro;        // [count][11]
  double* nu;           // [count]
  int* status;
};

// compute_macro (proj/src/physics.cpp:17-67).  Each of the reference's 16
// convolutions (tt_tensor.cpp:195-204) is u^T first * (sum_j v_j M_j) *
// last w; the three per-axis weight families are contracted with the cores
// once per pass.  Pass 1 uses {w, xi w, xi^2 w} (n, n u, e2); pass 2 the
// c-shifted {w, c w, c^2 w, c^3 w} of each axis (S), exactly the weights the
// reference builds (physics.cpp:44-61).  One CTA per tensor; the middle core
// is streamed with coalesced loads (HBM-bound).
__global__ void __launch_bounds__(MT) macro_kernel(MacroArgs p) {
  const int c = blockIdx.x;
  if (c >= p.count) return;
  const int n = p.n;
  const int r1 = p.set.ranks[2 * c], r2 = p.set.ranks[2 * c + 1];
  const double* F = p.set.base + p.set.off[c];
  const double* M = F + (long long)n * r1;
  const double* L = M + (long long)n * r1 * r2;
  double sc = p.set.uscale;
  if (p.set.tscale) sc *= p.set.tscale[c];

  extern __shared__ double sm[];
  // weights wa[axis][4][n]
  double* wa = sm;                 // 3*4*n
  double* a1 = wa + 12 * n;        // 4 x r1
  double* a3 = a1 + 4 * r1;        // 4 x r2
  double* bm = a3 + 4 * r2;        // 4 x r1 x r2
  __shared__ double red[MT / 32];
  __shared__ double mac[16];

  const double R = p.gas[1];
  for (int pass = 0; pass < 2; ++pass) {
    // ---- weights ----
    for (int i = threadIdx.x; i < n; i += MT) {
      const double w = p.weights[i], x = p.nodes[i];
      for (int ax = 0; ax < 3; ++ax) {
        double* W = wa + ax * 4 * n;
        if (pass == 0) {
          const double xw = x * w;
          W[i] = w;
          W[n + i] = xw;
          W[2 * n + i] = x * xw;
          W[3 * n + i] = 0.0;
        } else {
          const double cc = (x - mac[1 + ax]) / mac[8];
          const double cw = cc * w, c2w = cc * cw;
          W[i] = w;
          W[n + i] = cw;
          W[2 * n + i] = c2w;
          W[3 * n + i] = cc * c2w;
        }
      }
    }
    __syncthreads();
    const int nw = pass == 0 ? 3 : 4;
    // a1[p][a] = sum_i W0[p][i] F(i,a) (scale folded here, as scaled() does)
    for (int e = threadIdx.x; e < nw * r1; e += MT) {
      const int q = e / r1, a = e % r1;
      const double* W = wa + q * n;
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += W[i] * (sc * F[i + n * a]);
      a1[q * r1 + a] = s;
    }
    for (int e = threadIdx.x; e < nw * r2; e += MT) {
      const int q = e / r2, b = e % r2;
      const double* W = wa + 2 * 4 * n + q * n;
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += L[b + r2 * k] * W[k];
      a3[q * r2 + b] = s;
    }
    for (int e = threadIdx.x; e < r1 * r2; e += MT) {
      const double* W = wa + 4 * n;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      for (int j = 0; j < n; ++j) {
        const double m = M[(long long)j * r1 * r2 + e];
        s0 += W[j] * m;
        s1 += W[n + j] * m;
        s2 += W[2 * n + j] * m;
        s3 += W[3 * n + j] * m;
      }
      bm[e] = s0;
      bm[r1 * r2 + e] = s1;
      bm[2 * r1 * r2 + e] = s2;
      bm[3 * r1 * r2 + e] = s3;
    }
    __syncthreads();
    // bilinear forms conv(p,q,r) = a1[p] . bm[q] . a3[r]
    // pass 0: (000) (100) (010) (001) (200) (020) (002)
    // pass 1: S0: (300) (120) (102); S1: (210) (030) (012); S2: (201) (021) (003)
    const int nf = pass == 0 ? 7 : 9;
    const int P0[7][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {2, 0, 0}, {0, 2, 0}, {0, 0, 2}};
    const int P1[9][3] = {{3, 0, 0}, {1, 2, 0}, {1, 0, 2}, {2, 1, 0}, {0, 3, 0},
                          {0, 1, 2}, {2, 0, 1}, {0, 2, 1}, {0, 0, 3}};
    double part[9];
#pragma unroll
    for (int f = 0; f < 9; ++f) part[f] = 0.0;
    for (int e = threadIdx.x; e < r1 * r2; e += MT) {
      const int a = e % r1, b = e / r1;
#pragma unroll
      for (int f = 0; f < 9; ++f) {
        if (f < nf) {
          const int* q = pass == 0 ? P0[f] : P1[f];
          part[f] += a1[q[0] * r1 + a] * bm[q[1] * r1 * r2 + e] * a3[q[2] * r2 + b];
        }
      }
    }
    double tot[9];
#pragma unroll
    for (int f = 0; f < 9; ++f) tot[f] = f < nf ? msum(part[f], red) : 0.0;
    if (threadIdx.x == 0) {
      if (pass == 0) {
        const double nd = tot[0];
        mac[0] = nd;
        int err = 0;
        if (!(nd > 0.0)) err = kErrDensity;
        const double u0 = tot[1] / nd, u1 = tot[2] / nd, u2 = tot[3] / nd;
        const double e2 = tot[4] + tot[5] + tot[6];
        const double T = (e2 - nd * (u0 * u0 + u1 * u1 + u2 * u2)) / (3.0 * nd * R);
        if (!err && !(T > 0.0)) err = kErrTemperature;
        mac[1] = u0;
        mac[2] = u1;
        mac[3] = u2;
        mac[4] = T;
        mac[8] = err ? 1.0 : sqrt(2.0 * R * T);
        mac[9] = err;
        if (err && atomicCAS(&p.status[kStError], 0, err) == 0) p.status[kStErrIdx] = c;
      } else {
        const double nd = mac[0];
        mac[5] = (tot[0] + tot[1] + tot[2]) / nd;
        mac[6] = (tot[3] + tot[4] + tot[5]) / nd;
        mac[7] = (tot[6] + tot[7] + tot[8]) / nd;
      }
    }
    __syncthreads();
    if (mac[9] != 0.0) return;  // blow-up reported; no S for this cell
  }
  if (threadIdx.x == 0) {
    const double m = p.gas[0], T = mac[4];
    const double rho = m * mac[0];
    const double pr = rho * R * T;
    const double mu = p.gas[3] * pow(T / p.gas[4], p.gas[5]);
    double* out = p.macro + 11LL * c;
    out[0] = mac[0];
    out[1] = mac[1];
    out[2] = mac[2];
    out[3] = mac[3];
    out[4] = T;
    out[5] = rho;
    out[6] = pr;
    out[7] = mac[5];
    out[8] = mac[6];
    out[9] = mac[7];
    out[10] = pr / mu;
    if (p.nu) p.nu[c] = pr / mu;
  }
}

size_t macro_smem_bytes(int n, int rmax) {
  return 8 * (size_t)(12 * n + 4 * rmax + 4 * rmax + 4 * rmax * rmax);
}

cudaError_t launch_macro(const MacroArgs& a, int rmax, cudaStream_t st) {
  if (a.count == 0) return cudaSuccess;
  const size_t smem = macro_smem_bytes(a.n, rmax);
  cudaError_t e =
      cudaFuncSetAttribute(macro_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  macro_kernel<<<a.count, MT, smem, st>>>(a);
  return cudaGetLastError();
}

// Raw S-model equilibrium f_S = f_M o (1 + 0.8(1-Pr)(S.c)(c^2 - 2.5))
// (shakhov_tt, proj/src/physics.cpp:89-108) written as its exact rank-
// (1,4,4,1) TT: g = sum_{p,s} x^p H_ps(y) z^s with x, y, z the three c
// components.  The reference assembles the same tensor at rank 13; the
// subsequent rounding (physics.cpp:109) sees the same tensor, hence the
// same truncation.  Layout: fixed stride 4n + 16n + 4n per cell.
__global__ void shakhov_raw_kernel(const double* macro, int count, int n, const double* nodes,
                                   double R, double prandtl, double* out) {
  const int c = blockIdx.x;
  if (c >= count) return;
  const double* m = macro + 11LL * c;
  const double nd = m[0], T = m[4];
  const double two_rt = 2.0 * R * T;
  const double norm1d = 1.0 / sqrt(M_PI * two_rt);
  const double s = sqrt(2.0 * R * T);
  const double kap = 0.8 * (1.0 - prandtl);
  const double a = kap * m[7], b = kap * m[8], d = kap * m[9];
  double* F = out + (long long)c * 24 * n;
  double* M = F + 4 * n;
  double* L = M + 16 * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double xi = nodes[i];
    double fm[3], cc[3];
    for (int ax = 0; ax < 3; ++ax) {
      const double v = xi - m[1 + ax];
      fm[ax] = norm1d * exp(-v * v / two_rt);
      cc[ax] = (xi - m[1 + ax]) / s;
    }
    fm[0] *= nd;
    // first (n x 4): fM0 * x^p
    const double x = cc[0];
    F[i] = fm[0];
    F[i + n] = fm[0] * x;
    F[i + 2 * n] = fm[0] * x * x;
    F[i + 3 * n] = fm[0] * x * x * x;
    // middle slice j = i (4 x 4 col-major): H(p, s)
    const double y = cc[1], y2 = y * y - 2.5;
    double* Mj = M + 16 * i;
    const double H[4][4] = {{1.0 + b * y * y2, d * y2, b * y, d},
                            {a * y2, 0.0, a, 0.0},
                            {b * y, d, 0.0, 0.0},
                            {a, 0.0, 0.0, 0.0}};
    for (int pp = 0; pp < 4; ++pp)
      for (int ss = 0; ss < 4; ++ss) Mj[pp + 4 * ss] = fm[1] * H[pp][ss];
    // last (4 x n): fM2 * z^s
    const double z = cc[2];
    L[0 + 4 * i] = fm[2];
    L[1 + 4 * i] = fm[2] * z;
    L[2 + 4 * i] = fm[2] * z * z;
    L[3 + 4 * i] = fm[2] * z * z * z;
  }
}

cudaError_t launch_shakhov_raw(const double* macro, int count, int n, const double* nodes,
                               double R, double prandtl, double* out, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  shakhov_raw_kernel<<<count, 64, 0, st>>>(macro, count, n, nodes, R, prandtl, out);
  return cudaGetLastError();
}

// Gather tensors of a set into cell order (download / halo packing).
__global__ void gather_kernel(TSet s, int count, const long long* dst_off, int n1, int n2, int n3,
                              double* dst) {
  const int t = blockIdx.x;
  if (t >= count) return;
  const int r1 = s.ranks[2 * t], r2 = s.ranks[2 * t + 1];
  const long long sz = (long long)n1 * r1 + (long long)n2 * r1 * r2 + (long long)r2 * n3;
  const double* src = s.base + s.off[t];
  double* d = dst + dst_off[t];
  for (long long e = threadIdx.x; e < sz; e += blockDim.x) d[e] = src[e];
}

// Copy tensors src_ids[i] of a set to dst_base + new_off[i] and register
// them as entries dst_ids[i] of the destination set (halo unpack / ghost
// carry-over).
__global__ void place_kernel(TSet s, const int* src_ids, int count, int n1, int n2, int n3,
                             int* dst_ranks, long long* dst_off, const int* dst_ids,
                             const long long* new_off, double* dst_base) {
  const int i = blockIdx.x;
  if (i >= count) return;
  const int t = src_ids ? src_ids[i] : i;
  const int r1 = s.ranks[2 * t], r2 = s.ranks[2 * t + 1];
  const long long sz = (long long)n1 * r1 + (long long)n2 * r1 * r2 + (long long)r2 * n3;
  const double* src = s.base + s.off[t];
  double* d = dst_base + new_off[i];
  for (long long e = threadIdx.x; e < sz; e += blockDim.x) d[e] = src[e];
  if (threadIdx.x == 0) {
    const int di = dst_ids[i];
    dst_ranks[2 * di] = r1;
    dst_ranks[2 * di + 1] = r2;
    dst_off[di] = new_off[i];
  }
}

cudaError_t launch_place(const TSet& s, const int* src_ids, int count, int n1, int n2, int n3,
                         int* dst_ranks, long long* dst_off, const int* dst_ids,
                         const long long* new_off, double* dst_base, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  place_kernel<<<count, 128, 0, st>>>(s, src_ids, count, n1, n2, n3, dst_ranks, dst_off, dst_ids,
                                      new_off, dst_base);
  return cudaGetLastError();
}

// Gather tensors src_ids[i] (or i) of a set into dst + dst_off[i].
__global__ void gather_ids_kernel(TSet s, const int* src_ids, int count, const long long* dst_off,
                                  int n1, int n2, int n3, double* dst) {
  const int i = blockIdx.x;
  if (i >= count) return;
  const int t = src_ids[i];
  const int r1 = s.ranks[2 * t], r2 = s.ranks[2 * t + 1];
  const long long sz = (long long)n1 * r1 + (long long)n2 * r1 * r2 + (long long)r2 * n3;
  const double* src = s.base + s.off[t];
  double* d = dst + dst_off[i];
  for (long long e = threadIdx.x; e < sz; e += blockDim.x) d[e] = src[e];
}

cudaError_t launch_gather_ids(const TSet& s, const int* src_ids, int count,
                              const long long* dst_off, int n1, int n2, int n3, double* dst,
                              cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  gather_ids_kernel<<<count, 128, 0, st>>>(s, src_ids, count, dst_off, n1, n2, n3, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather(const TSet& s, int count, const long long* dst_off, int n1, int n2,
                          int n3, double* dst, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  gather_kernel<<<count, 128, 0, st>>>(s, count, dst_off, n1, n2, n3, dst);
  return cudaGetLastError();
}

}  // namespace ttdvm

namespace ttdvm {
// FP64 FMA throughput probe: independent DFMA chains per thread, one wave
// of resident CTAs per SM; returns FLOP count (2 per FMA).
__global__ void dfma_probe_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0;
  double x4 = x0 + 4.0, x5 = x0 + 5.0, x6 = x0 + 6.0, x7 = x0 + 7.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains live
}

cudaError_t launch_dfma_probe(double* out, int blocks, int threads, int iters, cudaStream_t st) {
  dfma_probe_kernel<<<blocks, threads, 0, st>>>(out, iters, 0.999999, 1e-7);
  return cudaGetLastError();
}
}  // namespace ttdvm
