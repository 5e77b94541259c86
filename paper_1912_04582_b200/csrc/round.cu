// Batched FP64 TT rounding of implicit sums.
//
// One CTA (256 threads) owns one output tensor.  Its input is a list of
// summands (Term) -- scaled, optionally face-factor-weighted and reflected
// TT tensors read straight from their arenas -- so the rank-inflated sum of
// a face flux, cell residual or update is never materialised
// (proj/src/tt_tensor.cpp:290-312 builds it with explicit block-diagonal
// zeros; here the block structure is used directly).
//
// Algorithm (same truncation decisions as TtTensor::rounded,
// proj/src/tt_tensor.cpp:139-193):
//   1. Householder QR of last^T (n3 x R2) -> R3, Q3 (reflectors kept).
//   2. Cut 1: the singular values of the mode-1 unfolding A_(1) equal those
//      of C = F R2^T (R1 <= n1, "W route": R2 from the QR of the stacked
//      (M_j R3^T)^T) or C = R_T^T (R1 > n1, "T route": R_T from the QR of
//      the stacked (F M_j R3^T)^T).  Both tall QRs run as a TSQR over
//      slices j with a structured Householder update of the running R
//      (only R is needed, never the tall Q).
//   3. One-sided Jacobi SVD of C -> sigma_1, U1; budget eps^2 ||A||^2 / 2
//      (reference :167-169); truncation_rank (reference :18-29).
//   4. Cut 2: S_j = (U1^T F) M_j R3^T, TSQR of the stacked S_j -> R_S,
//      Jacobi SVD with V -> sigma_2, V2; truncation_rank.
//   5. Output first = U1, middle_j = S_j V2, last = (Q3 V2)^T.
// All arithmetic FP64.  Reconstructions equal the reference's up to
// roundoff; cores differ by the usual orthogonal gauge (the reference puts
// Sigma_2 into last, here it sits in middle).
#include <math.h>

#include "ttdvm_device.cuh"

namespace ttdvm {

namespace {

constexpr int NT = kRoundThreads;
constexpr int NW = NT / 32;

struct TermInfo {
  const double* base;
  const double* u[3];
  double scale;
  int r1, r2, off1, off2, refl;
};

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

// LAPACK dlarfg on (alpha, ||x||^2): H = I - tau v v^T, v = [1; x*scale].
__device__ __forceinline__ void larfg(double alpha, double sigma2, double& beta, double& tau,
                                      double& scale) {
  if (sigma2 == 0.0) {
    beta = alpha;
    tau = 0.0;
    scale = 0.0;
    return;
  }
  const double nrm = sqrt(alpha * alpha + sigma2);
  beta = alpha >= 0.0 ? -nrm : nrm;
  tau = (beta - alpha) / beta;
  scale = 1.0 / (alpha - beta);
}

__device__ __forceinline__ int floor_pow2(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

// Householder QR of A (m x ncols, col-major, lda) in place: R in the upper
// triangle, reflector tails below the diagonal, tau[k].
__device__ void qr_inplace(double* A, int lda, int m, int ncols, double* tau, double* sh) {
  const int kmax = min(m, ncols);
  for (int k = 0; k < kmax; ++k) {
    // sigma2 = ||A[k+1:m, k]||^2 by warp 0
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int i = k + 1 + threadIdx.x; i < m; i += 32) s += A[i + lda * k] * A[i + lda * k];
      s = warp_sum(s);
      if (threadIdx.x == 0) {
        double beta, t, sc;
        larfg(A[k + lda * k], s, beta, t, sc);
        sh[0] = t;
        sh[1] = sc;
        sh[2] = beta;
      }
    }
    __syncthreads();
    const double t = sh[0], sc = sh[1];
    if (t != 0.0) {
      for (int i = k + 1 + threadIdx.x; i < m; i += NT) A[i + lda * k] *= sc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tau[k] = t;
      if (t != 0.0) A[k + lda * k] = sh[2];
    }
    if (t != 0.0) {
      for (int l = k + 1 + threadIdx.x; l < ncols; l += NT) {
        double* col = A + lda * l;
        double w = col[k];
        const double* v = A + lda * k;
        for (int i = k + 1; i < m; ++i) w += v[i] * col[i];
        w *= t;
        col[k] -= w;
        for (int i = k + 1; i < m; ++i) col[i] -= w * v[i];
      }
    }
    __syncthreads();
  }
}

// QR of [R; B] -> R, R upper c x c (ld ldr), B h x c (ld ldb); B destroyed.
// Threads: groups of tpc lanes per column, rows strided inside the group.
template <int TPC>
__device__ void qr_update_t(double* R, int ldr, double* B, int ldb, int h, int c, double* sh) {
  const int g = threadIdx.x / TPC, sub = threadIdx.x % TPC;
  const int ngroups = NT / TPC;
  // sigma2 of column 0 (all of warp 0 reaches the shuffles)
  if (threadIdx.x < 32) {
    double s = 0.0;
    if (g == 0)
      for (int i = sub; i < h; i += TPC) s += B[i] * B[i];
    s = group_sum<TPC>(s);
    if (g == 0 && sub == 0) sh[0] = s;
  }
  __syncthreads();
  for (int k = 0; k < c; ++k) {
    double beta, t, sc;
    larfg(R[k + ldr * k], sh[k & 1], beta, t, sc);
    if (t != 0.0) {
      // the group owning column k scales v (groups are assigned l - k - 1)
      for (int i = threadIdx.x; i < h; i += NT) B[i + ldb * k] *= sc;
    }
    __syncthreads();
    if (threadIdx.x == 0 && t != 0.0) R[k + ldr * k] = beta;
    const double* v = B + ldb * k;
    // uniform trip count across the block: every lane reaches the shuffles
    for (int base = k + 1; base < c; base += ngroups) {
      const int l = base + g;
      const bool act = l < c;
      double* col = B + ldb * (act ? l : k);
      double w = 0.0;
      if (t != 0.0) {
        if (act)
          for (int i = sub; i < h; i += TPC) w += v[i] * col[i];
        w = group_sum<TPC>(w);
        if (act) w = t * (w + R[k + ldr * l]);
      }
      double s = 0.0;
      if (act) {
        for (int i = sub; i < h; i += TPC) {
          const double x = col[i] - w * v[i];
          col[i] = x;
          s += x * x;
        }
        if (sub == 0) R[k + ldr * l] -= w;
      }
      s = group_sum<TPC>(s);
      if (act && l == k + 1 && sub == 0) sh[(k + 1) & 1] = s;
    }
    __syncthreads();
  }
}

__device__ void qr_update(double* R, int ldr, double* B, int ldb, int h, int c, double* sh) {
  const int tpc = min(32, floor_pow2(max(1, NT / max(c, 1))));
  switch (tpc) {
    case 32: qr_update_t<32>(R, ldr, B, ldb, h, c, sh); break;
    case 16: qr_update_t<16>(R, ldr, B, ldb, h, c, sh); break;
    case 8: qr_update_t<8>(R, ldr, B, ldb, h, c, sh); break;
    case 4: qr_update_t<4>(R, ldr, B, ldb, h, c, sh); break;
    case 2: qr_update_t<2>(R, ldr, B, ldb, h, c, sh); break;
    default: qr_update_t<1>(R, ldr, B, ldb, h, c, sh); break;
  }
}

// One-sided (Hestenes) Jacobi SVD of A (m x c, ld lda) in place: on exit
// the columns of A are U*Sigma (unsorted) and V (c x c, ld ldv, optional,
// must hold the identity on entry) accumulates the rotations.
template <int TPP>
__device__ void jacobi_t(double* A, int lda, int m, int c, double* V, int ldv, int* flag) {
  const int cp = c + (c & 1);
  const int npairs = cp / 2;
  const int pi = threadIdx.x / TPP, sub = threadIdx.x % TPP;
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int r = 0; r < cp - 1; ++r) {
      for (int base = 0; base < npairs; base += NT / TPP) {
        const int pp = base + pi;
        const int a = pp == 0 ? 0 : ((pp + r - 1) % (cp - 1)) + 1;
        const int b = ((cp - 1 - pp + r - 1) % (cp - 1)) + 1;
        const bool live = pp < npairs && a < c && b < c;
        double al = 0.0, be = 0.0, ga = 0.0;
        double* x = A + lda * (live ? a : 0);
        double* y = A + lda * (live ? b : 0);
        if (live) {
          for (int i = sub; i < m; i += TPP) {
            const double xi = x[i], yi = y[i];
            al += xi * xi;
            be += yi * yi;
            ga += xi * yi;
          }
        }
        al = group_sum<TPP>(al);
        be = group_sum<TPP>(be);
        ga = group_sum<TPP>(ga);
        if (live && ga != 0.0 && fabs(ga) > tol * sqrt(al) * sqrt(be)) {
          rotated = true;
          const double zeta = (be - al) / (2.0 * ga);
          double t;
          if (fabs(zeta) > 1e150) {
            t = 0.5 / zeta;
          } else {
            t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          }
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          for (int i = sub; i < m; i += TPP) {
            const double xi = x[i], yi = y[i];
            x[i] = cs * xi - sn * yi;
            y[i] = sn * xi + cs * yi;
          }
          if (V) {
            double* vx = V + ldv * a;
            double* vy = V + ldv * b;
            for (int i = sub; i < c; i += TPP) {
              const double xi = vx[i], yi = vy[i];
              vx[i] = cs * xi - sn * yi;
              vy[i] = sn * xi + cs * yi;
            }
          }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated ? 1 : 0)) break;
  }
  (void)flag;
}

__device__ void jacobi(double* A, int lda, int m, int c, double* V, int ldv) {
  const int npairs = (c + 1) / 2;
  const int tpp = min(32, floor_pow2(max(1, NT / max(npairs, 1))));
  switch (tpp) {
    case 32: jacobi_t<32>(A, lda, m, c, V, ldv, nullptr); break;
    case 16: jacobi_t<16>(A, lda, m, c, V, ldv, nullptr); break;
    case 8: jacobi_t<8>(A, lda, m, c, V, ldv, nullptr); break;
    case 4: jacobi_t<4>(A, lda, m, c, V, ldv, nullptr); break;
    case 2: jacobi_t<2>(A, lda, m, c, V, ldv, nullptr); break;
    default: jacobi_t<1>(A, lda, m, c, V, ldv, nullptr); break;
  }
}

// Column norms of A (m x c) -> sig sorted descending with perm.
__device__ void sorted_norms(const double* A, int lda, int m, int c, double* sig_raw, double* sig,
                             int* perm) {
  for (int p = threadIdx.x; p < c; p += NT) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += A[i + lda * p] * A[i + lda * p];
    sig_raw[p] = sqrt(s);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < c; p += NT) {
    const double v = sig_raw[p];
    int rank = 0;
    for (int q = 0; q < c; ++q) {
      const double w = sig_raw[q];
      rank += (w > v) || (w == v && q < p);
    }
    sig[rank] = v;
    perm[rank] = p;
  }
  __syncthreads();
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

// SURVEY.md Appendix A canonical FLOPs of TtTensor::rounded(n; R1,R2 -> t1,t2)
// (the reference algorithm, not the cheaper one run here).
__device__ double qr_f(double m, double k) {
  const double p = fmin(m, k);
  return 2.0 * m * k * p - 2.0 / 3.0 * p * p * p;
}
__device__ double q_f(double m, double k) {
  const double p = fmin(m, k);
  return 2.0 * m * p * p - 2.0 / 3.0 * p * p * p;
}
__device__ double svd_f(double m, double k) {
  const double M = fmax(m, k), P = fmin(m, k);
  return 6.0 * M * P * P + 20.0 * P * P * P;
}
__device__ double round_flops(double n, double R1, double R2, double t1, double t2) {
  const double q3 = fmin(n, R2), q2 = fmin(n * q3, R1);
  return qr_f(n, R2) + q_f(n, R2) + n * 2.0 * R1 * R2 * q3 + qr_f(n * q3, R1) +
         q_f(n * q3, R1) + 2.0 * n * R1 * q2 + 2.0 * n * q2 + svd_f(n, q2) + t1 * q2 +
         n * 2.0 * t1 * q2 * q3 + svd_f(n * t1, q3) + 2.0 * t2 * q3 * n;
}

__device__ __forceinline__ double mid_val(const TermInfo& t, int n1, int n2, int j, int a,
                                          int b) {
  const int jj = t.refl == 2 ? n2 - 1 - j : j;
  double v = t.base[(long long)n1 * t.r1 + (long long)jj * t.r1 * t.r2 + a + t.r1 * b];
  if (t.u[1]) v *= t.u[1][j];
  return v;
}

}  // namespace

__global__ void __launch_bounds__(NT) round_sums_kernel(RoundArgs p) {
  extern __shared__ double sm[];
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3;
  const int mx = max(n1, n3);
  const int RM1 = p.RM1, RM2 = p.RM2, HMAX = p.HMAX;
  // ---- shared-memory carve-up (doubles) ----
  double* F = sm;                          // n1 x RM1
  double* lastT = F + n1 * RM1;            // n3 x RM2
  double* tau = lastT + n3 * RM2;          // mx
  double* Rr = tau + mx;                   // mx x mx
  double* B = Rr + mx * mx;                // HMAX x mx
  double* X = B + HMAX * mx;               // n1 x RM2
  double* P = X + n1 * RM2;                // n1 x RM1
  double* U1 = P + n1 * RM1;               // n1 x n1
  double* V2 = U1 + n1 * n1;               // n3 x n3
  double* sig = V2 + n3 * n3;              // mx
  double* sraw = sig + mx;                 // mx
  double* sh = sraw + mx;                  // 32 scalars
  int* perm = reinterpret_cast<int*>(sh + 32);          // mx
  int* colterm = perm + mx;                              // RM2 (col -> term)
  int* rowterm = colterm + RM2;                          // RM1 (col of F -> term)
  TermInfo* terms = reinterpret_cast<TermInfo*>(
      reinterpret_cast<double*>(rowterm + RM1 + (((RM1 + RM2 + mx) & 1) ? 1 : 0)));
  __shared__ int s_meta[8];

  const int o = blockIdx.x;
  if (o >= p.nout) return;
  const long long t0 = p.term_off ? p.term_off[o] : o;
  const int K = p.term_off ? (int)(p.term_off[o + 1] - t0) : 1;

  if (threadIdx.x == 0) {
    int off1 = 0, off2 = 0;
    for (int k = 0; k < K; ++k) {
      const Term tm = p.terms[t0 + k];
      const TSet& s = p.sets[tm.set];
      TermInfo ti;
      ti.r1 = s.ranks[2 * tm.idx];
      ti.r2 = s.ranks[2 * tm.idx + 1];
      ti.base = s.base + s.off[tm.idx];
      double sc = tm.scale * s.uscale;
      if (s.tscale) sc *= s.tscale[tm.idx];
      ti.scale = sc;
      ti.refl = tm.refl;
      const double* fac = tm.fac >= 0 ? p.factors + (long long)tm.fac * (n1 + n2 + n3) : nullptr;
      ti.u[0] = fac ? fac : nullptr;
      ti.u[1] = fac ? fac + n1 : nullptr;
      ti.u[2] = fac ? fac + n1 + n2 : nullptr;
      ti.off1 = off1;
      ti.off2 = off2;
      off1 += ti.r1;
      off2 += ti.r2;
      terms[k] = ti;
    }
    s_meta[0] = off1;
    s_meta[1] = off2;
  }
  __syncthreads();
  const int R1 = s_meta[0], R2 = s_meta[1];
  // column -> term maps
  for (int k = 0; k < K; ++k) {
    const TermInfo& t = terms[k];
    for (int a = threadIdx.x; a < t.r1; a += NT) rowterm[t.off1 + a] = k;
    for (int b = threadIdx.x; b < t.r2; b += NT) colterm[t.off2 + b] = k;
  }
  // ---- materialise F (n1 x R1) and last^T (n3 x R2) ----
  for (int k = 0; k < K; ++k) {
    const TermInfo& t = terms[k];
    for (int e = threadIdx.x; e < n1 * t.r1; e += NT) {
      const int i = e % n1, a = e / n1;
      const int ii = t.refl == 1 ? n1 - 1 - i : i;
      double v = t.scale * t.base[ii + n1 * a];
      if (t.u[0]) v *= t.u[0][i];
      F[i + n1 * (t.off1 + a)] = v;
    }
    const double* L = t.base + (long long)n1 * t.r1 + (long long)n2 * t.r1 * t.r2;
    for (int e = threadIdx.x; e < n3 * t.r2; e += NT) {
      const int b = e % t.r2, kk = e / t.r2;  // coalesced read of last (b fastest)
      const int kr = t.refl == 3 ? n3 - 1 - kk : kk;
      double v = L[b + t.r2 * kr];
      if (t.u[2]) v *= t.u[2][kk];
      lastT[kk + n3 * (t.off2 + b)] = v;
    }
  }
  __syncthreads();

  // ---- 1. QR of last^T ----
  qr_inplace(lastT, n3, n3, R2, tau, sh);
  const int q3 = min(n3, R2);
  // R3(c, b) = lastT[c + n3*b] for c <= b
  auto r3 = [&](int c, int b) -> double { return c <= b ? lastT[c + n3 * b] : 0.0; };

  // ---- 2. cut 1 TSQR ----
  const bool troute = R1 > n1;
  const int c1 = troute ? n1 : R1;
  for (int e = threadIdx.x; e < mx * mx; e += NT) Rr[e] = 0.0;
  const int ns1 = max(1, HMAX / q3);
  for (int j0 = 0; j0 < n2; j0 += ns1) {
    const int jn = min(n2, j0 + ns1);
    __syncthreads();
    for (int j = j0; j < jn; ++j) {
      const int row0 = (j - j0) * q3;
      if (troute) {
        // X = F blockdiag(M_j)  (n1 x R2)
        for (int e = threadIdx.x; e < n1 * R2; e += NT) {
          const int i = e % n1, col = e / n1;
          const TermInfo& t = terms[colterm[col]];
          const int b = col - t.off2;
          double s = 0.0;
          for (int a = 0; a < t.r1; ++a) s += F[i + n1 * (t.off1 + a)] * mid_val(t, n1, n2, j, a, b);
          X[i + n1 * col] = s;
        }
        __syncthreads();
        // B(row0 + c, i) = sum_b X(i, b) R3(c, b)
        for (int e = threadIdx.x; e < q3 * n1; e += NT) {
          const int c = e % q3, i = e / q3;
          double s = 0.0;
          for (int b = c; b < R2; ++b) s += X[i + n1 * b] * lastT[c + n3 * b];
          B[row0 + c + HMAX * i] = s;
        }
        __syncthreads();
      } else {
        // B(row0 + c, off1 + a) = sum_b R3(c, off2 + b) M_tj(a, b)
        for (int e = threadIdx.x; e < q3 * R1; e += NT) {
          const int c = e % q3, col = e / q3;
          const TermInfo& t = terms[rowterm[col]];
          const int a = col - t.off1;
          double s = 0.0;
          for (int b = 0; b < t.r2; ++b) s += r3(c, t.off2 + b) * mid_val(t, n1, n2, j, a, b);
          B[row0 + c + HMAX * col] = s;
        }
      }
    }
    __syncthreads();
    qr_update(Rr, mx, B, HMAX, (jn - j0) * q3, c1, sh);
  }
  __syncthreads();

  // ---- 3. C (n1 x c1) into B, norm, Jacobi SVD ----
  double loc = 0.0;
  for (int e = threadIdx.x; e < n1 * c1; e += NT) {
    const int i = e % n1, pp = e / n1;
    double v;
    if (troute) {
      v = pp <= i ? Rr[pp + mx * i] : 0.0;
    } else {
      v = 0.0;
      for (int a = pp; a < R1; ++a) v += F[i + n1 * a] * Rr[pp + mx * a];
    }
    B[i + HMAX * pp] = v;
    loc += v * v;
  }
  const double norm2 = block_sum(loc, sh + 8);
  if (norm2 == 0.0 || !isfinite(norm2)) {
    // canonical zero, TtTensor::constant(n1, n2, n3, 0) (reference :168)
    if (threadIdx.x == 0) {
      const long long sz = n1 + n2 + n3;
      const unsigned long long at = atomicAdd(p.out.used, (unsigned long long)sz);
      const bool ok = (long long)(at + sz) <= p.out.capacity;
      if (!ok) atomicExch(&p.status[kStOverflow], 1);
      if (!isfinite(norm2)) {
        if (atomicCAS(&p.status[kStError], 0, kErrNonFinite) == 0) p.status[kStErrIdx] = o;
      }
      p.out.ranks[2 * o] = 1;
      p.out.ranks[2 * o + 1] = 1;
      p.out.off[o] = ok ? (long long)at : -1;
      s_meta[2] = ok ? 1 : 0;
      s_meta[3] = (int)0;
      reinterpret_cast<long long*>(sh)[20] = (long long)at;
      if (p.margins) {
        p.margins[2 * o] = INFINITY;
        p.margins[2 * o + 1] = INFINITY;
      }
    }
    __syncthreads();
    if (s_meta[2]) {
      double* dst = p.out.base + reinterpret_cast<long long*>(sh)[20];
      for (int e = threadIdx.x; e < n1 + n2 + n3; e += NT) dst[e] = e < n1 ? 0.0 : 1.0;
    }
    return;
  }
  const double budget2 = p.eps * p.eps * norm2 / 2.0;
  jacobi(B, HMAX, n1, c1, nullptr, 0);
  sorted_norms(B, HMAX, n1, c1, sraw, sig, perm);
  if (threadIdx.x == 0) {
    double mg;
    s_meta[4] = truncation_rank(sig, c1, budget2, p.cap, &mg);
    if (p.margins) p.margins[2 * o] = mg;
  }
  __syncthreads();
  const int t1 = s_meta[4];
  // U1(:, r) = C V(:, perm[r]) / sigma_r
  for (int e = threadIdx.x; e < n1 * t1; e += NT) {
    const int i = e % n1, r = e / n1;
    U1[i + n1 * r] = B[i + HMAX * perm[r]] / sig[r];
  }
  __syncthreads();
  // P = U1^T F (t1 x R1)
  for (int e = threadIdx.x; e < t1 * R1; e += NT) {
    const int r = e % t1, col = e / t1;
    double s = 0.0;
    for (int i = 0; i < n1; ++i) s += U1[i + n1 * r] * F[i + n1 * col];
    P[r + n1 * col] = s;
  }

  // ---- 4. cut 2 TSQR over S_j = P blockdiag(M_j) R3^T (t1 x q3) ----
  for (int e = threadIdx.x; e < mx * mx; e += NT) Rr[e] = 0.0;
  const int ns2 = max(1, HMAX / t1);
  for (int j0 = 0; j0 < n2; j0 += ns2) {
    const int jn = min(n2, j0 + ns2);
    __syncthreads();
    for (int j = j0; j < jn; ++j) {
      const int row0 = (j - j0) * t1;
      for (int e = threadIdx.x; e < t1 * R2; e += NT) {
        const int r = e % t1, col = e / t1;
        const TermInfo& t = terms[colterm[col]];
        const int b = col - t.off2;
        double s = 0.0;
        for (int a = 0; a < t.r1; ++a) s += P[r + n1 * (t.off1 + a)] * mid_val(t, n1, n2, j, a, b);
        X[r + n1 * col] = s;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < t1 * q3; e += NT) {
        const int r = e % t1, c = e / t1;
        double s = 0.0;
        for (int b = c; b < R2; ++b) s += X[r + n1 * b] * lastT[c + n3 * b];
        B[row0 + r + HMAX * c] = s;
      }
      __syncthreads();
    }
    qr_update(Rr, mx, B, HMAX, (jn - j0) * t1, q3, sh);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < q3 * q3; e += NT) {
    const int i = e % q3, c = e / q3;
    V2[i + n3 * c] = i == c ? 1.0 : 0.0;
  }
  __syncthreads();
  jacobi(Rr, mx, q3, q3, V2, n3);
  sorted_norms(Rr, mx, q3, q3, sraw, sig, perm);
  if (threadIdx.x == 0) {
    double mg;
    const int t2 = truncation_rank(sig, q3, budget2, p.cap, &mg);
    if (p.margins) p.margins[2 * o + 1] = mg;
    const long long sz = (long long)n1 * t1 + (long long)n2 * t1 * t2 + (long long)t2 * n3;
    const unsigned long long at = atomicAdd(p.out.used, (unsigned long long)sz);
    const bool ok = (long long)(at + sz) <= p.out.capacity;
    if (!ok) atomicExch(&p.status[kStOverflow], 1);
    p.out.ranks[2 * o] = t1;
    p.out.ranks[2 * o + 1] = t2;
    p.out.off[o] = ok ? (long long)at : -1;
    atomicMax(&p.status[kStMaxR1], t1);
    atomicMax(&p.status[kStMaxR2], t2);
    if (p.acc) {
      double in_sz = 0.0;
      for (int k = 0; k < K; ++k)
        in_sz += (double)n1 * terms[k].r1 + (double)n2 * terms[k].r1 * terms[k].r2 +
                 (double)terms[k].r2 * n3;
      atomicAdd(&p.acc[0], round_flops((double)n2, (double)R1, (double)R2, (double)t1, (double)t2));
      atomicAdd(&p.acc[1], 8.0 * (in_sz + (double)sz));
    }
    s_meta[2] = ok ? 1 : 0;
    s_meta[5] = t2;
    reinterpret_cast<long long*>(sh)[20] = (long long)at;
  }
  __syncthreads();
  if (!s_meta[2]) return;
  const int t2 = s_meta[5];
  double* dst = p.out.base + reinterpret_cast<long long*>(sh)[20];
  double* dmid = dst + (long long)n1 * t1;
  double* dlast = dmid + (long long)n2 * t1 * t2;
  // ---- 5. outputs ----
  for (int e = threadIdx.x; e < n1 * t1; e += NT) dst[e] = U1[e];
  // W2 = V2(:, perm[:t2]) (q3 x t2) kept in the tail of sraw/sig? use B rows
  // beyond the S_j block: store W2 in Rr (free now).
  for (int e = threadIdx.x; e < q3 * t2; e += NT) {
    const int c = e % q3, s = e / q3;
    Rr[c + mx * s] = V2[c + n3 * perm[s]];
  }
  __syncthreads();
  for (int j = 0; j < n2; ++j) {
    for (int e = threadIdx.x; e < t1 * R2; e += NT) {
      const int r = e % t1, col = e / t1;
      const TermInfo& t = terms[colterm[col]];
      const int b = col - t.off2;
      double s = 0.0;
      for (int a = 0; a < t.r1; ++a) s += P[r + n1 * (t.off1 + a)] * mid_val(t, n1, n2, j, a, b);
      X[r + n1 * col] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < t1 * q3; e += NT) {
      const int r = e % t1, c = e / t1;
      double s = 0.0;
      for (int b = c; b < R2; ++b) s += X[r + n1 * b] * lastT[c + n3 * b];
      B[r + HMAX * c] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < t1 * t2; e += NT) {
      const int r = e % t1, s = e / t1;
      double acc = 0.0;
      for (int c = 0; c < q3; ++c) acc += B[r + HMAX * c] * Rr[c + mx * s];
      dmid[(long long)j * t1 * t2 + r + t1 * s] = acc;
    }
    __syncthreads();
  }
  // last = (Q3 [W2; 0])^T : G (n3 x t2) in B
  for (int e = threadIdx.x; e < n3 * t2; e += NT) {
    const int c = e % n3, s = e / n3;
    B[c + HMAX * s] = c < q3 ? Rr[c + mx * s] : 0.0;
  }
  __syncthreads();
  const int kmax = min(n3, R2);
  for (int k = kmax - 1; k >= 0; --k) {
    const double t = tau[k];
    if (t != 0.0) {
      for (int s = threadIdx.x; s < t2; s += NT) {
        double* g = B + HMAX * s;
        double w = g[k];
        for (int i = k + 1; i < n3; ++i) w += lastT[i + n3 * k] * g[i];
        w *= t;
        g[k] -= w;
        for (int i = k + 1; i < n3; ++i) g[i] -= w * lastT[i + n3 * k];
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < t2 * n3; e += NT) {
    const int s = e % t2, kk = e / t2;
    dlast[s + t2 * kk] = B[kk + HMAX * s];
  }
}

// Shared-memory bytes of the plan above.
size_t round_smem_bytes(int n1, int n2, int n3, int RM1, int RM2, int HMAX) {
  (void)n2;
  const size_t mx = n1 > n3 ? n1 : n3;
  size_t d = (size_t)n1 * RM1 + (size_t)n3 * RM2 + mx + mx * mx + (size_t)HMAX * mx +
             (size_t)n1 * RM2 + (size_t)n1 * RM1 + (size_t)n1 * n1 + (size_t)n3 * n3 + 2 * mx +
             32;
  size_t ints = mx + RM2 + RM1 + 1;
  size_t bytes = d * 8 + ((ints * 4 + 7) / 8) * 8 + sizeof(TermInfo) * kMaxTerms + 64;
  return bytes;
}

cudaError_t launch_round(const RoundArgs& a, cudaStream_t st) {
  if (a.nout == 0) return cudaSuccess;
  const size_t smem = round_smem_bytes(a.n1, a.n2, a.n3, a.RM1, a.RM2, a.HMAX);
  cudaError_t e = cudaFuncSetAttribute(round_sums_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  round_sums_kernel<<<a.nout, NT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace ttdvm
