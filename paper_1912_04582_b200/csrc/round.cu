// Batched FP64 TT rounding of implicit sums.
//
// One CTA (128 threads) owns one output tensor.  Its input is a list of
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
//   3. SVD of C: column-pivoted QR of C^T, then one-sided Jacobi on R^T
//      (Drmac-Veselic preconditioning: ~5 sweeps instead of ~12), which
//      yields sigma_1 and U1 without accumulating rotations; budget
//      eps^2 ||A||^2 / 2 (reference :167-169); truncation_rank (:18-29).
//   4. Cut 2: S_j = (U1^T F) M_j R3^T, TSQR of the stacked S_j -> R_S, the
//      same SVD on R_S^T -> sigma_2 and the right vectors V2.
//   5. Output first = U1, middle_j = (U1^T F) M_j (R3^T V2), last = (Q3 V2)^T.
// The middle slices of all summands for the current j are staged in shared
// memory once per use.  All arithmetic FP64.  Reconstructions equal the
// reference's up to roundoff; cores differ by an orthogonal gauge (the
// reference keeps Sigma_2 in last, here it sits in middle).
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "linalg.cuh"

namespace ttdvm {

namespace {


struct TermInfo {
  const double* base;   // state-like operand (ranks b1, b2)
  const double* fb;     // Hadamard TT factor (ranks fa1, fa2) or null
  const double* u[3];   // rank-1 face factor (axis-aligned normals) or null
  double scale;
  int r1, r2, off1, off2, refl, ms;
  int b1, b2, fa1, fa2;
};

// x / d for 0 <= x < 2^20 and 1 <= d <= 2^10 through the FP32 reciprocal
// inv = rn(1/d): (x + 0.5) inv is (x + 0.5) / d within 2^-23 relative, and
// that quotient is at least 0.5 / d (>= 2^-21 relative) from the nearest
// integer, so truncation is exact.
__device__ __forceinline__ int small_div(int x, float inv) {
  return __float2int_rz(((float)x + 0.5f) * inv);
}

// prefetch.global.L1 of the 128-byte lines covering [p, p + count)
__device__ __forceinline__ void prefetch_l1(const double* p, long long count) {
  const unsigned long long a0 = reinterpret_cast<unsigned long long>(p) & ~127ull;
  const unsigned long long a1 = reinterpret_cast<unsigned long long>(p + count);
  for (unsigned long long a = a0 + 128ull * threadIdx.x; a < a1; a += 128ull * NT)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
}

// ---- operand cache: TMA bulk copies of whole operand tensors ---------------
// Every operand (a cell's f, a face flux, J, the xi_n / |xi_n| factor of a
// face) is one contiguous [first | middle | last] block of its arena, so one
// cp.async.bulk per distinct operand brings all of an output's inputs into
// shared memory while the CTA sets up; completion is tracked by an mbarrier
// (complete_tx).  The phases that follow -- materialising F / last^T, the
// slice stages of both cuts and of the output -- then read shared memory
// instead of taking an L2 / HBM round trip each.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  const unsigned a = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// Resolve the summands of output o into TermInfo (thread k reads term k;
// thread 0 then forms the running offsets from shared memory) and the row /
// column -> term maps.  A term's ranks are (fa1 b1, fa2 b2): the Hadamard
// product fb o base (proj/src/tt_tensor.cpp:212-245) is never formed, its
// Kronecker-structured cores are built on the fly where they are consumed.
__device__ void setup_terms(const RoundArgs& p, int o, TermInfo* terms, int* rowterm,
                            int* colterm, int* s_meta, int& K, int& R1, int& R2,
                            double* ocbuf = nullptr, int OC = 0,
                            unsigned long long* ocbar = nullptr, bool prefetch = true) {
  const long long t0 = p.term_off ? p.term_off[o] : (long long)o;
  K = p.term_off ? (int)(p.term_off[o + 1] - t0) : 1;
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3;
  for (int k = threadIdx.x; k < K; k += NT) {
    const Term tm = p.terms[t0 + k];
    const TSet& s = p.sets[tm.set];
    TermInfo ti;
    ti.b1 = s.ranks[2 * tm.idx];
    ti.b2 = s.ranks[2 * tm.idx + 1];
    ti.base = s.base + s.off[tm.idx];
    double sc = tm.scale * s.uscale;
    if (s.tscale) sc *= s.tscale[tm.idx];
    if (tm.dsi >= 0) sc *= p.dscale[tm.dsi];
    ti.scale = sc;
    ti.refl = tm.refl;
    const double* fac = tm.fac >= 0 ? p.factors + (long long)tm.fac * (n1 + n2 + n3) : nullptr;
    ti.u[0] = fac ? fac : nullptr;
    ti.u[1] = fac ? fac + n1 : nullptr;
    ti.u[2] = fac ? fac + n1 + n2 : nullptr;
    if (tm.fset >= 0) {
      const TSet& f = p.sets[tm.fset];
      ti.fa1 = f.ranks[2 * tm.fidx];
      ti.fa2 = f.ranks[2 * tm.fidx + 1];
      ti.fb = f.base + f.off[tm.fidx];
    } else {
      ti.fa1 = ti.fa2 = 1;
      ti.fb = nullptr;
    }
    ti.r1 = ti.fa1 * ti.b1;
    ti.r2 = ti.fa2 * ti.b2;
    terms[k] = ti;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int off1 = 0, off2 = 0, ms = 0;
    for (int k = 0; k < K; ++k) {
      TermInfo& t = terms[k];
      t.off1 = off1;
      t.off2 = off2;
      t.ms = ms;
      off1 += t.r1;
      off2 += t.r2;
      ms += t.r1 * t.r2;
    }
    s_meta[0] = off1;
    s_meta[1] = off2;
    if (OC > 0) {
      // one bulk copy per distinct operand; a term whose operand another
      // term already fetched (f_L under both xi_n and |xi_n|) shares the copy
      const double* src[2 * kMaxTerms];
      double* dst[2 * kMaxTerms];
      int cnt[2 * kMaxTerms];
      int nsrc = 0, used = 0;
      unsigned tx = 0;
      auto place = [&](const double* g, long long doubles) -> const double* {
        for (int q = 0; q < nsrc; ++q)
          if (src[q] == g) return dst[q];
        // 16-byte aligned source and size (even n always is; else stay on global loads)
        if ((reinterpret_cast<unsigned long long>(g) & 15ull) || (doubles & 1) ||
            used + doubles > OC)
          return g;
        src[nsrc] = g;
        dst[nsrc] = ocbuf + used;
        cnt[nsrc] = (int)doubles;
        used += (int)doubles;
        tx += 8u * (unsigned)doubles;
        return dst[nsrc++];
      };
      for (int k = 0; k < K; ++k) {
        TermInfo& t = terms[k];
        t.base = place(t.base, (long long)n1 * t.b1 + (long long)n2 * t.b1 * t.b2 + (long long)t.b2 * n3);
        if (t.fb)
          t.fb = place(t.fb, (long long)n1 * t.fa1 + (long long)n2 * t.fa1 * t.fa2 + (long long)t.fa2 * n3);
      }
      mbar_init(ocbar, 1);
      mbar_expect_tx(ocbar, tx);
      for (int q = 0; q < nsrc; ++q) bulk_g2s(dst[q], src[q], 8u * (unsigned)cnt[q], ocbar);
    }
  }
  __syncthreads();
  R1 = s_meta[0];
  R2 = s_meta[1];
  for (int k = 0; k < K; ++k) {
    const TermInfo& t = terms[k];
    for (int a = threadIdx.x; a < t.r1; a += NT) rowterm[t.off1 + a] = k;
    for (int b = threadIdx.x; b < t.r2; b += NT) colterm[t.off2 + b] = k;
  }
  // Pull every summand's cores (and Hadamard factor cores) toward L1 now:
  // the slice stages of both cuts and the output read them many phases
  // later, and their loads sit on the critical path of each phase.
  const double* oc_lo = ocbuf;
  const double* oc_hi = ocbuf + OC;
  for (int k = 0; prefetch && k < K; ++k) {
    const TermInfo& t = terms[k];
    const long long nb = (long long)n1 * t.b1 + (long long)n2 * t.b1 * t.b2 + (long long)t.b2 * n3;
    if (!(OC > 0 && t.base >= oc_lo && t.base < oc_hi)) prefetch_l1(t.base, nb);
    if (t.fb && !(OC > 0 && t.fb >= oc_lo && t.fb < oc_hi))
      prefetch_l1(t.fb, (long long)n1 * t.fa1 + (long long)n2 * t.fa1 * t.fa2 + (long long)t.fa2 * n3);
  }
  if (OC > 0) mbar_wait(ocbar, 0);  // the operands have landed
}

// F (n1 x R1, ld n1) and last^T (n3 x R2, ld n3) of the implicit sum.
// Hadamard column order follows the reference: (p, q) -> p * b + q.
__device__ void materialise_outer(double* F, double* lastT, const TermInfo* terms, int K, int n1,
                                  int n2, int n3) {
  for (int k = 0; k < K; ++k) {
    const TermInfo& t = terms[k];
    for2d(n1, t.r1, [&](int i, int c) {
      int p = 0, q = c;
      if (t.fb) {
        p = c / t.b1;
        q = c - p * t.b1;
      }
      const int ii = t.refl == 1 ? n1 - 1 - i : i;
      double v = t.scale * t.base[ii + n1 * q];
      if (t.u[0]) v *= t.u[0][i];
      if (t.fb) v *= t.fb[i + n1 * p];
      F[i + n1 * (t.off1 + c)] = v;
    });
    const double* L = t.base + (long long)n1 * t.b1 + (long long)n2 * t.b1 * t.b2;
    const double* FL =
        t.fb ? t.fb + (long long)n1 * t.fa1 + (long long)n2 * t.fa1 * t.fa2 : nullptr;
    for2d(t.r2, n3, [&](int c, int kk) {  // coalesced read of last (c fastest)
      int p = 0, q = c;
      if (t.fb) {
        p = c / t.b2;
        q = c - p * t.b2;
      }
      const int kr = t.refl == 3 ? n3 - 1 - kk : kk;
      double v = L[q + t.b2 * kr];
      if (t.u[2]) v *= t.u[2][kk];
      if (FL) v *= FL[p + t.fa2 * kk];
      lastT[kk + n3 * (t.off2 + c)] = v;
    });
  }
}


// Householder QR of A (m x ncols, col-major, lda) in place: R in the upper
// triangle, reflector tails below the diagonal, tau[k].
__device__ __noinline__ void qr_inplace(double* A, int lda, int m, int ncols, double* tau, double* sh) {
  const int kmax = min(m, ncols);
  for (int k = 0; k < kmax; ++k) {
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

// qr_inplace with one barrier per column step: a group of TPC threads owns
// each column (c * TPC <= NT) and its rows (sub, sub + TPC, ...); the owner
// of column k forms its reflector (larfg, scaled tail in place) while the
// other groups are still updating for step k - 1, and learns its squared
// norm while applying step k - 1.  Same reflector format as qr_inplace.
template <int TPC>
__device__ void qr_grp_t(double* A, int lda, int m, int c, double* tau, double* sh) {
  const int g = threadIdx.x / TPC, sub = threadIdx.x % TPC;
  const int kmax = min(m, c);
  const bool own = g < c;
  double* col = A + lda * (own ? g : 0);
  double s2 = 0.0;
  if (g == 0 && own)
    for (int i = 1 + sub; i < m; i += TPC) s2 += col[i] * col[i];
  s2 = group_sum<TPC>(s2);
  for (int k = 0; k < kmax; ++k) {
    if (g == k) {  // reflector of column k (rows > k), alpha from the row-k owner
      double beta, t, sc;
      larfg(col[k], s2, beta, t, sc);  // row k: visible to the group since the last __syncwarp
      if (t != 0.0) {
        for (int i = k + 1 + ((sub - k - 1) % TPC + TPC) % TPC; i < m; i += TPC) col[i] *= sc;
        if (sub == 0) col[k] = beta;
      }
      if (sub == 0) {
        tau[k] = t;
        sh[k & 1] = t;
      }
    }
    __syncthreads();
    const double t = sh[k & 1];
    const bool act = own && g > k && t != 0.0;
    const double* v = A + lda * k;
    double w = 0.0;
    const int i0 = k + 1 + ((sub - k - 1) % TPC + TPC) % TPC;  // first own row > k
    if (act)
      for (int i = i0; i < m; i += TPC) w += v[i] * col[i];
    w = group_sum<TPC>(w);
    double ss = 0.0;
    if (act) {
      w = t * (w + col[k]);
      for (int i = i0; i < m; i += TPC) {
        const double x = col[i] - w * v[i];
        col[i] = x;
        if (i > k + 1) ss += x * x;
      }
    } else if (own && g == k + 1) {
      for (int i = i0; i < m; i += TPC)
        if (i > k + 1) ss += col[i] * col[i];
    }
    ss = group_sum<TPC>(ss);
    if (g == k + 1) s2 = ss;
    __syncwarp();  // every lane of the group has read row k
    if (act && sub == 0) col[k] -= w;
    __syncwarp();
  }
  __syncthreads();
}

__device__ __noinline__ void qr_grp(double* A, int lda, int m, int c, double* tau, double* sh) {
  if (c * 32 <= NT) qr_grp_t<32>(A, lda, m, c, tau, sh);
  else if (c * 16 <= NT) qr_grp_t<16>(A, lda, m, c, tau, sh);
  else if (c * 8 <= NT) qr_grp_t<8>(A, lda, m, c, tau, sh);
  else if (c * 4 <= NT) qr_grp_t<4>(A, lda, m, c, tau, sh);
  else if (c * 2 <= NT) qr_grp_t<2>(A, lda, m, c, tau, sh);
  else qr_grp_t<1>(A, lda, m, c, tau, sh);
}

// QR of [R; B] -> R, R upper c x c (ld ldr), B h x c (ld ldb) read once.
// Groups of TPC threads own one column each (c <= NT / TPC) and keep its
// rows (sub, sub + TPC, ...) in registers; the Householder vector of step k
// is broadcast through vbuf (double-buffered), so each column step costs one
// __syncthreads.  The owner of column k + 1 learns its squared norm while
// applying step k.
template <int TPC, int NR>
__device__ void qr_update_reg(double* R, int ldr, const double* B, int ldb, int h, int c,
                              double* vbuf, int vld, double* sh) {
  const int g = threadIdx.x / TPC, sub = threadIdx.x % TPC;
  double x[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const int row = sub + TPC * q;
    x[q] = (g < c && row < h) ? B[row + ldb * g] : 0.0;
  }
  double s2 = 0.0;  // squared norm of the own column (valid in the owner of k)
#pragma unroll
  for (int q = 0; q < NR; ++q) s2 += x[q] * x[q];
  s2 = group_sum<TPC>(s2);
  __syncthreads();  // B may be overwritten by the caller only after all loads
  for (int k = 0; k < c; ++k) {
    double* v = vbuf + (k & 1) * vld;
    if (g == k) {
      double beta, t, sc;
      larfg(R[k + ldr * k], s2, beta, t, sc);
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int row = sub + TPC * q;
        x[q] *= sc;
        if (row < h) v[row] = x[q];
      }
      if (sub == 0) {
        sh[(k & 1)] = t;
        if (t != 0.0) R[k + ldr * k] = beta;
      }
    }
    __syncthreads();
    const double t = sh[k & 1];
    const bool act = g > k && g < c;
    double w = 0.0, rkl = 0.0;
    if (act && t != 0.0) {
      rkl = R[k + ldr * g];
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int row = sub + TPC * q;
        if (row < h) w += v[row] * x[q];
      }
    }
    w = group_sum<TPC>(w);
    double ss = 0.0;
    if (act && t != 0.0) {
      w = t * (w + rkl);
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int row = sub + TPC * q;
        if (row < h) x[q] -= w * v[row];
      }
      if (sub == 0) R[k + ldr * g] = rkl - w;
    }
    if (g == k + 1) {  // next pivot column: its squared norm for step k + 1
#pragma unroll
      for (int q = 0; q < NR; ++q) ss += x[q] * x[q];
    }
    ss = group_sum<TPC>(ss);
    if (g == k + 1) s2 = ss;
  }
  __syncthreads();
}

// SMALL variant (n <= 32): one slice per update, h <= 32 rows, 8 per thread;
// large variant (n <= 48): h <= 48, 24 rows per thread.
template <bool SMALL>
__device__ void qr_update(double* R, int ldr, const double* B, int ldb, int h, int c,
                          double* vbuf, int vld, double* sh) {
  if (SMALL) {
    qr_update_reg<4, 8>(R, ldr, B, ldb, h, c, vbuf, vld, sh);  // c <= 32, h <= 32
  } else if (c <= NT / 4) {
    qr_update_reg<4, 12>(R, ldr, B, ldb, h, c, vbuf, vld, sh);  // h <= 48
  } else {
    qr_update_reg<2, 24>(R, ldr, B, ldb, h, c, vbuf, vld, sh);  // h <= 48, c <= 64
  }
}

// Column-pivoted Householder QR of M (p x m, ld ldm) in place (dgeqp3
// semantics, Q discarded): on exit the upper trapezoid holds R (k x m,
// k = min(p, m)) of M Pi, piv[i] = original column at position i.
__device__ __noinline__ void qrp_inplace(double* M, int ldm, int p, int m, double* vn, int* piv, double* sh) {
  const int kmax = min(p, m);
  for (int j = threadIdx.x; j < m; j += NT) {
    double s = 0.0;
    for (int i = 0; i < p; ++i) s += M[i + ldm * j] * M[i + ldm * j];
    vn[j] = s;
    piv[j] = j;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < kmax; ++k) {
    // argmax_{j >= k} vn[j], computed redundantly by every warp
    double bv = -1.0;
    int bi = k;
    for (int j = k + lane; j < m; j += 32) {
      const double v = vn[j];
      if (v > bv) {
        bv = v;
        bi = j;
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
    const int pv = bi;
    __syncthreads();  // everyone has read vn
    if (pv != k) {
      for (int i = threadIdx.x; i < p; i += NT) {
        const double a = M[i + ldm * k];
        M[i + ldm * k] = M[i + ldm * pv];
        M[i + ldm * pv] = a;
      }
      if (threadIdx.x == 0) {
        const double a = vn[k];
        vn[k] = vn[pv];
        vn[pv] = a;
        const int q = piv[k];
        piv[k] = piv[pv];
        piv[pv] = q;
      }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int i = k + 1 + threadIdx.x; i < p; i += 32) s += M[i + ldm * k] * M[i + ldm * k];
      s = warp_sum(s);
      if (threadIdx.x == 0) {
        double beta, t, sc;
        larfg(M[k + ldm * k], s, beta, t, sc);
        sh[0] = t;
        sh[1] = sc;
        sh[2] = beta;
      }
    }
    __syncthreads();
    const double t = sh[0], sc = sh[1];
    for (int l = k + 1 + threadIdx.x; l < m; l += NT) {
      double* col = M + ldm * l;
      double s = 0.0;
      if (t != 0.0) {
        const double* v = M + ldm * k;
        double w = col[k];
        for (int i = k + 1; i < p; ++i) w += (v[i] * sc) * col[i];
        w *= t;
        col[k] -= w;
        for (int i = k + 1; i < p; ++i) {
          const double x = col[i] - w * (v[i] * sc);
          col[i] = x;
          s += x * x;
        }
      } else {
        for (int i = k + 1; i < p; ++i) s += col[i] * col[i];
      }
      vn[l] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0 && t != 0.0) M[k + ldm * k] = sh[2];
    __syncthreads();
  }
}


// Singular values and the leading left singular vectors of C = M^T, where
// M is p x m (ld ldm, destroyed): M Pi = Q R, X = R^T (m x k), Jacobi on
// X; C = Pi X Q^T so U_C = Pi * normalised columns of X.  Writes U (m x t,
// ld ldu); returns the truncation rank (all threads).
__device__ __noinline__ int svd_left(double* M, int ldm, int p, int m, const SvdWork& w, double budget2,
                        int cap, double* U, int ldu, double* margin_out, int* s_int) {
  const int k = min(p, m);
  qrp_inplace(M, ldm, p, m, w.vn, w.piv, w.sh);
  for2d(m, k, [&](int i, int r) { w.Xs[i + w.ldx * r] = i >= r ? M[r + ldm * i] : 0.0; });
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
    U[w.piv[i] + ldu * r] = w.Xs[i + w.ldx * w.perm[r]] / w.sig[r];
  });
  __syncthreads();
  return t;
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

// Stage slice j of every summand's middle core (factor u2[j] and mode-2
// reflection applied) into Ms with coalesced loads.
__device__ void stage_slice(double* Ms, const TermInfo* terms, int K, int n1, int n2, int j) {
  for (int k = 0; k < K; ++k) {
    const TermInfo& t = terms[k];
    const int jj = t.refl == 2 ? n2 - 1 - j : j;
    const double* src = t.base + (long long)n1 * t.b1 + (long long)jj * t.b1 * t.b2;
    const double f = t.u[1] ? t.u[1][j] : 1.0;
    if (!t.fb) {
      const int sz = t.r1 * t.r2;
      for (int e = threadIdx.x; e < sz; e += NT) Ms[t.ms + e] = f * src[e];
    } else {
      // Kronecker block A2_j (x) B2_j: (p*b1 + q, p'*b2 + q') = A(p,p') B(q,q')
      const double* fs = t.fb + (long long)n1 * t.fa1 + (long long)j * t.fa1 * t.fa2;
      for2d(t.r1, t.r2, [&](int r, int c) {
        const int p = r / t.b1, q = r - p * t.b1;
        const int pp = c / t.b2, qq = c - pp * t.b2;
        Ms[t.ms + r + t.r1 * c] = f * fs[p + t.fa1 * pp] * src[q + t.b1 * qq];
      });
    }
  }
}


// ---- FP64 tensor-core (DMMA) slice products --------------------------------
// The dense products of the T route and of the high-rank bins (config 3:
// 32 x 72 x 32 per slice; config 5 residuals and the disturbed faces of
// config 4: 44..64 x ~100 x 44..64) run on mma.sync.m8n8k4.f64: each warp
// owns 16 x 16 output super-tiles (2 x 2 register-blocked 8 x 8 tiles, four
// DMMAs per four fragment loads), so a multiply-add costs 1/16 shared-memory
// load instead of the 5/4 of the 4-row FMA strips below -- those ran
// shared-memory-bound at ~6 % of the FP64 peak.  Products are IEEE FMAs
// (same per-term rounding as DFMA; the k order inside a dot product differs).
// The exact double-double Gram accumulation stays on DFMA.
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// C(i, j) = sum_{k in [kb(j0), ke(j0))} A(i, k) B(k, j) for i < M, j < N over
// `nbatch` independent problems (slices); a(q, i, k), b(q, k, j) return 0
// outside their operand, cst(q, i, j, v) stores inside bounds.  krange(j0,
// kb, ke) narrows the k loop of a 16-column super-tile (block-diagonal or
// triangular B).  Every warp of the CTA must call this (mma.sync).
template <class FA, class FB, class FC, class FK>
__device__ __forceinline__ void dmma_gemm(int nbatch, int M, int N, FA&& a, FB&& b, FC&& cst,
                                          FK&& krange) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gr = lane >> 2, gc = lane & 3;
  const int sm_ = (M + 15) >> 4, sn_ = (N + 15) >> 4;
  const int per = sm_ * sn_;
  for (int s = warp; s < nbatch * per; s += NW) {
    const int q = s / per, t = s - q * per;
    const int j0 = (t / sm_) << 4, i0 = (t - (t / sm_) * sm_) << 4;
    int kb, ke;
    krange(j0, kb, ke);
    double c00[2] = {0.0, 0.0}, c01[2] = {0.0, 0.0}, c10[2] = {0.0, 0.0}, c11[2] = {0.0, 0.0};
    const bool two_i = i0 + 8 < M, two_j = j0 + 8 < N;
    // two k-steps per iteration: eight fragment loads issued before the
    // eight DMMAs that consume them (a and b return 0 past their operand /
    // outside the block, so running up to 4 past ke adds zeros)
#pragma unroll 2
    for (int k0 = kb; k0 < ke; k0 += 8) {
      const int k1 = k0 + 4;
      const double a0 = a(q, i0 + gr, k0 + gc), a0n = a(q, i0 + gr, k1 + gc);
      const double b0 = b(q, k0 + gc, j0 + gr), b0n = b(q, k1 + gc, j0 + gr);
      double a1 = 0.0, a1n = 0.0, b1 = 0.0, b1n = 0.0;
      if (two_i) {
        a1 = a(q, i0 + 8 + gr, k0 + gc);
        a1n = a(q, i0 + 8 + gr, k1 + gc);
      }
      if (two_j) {
        b1 = b(q, k0 + gc, j0 + 8 + gr);
        b1n = b(q, k1 + gc, j0 + 8 + gr);
      }
      dmma884(c00, a0, b0);
      if (two_j) dmma884(c01, a0, b1);
      if (two_i) dmma884(c10, a1, b0);
      if (two_i && two_j) dmma884(c11, a1, b1);
      dmma884(c00, a0n, b0n);
      if (two_j) dmma884(c01, a0n, b1n);
      if (two_i) dmma884(c10, a1n, b0n);
      if (two_i && two_j) dmma884(c11, a1n, b1n);
    }
    const int r = i0 + gr, cc = j0 + 2 * gc;
    cst(q, r, cc, c00[0]);
    cst(q, r, cc + 1, c00[1]);
    if (two_j) {
      cst(q, r, cc + 8, c01[0]);
      cst(q, r, cc + 9, c01[1]);
    }
    if (two_i) {
      cst(q, r + 8, cc, c10[0]);
      cst(q, r + 8, cc + 1, c10[1]);
      if (two_j) {
        cst(q, r + 8, cc + 8, c11[0]);
        cst(q, r + 8, cc + 9, c11[1]);
      }
    }
  }
}

// Products worth the tensor cores: at least a full 8 x 8 tile in every
// dimension (the bulk low-rank bins keep the FMA strips).
__device__ __forceinline__ bool dmma_worth(int M, int N, int K) {
  return M >= 8 && N >= 8 && K >= 8;
}

// X_q (rows x R2, ld ldx, batch stride xs) = L (rows x R1, ld ldl) blockdiag(Ms_q):
// the k range of a column super-tile is the row range of the summands it meets.
__device__ void dmma_left_times_blockdiag(double* X, int ldx, int xs, const double* L, int ldl,
                                          int rows, int R1, int R2, const double* Ms, int msld,
                                          const TermInfo* terms, const int* colterm, int jn) {
  dmma_gemm(
      jn, rows, R2,
      [&](int, int i, int k) { return (i < rows && k < R1) ? L[i + ldl * k] : 0.0; },
      [&](int q, int k, int j) {
        if (j >= R2 || k >= R1) return 0.0;
        const TermInfo& t = terms[colterm[j]];
        const int a = k - t.off1;
        return (a >= 0 && a < t.r1) ? Ms[q * msld + t.ms + a + t.r1 * (j - t.off2)] : 0.0;
      },
      [&](int q, int i, int j, double v) {
        if (i < rows && j < R2) X[q * xs + i + ldx * j] = v;
      },
      [&](int j0, int& kb, int& ke) {
        const TermInfo& lo = terms[colterm[min(j0, R2 - 1)]];
        const TermInfo& hi = terms[colterm[min(j0 + 15, R2 - 1)]];
        kb = lo.off1 & ~3;
        ke = hi.off1 + hi.r1;
      });
}

// out_q(r, c) = sum_{b >= c} X_q(r, b) R3(c, b), R3 upper trapezoidal in
// lastT (ld n3; below the diagonal it holds reflectors, masked here);
// stored at out[q * os + (trans ? c + ldo * r : r + ldo * c)].
__device__ void dmma_times_r3t(double* out, int ldo, int os, bool trans, const double* X, int ldx,
                               int xs, int rows, int ncol, int R2, const double* lastT, int n3,
                               int jn) {
  dmma_gemm(
      jn, rows, ncol,
      [&](int q, int i, int k) { return (i < rows && k < R2) ? X[q * xs + i + ldx * k] : 0.0; },
      [&](int, int k, int j) { return (j < ncol && k < R2 && k >= j) ? lastT[j + n3 * k] : 0.0; },
      [&](int q, int i, int j, double v) {
        if (i < rows && j < ncol) out[q * os + (trans ? j + ldo * i : i + ldo * j)] = v;
      },
      [&](int j0, int& kb, int& ke) {
        kb = j0 & ~3;
        ke = R2;
      });
}

// X (rows x R2, ld ldxp) = L (rows x R1, ld ldl) blockdiag(Ms_t); each
// thread computes a 4-row strip of one column (4 independent FMA chains,
// one broadcast Ms load per 4 FMAs).
__device__ void left_times_blockdiag(double* X, int ldxp, const double* L, int ldl, int rows,
                                     int R2, const double* Ms, const TermInfo* terms,
                                     const int* colterm, int R1 = 0) {
  if (R1 > 0 && dmma_worth(rows, R2, R1)) {
    dmma_left_times_blockdiag(X, ldxp, 0, L, ldl, rows, R1, R2, Ms, 0, terms, colterm, 1);
    return;
  }
  const int ngr = (rows + 3) >> 2;
  for2d(ngr, R2, [&](int ig, int col) {
    const int i0 = ig << 2;
    const TermInfo& t = terms[colterm[col]];
    const int b = col - t.off2;
    const double* mcol = Ms + t.ms + t.r1 * b;
    const double* lr = L + ldl * t.off1;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (i0 + 3 < rows) {
      for (int a = 0; a < t.r1; ++a) {
        const double m = mcol[a];
        const double* l = lr + ldl * a + i0;
        a0 += l[0] * m;
        a1 += l[1] * m;
        a2 += l[2] * m;
        a3 += l[3] * m;
      }
      double* xo = X + i0 + ldxp * col;
      xo[0] = a0;
      xo[1] = a1;
      xo[2] = a2;
      xo[3] = a3;
    } else {
      for (int a = 0; a < t.r1; ++a) {
        const double m = mcol[a];
        const double* l = lr + ldl * a;
        a0 += l[i0] * m;
        if (i0 + 1 < rows) a1 += l[i0 + 1] * m;
        if (i0 + 2 < rows) a2 += l[i0 + 2] * m;
      }
      X[i0 + ldxp * col] = a0;
      if (i0 + 1 < rows) X[i0 + 1 + ldxp * col] = a1;
      if (i0 + 2 < rows) X[i0 + 2 + ldxp * col] = a2;
    }
  });
}

// out(r, c) = sum_{b >= c} X(r, b) R3(c, b) for r < rows, c < ncol, with
// R3 upper trapezoidal in lastT (ld n3); out index r + ldo*c, or c + ldo*r
// when trans.  4-row strips per thread.
__device__ void times_r3t(double* out, int ldo, bool trans, const double* X, int ldxp, int rows,
                          int ncol, int R2, const double* lastT, int n3, bool tensor = false) {
  if (tensor && dmma_worth(rows, ncol, R2)) {
    dmma_times_r3t(out, ldo, 0, trans, X, ldxp, 0, rows, ncol, R2, lastT, n3, 1);
    return;
  }
  const int ngr = (rows + 3) >> 2;
  for2d(ngr, ncol, [&](int ig, int c) {
    const int r0 = ig << 2;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int nr = min(4, rows - r0);
    if (nr == 4) {
      for (int b = c; b < R2; ++b) {
        const double l = lastT[c + n3 * b];
        const double* xp = X + r0 + ldxp * b;
        a0 += xp[0] * l;
        a1 += xp[1] * l;
        a2 += xp[2] * l;
        a3 += xp[3] * l;
      }
    } else {
      for (int b = c; b < R2; ++b) {
        const double l = lastT[c + n3 * b];
        const double* xp = X + r0 + ldxp * b;
        a0 += xp[0] * l;
        if (nr > 1) a1 += xp[1] * l;
        if (nr > 2) a2 += xp[2] * l;
      }
    }
    const double acc[4] = {a0, a1, a2, a3};
    for (int u = 0; u < nr; ++u) {
      const int r = r0 + u;
      out[trans ? (c + ldo * r) : (r + ldo * c)] = acc[u];
    }
  });
}


// Gram accumulation of the rows of T (rows x ncol, ld ldt) into the
// register-resident upper-triangle entries (ei, ej) of this thread.
// ---- slice-batched helpers of the exact-Gram kernel: jn consecutive
// slices j0 .. j0 + jn - 1 per call, flattened over (slice, element) so all
// threads stay busy when the per-slice blocks are small ----
__device__ void stage_slices(double* Ms, int msld, const TermInfo* terms, int K, int n1, int n2,
                             int j0, int jn) {
  // a thread keeps one in-slice element r (its Kronecker indices are formed
  // once) and walks the slices jj: no integer division in the loop
  for (int k = 0; k < K; ++k) {
    const TermInfo& t = terms[k];
    const int r1 = t.r1, sz = r1 * t.r2, b1 = t.b1, b2 = t.b2, fa1 = t.fa1, fa2 = t.fa2;
    const int lg = sz <= 1 ? 0 : min(LOG_NT, 32 - __clz(sz - 1));
    const int step = NT >> lg;
    const double* mb = t.base + (long long)n1 * b1;
    const double* mf = t.fb ? t.fb + (long long)n1 * fa1 : nullptr;
    const double* u1 = t.u[1];
    const bool rev = t.refl == 2;
    const float ir1 = __frcp_rn((float)r1), ib1 = __frcp_rn((float)b1), ib2 = __frcp_rn((float)b2);
    double* dst = Ms + t.ms;
    for (int r = threadIdx.x & ((1 << lg) - 1); r < sz; r += 1 << lg) {
      int os = r, of = 0;
      if (mf) {  // Kronecker block A2_j (x) B2_j: (p*b1 + q, p'*b2 + q') = A(p,p') B(q,q')
        const int c = small_div(r, ir1), a = r - c * r1;
        const int pa = small_div(a, ib1), q = a - pa * b1;
        const int pc = small_div(c, ib2), qq = c - pc * b2;
        os = q + b1 * qq;
        of = pa + fa1 * pc;
      }
#pragma unroll 1
      for (int jj = threadIdx.x >> lg; jj < jn; jj += step) {
        const int j = j0 + jj;
        const int jr = rev ? n2 - 1 - j : j;
        double v = mb[(long long)jr * b1 * b2 + os];
        if (mf) v *= mf[(long long)j * fa1 * fa2 + of];
        if (u1) v *= u1[j];
        dst[jj * msld + r] = v;
      }
    }
  }
}

// X_jj (rows x R2, ld ldx, slice stride xs) = L (rows x R1, ld ldl) blockdiag(Ms_jj)
__device__ void left_times_blockdiag_b(double* X, int ldx, int xs, const double* L, int ldl,
                                       int rows, int R2, const double* Ms, int msld,
                                       const TermInfo* terms, const int* colterm, int jn,
                                       int R1 = 0) {
  if (R1 > 0 && dmma_worth(rows, R2, R1)) {
    dmma_left_times_blockdiag(X, ldx, xs, L, ldl, rows, R1, R2, Ms, msld, terms, colterm, jn);
    return;
  }
  const int ngr = (rows + 3) >> 2;
  for2d(ngr, jn * R2, [&](int ig, int jc) {
    const int jj = jc / R2, col = jc - jj * R2;
    const int i0 = ig << 2;
    const TermInfo& t = terms[colterm[col]];
    const double* mcol = Ms + jj * msld + t.ms + t.r1 * (col - t.off2);
    const double* lr = L + ldl * t.off1;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int a = 0; a < t.r1; ++a) {
      const double m = mcol[a];
      const double* l = lr + ldl * a + i0;
      a0 += l[0] * m;
      if (i0 + 1 < rows) a1 += l[1] * m;
      if (i0 + 2 < rows) a2 += l[2] * m;
      if (i0 + 3 < rows) a3 += l[3] * m;
    }
    double* xo = X + jj * xs + ldx * col + i0;
    xo[0] = a0;
    if (i0 + 1 < rows) xo[1] = a1;
    if (i0 + 2 < rows) xo[2] = a2;
    if (i0 + 3 < rows) xo[3] = a3;
  });
}

// out_jj(c, r) = sum_{b >= c} X_jj(r, b) R3(c, b) (transposed, ld ldo, slice
// stride os) for r < rows, c < ncol; X_jj at X + jj * xs (ld ldx)
__device__ void times_r3t_b(double* out, int ldo, int os, const double* X, int ldx, int xs,
                            int rows, int ncol, int R2, const double* lastT, int n3, int jn,
                            bool tensor = false) {
  if (tensor && dmma_worth(rows, ncol, R2)) {
    dmma_times_r3t(out, ldo, os, true, X, ldx, xs, rows, ncol, R2, lastT, n3, jn);
    return;
  }
  const int ngr = (rows + 3) >> 2;
  for2d(ngr, jn * ncol, [&](int ig, int jc) {
    const int jj = jc / ncol, c = jc - jj * ncol;
    const int r0 = ig << 2;
    const double* xb = X + jj * xs + r0;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int b = c; b < R2; ++b) {
      const double l = lastT[c + n3 * b];
      const double* xp = xb + ldx * b;
      a0 += xp[0] * l;
      if (r0 + 1 < rows) a1 += xp[1] * l;
      if (r0 + 2 < rows) a2 += xp[2] * l;
      if (r0 + 3 < rows) a3 += xp[3] * l;
    }
    double* o = out + jj * os + c;
    o[ldo * r0] = a0;
    if (r0 + 1 < rows) o[ldo * (r0 + 1)] = a1;
    if (r0 + 2 < rows) o[ldo * (r0 + 2)] = a2;
    if (r0 + 3 < rows) o[ldo * (r0 + 3)] = a3;
  });
}

// Block or single-warp pivoted dd Cholesky / svd_from_r by size; results
// (rank, truncation) broadcast to the CTA through s_int.
template <bool LEAN = false>
__device__ __forceinline__ int chol_any(double* Gh, double* Gl, int d, double thresh, double* R,
                                        int ldr, int* piv, double* sh, int* s_int) {
  if constexpr (!LEAN) {
    if (d > kWarpMaxD) return chol_piv_dd(Gh, Gl, d, thresh, R, ldr, piv, sh);
  }
  if (threadIdx.x < 32) {
    const int k = chol_piv_dd_warp(Gh, Gl, d, thresh, R, ldr, piv);
    if (threadIdx.x == 0) *s_int = k;
  }
  __syncthreads();
  return *s_int;
}

template <bool LEAN = false>
__device__ __forceinline__ int svd_r_any(const double* R, int ldr, int k, int m, const int* piv,
                                         const SvdWork& w, double budget2, int cap, double* U,
                                         int ldu, double* margin_out, int* s_int) {
  if constexpr (!LEAN) {
    if (k > kWarpMaxD)
      return svd_from_r(R, ldr, k, m, piv, w, budget2, cap, U, ldu, margin_out, s_int);
  }
  if (threadIdx.x < 32) {
    const int t = svd_from_r_warp(R, ldr, k, m, piv, w, budget2, cap, U, ldu, margin_out);
    if (threadIdx.x == 0) *s_int = t;
  }
  __syncthreads();
  return *s_int;
}

template <int Q>
__device__ __forceinline__ void gram_rows_acc(double (&gh)[Q], double (&gl)[Q], const int (&ei)[Q],
                                              const int (&ej)[Q], const double* T, int ldt,
                                              int ncol) {
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (ei[q] < 0) continue;
    const double* a = T + ei[q];
    const double* b = T + ej[q];
    double h = gh[q], l = gl[q];
    for (int c = 0; c < ncol; ++c) dd_fma_acc(h, l, a[ldt * c], b[ldt * c]);
    gh[q] = h;
    gl[q] = l;
  }
}

template <int Q>
__device__ __forceinline__ void gram_store(double* Gh, double* Gl, int d, double (&gh)[Q],
                                           double (&gl)[Q], const int (&ei)[Q], const int (&ej)[Q]) {
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (ei[q] < 0) continue;
    double h = gh[q], l = gl[q];
    dd_norm(h, l);
    Gh[ei[q] + d * ej[q]] = h;
    Gl[ei[q] + d * ej[q]] = l;
    Gh[ej[q] + d * ei[q]] = h;
    Gl[ej[q] + d * ei[q]] = l;
  }
}

}  // namespace

#ifndef TTDVM_GRAM_ONLY
template <bool SMALL>
__global__ void __launch_bounds__(NT, SMALL ? 5 : 3) round_sums_kernel(RoundArgs p) {
  extern __shared__ double sm[];
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3;
  const int mx = max(n1, n3);
  const int RM1 = p.RM1, RM2 = p.RM2, HMAX = p.HMAX;
  const int RMX = max(RM1, RM2);
  const int BROWS = max(HMAX, RM2);
  // ---- shared-memory carve-up (doubles); see round_smem_bytes ----
  double* F = sm;                          // n1 x RMX   (cut 2 / output: X2)
  double* lastT = F + n1 * RMX;            // n3 x RM2
  double* tau = lastT + n3 * RM2;          // mx
  double* Rr = tau + mx;                   // mx x mx
  double* B = Rr + mx * mx;                // BROWS x mx
  double* XP = B + BROWS * mx;             // n1 x RMX   (cut 1: X; cut 2: P)
  double* U1 = XP + n1 * RMX;              // n1 x n1
  double* Xs = U1 + n1 * n1;               // mx x mx
  double* Ms = Xs + mx * mx;               // p.MSMAX
  double* vbuf = Ms + p.MSMAX;             // 2 x HMAX
  double* sig = vbuf + 2 * HMAX;           // mx
  double* sraw = sig + mx;                 // mx
  double* vn = sraw + mx;                  // mx
  double* sh = vn + mx;                    // 32 scalars
  int* perm = reinterpret_cast<int*>(sh + 32);          // mx
  int* piv = perm + mx;                                  // mx
  int* colterm = piv + mx;                               // RM2
  int* rowterm = colterm + RM2;                          // RM1
  TermInfo* terms = reinterpret_cast<TermInfo*>(
      reinterpret_cast<double*>(rowterm + RM1 + (((RM1 + RM2) & 1) ? 1 : 0)));
  __shared__ int s_meta[8];

  const int o = blockIdx.x;
  if (o >= p.nout) return;
  long long prof_t = p.prof ? clock64() : 0;
#define PROF(k)                                                      \
  if (p.prof && threadIdx.x == 0) {                                  \
    const long long t_ = clock64();                                  \
    atomicAdd(&p.prof[k], (unsigned long long)(t_ - prof_t));        \
    prof_t = t_;                                                     \
  }
  int K, R1, R2;
  setup_terms(p, o, terms, rowterm, colterm, s_meta, K, R1, R2);
  materialise_outer(F, lastT, terms, K, n1, n2, n3);
  __syncthreads();
  PROF(0);
  // ---- 1. QR of last^T ----
  qr_inplace(lastT, n3, n3, R2, tau, sh);
  const int q3 = min(n3, R2);
  PROF(1);

  // ---- 2. cut 1 TSQR ----
  const bool troute = R1 > n1;
  const int c1 = troute ? n1 : R1;
  for (int e = threadIdx.x; e < mx * mx; e += NT) Rr[e] = 0.0;
  const int ns1 = max(1, HMAX / q3);
  for (int j0 = 0; j0 < n2; j0 += ns1) {
    const int jn = min(n2, j0 + ns1);
    for (int j = j0; j < jn; ++j) {
      const int row0 = (j - j0) * q3;
      __syncthreads();
      stage_slice(Ms, terms, K, n1, n2, j);
      __syncthreads();
      if (troute) {
        // T_j^T block: B(row0 + c, i) = sum_b X(i, b) R3(c, b), X = F M_j
        left_times_blockdiag(XP, n1, F, n1, n1, R2, Ms, terms, colterm);
        __syncthreads();
        times_r3t(B + row0, HMAX, true, XP, n1, n1, q3, R2, lastT, n3);
      } else {
        // (M_j R3^T)^T block: B(row0 + c, off1 + a) = sum_b R3(c, off2 + b) M_t(a, b)
        for2d(q3, R1, [&](int c, int col) {
          const TermInfo& t = terms[rowterm[col]];
          const int a = col - t.off1;
          double s = 0.0;
          for (int b = max(0, c - t.off2); b < t.r2; ++b)
            s += lastT[c + n3 * (t.off2 + b)] * Ms[t.ms + a + t.r1 * b];
          B[row0 + c + HMAX * col] = s;
        });
      }
    }
    __syncthreads();
    PROF(2);
    qr_update<SMALL>(Rr, mx, B, HMAX, (jn - j0) * q3, c1, vbuf, HMAX, sh);
    PROF(3);
  }
  __syncthreads();

  // ---- 3. SVD of C, through M = C^T (c1 x n1) ----
  double* Mc;
  int ldmc;
  if (troute) {
    Mc = Rr;  // C^T = R_T
    ldmc = mx;
  } else {
    for2d(c1, n1, [&](int pp, int i) {  // C^T = R2 F^T
      double v = 0.0;
      for (int a = pp; a < R1; ++a) v += Rr[pp + mx * a] * F[i + n1 * a];
      B[pp + HMAX * i] = v;
    });
    Mc = B;
    ldmc = HMAX;
  }
  __syncthreads();
  double loc = 0.0;
  for2d(c1, n1, [&](int pp, int i) {
    const double v = Mc[pp + ldmc * i];
    loc += v * v;
  });
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
  const SvdWork sw{p.prof, Xs, vn, sig, sraw, piv, perm, sh, mx};
  PROF(4);
  double mg1 = 0.0;
  const int t1 = svd_left(Mc, ldmc, c1, n1, sw, budget2, p.cap, U1, n1, &mg1, &s_meta[4]);
  if (p.margins && threadIdx.x == 0) p.margins[2 * o] = mg1;
  PROF(5);
  // P = U1^T F (t1 x R1) into XP (ld n1)
  for2d(t1, R1, [&](int r, int col) {
    double s = 0.0;
    for (int i = 0; i < n1; ++i) s += U1[i + n1 * r] * F[i + n1 * col];
    XP[r + n1 * col] = s;
  });

  // ---- 4. cut 2 TSQR over S_j = P blockdiag(M_j) R3^T (t1 x q3) ----
  for (int e = threadIdx.x; e < mx * mx; e += NT) Rr[e] = 0.0;
  double* X2 = F;  // F is dead once P exists
  const int ns2 = max(1, HMAX / t1);
  for (int j0 = 0; j0 < n2; j0 += ns2) {
    const int jn = min(n2, j0 + ns2);
    for (int j = j0; j < jn; ++j) {
      const int row0 = (j - j0) * t1;
      __syncthreads();
      stage_slice(Ms, terms, K, n1, n2, j);
      __syncthreads();
      left_times_blockdiag(X2, n1, XP, n1, t1, R2, Ms, terms, colterm);
      __syncthreads();
      times_r3t(B + row0, HMAX, false, X2, n1, t1, q3, R2, lastT, n3);
    }
    __syncthreads();
    PROF(6);
    qr_update<SMALL>(Rr, mx, B, HMAX, (jn - j0) * t1, q3, vbuf, HMAX, sh);
    PROF(7);
  }
  __syncthreads();
  PROF(8);
  // ---- SVD through M = R_S (q3 x q3): left vectors of R_S^T = V2 -> B ----
  double mg2 = 0.0;
  const int t2 = svd_left(Rr, mx, q3, q3, sw, budget2, p.cap, B, HMAX, &mg2, &s_meta[5]);
  PROF(9);
  if (threadIdx.x == 0) {
    if (p.margins) p.margins[2 * o + 1] = mg2;
    const long long sz = (long long)n1 * t1 + (long long)n2 * t1 * t2 + (long long)t2 * n3;
    const unsigned long long at = atomicAdd(p.out.used, (unsigned long long)sz);
    const bool ok = (long long)(at + sz) <= p.out.capacity;
    if (!ok) atomicExch(&p.status[kStOverflow], 1);
    p.out.ranks[2 * o] = t1;
    p.out.ranks[2 * o + 1] = t2;
    p.out.off[o] = ok ? (long long)at : -1;
    // contended global atomics are spread / skipped: ranks only when larger,
    // work counters over kAccSlots slots (summed by the host)
    if (t1 > *(volatile int*)&p.status[kStMaxR1]) atomicMax(&p.status[kStMaxR1], t1);
    if (t2 > *(volatile int*)&p.status[kStMaxR2]) atomicMax(&p.status[kStMaxR2], t2);
    if (p.acc) {
      double in_sz = 0.0;
      for (int k = 0; k < K; ++k)
        in_sz += (double)n1 * terms[k].b1 + (double)n2 * terms[k].b1 * terms[k].b2 +
                 (double)terms[k].b2 * n3 +
                 (terms[k].fb ? (double)n1 * terms[k].fa1 + (double)n2 * terms[k].fa1 * terms[k].fa2 +
                                    (double)terms[k].fa2 * n3
                              : 0.0);
      double* slot = p.acc + 2 * (blockIdx.x % kAccSlots);
      atomicAdd(&slot[0], round_flops((double)n2, (double)R1, (double)R2, (double)t1, (double)t2));
      atomicAdd(&slot[1], 8.0 * (in_sz + (double)sz));
    }
    s_meta[2] = ok ? 1 : 0;
    reinterpret_cast<long long*>(sh)[20] = (long long)at;
  }
  __syncthreads();
  if (!s_meta[2]) return;
  double* dst = p.out.base + reinterpret_cast<long long*>(sh)[20];
  double* dmid = dst + (long long)n1 * t1;
  double* dlast = dmid + (long long)n2 * t1 * t2;
  // ---- 5. outputs ----
  for (int e = threadIdx.x; e < n1 * t1; e += NT) dst[e] = U1[e];
  // W2 = V2 (q3 x t2) from B into Rr (ld mx); G = [W2; 0] into Xs (ld mx)
  for2d(n3, t2, [&](int c, int s) {
    const double v = c < q3 ? B[c + HMAX * s] : 0.0;
    Xs[c + mx * s] = v;
    if (c < q3) Rr[c + mx * s] = v;
  });
  __syncthreads();
  // Z = R3^T W2 (R2 x t2, ld BROWS) into B
  double* Z = B;
  for2d(R2, t2, [&](int b, int s) {
    double acc = 0.0;
    const int cm = min(b, q3 - 1);
    for (int c = 0; c <= cm; ++c) acc += lastT[c + n3 * b] * Rr[c + mx * s];
    Z[b + BROWS * s] = acc;
  });
  // last = (Q3 G)^T, Q3 = H_0 ... H_{q3-1}: columns of G are independent,
  // one thread applies every reflector to its column
  const int kmax = min(n3, R2);
  for (int s = threadIdx.x; s < t2; s += NT) {
    double* g = Xs + mx * s;
    for (int k = kmax - 1; k >= 0; --k) {
      const double t = tau[k];
      if (t == 0.0) continue;
      double w = g[k];
      for (int i = k + 1; i < n3; ++i) w += lastT[i + n3 * k] * g[i];
      w *= t;
      g[k] -= w;
      for (int i = k + 1; i < n3; ++i) g[i] -= w * lastT[i + n3 * k];
    }
  }
  __syncthreads();
  for2d(t2, n3, [&](int s, int kk) { dlast[s + t2 * kk] = Xs[kk + mx * s]; });
  // middle_j = (P blockdiag(M_j)) Z
  for (int j = 0; j < n2; ++j) {
    __syncthreads();
    stage_slice(Ms, terms, K, n1, n2, j);
    __syncthreads();
    left_times_blockdiag(X2, n1, XP, n1, t1, R2, Ms, terms, colterm);
    __syncthreads();
    for2d(t1, t2, [&](int r, int s) {
      double a0 = 0.0, a1 = 0.0;
      int b = 0;
      for (; b + 1 < R2; b += 2) {
        a0 += X2[r + n1 * b] * Z[b + BROWS * s];
        a1 += X2[r + n1 * (b + 1)] * Z[b + 1 + BROWS * s];
      }
      if (b < R2) a0 += X2[r + n1 * b] * Z[b + BROWS * s];
      dmid[(long long)j * t1 * t2 + r + t1 * s] = a0 + a1;
    });
  }
  __syncthreads();
  PROF(10);
#undef PROF
}

#endif  // TTDVM_GRAM_ONLY

// ---------------------------------------------------------------------------
// Exact-Gram route (default): the two tall QRs of the TSQR route are
// replaced by Gram matrices accumulated in double-double (every product
// TwoProd-exact) and a pivoted double-double Cholesky, then the same
// one-sided Jacobi on R^T.  The Gram of the FP64-computed slices is exact
// to ~1e-32 relative, so sigma(R) carries the same ~u ||A|| absolute error
// as the Householder R (rounding R to FP64) -- the rank decisions keep the
// accuracy of the QR route -- while the slice loop has no sequential
// column steps (3 barriers per slice instead of 2 per column).
// The exact-Gram kernel and its launchers are compiled for two CTA widths:
// 128 threads here (namespace g128) and 256 threads in round256.cu
// (namespace g256, TTDVM_GRAM_ONLY).  Measured: the small Gram tiles of the
// config-4 face fluxes run best on 128 threads (their phases are short and
// four CTAs share an SM), the larger ones (cell residuals, config 3,
// n = 64) on 256 (more threads per dense slice product).
#if TTDVM_ROUND_NT == 512
#define RG_NS g512
#elif TTDVM_ROUND_NT == 256
#define RG_NS g256
#elif TTDVM_ROUND_NT == 32
#define RG_NS g32
#else
#define RG_NS g128
#endif
namespace RG_NS {

// Buffer plan of the exact-Gram kernel (doubles).  Shared: everything;
// with `spill`, F, last^T, XP and the Gram region move to a per-CTA global
// scratch slice (gdoubles) and JB must be 1.
struct GramPlan {
  int mx, RMX, D1, D3, D, GZ, TBZ;
};
__host__ __device__ inline GramPlan gram_plan(int n1, int n3, int RM1, int RM2, int JB) {
  GramPlan g;
  g.mx = n1 > n3 ? n1 : n3;
  g.RMX = RM1 > RM2 ? RM1 : RM2;
  g.D1 = n1 < RM1 ? n1 : RM1;
  g.D3 = n3 < RM2 ? n3 : RM2;
  g.D = g.D1 > g.D3 ? g.D1 : g.D3;
  g.GZ = 2 * g.D * g.D > RM2 * g.D ? 2 * g.D * g.D : RM2 * g.D;
  g.TBZ = g.mx * g.D > JB * g.D1 * g.D3 ? g.mx * g.D : JB * g.D1 * g.D3;
  return g;
}

// One output per call (one CTA of NT threads).  SPILL: see gram_plan.
// LEAN: the launch's summed ranks stay below the mode sizes and its Gram
// dimensions within the single-warp factorizations (RM1 < n1, RM2 <= n3,
// D <= kWarpMaxD: the bulk bins of the step), so only the W route, the
// grouped QR of last^T and the warp-level Cholesky / Jacobi are compiled in
// -- a third of the instructions of the general body (the general kernel
// showed 14 % of its warp stalls waiting on instruction fetch).
template <int Q, bool SPILL, bool LEAN = false>
__device__ __forceinline__ void round_gram_body(const RoundArgs& p, const int o, double* sm,
                                                int* s_meta) {
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3;
  const int RM1 = p.RM1, RM2 = p.RM2;
  // Buffers scale with D = max(min(n1, RM1), min(n3, RM2)) -- the largest
  // Gram / SVD dimension of this launch -- not with n^2, so launches of
  // low-rank sums (the rank bins of run_round) fit several CTAs per SM.
  // JB slices per barrier phase in the W route, cut 2 and the output (the
  // T route stages one slice at a time); chosen by the host from the budget
  const int JB = SPILL ? 1 : p.JB;
  const GramPlan gp = gram_plan(n1, n3, RM1, RM2, JB);
  const int mx = gp.mx, RMX = gp.RMX, D1 = gp.D1, D3 = gp.D3, D = gp.D;
  const int OC = SPILL ? 0 : p.OC;
  double* ocbuf = sm;              // OC doubles, 16-byte aligned (operand cache)
  double* cur = sm + ((OC + 1) & ~1);
  double *F, *lastT, *XP, *G;
  if (SPILL) {
    F = p.gscratch + (long long)blockIdx.x * p.gstride;  // n1 x RMX
    lastT = F + n1 * RMX;                                 // n3 x RM2
    XP = lastT + n3 * RM2;                                // n1 x RMX
    G = XP + n1 * RMX;                                    // GZ
  } else {
    F = cur;                       // n1 x RMX   (cut 2 / output: X2 when JB = 1)
    cur += n1 * RMX;
    lastT = cur;                   // n3 x RM2
    cur += n3 * RM2;
  }
  double* tau = cur;               // mx
  cur += mx;
  double* Tb = cur;                // TBZ        (slice blocks, C^T; V2 at the end)
  cur += gp.TBZ;
  if (!SPILL) {
    G = cur;                       // GZ         (Gram hi/lo planes; Z at the end)
    cur += gp.GZ;
    XP = cur;                      // n1 x RMX   (cut 1: X; cut 2: P)
    cur += n1 * RMX;
  }
  double* Gl = G + D * D;
  double* U1 = cur;                // n1 x D1
  cur += n1 * D1;
  double* Xs = cur;                // mx x D     (Jacobi workspace)
  cur += mx * D;
  double* Rc = cur;                // D x D      (Cholesky factor)
  cur += D * D;
  double* Ms = cur;                // JB x p.MSMAX (staged middle slices)
  cur += JB * p.MSMAX;
  double* X2c = cur;               // JB x D1 x RMX when JB > 1 (P M_j per slice)
  cur += JB > 1 ? JB * D1 * RMX : 0;
  double* sig = cur;               // mx
  double* sraw = sig + mx;         // mx
  double* vn = sraw + mx;          // mx
  double* sh = vn + mx;            // 32 scalars
  int* perm = reinterpret_cast<int*>(sh + 32);          // mx
  int* piv = perm + mx;                                  // mx
  int* colterm = piv + mx;                               // RM2
  int* rowterm = colterm + RM2;                          // RM1
  TermInfo* terms = reinterpret_cast<TermInfo*>(
      reinterpret_cast<double*>(rowterm + RM1 + (((RM1 + RM2) & 1) ? 1 : 0)));

  long long prof_t = p.prof ? clock64() : 0;
  // diagnostics: per-phase cycles of thread 0, with a barrier first so a
  // phase is charged to the phase that did the work (profiling runs only)
#define PROF(k)                                                      \
  if (p.prof) {                                                      \
    __syncthreads();                                                 \
    if (threadIdx.x == 0) {                                          \
      const long long t_ = clock64();                                \
      atomicAdd(&p.prof[k], (unsigned long long)(t_ - prof_t));      \
      prof_t = t_;                                                   \
    }                                                                \
  }
  int K, R1, R2;
  setup_terms(p, o, terms, rowterm, colterm, s_meta, K, R1, R2, ocbuf, OC,
              reinterpret_cast<unsigned long long*>(s_meta + 8));
  materialise_outer(F, lastT, terms, K, n1, n2, n3);
  __syncthreads();
  PROF(0);
  if (LEAN || R2 <= NT) {
    qr_grp(lastT, n3, n3, R2, tau, sh);
  } else {
    qr_inplace(lastT, n3, n3, R2, tau, sh);
  }
  const int q3 = min(n3, R2);
  PROF(1);

  // ---- cut 1 ----
  // T route (R1 >= n1): G1 = sum_j T_j T_j^T (n1 x n1), T_j = F M_j R3^T;
  //   sigma(A_(1)) and U1 from its pivoted Cholesky factor.
  // W route (R1 < n1): G_W = sum_j Z_j Z_j^T (R1 x R1), Z_j = M_j R3^T, so
  //   A_(1) A_(1)^T = C C^T with C = F Pi R_W^T (n1 x k); sigma and U1 from
  //   the column-pivoted QR + Jacobi of C^T (svd_left).  R1 x R1 work per
  //   slice instead of n1 x n1 -- the common case of low-rank sums.
  const bool wroute = LEAN || R1 < n1;
  const int d1 = wroute ? R1 : n1;
  int ei[Q], ej[Q];
  double gh[Q], gl[Q];
  {
    const int ne = d1 * (d1 + 1) / 2;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int e = threadIdx.x + NT * q;
      gh[q] = gl[q] = 0.0;
      if (e < ne) tri_index(e, d1, ei[q], ej[q]);
      else ei[q] = ej[q] = -1;
    }
  }
  if (LEAN || wroute) {
    for (int j0 = 0; j0 < n2; j0 += JB) {
      const int jn = min(JB, n2 - j0);
      __syncthreads();
      PROF(2);
      stage_slices(Ms, p.MSMAX, terms, K, n1, n2, j0, jn);
      __syncthreads();
      PROF(11);
      // Z_j^T: Tb(a, (jj, c)) = sum_b M_t(a, b) R3(c, off2 + b), R3 upper
      // trapezoidal.  Row a is fixed per thread (its term is looked up once);
      // (jj, c) advance without division.
      {
        const int lg = R1 <= 1 ? 0 : min(LOG_NT, 32 - __clz(R1 - 1));
        const int a = threadIdx.x & ((1 << lg) - 1), step = NT >> lg;
        const int ncol = jn * q3;
        for (int a2 = a; a2 < R1; a2 += (1 << lg)) {
          const TermInfo& t = terms[rowterm[a2]];
          const int r1 = t.r1, r2 = t.r2, off2 = t.off2;
          const double* mbase = Ms + t.ms + (a2 - t.off1);
          const double* lb = lastT + n3 * off2;
          int jc = threadIdx.x >> lg;
          int jj = jc / q3, c = jc - jj * q3;
#pragma unroll 1
          for (; jc < ncol; jc += step) {
            const double* mj = mbase + jj * p.MSMAX;
            double s = 0.0;
            for (int b = max(0, c - off2); b < r2; ++b) s += lb[c + n3 * b] * mj[r1 * b];
            Tb[a2 + d1 * jc] = s;
            c += step;
            while (c >= q3) {
              c -= q3;
              ++jj;
            }
          }
        }
      }
      __syncthreads();
      PROF(4);
      gram_rows_acc<Q>(gh, gl, ei, ej, Tb, d1, jn * q3);
    }
  } else if constexpr (!LEAN) {
    for (int j = 0; j < n2; ++j) {
      __syncthreads();
      stage_slice(Ms, terms, K, n1, n2, j);
      __syncthreads();
      left_times_blockdiag(XP, n1, F, n1, n1, R2, Ms, terms, colterm, p.no_dmma ? 0 : R1);
      __syncthreads();
      times_r3t(Tb, n1, false, XP, n1, n1, q3, R2, lastT, n3, !p.no_dmma);
      __syncthreads();
      gram_rows_acc<Q>(gh, gl, ei, ej, Tb, d1, q3);
    }
  }
  __syncthreads();
  gram_store<Q>(G, Gl, d1, gh, gl, ei, ej);
  __syncthreads();
  PROF(2);
  double loc = 0.0;
  for (int i = threadIdx.x; i < d1; i += NT) loc += G[i + d1 * i] + Gl[i + d1 * i];
  const double trace = block_sum(loc, sh + 8);
  double norm2 = trace;
  int k1 = 0;
  if (wroute && trace > 0.0 && isfinite(trace)) {
    k1 = chol_any<LEAN>(G, Gl, d1, 1e-31 * trace, Rc, D, piv, sh, &s_meta[6]);
    // M = C^T (k1 x n1, ld D1) into Tb: M(r, i) = sum_{v >= r} R_W(r, v) F(i, piv[v])
    double l2 = 0.0;
    for2d(k1, n1, [&](int r, int i) {
      double s = 0.0;
      for (int v = r; v < d1; ++v) s += Rc[r + D * v] * F[i + n1 * piv[v]];
      Tb[r + D1 * i] = s;
      l2 += s * s;
    });
    norm2 = block_sum(l2, sh + 8);
  }
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
  const double cthresh = 1e-31 * norm2;
  const SvdWork sw{p.prof, Xs, vn, sig, sraw, piv, perm, sh, mx};
  double mg1 = 0.0;
  int t1;
  if (LEAN || (wroute && k1 <= kWarpMaxD)) {
    // sigma and U1 of C (n1 x k1, C^T in Tb) through its k1 x k1 Gram:
    // exact dd Gram -> pivoted dd Cholesky Rg -> Jacobi on Rg^T gives sigma
    // and the right vectors V (into XP, k1 x t1); U1 = C V / sigma.  The
    // retained sigma are >= eps ||A|| / sqrt(2), so U1 carries at most
    // ~u / eps relative error; the rank decisions see sigma to ~u ||A||.
    PROF(3);
    {
      const int ne = k1 * (k1 + 1) / 2;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int e = threadIdx.x + NT * q;
        gh[q] = gl[q] = 0.0;
        if (e < ne) tri_index(e, k1, ei[q], ej[q]);
        else ei[q] = ej[q] = -1;
      }
    }
    gram_rows_acc<Q>(gh, gl, ei, ej, Tb, D1, n1);
    gram_store<Q>(G, Gl, k1, gh, gl, ei, ej);
    __syncthreads();
    const int kc = chol_any<LEAN>(G, Gl, k1, cthresh, Rc, D, piv, sh, &s_meta[6]);
    double* V = XP;  // k1 x t1
    t1 = svd_r_any<LEAN>(Rc, D, kc, k1, piv, sw, budget2, p.cap, V, k1, &mg1, &s_meta[4]);
    for2d(n1, t1, [&](int i, int r) {
      double a0 = 0.0, a1 = 0.0;
      int v = 0;
      for (; v + 1 < k1; v += 2) {
        a0 += Tb[v + D1 * i] * V[v + k1 * r];
        a1 += Tb[v + 1 + D1 * i] * V[v + 1 + k1 * r];
      }
      if (v < k1) a0 += Tb[v + D1 * i] * V[v + k1 * r];
      U1[i + n1 * r] = (a0 + a1) / sig[r];
    });
    __syncthreads();
  } else if constexpr (!LEAN) {
    if (wroute) {
      PROF(3);
      t1 = svd_left(Tb, D1, k1, n1, sw, budget2, p.cap, U1, n1, &mg1, &s_meta[4]);
    } else {
      k1 = chol_any(G, Gl, n1, cthresh, Rc, D, piv, sh, &s_meta[6]);
      PROF(3);
      t1 = svd_r_any(Rc, D, k1, n1, piv, sw, budget2, p.cap, U1, n1, &mg1, &s_meta[4]);
    }
  }
  if (p.margins && threadIdx.x == 0) p.margins[2 * o] = mg1;
  PROF(5);
  for2d(t1, R1, [&](int r, int col) {  // P = U1^T F
    double s = 0.0;
    for (int i = 0; i < n1; ++i) s += U1[i + n1 * r] * F[i + n1 * col];
    XP[r + n1 * col] = s;
  });

  // ---- cut 2: G2 = sum_j S_j^T S_j (q3 x q3), S_j = P M_j R3^T ----
  {
    const int ne = q3 * (q3 + 1) / 2;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int e = threadIdx.x + NT * q;
      gh[q] = gl[q] = 0.0;
      if (e < ne) tri_index(e, q3, ei[q], ej[q]);
      else ei[q] = ej[q] = -1;
    }
  }
  // X2_j = P blockdiag(M_j) (t1 x R2, ld t1), JB slices per phase.  When
  // every slice's X2_j fits the region at once (small t1), they are kept for
  // the output stage; when the W route staged all slices at once, cut 2
  // reuses them.
  double* X2 = JB > 1 ? X2c : F;
  const bool keepX2 =
      (long long)n2 * t1 * R2 <= (long long)(JB > 1 ? JB * D1 * RMX : n1 * RMX);
  const bool staged_all = wroute && JB >= n2;
  for (int j0 = 0; j0 < n2; j0 += JB) {
    const int jn = min(JB, n2 - j0);
    double* X2j = keepX2 ? X2 + j0 * t1 * R2 : X2;
    __syncthreads();
    PROF(6);
    if (!staged_all) {
      stage_slices(Ms, p.MSMAX, terms, K, n1, n2, j0, jn);
      __syncthreads();
    }
    PROF(11);
    left_times_blockdiag_b(X2j, t1, t1 * R2, XP, n1, t1, R2, Ms, p.MSMAX, terms, colterm, jn,
                           (LEAN || p.no_dmma) ? 0 : R1);
    __syncthreads();
    // S_j^T (q3 x t1) at column block jj
    times_r3t_b(Tb, q3, q3 * t1, X2j, t1, t1 * R2, t1, q3, R2, lastT, n3, jn, !LEAN && !p.no_dmma);
    __syncthreads();
    PROF(8);
    gram_rows_acc<Q>(gh, gl, ei, ej, Tb, q3, jn * t1);
  }
  __syncthreads();
  gram_store<Q>(G, Gl, q3, gh, gl, ei, ej);
  __syncthreads();
  PROF(6);
  const int k2 = chol_any<LEAN>(G, Gl, q3, cthresh, Rc, D, piv, sh, &s_meta[6]);
  PROF(7);
  double mg2 = 0.0;
  double* W2 = Tb;  // V2 (q3 x t2), ld D3
  const int t2 = svd_r_any<LEAN>(Rc, D, k2, q3, piv, sw, budget2, p.cap, W2, D3, &mg2, &s_meta[5]);
  PROF(9);
  if (threadIdx.x == 0) {
    if (p.margins) p.margins[2 * o + 1] = mg2;
    const long long sz = (long long)n1 * t1 + (long long)n2 * t1 * t2 + (long long)t2 * n3;
    const unsigned long long at = atomicAdd(p.out.used, (unsigned long long)sz);
    const bool ok = (long long)(at + sz) <= p.out.capacity;
    if (!ok) atomicExch(&p.status[kStOverflow], 1);
    p.out.ranks[2 * o] = t1;
    p.out.ranks[2 * o + 1] = t2;
    p.out.off[o] = ok ? (long long)at : -1;
    // contended global atomics are spread / skipped: ranks only when larger,
    // work counters over kAccSlots slots (summed by the host)
    if (t1 > *(volatile int*)&p.status[kStMaxR1]) atomicMax(&p.status[kStMaxR1], t1);
    if (t2 > *(volatile int*)&p.status[kStMaxR2]) atomicMax(&p.status[kStMaxR2], t2);
    if (p.acc) {
      double in_sz = 0.0;
      for (int k = 0; k < K; ++k)
        in_sz += (double)n1 * terms[k].b1 + (double)n2 * terms[k].b1 * terms[k].b2 +
                 (double)terms[k].b2 * n3 +
                 (terms[k].fb ? (double)n1 * terms[k].fa1 + (double)n2 * terms[k].fa1 * terms[k].fa2 +
                                    (double)terms[k].fa2 * n3
                              : 0.0);
      double* slot = p.acc + 2 * (blockIdx.x % kAccSlots);
      atomicAdd(&slot[0], round_flops((double)n2, (double)R1, (double)R2, (double)t1, (double)t2));
      atomicAdd(&slot[1], 8.0 * (in_sz + (double)sz));
    }
    s_meta[2] = ok ? 1 : 0;
    reinterpret_cast<long long*>(sh)[20] = (long long)at;
  }
  __syncthreads();
  if (!s_meta[2]) return;
  double* dst = p.out.base + reinterpret_cast<long long*>(sh)[20];
  double* dmid = dst + (long long)n1 * t1;
  double* dlast = dmid + (long long)n2 * t1 * t2;
  for (int e = threadIdx.x; e < n1 * t1; e += NT) dst[e] = U1[e];
  // G = [W2; 0] (n3 x t2) into Xs; Z = R3^T W2 (R2 x t2, ld RM2) into the Gram region
  for2d(n3, t2, [&](int c, int s) { Xs[c + mx * s] = c < q3 ? W2[c + D3 * s] : 0.0; });
  double* Z = G;
  for2d(R2, t2, [&](int b, int s) {
    double acc = 0.0;
    const int cm = min(b, q3 - 1);
    for (int c = 0; c <= cm; ++c) acc += lastT[c + n3 * b] * W2[c + D3 * s];
    Z[b + RM2 * s] = acc;
  });
  __syncthreads();
  const int kmax = min(n3, R2);
  {  // one warp per column of G, lanes over rows
    const int lane = threadIdx.x & 31;
    for (int s = threadIdx.x >> 5; s < t2; s += NW) {
      double* g = Xs + mx * s;
      for (int k = kmax - 1; k >= 0; --k) {
        const double t = tau[k];
        if (t == 0.0) continue;
        const double* v = lastT + n3 * k;
        double w = 0.0;
        for (int i = k + 1 + lane; i < n3; i += 32) w += v[i] * g[i];
        w = t * (warp_sum(w) + g[k]);
        __syncwarp();
        if (lane == 0) g[k] -= w;
        for (int i = k + 1 + lane; i < n3; i += 32) g[i] -= w * v[i];
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for2d(t2, n3, [&](int s, int kk) { dlast[s + t2 * kk] = Xs[kk + mx * s]; });
  for (int j0 = 0; j0 < n2; j0 += (keepX2 ? n2 : JB)) {
    const int jn = keepX2 ? n2 : min(JB, n2 - j0);
    __syncthreads();
    if (!keepX2) {
      stage_slices(Ms, p.MSMAX, terms, K, n1, n2, j0, jn);
      __syncthreads();
      left_times_blockdiag_b(X2, t1, t1 * R2, XP, n1, t1, R2, Ms, p.MSMAX, terms, colterm, jn,
                             (LEAN || p.no_dmma) ? 0 : R1);
      __syncthreads();
    }
    // middle_j = (P blockdiag(M_j)) Z
    if (!LEAN && !p.no_dmma && dmma_worth(t1, t2, R2)) {
      double* dm = dmid + (long long)j0 * t1 * t2;
      dmma_gemm(
          jn, t1, t2,
          [&](int q, int i, int k) { return (i < t1 && k < R2) ? X2[q * t1 * R2 + i + t1 * k] : 0.0; },
          [&](int, int k, int j) { return (k < R2 && j < t2) ? Z[k + RM2 * j] : 0.0; },
          [&](int q, int i, int j, double v) {
            if (i < t1 && j < t2) dm[(long long)q * t1 * t2 + i + t1 * j] = v;
          },
          [&](int, int& kb, int& ke) {
            kb = 0;
            ke = R2;
          });
    } else
    for2d(t1, jn * t2, [&](int r, int js) {
      const int jj = js / t2, s = js - jj * t2;
      const double* x = X2 + jj * t1 * R2 + r;
      const double* z = Z + RM2 * s;
      double a0 = 0.0, a1 = 0.0;
      int b = 0;
      for (; b + 1 < R2; b += 2) {
        a0 += x[t1 * b] * z[b];
        a1 += x[t1 * (b + 1)] * z[b + 1];
      }
      if (b < R2) a0 += x[t1 * b] * z[b];
      dmid[(long long)(j0 + jj) * t1 * t2 + r + t1 * s] = a0 + a1;
    });
  }
  __syncthreads();
  PROF(10);
#undef PROF
}

// Shared-memory plans: one CTA per output (6 / 4 / 3 CTAs per SM by Gram
// size); SPILL launches are persistent (grid = resident CTAs) and loop.
// Q = 0 is the Q = 1 body built for 1024 / NT resident CTAs (64 registers at
// 128 threads): tiny Gram tiles (D <= kTinyD), whose plans fit eight CTAs
// per SM in shared memory.
#ifndef TTDVM_TINY_MINB
#define TTDVM_TINY_MINB 8
#endif
template <int Q, bool SPILL, bool LEAN = false>
__global__ void __launch_bounds__(NT, SPILL ? 1 : (Q == 0 ? TTDVM_TINY_MINB * 128 / NT : (Q <= 3 ? 512 / NT : (Q <= 10 ? (NT == 128 ? 3 : 1) : 1))))
    round_gram_kernel(RoundArgs p) {
  constexpr int QB = Q == 0 ? 1 : Q;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) int s_meta[10];  // [8..9]: the operand cache's mbarrier
  if constexpr (!SPILL) {
    const int o = p.olist ? p.olist[blockIdx.x] : blockIdx.x;
    if (o < p.nout) round_gram_body<QB, false, LEAN>(p, o, sm, s_meta);
  } else {
    for (int b = blockIdx.x; b < p.nblk; b += gridDim.x) {
      const int o = p.olist ? p.olist[b] : b;
      __syncthreads();  // the previous output's shared-memory readers are done
      if (o < p.nout) round_gram_body<QB, true>(p, o, sm, s_meta);
    }
  }
}

size_t round_gram_smem_bytes(int n1, int n3, int RM1, int RM2, int MSMAX, int JB, bool spill) {
  if (spill) JB = 1;
  const GramPlan g = gram_plan(n1, n3, RM1, RM2, JB);
  const size_t big = spill ? 0
                           : (size_t)n1 * g.RMX + (size_t)n3 * RM2 + (size_t)g.GZ +
                                 (size_t)n1 * g.RMX;
  size_t d = big + g.mx + g.TBZ + (size_t)n1 * g.D1 + (size_t)g.mx * g.D + (size_t)g.D * g.D +
             (size_t)JB * MSMAX + (JB > 1 ? (size_t)JB * g.D1 * g.RMX : 0) + 3 * g.mx + 32;
  size_t ints = 2 * g.mx + RM2 + RM1 + 1;
  return d * 8 + ((ints * 4 + 7) / 8) * 8 + sizeof(TermInfo) * kMaxTerms + 64;
}

// Doubles of one CTA's global scratch slice in the spill plan (32-aligned).
long long round_gram_spill_doubles(int n1, int n3, int RM1, int RM2) {
  const GramPlan g = gram_plan(n1, n3, RM1, RM2, 1);
  const long long d = 2LL * n1 * g.RMX + (long long)n3 * RM2 + g.GZ;
  return (d + 31) / 32 * 32;
}

// Largest Gram dimension D that takes the 8-CTA tiny variant (128-thread
// build): TTDVM_TINY_D, default 0 = off.  Measured on config 4 (half scale,
// same box): D <= 8 cuts the collision roundings by ~24 % but slows the
// update roundings about as much (spills at 64 registers); D <= 12 doubles
// the flux phase.
int round_gram_tiny_d() {
  static const int v = [] {
    const char* e = getenv("TTDVM_TINY_D");
    return e ? atoi(e) : 0;
  }();
  return NT == 128 ? v : 0;
}
int round_gram_tiny_minb() { return TTDVM_TINY_MINB; }

template <bool SPILL>
static cudaError_t launch_gram_q(const RoundArgs& a, int grid, size_t smem, cudaStream_t st,
                                 int* resident) {
  const int D1 = a.n1 < a.RM1 ? a.n1 : a.RM1, D3 = a.n3 < a.RM2 ? a.n3 : a.RM2;
  const int D = D1 > D3 ? D1 : D3;
  const int ne = D * (D + 1) / 2;
  cudaError_t e = cudaSuccess;
  // the pruned build for the bulk bins (see round_gram_body); TTDVM_LEAN=0
  // keeps the general kernel (A/B)
  static const bool lean_on = [] {
    const char* e = getenv("TTDVM_LEAN");
    return !(e && *e == '0');
  }();
  const bool lean = !SPILL && lean_on && a.RM1 < a.n1 && a.RM2 <= a.n3 && D <= kWarpMaxD;
#define LAUNCH_Q(QV)                                                                         \
  if (lean && (QV) >= 1 && (QV) <= 5) {                                                      \
    constexpr int QL = (QV) >= 1 && (QV) <= 5 ? (QV) : 1;                                    \
    auto kern = round_gram_kernel<QL, false, true>;                                          \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    if (e != cudaSuccess) return e;                                                          \
    kern<<<grid, NT, smem, st>>>(a);                                                         \
  } else {                                                                                   \
    auto kern = round_gram_kernel<QV, SPILL>;                                                \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
    if (e != cudaSuccess) return e;                                                          \
    if (resident) {                                                                          \
      int per = 0, dev = 0, sms = 0;                                                         \
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NT, smem);               \
      if (e != cudaSuccess) return e;                                                        \
      cudaGetDevice(&dev);                                                                   \
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);                     \
      *resident = per * sms;                                                                 \
      return cudaSuccess;                                                                    \
    }                                                                                        \
    kern<<<grid, NT, smem, st>>>(a);                                                         \
  }
  bool tiny = false;
  if constexpr (!SPILL && NT == 128) {
    if (D <= round_gram_tiny_d()) {
      tiny = true;
      LAUNCH_Q(0)
    }
  }
  if (tiny) {
  } else if (ne <= NT) {
    LAUNCH_Q(1)
  } else if (ne <= 3 * NT) {
    LAUNCH_Q(3)
  } else if (ne <= 5 * NT) {
    LAUNCH_Q(5)
  } else if (ne <= 10 * NT) {
    LAUNCH_Q(10)
  } else if (ne <= 17 * NT) {
    LAUNCH_Q(17)
  } else if (NT < 256 && ne <= 33 * NT) {
    LAUNCH_Q(33)
  } else {
    return cudaErrorInvalidValue;
  }
#undef LAUNCH_Q
  return cudaGetLastError();
}

// Resident CTAs of the spill plan (persistent grid size), from the occupancy API.
cudaError_t round_gram_resident(const RoundArgs& a, int* resident) {
  const size_t smem = round_gram_smem_bytes(a.n1, a.n3, a.RM1, a.RM2, a.MSMAX, 1, true);
  return launch_gram_q<true>(a, 0, smem, nullptr, resident);
}

// a.gscratch != null selects the spill plan: grid CTAs loop over a.nblk outputs.
cudaError_t launch_round_gram(const RoundArgs& a, int nblocks, cudaStream_t st) {
  if (nblocks == 0) return cudaSuccess;
  if (a.gscratch) {
    const size_t smem = round_gram_smem_bytes(a.n1, a.n3, a.RM1, a.RM2, a.MSMAX, 1, true);
    return launch_gram_q<true>(a, nblocks, smem, st, nullptr);
  }
  const size_t smem = round_gram_smem_bytes(a.n1, a.n3, a.RM1, a.RM2, a.MSMAX, a.JB, false) +
                      8 * (size_t)((a.OC + 1) & ~1);
  return launch_gram_q<false>(a, nblocks, smem, st, nullptr);
}

#include "round_pipe.cuh"

}  // namespace RG_NS

#ifndef TTDVM_GRAM_ONLY
// Shared-memory bytes of the plan above.
size_t round_smem_bytes(int n1, int n2, int n3, int RM1, int RM2, int HMAX, int MSMAX) {
  (void)n2;
  const size_t mx = n1 > n3 ? n1 : n3;
  const size_t RMX = RM1 > RM2 ? RM1 : RM2;
  const size_t BROWS = HMAX > RM2 ? HMAX : RM2;
  size_t d = (size_t)n1 * RMX + (size_t)n3 * RM2 + mx + mx * mx + BROWS * mx +
             (size_t)n1 * RMX + (size_t)n1 * n1 + mx * mx + (size_t)MSMAX + 2 * (size_t)HMAX +
             3 * mx + 32;
  size_t ints = 2 * mx + RM2 + RM1 + 1;
  size_t bytes = d * 8 + ((ints * 4 + 7) / 8) * 8 + sizeof(TermInfo) * kMaxTerms + 64;
  return bytes;
}

// Rank bins (SURVEY.md §7 hard part 3): outputs are grouped by the largest
// summed rank max(R1, R2) so that each launch's shared-memory plan -- and
// with it the CTAs per SM -- fits its own outputs.  bins[b] lists the
// outputs with kRankEdges[b-1] < key <= kRankEdges[b]; bmax[4 b + {0,1,2}]
// are the bin's RM1, RM2, MSMAX.  Order inside a bin is nondeterministic;
// every output is computed independently, so results are not.
__global__ void __launch_bounds__(256) round_bin_kernel(RoundArgs p, int* counts, int* bmax,
                                                        int* lists) {
  // Block-aggregated: per-bin counts and maxima are reduced in shared memory
  // and each block reserves one range per bin with a single global atomic
  // (the per-output global atomics of a 1.5 M-output launch contended on 44
  // addresses).
  __shared__ int s_cnt[kRankBins], s_base[kRankBins], s_max[kRankBins * kBinWords];
  for (int o0 = blockIdx.x * blockDim.x; o0 < p.nout; o0 += gridDim.x * blockDim.x) {
    for (int i = threadIdx.x; i < kRankBins * (1 + kBinWords); i += blockDim.x) {
      if (i < kRankBins) s_cnt[i] = 0;
      else s_max[i - kRankBins] = 0;
    }
    __syncthreads();
    const int o = o0 + threadIdx.x;
    int bin = -1, pos = 0;
    if (o < p.nout) {
      const long long t0 = p.term_off ? p.term_off[o] : o;
      const int K = p.term_off ? (int)(p.term_off[o + 1] - t0) : 1;
      int r1 = 0, r2 = 0, ms = 0, oc = 0;
      for (int k = 0; k < K; ++k) {
        const Term tm = p.terms[t0 + k];
        const TSet& s = p.sets[tm.set];
        int a = s.ranks[2 * tm.idx], b = s.ranks[2 * tm.idx + 1];
        // doubles of the distinct operands (operand cache): an operand that an
        // earlier summand of this output already names is counted once
        bool dup = false, fdup = tm.fset < 0;
        for (int q = 0; q < k; ++q) {
          const Term tq = p.terms[t0 + q];
          dup |= tq.set == tm.set && tq.idx == tm.idx;
          fdup |= tq.fset == tm.fset && tq.fidx == tm.fidx;
        }
        if (!dup) oc += p.n1 * a + p.n2 * a * b + b * p.n3;
        if (tm.fset >= 0) {
          const int fa = p.sets[tm.fset].ranks[2 * tm.fidx], fb = p.sets[tm.fset].ranks[2 * tm.fidx + 1];
          if (!fdup) oc += p.n1 * fa + p.n2 * fa * fb + fb * p.n3;
          a *= fa;
          b *= fb;
        }
        r1 += a;
        r2 += b;
        ms += a * b;
      }
      const int key = max(r1, r2);
      bin = 0;
      while (bin < kRankBins - 1 && key > kRankEdges[bin]) ++bin;
      pos = atomicAdd(&s_cnt[bin], 1);
      atomicMax(&s_max[kBinWords * bin], r1);
      atomicMax(&s_max[kBinWords * bin + 1], r2);
      atomicMax(&s_max[kBinWords * bin + 2], ms);
      atomicMax(&s_max[kBinWords * bin + 3], K);
      atomicMax(&s_max[kBinWords * bin + 4], oc);
    }
    __syncthreads();
    if (threadIdx.x < kRankBins) {
      const int b = threadIdx.x;
      if (s_cnt[b] > 0) {
        s_base[b] = atomicAdd(&counts[b], s_cnt[b]);
        for (int w = 0; w < kBinWords; ++w)
          if (s_max[kBinWords * b + w] > bmax[kBinWords * b + w])
            atomicMax(&bmax[kBinWords * b + w], s_max[kBinWords * b + w]);
      }
    }
    __syncthreads();
    if (bin >= 0) lists[(long long)bin * p.nout + s_base[bin] + pos] = o;
    __syncthreads();
  }
}

cudaError_t launch_round_bins(const RoundArgs& a, int* counts, int* bmax, int* lists,
                              cudaStream_t st) {
  if (a.nout == 0) return cudaSuccess;
  const int blocks = min(1184, (a.nout + 255) / 256);
  round_bin_kernel<<<blocks, 256, 0, st>>>(a, counts, bmax, lists);
  return cudaGetLastError();
}

cudaError_t launch_round(const RoundArgs& a, cudaStream_t st) {
  if (a.nout == 0) return cudaSuccess;
  const size_t smem = round_smem_bytes(a.n1, a.n2, a.n3, a.RM1, a.RM2, a.HMAX, a.MSMAX);
  const bool small = a.n1 <= 32 && a.n3 <= 32 && a.HMAX <= 32;
  cudaError_t e = small ? cudaFuncSetAttribute(round_sums_kernel<true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                        : cudaFuncSetAttribute(round_sums_kernel<false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (small)
    round_sums_kernel<true><<<a.nout, NT, smem, st>>>(a);
  else
    round_sums_kernel<false><<<a.nout, NT, smem, st>>>(a);
  return cudaGetLastError();
}

#endif  // TTDVM_GRAM_ONLY

}  // namespace ttdvm
