// round_pipe.cuh -- the rounding of the bulk rank bins as a PIPELINE of six
// batched phase kernels (included by round.cu inside namespace
// g32, the one-warp-CTA build).
//
// The one-CTA-per-output kernel (round_gram_body) walks an output through
// ~12 dependent phases inside one CTA: three n x D shared-memory buffers and
// 128 registers per thread cap it at 12-16 outputs per SM, and three of its
// four warps idle during the single-warp factorizations.  Here each phase is
// its own kernel over all outputs of a chunk, ONE WARP PER OUTPUT, with only
// the buffers that phase needs in shared memory (6-15 KB) and the
// intermediates that cross a phase boundary in a per-output record in
// global memory (L2-resident between launches):
//
//   P1 prep      summands -> F, last^T; Householder QR of last^T       -> F, LT, tau
//   P2 gram1     per slice Z_j = M_j R3^T; G_W = sum_j Z_j Z_j^T (dd)  -> G
//   P3 factor1   chol(G_W), C = F Pi R_W^T, Gram/chol/Jacobi of C       -> t1, U1, P = U1^T F
//   P4 gram2     S_j = P M_j R3^T; G2 = sum_j S_j^T S_j (dd)            -> G
//   P5 factor2   chol/Jacobi of G2 -> t2, V2; allocate the output;
//                first = U1, last = (Q3 [V2; 0])^T, Z = R3^T V2         -> Z, offset
//   P6 middle    middle_j = (P M_j) Z
//
// Same arithmetic, in the same order, as the LEAN instantiation of
// round_gram_body (W route, grouped QR, warp-level pivoted double-double
// Cholesky and one-sided Jacobi): the helpers are the same functions, so
// the truncation decisions and the cores are those of the one-kernel path.
// Eligibility is the LEAN condition (RM1 < n1, RM2 <= n3, D <= kWarpMaxD).
#if TTDVM_ROUND_NT == 32

struct PipeArgs {
  RoundArgs p;
  double* rec;         // [count] records of `stride` doubles
  long long stride;
  int first;           // first entry of p.olist (or first output) of this chunk
  int count;
  int JB;              // slices per stage in P2 / P4 / P6
  int il;              // Gram accumulation with the lane's entries interleaved (pipe_gram_acc)
  int zt;              // P2: Z_j rows per lane, transposed Z buffer, vector loads in the Gram loop
  int oF, oLT, oTau, oG, oU1, oP, oZ, oS, oX2, oMs;  // record offsets (doubles)
  int keepms;          // P2 stores the staged middle slices; P4 / P6 copy them instead of restaging
  int tkeep;           // outputs with t1 <= tkeep keep X2_j = P M_j (all slices) for P6
};

// record scalars at oS: doubles [0] budget2, [1] cthresh, [2] input doubles
// (work counter); ints at +4: [0] t1, [1] t2, [2] flag (0 live, 1 finished
// early or dropped), [3] R1, [4] R2; long long at +8: output offset.
struct PipeRec {
  double *F, *LT, *tau, *G, *U1, *P, *Z, *sc, *X2, *Ms;
  int* iv;
  long long* off;
};
__device__ __forceinline__ PipeRec pipe_rec(const PipeArgs& a, int slot) {
  double* r = a.rec + (long long)slot * a.stride;
  PipeRec q;
  q.F = r + a.oF;
  q.LT = r + a.oLT;
  q.tau = r + a.oTau;
  q.G = r + a.oG;
  q.U1 = r + a.oU1;
  q.P = r + a.oP;
  q.Z = r + a.oZ;
  q.sc = r + a.oS;
  q.X2 = r + a.oX2;
  q.Ms = r + a.oMs;
  q.iv = reinterpret_cast<int*>(r + a.oS + 4);
  q.off = reinterpret_cast<long long*>(r + a.oS + 8);
  return q;
}

__device__ __forceinline__ int pipe_output(const PipeArgs& a, int slot) {
  return a.p.olist ? a.p.olist[a.first + slot] : a.first + slot;
}

// shared-memory tail common to the phases that stage slices: TermInfo table
// and the row / column -> summand maps
struct PipeTerms {
  TermInfo* terms;
  int *rowterm, *colterm;
};
__device__ __forceinline__ PipeTerms pipe_terms(double* at, int RM1, int RM2) {
  PipeTerms t;
  t.colterm = reinterpret_cast<int*>(at);
  t.rowterm = t.colterm + RM2;
  t.terms = reinterpret_cast<TermInfo*>(
      reinterpret_cast<double*>(t.rowterm + RM1 + (((RM1 + RM2) & 1) ? 1 : 0)));
  return t;
}
static size_t pipe_terms_bytes(int RM1, int RM2) {
  return (((size_t)(RM1 + RM2 + 1) * 4 + 7) / 8) * 8 + sizeof(TermInfo) * kMaxTerms;
}

// leading dimension of P2's transposed Z buffer: the batch's columns rounded
// up to even (16-byte rows) plus two, so consecutive rows start 16 bytes
// apart modulo the bank period
__host__ __device__ inline int pipe_ldz(int JB, int D3) { return ((JB * D3 + 1) & ~1) + 2; }

// R3 (upper trapezoid of the factored last^T, rows < q3) from the record
// into shared memory with leading dimension ld
__device__ __forceinline__ void pipe_load_r3(double* R3, int ld, const double* LT, int n3, int q3,
                                             int R2) {
  for (int e = threadIdx.x; e < q3 * R2; e += NT) {
    const int b = e / q3, c = e - b * q3;
    R3[c + ld * b] = c <= b ? LT[c + n3 * b] : 0.0;
  }
}

// Householder QR of A (m x c, m <= 64, ld lda) by ONE warp with the lanes over
// the ROWS (two per lane, in registers for the current reflector): every
// trailing column costs two FMAs, one warp sum and two FMAs per lane, and
// four columns are in flight at a time.  qr_grp's column-owner layout leaves
// a one-warp CTA with two lanes per column and the finished columns' lanes
// idle (~7.5k warp instructions for 44 x 12 against ~1.7k here).  Same
// reflector format (larfg, scaled tails below the diagonal, tau) -- the sums
// are associated differently, as they already are between the 32- and
// 128-thread builds of qr_grp.
#ifndef TTDVM_PIPE_QR_ROWS
#define TTDVM_PIPE_QR_ROWS 1
#endif
__device__ __forceinline__ void pipe_qr_rows(double* A, int lda, int m, int c, double* tau) {
  const int lane = threadIdx.x & 31;
  const int i0 = lane, i1 = lane + 32;
  const int kmax = min(m, c);
  for (int k = 0; k < kmax; ++k) {
    double* ck = A + lda * k;
    const bool in0 = i0 > k && i0 < m, in1 = i1 > k && i1 < m;
    double v0 = in0 ? ck[i0] : 0.0, v1 = in1 ? ck[i1] : 0.0;
    const double s2 = warp_sum(v0 * v0 + v1 * v1);
    double beta, t, sc;
    larfg(ck[k], s2, beta, t, sc);  // every lane: same inputs, same result
    __syncwarp();
    if (lane == 0) {
      tau[k] = t;
      if (t != 0.0) ck[k] = beta;
    }
    if (t == 0.0) continue;
    v0 *= sc;
    v1 *= sc;
    if (in0) ck[i0] = v0;
    if (in1) ck[i1] = v1;
    int l = k + 1;
    for (; l + 3 < c; l += 4) {
      double* c0 = A + lda * l;
      double* c1 = c0 + lda;
      double* c2 = c1 + lda;
      double* c3 = c2 + lda;
      const double a00 = in0 ? c0[i0] : 0.0, a01 = in1 ? c0[i1] : 0.0;
      const double a10 = in0 ? c1[i0] : 0.0, a11 = in1 ? c1[i1] : 0.0;
      const double a20 = in0 ? c2[i0] : 0.0, a21 = in1 ? c2[i1] : 0.0;
      const double a30 = in0 ? c3[i0] : 0.0, a31 = in1 ? c3[i1] : 0.0;
      double w0 = v0 * a00 + v1 * a01, w1 = v0 * a10 + v1 * a11;
      double w2 = v0 * a20 + v1 * a21, w3 = v0 * a30 + v1 * a31;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        w0 += __shfl_xor_sync(0xffffffffu, w0, o);
        w1 += __shfl_xor_sync(0xffffffffu, w1, o);
        w2 += __shfl_xor_sync(0xffffffffu, w2, o);
        w3 += __shfl_xor_sync(0xffffffffu, w3, o);
      }
      w0 = t * (w0 + c0[k]);
      w1 = t * (w1 + c1[k]);
      w2 = t * (w2 + c2[k]);
      w3 = t * (w3 + c3[k]);
      __syncwarp();  // every lane has read row k
      if (in0) {
        c0[i0] = a00 - w0 * v0;
        c1[i0] = a10 - w1 * v0;
        c2[i0] = a20 - w2 * v0;
        c3[i0] = a30 - w3 * v0;
      }
      if (in1) {
        c0[i1] = a01 - w0 * v1;
        c1[i1] = a11 - w1 * v1;
        c2[i1] = a21 - w2 * v1;
        c3[i1] = a31 - w3 * v1;
      }
      if (lane == 0) {
        c0[k] -= w0;
        c1[k] -= w1;
        c2[k] -= w2;
        c3[k] -= w3;
      }
    }
    for (; l < c; ++l) {
      double* c0 = A + lda * l;
      const double a00 = in0 ? c0[i0] : 0.0, a01 = in1 ? c0[i1] : 0.0;
      double w0 = warp_sum(v0 * a00 + v1 * a01);
      w0 = t * (w0 + c0[k]);
      __syncwarp();
      if (in0) c0[i0] = a00 - w0 * v0;
      if (in1) c0[i1] = a01 - w0 * v1;
      if (lane == 0) c0[k] -= w0;
    }
    __syncwarp();
  }
  __syncwarp();
}

// ---- P1 ---------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 16) pipe_prep_kernel(PipeArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) int s_meta[10];
  const int slot = blockIdx.x;
  if (slot >= a.count) return;
  const RoundArgs& p = a.p;
  const int o = pipe_output(a, slot);
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3, RM1 = p.RM1, RM2 = p.RM2;
  double* F = sm;
  double* lastT = F + n1 * RM1;
  double* tau = lastT + n3 * RM2;
  double* sh = tau + n3;
  PipeTerms pt = pipe_terms(sh + 32, RM1, RM2);
  int K, R1, R2;
  setup_terms(p, o, pt.terms, pt.rowterm, pt.colterm, s_meta, K, R1, R2);
  materialise_outer(F, lastT, pt.terms, K, n1, n2, n3);
  __syncthreads();
  if (TTDVM_PIPE_QR_ROWS && n3 <= 64) pipe_qr_rows(lastT, n3, n3, R2, tau);
  else qr_grp(lastT, n3, n3, R2, tau, sh);
  __syncthreads();
  PipeRec r = pipe_rec(a, slot);
  for (int e = threadIdx.x; e < n1 * R1; e += NT) r.F[e] = F[e];
  for (int e = threadIdx.x; e < n3 * R2; e += NT) r.LT[e] = lastT[e];
  for (int e = threadIdx.x; e < R2; e += NT) r.tau[e] = tau[e];
  if (threadIdx.x == 0) {
    double in_sz = 0.0;
    for (int k = 0; k < K; ++k) {
      const TermInfo& t = pt.terms[k];
      in_sz += (double)n1 * t.b1 + (double)n2 * t.b1 * t.b2 + (double)t.b2 * n3 +
               (t.fb ? (double)n1 * t.fa1 + (double)n2 * t.fa1 * t.fa2 + (double)t.fa2 * n3 : 0.0);
    }
    r.sc[2] = in_sz;
    r.iv[0] = 0;
    r.iv[1] = 0;
    r.iv[2] = 0;
    r.iv[3] = R1;
    r.iv[4] = R2;
  }
}

// Z_j^T of the W route: Tb(a, (jj, c)) = sum_b M_t(a, b) R3(c, off2 + b)
// (the loop of round_gram_body's cut 1, R3 with leading dimension ldr)
__device__ __forceinline__ void pipe_zj(double* Tb, const double* Ms, int msmax,
                                        const TermInfo* terms, const int* rowterm, const double* R3,
                                        int ldr, int R1, int q3, int jn) {
  const int lg = R1 <= 1 ? 0 : min(LOG_NT, 32 - __clz(R1 - 1));
  const int a = threadIdx.x & ((1 << lg) - 1), step = NT >> lg;
  const int ncol = jn * q3;
  for (int a2 = a; a2 < R1; a2 += (1 << lg)) {
    const TermInfo& t = terms[rowterm[a2]];
    const int r1 = t.r1, r2 = t.r2, off2 = t.off2;
    const double* mbase = Ms + t.ms + (a2 - t.off1);
    const double* lb = R3 + ldr * off2;
    int jc = threadIdx.x >> lg;
    int jj = jc / q3, c = jc - jj * q3;
#pragma unroll 1
    for (; jc < ncol; jc += step) {
      const double* mj = mbase + jj * msmax;
      double s = 0.0;
      for (int b = max(0, c - off2); b < r2; ++b) s += lb[c + ldr * b] * mj[r1 * b];
      Tb[a2 + R1 * jc] = s;
      c += step;
      while (c >= q3) {
        c -= q3;
        ++jj;
      }
    }
  }
}

// gram_rows_acc with the Q entries of a lane advanced together: one column
// loop for all of them (a third of the loop overhead at Q = 3) and Q
// independent double-double chains in flight.  Every entry still sums its
// columns in ascending order, so the Gram is bitwise that of gram_rows_acc.
template <int Q>
__device__ __forceinline__ void pipe_gram_acc(double (&gh)[Q], double (&gl)[Q], const int (&ei)[Q],
                                              const int (&ej)[Q], const double* T, int ldt,
                                              int ncol) {
  const double* pa[Q];
  const double* pb[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    pa[q] = T + (ei[q] < 0 ? 0 : ei[q]);
    pb[q] = T + (ei[q] < 0 ? 0 : ej[q]);
  }
#pragma unroll 2
  for (int c = 0; c < ncol; ++c) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (ei[q] >= 0) dd_fma_acc(gh[q], gl[q], *pa[q], *pb[q]);
      pa[q] += ldt;
      pb[q] += ldt;
    }
  }
}

template <int Q>
__device__ __forceinline__ void pipe_gram_init(int d, int (&ei)[Q], int (&ej)[Q], double (&gh)[Q],
                                               double (&gl)[Q]) {
  const int ne = d * (d + 1) / 2;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int e = threadIdx.x + NT * q;
    gh[q] = gl[q] = 0.0;
    if (e < ne) tri_index(e, d, ei[q], ej[q]);
    else ei[q] = ej[q] = -1;
  }
}

// Z_j of the W route with ONE (row a, slice jj) PAIR PER LANE: the lane keeps
// its row of M_t in registers and walks the q3 columns, so a multiply-add
// costs one shared-memory load of R3 (broadcast among the lanes of a summand)
// instead of two loads plus the per-element index arithmetic of pipe_zj.
// Stored transposed, Zt(a, jj * q3 + c) at Zt[jj * q3 + c + ldz * a]: the
// Gram loop then reads consecutive columns with 16-byte loads.  R3 is zero
// below its diagonal and padded by four zero columns, so the b loop needs no
// bounds; every sum still adds its terms in ascending b (the skipped ones
// are exact zeros): the values are those of pipe_zj.
__device__ __forceinline__ void pipe_zj_rows(double* Zt, int ldz, const double* Ms, int msmax,
                                             const TermInfo* terms, const int* rowterm,
                                             const double* R3, int ldr, int R1, int q3, int jn) {
  for (int pr = threadIdx.x; pr < R1 * jn; pr += NT) {
    const int jj = pr / R1, a2 = pr - jj * R1;
    const TermInfo& t = terms[rowterm[a2]];
    const int r1 = t.r1, r2 = t.r2;
    const double* mj = Ms + jj * msmax + t.ms + (a2 - t.off1);
    const double* lb = R3 + ldr * t.off2;
    double* z = Zt + jj * q3 + ldz * a2;
    if (r2 <= 4) {
      const double m0 = mj[0], m1 = r2 > 1 ? mj[r1] : 0.0, m2 = r2 > 2 ? mj[2 * r1] : 0.0,
                   m3 = r2 > 3 ? mj[3 * r1] : 0.0;
#pragma unroll 4
      for (int c = 0; c < q3; ++c) {
        double sacc = m0 * lb[c];
        sacc = fma(m1, lb[c + ldr], sacc);
        sacc = fma(m2, lb[c + 2 * ldr], sacc);
        sacc = fma(m3, lb[c + 3 * ldr], sacc);
        z[c] = sacc;
      }
    } else {
      for (int c = 0; c < q3; ++c) {
        double sacc = 0.0;
        for (int b = max(0, c - t.off2); b < r2; ++b) sacc += lb[c + ldr * b] * mj[r1 * b];
        z[c] = sacc;
      }
    }
  }
}

// Gram accumulation over the rows of the transposed buffer (entry (i, j) =
// sum_c Zt[c + ld i] Zt[c + ld j]), columns in ascending order, four per
// iteration through 16-byte loads.
template <int Q>
__device__ __forceinline__ void pipe_gram_acc_t(double (&gh)[Q], double (&gl)[Q],
                                                const int (&ei)[Q], const int (&ej)[Q],
                                                const double* T, int ld, int ncol) {
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (ei[q] < 0) continue;
    const double* x = T + ld * ei[q];
    const double* y = T + ld * ej[q];
    double h = gh[q], l = gl[q];
    int c = 0;
    for (; c + 4 <= ncol; c += 4) {
      const double2 x0 = *reinterpret_cast<const double2*>(x + c);
      const double2 x1 = *reinterpret_cast<const double2*>(x + c + 2);
      const double2 y0 = *reinterpret_cast<const double2*>(y + c);
      const double2 y1 = *reinterpret_cast<const double2*>(y + c + 2);
      dd_fma_acc(h, l, x0.x, y0.x);
      dd_fma_acc(h, l, x0.y, y0.y);
      dd_fma_acc(h, l, x1.x, y1.x);
      dd_fma_acc(h, l, x1.y, y1.y);
    }
    for (; c < ncol; ++c) dd_fma_acc(h, l, x[c], y[c]);
    gh[q] = h;
    gl[q] = l;
  }
}

// ---- P2 ---------------------------------------------------------------------
template <int Q>
#ifndef TTDVM_PIPE_P2_MINB
#define TTDVM_PIPE_P2_MINB 24
#endif
__global__ void __launch_bounds__(NT, TTDVM_PIPE_P2_MINB) pipe_gram1_kernel(PipeArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) int s_meta[10];
  const int slot = blockIdx.x;
  if (slot >= a.count) return;
  const RoundArgs& p = a.p;
  const int o = pipe_output(a, slot);
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3, RM1 = p.RM1, RM2 = p.RM2, JB = a.JB;
  const int D3 = RM2;
  const int ldz = pipe_ldz(JB, D3);
  double* R3 = sm;                        // D3 x (RM2 + 4), zero below the diagonal and in the pad
  double* Tb = R3 + ((D3 * (RM2 + 4) + 1) & ~1);  // Z batch (16-byte aligned): JB x RM1 x D3, or
                                                  // RM1 rows of ldz (transposed)
  double* Ms = Tb + RM1 * ldz;            // JB x MSMAX
  PipeTerms pt = pipe_terms(Ms + JB * p.MSMAX, RM1, RM2);
  PipeRec r = pipe_rec(a, slot);
  int K, R1, R2;
  setup_terms(p, o, pt.terms, pt.rowterm, pt.colterm, s_meta, K, R1, R2);
  const int q3 = min(n3, R2);
  for (int e = threadIdx.x; e < D3 * (RM2 + 4); e += NT) R3[e] = 0.0;
  __syncthreads();
  pipe_load_r3(R3, D3, r.LT, n3, q3, R2);
  int ei[Q], ej[Q];
  double gh[Q], gl[Q];
  pipe_gram_init<Q>(R1, ei, ej, gh, gl);
  if (a.keepms) {
    // every slice of every summand staged ONCE, straight into the record
    // (one set-up of the Kronecker indices per summand, all lanes busy over
    // the 44 slices); the batches below and P4 / P6 read plain copies
    stage_slices(r.Ms, p.MSMAX, pt.terms, K, n1, n2, 0, n2);
  }
  for (int j0 = 0; j0 < n2; j0 += JB) {
    const int jn = min(JB, n2 - j0);
    __syncthreads();  // (first pass: the record's slices written by this CTA are visible)
    if (a.keepms) {
      const double* mg = r.Ms + (long long)j0 * p.MSMAX;
      for (int e = threadIdx.x; e < jn * p.MSMAX; e += NT) Ms[e] = mg[e];
    } else {
      stage_slices(Ms, p.MSMAX, pt.terms, K, n1, n2, j0, jn);
    }
    __syncthreads();
    if (a.zt) {
      pipe_zj_rows(Tb, ldz, Ms, p.MSMAX, pt.terms, pt.rowterm, R3, D3, R1, q3, jn);
      __syncthreads();
      pipe_gram_acc_t<Q>(gh, gl, ei, ej, Tb, ldz, jn * q3);
    } else {
      pipe_zj(Tb, Ms, p.MSMAX, pt.terms, pt.rowterm, R3, D3, R1, q3, jn);
      __syncthreads();
      if (a.il) pipe_gram_acc<Q>(gh, gl, ei, ej, Tb, R1, jn * q3);
      else gram_rows_acc<Q>(gh, gl, ei, ej, Tb, R1, jn * q3);
    }
  }
  gram_store<Q>(r.G, r.G + RM1 * RM1, R1, gh, gl, ei, ej);
}

// ---- P3 ---------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(NT, 12) pipe_factor1_kernel(PipeArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int slot = blockIdx.x;
  if (slot >= a.count) return;
  const RoundArgs& p = a.p;
  const int o = pipe_output(a, slot);
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3, RM1 = p.RM1, RM2 = p.RM2;
  const int D1 = RM1, D = RM1 > RM2 ? RM1 : RM2;
  PipeRec r = pipe_rec(a, slot);
  const int R1 = r.iv[3];
  double* F = sm;                  // n1 x R1
  double* Tb = F + n1 * RM1;       // C^T: k1 x n1, ld D1
  double* G = Tb + n1 * D1;        // D x D
  double* Gl = G + D * D;
  double* Rc = Gl + D * D;         // D x D
  double* V = Rc + D * D;          // k1 x t1
  double* Xs = V + D * D;          // D x D (Jacobi workspace)
  double* sig = Xs + D * D;
  double* sraw = sig + D;
  double* vn = sraw + D;
  double* sh = vn + D;             // 32
  int* piv = reinterpret_cast<int*>(sh + 32);
  int* perm = piv + D;
  for (int e = threadIdx.x; e < n1 * R1; e += NT) F[e] = r.F[e];
  for (int e = threadIdx.x; e < R1 * R1; e += NT) {
    G[e] = r.G[e];
    Gl[e] = r.G[RM1 * RM1 + e];
  }
  __syncthreads();
  double loc = 0.0;
  for (int i = threadIdx.x; i < R1; i += NT) loc += G[i + R1 * i] + Gl[i + R1 * i];
  const double trace = block_sum(loc, sh + 8);
  double norm2 = trace;
  int k1 = 0;
  if (trace > 0.0 && isfinite(trace)) {
    k1 = chol_piv_dd_warp(G, Gl, R1, 1e-31 * trace, Rc, D, piv);
    __syncthreads();
    double l2 = 0.0;
    for2d(k1, n1, [&](int rr, int i) {
      double s = 0.0;
      for (int v = rr; v < R1; ++v) s += Rc[rr + D * v] * F[i + n1 * piv[v]];
      Tb[rr + D1 * i] = s;
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
      r.iv[2] = 1;
      r.off[0] = ok ? (long long)at : -1;
      if (p.margins) {
        p.margins[2 * o] = INFINITY;
        p.margins[2 * o + 1] = INFINITY;
      }
    }
    __syncthreads();
    const long long at = r.off[0];
    if (at >= 0) {
      double* dst = p.out.base + at;
      for (int e = threadIdx.x; e < n1 + n2 + n3; e += NT) dst[e] = e < n1 ? 0.0 : 1.0;
    }
    return;
  }
  const double budget2 = p.eps * p.eps * norm2 / 2.0;
  const double cthresh = 1e-31 * norm2;
  const SvdWork sw{p.prof, Xs, vn, sig, sraw, piv, perm, sh, D};
  int ei[Q], ej[Q];
  double gh[Q], gl[Q];
  pipe_gram_init<Q>(k1, ei, ej, gh, gl);
  gram_rows_acc<Q>(gh, gl, ei, ej, Tb, D1, n1);
  gram_store<Q>(G, Gl, k1, gh, gl, ei, ej);
  __syncthreads();
  const int kc = chol_piv_dd_warp(G, Gl, k1, cthresh, Rc, D, piv);
  __syncthreads();
  double mg1 = 0.0;
  const int t1 = svd_from_r_warp(Rc, D, kc, k1, piv, sw, budget2, p.cap, V, k1, &mg1);
  __syncthreads();
  for2d(n1, t1, [&](int i, int rr) {
    double a0 = 0.0, a1 = 0.0;
    int v = 0;
    for (; v + 1 < k1; v += 2) {
      a0 += Tb[v + D1 * i] * V[v + k1 * rr];
      a1 += Tb[v + 1 + D1 * i] * V[v + 1 + k1 * rr];
    }
    if (v < k1) a0 += Tb[v + D1 * i] * V[v + k1 * rr];
    r.U1[i + n1 * rr] = (a0 + a1) / sig[rr];
  });
  __syncthreads();  // U1 (global) written by this CTA is visible to it
  for2d(t1, R1, [&](int rr, int col) {  // P = U1^T F
    double s = 0.0;
    for (int i = 0; i < n1; ++i) s += r.U1[i + n1 * rr] * F[i + n1 * col];
    r.P[rr + D1 * col] = s;
  });
  if (threadIdx.x == 0) {
    r.sc[0] = budget2;
    r.sc[1] = cthresh;
    r.iv[0] = t1;
    if (p.margins) p.margins[2 * o] = mg1;
  }
  (void)n3;
  (void)RM2;
}

// ---- P4 ---------------------------------------------------------------------
template <int Q>
__global__ void __launch_bounds__(NT, 24) pipe_gram2_kernel(PipeArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) int s_meta[10];
  const int slot = blockIdx.x;
  if (slot >= a.count) return;
  const RoundArgs& p = a.p;
  PipeRec r = pipe_rec(a, slot);
  if (r.iv[2]) return;
  const int o = pipe_output(a, slot);
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3, RM1 = p.RM1, RM2 = p.RM2, JB = a.JB;
  const int D1 = RM1, D3 = RM2;
  const int t1 = r.iv[0];
  double* R3 = sm;                        // D3 x RM2
  double* XP = R3 + D3 * RM2;             // t1 x R1, ld D1
  double* X2 = XP + D1 * RM1;             // JB x t1 x R2
  double* Tb = X2 + JB * D1 * RM2;        // JB x q3 x t1
  double* Ms = Tb + JB * D3 * D1;         // JB x MSMAX
  PipeTerms pt = pipe_terms(Ms + JB * p.MSMAX, RM1, RM2);
  int K, R1, R2;
  setup_terms(p, o, pt.terms, pt.rowterm, pt.colterm, s_meta, K, R1, R2, nullptr, 0, nullptr,
              !a.keepms);
  const int q3 = min(n3, R2);
  pipe_load_r3(R3, D3, r.LT, n3, q3, R2);
  for (int e = threadIdx.x; e < D1 * R1; e += NT) XP[e] = r.P[e];
  int ei[Q], ej[Q];
  double gh[Q], gl[Q];
  pipe_gram_init<Q>(q3, ei, ej, gh, gl);
  for (int j0 = 0; j0 < n2; j0 += JB) {
    const int jn = min(JB, n2 - j0);
    __syncthreads();
    if (a.keepms) {
      const double* mg = r.Ms + (long long)j0 * p.MSMAX;
      for (int e = threadIdx.x; e < jn * p.MSMAX; e += NT) Ms[e] = mg[e];
    } else {
      stage_slices(Ms, p.MSMAX, pt.terms, K, n1, n2, j0, jn);
    }
    __syncthreads();
    left_times_blockdiag_b(X2, t1, t1 * R2, XP, D1, t1, R2, Ms, p.MSMAX, pt.terms, pt.colterm, jn);
    __syncthreads();
    if (t1 <= a.tkeep) {  // low-rank outputs keep P M_j for the output stage (no restaging in P6)
      double* xg = r.X2 + (long long)j0 * t1 * R2;
      for (int e = threadIdx.x; e < jn * t1 * R2; e += NT) xg[e] = X2[e];
    }
    times_r3t_b(Tb, q3, q3 * t1, X2, t1, t1 * R2, t1, q3, R2, R3, D3, jn);
    __syncthreads();
    if (a.il) pipe_gram_acc<Q>(gh, gl, ei, ej, Tb, q3, jn * t1);
    else gram_rows_acc<Q>(gh, gl, ei, ej, Tb, q3, jn * t1);
  }
  gram_store<Q>(r.G, r.G + RM2 * RM2, q3, gh, gl, ei, ej);
}

// ---- P5 ---------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 12) pipe_factor2_kernel(PipeArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int slot = blockIdx.x;
  if (slot >= a.count) return;
  const RoundArgs& p = a.p;
  PipeRec r = pipe_rec(a, slot);
  if (r.iv[2]) return;
  const int o = pipe_output(a, slot);
  const int n1 = p.n1, n2 = p.n2, n3 = p.n3, RM1 = p.RM1, RM2 = p.RM2;
  const int D3 = RM2, D = RM1 > RM2 ? RM1 : RM2;
  const int t1 = r.iv[0], R1 = r.iv[3], R2 = r.iv[4];
  const int q3 = min(n3, R2);
  double* lastT = sm;              // n3 x R2 (reflectors + R3)
  double* tau = lastT + n3 * RM2;  // R2
  double* Xq = tau + n3;           // n3 x t2 (Q3 [V2; 0])
  double* G = Xq + n3 * D3;        // D x D
  double* Gl = G + D * D;
  double* Rc = Gl + D * D;
  double* W2 = Rc + D * D;         // q3 x t2, ld D3
  double* Xs = W2 + D * D;         // D x D
  double* sig = Xs + D * D;
  double* sraw = sig + D;
  double* vn = sraw + D;
  double* sh = vn + D;             // 32
  int* piv = reinterpret_cast<int*>(sh + 32);
  int* perm = piv + D;
  for (int e = threadIdx.x; e < q3 * q3; e += NT) {
    G[e] = r.G[e];
    Gl[e] = r.G[RM2 * RM2 + e];
  }
  for (int e = threadIdx.x; e < n3 * R2; e += NT) lastT[e] = r.LT[e];
  for (int e = threadIdx.x; e < R2; e += NT) tau[e] = r.tau[e];
  __syncthreads();
  const double budget2 = r.sc[0], cthresh = r.sc[1];
  const SvdWork sw{p.prof, Xs, vn, sig, sraw, piv, perm, sh, D};
  const int k2 = chol_piv_dd_warp(G, Gl, q3, cthresh, Rc, D, piv);
  __syncthreads();
  double mg2 = 0.0;
  const int t2 = svd_from_r_warp(Rc, D, k2, q3, piv, sw, budget2, p.cap, W2, D3, &mg2);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (p.margins) p.margins[2 * o + 1] = mg2;
    const long long sz = (long long)n1 * t1 + (long long)n2 * t1 * t2 + (long long)t2 * n3;
    const unsigned long long at = atomicAdd(p.out.used, (unsigned long long)sz);
    const bool ok = (long long)(at + sz) <= p.out.capacity;
    if (!ok) atomicExch(&p.status[kStOverflow], 1);
    p.out.ranks[2 * o] = t1;
    p.out.ranks[2 * o + 1] = t2;
    p.out.off[o] = ok ? (long long)at : -1;
    if (t1 > *(volatile int*)&p.status[kStMaxR1]) atomicMax(&p.status[kStMaxR1], t1);
    if (t2 > *(volatile int*)&p.status[kStMaxR2]) atomicMax(&p.status[kStMaxR2], t2);
    if (p.acc) {
      double* slotp = p.acc + 2 * (blockIdx.x % kAccSlots);
      atomicAdd(&slotp[0], round_flops((double)n2, (double)R1, (double)R2, (double)t1, (double)t2));
      atomicAdd(&slotp[1], 8.0 * (r.sc[2] + (double)sz));
    }
    r.iv[1] = t2;
    r.iv[2] = ok ? 0 : 1;
    r.off[0] = ok ? (long long)at : -1;
  }
  __syncthreads();
  const long long at = r.off[0];
  if (at < 0) return;
  double* dst = p.out.base + at;
  double* dlast = dst + (long long)n1 * t1 + (long long)n2 * t1 * t2;
  for (int e = threadIdx.x; e < n1 * t1; e += NT) dst[e] = r.U1[e];
  // G = [W2; 0] (n3 x t2); Z = R3^T W2 (R2 x t2, ld RM2) into the record
  for2d(n3, t2, [&](int c, int s) { Xq[c + n3 * s] = c < q3 ? W2[c + D3 * s] : 0.0; });
  for2d(R2, t2, [&](int b, int s) {
    double acc = 0.0;
    const int cm = min(b, q3 - 1);
    for (int c = 0; c <= cm; ++c) acc += lastT[c + n3 * b] * W2[c + D3 * s];
    r.Z[b + RM2 * s] = acc;
  });
  __syncthreads();
  const int kmax = min(n3, R2);
  {  // the warp applies Q3 = H_0 ... H_{kmax-1} to each column of G, lanes over rows
    const int lane = threadIdx.x & 31;
    int s = 0;
    for (; TTDVM_PIPE_QR_ROWS && s + 1 < t2; s += 2) {  // two columns in flight (same sums per column)
      double* g = Xq + n3 * s;
      double* h = g + n3;
      for (int k = kmax - 1; k >= 0; --k) {
        const double t = tau[k];
        if (t == 0.0) continue;
        const double* v = lastT + n3 * k;
        double w = 0.0, x = 0.0;
        for (int i = k + 1 + lane; i < n3; i += 32) {
          w += v[i] * g[i];
          x += v[i] * h[i];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          w += __shfl_xor_sync(0xffffffffu, w, o);
          x += __shfl_xor_sync(0xffffffffu, x, o);
        }
        w = t * (w + g[k]);
        x = t * (x + h[k]);
        __syncwarp();
        if (lane == 0) {
          g[k] -= w;
          h[k] -= x;
        }
        for (int i = k + 1 + lane; i < n3; i += 32) {
          g[i] -= w * v[i];
          h[i] -= x * v[i];
        }
        __syncwarp();
      }
    }
    for (; s < t2; ++s) {
      double* g = Xq + n3 * s;
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
  for2d(t2, n3, [&](int s, int kk) { dlast[s + t2 * kk] = Xq[kk + n3 * s]; });
}

// ---- P6 ---------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 24) pipe_middle_kernel(PipeArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) int s_meta[10];
  const int slot = blockIdx.x;
  if (slot >= a.count) return;
  const RoundArgs& p = a.p;
  PipeRec r = pipe_rec(a, slot);
  if (r.iv[2]) return;
  const int o = pipe_output(a, slot);
  const int n1 = p.n1, n2 = p.n2, RM1 = p.RM1, RM2 = p.RM2, JB = a.JB;
  const int D1 = RM1;
  const int t1 = r.iv[0], t2 = r.iv[1];
  double* XP = sm;                        // t1 x R1, ld D1
  double* Z = XP + D1 * RM1;              // R2 x t2, ld RM2
  double* X2 = Z + RM2 * RM2;             // JB x t1 x R2
  double* Ms = X2 + JB * D1 * RM2;        // JB x MSMAX
  PipeTerms pt = pipe_terms(Ms + JB * p.MSMAX, RM1, RM2);
  double* dmid = p.out.base + r.off[0] + (long long)n1 * t1;
  for (int e = threadIdx.x; e < RM2 * t2; e += NT) Z[e] = r.Z[e];
  if (t1 <= a.tkeep) {
    // X2_j = P M_j of every slice was kept by P4: one product, no staging
    const int R2k = r.iv[4];
    const double* xg = r.X2;
    __syncthreads();
    for2d(t1, n2 * t2, [&](int rr, int js) {
      const int jj = js / t2, s = js - jj * t2;
      const double* x = xg + (long long)jj * t1 * R2k + rr;
      const double* z = Z + RM2 * s;
      double a0 = 0.0, a1 = 0.0;
      int b = 0;
      for (; b + 1 < R2k; b += 2) {
        a0 += x[t1 * b] * z[b];
        a1 += x[t1 * (b + 1)] * z[b + 1];
      }
      if (b < R2k) a0 += x[t1 * b] * z[b];
      dmid[(long long)jj * t1 * t2 + rr + t1 * s] = a0 + a1;
    });
    return;
  }
  int K, R1, R2;
  setup_terms(p, o, pt.terms, pt.rowterm, pt.colterm, s_meta, K, R1, R2, nullptr, 0, nullptr,
              !a.keepms);
  for (int e = threadIdx.x; e < D1 * R1; e += NT) XP[e] = r.P[e];
  for (int j0 = 0; j0 < n2; j0 += JB) {
    const int jn = min(JB, n2 - j0);
    __syncthreads();
    if (a.keepms) {
      const double* mg = r.Ms + (long long)j0 * p.MSMAX;
      for (int e = threadIdx.x; e < jn * p.MSMAX; e += NT) Ms[e] = mg[e];
    } else {
      stage_slices(Ms, p.MSMAX, pt.terms, K, n1, n2, j0, jn);
    }
    __syncthreads();
    left_times_blockdiag_b(X2, t1, t1 * R2, XP, D1, t1, R2, Ms, p.MSMAX, pt.terms, pt.colterm, jn);
    __syncthreads();
    for2d(t1, jn * t2, [&](int rr, int js) {
      const int jj = js / t2, s = js - jj * t2;
      const double* x = X2 + jj * t1 * R2 + rr;
      const double* z = Z + RM2 * s;
      double a0 = 0.0, a1 = 0.0;
      int b = 0;
      for (; b + 1 < R2; b += 2) {
        a0 += x[t1 * b] * z[b];
        a1 += x[t1 * (b + 1)] * z[b + 1];
      }
      if (b < R2) a0 += x[t1 * b] * z[b];
      dmid[(long long)(j0 + jj) * t1 * t2 + rr + t1 * s] = a0 + a1;
    });
  }
}

// ---- host side ----------------------------------------------------------------
// Record layout and shared-memory sizes for a bin (RM1, RM2 <= kWarpMaxD).
static void pipe_layout(PipeArgs& a) {
  const RoundArgs& p = a.p;
  const int RM1 = p.RM1, RM2 = p.RM2, D = RM1 > RM2 ? RM1 : RM2;
  auto even = [](long long v) { return (v + 1) & ~1LL; };
  long long o = 0;
  a.oF = (int)o;
  o += even((long long)p.n1 * RM1);
  a.oLT = (int)o;
  o += even((long long)p.n3 * RM2);
  a.oTau = (int)o;
  o += even(RM2);
  a.oG = (int)o;
  o += 2LL * D * D;
  a.oU1 = (int)o;
  o += even((long long)p.n1 * RM1);
  a.oP = (int)o;
  o += even((long long)RM1 * RM1);
  a.oZ = (int)o;
  o += even((long long)RM2 * RM2);
  a.oS = (int)o;
  o += 12;
  a.oX2 = (int)o;
  static const int tkeep_env = [] {  // TTDVM_PIPE_TKEEP=0: always restage in P6 (A/B)
    const char* e = getenv("TTDVM_PIPE_TKEEP");
    return e ? atoi(e) : 2;
  }();
  a.tkeep = std::min(tkeep_env, RM1);
  o += even((long long)p.n2 * a.tkeep * RM2);
  static const int keepms_env = [] {  // TTDVM_PIPE_KEEPMS=0: P4 / P6 restage from the operands (A/B)
    const char* e = getenv("TTDVM_PIPE_KEEPMS");
    return e ? atoi(e) : 1;
  }();
  a.keepms = keepms_env;
  a.oMs = (int)o;
  if (a.keepms) o += even((long long)p.n2 * p.MSMAX);
  a.stride = (o + 15) / 16 * 16;
}

long long round_pipe_record_doubles(const RoundArgs& p) {
  PipeArgs a;
  a.p = p;
  pipe_layout(a);
  return a.stride;
}

bool round_pipe_eligible(const RoundArgs& p) {
  const int D = (p.RM1 > p.RM2 ? p.RM1 : p.RM2);
  return p.RM1 < p.n1 && p.RM2 <= p.n3 && D <= kWarpMaxD && p.n1 <= 64 && p.n3 <= 64;
}

// Round outputs [first, first + count) of the launch (entries of p.olist)
// through the six phase kernels; `rec` holds count records.
cudaError_t launch_round_pipe(const RoundArgs& p, int first, int count, double* rec,
                              cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  PipeArgs a;
  a.p = p;
  a.rec = rec;
  a.first = first;
  a.count = count;
  pipe_layout(a);
  const int n1 = p.n1, n3 = p.n3, RM1 = p.RM1, RM2 = p.RM2, D = RM1 > RM2 ? RM1 : RM2;
  // slices per stage: about 512 doubles of Z_j per batch (TTDVM_PIPE_JB overrides, A/B)
  static const int jb_env = [] {
    const char* e = getenv("TTDVM_PIPE_JB");
    return e ? atoi(e) : 0;
  }();
  a.JB = std::max(1, std::min(p.n2, jb_env > 0 ? jb_env : 512 / std::max(1, RM1 * RM2)));
  // TTDVM_PIPE_IL=1: the lane's Gram entries interleaved in one column loop
  // (measured neutral at Q = 3, 6 % slower at Q = 5: off by default)
  static const int il_env = [] {
    const char* e = getenv("TTDVM_PIPE_IL");
    return e ? atoi(e) : 0;
  }();
  a.il = il_env;
  static const int zt_env = [] {  // TTDVM_PIPE_ZT=0: P2 with pipe_zj + gram_rows_acc (A/B)
    const char* e = getenv("TTDVM_PIPE_ZT");
    return e ? atoi(e) : 1;
  }();
  a.zt = zt_env;
  const size_t tb = pipe_terms_bytes(RM1, RM2);
  const size_t small = (size_t)(5 * D * D + 3 * D + 32) * 8 + (size_t)2 * D * 4 + 16;
  const size_t s1 = (size_t)(n1 * RM1 + n3 * RM2 + n3 + 32) * 8 + tb;
  const size_t s2 =
      (size_t)(((RM2 * (RM2 + 4) + 1) & ~1) + RM1 * pipe_ldz(a.JB, RM2) + a.JB * p.MSMAX) * 8 + tb;
  const size_t s3 = (size_t)(2 * n1 * RM1) * 8 + small;
  const size_t s4 = (size_t)(RM2 * RM2 + RM1 * RM1 + 2 * a.JB * RM1 * RM2 + a.JB * p.MSMAX) * 8 + tb;
  const size_t s5 = (size_t)(2 * n3 * RM2 + n3) * 8 + small;
  const size_t s6 = (size_t)(RM1 * RM1 + RM2 * RM2 + a.JB * RM1 * RM2 + a.JB * p.MSMAX) * 8 + tb;
  const int ne = D * (D + 1) / 2;
  cudaError_t e;
#define PIPE_ATTR(kern, bytes)                                                                  \
  if ((bytes) > 48 * 1024) {                                                                    \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes));  \
    if (e != cudaSuccess) return e;                                                             \
  }
#define PIPE_Q(kern, bytes)                                  \
  if (ne <= NT) {                                            \
    PIPE_ATTR(kern<1>, bytes)                                \
    kern<1><<<count, NT, bytes, st>>>(a);                    \
  } else if (ne <= 3 * NT) {                                 \
    PIPE_ATTR(kern<3>, bytes)                                \
    kern<3><<<count, NT, bytes, st>>>(a);                    \
  } else {                                                   \
    PIPE_ATTR(kern<5>, bytes)                                \
    kern<5><<<count, NT, bytes, st>>>(a);                    \
  }
  PIPE_ATTR(pipe_prep_kernel, s1)
  pipe_prep_kernel<<<count, NT, s1, st>>>(a);
  PIPE_Q(pipe_gram1_kernel, s2)
  PIPE_Q(pipe_factor1_kernel, s3)
  PIPE_Q(pipe_gram2_kernel, s4)
  PIPE_ATTR(pipe_factor2_kernel, s5)
  pipe_factor2_kernel<<<count, NT, s5, st>>>(a);
  PIPE_ATTR(pipe_middle_kernel, s6)
  pipe_middle_kernel<<<count, NT, s6, st>>>(a);
#undef PIPE_Q
#undef PIPE_ATTR
  return cudaGetLastError();
}

#endif  // TTDVM_ROUND_NT == 32
