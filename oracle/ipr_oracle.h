/*
 * ipr_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the Bini et al. inverse p-th root
 * iteration studied in arXiv:1703.02283 ("approximate computing for inverse matrix
 * p-th roots").  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this.  It shares NO code, header, table or constant
 * generator with the CUDA path under paper_1703_02283_b200/ (which must never load it).
 *
 * Citations are PAPER.md line numbers (section / equation in brackets):
 *   Eq. (1)  PAPER.md:71-73  [Sec. 2]   C_{k+1} = ((p+1) C_k - C_k^{p+1} A) / p
 *   Eq. (2)  PAPER.md:76-78  [Sec. 2]   ||I - C_0^p A||_2 < 1  => convergence
 *   Eq. (3)  PAPER.md:84-86  [Sec. 2]   C_0 = (||A||_1 ||A||_inf)^{-1} A^T
 *   approximate arithmetic / storage: PAPER.md:101-145 [Sec. 3], :149-155 [Sec. 4]
 *   dynamic precision scaling: PAPER.md:256-261 [Sec. 4.3.1]
 * Readings of silent/ambiguous passages (R-1 ... R-21) are listed in DESIGN.md.
 *
 * Parity status: every function below is pinned by tests in tests/test_oracle_*.py
 * against closed forms, library routines or hand values, EXCEPT the paper's own
 * curves (Figs. 2-5 are missing from PAPER.md): "parity unpinned" for those (R-21).
 */
#ifndef IPR_ORACLE_H
#define IPR_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Operand (GEMM input) formats.  Values are independent of include/ipr.h on purpose. */
/* ORC_FP64_OZ (= 6): an FP64 phase whose GPU GEMMs are emulated on INT8 tensor cores (Ozaki scheme,
 * reading R-23).  The oracle computes it exactly like ORC_FP64: the emulation is an FP64-accurate
 * GEMM, so the two sides differ by FP64-level rounding only (Level 2 tolerance, not bit-exact). */
/* ORC_FP64_CRT (= 7): an FP64 phase whose GPU GEMMs run on INT8 tensor cores by the Chinese remainder
 * theorem (Ozaki scheme II, reading R-28).  Unlike FP64_OZ its products are NOT FP64-accurate by design:
 * each row of the left operand / column of the right one is quantised to b-bit integers relative to its
 * maximum.  The oracle computes that definition exactly (orc_gemm_crt: exact integer product, one
 * rounding), so the GPU's CRT phases have a true reference. */
enum { ORC_FP64 = 0, ORC_TF32 = 1, ORC_BF16 = 2, ORC_FP16 = 3, ORC_FP8 = 4, ORC_INT8 = 5, ORC_FP64_OZ = 6,
       ORC_FP64_CRT = 7 };
enum { ORC_RNE = 0, ORC_RTZ = 1 };
enum { ORC_CONTINUE = 0, ORC_CONVERGED = 1, ORC_ITER_LIMIT = 2, ORC_DIVERGED = 3,
       ORC_NONFINITE = 4, ORC_SWITCH = 5 };

/* q_m: round x to a binary format with E exponent bits and m stored mantissa bits,
 * subnormals kept, overflow -> +-Inf (RNE) or +-max finite (RTZ), NaN -> NaN,
 * -0 kept.  Definition written out with frexp/ldexp (no bit tricks). */
double orc_qm(double x, int E, int m, int rtz);
void   orc_qm_array(int64_t len, const double *x, double *y, int E, int m, int rtz);

/* Operand format of a precision: (E, M).  Container exponent bits of a phase. */
void orc_prec_format(int prec, int *E, int *M);
int  orc_container_E(int prec);
int  orc_native_m(int prec);

/* Norms of Eq. (3): out[0] = ||A||_1 (max column abs-sum), out[1] = ||A||_inf (max row
 * abs-sum), out[2] = max diagonal.  Sums sequential in ascending index. */
void orc_norms(int64_t n, const double *A, double *out3);

/* 1 if A == A^T bit for bit, else 0. */
int orc_is_symmetric(int64_t n, const double *A);

/* Z = X * Y (all n x n row-major), i-k-j loops, FP64 accumulator, no FMA. */
void orc_gemm(int64_t n, const double *X, const double *Y, double *Z);
/* Columns [c0, c1) of Z = X Y, same per-element k order (column-panel decomposition tests). */
void orc_gemm_cols(int64_t n, int64_t c0, int64_t c1, const double *X, const double *Y, double *Z);
/* Rows [r0, r1) of Z = X Y, same loops (bounded timing sample for the CPU baseline). */
void orc_gemm_rows(int64_t n, int64_t r0, int64_t r1, const double *X, const double *Y, double *Z);
/* y = X v (row-major), sequential sums. */
void orc_matvec(int64_t n, const double *X, const double *v, double *y);

typedef struct {
  int    prec;          /* ORC_FP64 / TF32 / BF16 / FP16                              */
  int    mant_bits;     /* m stored bits of C (and A) in this phase; -1 = native      */
  int    round;         /* ORC_RNE / ORC_RTZ for stored C (and A)                     */
  double switch_tol;    /* leave phase when rho <= switch_tol; 0 = off                */
  double plateau_ratio; /* armed plateau: rho_k > ratio * rho_{k-1}; 0 = off          */
  double plateau_arm;   /* armed when rho_hat_k < plateau_arm                          */
  int    max_iters;     /* per-phase cap on chains; 0 = unlimited                     */
  int    corr_prec;     /* ORC_FORM_SYMMETRIC: operand format of the correction GEMM  */
                        /* W = qc(C) Rhat; -1 = prec.  Ignored by the other forms.    */
} orc_phase;

typedef struct {
  int k, phase, prec, mant_bits, decision;
  double rho, rho_hat, delta, gamma;
  double rho_cert;     /* ORC_FORM_SYMMETRIC: certified ||I - C^p A||_F (FP64) when the */
                       /* in-chain rho_s met final_tol; NaN otherwise                   */
} orc_record;

/* Controller (reading R-5 of DESIGN.md).  Pure state machine, no matrices. */
typedef struct {
  int phase, nphases, it_in_phase;
  int64_t n;
  double rho_prev, rho_best, rhohat_min, final_tol;
  int best_is_new;                     /* out: 1 if this rho became the new best */
} orc_ctrl;
void orc_ctrl_init(orc_ctrl *c, int64_t n, int nphases, double final_tol);
int  orc_ctrl_decide(orc_ctrl *c, const orc_phase *ph, double rho);
void orc_ctrl_enter_next_phase(orc_ctrl *c);

/* Scalars of the phase-0 initial guess: C0 = q_m0(A^T / s), s = ||A||_1 ||A||_inf. */
void orc_c0(int64_t n, const double *A, double s, const orc_phase *ph0, double *C0);

/* One full Bini iteration from C_k at phase ph (R-1 right-to-left chain):
 *   Chat = qin(C), Ahat = qin(q_m(A)), T_1 = Chat Ahat, T_j = Chat qin(T_{j-1}),
 *   rho = ||I - T_p||_F (unrounded T_p), P = Chat qin(T_p),
 *   C_next = q_m(((p+1) C - P) / p)  (three FP64 ops, one rounding; R-2).
 * C_next may be NULL (chain + residual only).  Returns rho; *delta = ||C_next - C||_F. */
double orc_step(int64_t n, int p, const double *A, const double *C, const orc_phase *ph,
                double *C_next, double *delta);

/* Full solve: init (norms, C0) + controller-driven iterations.
 *   rec[cap_rec] trace; C_best (n*n) answer; C_hist (hist_cap * n*n, may be NULL) keeps
 *   the iterate evaluated by each record (C_k of record k);
 *   gamma_normA2 > 0 => record gamma_k = ||C A - A C||_F / (||C||_F gamma_normA2).
 * Returns outcome (ORC_CONVERGED, ...); *nrec = records written. */
int orc_solve(int64_t n, int p, const double *A, const orc_phase *phases, int nphases,
              double final_tol, int max_total, orc_record *rec, int cap_rec, int *nrec,
              double *C_best, double *C_hist, int hist_cap, double gamma_normA2,
              double *s_out);

/* Iteration forms: ORC_FORM_LITERAL = Eq. (1) as printed (right-to-left chain, reading R-1);
 * ORC_FORM_NEWTON_SCHULZ = p = 1 only, X_{k+1} = X_k (2I - A X_k) (NEXT-1). */
/* ORC_FORM_SYMMETRIC_TRI (p = 2): as ORC_FORM_SYMMETRIC with Z_2 = C A C replaced by the mirror
 * of its upper triangle (Z_2[i][j] := Z_2[min(i,j)][max(i,j)]), so R is exactly symmetric. */
/* ORC_FORM_COUPLED (NEXT-2 (ii)): X_{k+1} = X_k N_k, M_{k+1} = N_k^p M_k, N = ((p+1)I - M)/p, M
 * re-anchored as X^p A at every phase start; rho = ||I - M_k||_F; convergence certified on
 * ||I - X^p A||_F like the symmetric forms.  No scaled formats. */
/* ORC_FORM_SYMMETRIC_TRIZ (reading R-37, p = 2): ORC_FORM_SYMMETRIC_TRI, and in an FP64_CRT phase Z_1 = Ahat Chat
 * is taken from its upper triangle too from the third chain of the phase on, while every in-phase ratio
 * rho_k / rho_{k-1} so far was <= 0.1 (sticky off).  orc_step_sym_form: tri = 2 is that chain. */
enum { ORC_FORM_LITERAL = 0, ORC_FORM_NEWTON_SCHULZ = 1, ORC_FORM_SYMMETRIC = 2,
       ORC_FORM_SYMMETRIC_TRI = 3, ORC_FORM_COUPLED = 4, ORC_FORM_SYMMETRIC_TRIZ = 5 };
/* Reading R-33: certificate-first iterates in the last phase of the symmetric forms (default on). */
void orc_set_predict_cert(int on);
int orc_solve_form(int64_t n, int p, int form, const double *A, const orc_phase *phases,
                   int nphases, double final_tol, int max_total, orc_record *rec, int cap_rec,
                   int *nrec, double *C_best, double *C_hist, int hist_cap, double gamma_normA2,
                   double *s_out);
/* One Newton-Schulz step from X: returns rho(X) = ||I - Ahat Xhat||_F; X_next may be NULL. */
double orc_step_ns(int64_t n, const double *A, const double *X, const orc_phase *ph,
                   double *X_next, double *delta);

/* One symmetrised-correction step (NEXT-2, p >= 2, no FP16): returns rho_s(C) =
 * ||I - C^{p-1} A C||_F (in-chain); C_next = q_m(C + (W + W^T)/(2p)), W = qc(C) qc(I - Z_p).
 * Returns NaN for p < 2 or an FP16 phase. */
double orc_step_sym(int64_t n, int p, const double *A, const double *C, const orc_phase *ph,
                    double *C_next, double *delta);
/* The same step for a form: tri = 0 ORC_FORM_SYMMETRIC, 1 ORC_FORM_SYMMETRIC_TRI (p = 2; Z_2 from its upper
 * triangle and -- reading R-36, in phases below the FP64 range -- the correction from W's upper triangle:
 * C_{k+1} = q_m(C + 2 W_{min(i,j),max(i,j)} / (2p))). */
double orc_step_sym_form(int64_t n, int p, int tri, const double *A, const double *C, const orc_phase *ph,
                         double *C_next, double *delta);

/* Cyclic Jacobi eigen-decomposition of a symmetric matrix (n small).
 * lambda ascending, V columns = eigenvectors (row-major n x n).  Returns sweeps used. */
int orc_jacobi(int64_t n, const double *A, double *lambda, double *V);
/* X = V diag(lambda^{-1/p}) V^T. */
void orc_inv_proot_eig(int64_t n, const double *lambda, const double *V, int p, double *X);

/* Spectral predictor: rho_hat_k (k = 0..kmax-1) of the exact-arithmetic iteration from
 * the eigenvalues lambda of A and s: t_0 = lambda^{p+1}/s^p, t <- t ((p+1-t)/p)^p. */
void orc_spectral(int64_t n, const double *lambda, int p, double s, int kmax, double *rho_hat);

/* FP16 phase operand scale exponent: sigma = 14 - floor(log2(max|X|)) (0 if max is 0
 * or non-finite).  Stored FP16 operand = q16(2^sigma X). */
int orc_fp16_sigma(double maxabs);
/* Scale exponent of the scaled operand formats: FP16 (as above), FP8 E4M3 and INT8 (scaled max
 * in [2^6, 2^7)); 0 otherwise.  INT8 quantiser: nearest-even integer saturated to +-127. */
int orc_sigma(int prec, double maxabs);

/* Dynamic precision inside an FP64_OZ phase (reading R-26): mant_bits = ORC_MANT_ADAPTIVE picks
 * the Ozaki digit count per iteration from the expected residual and stores C with
 * orc_oz_adaptive_m(S) = min(52, 7 S - 4) bits. */
enum { ORC_MANT_ADAPTIVE = -2 };
int orc_oz_digits(double rho_hat_target, int64_t n);
int orc_oz_adaptive_m(int S);
/* Digits S of a fixed-m FP64_OZ / FP64_CRT phase: S = clamp(ceil((m + 12) / 7), 2, 9) (reading R-23). */
int orc_digits_for_m(int m);
/* Bits b of an FP64_CRT product with S Ozaki-equivalent digits at order n (reading R-28):
 * b = min(7 S - 4, 62), lowered while 2 b + log2 n + 1.02 >= log2 of the product of the 18 moduli
 * (the exact integer product must stay below M / 2^1.02 for its reconstruction to be unique). */
int orc_crt_bits(int S, int64_t n);
/* Z = X (x)_b Y (n x n row-major): the CRT product's definition (reading R-28).
 *   Xbar_ik = rint(2^{e_i} x_ik), e_i = b - 1 - floor(log2 max_k |x_ik|)  (0 for a zero row)
 *   Ybar_kj = rint(2^{f_j} y_kj), f_j = b - 1 - floor(log2 max_k |y_kj|)  (0 for a zero column)
 *   Z_ij    = RN( 2^{-(e_i + f_j)} sum_k Xbar_ik Ybar_kj )   -- the integer sum exact, ONE rounding.
 * rint = round half to even.  1 <= b <= 62. */
void orc_gemm_crt(int64_t n, int b, const double *X, const double *Y, double *Z);
/* Selected elements of the same product: Z[q] = (X (x)_b Y)[I[q]][J[q]], q < npairs (the exponents from
 * the FULL row I[q] of X and column J[q] of Y) -- sampled outputs of full-size products. */
void orc_gemm_crt_pairs(int64_t n, int b, const double *X, const double *Y, int64_t npairs, const int64_t *I,
                        const int64_t *J, double *Z);
double orc_q_int8(double x);

/* The CRT certificate of the symmetric forms (reading R-35; not in the paper: it makes the
 * north star's "residual <= 1e-12" a proven statement about the returned matrix).
 * orc_cert_grid: the certified matrix Ct of a candidate C (n x n row-major): with the row exponents
 *   e_i = b - 1 - floor(log2 max_k |c_ik|) of orc_gemm_crt (0 for a zero row),
 *   Ct_ij = 2^{-g} rint(2^{g} c_ij),  g = min(e_i, e_j)   (rint = half to even)
 * i.e. C rounded to the coarser of its row's and its column's b-bit grids -- so 2^{e_i} Ct_ij is an
 * integer for every i, j and the row AND column quantisation of Ct to b bits is exact.  A symmetric C
 * gives a symmetric Ct; |Ct_ij - c_ij| <= 2^{-g-1}; elements within 2^{b-53} of both maxima are kept.
 * orc_resid_dd: ||I - X^p A||_F evaluated in double-double arithmetic (the right-to-left chain
 *   T_1 = X A, T_j = X T_{j-1}, every product accumulated in double-double, R = I - T_p in
 *   double-double): ~2^-100 relative per product, i.e. the exact residual of the FP64 matrices X, A
 *   for every digit that matters (an FP64 evaluation carries ~n u |X||A| of rounding noise).
 * orc_set_cert_mode: how orc_solve_form's symmetric forms certify (R-30): 0 = FP64 literal chain
 *   (default); 1 = CRT (R-35): the candidate's Ct = orc_cert_grid(C, 62) is certified by
 *   orc_resid_dd(Ct) and, when certified, Ct is the answer. */
void orc_cert_grid(int64_t n, int b, const double *C, double *Ct);
double orc_resid_dd(int64_t n, int p, const double *A, const double *X);
void orc_set_cert_mode(int mode);
/* Rows of the same residual: out[q] = sum_j (I - X^p A)[rows[q]][j]^2 in double-double arithmetic
 * (row i of X^p A = ((x_i^T X) ... X) A, every vector-matrix product accumulated in double-double) --
 * sampled rows of full-size residuals. */
void orc_resid_rows_dd(int64_t n, int p, const double *A, const double *X, int64_t nrows, const int64_t *rows,
                       double *out);

#ifdef __cplusplus
}
#endif
#endif
