/*
 * ipr_oracle.c -- TEST INFRASTRUCTURE ONLY (see ipr_oracle.h).
 *
 * Plain FP64 CPU oracle for the Bini inverse p-th root iteration of arXiv:1703.02283.
 * Compiled with -ffp-contract=off (no FMA contraction) so every line below is the
 * IEEE operation it reads as.  No BLAS, no bit tricks: rounding is written with
 * frexp/ldexp/nearbyint, products are i-k-j triple loops with an FP64 accumulator.
 * Nothing here is shared with, or loaded by, the CUDA path.
 */
#include "ipr_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------
 * q_m -- approximate storage / arithmetic as custom-precision rounding.
 * PAPER.md:191-194 [Sec. 4.2] "floating-point types with a custom number of bits in the
 * exponent and mantissa"; PAPER.md:106-111 footnotes give the (exponent, stored mantissa)
 * splits of half (5,10), single (8,23), double (11,52).
 * Reading R-7: round-to-nearest-even by default, RTZ ("bit truncation")
 * selectable.  Reading R-8: subnormals kept.  Overflow: RNE -> Inf, RTZ -> max finite.
 * Definition: with e = max(floor(log2|x|), emin) the representable neighbours of x are
 * the integer multiples of ulp = 2^(e-m); x/ulp and q*ulp are exact power-of-two
 * scalings, nearbyint() rounds half-to-even in the default rounding mode.
 * ------------------------------------------------------------------------------ */
double orc_qm(double x, int E, int m, int rtz) {
  if (isnan(x) || isinf(x) || x == 0.0) return x;
  const int bias = (1 << (E - 1)) - 1;
  const int emin = 1 - bias, emax = bias;
  int ex;
  frexp(fabs(x), &ex);            /* |x| = f 2^ex, f in [0.5, 1)  =>  floor(log2|x|) = ex-1 */
  int e = ex - 1;
  if (e < emin) e = emin;         /* subnormal range: fixed spacing 2^(emin-m) */
  const double ulp = ldexp(1.0, e - m);
  const double r = x / ulp;
  const double q = rtz ? trunc(r) : nearbyint(r);
  double y = q * ulp;
  const double maxf = ldexp(2.0 - ldexp(1.0, -m), emax);
  if (fabs(y) > maxf) y = rtz ? copysign(maxf, x) : copysign(INFINITY, x);
  return y;
}

void orc_qm_array(int64_t len, const double *x, double *y, int E, int m, int rtz) {
  for (int64_t i = 0; i < len; ++i) y[i] = orc_qm(x[i], E, m, rtz);
}

/* Operand formats (R-9, R-10): BF16 = e8m7, FP16 = e5m10 (PAPER.md:106-107 footnote),
 * FP8 = e4m3 (NEXT-3; scaled so |values| < 2^7: the IEEE-like e4m3 grid and the hardware's
 * E4M3 "fn" grid coincide there), INT8 = 8-bit two's-complement fixed point (NEXT-3, the
 * fixed-point analogue of PAPER.md:268-281; M = 7 magnitude bits, no exponent field),
 * TF32 = e8m10, FP64 = e11m52 (PAPER.md:110-111 footnote). */
void orc_prec_format(int prec, int *E, int *M) {
  switch (prec) {
    case ORC_TF32: *E = 8;  *M = 10; break;
    case ORC_BF16: *E = 8;  *M = 7;  break;
    case ORC_FP16: *E = 5;  *M = 10; break;
    case ORC_FP8:  *E = 4;  *M = 3;  break;
    case ORC_INT8: *E = 0;  *M = 7;  break;
    default:       *E = 11; *M = 52; break;
  }
}
/* Reading R-8: container of a phase = its accumulate format: e8 (FP32) for the
 * BF16/FP16/TF32 phases, e11 (FP64) for FP64 phases. */
static int is_f64p(int prec) { return prec == ORC_FP64 || prec == ORC_FP64_OZ || prec == ORC_FP64_CRT; }
int orc_container_E(int prec) { return is_f64p(prec) ? 11 : 8; }
int orc_native_m(int prec) { int E, M; orc_prec_format(prec, &E, &M); return M; }

static int phase_m(const orc_phase *ph) {
  return ph->mant_bits < 0 ? orc_native_m(ph->prec) : ph->mant_bits;
}

/* ---------------------------------------------------------------------------------
 * Dynamic precision inside an FP64_OZ phase (mant_bits = ORC_MANT_ADAPTIVE; reading R-26).
 * PAPER.md:256-261 [Sec. 4.3.1]: "the necessity of increased precision can be detected at
 * runtime".  Before the chain of C_k the GPU picks its Ozaki digit count S_k from the residual it
 * expects for C_{k+1}, rho_hat_{k-1} q^2 (q = the last in-phase contraction ratio, clamped to
 * [1e-3, 1], 0.03 without history): S = clamp(ceil((log2(30 sqrt n) - log2 target) / 7), 3, 9);
 * C_{k+1} is then stored with m = min(52, 7 S - 4) bits.  The oracle's arithmetic stays FP64, so
 * only that storage rule is mirrored here.
 * ------------------------------------------------------------------------------ */
int orc_oz_digits(double rho_hat_target, int64_t n) {
  if (!(rho_hat_target > 0.0) || !isfinite(rho_hat_target)) return 9;
  const double b = log2(30.0 * sqrt((double)n)) - log2(rho_hat_target);
  int S = (int)ceil(b / 7.0);
  if (S < 3) S = 3;
  if (S > 9) S = 9;
  return S;
}
int orc_oz_adaptive_m(int S) { return 7 * S - 4 < 52 ? 7 * S - 4 : 52; }
static int is_adaptive(const orc_phase *ph) {
  return (ph->prec == ORC_FP64_OZ || ph->prec == ORC_FP64_CRT) && ph->mant_bits == ORC_MANT_ADAPTIVE;
}
int orc_digits_for_m(int m) {
  int S = (m + 12 + 6) / 7;               /* ceil((m + 12) / 7) for m >= 0 */
  return S < 2 ? 2 : S > 9 ? 9 : S;
}

/* ---------------------------------------------------------------------------------
 * FP64-range products by the Chinese remainder theorem (Ozaki scheme II; reading R-28 --
 * not in the paper; its "custom number of mantissa bits", PAPER.md:191-194 [Sec. 4.2], applied to
 * the operands of an integer product).  What the GPU emulation computes is, by definition, the EXACT
 * product of the b-bit integer quantisations of the operands' rows (left) and columns (right),
 * rescaled and rounded once; the moduli, residues and CRT reconstruction are only the GPU's way of
 * forming that integer product, so none of them appears here except the moduli's product, which caps b.
 * ------------------------------------------------------------------------------ */
static const int crt_moduli_def[18] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217,
                                       211, 199, 197, 193, 191, 181};   /* DESIGN.md R-28 */
int orc_crt_bits(int S, int64_t n) {
  double log2M = 0.0;
  for (int l = 0; l < 18; ++l) log2M += log2((double)crt_moduli_def[l]);
  int b = 7 * S - 4 < 62 ? 7 * S - 4 : 62;
  while (b > 2 && !(2.0 * b + log2((double)(n < 1 ? 1 : n)) + 1.02 < log2M)) --b;
  return b;
}

/* exponent that puts max|x| into [2^(b-1), 2^b): b - 1 - floor(log2 max|x|) */
static int crt_exp(double mx, int b) {
  if (!(mx > 0.0)) return 0;
  int ex;
  frexp(mx, &ex);                          /* mx = f 2^ex, f in [0.5, 1): floor(log2 mx) = ex - 1 */
  return b - 1 - (ex - 1);
}

/* unsigned 192-bit magnitude, little-endian 64-bit words */
typedef struct { uint64_t w[3]; } u192;
static void u192_add(u192 *a, unsigned __int128 v) {
  unsigned __int128 s = (unsigned __int128)a->w[0] + (uint64_t)v;
  a->w[0] = (uint64_t)s;
  s = (unsigned __int128)a->w[1] + (uint64_t)(v >> 64) + (uint64_t)(s >> 64);
  a->w[1] = (uint64_t)s;
  a->w[2] += (uint64_t)(s >> 64);
}
static int u192_cmp(const u192 *a, const u192 *b) {
  for (int i = 2; i >= 0; --i) if (a->w[i] != b->w[i]) return a->w[i] > b->w[i] ? 1 : -1;
  return 0;
}
static u192 u192_sub(const u192 *a, const u192 *b) {   /* a - b, a >= b */
  u192 r;
  uint64_t br = 0;
  for (int i = 0; i < 3; ++i) {
    const uint64_t t = a->w[i] - b->w[i] - br;
    br = (a->w[i] < b->w[i] || (a->w[i] == b->w[i] && br)) ? 1 : 0;
    r.w[i] = t;
  }
  return r;
}
static int u192_bit(const u192 *a, int k) { return (int)((a->w[k >> 6] >> (k & 63)) & 1u); }
/* RN(a 2^scale): round the integer a to 53 significant bits (ties to even), then scale by 2^scale
 * (exact for the normal results these products have) */
static double u192_to_double(const u192 *a, int scale) {
  int top = -1;
  for (int k = 191; k >= 0; --k) if (u192_bit(a, k)) { top = k; break; }
  if (top < 0) return 0.0;
  if (top < 53) return ldexp((double)a->w[0], scale);   /* exact: fewer than 54 bits */
  const int sh = top - 52;                              /* keep bits [sh, top] */
  uint64_t mant = 0;
  for (int k = top; k >= sh; --k) mant = (mant << 1) | (uint64_t)u192_bit(a, k);
  const int guard = u192_bit(a, sh - 1);
  int sticky = 0;
  for (int k = sh - 2; k >= 0 && !sticky; --k) sticky = u192_bit(a, k);
  if (guard && (sticky || (mant & 1u))) mant += 1;      /* may carry to 2^53: still exact in FP64 */
  return ldexp((double)mant, sh + scale);
}

/* the exact element (Xbar_i. Ybar_.j) 2^-(e+f), rounded once */
static double crt_elem(int64_t n, const int64_t *xr, int64_t xs, const int64_t *yc, int64_t ys, int e, int f) {
  u192 pos = {{0, 0, 0}}, neg = {{0, 0, 0}};
  for (int64_t k = 0; k < n; ++k) {
    const __int128 pr = (__int128)xr[k * xs] * (__int128)yc[k * ys];   /* |pr| <= 2^124 */
    if (pr >= 0) u192_add(&pos, (unsigned __int128)pr);
    else u192_add(&neg, (unsigned __int128)(-pr));
  }
  if (u192_cmp(&pos, &neg) >= 0) { const u192 d = u192_sub(&pos, &neg); return u192_to_double(&d, -(e + f)); }
  const u192 d = u192_sub(&neg, &pos);
  return -u192_to_double(&d, -(e + f));
}

void orc_gemm_crt_pairs(int64_t n, int b, const double *X, const double *Y, int64_t npairs, const int64_t *I,
                        const int64_t *J, double *Z) {
  #pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < npairs; ++q) {
    int64_t *xr = (int64_t *)malloc((size_t)n * sizeof(int64_t)), *yc = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    const int64_t i = I[q], j = J[q];
    double mx = 0.0, my = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      if (fabs(X[i * n + k]) > mx) mx = fabs(X[i * n + k]);
      if (fabs(Y[k * n + j]) > my) my = fabs(Y[k * n + j]);
    }
    const int e = crt_exp(mx, b), f = crt_exp(my, b);
    for (int64_t k = 0; k < n; ++k) {
      xr[k] = (int64_t)nearbyint(ldexp(X[i * n + k], e));
      yc[k] = (int64_t)nearbyint(ldexp(Y[k * n + j], f));
    }
    Z[q] = crt_elem(n, xr, 1, yc, 1, e, f);
    free(xr); free(yc);
  }
}

void orc_gemm_crt(int64_t n, int b, const double *X, const double *Y, double *Z) {
  int64_t *Xb = (int64_t *)malloc((size_t)(n * n) * sizeof(int64_t));
  int64_t *Yb = (int64_t *)malloc((size_t)(n * n) * sizeof(int64_t));
  int *e = (int *)malloc((size_t)n * sizeof(int)), *f = (int *)malloc((size_t)n * sizeof(int));
  for (int64_t i = 0; i < n; ++i) {                      /* rows of X */
    double mx = 0.0;
    for (int64_t k = 0; k < n; ++k) if (fabs(X[i * n + k]) > mx) mx = fabs(X[i * n + k]);
    e[i] = crt_exp(mx, b);
    for (int64_t k = 0; k < n; ++k) Xb[i * n + k] = (int64_t)nearbyint(ldexp(X[i * n + k], e[i]));
  }
  for (int64_t j = 0; j < n; ++j) {                      /* columns of Y */
    double mx = 0.0;
    for (int64_t k = 0; k < n; ++k) if (fabs(Y[k * n + j]) > mx) mx = fabs(Y[k * n + j]);
    f[j] = crt_exp(mx, b);
    for (int64_t k = 0; k < n; ++k) Yb[k * n + j] = (int64_t)nearbyint(ldexp(Y[k * n + j], f[j]));
  }
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) Z[i * n + j] = crt_elem(n, Xb + i * n, 1, Yb + j, n, e[i], f[j]);
  free(Xb); free(Yb); free(e); free(f);
}
static double clampq(double q) { return q < 1e-3 ? 1e-3 : q > 1.0 ? 1.0 : q; }
/* stored value of a phase: q_m in the container (approximate storage) */
static double store_q(const orc_phase *ph, double x) {
  return orc_qm(x, orc_container_E(ph->prec), phase_m(ph), ph->round == ORC_RTZ);
}

int orc_fp16_sigma(double maxabs) {
  if (!(maxabs > 0.0) || !isfinite(maxabs)) return 0;
  int ex;
  frexp(maxabs, &ex);
  return 14 - (ex - 1);        /* scaled max in [2^14, 2^15), below FP16 max 65504 */
}

/* Scale exponent of a scaled operand format: FP16 as above; FP8 and INT8: scaled max in
 * [2^6, 2^7) (below the E4M3 max 448 and inside the int8 range).  0 for unscaled formats. */
int orc_sigma(int prec, double maxabs) {
  if (prec == ORC_FP16) return orc_fp16_sigma(maxabs);
  if (prec != ORC_FP8 && prec != ORC_INT8) return 0;
  if (!(maxabs > 0.0) || !isfinite(maxabs)) return 0;
  int ex;
  frexp(maxabs, &ex);
  return 6 - (ex - 1);
}

/* INT8 fixed point: nearest integer (ties to even), saturated to [-127, 127]. */
double orc_q_int8(double x) {
  if (isnan(x)) return x;
  double q = nearbyint(x);
  if (q > 127.0) q = 127.0;
  if (q < -127.0) q = -127.0;
  return q;
}

static double maxabs_of(int64_t len, const double *x) {
  double m = 0.0;
  for (int64_t i = 0; i < len; ++i) { double a = fabs(x[i]); if (a > m || isnan(a)) m = a; }
  return m;
}

/* Operand quantisation qin (hardware round-to-nearest-even conversion, R-9).
 * FP16 phase (reading R-20): operand = q16(2^sigma X), sigma from max|X|; returns sigma. */
static int qin_matrix(int prec, int64_t len, const double *x, double *y) {
  int E, M;
  orc_prec_format(prec, &E, &M);
  if (is_f64p(prec)) { if (y != x) memcpy(y, x, (size_t)len * sizeof(double)); return 0; }
  const int sigma = orc_sigma(prec, maxabs_of(len, x));
  if (prec == ORC_INT8) {
    for (int64_t i = 0; i < len; ++i) y[i] = orc_q_int8(ldexp(x[i], sigma));
    return sigma;
  }
  for (int64_t i = 0; i < len; ++i) y[i] = orc_qm(ldexp(x[i], sigma), E, M, 0);
  return sigma;
}

/* ---------------------------------------------------------------------------------
 * Norms of Eq. (3): ||A||_1 = max_j sum_i |a_ij|, ||A||_inf =
 * max_i sum_j |a_ij|; sums sequential in ascending index.  Plus max diagonal (the
 * sufficient condition of reading R-12).
 * ------------------------------------------------------------------------------ */
void orc_norms(int64_t n, const double *A, double *out3) {
  double n1 = 0.0, ninf = 0.0, md = -INFINITY;
  for (int64_t j = 0; j < n; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += fabs(A[i * n + j]);
    if (s > n1 || isnan(s)) n1 = s;
  }
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s += fabs(A[i * n + j]);
    if (s > ninf || isnan(s)) ninf = s;
    if (A[i * n + i] > md) md = A[i * n + i];
  }
  out3[0] = n1; out3[1] = ninf; out3[2] = md;
}

int orc_is_symmetric(int64_t n, const double *A) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j)
      if (memcmp(&A[i * n + j], &A[j * n + i], sizeof(double)) != 0) return 0;
  return 1;
}

/* Rows [r0, r1) of Z = X Y (the same loops as orc_gemm; used to time a bounded sample). */
void orc_gemm_rows(int64_t n, int64_t r0, int64_t r1, const double *X, const double *Y, double *Z) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = r0; i < r1; ++i) {
    double *z = Z + i * n;
    for (int64_t j = 0; j < n; ++j) z[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double x = X[i * n + k];
      const double *y = Y + k * n;
      for (int64_t j = 0; j < n; ++j) z[j] += x * y[j];
    }
  }
}

/* Columns [c0, c1) of Z = X Y (same per-element k order as orc_gemm; column-panel tests). */
void orc_gemm_cols(int64_t n, int64_t c0, int64_t c1, const double *X, const double *Y, double *Z) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double *z = Z + i * n;
    for (int64_t j = c0; j < c1; ++j) z[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double x = X[i * n + k];
      const double *y = Y + k * n;
      for (int64_t j = c0; j < c1; ++j) z[j] += x * y[j];
    }
  }
}

/* Z = X Y: the matrix product of Eq. (1), written as the textbook triple loop. */
void orc_gemm(int64_t n, const double *X, const double *Y, double *Z) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double *z = Z + i * n;
    for (int64_t j = 0; j < n; ++j) z[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double x = X[i * n + k];
      const double *y = Y + k * n;
      for (int64_t j = 0; j < n; ++j) z[j] += x * y[j];
    }
  }
}

void orc_matvec(int64_t n, const double *X, const double *v, double *y) {
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s += X[i * n + k] * v[k];
    y[i] = s;
  }
}

/* ---------------------------------------------------------------------------------
 * Initial guess, Eq. (3): C_0 = (||A||_1 ||A||_inf)^{-1} A^T, then the
 * phase-0 storage rounding ("as well as the input data itself").
 * ------------------------------------------------------------------------------ */
void orc_c0(int64_t n, const double *A, double s, const orc_phase *ph0, double *C0) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) C0[i * n + j] = store_q(ph0, A[j * n + i] / s);
}

/* ---------------------------------------------------------------------------------
 * Controller, reading R-5 ("Increasing the precision in later
 * iterations ... the necessity of increased precision can be detected at runtime";
 * divergence rule from SPEC.md solver: residual > 10x running minimum and > 1).
 * ------------------------------------------------------------------------------ */
void orc_ctrl_init(orc_ctrl *c, int64_t n, int nphases, double final_tol) {
  c->phase = 0; c->nphases = nphases; c->it_in_phase = 0; c->n = n;
  c->rho_prev = NAN; c->rho_best = INFINITY; c->rhohat_min = INFINITY;
  c->final_tol = final_tol; c->best_is_new = 0;
}

int orc_ctrl_decide(orc_ctrl *c, const orc_phase *ph, double rho) {
  const int last = (c->phase == c->nphases - 1);
  const double rhohat = rho / sqrt((double)c->n);
  const int fin = isfinite(rho);
  int d;
  c->best_is_new = 0;
  if (fin && rho < c->rho_best) { c->rho_best = rho; c->best_is_new = 1; }
  if (!fin)
    d = last ? ORC_NONFINITE : ORC_SWITCH;
  else if (last && rho <= c->final_tol)
    d = ORC_CONVERGED;
  else if (rhohat > 10.0 * c->rhohat_min && rhohat > 1.0)
    d = last ? ORC_DIVERGED : ORC_SWITCH;
  else if (!last && ph->switch_tol > 0.0 && rho <= ph->switch_tol)
    d = ORC_SWITCH;
  else if (!last && ph->plateau_ratio > 0.0 && rhohat < ph->plateau_arm &&
           isfinite(c->rho_prev) && rho > ph->plateau_ratio * c->rho_prev)
    d = ORC_SWITCH;
  else if (ph->max_iters > 0 && c->it_in_phase + 1 >= ph->max_iters)
    d = last ? ORC_ITER_LIMIT : ORC_SWITCH;
  else
    d = ORC_CONTINUE;
  if (fin && rhohat < c->rhohat_min) c->rhohat_min = rhohat;
  c->rho_prev = rho;
  c->it_in_phase += 1;
  return d;
}

void orc_ctrl_enter_next_phase(orc_ctrl *c) {
  c->phase += 1; c->it_in_phase = 0; c->rho_prev = NAN;
}

/* ---------------------------------------------------------------------------------
 * One iteration of Eq. (1), in the reading of DESIGN.md:
 *  R-1 right-to-left chain  T_1 = Chat Ahat,  T_j = Chat qin(T_{j-1}),  P = Chat qin(T_p)
 *  R-9 Ahat = qin(q_m(A)) and Chat = qin(C); intermediates take the operand format
 *  R-2 C_next = q_m( ((p+1) C - P) / p )  -- three FP64 operations, one rounding
 *  residual rho = ||I - T_p||_F from the unrounded T_p (T_p = C^p A).
 * ------------------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  double *Chat, *X, *T;
  int sigC, sigX;
  int sigR;                   /* symmetric form: sigma of Rhat when the correction format is scaled */
  int crt_b;                  /* FP64_CRT phase: bits b of this chain's products (0: exact FP64 GEMMs) */
} chain_ws;

/* a chain product of the symmetric forms: the FP64 GEMM, or the CRT product of an FP64_CRT phase */
static void chain_gemm(const chain_ws *w, int64_t n, const double *X, const double *Y, double *Z) {
  if (w->crt_b > 0) orc_gemm_crt(n, w->crt_b, X, Y, Z);
  else orc_gemm(n, X, Y, Z);
}

static double chain(int64_t n, int p, const double *A, const double *C, const orc_phase *ph,
                    chain_ws *w) {
  const int64_t nn = n * n;
  /* Ahat = qin(q_m(A)) */
  for (int64_t i = 0; i < nn; ++i) w->T[i] = store_q(ph, A[i]);
  w->sigX = qin_matrix(ph->prec, nn, w->T, w->X);
  w->sigC = qin_matrix(ph->prec, nn, C, w->Chat);
  double rho = 0.0;
  for (int j = 1; j <= p; ++j) {
    orc_gemm(n, w->Chat, w->X, w->T);                      /* T_j = Chat X */
    if (w->sigC + w->sigX != 0)
      for (int64_t i = 0; i < nn; ++i) w->T[i] = ldexp(w->T[i], -(w->sigC + w->sigX));
    if (j == p) {                                           /* rho = ||I - T_p||_F */
      double s2 = 0.0;
      for (int64_t r = 0; r < n; ++r)
        for (int64_t c = 0; c < n; ++c) {
          const double d = (r == c ? 1.0 : 0.0) - w->T[r * n + c];
          s2 += d * d;
        }
      rho = sqrt(s2);
    }
    w->sigX = qin_matrix(ph->prec, nn, w->T, w->X);        /* X = qin(T_j) */
  }
  return rho;
}

static double update(int64_t n, int p, const double *C, const orc_phase *ph, chain_ws *w,
                     double *C_next) {
  const int64_t nn = n * n;
  orc_gemm(n, w->Chat, w->X, w->T);                        /* P = Chat qin(T_p) */
  if (w->sigC + w->sigX != 0)
    for (int64_t i = 0; i < nn; ++i) w->T[i] = ldexp(w->T[i], -(w->sigC + w->sigX));
  const double pp1 = (double)(p + 1), pd = (double)p;
  double s2 = 0.0;
  for (int64_t i = 0; i < nn; ++i) {
    const double a = pp1 * C[i];
    const double d = a - w->T[i];
    const double e = d / pd;
    const double c1 = store_q(ph, e);
    const double dd = c1 - C[i];
    s2 += dd * dd;
    C_next[i] = c1;
  }
  return sqrt(s2);
}

/* ---------------------------------------------------------------------------------
 * NEXT-1: the Newton-Schulz ordering of the p = 1 iteration.
 * [Sec. 2]: "For p=1 the algorithm corresponds to the well-known Newton-Schulz method"; the
 * textbook Newton-Schulz step is X_{k+1} = X_k (2I - A X_k):
 *   Xhat = qin(X), Ahat = qin(q_m(A)), T = Ahat Xhat (FP64 accumulator),
 *   rho = ||I - T||_F (unrounded T), What = qin(2I - T) (one FP64 subtraction per element),
 *   X_{k+1} = q_m(Xhat What)  (FP64 accumulator, one rounding to m bits).
 * ------------------------------------------------------------------------------ */
static double chain_ns(int64_t n, const double *A, const double *X, const orc_phase *ph, chain_ws *w) {
  const int64_t nn = n * n;
  for (int64_t i = 0; i < nn; ++i) w->T[i] = store_q(ph, A[i]);
  const int sigA = qin_matrix(ph->prec, nn, w->T, w->X);   /* w->X = Ahat (scratch) */
  w->sigC = qin_matrix(ph->prec, nn, X, w->Chat);           /* w->Chat = Xhat        */
  orc_gemm(n, w->X, w->Chat, w->T);                         /* T = Ahat Xhat         */
  if (sigA + w->sigC != 0)
    for (int64_t i = 0; i < nn; ++i) w->T[i] = ldexp(w->T[i], -(sigA + w->sigC));
  double s2 = 0.0;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t c = 0; c < n; ++c) {
      const double d = (r == c ? 1.0 : 0.0) - w->T[r * n + c];
      s2 += d * d;
    }
  for (int64_t r = 0; r < n; ++r)                           /* W = 2I - T            */
    for (int64_t c = 0; c < n; ++c) w->T[r * n + c] = (r == c ? 2.0 : 0.0) - w->T[r * n + c];
  w->sigX = qin_matrix(ph->prec, nn, w->T, w->X);           /* w->X = What           */
  return sqrt(s2);
}

static double update_ns(int64_t n, const double *X, const orc_phase *ph, chain_ws *w, double *X_next) {
  const int64_t nn = n * n;
  orc_gemm(n, w->Chat, w->X, w->T);                         /* Xhat What             */
  if (w->sigC + w->sigX != 0)
    for (int64_t i = 0; i < nn; ++i) w->T[i] = ldexp(w->T[i], -(w->sigC + w->sigX));
  double s2 = 0.0;
  for (int64_t i = 0; i < nn; ++i) {
    const double x1 = store_q(ph, w->T[i]);
    const double dd = x1 - X[i];
    s2 += dd * dd;
    X_next[i] = x1;
  }
  return sqrt(s2);
}

/* ---------------------------------------------------------------------------------
 * NEXT-2: the symmetrised-correction form for p >= 2.  Not printed in the
 * paper: it is the Newton correction of Eq. (1) (PAPER.md:71-73 reads C_{k+1} = C_k +
 * C_k (I - C_k^p A) / p) with the residual taken as R = I - C^{p-1} A C and the correction
 * symmetrised, so that noise which does not commute with A is damped (R-22):
 *   Chat = qin(C), Ahat = qin(q_m(A)),  Z_1 = Ahat Chat,  Z_j = Chat qin(Z_{j-1}) (j = 2..p)
 *   rho_s = ||I - Z_p||_F (unrounded Z_p),  Rhat = qc(I - Z_p)   (one FP64 subtraction)
 *   W = qc(C) Rhat  (FP64 accumulator),   C_{k+1}[i][j] = q_m(C_ij + (W_ij + W_ji) / (2p))
 * where qc is the operand format of the correction GEMM (corr_prec; = prec by default).
 * C_{k+1} is exactly symmetric whenever C_k is (W_ij + W_ji is commutative in IEEE).
 * Scaled formats (FP16/FP8/INT8) scale Chat, Ahat and qin(Z_j) by powers of two (reading R-20)
 * and unscale every product exactly; the correction format is BF16, TF32 or FP64, or the phase's
 * own scaled format (an FP8 phase with an FP8 correction, R-29): then Rhat = 2^sigR R and
 * qc(C) = Chat carry their own sigmas and W is unscaled by 2^-(sigC + sigR), exactly.
 * ------------------------------------------------------------------------------ */
static int is_scaled(int prec) { return prec == ORC_FP16 || prec == ORC_FP8 || prec == ORC_INT8; }
/* default correction format: the phase's own, BF16 for the scaled formats */
static int corr_of(const orc_phase *ph) {
  if (ph->corr_prec >= 0) return ph->corr_prec;
  return is_scaled(ph->prec) ? ORC_BF16 : ph->prec;
}

/* Reading R-36: the symmetric forms in a reduced-precision phase (not FP64 / FP64_OZ / FP64_CRT) take every
 * product from its upper triangle: each Z_j := the mirror of its upper triangle (j = 1..p) and the correction
 * S_ij = 2 W_{min(i,j), max(i,j)} instead of W_ij + W_ji -- each differs from the full product by a commutator
 * ([A, C], [C, Z_j], [C, R]) that sits at the phase's own rounding level there (C_k is a polynomial in A up to
 * that noise); FP64-range phases keep the full products (the symmetrisation of W + W^T sets R-22's linear
 * rate), except the tri form's Z_2 = C A C (symmetric in exact arithmetic, ORC_FORM_SYMMETRIC_TRI). */
/* Reading R-37 (ORC_FORM_SYMMETRIC_TRIZ, p = 2): in an FP64_CRT phase the chain's Z_1 = Ahat Chat is ALSO taken from
 * its upper triangle (tri == 2 below) while the phase contracts fast: from the third chain of the phase on, as long
 * as every in-phase ratio rho_k / rho_{k-1} so far was <= ORC_ZTRI_RATIO (sticky: one slower step and the phase keeps
 * the full Z_1 for good -- the mirror feeds the commutator [A, C] back into R, which only pays while the symmetric
 * update removes it much faster than that).  W + W^T stays full. */
#define ORC_ZTRI_RATIO 0.1
static int tri_w_phase(int tri, const orc_phase *ph) {
  (void)tri;
  return ph->prec != ORC_FP64 && ph->prec != ORC_FP64_OZ && ph->prec != ORC_FP64_CRT;
}

static double chain_sym(int64_t n, int p, int tri, const double *A, const double *C,
                        const orc_phase *ph, chain_ws *w) {
  const int64_t nn = n * n;
  for (int64_t i = 0; i < nn; ++i) w->T[i] = store_q(ph, A[i]);
  const int sigA = qin_matrix(ph->prec, nn, w->T, w->X);    /* w->X = Ahat            */
  w->sigC = qin_matrix(ph->prec, nn, C, w->Chat);           /* w->Chat = Chat         */
  chain_gemm(w, n, w->X, w->Chat, w->T);                    /* Z_1 = Ahat Chat        */
  int sigX = sigA;                                           /* scaled formats: unscale */
  for (int j = 1; j <= p; ++j) {
    if (j > 1) chain_gemm(w, n, w->Chat, w->X, w->T);       /* Z_j = Chat qin(Z_{j-1}) */
    if (sigX + w->sigC != 0)
      for (int64_t i = 0; i < nn; ++i) w->T[i] = ldexp(w->T[i], -(sigX + w->sigC));
    if (j < p && (tri_w_phase(tri, ph) || tri == 2))        /* R-36 / R-37: Z_j from its upper triangle */
      for (int64_t r = 0; r < n; ++r)
        for (int64_t c = 0; c < r; ++c) w->T[r * n + c] = w->T[c * n + r];
    if (j < p) sigX = qin_matrix(ph->prec, nn, w->T, w->X); /* qin(Z_j)               */
  }
  if (tri || tri_w_phase(tri, ph))   /* ORC_FORM_SYMMETRIC_TRI: Z_2 = C A C from its upper triangle; R-36: Z_p */
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c < r; ++c) w->T[r * n + c] = w->T[c * n + r];
  double s2 = 0.0;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t c = 0; c < n; ++c) {
      const double d = (r == c ? 1.0 : 0.0) - w->T[r * n + c];   /* R = I - Z_p        */
      s2 += d * d;
      w->T[r * n + c] = d;
    }
  w->sigR = qin_matrix(corr_of(ph), nn, w->T, w->X);        /* w->X = Rhat (2^sigR R)  */
  return sqrt(s2);
}


static double update_sym(int64_t n, int p, int tri, const double *C, const orc_phase *ph, chain_ws *w,
                         double *C_next) {
  const int triw = tri_w_phase(tri, ph);
  const int64_t nn = n * n;
  const int sigCc = qin_matrix(corr_of(ph), nn, C, w->Chat); /* qc(C)                 */
  orc_gemm(n, w->Chat, w->X, w->T);                         /* W = qc(C) Rhat         */
  if (sigCc + w->sigR != 0)   /* a scaled (FP8) correction: unscale exactly, as the chain does */
    for (int64_t i = 0; i < nn; ++i) w->T[i] = ldexp(w->T[i], -(sigCc + w->sigR));
  const double tp = (double)(2 * p);
  double s2 = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const double sw = triw ? 2.0 * w->T[(i < j ? i : j) * n + (i < j ? j : i)]
                             : w->T[i * n + j] + w->T[j * n + i];
      const double e = sw / tp;
      const double c1 = store_q(ph, C[i * n + j] + e);
      const double dd = c1 - C[i * n + j];
      s2 += dd * dd;
      C_next[i * n + j] = c1;
    }
  return sqrt(s2);
}

/* ---------------------------------------------------------------------------------
 * NEXT-2 (ii): the coupled (M-carrying) form of the same iteration.  With
 * M_k = X_k^p A and N_k = ((p+1) I - M_k) / p, Eq. (1) reads X_{k+1} = X_k N_k and
 * (in exact arithmetic) M_{k+1} = N_k^p M_k.  Carrying M keeps the error bounded after convergence
 * for any kappa (SURVEY Table A3) but, unlike the symmetrised form, does not remove noise that
 * earlier phases left in X.  In the order the GPU evaluates it (R-27):
 *   anchor (first chain of a phase):  T_1 = qin(X) Ahat, T_j = qin(X) qin(T_{j-1}) (j = 2..p)
 *   finish of a chain ending in T:    rho = ||I - T||_F (unrounded); w = q_m(T);
 *                                     Mhat = qin(w); N = ((p+1) delta - w) / p (three FP64 ops,
 *                                     the integers exact); Nhat = qin(N)
 *   step:  X_{k+1} = q_m(qin(X_k) Nhat);  T_1 = Nhat Mhat, T_j = Nhat qin(T_{j-1});  finish(T_p)
 * Scaled (FP16/FP8/INT8) formats are not defined for this form.
 * ------------------------------------------------------------------------------ */
static double coupled_finish(int64_t n, int p, const orc_phase *ph, const double *T, double *Mh, double *Nh) {
  double s2 = 0.0;
  const double pp1 = (double)(p + 1), pd = (double)p;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t c = 0; c < n; ++c) {
      const double v = T[r * n + c];
      const double d = (r == c ? 1.0 : 0.0) - v;
      s2 += d * d;
      const double wv = store_q(ph, v);
      Mh[r * n + c] = wv;
      const double a = r == c ? pp1 : 0.0;
      Nh[r * n + c] = (a - wv) / pd;
    }
  qin_matrix(ph->prec, n * n, Mh, Mh);
  qin_matrix(ph->prec, n * n, Nh, Nh);
  return sqrt(s2);
}

static double coupled_anchor(int64_t n, int p, const double *A, const double *X, const orc_phase *ph,
                             chain_ws *w, double *Mh, double *Nh) {
  const int64_t nn = n * n;
  for (int64_t i = 0; i < nn; ++i) w->T[i] = store_q(ph, A[i]);
  qin_matrix(ph->prec, nn, w->T, w->X);                     /* Ahat                   */
  qin_matrix(ph->prec, nn, X, w->Chat);                     /* Xhat                   */
  for (int j = 1; j <= p; ++j) {
    orc_gemm(n, w->Chat, w->X, w->T);                       /* T_j = Xhat qin(T_{j-1}) */
    if (j < p) qin_matrix(ph->prec, nn, w->T, w->X);
  }
  return coupled_finish(n, p, ph, w->T, Mh, Nh);
}

/* X_next = q_m(qin(X) Nhat); M chain; returns delta = ||X_next - X||_F, *rho_next from finish */
static double coupled_step(int64_t n, int p, const double *X, const orc_phase *ph, chain_ws *w,
                           double *Mh, double *Nh, double *X_next, double *rho_next) {
  const int64_t nn = n * n;
  qin_matrix(ph->prec, nn, X, w->Chat);
  orc_gemm(n, w->Chat, Nh, w->T);                           /* X Nhat                 */
  double s2 = 0.0;
  for (int64_t i = 0; i < nn; ++i) {
    const double x1 = store_q(ph, w->T[i]);
    const double dd = x1 - X[i];
    s2 += dd * dd;
    X_next[i] = x1;
  }
  orc_gemm(n, Nh, Mh, w->T);                                /* T_1 = Nhat Mhat        */
  for (int j = 2; j <= p; ++j) {
    qin_matrix(ph->prec, nn, w->T, w->X);
    orc_gemm(n, Nh, w->X, w->T);                            /* T_j = Nhat qin(T_{j-1}) */
  }
  *rho_next = coupled_finish(n, p, ph, w->T, Mh, Nh);
  return sqrt(s2);
}

static int ws_alloc(chain_ws *w, int64_t n) {
  const size_t b = (size_t)(n * n) * sizeof(double);
  w->n = n;
  w->Chat = (double *)malloc(b); w->X = (double *)malloc(b); w->T = (double *)malloc(b);
  w->crt_b = 0;
  return w->Chat && w->X && w->T;
}
static void ws_free(chain_ws *w) { free(w->Chat); free(w->X); free(w->T); }

double orc_step(int64_t n, int p, const double *A, const double *C, const orc_phase *ph,
                double *C_next, double *delta) {
  chain_ws w;
  if (!ws_alloc(&w, n)) { ws_free(&w); return NAN; }
  const double rho = chain(n, p, A, C, ph, &w);
  if (C_next) { const double d = update(n, p, C, ph, &w, C_next); if (delta) *delta = d; }
  ws_free(&w);
  return rho;
}

static double gamma_of(int64_t n, const double *C, const double *A, double normA2,
                       double *t1, double *t2) {
  orc_gemm(n, C, A, t1);
  orc_gemm(n, A, C, t2);
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n * n; ++i) {
    const double d = t1[i] - t2[i];
    s += d * d; c += C[i] * C[i];
  }
  return sqrt(s) / (sqrt(c) * normA2);
}

/* Re-container an FP64 copy of an iterate into phase ph's storage format (reading R-5:
 * the next phase restarts from the best iterate). */
static void recontainer(int64_t nn, const double *src, const orc_phase *ph, double *dst) {
  for (int64_t i = 0; i < nn; ++i) dst[i] = store_q(ph, src[i]);
}

double orc_step_ns(int64_t n, const double *A, const double *X, const orc_phase *ph,
                   double *X_next, double *delta) {
  chain_ws w;
  if (!ws_alloc(&w, n)) { ws_free(&w); return NAN; }
  const double rho = chain_ns(n, A, X, ph, &w);
  if (X_next) { const double d = update_ns(n, X, ph, &w, X_next); if (delta) *delta = d; }
  ws_free(&w);
  return rho;
}

double orc_step_sym(int64_t n, int p, const double *A, const double *C, const orc_phase *ph,
                    double *C_next, double *delta) {
  return orc_step_sym_form(n, p, 0, A, C, ph, C_next, delta);
}

double orc_step_sym_form(int64_t n, int p, int tri, const double *A, const double *C, const orc_phase *ph,
                         double *C_next, double *delta) {
  if (p < 2 || (is_scaled(corr_of(ph)) && corr_of(ph) != ph->prec) || (tri && p != 2)) return NAN;
  chain_ws w;
  if (!ws_alloc(&w, n)) { ws_free(&w); return NAN; }
  if (ph->prec == ORC_FP64_CRT)   /* a single step: the digits of the phase's fixed m (9 if adaptive) */
    w.crt_b = orc_crt_bits(is_adaptive(ph) ? 9 : orc_digits_for_m(phase_m(ph)), n);
  const double rho = chain_sym(n, p, tri, A, C, ph, &w);
  if (C_next) { const double d = update_sym(n, p, tri, C, ph, &w, C_next); if (delta) *delta = d; }
  ws_free(&w);
  return rho;
}

int orc_solve(int64_t n, int p, const double *A, const orc_phase *phases, int nphases,
              double final_tol, int max_total, orc_record *rec, int cap_rec, int *nrec,
              double *C_best, double *C_hist, int hist_cap, double gamma_normA2,
              double *s_out) {
  return orc_solve_form(n, p, ORC_FORM_LITERAL, A, phases, nphases, final_tol, max_total, rec,
                        cap_rec, nrec, C_best, C_hist, hist_cap, gamma_normA2, s_out);
}

/* Reading R-33: after an update in the last phase of a symmetric form, the in-phase
 * linear rate q = rho_k / rho_{k-1} predicts rho_{k+1} ~ rho_k q; when that is <= final_tol / 2 the
 * next iterate is certified (FP64 literal chain) before its own chain, and the chain runs only if the
 * certificate misses.  The GPU engine's default (IPR_CERT_FP64); 0 = trigger on the chain only. */
static int g_predict_cert = 1;
void orc_set_predict_cert(int on) { g_predict_cert = on != 0; }

/* Certificate of a symmetric form's candidate C (R-30; R-35 with orc_set_cert_mode(1)): returns the
 * certified residual; Ct receives the matrix it is the residual of (the answer when it passes). */
static int g_cert_mode = 0;
void orc_set_cert_mode(int mode) { g_cert_mode = mode; }
static double sym_cert(int64_t n, int p, const double *A, const double *C, chain_ws *w, double *Ct) {
  if (g_cert_mode == 1) {
    orc_cert_grid(n, 62, C, Ct);
    return orc_resid_dd(n, p, A, Ct);
  }
  const orc_phase ph64 = {ORC_FP64, -1, ORC_RNE, 0.0, 0.0, 0.0, 0, -1};
  memcpy(Ct, C, (size_t)(n * n) * sizeof(double));
  return chain(n, p, A, C, &ph64, w);
}

int orc_solve_form(int64_t n, int p, int form, const double *A, const orc_phase *phases,
                   int nphases, double final_tol, int max_total, orc_record *rec, int cap_rec,
                   int *nrec, double *C_best, double *C_hist, int hist_cap, double gamma_normA2,
                   double *s_out) {
  *nrec = 0;
  if (n <= 0 || p < 1 || nphases < 1) return -1;
  if (form == ORC_FORM_NEWTON_SCHULZ && p != 1) return -1;
  if (form == ORC_FORM_COUPLED)
    for (int i = 0; i < nphases; ++i)
      if (is_scaled(phases[i].prec)) return -1;
  const int triz = form == ORC_FORM_SYMMETRIC_TRIZ;
  if (triz) form = ORC_FORM_SYMMETRIC_TRI;   /* R-37: the tri form + the Z_1 rule below */
  const int sym = form == ORC_FORM_SYMMETRIC || form == ORC_FORM_SYMMETRIC_TRI;
  if (sym) {
    if (p < 2 || (form == ORC_FORM_SYMMETRIC_TRI && p != 2)) return -1;
    for (int i = 0; i < nphases; ++i)
      if (is_scaled(corr_of(&phases[i])) && corr_of(&phases[i]) != phases[i].prec) return -1;
  }
  if (form < ORC_FORM_LITERAL || form > ORC_FORM_COUPLED) return -1;
  for (int i = 0; i < nphases; ++i)   /* FP64_CRT products are defined for the symmetric forms only */
    if (phases[i].prec == ORC_FP64_CRT && !sym) return -1;
  if (!orc_is_symmetric(n, A)) return -2;
  const int64_t nn = n * n;
  double nrm[3];
  orc_norms(n, A, nrm);
  const double s = nrm[0] * nrm[1];
  if (s_out) *s_out = s;
  double *C = (double *)malloc((size_t)nn * sizeof(double));
  double *Cn = (double *)malloc((size_t)nn * sizeof(double));
  double *Ct = (double *)malloc((size_t)nn * sizeof(double));   /* the certified matrix (R-35) */
  double *g1 = NULL, *g2 = NULL;
  if (gamma_normA2 > 0) {
    g1 = (double *)malloc((size_t)nn * sizeof(double));
    g2 = (double *)malloc((size_t)nn * sizeof(double));
  }
  chain_ws w;
  ws_alloc(&w, n);
  const int coupled = form == ORC_FORM_COUPLED;
  double *Mh = coupled ? (double *)malloc((size_t)nn * sizeof(double)) : NULL;
  double *Nh = coupled ? (double *)malloc((size_t)nn * sizeof(double)) : NULL;
  int anchor = 1;
  double rho_next = NAN;
  orc_c0(n, A, s, &phases[0], C);
  memcpy(C_best, C, (size_t)nn * sizeof(double));
  orc_ctrl ctl;
  orc_ctrl_init(&ctl, n, nphases, final_tol);
  int outcome = ORC_CONTINUE;
  /* R-26 state: last residual (any phase), the last two in-phase residuals, the stored m of C */
  double last_rho_hat = NAN, ph_r1 = NAN, ph_r2 = NAN;
  int z_ok = 1;                       /* R-37: no in-phase ratio above ORC_ZTRI_RATIO so far */
  int m_of_C = is_adaptive(&phases[0]) ? 52 : phase_m(&phases[0]);
  int cert_pending = 0;               /* R-33 */
  for (int k = 0; k < max_total; ++k) {
    const orc_phase *ph = &phases[ctl.phase];
    double cert_pre = NAN;
    if (cert_pending) {               /* R-33: the predicted-converged iterate, certificate first */
      cert_pending = 0;
      if (C_hist && k < hist_cap) memcpy(C_hist + (int64_t)k * nn, C, (size_t)nn * sizeof(double));
      cert_pre = sym_cert(n, p, A, C, &w, Ct);
      if (cert_pre <= final_tol) {
        orc_record r;
        r.k = k; r.phase = ctl.phase; r.prec = ph->prec; r.mant_bits = m_of_C;
        r.decision = ORC_CONVERGED; r.rho = NAN; r.rho_hat = NAN; r.delta = NAN;
        r.gamma = (gamma_normA2 > 0) ? gamma_of(n, C, A, gamma_normA2, g1, g2) : NAN;
        r.rho_cert = cert_pre;
        memcpy(C_best, Ct, (size_t)nn * sizeof(double));  /* the certified matrix is the answer */
        if (*nrec < cap_rec) rec[*nrec] = r;
        *nrec += 1;
        outcome = ORC_CONVERGED;
        break;
      }
    }
    orc_phase ph_k = *ph;             /* the phase with this iteration's storage bits */
    int S_k = orc_digits_for_m(phase_m(ph));
    if (is_adaptive(ph)) {
      const double q = (isfinite(ph_r1) && isfinite(ph_r2) && ph_r2 > 0.0) ? clampq(ph_r1 / ph_r2) : 0.03;
      S_k = k == 0 ? 9 : orc_oz_digits(last_rho_hat * q * q, n);
      ph_k.mant_bits = orc_oz_adaptive_m(S_k);
    }
    /* FP64_CRT: this chain's products at b = orc_crt_bits(S_k) (R-26 digits, R-28 bits) */
    w.crt_b = ph->prec == ORC_FP64_CRT ? orc_crt_bits(S_k, n) : 0;
    if (C_hist && k < hist_cap) memcpy(C_hist + (int64_t)k * nn, C, (size_t)nn * sizeof(double));
    double rho;
    if (coupled) {
      rho = anchor ? coupled_anchor(n, p, A, C, ph, &w, Mh, Nh) : rho_next;
      anchor = 0;
    } else {
      rho = form == ORC_FORM_NEWTON_SCHULZ ? chain_ns(n, A, C, ph, &w)
            : sym ? chain_sym(n, p, form == ORC_FORM_SYMMETRIC_TRI
                                        ? (triz && ph->prec == ORC_FP64_CRT && z_ok && isfinite(ph_r1) && isfinite(ph_r2) ? 2 : 1)
                                        : 0, A, C, ph, &w)
                  : chain(n, p, A, C, ph, &w);
    }
    const int phase_now = ctl.phase;
    int d = orc_ctrl_decide(&ctl, ph, rho);
    if (ctl.best_is_new) memcpy(C_best, C, (size_t)nn * sizeof(double));
    orc_record r;
    r.k = k; r.phase = phase_now; r.prec = ph->prec; r.mant_bits = m_of_C;
    r.decision = d; r.rho = rho; r.rho_hat = rho / sqrt((double)n); r.delta = NAN;
    r.gamma = (gamma_normA2 > 0) ? gamma_of(n, C, A, gamma_normA2, g1, g2) : NAN;
    r.rho_cert = cert_pre;
    if (d == ORC_CONVERGED && coupled) {
      /* rho = ||I - M_k||_F tracks ||I - X_k^p A||_F only up to drift: certify on X_k itself
       * (the best iterate), continue with the step if it misses (as the GPU engine does) */
      const orc_phase ph64 = {ORC_FP64, -1, ORC_RNE, 0.0, 0.0, 0.0, 0, -1};
      r.rho_cert = chain(n, p, A, C, &ph64, &w);
      if (!(r.rho_cert <= final_tol)) {
        d = ORC_CONTINUE;
        r.decision = d;
        r.delta = coupled_step(n, p, C, ph, &w, Mh, Nh, Cn, &rho_next);
        double *t = C; C = Cn; Cn = t;
        m_of_C = phase_m(ph);
        if (ph->max_iters > 0 && ctl.it_in_phase >= ph->max_iters) { d = ORC_ITER_LIMIT; r.decision = d; }
      } else {
        memcpy(C_best, C, (size_t)nn * sizeof(double));   /* the certified iterate is the answer (R-30) */
      }
    } else if (d == ORC_CONVERGED && sym) {
      /* rho_s = ||I - C^{p-1} A C||_F is not the north-star residual: certify
       * ||I - C^p A||_F with the FP64 literal chain (reading R-3); if it misses final_tol the
       * iteration continues from the update computed first (as the GPU engine does). */
      r.delta = update_sym(n, p, form == ORC_FORM_SYMMETRIC_TRI, C, &ph_k, &w, Cn);
      r.rho_cert = isfinite(cert_pre) ? cert_pre : sym_cert(n, p, A, C, &w, Ct);   /* R-33: once */
      if (!(r.rho_cert <= final_tol)) {
        d = ORC_CONTINUE;
        r.decision = d;
        double *t = C; C = Cn; Cn = t;
        m_of_C = phase_m(&ph_k);
        /* the last phase's cap still applies after a missed certificate (as the GPU engine) */
        if (ph->max_iters > 0 && ctl.it_in_phase >= ph->max_iters) { d = ORC_ITER_LIMIT; r.decision = d; }
      } else {
        memcpy(C_best, Ct, (size_t)nn * sizeof(double));  /* the certified matrix is the answer (R-30, R-35) */
      }
    } else if (d == ORC_CONTINUE && coupled) {
      r.delta = coupled_step(n, p, C, ph, &w, Mh, Nh, Cn, &rho_next);
      double *t = C; C = Cn; Cn = t;
      m_of_C = phase_m(ph);
    } else if (d == ORC_CONTINUE) {
      r.delta = form == ORC_FORM_NEWTON_SCHULZ ? update_ns(n, C, ph, &w, Cn)
                : sym                           ? update_sym(n, p, form == ORC_FORM_SYMMETRIC_TRI, C, &ph_k, &w, Cn)
                                                : update(n, p, C, ph, &w, Cn);
      double *t = C; C = Cn; Cn = t;
      m_of_C = phase_m(&ph_k);
    } else if (d == ORC_SWITCH) {
      orc_ctrl_enter_next_phase(&ctl);
      orc_phase pe = phases[ctl.phase];
      if (is_adaptive(&pe))   /* entry storage from the digits the entering chain will use */
        pe.mant_bits = orc_oz_adaptive_m(orc_oz_digits(rho / sqrt((double)n) * 0.03 * 0.03, n));
      recontainer(nn, C_best, &pe, C);
      m_of_C = phase_m(&pe);
      anchor = 1;                     /* coupled: re-anchor M = X^p A in the new phase */
    }
    /* R-26 bookkeeping */
    last_rho_hat = rho / sqrt((double)n);
    if (d == ORC_SWITCH) { ph_r1 = NAN; ph_r2 = NAN; z_ok = 1; }
    else {
      ph_r2 = ph_r1; ph_r1 = rho;
      if (isfinite(ph_r2) && !(ph_r1 <= ORC_ZTRI_RATIO * ph_r2)) z_ok = 0;
    }
    /* R-33: certify the next iterate first when the last phase's rate predicts it converged */
    if (d == ORC_CONTINUE && sym && g_predict_cert && ctl.phase == nphases - 1 && isfinite(ph_r1) &&
        isfinite(ph_r2) && ph_r2 > 0.0 && ph_r1 < ph_r2 && ph_r1 * (ph_r1 / ph_r2) <= 0.5 * final_tol)
      cert_pending = 1;
    if (*nrec < cap_rec) rec[*nrec] = r;
    *nrec += 1;
    if (d != ORC_CONTINUE && d != ORC_SWITCH) { outcome = d; break; }
  }
  ws_free(&w);
  free(C); free(Cn); free(Ct); free(g1); free(g2); free(Mh); free(Nh);
  return outcome;
}

/* ---------------------------------------------------------------------------------
 * Brute-force limit for small n (SPEC.md oracle module; the paper's "solution that was
 * precomputed using double-precision"): cyclic Jacobi rotations
 * (Golub & Van Loan, Alg. 8.5.3) and X = V diag(lambda^{-1/p}) V^T.
 * ------------------------------------------------------------------------------ */
int orc_jacobi(int64_t n, const double *A0, double *lambda, double *V) {
  double *A = (double *)malloc((size_t)(n * n) * sizeof(double));
  memcpy(A, A0, (size_t)(n * n) * sizeof(double));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) V[i * n + j] = (i == j) ? 1.0 : 0.0;
  double fro = 0.0;
  for (int64_t i = 0; i < n * n; ++i) fro += A[i] * A[i];
  fro = sqrt(fro);
  int sweep;
  for (sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j)
        if (i != j) off += A[i * n + j] * A[i * n + j];
    if (sqrt(off) <= 1e-15 * fro) break;
    for (int64_t pi = 0; pi < n - 1; ++pi)
      for (int64_t qi = pi + 1; qi < n; ++qi) {
        const double apq = A[pi * n + qi];
        if (apq == 0.0) continue;
        const double theta = (A[qi * n + qi] - A[pi * n + pi]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(1.0 + theta * theta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = t * c;
        for (int64_t k = 0; k < n; ++k) {           /* A <- A J (columns p, q) */
          const double akp = A[k * n + pi], akq = A[k * n + qi];
          A[k * n + pi] = c * akp - sn * akq;
          A[k * n + qi] = sn * akp + c * akq;
        }
        for (int64_t k = 0; k < n; ++k) {           /* A <- J^T A (rows p, q) */
          const double apk = A[pi * n + k], aqk = A[qi * n + k];
          A[pi * n + k] = c * apk - sn * aqk;
          A[qi * n + k] = sn * apk + c * aqk;
        }
        for (int64_t k = 0; k < n; ++k) {           /* V <- V J */
          const double vkp = V[k * n + pi], vkq = V[k * n + qi];
          V[k * n + pi] = c * vkp - sn * vkq;
          V[k * n + qi] = sn * vkp + c * vkq;
        }
      }
  }
  for (int64_t i = 0; i < n; ++i) lambda[i] = A[i * n + i];
  /* selection sort ascending, permuting V's columns with lambda */
  for (int64_t i = 0; i < n; ++i) {
    int64_t m = i;
    for (int64_t j = i + 1; j < n; ++j) if (lambda[j] < lambda[m]) m = j;
    if (m != i) {
      double t = lambda[i]; lambda[i] = lambda[m]; lambda[m] = t;
      for (int64_t k = 0; k < n; ++k) {
        double u = V[k * n + i]; V[k * n + i] = V[k * n + m]; V[k * n + m] = u;
      }
    }
  }
  free(A);
  return sweep;
}

void orc_inv_proot_eig(int64_t n, const double *lambda, const double *V, int p, double *X) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k)
        s += V[i * n + k] * pow(lambda[k], -1.0 / (double)p) * V[j * n + k];
      X[i * n + j] = s;
    }
}

/* ---------------------------------------------------------------------------------
 * Spectral predictor (exact arithmetic).  C_0 = A/s is a polynomial in A, hence so is
 * every C_k (Eq. 1); in A's eigenbasis c_{k+1} = c_k ((p+1) - c_k^p lambda)/p.  With
 * t = c^p lambda:  t_0 = lambda^{p+1}/s^p,  t_{k+1} = t_k ((p+1 - t_k)/p)^p,  and
 * ||I - C_k^p A||_F^2 = sum_i (1 - t_i)^2.
 * ------------------------------------------------------------------------------ */
void orc_spectral(int64_t n, const double *lambda, int p, double s, int kmax, double *rho_hat) {
  double *t = (double *)malloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) t[i] = pow(lambda[i], (double)(p + 1)) / pow(s, (double)p);
  for (int k = 0; k < kmax; ++k) {
    double s2 = 0.0;
    for (int64_t i = 0; i < n; ++i) s2 += (1.0 - t[i]) * (1.0 - t[i]);
    rho_hat[k] = sqrt(s2 / (double)n);
    for (int64_t i = 0; i < n; ++i) t[i] = t[i] * pow(((double)(p + 1) - t[i]) / (double)p, (double)p);
  }
  free(t);
}

/* ---------------------------------------------------------------------------------------------
 * The CRT certificate (reading R-35): the grid rounding of the certified matrix and the
 * double-double residual that the oracle certifies it with.
 * ------------------------------------------------------------------------------------------- */
void orc_cert_grid(int64_t n, int b, const double *C, double *Ct) {
  int *e = (int *)malloc((size_t)n * sizeof(int));
  for (int64_t i = 0; i < n; ++i) {
    double mx = 0.0;
    for (int64_t k = 0; k < n; ++k) if (fabs(C[i * n + k]) > mx) mx = fabs(C[i * n + k]);
    int ex = 0;
    if (mx > 0.0) frexp(mx, &ex);        /* mx = f 2^ex, f in [0.5, 1): floor(log2 mx) = ex - 1 */
    e[i] = mx > 0.0 ? b - 1 - (ex - 1) : 0;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const int g = e[i] < e[j] ? e[i] : e[j];
      Ct[i * n + j] = ldexp(rint(ldexp(C[i * n + j], g)), -g);
    }
  free(e);
}

/* double-double helpers (Knuth two-sum, fma two-product; no contraction is involved: fma() is
 * called explicitly and is exact before its one rounding) */
typedef struct { double hi, lo; } orc_dd;
static orc_dd dd_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  orc_dd r = {s, (a - (s - bb)) + (b - bb)};
  return r;
}
static orc_dd dd_fast(double a, double b) {   /* |a| >= |b| */
  const double s = a + b;
  orc_dd r = {s, b - (s - a)};
  return r;
}
static orc_dd dd_add(orc_dd x, orc_dd y) {
  orc_dd s = dd_two_sum(x.hi, y.hi), t = dd_two_sum(x.lo, y.lo);
  s.lo += t.hi;
  s = dd_fast(s.hi, s.lo);
  s.lo += t.lo;
  return dd_fast(s.hi, s.lo);
}
static orc_dd dd_mul_d(orc_dd x, double y) {
  const double p = x.hi * y;
  double e = fma(x.hi, y, -p);
  e += x.lo * y;
  return dd_fast(p, e);
}

double orc_resid_dd(int64_t n, int p, const double *A, const double *X) {
  const int64_t nn = n * n;
  orc_dd *T = (orc_dd *)malloc((size_t)nn * sizeof(orc_dd));
  orc_dd *U = (orc_dd *)malloc((size_t)nn * sizeof(orc_dd));
  for (int64_t q = 0; q < nn; ++q) { T[q].hi = A[q]; T[q].lo = 0.0; }
  for (int j = 1; j <= p; ++j) {       /* T_j = X T_{j-1} (reading R-1's right-to-left chain) */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      orc_dd *u = U + i * n;
      for (int64_t c = 0; c < n; ++c) { u[c].hi = 0.0; u[c].lo = 0.0; }
      for (int64_t k = 0; k < n; ++k) {
        const double x = X[i * n + k];
        const orc_dd *t = T + k * n;
        for (int64_t c = 0; c < n; ++c) u[c] = dd_add(u[c], dd_mul_d(t[c], x));
      }
    }
    orc_dd *w = T; T = U; U = w;
  }
  orc_dd ss = {0.0, 0.0};
  for (int64_t i = 0; i < n; ++i)
    for (int64_t c = 0; c < n; ++c) {
      orc_dd r = {i == c ? 1.0 : 0.0, 0.0};
      orc_dd t = T[i * n + c];
      t.hi = -t.hi; t.lo = -t.lo;
      r = dd_add(r, t);                /* R_ic = delta_ic - T_p[i][c] */
      const double v = r.hi + r.lo;
      orc_dd sq = {v * v, fma(v, v, -(v * v))};
      ss = dd_add(ss, sq);
    }
  free(T); free(U);
  return sqrt(ss.hi + ss.lo);
}

void orc_resid_rows_dd(int64_t n, int p, const double *A, const double *X, int64_t nrows, const int64_t *rows,
                       double *out) {
  orc_dd *v = (orc_dd *)malloc((size_t)n * sizeof(orc_dd));
  orc_dd *u = (orc_dd *)malloc((size_t)n * sizeof(orc_dd));
  for (int64_t q = 0; q < nrows; ++q) {
    const int64_t i = rows[q];
    for (int64_t c = 0; c < n; ++c) { v[c].hi = X[i * n + c]; v[c].lo = 0.0; }   /* x_i^T */
    for (int j = 1; j <= p; ++j) {     /* v <- v X (p - 1 times), then v <- v A */
      const double *M = j < p ? X : A;
      #pragma omp parallel for schedule(static)
      for (int64_t c = 0; c < n; ++c) {
        orc_dd acc = {0.0, 0.0};
        for (int64_t k = 0; k < n; ++k) acc = dd_add(acc, dd_mul_d(v[k], M[k * n + c]));
        u[c] = acc;
      }
      orc_dd *w = v; v = u; u = w;
    }
    orc_dd ss = {0.0, 0.0};
    for (int64_t c = 0; c < n; ++c) {
      orc_dd r = {c == i ? 1.0 : 0.0, 0.0};
      orc_dd t = v[c];
      t.hi = -t.hi; t.lo = -t.lo;
      r = dd_add(r, t);
      const double e = r.hi + r.lo;
      orc_dd sq = {e * e, fma(e, e, -(e * e))};
      ss = dd_add(ss, sq);
    }
    out[q] = ss.hi + ss.lo;
  }
  free(v); free(u);
}
