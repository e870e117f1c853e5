/*
 * ipr.h -- C-ABI of the B200-native (sm_100a) inverse matrix p-th root library.
 *
 * The library computes A^{-1/p} for a symmetric positive definite A with the iteration of
 * Bini et al. studied in arXiv:1703.02283:
 *
 *   Eq. (1)  PAPER.md:71-73  [Sec. 2]   C_{k+1} = ((p+1) C_k - C_k^{p+1} A) / p
 *   Eq. (3)  PAPER.md:84-86  [Sec. 2]   C_0 = (||A||_1 ||A||_inf)^{-1} A^T
 *   Eq. (2)  PAPER.md:76-79  [Sec. 2]   ||I - C_0^p A||_2 < 1  =>  C_k -> A^{-1/p}
 *
 * running "approximate" (reduced precision) phases first -- approximate arithmetic
 * (Sec. 3.1) and approximate storage / data exchange (PAPER.md:129-141,
 * Sec. 3.2) -- and switching to higher precision at runtime (dynamic precision scaling,
 * PAPER.md:256-261, Sec. 4.3.1), ending with FP64 refinement.
 *
 * Readings of passages the paper leaves open (product order, update form, rounding,
 * controller rules, forms, emulated FP64, certificates ...) are numbered R-1 ... R-32 in DESIGN.md and cited below.
 *
 * General conventions
 *  - Every function returns ipr_status (IPR_OK == 0).  No function aborts the process and
 *    there is NO CPU fallback: anything the GPU path cannot do returns IPR_E_UNSUPPORTED.
 *  - Numerical failure is NOT an error: it is reported as an ipr_outcome (IPR_DIVERGED,
 *    IPR_NONFINITE) with status IPR_OK.  Misuse (bad arguments, wrong call order,
 *    non-symmetric A) is an error status.
 *  - Matrices at the boundary are FP64, row-major, with a leading dimension (elements) >= n, on
 *    the device (or, for ipr_init's A and ipr_finalize's / ipr_set_output's C, in host memory).
 *    The caller owns them.  The library owns every internal buffer.
 *  - One context per host thread; contexts are independent.  All device work is enqueued
 *    on the caller's stream; ipr_iterate/ipr_residual/ipr_finalize synchronise it.
 *  - ipr_last_error(NULL) returns the message of the last failed call on this thread.
 */
#ifndef IPR_H
#define IPR_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct ipr_ctx ipr_ctx;

typedef enum {
  IPR_OK = 0,
  IPR_E_INVALID_ARG = 1,   /* null pointer, n <= 0, lda < n, bad p / schedule ...            */
  IPR_E_NOT_SYMMETRIC = 2, /* A != A^T bit for bit (reading R-13)                            */
  IPR_E_STATE = 3,         /* wrong call order (e.g. iterate before set_schedule)            */
  IPR_E_UNSUPPORTED = 4,   /* combination the GPU path does not implement (never CPU)       */
  IPR_E_OOM = 5,           /* device allocation failed                                       */
  IPR_E_CUDA = 6,          /* CUDA runtime / driver error (message in ipr_last_error)        */
  IPR_E_NCCL = 7           /* NCCL error or NCCL library not loadable                        */
} ipr_status;

/* GEMM input (operand) format of a phase.  Accumulation is FP32 for BF16/FP16/TF32/FP8
 * (tcgen05 tensor cores, kind::f16 / kind::tf32 / kind::f8f6f4), exact INT32 for INT8
 * (kind::i8) and FP64 for FP64 (DMMA).
 * Scaled formats carry a per-tensor power-of-two scale 2^sigma chosen from max|X| (reading R-20;
 * every product is unscaled exactly in FP64):
 *   IPR_FP16  e5m10,  scaled max in [2^14, 2^15)
 *   IPR_FP8   E4M3 (PAPER.md:263-267 finds 2 stored mantissa bits still
 *             converge in storage-only mode), scaled max in [2^6, 2^7), one RNE rounding
 *   IPR_INT8  8-bit fixed point q = sat_127(rint(2^sigma x)), scaled max in [2^6, 2^7) -- the
 *             tensor-core analogue of the paper's fixed-point storage.
 *
 * IPR_FP64_OZ: an FP64 phase (FP64 operands and storage, m <= 52) whose GEMMs run on the INT8
 *             tensor cores by the Ozaki scheme I (reading R-23): 9 signed 7-bit digits per element
 *             relative to its row / column maximum, the 45 digit products with s + t <= 10 as 9
 *             K-concatenated kind::i8 GEMMs (exact INT32), combined in FP64.  Accuracy at the FP64
 *             GEMM level (not bit-identical to DMMA).  Symmetric forms only, world = 1.
 * IPR_FP64_CRT: the same FP64 phase with its GEMMs on the INT8 tensor cores by the Ozaki scheme II
 *             (reading R-28): rows / columns quantised to b-bit integers relative to their maximum
 *             (b = 7 S - 4 for the phase's digit count S -- the stored bits of the R-26 rule -- capped at
 *             62 and at what 18 moduli allow at n), the integer product computed exactly modulo N pairwise
 *             coprime moduli <= 256 (one kind::i8 GEMM each; N = 17 at b = 59, n = 8192) and rebuilt by
 *             the Chinese remainder theorem in exact sliced FP64 arithmetic.  Error: the quantisation
 *             (2^-b relative to the row / column maximum; the reconstruction adds <= ~0.06 of that).
 *             Symmetric forms only, any 1 x world grid, n <= 65535. */
typedef enum { IPR_FP64 = 0, IPR_TF32 = 1, IPR_BF16 = 2, IPR_FP16 = 3, IPR_FP8 = 4, IPR_INT8 = 5,
               IPR_FP64_OZ = 6, IPR_FP64_CRT = 7 } ipr_prec;

/* ipr_phase.mant_bits = IPR_MANT_ADAPTIVE (IPR_FP64_OZ / IPR_FP64_CRT phases only): dynamic precision inside the
 * phase (reading R-26, "the necessity of increased precision can be detected at
 * runtime").  Before the chain of C_k the engine picks the Ozaki digits from the residual it
 * expects for C_{k+1}: target = rho_hat_{k-1} q^2 (q = last in-phase contraction rho_{k-1} /
 * rho_{k-2} clamped to [1e-3, 1], 0.03 without history), S = clamp(ceil((log2(30 sqrt n) -
 * log2 target) / 7), 3, 9); C_{k+1} is stored with m = min(52, 7 S - 4) bits.  The first chain of a
 * run uses S = 9; a phase entry stores C with the bits of the digits its first chain will use. */
enum { IPR_MANT_ADAPTIVE = -2 };

/* Rounding of the stored iterate (reading R-7: RNE default; RTZ = "bit truncation",
 * PAPER.md:26).  Operand conversions are always round-to-nearest-even (hardware cvt.rn). */
typedef enum { IPR_RNE = 0, IPR_RTZ = 1 } ipr_round;

typedef enum {
  IPR_RUNNING = 0,    /* ipr_iterate's max_iters budget ran out; call again to continue     */
  IPR_CONVERGED = 1,  /* rho <= final_tol in the last phase                                  */
  IPR_ITER_LIMIT = 2, /* last phase hit its max_iters                                        */
  IPR_DIVERGED = 3,   /* rho_hat > 10 * min rho_hat and rho_hat > 1 in the last phase (R-5)  */
  IPR_NONFINITE = 4   /* rho not finite in the last phase                                    */
} ipr_outcome;

/* Controller decisions recorded in the trace (reading R-5). */
typedef enum { IPR_DEC_CONTINUE = 0, IPR_DEC_CONVERGED = 1, IPR_DEC_ITER_LIMIT = 2,
               IPR_DEC_DIVERGED = 3, IPR_DEC_NONFINITE = 4, IPR_DEC_SWITCH = 5 } ipr_decision;

/* One precision phase ("imprecise arithmetic for the majority of iterations and
 * then refining ... using precise arithmetic").  rho = ||I - C_k^p A||_F (absolute), rho_hat =
 * rho / sqrt(n).  A phase is left (reading R-5) when rho <= switch_tol, or when armed
 * (rho_hat < plateau_arm) and rho_k > plateau_ratio * rho_{k-1}, or on divergence /
 * non-finite rho, or after max_iters chains; the next phase restarts from the best iterate. */
typedef struct {
  ipr_prec  prec;          /* operand format of the p+1 GEMMs                                */
  int       mant_bits;     /* m: stored mantissa bits of C and A (R-8 container: e8 for      */
                           /* BF16/FP16/TF32 phases, m <= 23; e11 for FP64, m <= 52); -1 =   */
                           /* the operand format's own (3 FP8, 7 BF16/INT8, 10 FP16/TF32,    */
                           /* 52 FP64)                                                        */
  ipr_round round;         /* rounding of stored C and A                                     */
  double    switch_tol;    /* 0 = off                                                         */
  double    plateau_ratio; /* 0 = off (typ. 0.7)                                              */
  double    plateau_arm;   /* typ. 0.5                                                        */
  int       max_iters;     /* per-phase cap on chains; 0 = unlimited                          */
  int       corr_prec;     /* IPR_FORM_SYMMETRIC only: ipr_prec of the correction GEMM        */
                           /* W = qc(C) qc(I - C^{p-1}AC); -1 = prec (BF16 for the scaled     */
                           /* FP16/FP8/INT8 phases).  Must be BF16, TF32 or FP64 (FP64     */
                           /* only in FP64 phases), or the phase's own scaled format (FP16 /  */
                           /* FP8 / INT8 = prec: R-29, R and C scaled by powers of two, W     */
                           /* unscaled exactly; else IPR_E_UNSUPPORTED at ipr_iterate).       */
                           /* A BF16/TF32 correction in an FP64 phase                         */
                           /* is mixed-precision refinement: R is small, so W needs only      */
                           /* relative accuracy (R-22).  Ignored by other forms.    */
} ipr_phase;

/* Trace record: one per evaluated iterate C_k (one chain of p GEMMs, or -- reading R-33 -- only the
 * FP64 certificate of an iterate predicted to converge, when that certificate passed). */
typedef struct {
  int    k;          /* record index (0-based)                                               */
  int    phase;      /* schedule index of the phase that evaluated C_k                       */
  int    prec;       /* ipr_prec of that phase                                               */
  int    mant_bits;  /* effective m of that phase                                            */
  int    decision;   /* ipr_decision taken after this residual                               */
  double rho;        /* in-chain ||I - C_k^p A||_F (reading R-4); NaN for a certificate-only */
                     /* record (R-33: rho_cert holds the FP64 residual, decision CONVERGED)    */
  double rho_hat;    /* rho / sqrt(n)                                                        */
  double delta;      /* ||C_{k+1} - C_k||_F of the update that followed (NaN if none)        */
  double gemm_ms;    /* device time of this record's GEMMs (chain + update), CUDA events     */
  double upd_ms;     /* the part of gemm_ms spent in the update (GEMM p+1 + its epilogue /    */
                     /* k_sym_update); gemm_ms - upd_ms = the chain's p GEMMs                  */
  int    digits;     /* IPR_FP64_OZ / _CRT: Ozaki digits S of this record's chain (OZ: S(S+1)/2 */
                     /* INT8 digit products per FP64 product; CRT: b = 7 S - 4 bits); else 0     */
  double rho_cert;   /* symmetric / coupled forms: ||I - C_k^p A||_F recomputed in FP64 when  */
                     /* the in-chain rho met final_tol, or before the chain when the last    */
                     /* phase's rate predicted it (R-33); converged iff rho_cert <= final_tol;*/
                     /* NaN otherwise                                                         */
  int    moduli;     /* IPR_FP64_CRT: CRT moduli of this record's chain (INT8 GEMMs per FP64   */
                     /* product); 0 otherwise                                                  */
  int    ztri;       /* IPR_FORM_SYMMETRIC_TRIZ: 1 if this record's chain took Z_1 from its upper  */
                     /* tiles (reading R-37: 2 n^2 (n + 1) instead of 2 n^3 + n^2 (n + 1) ops per    */
                     /* modulus); 0 otherwise (fills the padding after moduli: the layout is unchanged) */
  double kern_ms;    /* IPR_FP64_CRT: device time of the chain's kind::i8 modulus GEMM launches  */
                     /* alone (CUDA events; the residue splits and the CRT reconstruction are   */
                     /* the rest of gemm_ms - upd_ms); 0 otherwise                              */
  double gap_ms;     /* device time between this chain's residual being ready and its update's   */
                     /* first kernel: the host round trip of the controller (decision + enqueue)  */
                     /* the GPU waits for (CUDA events); NaN when no update followed            */
} ipr_record;

/* Create a context for an n x n SPD matrix A (FP64, row-major, leading dimension lda >= n).  A on the
 * device is borrowed read-only until ipr_finalize; A in host memory (pinned for full link speed, or
 * pageable) is copied once into a library-owned device copy on cuda_stream (the caller may reuse it
 * after this call returns).  Checks exact symmetry (IPR_E_NOT_
 * SYMMETRIC otherwise), computes ||A||_1, ||A||_inf and max diagonal on the GPU (Eq. 3) and
 * records a warning (ipr_last_error) if the sufficient condition of reading R-12 for Eq. (2)
 * fails; that never fails init.
 * Multi-GPU: world > 1 ranks, one process per GPU, each passing
 * the FULL A; nccl_unique_id = 128 bytes from ipr_nccl_unique_id on rank 0 broadcast by the caller.
 * grid_rows x grid_cols must equal world (else IPR_E_INVALID_ARG):
 *   1 x world (default): column panels -- every form and format except IPR_FP64_OZ;
 *   P_r x P_c, P_r > 1: 2-D blocks, rank = r * P_c + c owns rows [r n/P_r, ...) x columns [c n/P_c, ...)
 *     (padded); the literal form with FP64 / TF32 / BF16 phases (else IPR_E_UNSUPPORTED at ipr_iterate),
 *     needs ncclCommSplit (NCCL >= 2.18).
 * Every decomposition reproduces world = 1 bit for bit (same tiles, same K order, partials reduced in the
 * same global order).  world == 1: nccl_unique_id may be NULL, grid 1 x 1.  cuda_stream: cudaStream_t
 * (NULL ok). */
ipr_status ipr_init(ipr_ctx **out, int64_t n, const double *A_dev, int64_t lda,
                    void *cuda_stream, int world, int rank, const void *nccl_unique_id,
                    int grid_rows, int grid_cols);

/* Root order p >= 1 and 1..16 phases; the precision (operand mantissa bits,
 * then m) must be non-decreasing along the schedule.  final_tol >= 0: stop when rho <=
 * final_tol in the last phase.  May be called again only before the first ipr_iterate. */
ipr_status ipr_set_schedule(ipr_ctx *c, int p, const ipr_phase *phases, int nphases,
                            double final_tol);

/* Iteration form.  IPR_FORM_LITERAL (default): Eq. (1) as printed, evaluated as
 * the right-to-left chain of reading R-1.  IPR_FORM_NEWTON_SCHULZ: p = 1 only, the textbook
 * Newton-Schulz ordering X_{k+1} = X_k (2I - A X_k) that PAPER.md:79-81 names (SURVEY 8(f)
 * NEXT-1): two GEMMs per iteration, T = Ahat Xhat with the fused residual ||I - T||_F and
 * What = qin(2I - T), then X_{k+1} = q_m(Xhat What).  Its error is quadratic in the deviation
 * (no linear term), so low-precision noise is removed by the FP64 phase.  Call before the
 * first ipr_iterate; a p != 1 schedule with this form fails at ipr_iterate (INVALID_ARG).
 *
 * IPR_FORM_SYMMETRIC (p >= 2; BF16/TF32/FP64 phases): the Newton correction
 * of Eq. (1) (C_{k+1} = C_k + C_k (I - C_k^p A) / p) with the residual taken as
 * R = I - C^{p-1} A C and the correction symmetrised (reading R-22):
 *   Z_1 = Ahat Chat, Z_j = Chat qin(Z_{j-1}) (j = 2..p), rho_s = ||I - Z_p||_F (fused),
 *   Rhat = qc(I - Z_p);  W = qc(C) Rhat;  C_{k+1} = q_m(C + (W + W^T) / (2p)).
 * C_k stays exactly symmetric; at the fixed point the error multiplier is
 * mu_ij = 1 - (x_i g_ij + x_j g_ji)/(2p) (|mu| <= 0.03 at kappa = 2, < 1 up to kappa ~ 34 for
 * p = 2), so low-precision noise is damped in the FP64 phase instead of persisting.
 * The trace's rho is rho_s; when it meets final_tol in the last phase the engine certifies
 * ||I - C_k^p A||_F (record.rho_cert, see ipr_set_cert; by default on the FP64 DMMA pipe -- exactly
 * the computation of ipr_residual(certify = 1)): converged iff that is <=
 * final_tol, and the certified C_k is the answer ipr_finalize returns; else the iteration continues
 * from C_{k+1}.
 *
 * IPR_FORM_SYMMETRIC_TRI (p = 2, 1 x world grids): as IPR_FORM_SYMMETRIC, but
 * Z_2 = C A C -- symmetric in exact arithmetic -- is computed on the upper triangle only (tiles
 * wholly below the diagonal are skipped: ~1/2 of GEMM 2) and R_ij = delta_ij - Z_2[min(i,j)][max(i,j)]
 * is exactly symmetric; rho_s sums the off-diagonal terms twice.  G > 1: each rank computes the upper
 * tiles of its own columns, the mirrors reach their owners by one all-to-all.  In phases below the FP64
 * range (FP8 / INT8 / FP16 / BF16 / TF32; reading R-36) both symmetric forms compute every chain
 * product and W on their upper tiles: each Z_j := the mirror of its upper triangle and the correction
 * S_ij = 2 W_{min(i,j),max(i,j)} (they differ from the full products by commutators at those phases' own
 * rounding level); FP64-range phases keep the full products and W + W^T.
 *
 * IPR_FORM_SYMMETRIC_TRIZ (reading R-37; p = 2): IPR_FORM_SYMMETRIC_TRI, and in an IPR_FP64_CRT phase
 * Z_1 = Ahat Chat is taken from its upper tiles too (mirrored; 2/3 of the chain's modulus GEMM work) from the
 * third chain of the phase on, while every in-phase ratio rho_k / rho_{k-1} so far was <= 0.1.  One slower step
 * switches the rule off for the rest of the phase (the full Z_1 of IPR_FORM_SYMMETRIC_TRI): on slowly
 * contracting inputs (kappa >~ 5 in the BASELINE family) the two forms run the same trajectory.  The
 * certificate (ipr_set_cert) does not depend on how the iterate was produced.
 *
 * IPR_FORM_COUPLED (any p; FP64 / TF32 / BF16 phases): the M-carrying form
 * of Eq. (1) (reading R-27): with M = X^p A and N = ((p+1) I - M) / p, X_{k+1} = X_k N_k
 * and M_{k+1} = N_k^p M_k -- p + 1 GEMMs per iteration (X Nhat; Nhat Mhat; Nhat qin(T)...).  The last
 * GEMM of each M chain stores Mhat = qin(q_m(M)) and Nhat = qin(((p+1)I - q_m(M))/p) and the
 * residual rho = ||I - M||_F; every phase start re-anchors M = X^p A with the literal chain.
 * Bounded after convergence for any kappa (it does not remove noise earlier phases left in X);
 * convergence is certified on ||I - X^p A||_F like the symmetric forms. */
typedef enum { IPR_FORM_LITERAL = 0, IPR_FORM_NEWTON_SCHULZ = 1, IPR_FORM_SYMMETRIC = 2,
               IPR_FORM_SYMMETRIC_TRI = 3, IPR_FORM_COUPLED = 4, IPR_FORM_SYMMETRIC_TRIZ = 5 } ipr_form;
ipr_status ipr_set_form(ipr_ctx *c, int form);

/* Convergence certificate of the symmetric and coupled forms, whose in-chain residual is not the
 * north-star residual ||I - C^p A||_F (reading R-3; R-30).  Call before the first ipr_iterate.
 *  IPR_CERT_FP64 (default): ||I - C_k^p A||_F of the candidate C_k on the FP64 DMMA pipe
 *    (deterministic): p = 2 as ||I - Y A||_F with Y = C C computed on its upper tiles and mirrored
 *    (C and so Y are bitwise symmetric; 1.5 GEMMs; R-32), other p by the literal chain
 *    T_1 = C A, T_j = C T_{j-1} (p GEMMs) -- the same function that
 *    ipr_residual(certify = 1) runs on the returned iterate -- so for a converged solve the two agree
 *    bit for bit, and "converged" means that FP64 residual is <= final_tol.
 *  IPR_CERT_PHASE: the same residual from the FP64-range phase's own product (IPR_FP64_CRT / _OZ: the
 *    INT8-emulated GEMM, reusing Z_1 = A C of the chain: p - 1 products instead of p DMMA GEMMs).  An
 *    ESTIMATE: it is more accurate than the DMMA evaluation (exact integer sums, 2^-b quantisation) but
 *    a different rounding, so ipr_residual(certify = 1) may exceed final_tol for a solve it accepted
 *    (measured: 9.72e-13 accepted, DMMA 1.004e-12, n = 4096, kappa = 5).  Diagnostics only.
 *  IPR_FP64 triggers the certificate of the symmetric forms in two ways (R-33): when the
 *    in-chain rho_s of C_k meets final_tol, and -- after an update in the last phase -- when the phase's
 *    linear rate predicts it, rho_k (rho_k / rho_{k-1}) <= final_tol / 2: then C_{k+1} is certified
 *    BEFORE its chain, which runs only if the certificate misses (the converged record then has
 *    rho = NaN).  IPR_CERT_FP64_CHAIN: the same certificate, triggered by the in-chain rho only.
 *  IPR_CERT_CRT (reading R-35; symmetric forms, p = 2 on 1 x G grids or p = 3 on one GPU, an IPR_FP64_CRT
 *    phase, FP64 last phase):
 *    a PROVEN upper bound on ||I - Ct^2 A||_F, where Ct is the candidate C_k rounded to the coarser of its
 *    row's and its column's 62-bit grids (|Ct - C_k| <= 2^-62 of the row / column maximum; the rounding
 *    makes Ct's integer quantisation exact), from exact integer products on the INT8 tensor cores
 *    (Y = Ct Ct on its upper tiles, then Y A; 1.5 x 18 modulus GEMMs; p = 3: Y, T = Ct Y, T A) plus the quantisation and
 *    reconstruction errors bounded a posteriori (||A||_2 <= ||A||_1, ||Y||_2 <= ||Y||_inf).  Converged
 *    means that bound is <= final_tol, and Ct is the answer (it replaces C_k; ipr_set_output streams Ct).
 *    Triggered like IPR_CERT_FP64 (R-33).  An FP64 DMMA evaluation carries ~n u |C|^2 |A| of rounding
 *    noise (4-6e-13 at n = 8192); this bound is a statement about the exact residual.  Candidates whose
 *    exponents leave (-400, 400) or that are not bitwise symmetric fall back to IPR_CERT_FP64's DMMA
 *    evaluation of Ct.  G > 1: every rank rounds and splits the gathered candidate, computes its column
 *    panel of Y (stored K-major: the rows S_g of the symmetric Y) and of Y A, and all-gathers Y's residue
 *    planes and row statistics -- the bound is bit-identical to G = 1.  Unsupported configurations fail at
 *    the first ipr_iterate (IPR_E_UNSUPPORTED).
 * Errors: IPR_E_INVALID_ARG (unknown mode), IPR_E_STATE (after the first ipr_iterate). */
typedef enum { IPR_CERT_FP64 = 0, IPR_CERT_PHASE = 1, IPR_CERT_FP64_CHAIN = 2, IPR_CERT_CRT = 3 } ipr_cert;
ipr_status ipr_set_cert(ipr_ctx *c, int mode);

/* Run at most max_iters (> 0) chains.  *iters_done = chains evaluated by this call,
 * *outcome = IPR_RUNNING if the budget ran out, else the terminal outcome.  Resumable. */
ipr_status ipr_iterate(ipr_ctx *c, int max_iters, int *iters_done, ipr_outcome *outcome);

/* certify == 0: the in-chain residual of the latest evaluated iterate (reading R-4).
 * certify == 1: ||I - C_best^p A||_F recomputed (IPR_CERT_FP64: with FP64 DMMA GEMMs) from the best iterate (the one
 * ipr_finalize returns), the last GEMM keeping only its residual partials (reading R-3) -- the
 * form's own FP64 certificate, bit for bit: the literal form's FP64 chain C (C A) (its in-chain
 * rho), the symmetric / coupled forms' IPR_CERT_FP64 ((C C) A for p = 2, R-32) -- or, with IPR_CERT_CRT,
 * that certificate's bound for Ct = the grid rounding of C_best (= C_best for a CRT-certified answer).
 * certify == 2: the FP64 DMMA evaluation of C_best whatever the certificate mode. */
ipr_status ipr_residual(ipr_ctx *c, int certify, double *rho);

/* Copy up to cap trace records; *count = total records so far (may exceed cap). */
ipr_status ipr_get_trace(ipr_ctx *c, ipr_record *buf, int cap, int *count);

/* Copy an iterate (FP64) to a caller device buffer: which = 0 the current C_k (the iterate
 * the next chain evaluates), which = 1 the best iterate (minimum rho, reading R-17). */
ipr_status ipr_get_iterate(ipr_ctx *c, int which, double *C_dev_out, int64_t ldc);

/* s = ||A||_1 * ||A||_inf and the norms: out4 = {||A||_1, ||A||_inf, max diag, s}. */
ipr_status ipr_get_norms(ipr_ctx *c, double *out4);

/* Optional: the destination the caller will pass to ipr_finalize (host -- pinned for full speed -- or
 * device, row-major, ldc >= n; NULL clears).  With world = 1 the engine then streams every candidate it
 * certifies in an FP64-range phase to C_out on a copy stream while the FP64 certificate runs; when the
 * solve converges on that candidate, ipr_finalize(c, C_out, ldc) only waits for the copy.  C_out is
 * written during ipr_iterate (possibly with a candidate that later misses): its content is defined only
 * after ipr_finalize.  Errors: IPR_E_INVALID_ARG. */
ipr_status ipr_set_output(ipr_ctx *c, double *C_out, int64_t ldc);

/* Write the best iterate (FP64, full matrix on every rank) to C_dev_out (device or host memory,
 * ldc >= n; may be NULL to discard) and free the context (also on error). */
ipr_status ipr_finalize(ipr_ctx *c, double *C_dev_out, int64_t ldc);

/* Message of the last failure (or init warning) of c; c == NULL: this thread's last. */
const char *ipr_last_error(const ipr_ctx *c);

/* Rank-0 bootstrap helper: 128-byte NCCL unique id (NCCL loaded with dlopen). */
ipr_status ipr_nccl_unique_id(void *out128);

/* Library version string. */
const char *ipr_version(void);

#ifdef __cplusplus
}
#endif
#endif
