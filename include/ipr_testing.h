/*
 * ipr_testing.h -- kernel-level entry points of libipr used by the parity tests.
 *
 * Same conventions as ipr.h (status codes, device pointers, no CPU fallback).  Each call
 * enqueues on `stream` (cudaStream_t, NULL = legacy default) and synchronises it before
 * returning, so the caller may read the outputs immediately.
 */
#ifndef IPR_TESTING_H
#define IPR_TESTING_H
#include <stdint.h>
#include "ipr.h"
#ifdef __cplusplus
extern "C" {
#endif

/* Device quantisers (approximate storage / operand formats, PAPER.md:191-194 and the format
 * footnotes PAPER.md:106-111; readings R-7, R-8, R-9, R-20):
 *   mode 0: FP64 in  -> FP32 out : q_m with e8 container (stored C/A of BF16/FP16/TF32 phases)
 *   mode 1: FP64 in  -> FP64 out : q_m with e11 container (stored C/A of FP64 phases)
 *   mode 2: FP32 in  -> BF16 out (uint16 bit patterns), round-to-nearest-even
 *   mode 3: FP32 in  -> FP32 out rounded to the TF32 grid (e8m10), round-to-nearest-even
 *   mode 4: FP32 in  -> FP16 out (uint16 bit patterns) of 2^sigma * x, RNE (R-20 scaling)
 *   mode 5: FP64 in  -> FP8 E4M3 out (uint8 bit patterns) of 2^sigma * x, one RNE rounding (NEXT-3)
 *   mode 6: FP64 in  -> INT8 out of sat_127(rint(2^sigma * x)) (fixed point, NEXT-3)
 *   mode 7: as mode 0, through the symmetric update's branch-free normal-range path + its fallback
 *   mode 8: as mode 1, likewise
 * m: stored mantissa bits (modes 0/1), round: ipr_round (modes 0/1).  len >= 0. */
ipr_status ipr_test_quantize(int mode, const void *in_dev, void *out_dev, int64_t len, int m,
                             int round, int sigma, void *stream);

/* One GEMM of the hot path with a plain FP64 store epilogue:  Z = X Y  (n x n).
 *   X  : row-major operand (element (i,k) at X[i*n + k])
 *   Yt : K-major operand   (element (k,j) of Y at Yt[j*n + k])
 *   Z  : FP64 row-major, the accumulator converted exactly (FP32 -> FP64 for tensor-core
 *        kinds).  Formats: prec = IPR_FP64 (double), IPR_TF32 (float on the TF32 grid),
 *        IPR_BF16 / IPR_FP16 (uint16 bit patterns), IPR_FP8 (E4M3 bytes, FP32 accumulate),
 *        IPR_INT8 (int8, exact INT32 accumulate).  Operands unscaled (sigma 0).
 *        n >= 1 (any n; ragged tiles handled). */
ipr_status ipr_test_gemm(int prec, int64_t n, const void *X_dev, const void *Yt_dev,
                         double *Z_dev, void *stream);
/* IPR_FP64_OZ / IPR_FP64_CRT products of ipr_test_gemm / ipr_bench_gemm use `digits` Ozaki digits
 * (OZ) or b = 7 digits - 4 bits (CRT, capped as in ipr.h); digits in [2, 9], default 9.  Process-wide. */
ipr_status ipr_test_set_digits(int digits);
/* IPR_FP64_CRT residue convention (process-wide): 0 (default) residues in [0, m) with u8 x u8 modulus
 * GEMMs while K 255^2 < 2^31 (K <= 33024), symmetric residues in [-128, 127] with s8 x s8 beyond;
 * 1 forces the symmetric convention at every K (tests of the large-K path at small sizes).  Set it
 * between solves / products only. */
ipr_status ipr_test_crt_signed(int on);
/* The NCCL transport's plumbing on one GPU (NCCL refuses two ranks on one device, so the multi-process
 * path cannot run here): dlopen and symbol binding, a 1-rank communicator from ipr_nccl_unique_id's
 * source, an in-place all-gather, the grouped send / recv all-to-all and ncclCommSplit, results checked
 * byte by byte.  IPR_E_NCCL (message in ipr_last_error) on any failure. */
ipr_status ipr_test_nccl_selftest(void);
/* The CRT constants of N moduli (1 <= N <= 18, host only, no GPU): out40[0..N-1] the moduli,
 * out40[20 + l] = inv_l = (M_N / m_l)^-1 mod m_l; dout64[3 l + 0..2] = H_l, L_l, R_l (W_l = M_N / m_l =
 * H_l 2^s1 + L_l 2^s2 + R_l, R_l rounded to FP64); dout64[54..56] = MH, ML, MR; dout64[57..58] =
 * 2^s1, 2^s2.  *n_for = the number of moduli a product with b bits at order n uses (-1: none);
 * *b_for = the bits b a phase with b Ozaki-equivalent digits S = b uses at order n (b = min(7 S - 4,
 * 62, what 18 moduli allow)) when 2 <= b <= 9, else 0. */
ipr_status ipr_test_crt_table(int N, int b, int64_t n, int *out40, double *dout64, int *n_for, int *b_for);

/* Throughput probe of the hot-path GEMM kernel of a format (measurement): allocates
 * two n x n operands (n rounded up to the tile: 256 tcgen05 / 128 DMMA) filled with pseudo-random
 * values on the format's grid, runs `warmup` untimed then `iters` timed launches of the chain GEMM
 * with the hot path's epilogue (qin(D) stored K-major; for the scaled FP16/FP8/INT8 formats the
 * FP32 scratch + per-tile max that precedes the operand scaling) on `stream`, and
 * writes the average device time per launch (CUDA events on `stream`) to *ms.  2 n^3 flop per
 * launch.  Frees everything before returning. */
ipr_status ipr_bench_gemm(int prec, int64_t n, int warmup, int iters, void *stream, double *ms);
/* Same with an explicit epilogue mode (diagnostics): epi = 0 the hot-path default above,
 * 1 none (accumulators read from TMEM / registers and dropped), 2 EPI_STORE_T, 3 EPI_TSCRATCH. */
ipr_status ipr_bench_gemm_epi(int prec, int64_t n, int warmup, int iters, int epi, void *stream, double *ms);

/* Host-side plan of the 1 x world column-panel decomposition; needs no GPU.
 * out8 = {npad (padded order), kp (columns per rank), col0 (first global column of `rank`),
 *         tile_m, tile_n (output tile of the GEMM kernel used for prec), tiles_m,
 *         tiles_n_total, first global partial slot of this rank = (col0 / tile_n) * tiles_m}.
 * Partial slot of output tile (tm, tn_global) = tn_global * tiles_m + tm, identical for
 * every world size, so per-tile partials reduce in the same order for any G. */
ipr_status ipr_plan(int64_t n, int world, int rank, int prec, int64_t *out8);

/* Read an intermediate of the last iteration of a symmetric-form context (test hook for the
 * full-size step parity of tests/test_gpu_fullsize.py: each stage of one step is checked on sampled
 * elements the oracle computes one by one from the previous stage's values).  After ipr_iterate has
 * evaluated C_k and computed C_{k+1} (outcome IPR_RUNNING), `what` selects:
 *   IPR_PEEK_AHAT   (0) Ahat of the phase, K-major [npad][npad] (element (k, j) at k + j npad)
 *   IPR_PEEK_CHAT   (1) Chat of C_k (the chain's operand), row-major [npad][npad]
 *   IPR_PEEK_Z1     (2) qin(Z_1) of C_k (the B operand of GEMM 2), K-major
 *   IPR_PEEK_RHAT   (3) Rhat = qc(I - Z_p) of C_k (the B operand of the W GEMM), K-major
 *   IPR_PEEK_W      (4) W = qc(C_k) Rhat as stored (FP32 / FP64), row-major
 *   IPR_PEEK_CHATC  (5) qc(C_k) (the correction GEMM's A operand; = Chat if the formats agree), row-major
 * The values are converted to FP64 and unscaled by the operand's 2^-sigma (exact); dst: npad^2 doubles
 * on the device, npad = *npad_out (zero padding beyond n).  G = 1, symmetric forms, non-Ozaki phases;
 * else IPR_E_UNSUPPORTED. */
enum { IPR_PEEK_AHAT = 0, IPR_PEEK_CHAT = 1, IPR_PEEK_Z1 = 2, IPR_PEEK_RHAT = 3, IPR_PEEK_W = 4, IPR_PEEK_CHATC = 5 };
ipr_status ipr_test_peek(ipr_ctx *c, int what, double *dst_dev, int64_t *npad_out);

/* In-process rank groups (SURVEY 8(e) on a one-GPU box).  A local group stands for `world` ranks that
 * live in ONE process on ONE device, each with its own context, CUDA stream and host thread: every
 * all-gather / all-to-all of the engine becomes stream-ordered device-to-device copies between the
 * ranks' buffers, fenced by CUDA events and host barriers (no kernel waits on another rank; the
 * column-panel arithmetic, layouts and exchanges are exactly those of the NCCL path).  Used by the
 * -m gpu tests to check that G = 2 / 4 ranks reproduce the G = 1 trajectory bit for bit (P11).
 * ipr_test_init_local is ipr_init with the group in place of the NCCL id: call it once per rank, each
 * from its own host thread (the exchanges block until every rank of the group arrives).  Destroy the
 * group after every context of it is finalized. */
typedef struct ipr_local_group ipr_local_group;
ipr_status ipr_test_local_group_create(int world, ipr_local_group **out);
ipr_status ipr_test_local_group_destroy(ipr_local_group *g);
ipr_status ipr_test_init_local(ipr_ctx **out, int64_t n, const double *A_dev, int64_t lda, void *cuda_stream,
                               ipr_local_group *group, int rank, int grid_rows, int grid_cols);

/* Guard bands (memory-safety check in place of compute-sanitizer, which this pool does not allow):
 * ipr_test_set_guards(1) makes every context allocated afterwards (process-wide, at its first
 * ipr_iterate) put a 4 KB band of a fixed byte pattern behind each of its arena buffers;
 * ipr_test_check_guards re-reads every band: *bad = index of the first altered band, -1 if all intact.
 * corrupt_first != 0 alters band 0 first (the test's positive control). */
ipr_status ipr_test_set_guards(int on);
ipr_status ipr_test_check_guards(ipr_ctx *c, int corrupt_first, int *bad);

/* Number of this process's kernel launches since load (all libipr kernels). */
int64_t ipr_launch_count(void);

/* The terms of the last IPR_CERT_CRT certificate of c (reading R-35; NaN before one ran):
 * out[0] the certified bound (record.rho_cert), [1] ||I - P||_F as evaluated from the exact product,
 * [2] beta (the bound's error terms), [3] ||Ytilde - Yh||_F, [4] ||Atilde - A||_F, [5] the ||A||_2 bound,
 * [6] the ||Y||_2 bound, [7] eY, [8] eP (reconstruction bounds), [9] moduli.  out has 10 slots. */
ipr_status ipr_test_cert_info(ipr_ctx *c, double *out10);

#ifdef __cplusplus
}
#endif
#endif
