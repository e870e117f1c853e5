// kernels.h -- host launchers of the HBM-bound kernels (kernels.cu).  Internal to libipr.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ipr {
cudaError_t launch_symcheck(const double *A, int64_t lda, int64_t n, int *flag, cudaStream_t s);
cudaError_t launch_norms(const double *A, int64_t lda, int64_t n, double *colsum, double *out3, cudaStream_t s);
cudaError_t launch_maxabs_qA(const double *A, int64_t lda, int64_t n, int cont64, int m, int rtz, float *pmax,
                             int nparts, cudaStream_t s);
cudaError_t launch_stage_a(const double *A, int64_t lda, int64_t n, int64_t npad, int64_t col0, int64_t kp, int prec,
                           int cont64, int m, int rtz, const int *sig, void *Aop, cudaStream_t s);
cudaError_t launch_c0(const double *A, int64_t lda, int64_t n, int64_t rows, int64_t row0, int64_t col0, int64_t kp,
                      double sv, int cont64, int m, int rtz, void *cont, cudaStream_t s);
cudaError_t launch_make_operand(const void *cont, int cont64, int64_t count, int prec, const int *sig, void *op,
                                cudaStream_t s);
cudaError_t launch_scale_op(const float *src, int64_t count, const int *sig, int prec, void *dst, cudaStream_t s);
cudaError_t launch_maxabs_cont(const void *cont, int cont64, int64_t count, float *pmax, int nparts, cudaStream_t s);
cudaError_t launch_mirror_unpack(const void *recv, int esz, int64_t kp, int64_t npad, int rank, int world, void *T,
                                 cudaStream_t s);
cudaError_t launch_select_partials(const double *partg, int64_t total, int64_t tiles_m, int tmsz, int tnsz, int64_t mr,
                                   int64_t kp, int gcols, double *part, cudaStream_t s);
cudaError_t launch_copy_out_blocks(const double *src, int64_t mr, int64_t kp, int gcols, int64_t n, double *dst,
                                   int64_t ldc, cudaStream_t s);
cudaError_t launch_peek(const void *src, int prec, const int *sig, int64_t count, double *dst, cudaStream_t s);
cudaError_t launch_cont_to_f64(const void *cont, int cont64, int64_t count, double *dst, cudaStream_t s);
cudaError_t launch_f64_to_cont(const double *src, int64_t count, int cont64, int m, int rtz, void *cont,
                               cudaStream_t s);
cudaError_t launch_reduce_sum(const double *part, int64_t count, double *out, cudaStream_t s);
cudaError_t launch_reduce_max(const float *part, int64_t count, double *out, int *sig, int prec, cudaStream_t s);
cudaError_t launch_copy_out(const double *src, int64_t npad, int64_t kp, int64_t n, double *dst, int64_t ldc,
                            cudaStream_t s);
cudaError_t launch_pad_copy(const void *src, int64_t n, int64_t npad, int esz, void *dst, cudaStream_t s);
cudaError_t launch_unpad_f64(const double *src, int64_t n, int64_t npad, double *dst, cudaStream_t s);
cudaError_t launch_transpose(const void *src, int64_t rows, int64_t cols, int esz, void *dst, cudaStream_t s);
// amax (nullable): atomicMax of the bits of max |C_{k+1}| (as float) -- the caller zeroes it first
cudaError_t launch_sym_update(const void *cold, int cont64, void *cnew, const void *W, int w64, int64_t npad,
                              int64_t kp, int64_t col0, int p, int m, int rtz, int prec, void *chat_new, int corr,
                              void *chat_corr_new, double *part, unsigned *amax, int wtri, cudaStream_t s);
cudaError_t launch_oz_split(const double *X, int64_t ld, int64_t rows, int64_t cols, int S, int8_t *planes,
                            int8_t *bcat, int *sig, cudaStream_t s);
cudaError_t launch_crt_split(const double *X, int64_t ld, int64_t rows, int64_t cols, int b, int nm, int8_t *planes,
                             int *sig, cudaStream_t s);
// the CRT certificate (reading R-35, ozaki.cu)
cudaError_t launch_cert_rowexp(const double *X, int64_t ld, int64_t rows, int64_t cols, int b, int *sig, double *scale,
                               cudaStream_t s);
// Xin: the candidate (row-major, ld), X: where Ct goes (may equal Xin); asum: row abs sums of Ct (nullable)
cudaError_t launch_cert_round_split(const double *Xin, double *X, int64_t ld, int64_t rows, int64_t cols, int nm,
                                    const int *sig, int8_t *planes, double *asum, cudaStream_t s);
// pstride: the residue plane stride (0: rows * cols); row r of X writes planes + l * pstride + r * cols
cudaError_t launch_cert_split(const double *Xh, const double *Xl, int64_t ld, int64_t rows, int64_t cols, int b, int nm,
                              int8_t *planes, int64_t pstride, int *sig, double *scale, double *err2, double *asum,
                              cudaStream_t s);
cudaError_t launch_cert_stats(const double *const *v, const int *op, int nv, int64_t len, double *out, cudaStream_t s);
cudaError_t launch_fill_operand(void *dst, int64_t count, int prec, uint32_t seed, cudaStream_t s);
cudaError_t launch_test_quant(int mode, const void *in, void *out, int64_t len, int m, int rtz, int sigma,
                              cudaStream_t s);
}  // namespace ipr
