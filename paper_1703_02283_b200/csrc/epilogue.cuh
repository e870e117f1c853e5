// epilogue.cuh -- the fused per-element epilogue shared by the FP64 (DMMA) and the tcgen05
// GEMM kernels.  Every GEMM of the hot path is D = Chat * X; what happens to D is:
//
//  EPI_STORE_T : T_j = D  ->  qin(T_j) stored transposed (K-major B operand of the next
//                GEMM, reading R-1: right-to-left chain T_j = Chat T_{j-1})
//  EPI_RESID   : partial of rho^2 = sum (delta_ij - T_p,ij)^2 from the unrounded accumulator
//                (the in-chain residual of reading R-4)
//  EPI_WSTORE  : W = D row-major (symmetric form, NEXT-2); the update C + (W + W^T)/(2p)
//                needs W^T, so it runs in k_sym_update (kernels.cu) after the GEMM
//  EPI_UPDATE  : C_{k+1} = q_m(((p+1) C_k - P) / p)  with P = D: three separately rounded FP64
//                operations and ONE rounding to m bits (reading R-2, Eq. (1) PAPER.md:71-73;
//                approximate storage PAPER.md:133-136), plus Chat_{k+1} = qin(C_{k+1}) and the
//                partial of delta^2 = sum (C_{k+1} - C_k)^2 ("changes introduced in each
//                iteration").
//
// __dmul_rn/__dsub_rn/__ddiv_rn are never contracted into FMAs, so the update is the exact
// IEEE sequence the oracle evaluates.
#pragma once
#include "common.cuh"

namespace ipr {

struct EpiAcc {
  double r2;    // residual partial
  double d2;    // delta partial
  float mx;     // max |.| partial
};

// v: accumulator value converted to FP64 (exact) and scaled (exact power of two).
// row: global row; col: local column (global = col0 + col).
// MODE >= 0: the epilogue mode is a compile-time constant (specialised kernels); -1: g.mode.
template <int MODE = -1>
__device__ __forceinline__ void epi_element(const GemmArgs &g, int64_t row, int64_t col,
                                            double v, EpiAcc &acc) {
  const int mode = MODE >= 0 ? MODE : g.mode;
  if (mode & EPI_STORE_N) store_operand(g.nout, row * g.ldn + col, g.tprec, v, 0);
  const bool mirror = g.tri && row != g.col0 + col;   // tri: (i,j), i < j, also stands for (j,i)
  if (g.tri && row > g.col0 + col) return;             // tri: lower triangle comes from the mirror
  if (mode & (EPI_STORE_T | EPI_TSCRATCH)) {
    double w = v;
    if (mode & EPI_DIAG_MINUS) {      // diag*I - D: NS What = 2I - A X, symmetric R = I - Z_p
      const int64_t gc = g.col0 + col;
      w = __dsub_rn((row == gc && row < g.n) ? g.diag : 0.0, v);
    }
    if (mode & EPI_STORE_T) {
      // FP16 T operands go through EPI_TSCRATCH + a scale kernel (sigma 0 here)
      store_operand(g.tout, col * g.ldt + row, g.tprec, w, 0);
      if (mirror) store_operand(g.mout, row * g.ldm + col, g.tprec, w, 0);
    } else {
      ((float *)g.tout)[col * g.ldt + row] = (float)w;
      acc.mx = fmaxf(acc.mx, fabsf((float)w));
    }
  }
  if (mode & EPI_NSUPDATE) {          // X_{k+1} = q_m(Xhat What): one rounding to m bits
    const int64_t ci = row * g.ldc + col;
    const double c = g.cont64 ? ((const double *)g.cold)[ci] : (double)((const float *)g.cold)[ci];
    double cn;
    if (g.cont64) {
      cn = q_e11(v, g.m, g.rtz);
      ((double *)g.cnew)[ci] = cn;
    } else {
      const float f = q_e8(v, g.m, g.rtz);
      ((float *)g.cnew)[ci] = f;
      cn = (double)f;
    }
    if (g.chat_new) {
      if (is_scaled(g.prec)) acc.mx = fmaxf(acc.mx, fabsf((float)cn));
      else store_operand(g.chat_new, row * g.ldh + col, g.prec, cn, 0);
    }
    const double dd = __dsub_rn(cn, c);
    acc.d2 = __fma_rn(dd, dd, acc.d2);
  }
  if (mode & EPI_COUPLED) {           // coupled form (R-27): M_{k+1} stored, N_{k+1} from it
    const int64_t gc = g.col0 + col;
    const double w = g.cont64 ? q_e11(v, g.m, g.rtz) : (double)q_e8(v, g.m, g.rtz);
    store_operand(g.tout, col * g.ldt + row, g.prec, w, 0);
    const double a = (row == gc && row < g.n) ? (double)(g.p + 1) : 0.0;
    const double d = __dsub_rn(a, w);
    const double e = ((g.p & (g.p - 1)) == 0) ? __dmul_rn(d, 1.0 / (double)g.p) : __ddiv_rn(d, (double)g.p);
    store_operand(g.nkout, col * g.ldt + row, g.prec, e, 0);
  }
  if (mode & EPI_RESID) {
    const int64_t gc = g.col0 + col;
    if (row < g.n && gc < g.n) {
      const double d = __dsub_rn(row == gc ? 1.0 : 0.0, v);
      acc.r2 = __fma_rn(mirror ? 2.0 * d : d, d, acc.r2);
    }
  }
  if (mode & EPI_UPDATE) {
    const int64_t ci = row * g.ldc + col;
    const double c = g.cont64 ? ((const double *)g.cold)[ci] : (double)((const float *)g.cold)[ci];
    const double a = __dmul_rn((double)(g.p + 1), c);
    const double d = __dsub_rn(a, v);
    // d / p; for p = 2^k the product with the exact reciprocal is the same IEEE result
    const double e = ((g.p & (g.p - 1)) == 0) ? __dmul_rn(d, 1.0 / (double)g.p) : __ddiv_rn(d, (double)g.p);
    double cn;
    if (g.cont64) {
      cn = q_e11(e, g.m, g.rtz);
      ((double *)g.cnew)[ci] = cn;
    } else {
      const float f = q_e8(e, g.m, g.rtz);
      ((float *)g.cnew)[ci] = f;
      cn = (double)f;
    }
    if (g.chat_new) {
      const int64_t hi = row * g.ldh + col;
      if (is_scaled(g.prec)) {
        // a scaled Chat is produced by a separate kernel once max|C_{k+1}| is known
        acc.mx = fmaxf(acc.mx, fabsf((float)cn));
      } else {
        store_operand(g.chat_new, hi, g.prec, cn, 0);
      }
    }
    const double dd = __dsub_rn(cn, c);
    acc.d2 = __fma_rn(dd, dd, acc.d2);
  }
  if (mode & EPI_F64) g.zout[row * g.ldz + col] = v;
  if (mode & EPI_WSTORE) {            // symmetric form: W = qc(C) Rhat, exact accumulator value
    if (g.w64) ((double *)g.wout)[row * g.ldw + col] = v;
    else ((float *)g.wout)[row * g.ldw + col] = (float)v;
  }
}

}  // namespace ipr
