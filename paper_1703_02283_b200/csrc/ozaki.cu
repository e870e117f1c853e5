// ozaki.cu -- FP64 GEMMs emulated on the INT8 tensor cores (tcgen05 kind::i8), Ozaki scheme I
// (reading R-23).  An FP64 phase whose format is P_FP64_OZ computes every product of
// the hot path this way instead of on the DMMA pipe:
//
//   split     x_ik = 2^sig_i * sum_{s=1..S} d_s,ik 2^-7s   (+ |rest| <= 2^(sig_i - 7S - 1))
//             per ROW of the left operand (sig_i from max_k |x_ik|) and per COLUMN of the right
//             operand; d_1 in [-127, 127], d_s in [-64, 64] (s >= 2), every step exact in FP64
//   products  P_g = sum_{s + t = g} D_s E_t  for g = 2 .. S+1: ONE int8 GEMM with the K-concatenated
//             operands [D_1 | ... | D_{g-1}] and [E_{g-1}; ...; E_1], exact in INT32:
//             |P_g| <= (2 * 127 * 64 + (S - 2) * 64 * 64) * n < 2^31 for n <= 47800 (S = 9)
//   combine   Z_ij = sum_g 2^(sig_i + tau_j - 7g) P_g,ij, in FP64, smallest groups first
//   finish    the hot path's FP64 epilogue (store / residual / update partials, epilogue.cuh) on Z
//
// An FP64_OZ phase storing m mantissa bits uses S = oz_digits(m) = ceil((m + 12) / 7) digits
// (clamped to 2..9): the arithmetic keeps ~12 bits more than the storage.
// S = 9 keeps 63 bits per operand relative to its row / column maximum; the dropped pairs
// (s + t > S + 1) and the digit remainder are below the FP64 GEMM's own rounding at the orders
// used here (measured in NumPy against 80-bit long double: Frobenius error 9e-16 vs 8.6e-15 for an
// FP64 GEMM at n = 512; tests/test_gpu_ozaki.py asserts "no worse than 2x DMMA" on the GPU).
// K-work: S(S+1)/2 = 45 int8 GEMMs of order n.
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace ipr {

// Digits of the rows of X (FP64, row-major, leading dimension ld): one block per row.
//   planes (A role, may be NULL): digit s of x_rk at planes[(s-1) * rows * cols + r * cols + k]
//   bcat   (B role, may be NULL): digit s of x_rk at bcat[r * S * cols + (S - s) * cols + k]
//   sig[r]: the row's scale exponent
__global__ void __launch_bounds__(256) k_oz_split(const double *__restrict__ X, int64_t ld, int64_t rows,
                                                  int64_t cols, int S, int8_t *planes, int8_t *bcat, int *sig) {
  __shared__ double red[8];
  const int64_t r = blockIdx.x;
  const double *x = X + r * ld;
  double mx = 0.0;
  for (int64_t k = threadIdx.x; k < cols; k += blockDim.x) mx = fmax(mx, fabs(x[k]));
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    red[0] = fmax(mx, red[0]);
  }
  __syncthreads();
  mx = red[0];
  // |x| 2^-sig * 128 <= 127: sig = floor(log2(mx * 128/127)) + 1 (0 for an all-zero row)
  const int sg = (mx > 0.0) ? ilogb(mx * (128.0 / 127.0)) + 1 : 0;
  if (threadIdx.x == 0) sig[r] = sg;
  const double sc = pow2(-sg);
  // 8 consecutive elements per thread: every digit plane gets one 8-byte store per thread
  // (cols is a multiple of 256, so k0 + 8 <= cols and the stores are 8-byte aligned)
  for (int64_t k0 = (int64_t)threadIdx.x * 8; k0 < cols; k0 += (int64_t)blockDim.x * 8) {
    double v[8];
    const double2 *xp = (const double2 *)(x + k0);
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 t = xp[u];
      v[2 * u] = __dmul_rn(t.x, sc);
      v[2 * u + 1] = __dmul_rn(t.y, sc);
    }
    for (int s = 1; s <= S; ++s) {
      uint64_t w = 0;
      #pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = __dmul_rn(v[u], 128.0);
        const double d = rint(v[u]);
        v[u] = __dsub_rn(v[u], d);
        w |= (uint64_t)(uint8_t)(int8_t)(int)d << (8 * u);
      }
      if (planes) *(uint64_t *)(planes + (int64_t)(s - 1) * rows * cols + r * cols + k0) = w;
      if (bcat) *(uint64_t *)(bcat + r * S * cols + (int64_t)(S - s) * cols + k0) = w;
    }
  }
}

cudaError_t launch_oz_split(const double *X, int64_t ld, int64_t rows, int64_t cols, int S, int8_t *planes,
                            int8_t *bcat, int *sig, cudaStream_t s) {
  if (S < 2 || S > OZ_S) return cudaErrorInvalidValue;
  k_oz_split<<<(unsigned)rows, 256, 0, s>>>(X, ld, rows, cols, S, planes, bcat, sig);
  ++g_launches;
  return cudaGetLastError();
}

// Z = X Y for a P_FP64_OZ GemmArgs: g.oz_a / g.oz_rsig hold the OZ_S digits of X (A role), g.oz_b /
// g.oz_csig those of Y (B role, per output column, layout stride OZ_S); the product keeps the
// digit pairs s + t <= g.oz_S + 1 (the leading g.oz_S digits of a 9-digit split ARE the g.oz_S-digit
// split).  One persistent kind::i8 launch per group g = S+1 .. 2 (K' = (g-1) npad over digit planes
// 1..g-1 and the B digits g-1..1), accumulating 2^(sig_i + tau_j - 7g) P_g in FP64 into g.ozacc
// (transposed); the group-2 launch applies the hot path's epilogue g.mode (store / residual partials
// / mirror) to the completed FP64 value (no separate finish pass).  Running all groups of a tile in
// one launch (oz_grouped = 1) keeps the accumulator in L2 but spreads the CTAs over every digit
// plane at once and measured slower (19.7 vs 16.6 ms at n = 8192).  G = 1: M = N = K = npad.
cudaError_t launch_gemm_ozaki(const GemmArgs &g, cudaStream_t s) {
  const int S = g.oz_S;
  if (!g.oz_a || !g.oz_b || !g.oz_rsig || !g.oz_csig || !g.ozacc || g.M != g.K || g.N != g.K || S < 2 || S > OZ_S)
    return cudaErrorInvalidValue;
  const int64_t np = g.K;
  GemmArgs q = g;
  q.prec = P_INT8;
  if (!is_f64(q.tprec) && q.tprec != P_BF16 && q.tprec != P_TF32) q.tprec = P_FP64;
  q.A = g.oz_a; q.a_kp = np; q.a_pstride = np * np;
  q.K = (int64_t)OZ_S * np;                      // map extents: all digit planes
  q.B = g.oz_b; q.ldb = (int64_t)OZ_S * np;
  q.oz_grouped = 2;                              // one launch per group, smallest contributions first
  q.sigA = nullptr; q.sigB = nullptr; q.pmax = nullptr;
  for (int gi = S + 1; gi >= 2; --gi) {
    q.oz_g = gi;
    cudaError_t e = launch_gemm_tc(q, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ipr
