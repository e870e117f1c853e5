// common.cuh -- shared device helpers of libipr (CUDA path only; shares no code with the oracle).
//
// Quantisers written at the bit level (the oracle uses an independent frexp/ldexp
// definition).  Citations: PAPER.md:191-194 [Sec. 4.2] custom exponent/mantissa widths;
// PAPER.md:106-111 format footnotes; readings R-7 (RNE default, RTZ option), R-8 (container
// e8 for BF16/FP16/TF32 phases, e11 for FP64 phases, subnormals kept), R-9 (operands take the
// MMA input format), R-20 (FP16 operands scaled by 2^sigma) -- see DESIGN.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

namespace ipr {

enum Prec { P_FP64 = 0, P_TF32 = 1, P_BF16 = 2, P_FP16 = 3, P_FP8 = 4, P_INT8 = 5, P_FP64_OZ = 6, P_FP64_CRT = 7 };

// FP64 storage/operand format (P_FP64_OZ / P_FP64_CRT: FP64 values, GEMMs emulated on INT8 tensor
// cores by the Ozaki scheme I (digits) / II (Chinese remainder theorem))
__host__ __device__ inline bool is_f64(int prec) { return prec == P_FP64 || prec == P_FP64_OZ || prec == P_FP64_CRT; }
__host__ __device__ inline bool is_emu(int prec) { return prec == P_FP64_OZ || prec == P_FP64_CRT; }
// Ozaki scheme I (reading R-23): at most OZ_S digits per operand (a product keeps the digit pairs
// s + t <= S + 1); an FP64_OZ phase storing m mantissa bits uses S = oz_digits(m) <= OZ_S
constexpr int OZ_S = 9;
__host__ __device__ inline int oz_digits(int m) {
  const int s = (m + 12 + 6) / 7;
  return s < 2 ? 2 : s > OZ_S ? OZ_S : s;
}

// Ozaki scheme II (reading R-28): a product of operands quantised to b-bit integers relative to their
// row / column maximum (b <= CRT_BMAX) is computed exactly modulo N pairwise coprime
// moduli m_l <= 256 (one kind::i8 GEMM each, residues in [-128, 127]) and reconstructed by the CRT.
// The table is per N (the modulus product M_N changes the CRT weights):
//   X = sum_l v_l W_l, W_l = M_N / m_l, v_l = (u_l inv_l) mod m_l, u_l = (product mod m_l);
//   W_l = H_l 2^s1 + L_l 2^s2 + R_l with H, L < 2^39 (those partial sums exact in FP64; R rounded
//   to FP64 when s2 > 53, an absolute error far below the result's own rounding);
//   P = X - q M_N, q = rint(X / M_N), with M_N = MH 2^s1 + ML 2^s2 + MR sliced the same way.
constexpr int CRT_MAX = 18, CRT_BMAX = 62;
struct CrtTab {
  int m[CRT_MAX];                    // moduli (descending, pairwise coprime)
  uint32_t mag[CRT_MAX];             // ceil(2^32 / m_l): x mod m_l by one multiply-high
  int off[CRT_MAX];                  // m_l ceil(2^30 / m_l): makes an INT32 GEMM sum non-negative
  double invm[CRT_MAX];              // 1 / m_l (RN)
  float invmf[CRT_MAX];
  int inv[CRT_MAX + 1][CRT_MAX];     // (M_N / m_l)^-1 mod m_l
  double H[CRT_MAX + 1][CRT_MAX], L[CRT_MAX + 1][CRT_MAX], R[CRT_MAX + 1][CRT_MAX];
  double MH[CRT_MAX + 1], ML[CRT_MAX + 1], MR[CRT_MAX + 1], invM[CRT_MAX + 1];
  double Lo[CRT_MAX + 1][CRT_MAX], MLo[CRT_MAX + 1];   // (W mod 2^s1) 2^-s1, rounded (two-slice form)
  double CH[CRT_MAX + 1], CL[CRT_MAX + 1];             // 256 sum_l H_l (exact), 256 sum_l Lo_l (bias of 256 + v)
  double p2s1[CRT_MAX + 1], p2s2[CRT_MAX + 1];
  double log2M[CRT_MAX + 1];
  // exact four-slice form (the CRT certificate, reading R-35): W_l = H 2^s1 + L 2^s2 + X3 2^s3 + X4,
  // every slice an integer < 2^39 (M: MH < 2^48), s2 = max(s1 - 39, 0), s3 = max(s2 - 39, 0); the
  // biases 256 sum_l slice_l are exact; every sum of (256 + v_l) slice_l is an integer < 2^53
  double X3[CRT_MAX + 1][CRT_MAX], X4[CRT_MAX + 1][CRT_MAX];
  double MX3[CRT_MAX + 1], MX4[CRT_MAX + 1];
  double CB2[CRT_MAX + 1], CB3[CRT_MAX + 1], CB4[CRT_MAX + 1];
  double p2s3[CRT_MAX + 1];
};
const CrtTab &crt_table();                       // host copy (ozaki.cu)
int crt_moduli(int b, int64_t n);                // smallest N with M_N > 2^1.02 n 2^(2b); -1 if none
// CRT residues in [0, m_l) (u8 x u8 modulus GEMMs) while every INT32 sum of K products of bytes stays
// below 2^31 (K 255^2 < 2^31: K <= 33025); symmetric residues in [-128, 127] (s8 x s8) beyond -- or
// always, with ipr_test_crt_signed(1) (tests of the large-K convention at small sizes).  Host-side
// decision: the split takes it as its template flag, the modulus GEMMs as GemmArgs::crt_u8.
bool crt_unsigned(int64_t k);
void crt_force_signed(int on);
int crt_bits(int S, int64_t n);                  // digits S -> bits b = min(7 S - 4, 62, what 18 moduli allow at n)

// Operand formats that carry a per-tensor power-of-two scale 2^sigma (reading R-20; NEXT-3).
__host__ __device__ inline bool is_scaled(int prec) { return prec == P_FP16 || prec == P_FP8 || prec == P_INT8; }

// Epilogue modes of the GEMM kernels (bit flags).
enum EpiMode : int {
  EPI_STORE_T = 1,    // write qin(scale*D) transposed (K-major operand for the next GEMM)
  EPI_RESID = 2,      // per-tile partial of sum (delta_ij - scale*D_ij)^2  (fused residual)
  EPI_UPDATE = 4,     // C_next = q_m(((p+1) C - scale*D) / p), Chat_next, delta partials
  EPI_F64 = 8,        // test hook: FP64 row-major store of scale*D
  EPI_TSCRATCH = 16,  // FP16 phase: FP32 store of scale*D transposed + per-tile max|.|
  EPI_DIAG_MINUS = 32,  // modifier of STORE_T/TSCRATCH: store diag*delta_ij - D (Newton-Schulz
                        // What = 2I - T with diag = 2; symmetric form R = I - Z_p with diag = 1)
  EPI_NSUPDATE = 64,  // Newton-Schulz: X_{k+1} = q_m(D) -> container, operand, delta partials
  EPI_WSTORE = 128,   // symmetric form: W = D row-major to wout[i * ldw + j] (FP32, or FP64 if w64)
  EPI_STORE_N = 256,  // also store qin(D) row-major (nout[i * ldn + j]): symmetric form, FP64,
                      // G = 1 -- D = A C row-major is the B operand of C (C A) for certification
  EPI_OZACC = 512,    // Ozaki group g: ozacc[j * ldoz + i] (+)= 2^(rsig_i + csig_j - 7 g) * D_ij (INT32 D)
  EPI_COUPLED = 1024, // coupled form: w = q_m(D); Mhat = qin(w) -> tout, Nhat = qin(((p+1)delta - w)/p)
                      // -> nkout (both K-major at col * ldt + row); with EPI_RESID for rho
  EPI_SYMUPD = 2048,  // symmetric-tri form, fused update (tcgen05, tri): D = S = W + W^T from the
                      // K-concatenated GEMM [Chat | Rhat] [Rhat ; Chat]; C_{k+1} = q_m(C + S/(2p)) at (i,j)
                      // and (j,i) -> cnew, + the next operands (chat_new in prec, qnext planes 0 and 2 in
                      // the correction format tprec), delta partials
};

struct GemmArgs {
  int64_t M, N, K;      // padded sizes (multiples of 128); N = local panel width
  int64_t n;            // true matrix order (residual masking)
  int64_t col0;         // global column of local column 0
  // A operand (Chat): element (i,k) at A + (k / a_kp) * a_pstride + i * a_kp + k % a_kp
  const void *A; int64_t a_kp, a_pstride;
  // B operand, K-major: element (k,j) at B + j * ldb + k
  const void *B; int64_t ldb;
  int prec, mode;
  int tprec;            // operand format of the EPI_STORE_T output (= prec except the symmetric
                        // form's Rhat, stored in the correction format)
  double diag;          // EPI_DIAG_MINUS coefficient
  int tri;              // symmetric-tri form (G = 1): D is symmetric in exact arithmetic; only
                        // elements with row <= col are computed, each stored at (i,j) AND (j,i),
                        // residual weight 2 off the diagonal; tiles wholly below are skipped
  const int *sigA, *sigB; // FP16 phase: device scale exponents of the A / B operands; else NULL
  // EPI_STORE_T / EPI_TSCRATCH: T(i,j) -> tout[j * ldt + i]
  void *tout; int64_t ldt;
  // partial sums: part[tile_n_global * tiles_m + tile_m]
  double *part; int64_t tiles_m;
  float *pmax;          // per-tile max |.| (EPI_TSCRATCH, EPI_UPDATE in FP16 phase)
  // EPI_UPDATE: container C(i,j) at cold/cnew[i * ldc + j]; operand Chat_next at chat_new[i*ldh+j]
  const void *cold; void *cnew; int64_t ldc;
  void *chat_new; int64_t ldh;
  int p, m, rtz, cont64;
  // EPI_F64
  double *zout; int64_t ldz;
  // EPI_WSTORE
  void *wout; int64_t ldw; int w64;
  // EPI_STORE_N
  void *nout; int64_t ldn;
  // EPI_COUPLED: the K-major Nhat output (same ldt as tout)
  void *nkout;
  // EPI_OZACC (FP64 accumulator stored transposed), and the Ozaki operands of a P_FP64_OZ GEMM
  double *ozacc; int64_t ldoz; const int *oz_rsig, *oz_csig; int oz_g, oz_first, oz_S;
  int oz_grouped;       // k_gemm_tc<kind::i8>: every group g = S+1..2 of a tile in one launch (K up to
                        // OZ_S * npad, B offset (OZ_S - g + 1) * npad), the finish epilogue g.mode
                        // fused into group 2; g.mode holds the FINISH mode
  const int8_t *oz_a;   // A-role digit planes [S][npad][npad] (row-major per plane)
  int64_t b_pstride;    // != 0: B is K-concatenated planes too, element (k,j) at
                        // B + (k / a_kp) * b_pstride + j * ldb + k % a_kp (3-D tensor map)
  void *qnext;          // EPI_SYMUPD: [3][npad][npad] correction-format buffer of the next iterate (planes
                        // 0 and 2 receive Chat_{k+1}); ldh is its row stride
  int hprec;            // EPI_SYMUPD: format of chat_new (the phase's operand; prec is the MMA format)
  const int8_t *oz_b;   // B-role digits, per output column j: [S * npad] = digit planes S..1 of column j
                        // (oz_grouped == 3, CRT: residue planes [crt_n][npad][npad] of both operands)
  int crt_n;            // oz_grouped == 3: number of moduli (one kind::i8 GEMM each)
  int crt_l0, crt_l1;   // CRT: the moduli [crt_l0, crt_l1) of this launch (modulus-major)
  uint8_t *crt_v;       // CRT: v_l of moduli 0..crt_n-1 at crt_v[(l * M + i) * ldv + j]
  int64_t ldv;
  // tri: the mirror (j, i) of an upper element (i, j) goes to mout[i * ldm + (j - col0)] -- at G = 1
  // mout = tout, ldm = ldt (the launchers fill them in when mout is null); a G > 1 rank points it at the
  // packed [G][kp][kp] send buffer of the mirror exchange (ldm = kp)
  void *mout; int64_t ldm;
  // 2-D grid (P_r x P_c ranks, literal form): the output block's first global row.  Epilogues use global
  // rows (diagonal, masking, partial slots); the engine offsets the output pointers by -row0 rows.
  int64_t row0;
  // B operand panels (b_pstride != 0): K-panel length of B (0: = a_kp) -- the 2-D grid's gathered
  // T column panel [P_r][kp][mr] has b_kp = mr
  int64_t b_kp;
  // diagnostics only (IPR_DIAG_EPI, read by launch_gemm_tc; results are wrong when set): bit 0 skips the
  // tri epilogue's residual terms, bit 1 its K-major stores, bit 2 its mirror stores
  int diag_epi;
  // CRT modulus launches after the first of a product (ozaki.cu): launched with programmatic stream
  // serialization, so a launch's CTAs start on the SMs its predecessor's tail frees (the launches are
  // independent: other residue planes, other v-byte planes); each waits for its predecessor before it
  // exits, so the finish kernel, launched normally, sees every modulus complete
  int pdl;
  int crt_u8;           // CRT: residues in [0, m) (u8 x u8 modulus GEMMs), else symmetric (s8 x s8)
  int crt_dd;           // CRT: reconstruct exactly as a double-double (the certificate, launch_crt_finish_dd)
};

// ------------------------------------------------------------------------------------
// Bit-level quantisers
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double bits2d(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ uint64_t d2bits(double x) { return (uint64_t)__double_as_longlong(x); }
// Round the magnitude bits `mag` of an IEEE encoding to keep `s` fewer low bits.
__device__ __forceinline__ uint64_t round_mag64(uint64_t mag, int s, int rtz) {
  if (s <= 0) return mag;
  const uint64_t mask = ~((1ull << s) - 1ull);
  if (rtz) return mag & mask;
  const uint64_t half = (1ull << (s - 1)) - 1ull;
  // parity of q = mag / 2^s (the oracle's integer multiple of the ulp); at s = 52 (m = 0) q is the
  // implicit bit: 1 (odd) for normals, 0 for subnormals -- not the exponent's low bit
  const uint64_t lsb = s >= 52 ? (uint64_t)((mag >> 52) != 0ull) : (mag >> s) & 1ull;
  return (mag + half + lsb) & mask;
}

// FP64 value -> m stored bits in an e11 (FP64) container.  Works for subnormal doubles (the
// encoding is fixed point there) and carries into Inf on RNE overflow.
__device__ __forceinline__ double q_e11(double x, int m, int rtz) {
  const uint64_t b = d2bits(x);
  const uint64_t sign = b & 0x8000000000000000ull, mag = b ^ sign;
  if (mag >= 0x7ff0000000000000ull) return x;            // Inf / NaN
  uint64_t r = round_mag64(mag, 52 - m, rtz);
  if (rtz && r >= 0x7ff0000000000000ull) r = 0x7fefffffffffffffull;  // unreachable, kept safe
  return bits2d(r | sign);
}

// FP64 value -> m stored bits in an e8 (FP32) container, single rounding from FP64.  q_e8d returns
// the result as the (exactly equal) double: callers that continue in FP64 skip two F2F conversions
// (XU pipe: the symmetric update was XU-bound).
__device__ __forceinline__ double q_e8d(double x, int m, int rtz) {
  const uint64_t b = d2bits(x);
  const uint64_t sign = b & 0x8000000000000000ull, mag = b ^ sign;
  if (mag >= 0x7ff0000000000000ull) return (double)(float)x;   // Inf / NaN (as the FP32 conversion)
  const uint64_t E128 = (uint64_t)(1023 + 128) << 52;    // 2^128: beyond e8
  const uint64_t E126 = (uint64_t)(1023 - 126) << 52;    // 2^-126: e8 normal minimum
  // max finite of e8 with m bits: (2 - 2^-m) 2^127
  const double maxf = bits2d(((uint64_t)(1023 + 127) << 52) | (((1ull << m) - 1ull) << (52 - m)));
  if (mag >= E128) return rtz ? copysign(maxf, x) : copysign(__longlong_as_double(0x7ff0000000000000ll), x);
  if (mag >= E126) {
    const uint64_t r = round_mag64(mag, 52 - m, rtz);
    if (r >= E128) return copysign(__longlong_as_double(0x7ff0000000000000ll), x);
    return bits2d(r | sign);                             // exact in FP32: <= m+1 significant bits
  }
  // e8 subnormal range: multiples of 2^(-126-m)
  const double up = bits2d((uint64_t)(1023 + 126 + m) << 52);
  const double dn = bits2d((uint64_t)(1023 - 126 - m) << 52);
  const double y = __dmul_rn(x, up);
  const double q = rtz ? trunc(y) : rint(y);
  return __dmul_rn(q, dn);                               // a multiple of 2^-149 below 2^-126: exact in FP32
}
__device__ __forceinline__ float q_e8(double x, int m, int rtz) { return (float)q_e8d(x, m, rtz); }

// Branch-free q_e8d / q_e11 for the common case (hot loops of the symmetric update): the caller
// hoists the rounding constants (QRound) and keeps q only if `ok` (the value and its rounding stay
// in the normal range of the container), else calls q_e8d / q_e11.  Same bits as those whenever ok.
struct QRound {
  uint64_t mask, half;
  int sh, rtz;
  __device__ __forceinline__ QRound(int m, int rtz_) : sh(52 - m), rtz(rtz_) {
    mask = sh > 0 ? ~((1ull << sh) - 1ull) : ~0ull;
    half = sh > 0 && !rtz_ ? (1ull << (sh - 1)) - 1ull : 0ull;
  }
  __device__ __forceinline__ uint64_t round(uint64_t mag) const {
    const uint64_t lsb = (sh > 0 && !rtz) ? (sh >= 52 ? (uint64_t)((mag >> 52) != 0ull) : (mag >> sh) & 1ull) : 0ull;
    return (mag + half + lsb) & mask;
  }
};
__device__ __forceinline__ double q_e8d_fast(double x, const QRound &q, bool &ok) {
  const uint64_t b = d2bits(x);
  const uint64_t sign = b & 0x8000000000000000ull, mag = b ^ sign;
  const uint64_t E128 = (uint64_t)(1023 + 128) << 52, E126 = (uint64_t)(1023 - 126) << 52;
  const uint64_t r = q.round(mag);
  ok = ok && (mag - E126 < E128 - E126) && r < E128;   // normal e8 input and result (0 goes slow)
  return bits2d(r | sign);
}
__device__ __forceinline__ double q_e11_fast(double x, const QRound &q, bool &ok) {
  const uint64_t b = d2bits(x);
  const uint64_t sign = b & 0x8000000000000000ull, mag = b ^ sign;
  ok = ok && mag < 0x7ff0000000000000ull;              // finite (q_e11 handles subnormals alike)
  return bits2d(q.round(mag) | sign);
}

// FP32 -> TF32 grid (e8m10), round-to-nearest-even, Inf/NaN kept (operand conversion).
__device__ __forceinline__ float to_tf32(float x) {
  const uint32_t b = __float_as_uint(x);
  const uint32_t sign = b & 0x80000000u, mag = b ^ sign;
  if (mag >= 0x7f800000u) return x;
  const uint32_t r = (mag + 0xfffu + ((mag >> 13) & 1u)) & ~0x1fffu;
  return __uint_as_float(r | sign);
}

// Scale exponent of a scaled operand (reading R-20): FP16 sigma = 14 - floor(log2 max) (scaled max
// in [2^14, 2^15)); FP8 E4M3 and INT8 sigma = 6 - floor(log2 max) (scaled max in [64, 128)).
// 0 if max <= 0 / NaN / Inf.
__device__ __forceinline__ int op_sigma(int prec, double mx) {
  if (!(mx > 0.0) || isinf(mx)) return 0;
  return (prec == P_FP16 ? 14 : 6) - ilogb(mx);
}

// exact 2^e as double (|e| <= 1000)
__device__ __forceinline__ double pow2(int e) { return bits2d((uint64_t)(1023 + e) << 52); }

// E4M3 grid (NEXT-3) of an FP64 value with |x| < 448: RNE to 3 mantissa bits for |x| >= 2^-6,
// multiples of 2^-9 below (subnormals) -- one rounding from FP64; the result is exactly
// representable, so the final cvt is exact.
__device__ __forceinline__ uint8_t to_e4m3(double x) {
  const double a = fabs(x);
  double q;
  if (a >= 0.015625) q = q_e11(x, 3, 0);
  else q = __dmul_rn(rint(__dmul_rn(x, 512.0)), 1.0 / 512.0);
  return (uint8_t)__nv_cvt_double_to_fp8(q, __NV_SATFINITE, __NV_E4M3);
}
// INT8 fixed point (NEXT-3): nearest-even integer, saturated to [-127, 127]
__device__ __forceinline__ int8_t to_int8(double x) {
  double q = rint(x);
  q = fmin(fmax(q, -127.0), 127.0);
  return (int8_t)(int)q;
}

// Operand store of an FP32/FP64 value in phase precision (RNE); scaled formats get 2^sig first.
__device__ __forceinline__ void store_operand(void *base, int64_t idx, int prec, double v, int sig) {
  switch (prec) {
    case P_FP64:
    case P_FP64_OZ:
    case P_FP64_CRT: ((double *)base)[idx] = v; break;
    case P_TF32: ((float *)base)[idx] = to_tf32((float)v); break;
    case P_BF16: ((__nv_bfloat16 *)base)[idx] = __float2bfloat16_rn((float)v); break;
    case P_FP16: ((__half *)base)[idx] = __float2half_rn((float)__dmul_rn(v, pow2(sig))); break;
    case P_FP8: ((uint8_t *)base)[idx] = to_e4m3(__dmul_rn(v, pow2(sig))); break;
    case P_INT8: ((int8_t *)base)[idx] = to_int8(__dmul_rn(v, pow2(sig))); break;
  }
}

__host__ __device__ inline int elt_size(int prec) {
  return is_f64(prec) ? 8 : (prec == P_BF16 || prec == P_FP16) ? 2 : (prec == P_FP8 || prec == P_INT8) ? 1 : 4;
}

// Deterministic block-wide sum of one double per thread (fixed shuffle tree + warp order).
template <int NT>
__device__ __forceinline__ double block_sum_det(double v, double *red) {
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NT / 32; ++i) s += red[i];
  }
  return s;  // valid in thread 0
}

template <int NT>
__device__ __forceinline__ float block_max(float v, float *red) {
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x == 0) for (int i = 0; i < NT / 32; ++i) s = fmaxf(s, red[i]);
  return s;
}

}  // namespace ipr

// Host-side launch declarations (implemented in kernels.cu / gemm_dmma.cu / gemm_tc.cu).
namespace ipr {
// Per-device "done once" flag for device state that a process sets up lazily (function attributes,
// __constant__ tables): one bit per device ordinal, so a second GPU in the process gets its own setup.
struct DeviceOnce {
  unsigned long long bits = 0ull;
  bool done() const { int d = 0; cudaGetDevice(&d); return d < 64 && ((bits >> d) & 1ull); }
  void set() { int d = 0; cudaGetDevice(&d); if (d < 64) bits |= 1ull << d; }
};
extern int64_t g_launches;
cudaError_t launch_gemm_dmma(const GemmArgs &a, cudaStream_t s);
cudaError_t launch_gemm_tc(const GemmArgs &a, cudaStream_t s);  // BF16 / FP16 / TF32 / FP8 / INT8
cudaError_t launch_gemm_ozaki(const GemmArgs &a, cudaStream_t s);  // FP64 on INT8 (ozaki.cu)
cudaError_t launch_gemm_crt(const GemmArgs &a, cudaStream_t s);    // FP64 on INT8, CRT (ozaki.cu)
cudaError_t tc_set_crt_table(const CrtTab &t);                      // upload (gemm_tc.cu)
cudaError_t launch_crt_finish(const GemmArgs &a, cudaStream_t s);  // CRT reconstruction + epilogue
cudaError_t launch_crt_finish_dd(const GemmArgs &a, cudaStream_t s);  // exact CRT reconstruction (R-35)
// Optional device timing of the kind::i8 GEMM launches of CRT products (the roofline's dominant kernel,
// without the residue splits and the reconstruction): while set on this host thread, launch_gemm_crt
// records an event pair around its GEMM launches (up to cap pairs; *used counts them).
struct CrtTimer { cudaEvent_t *ev; int cap; int used; };
void crt_set_timer(CrtTimer *t);
bool tc_supported(int prec);
const char *tc_last_error();
int gemm_tile_n(int prec);   // BN of the kernel used for a precision (partial layout)
int dmma_tile_n();
int gemm_tile_m(int prec);
}  // namespace ipr
