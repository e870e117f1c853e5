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
#include <cmath>
#include <cstdlib>
#include <cstring>

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

namespace ipr {

// =========================================================================================
// Ozaki scheme II (reading R-28): FP64 products by the Chinese remainder theorem on INT8 moduli.
//
//   quantise  Xbar_ik = rint(2^e_i x_ik), e_i = b - 1 - floor(log2 max_k |x_ik|)  (|Xbar| <= 2^b, an
//             FP64 integer for any b: x 2^e is exact, rint of a double is a double; b <= 62, so it is
//             also an int64); the same per column of the right operand (exponent f_j)
//   products  for l = 1..N: U_l = (Xbar mod m_l)(Ybar mod m_l), symmetric residues in [-128, 127],
//             ONE kind::i8 GEMM each, exact in INT32 (|U_l| <= 2^14 n < 2^31 for n < 131072)
//   CRT       Pbar = Xbar Ybar is the unique integer with |Pbar| < M_N / 2 and Pbar = U_l mod m_l:
//             Pbar = sum_l v_l W_l - q M_N, v_l = (U_l inv_l) mod m_l, W_l = M_N / m_l (exact sliced
//             FP64 arithmetic in k_crt_finish: an exact 39-bit slice and a rounded low slice, common.cuh
//             CrtTab); M_N > 2^1.02 n 2^(2b) >= 2.03 max |Pbar| puts X / M_N within 0.493 of an integer,
//             so q = rint(X / M_N) is exact (X / M_N is evaluated to ~2^-45)
//   bits      b = 7 S - 4 for the phase's Ozaki-equivalent digits S (crt_bits); N = crt_moduli(b, n)
//   scale     Z_ij = 2^-(e_i + f_j) Pbar_ij (exact)
// Error: only the quantisation, |Xbar_ik - 2^e_i x_ik| <= 1/2, i.e. 2^-b relative to the row maximum.
// =========================================================================================
// pairwise coprime moduli <= 256, descending: 2^8, 3*5*17, 11*23, 251, 13*19, then primes and 7*31
constexpr int kModuli[CRT_MAX] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193,
                                  191, 181};
namespace {
// little multi-word unsigned integer (M_18 ~ 2^141 exceeds 128 bits)
struct Big {
  uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  void mul(uint32_t m) { uint64_t c = 0; for (auto &x : w) { c += (uint64_t)x * m; x = (uint32_t)c; c >>= 32; } }
  uint32_t divmod(uint32_t m) {   // *this /= m, returns the remainder
    uint64_t r = 0;
    for (int i = 7; i >= 0; --i) { r = (r << 32) | w[i]; w[i] = (uint32_t)(r / m); r %= m; }
    return (uint32_t)r;
  }
  int bitlen() const { for (int i = 7; i >= 0; --i) if (w[i]) return 32 * i + 32 - __builtin_clz(w[i]); return 0; }
  uint64_t bits(int lo, int cnt) const {   // bits [lo, lo + cnt) (cnt <= 64)
    uint64_t v = 0;
    for (int k = 0; k < cnt; ++k) { const int b = lo + k; if (b < 256 && ((w[b >> 5] >> (b & 31)) & 1u)) v |= 1ull << k; }
    return v;
  }
  long double ld(int below = 256) const {  // value of bits [0, below), as long double
    long double v = 0.0L;
    for (int i = 7; i >= 0; --i) {
      uint32_t x = w[i];
      if (32 * i >= below) x = 0;
      else if (32 * i + 32 > below) x &= (uint32_t)((1ull << (below - 32 * i)) - 1);
      v = v * 4294967296.0L + (long double)x;
    }
    return v;
  }
};
int64_t modinv(int64_t a, int64_t m) {   // a^-1 mod m (gcd(a, m) = 1)
  int64_t g = m, x = 0, x1 = 1, aa = a % m;
  while (aa) { const int64_t q = g / aa, t = g - q * aa; g = aa; aa = t; const int64_t tx = x - q * x1; x = x1; x1 = tx; }
  return ((x % m) + m) % m;
}
CrtTab make_crt_table() {
  CrtTab t;
  memset(&t, 0, sizeof t);
  for (int l = 0; l < CRT_MAX; ++l) {
    t.m[l] = kModuli[l];
    t.invm[l] = 1.0 / (double)kModuli[l];
    t.invmf[l] = 1.0f / (float)kModuli[l];
    t.mag[l] = (uint32_t)((((uint64_t)1 << 32) + kModuli[l] - 1) / kModuli[l]);
    t.off[l] = kModuli[l] * (int)(((1 << 30) + kModuli[l] - 1) / kModuli[l]);
  }
  for (int N = 1; N <= CRT_MAX; ++N) {
    Big M;
    M.w[0] = 1;
    for (int l = 0; l < N; ++l) M.mul((uint32_t)kModuli[l]);
    int E = 0;
    for (int l = 0; l < N; ++l) { Big W = M; W.divmod((uint32_t)kModuli[l]); E = W.bitlen() > E ? W.bitlen() : E; }
    // W = H 2^s1 + L 2^s2 + R: H, L < 2^39 exact; R < 2^s2 rounded to FP64 when s2 > 53 (its products
    // then carry an absolute error ~2^(s2 - 40), far below the result's own rounding 2^(2b + log2 n - 53)).
    // Lo = L 2^(s2 - s1) + R 2^-s1 = (W mod 2^s1) 2^-s1 rounded to FP64: the two-slice form of the
    // finish kernel (the rounding of sum v Lo ~2^(s1 - 45), negligible likewise)
    // 39-bit H: the finish kernel accumulates (256 + v_l) H_l, 18 * 511 * 2^39 < 2^53
    const int s1 = E > 39 ? E - 39 : 0, s2 = s1 > 39 ? s1 - 39 : 0;
    auto slice = [&](const Big &W, double &h, double &lo, double &r, double &low) {
      h = (double)W.bits(s1, 39 + 9);
      lo = (double)W.bits(s2, s1 - s2);
      r = (double)W.ld(s2);
      low = (double)(W.ld(s1) / ldexpl(1.0L, s1));
    };
    const int s3 = s2 > 39 ? s2 - 39 : 0;
    double b2 = 0.0, b3 = 0.0, b4 = 0.0;
    for (int l = 0; l < N; ++l) {
      Big W = M;
      W.divmod((uint32_t)kModuli[l]);
      Big Wc = W;
      t.inv[N][l] = (int)modinv((int64_t)Wc.divmod((uint32_t)kModuli[l]), kModuli[l]);
      slice(W, t.H[N][l], t.L[N][l], t.R[N][l], t.Lo[N][l]);
      t.X3[N][l] = (double)W.bits(s3, s2 - s3);
      t.X4[N][l] = (double)W.bits(0, s3);
      b2 += 256.0 * t.L[N][l]; b3 += 256.0 * t.X3[N][l]; b4 += 256.0 * t.X4[N][l];   // exact: < 2^52
    }
    slice(M, t.MH[N], t.ML[N], t.MR[N], t.MLo[N]);
    t.MX3[N] = (double)M.bits(s3, s2 - s3);
    t.MX4[N] = (double)M.bits(0, s3);
    t.CB2[N] = b2; t.CB3[N] = b3; t.CB4[N] = b4;
    t.p2s3[N] = ldexp(1.0, s3);
    double ch = 0.0;
    long double cl = 0.0L;
    for (int l = 0; l < N; ++l) { ch += 256.0 * t.H[N][l]; cl += 256.0L * (long double)t.Lo[N][l]; }
    t.CH[N] = ch;                                 // exact: < 2^52
    t.CL[N] = (double)cl;
    t.invM[N] = (double)(1.0L / M.ld());
    t.p2s1[N] = ldexp(1.0, s1);
    t.p2s2[N] = ldexp(1.0, s2);
    t.log2M[N] = (double)log2l(M.ld());
  }
  return t;
}
}  // namespace

const CrtTab &crt_table() {
  static const CrtTab t = make_crt_table();
  return t;
}
static int g_crt_signed = 0;   // ipr_test_crt_signed
void crt_force_signed(int on) { g_crt_signed = on != 0; }
bool crt_unsigned(int64_t k) { return !g_crt_signed && k <= 33024; }
int crt_moduli(int b, int64_t n) {
  const double need = 2.0 * b + std::log2((double)(n < 1 ? 1 : n)) + 1.02;
  for (int N = 2; N <= CRT_MAX; ++N)
    if (crt_table().log2M[N] > need) return N;
  return -1;
}
int crt_bits(int S, int64_t n) {
  // b = 7 S - 4: the stored bits of R-26's rule for S digits (m = min(52, 7 S - 4)); the Ozaki-I
  // equivalent 7 S - 1 costs ~1 modulus more per product for the same trajectory (measured: 7 S - 4
  // and 7 S - 7 certify in the same 19 + 8 iterations, 7 S - 10 stalls at 2.9e-6).  IPR_CRT_BOFF
  // overrides the 4 (experiments only).
  static int boff = -1;
  if (boff < 0) { const char *v = getenv("IPR_CRT_BOFF"); boff = v ? atoi(v) : 4; }
  int b = 7 * S - boff < CRT_BMAX ? 7 * S - boff : CRT_BMAX;
  while (b > 2 && crt_moduli(b, n) < 0) --b;
  return b;
}

// Symmetric residue byte of y = yb - 2^62 modulo the compile-time modulus M, yb = y + 2^62 in [0, 2^63)
// given as its two 32-bit halves (eight unsigned bytes b_t): yb mod M = (sum_t b_t (2^(8t) mod M)) mod M,
// the byte sum as two __dp4a (< 8 * 255 * 255 + M < 2^20) with h - 2^62 mod M folded into the first
// accumulator, then one exact multiply-high reduction (x < 2^20, magic ceil(2^32 / M): error < 2^-12
// < 1/M) and the shift by the symmetric offset h.  ~5 integer operations per residue.
// UNS: the residue in [0, M) itself (u8 x u8 modulus GEMMs, crt_unsigned): no symmetric shift, and for
// M = 256 the low byte of the sum directly.
template <int M, bool UNS = false>
__device__ __forceinline__ uint32_t crt_res8(uint32_t lo, uint32_t hi) {
  constexpr uint32_t h = UNS ? 0u : M == 256 ? 128 : (M - 1) / 2;
  constexpr uint32_t w0 = 1u % M, w1 = (1u << 8) % M, w2 = (1u << 16) % M, w3 = (1u << 24) % M;
  constexpr uint32_t w4 = (uint32_t)((1ull << 32) % M), w5 = (uint32_t)((1ull << 40) % M);
  constexpr uint32_t w6 = (uint32_t)((1ull << 48) % M), w7 = (uint32_t)((1ull << 56) % M);
  constexpr uint32_t KL = w0 | (w1 << 8) | (w2 << 16) | (w3 << 24), KH = w4 | (w5 << 8) | (w6 << 16) | (w7 << 24);
  constexpr uint32_t K3 = (uint32_t)((h + M - (uint32_t)((1ull << 62) % M)) % M);
  constexpr uint32_t MAG = (uint32_t)(((1ull << 32) + M - 1) / M);
  if (UNS && M == 256) return lo;                 // y mod 256: the low byte (2^62 = 0 mod 256)
  const uint32_t r = __dp4a(hi, KH, __dp4a(lo, KL, K3));
  const uint32_t u = r - __umulhi(r, MAG) * (uint32_t)M;
  return UNS ? u : u - h;                         // the low byte is the residue (packed by PRMT)
}
template <int L, bool UNS>
__device__ __forceinline__ void crt_split4(const uint32_t (&lo)[4], const uint32_t (&hi)[4], int nm, int8_t *dst,
                                           int64_t plane) {
  if constexpr (L < CRT_MAX) {
    if (L < nm) {
      uint32_t b[4];
      #pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = crt_res8<kModuli[L], UNS>(lo[u], hi[u]);
      *(uint32_t *)(dst + (int64_t)L * plane) =
          __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
      crt_split4<L + 1, UNS>(lo, hi, nm, dst, plane);
    }
  }
}

// Residues of the rows of X (FP64, row-major, leading dimension ld): one block per row; plane l of
// `planes` holds (Xbar mod m_l) at planes[l * rows * cols + r * cols + k]; sig[r] = e_r.
// SMEM: the row is staged in shared memory (cols * 8 B <= 64 KB), so the maximum pass and the residue
// pass read it from DRAM once (with two global passes the residue writes evicted it between them).
template <bool SMEM, bool UNS>
__global__ void __launch_bounds__(256, 3) k_crt_split(const double *__restrict__ X, int64_t ld, int64_t rows,
                                                      int64_t cols, int b, int nm, int8_t *planes, int *sig) {
  extern __shared__ double srow[];
  __shared__ double red[8];
  const int64_t r = blockIdx.x;
  const double *x = X + r * ld;
  double mx = 0.0;
  if (SMEM) {
    for (int64_t k = (int64_t)threadIdx.x * 2; k < cols; k += (int64_t)blockDim.x * 2) {
      const double2 t = *(const double2 *)(x + k);
      *(double2 *)(srow + k) = t;
      mx = fmax(mx, fmax(fabs(t.x), fabs(t.y)));
    }
  } else {
    for (int64_t k = threadIdx.x; k < cols; k += blockDim.x) mx = fmax(mx, fabs(x[k]));
  }
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
  // scaled row maximum in [2^(b-1), 2^b): |Xbar| <= 2^b <= 2^62
  const int e = (mx > 0.0) ? b - 1 - ilogb(mx) : 0;
  if (threadIdx.x == 0) sig[r] = e;
  // 2^e in two exact factors: |e| can exceed the FP64 exponent range for tiny / huge rows
  const double sc1 = pow2(e / 2), sc2 = pow2(e - e / 2);
  const int64_t plane = rows * cols;
  const double *src = SMEM ? (const double *)srow : x;
  #pragma unroll 2
  for (int64_t k0 = (int64_t)threadIdx.x * 4; k0 < cols; k0 += (int64_t)blockDim.x * 4) {
    uint32_t lo[4], hi[4];
    const double2 *xp = (const double2 *)(src + k0);
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 t = xp[u >> 1];
      // Xbar + 2^62 in [0, 2^63): eight unsigned bytes
      const uint64_t y = (uint64_t)__double2ll_rn(__dmul_rn(__dmul_rn((u & 1) ? t.y : t.x, sc1), sc2)) + (1ull << 62);
      lo[u] = (uint32_t)y; hi[u] = (uint32_t)(y >> 32);
    }
    crt_split4<0, UNS>(lo, hi, nm, planes + r * cols + k0, plane);
  }
}

cudaError_t launch_crt_split(const double *X, int64_t ld, int64_t rows, int64_t cols, int b, int nm, int8_t *planes,
                             int *sig, cudaStream_t s) {
  if (b < 2 || b > CRT_BMAX || nm < 2 || nm > CRT_MAX || cols % 4) return cudaErrorInvalidValue;
  const bool uns = crt_unsigned(cols);           // cols = the GEMM's K (row length of the residue planes)
  if (cols * 8 <= 65536 && ld % 2 == 0) {
    static DeviceOnce attr;
    if (!attr.done()) {
      cudaError_t e = cudaFuncSetAttribute(k_crt_split<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_crt_split<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      if (e != cudaSuccess) return e;
      attr.set();
    }
    if (uns) k_crt_split<true, true><<<(unsigned)rows, 256, (size_t)cols * 8, s>>>(X, ld, rows, cols, b, nm, planes, sig);
    else k_crt_split<true, false><<<(unsigned)rows, 256, (size_t)cols * 8, s>>>(X, ld, rows, cols, b, nm, planes, sig);
  } else if (uns) {   // rows longer than 8192: two passes over the row (L2), the same residue convention
    k_crt_split<false, true><<<(unsigned)rows, 256, 0, s>>>(X, ld, rows, cols, b, nm, planes, sig);
  } else {
    k_crt_split<false, false><<<(unsigned)rows, 256, 0, s>>>(X, ld, rows, cols, b, nm, planes, sig);
  }
  ++g_launches;
  return cudaGetLastError();
}

thread_local CrtTimer *t_crt_timer = nullptr;
void crt_set_timer(CrtTimer *t) { t_crt_timer = t; }

// Z = X Y for a P_FP64_CRT GemmArgs: g.oz_a / g.oz_rsig the residue planes and exponents of X (A
// role, rows), g.oz_b / g.oz_csig those of the rows of the K-major B operand, g.crt_n moduli,
// g.crt_v the crt_n x npad x npad byte scratch.  One persistent kind::i8 launch over every modulus,
// modulus-major (the CTA pairs stream one residue plane pair at a time, L2 reuse as in a plain GEMM;
// a tile-major order measured 50 GB of DRAM reads per n = 8192 product), each tile's epilogue
// storing v_l bytes; then k_crt_finish reconstructs and applies the hot path's epilogue g.mode
// (fused into the last modulus' epilogue it thrashed L1 on the residue loads: 3.4 ms).
cudaError_t launch_gemm_crt(const GemmArgs &g, cudaStream_t s) {
  static DeviceOnce uploaded;                   // the __constant__ table is per device
  if (!uploaded.done()) {
    cudaError_t e = tc_set_crt_table(crt_table());
    if (e != cudaSuccess) return e;
    uploaded.set();
  }
  // M = K = npad; N = npad (G = 1) or the column panel width kp (G > 1: B residues [crt_n][kp][npad])
  if (!g.oz_a || !g.oz_b || !g.oz_rsig || !g.oz_csig || !g.crt_v || g.M != g.K || g.N > g.K || g.crt_n < 2 ||
      g.crt_n > CRT_MAX)
    return cudaErrorInvalidValue;
  const int64_t np = g.K;
  GemmArgs q = g;
  q.prec = P_INT8;
  if (!is_f64(q.tprec) && q.tprec != P_BF16 && q.tprec != P_TF32) q.tprec = P_FP64;
  q.A = g.oz_a; q.a_kp = np; q.a_pstride = np * np;
  q.K = (int64_t)g.crt_n * np;                   // map extents: all residue planes
  q.B = g.oz_b; q.ldb = np;
  q.oz_grouped = 3;
  q.crt_u8 = crt_unsigned(np) ? 1 : 0;           // the split of these residues took the same decision
  q.sigA = nullptr; q.sigB = nullptr; q.pmax = nullptr;
  q.ldv = np;
  CrtTimer *tm = t_crt_timer;
  const bool timed = tm && tm->used < tm->cap;
  if (timed) { cudaError_t e = cudaEventRecord(tm->ev[2 * tm->used], s); if (e != cudaSuccess) return e; }
  static int per = 0;                            // moduli per launch (bounds the drift of the CTA pairs)
  if (!per) { const char *v = getenv("IPR_CRT_PER"); per = v ? atoi(v) : 2; per = per < 1 ? 1 : per; }
  static int pdl = -1;                           // IPR_CRT_PDL=0: plain stream order (A/B measurements)
  if (pdl < 0) { const char *v = getenv("IPR_CRT_PDL"); pdl = v ? atoi(v) != 0 : 1; }
  for (int l0 = 0; l0 < g.crt_n; l0 += per) {    // residue bytes of every modulus
    q.crt_l0 = l0; q.crt_l1 = l0 + per < g.crt_n ? l0 + per : g.crt_n;
    q.pdl = pdl && l0 > 0;                       // overlap a launch's ramp with its predecessor's tail
    cudaError_t e = launch_gemm_tc(q, s);
    if (e != cudaSuccess) return e;
  }
  if (timed) { cudaError_t e = cudaEventRecord(tm->ev[2 * tm->used + 1], s); if (e != cudaSuccess) return e; ++tm->used; }
  return g.crt_dd ? launch_crt_finish_dd(q, s)  // the certificate's exact reconstruction (R-35)
                  : launch_crt_finish(q, s);     // reconstruction + the hot path's epilogue
}

}  // namespace ipr

namespace ipr {

// =========================================================================================
// The CRT certificate (reading R-35): ||I - Ct^2 A||_F of the certified matrix Ct (the candidate C
// rounded to the coarser of its row's and its column's b-bit grids) from EXACT integer products,
// with every remaining error bounded a posteriori (engine.cu certify_crt):
//   k_cert_rowexp       e_r of the candidate's rows (the split's exponent rule), the row scale 2^-e_r
//   k_cert_round_split  Ct_rk = 2^-g rint(2^g c_rk), g = min(e_r, e_k), in place, and the residues of
//                       2^e_r Ct_rk (an integer: the quantisation of Ct is exact in rows AND columns)
//   k_cert_split        the residues of an operand given as a double-double (hi, lo) -- or a plain
//                       FP64 matrix -- with its quantisation error sum_k d_rk^2 and sum_k |x_rk| per row
// Residues of y + 2^63 (|y| <= 2^62 + 2^10 here: the double-double rows may exceed 2^b by a few ulps).
// =========================================================================================
template <int M, bool UNS>
__device__ __forceinline__ uint32_t cert_res8(uint32_t lo, uint32_t hi) {
  constexpr uint32_t h = UNS ? 0u : M == 256 ? 128 : (M - 1) / 2;
  constexpr uint32_t w0 = 1u % M, w1 = (1u << 8) % M, w2 = (1u << 16) % M, w3 = (1u << 24) % M;
  constexpr uint32_t w4 = (uint32_t)((1ull << 32) % M), w5 = (uint32_t)((1ull << 40) % M);
  constexpr uint32_t w6 = (uint32_t)((1ull << 48) % M), w7 = (uint32_t)((1ull << 56) % M);
  constexpr uint32_t KL = w0 | (w1 << 8) | (w2 << 16) | (w3 << 24), KH = w4 | (w5 << 8) | (w6 << 16) | (w7 << 24);
  constexpr uint32_t K3 = (uint32_t)((h + M - (uint32_t)((1ull << 63) % M)) % M);
  constexpr uint32_t MAG = (uint32_t)(((1ull << 32) + M - 1) / M);
  if (UNS && M == 256) return lo;                 // y mod 256: the low byte (2^63 = 0 mod 256)
  const uint32_t r = __dp4a(hi, KH, __dp4a(lo, KL, K3));
  const uint32_t u = r - __umulhi(r, MAG) * (uint32_t)M;
  return UNS ? u : u - h;
}
template <int L, bool UNS>
__device__ __forceinline__ void cert_split4(const uint32_t (&lo)[4], const uint32_t (&hi)[4], int nm, int8_t *dst,
                                            int64_t plane) {
  if constexpr (L < CRT_MAX) {
    if (L < nm) {
      uint32_t b[4];
      #pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = cert_res8<kModuli[L], UNS>(lo[u], hi[u]);
      *(uint32_t *)(dst + (int64_t)L * plane) =
          __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
      cert_split4<L + 1, UNS>(lo, hi, nm, dst, plane);
    }
  }
}
// 2^e x exactly for |e| <= 2000 (two power-of-two factors)
__device__ __forceinline__ double scale2(double x, int e) { return __dmul_rn(__dmul_rn(x, pow2(e / 2)), pow2(e - e / 2)); }
__device__ __forceinline__ double row_absmax(const double *x, int64_t cols, double *red) {
  double mx = 0.0;
  for (int64_t k = threadIdx.x; k < cols; k += blockDim.x) mx = fmax(mx, fabs(x[k]));
  #pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]);
    red[0] = fmax(mx, red[0]);
  }
  __syncthreads();
  return red[0];
}
// exponent rule of the split (k_crt_split): scaled row maximum in [2^(b-1), 2^b); 0 for a zero row.
// Rows outside |e| <= 400 (maxima beyond 2^+-340) are flagged: the certificate then falls back.
__device__ __forceinline__ int cert_exp(double mx, int b, bool *ok) {
  if (!(mx > 0.0)) { *ok = mx == 0.0; return 0; }
  const int e = b - 1 - ilogb(mx);
  *ok = e >= -400 && e <= 400;
  return e;
}

__global__ void __launch_bounds__(256) k_cert_rowexp(const double *__restrict__ X, int64_t ld, int64_t cols, int b,
                                                     int *sig, double *scale) {
  __shared__ double red[8];
  const int64_t r = blockIdx.x;
  const double mx = row_absmax(X + r * ld, cols, red);
  bool ok;
  const int e = cert_exp(mx, b, &ok);
  if (threadIdx.x == 0) { sig[r] = e; scale[r] = !ok ? NAN : mx > 0.0 ? scale2(1.0, -e) : 0.0; }
}

template <bool UNS>
__global__ void __launch_bounds__(256, 3) k_cert_round_split(const double *Xin, double *X, int64_t ld, int64_t rows,
                                                             int64_t cols, int nm, const int *__restrict__ sig,
                                                             int8_t *planes, double *asum) {
  __shared__ double red[8];
  double as = 0.0;
  const int64_t r = blockIdx.x;
  const double *xi = Xin + r * ld;                 // the candidate (may be X itself: in place)
  double *x = X + r * ld;
  const int er = sig[r];
  const int64_t plane = rows * cols;
  for (int64_t k0 = (int64_t)threadIdx.x * 4; k0 < cols; k0 += (int64_t)blockDim.x * 4) {
    uint32_t lo[4], hi[4];
    double v[4];
    const double2 a = *(const double2 *)(xi + k0), c = *(const double2 *)(xi + k0 + 2);
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
    const int4 ek = *(const int4 *)(sig + k0);
    const int es[4] = {ek.x, ek.y, ek.z, ek.w};
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int g = min(er, es[u]);
      v[u] = scale2(rint(scale2(v[u], g)), -g);                    // Ct_rk on the grid 2^-g (exact)
      as += fabs(v[u]);
      const uint64_t y = (uint64_t)__double2ll_rn(scale2(v[u], er)) + (1ull << 63);   // 2^e_r Ct_rk: an integer
      lo[u] = (uint32_t)y; hi[u] = (uint32_t)(y >> 32);
    }
    *(double2 *)(x + k0) = make_double2(v[0], v[1]);
    *(double2 *)(x + k0 + 2) = make_double2(v[2], v[3]);
    cert_split4<0, UNS>(lo, hi, nm, planes + r * cols + k0, plane);
  }
  if (asum) {                                                        // sum_k |Ct_rk| (||Ct||_inf, p >= 3)
    as = block_sum_det<256>(as, red);
    if (threadIdx.x == 0) asum[r] = as;
  }
}

template <bool UNS, bool LO>
__global__ void __launch_bounds__(256, 3) k_cert_split(const double *__restrict__ Xh, const double *__restrict__ Xl,
                                                       int64_t ld, int64_t plane, int64_t cols, int b, int nm,
                                                       int8_t *planes, int *sig, double *scale, double *err2,
                                                       double *asum) {
  __shared__ double red[8];
  const int64_t r = blockIdx.x;
  const double *xh = Xh + r * ld;
  const double *xl = LO ? Xl + r * ld : nullptr;
  const double mx = row_absmax(xh, cols, red);
  bool ok;
  const int e = cert_exp(mx, b, &ok);
  double es = 0.0, as = 0.0;
  for (int64_t k0 = (int64_t)threadIdx.x * 4; k0 < cols; k0 += (int64_t)blockDim.x * 4) {
    uint32_t lo[4], hi[4];
    double vh[4], vl[4] = {0.0, 0.0, 0.0, 0.0};
    {
      const double2 a = *(const double2 *)(xh + k0), c = *(const double2 *)(xh + k0 + 2);
      vh[0] = a.x; vh[1] = a.y; vh[2] = c.x; vh[3] = c.y;
    }
    if (LO) {
      const double2 a = *(const double2 *)(xl + k0), c = *(const double2 *)(xl + k0 + 2);
      vl[0] = a.x; vl[1] = a.y; vl[2] = c.x; vl[3] = c.y;
    }
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      as += fabs(vh[u]) + fabs(vl[u]);
      const double hs = scale2(vh[u], e), ls = scale2(vl[u], e);
      long long y;
      double d;
      if (fabs(hs) >= 4503599627370496.0) {                      // hs an integer: y = hs + rint(ls)
        const double fl = rint(ls);
        y = __double2ll_rn(hs) + __double2ll_rn(fl);
        d = __dsub_rn(ls, fl);
      } else {                                                     // |ls| <= ulp(hs) / 2 <= 1/4
        const double fh = rint(hs);
        y = __double2ll_rn(fh);
        d = __dadd_rn(__dsub_rn(hs, fh), ls);                      // hs - fh exact
      }
      es = __fma_rn(d, d, es);
      const uint64_t yy = (uint64_t)y + (1ull << 63);
      lo[u] = (uint32_t)yy; hi[u] = (uint32_t)(yy >> 32);
    }
    cert_split4<0, UNS>(lo, hi, nm, planes + r * cols + k0, plane);
  }
  es = block_sum_det<256>(es, red);
  __syncthreads();
  as = block_sum_det<256>(as, red);
  if (threadIdx.x == 0) {
    sig[r] = e;
    scale[r] = !ok ? NAN : mx > 0.0 ? scale2(1.0, -e) : 0.0;
    err2[r] = !ok ? NAN : scale2(es, -2 * e);                    // sum_k (2^-e d_rk)^2
    asum[r] = as;
  }
}

cudaError_t launch_cert_rowexp(const double *X, int64_t ld, int64_t rows, int64_t cols, int b, int *sig, double *scale,
                               cudaStream_t s) {
  k_cert_rowexp<<<(unsigned)rows, 256, 0, s>>>(X, ld, cols, b, sig, scale);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t launch_cert_round_split(const double *Xin, double *X, int64_t ld, int64_t rows, int64_t cols, int nm,
                                    const int *sig, int8_t *planes, double *asum, cudaStream_t s) {
  if (nm < 2 || nm > CRT_MAX || cols % 4 || ld % 2) return cudaErrorInvalidValue;
  if (crt_unsigned(cols)) k_cert_round_split<true><<<(unsigned)rows, 256, 0, s>>>(Xin, X, ld, rows, cols, nm, sig, planes, asum);
  else k_cert_round_split<false><<<(unsigned)rows, 256, 0, s>>>(Xin, X, ld, rows, cols, nm, sig, planes, asum);
  ++g_launches;
  return cudaGetLastError();
}
cudaError_t launch_cert_split(const double *Xh, const double *Xl, int64_t ld, int64_t rows, int64_t cols, int b, int nm,
                              int8_t *planes, int64_t pstride, int *sig, double *scale, double *err2, double *asum,
                              cudaStream_t s) {
  if (b < 2 || b > CRT_BMAX || nm < 2 || nm > CRT_MAX || cols % 4 || ld % 2) return cudaErrorInvalidValue;
  const bool uns = crt_unsigned(cols);
  const int64_t plane = pstride ? pstride : rows * cols;
#define CERT_SPLIT(U, L) k_cert_split<U, L><<<(unsigned)rows, 256, 0, s>>>(Xh, Xl, ld, plane, cols, b, nm, planes, sig, scale, err2, asum)
  if (uns) { if (Xl) CERT_SPLIT(true, true); else CERT_SPLIT(true, false); }
  else { if (Xl) CERT_SPLIT(false, true); else CERT_SPLIT(false, false); }
#undef CERT_SPLIT
  ++g_launches;
  return cudaGetLastError();
}

// Deterministic reductions of the per-row certificate quantities: out[q] = sum (op 0) or max (op 1) of
// v[q][0 .. len) (NaN propagates through both), one block, fixed order.
struct CertStatArgs { const double *v[8]; int op[8]; };
__global__ void __launch_bounds__(256) k_cert_stats(const CertStatArgs a, int nv, int64_t len, double *out) {
  __shared__ double red[8];
  for (int q = 0; q < nv; ++q) {
    const double *x = a.v[q];
    const bool mx = a.op[q] != 0;
    double t = 0.0;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
      const double y = x[i];
      t = mx ? ((y > t || y != y) ? y : t) : t + y;
    }
    if (!mx) {
      t = block_sum_det<256>(t, red);
    } else {
      #pragma unroll
      for (int o = 16; o > 0; o >>= 1) { const double y = __shfl_xor_sync(0xffffffffu, t, o); t = (y > t || y != y) ? y : t; }
      __syncthreads();
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
      __syncthreads();
      if (threadIdx.x == 0) for (int w = 0; w < 8; ++w) t = (red[w] > t || red[w] != red[w]) ? red[w] : t;
    }
    if (threadIdx.x == 0) out[q] = t;
    __syncthreads();
  }
}
cudaError_t launch_cert_stats(const double *const *v, const int *op, int nv, int64_t len, double *out, cudaStream_t s) {
  if (nv < 1 || nv > 8) return cudaErrorInvalidValue;
  CertStatArgs a;
  memset(&a, 0, sizeof a);
  for (int q = 0; q < nv; ++q) { a.v[q] = v[q]; a.op[q] = op[q]; }
  k_cert_stats<<<1, 256, 0, s>>>(a, nv, len, out);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace ipr
