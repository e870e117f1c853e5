// tools/probes/crt_split_probe.cu -- standalone timing of the CRT residue split (k_crt_split of
// ozaki.cu, copied) with and without its row-maximum pass (measurement only, not the product path).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int CRT_MAX = 18;
constexpr int kModuli[CRT_MAX] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193, 191, 181};
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)((uint64_t)(1023 + e) << 52)); }
// Symmetric residue byte of y = c2 2^42 + c1 2^21 + c0 - 2^62 modulo the compile-time modulus M
// (c0, c1, c2 in [0, 2^21): the caller biased y by 2^62).  Integer ALU only, ~7 operations:
// r = c0 + c1 K1 + c2 K2 + K3 < 2^30 (K3 = h - 2^62 mod M, h = the symmetric offset), u = r mod M
// by an exact multiply-high (x < 2^30, magic ceil(2^39 / M) < 2^32: error < 2^-9 < 1/M), v = u - h.
template <int M>
__device__ __forceinline__ uint32_t crt_res8(uint32_t c0, uint32_t c1, uint32_t c2) {
  constexpr uint32_t h = M == 256 ? 128 : (M - 1) / 2;
  constexpr uint32_t K1 = (1u << 21) % M, K2 = (uint32_t)((1ull << 42) % M);
  constexpr uint32_t K3 = (uint32_t)((h + M - (uint32_t)((1ull << 62) % M)) % M);
  constexpr uint32_t MAG = (uint32_t)(((1ull << 39) + M - 1) / M);
  const uint32_t r = c2 * K2 + (c1 * K1 + (c0 + K3));
  const uint32_t u = r - (__umulhi(r, MAG) >> 7) * (uint32_t)M;
  return u - h;                                   // the low byte is the residue (packed by PRMT)
}
template <int L>
__device__ __forceinline__ void crt_split4(const uint32_t (&c0)[4], const uint32_t (&c1)[4], const uint32_t (&c2)[4],
                                           int nm, int8_t *dst, int64_t plane) {
  if constexpr (L < CRT_MAX) {
    if (L < nm) {
      uint32_t b[4];
      #pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = crt_res8<kModuli[L]>(c0[u], c1[u], c2[u]);
      *(uint32_t *)(dst + (int64_t)L * plane) =
          __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
      crt_split4<L + 1>(c0, c1, c2, nm, dst, plane);
    }
  }
}

// Residues of the rows of X (FP64, row-major, leading dimension ld): one block per row; plane l of
// `planes` holds (Xbar mod m_l) at planes[l * rows * cols + r * cols + k]; sig[r] = e_r.
__global__ void __launch_bounds__(256, 4) k_split_full(const double *__restrict__ X, int64_t ld, int64_t rows, int64_t cols,
                                                   int b, int nm, int8_t *planes, int *sig) {
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
  // scaled row maximum in [2^(b-1), 2^b): |Xbar| <= 2^b <= 2^62
  const int e = (mx > 0.0) ? b - 1 - ilogb(mx) : 0;
  if (threadIdx.x == 0) sig[r] = e;
  const double sc = pow2(e);
  const int64_t plane = rows * cols;
  for (int64_t k0 = (int64_t)threadIdx.x * 4; k0 < cols; k0 += (int64_t)blockDim.x * 4) {
    uint32_t c0[4], c1[4], c2[4];
    const double2 *xp = (const double2 *)(x + k0);
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 t = xp[u >> 1];
      // Xbar + 2^62 in [0, 2^63): three 21-bit fields
      const uint64_t y = (uint64_t)__double2ll_rn(__dmul_rn((u & 1) ? t.y : t.x, sc)) + (1ull << 62);
      c0[u] = (uint32_t)y & 0x1fffffu; c1[u] = (uint32_t)(y >> 21) & 0x1fffffu; c2[u] = (uint32_t)(y >> 42);
    }
    crt_split4<0>(c0, c1, c2, nm, planes + r * cols + k0, plane);
  }
}


// variant: exponents given (no max pass)
__global__ void __launch_bounds__(256, 4) k_split_noexp(const double *__restrict__ X, int64_t ld, int64_t rows, int64_t cols,
                                                   int b, int nm, int8_t *planes, const int *sig) {
  const int64_t r = blockIdx.x;
  const double *x = X + r * ld;
  const double sc = pow2(sig[r]);
  const int64_t plane = rows * cols;
  for (int64_t k0 = (int64_t)threadIdx.x * 4; k0 < cols; k0 += (int64_t)blockDim.x * 4) {
    uint32_t c0[4], c1[4], c2[4];
    const double2 *xp = (const double2 *)(x + k0);
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double2 t = xp[u >> 1];
      const uint64_t y = (uint64_t)__double2ll_rn(__dmul_rn((u & 1) ? t.y : t.x, sc)) + (1ull << 62);
      c0[u] = (uint32_t)y & 0x1fffffu; c1[u] = (uint32_t)(y >> 21) & 0x1fffffu; c2[u] = (uint32_t)(y >> 42);
    }
    crt_split4<0>(c0, c1, c2, nm, planes + r * cols + k0, plane);
  }
}
// variant: only the max pass
__global__ void __launch_bounds__(256) k_maxonly(const double *__restrict__ X, int64_t ld, int64_t cols, int b, int *sig) {
  __shared__ double red[8];
  const int64_t r = blockIdx.x;
  const double *x = X + r * ld;
  double mx = 0.0;
  for (int64_t k = threadIdx.x; k < cols; k += blockDim.x) mx = fmax(mx, fabs(x[k]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) { for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w]); sig[r] = b - 1 - ilogb(mx); }
}
__global__ void fill(double *x, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { uint32_t h = (uint32_t)i * 2654435761u; h ^= h >> 13; x[i] = ((double)(h & 0xffffff) / 8388608.0 - 1.0) * 1e-3; }
}
int main() {
  const int64_t n = 8192;
  double *X; int8_t *P; int *sig;
  cudaMalloc(&X, n * n * 8); cudaMalloc(&P, n * n * 18); cudaMalloc(&sig, n * 4);
  fill<<<(unsigned)((n * n + 255) / 256), 256>>>(X, n * n);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int nm : {17, 10}) {
    float t[3] = {0, 0, 0};
    for (int v = 0; v < 3; ++v) {
      for (int rep = 0; rep < 6; ++rep) {
        if (rep == 1) cudaEventRecord(a);
        if (v == 0) k_split_full<<<(unsigned)n, 256>>>(X, n, n, n, 59, nm, P, sig);
        else if (v == 1) k_split_noexp<<<(unsigned)n, 256>>>(X, n, n, n, 59, nm, P, sig);
        else k_maxonly<<<(unsigned)n, 256>>>(X, n, n, 59, sig);
      }
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&t[v], a, b);
    }
    printf("nm=%d full %.3f ms  no-max %.3f ms  max-only %.3f ms  (%s)\n", nm, t[0] / 5, t[1] / 5, t[2] / 5,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
