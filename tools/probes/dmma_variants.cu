// Probe: FP64 DMMA GEMM tiling variants at n = 8192 (plain store epilogue).  Used to choose the
// configuration of paper_1703_02283_b200/csrc/gemm_dmma.cu.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N> __device__ __forceinline__ void wait_g() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
// BK doubles per row = BK*8 bytes = BK/2 chunks of 16 B; swizzle chunk ^ ((row&1)<<2) within 8-chunk groups
template <int BK> __device__ __forceinline__ int sw(int row, int c) { return c ^ ((row & 1) << 2); }

// WTM x WTN warp tile = (WTM/8) x (WTN/8) DMMA tiles
template <int BM, int BN, int BK, int ST, int WM, int WN, int MINB>
__global__ void __launch_bounds__(WM * WN * 32, MINB) kgemm(const double *A, const double *B, double *C, int n) {
  constexpr int NT = WM * WN * 32, WTM = BM / WM, WTN = BN / WN, MI = WTM / 8, NI = WTN / 8;
  constexpr int CH = BK / 2;  // 16B chunks per row
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int nkb = n / BK;
  auto sA = [&](int s) { return smem + s * (BM + BN) * BK; };
  auto sB = [&](int s) { return smem + s * (BM + BN) * BK + BM * BK; };
  auto load = [&](int s, int kb) {
    const int64_t k0 = (int64_t)kb * BK;
    for (int idx = tid; idx < BM * CH; idx += NT) {
      const int r = idx / CH, c = idx % CH;
      cp_async16(sA(s) + r * BK + sw<BK>(r, c) * 2, A + (m0 + r) * n + k0 + c * 2);
    }
    for (int idx = tid; idx < BN * CH; idx += NT) {
      const int r = idx / CH, c = idx % CH;
      cp_async16(sB(s) + r * BK + sw<BK>(r, c) * 2, B + (n0 + r) * n + k0 + c * 2);
    }
  };
  double acc[MI][NI][2];
  #pragma unroll
  for (int i = 0; i < MI; ++i)
    #pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  #pragma unroll
  for (int s = 0; s < ST - 1; ++s) { if (s < nkb) load(s, s); commit(); }
  const int fr = lane >> 2, fk = lane & 3;
  for (int kb = 0; kb < nkb; ++kb) {
    wait_g<ST - 2>();
    __syncthreads();
    { const int nk = kb + ST - 1; if (nk < nkb) load(nk % ST, nk); commit(); }
    const double *a = sA(kb % ST), *b = sB(kb % ST);
    #pragma unroll
    for (int kk = 0; kk < BK / 8; ++kk) {
      const int chunk = kk * 4 + fk;
      double2 af[MI], bf[NI];
      #pragma unroll
      for (int mi = 0; mi < MI; ++mi) { const int r = wm * WTM + mi * 8 + fr; af[mi] = *(const double2 *)(a + r * BK + sw<BK>(r, chunk) * 2); }
      #pragma unroll
      for (int ni = 0; ni < NI; ++ni) { const int r = wn * WTN + ni * 8 + fr; bf[ni] = *(const double2 *)(b + r * BK + sw<BK>(r, chunk) * 2); }
      #pragma unroll
      for (int mi = 0; mi < MI; ++mi)
        #pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], af[mi].x, bf[ni].x);
      #pragma unroll
      for (int mi = 0; mi < MI; ++mi)
        #pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni], af[mi].y, bf[ni].y);
    }
  }
  wait_g<0>();
  #pragma unroll
  for (int mi = 0; mi < MI; ++mi)
    #pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int64_t row = m0 + wm * WTM + mi * 8 + fr, col = n0 + wn * WTN + ni * 8 + fk * 2;
      *(double2 *)(C + row * n + col) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
    }
}

template <int BM, int BN, int BK, int ST, int WM, int WN, int MINB>
void run(const char *name, const double *A, const double *B, double *C, int n) {
  auto k = kgemm<BM, BN, BK, ST, WM, WN, MINB>;
  const int smem = ST * (BM + BN) * BK * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  dim3 grid(n / BN, n / BM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<grid, WM * WN * 32, smem>>>(A, B, C, n);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k<<<grid, WM * WN * 32, smem>>>(A, B, C, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  printf("%-40s regs=%3d smem=%6d : %.2f TFLOP/s  (%s)\n", name, fa.numRegs, smem, 2.0 * n * n * (double)n * 3 / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

__global__ void fill(double *x, int64_t len, uint64_t seed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < len) { uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed; z ^= z >> 29; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 32; x[i] = (double)(z % 2001) / 1000.0 - 1.0; }
}

int main() {
  const int n = 8192;
  double *A, *B, *C;
  cudaMalloc(&A, (size_t)n * n * 8); cudaMalloc(&B, (size_t)n * n * 8); cudaMalloc(&C, (size_t)n * n * 8);
  fill<<<(n * (int64_t)n + 255) / 256, 256>>>(A, (int64_t)n * n, 1);
  fill<<<(n * (int64_t)n + 255) / 256, 256>>>(B, (int64_t)n * n, 2);
  run<128, 64, 16, 4, 4, 2, 2>("128x64x16 st4 w4x2 2cta", A, B, C, n);
  run<128, 64, 16, 3, 4, 2, 2>("128x64x16 st3 w4x2 2cta", A, B, C, n);
  run<128, 64, 16, 5, 4, 2, 2>("128x64x16 st5 w4x2 2cta", A, B, C, n);
  run<128, 64, 32, 2, 4, 2, 2>("128x64x32 st2 w4x2 2cta", A, B, C, n);
  run<128, 64, 16, 4, 2, 2, 2>("128x64x16 st4 w2x2 2cta (64x32)", A, B, C, n);
  run<64, 64, 16, 6, 2, 2, 4>("64x64x16 st6 w2x2 4cta", A, B, C, n);
  run<64, 64, 32, 3, 2, 2, 4>("64x64x32 st3 w2x2 4cta", A, B, C, n);
  run<128, 64, 16, 4, 2, 2, 3>("128x64x16 st4 w2x2 3cta", A, B, C, n);
  run<64, 128, 16, 4, 2, 2, 2>("64x128x16 st4 w2x2 2cta (32x64)", A, B, C, n);
  run<128, 32, 16, 4, 4, 1, 3>("128x32x16 st4 w4x1 3cta", A, B, C, n);
  return 0;
}
