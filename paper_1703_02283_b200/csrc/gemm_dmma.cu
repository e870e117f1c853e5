// gemm_dmma.cu -- FP64 GEMM of the hot path on the FP64 tensor pipe (SASS DMMA.8x8x4).
//
// tcgen05.mma has no f64 kind on sm_100a (ptxas 12.9), so FP64 phases use the
// warp-level mma.sync.aligned.m8n8k4.row.col.f64 (DMMA), fed by a 4-stage cp.async
// (LDGSTS) shared-memory pipeline.  On B200 the DMMA issue peak measured 37.1 TFLOP/s
// (profiles/r01_calibration.md).
//
// Tile 128 x 64 x 16 per CTA, 4 warps (2 x 2) with 64 x 32 warp tiles = 8 x 4 DMMA tiles and
// 64 FP64 accumulators per thread; two CTAs per SM (8 warps/SM) so one CTA's barrier / refill
// bubble is covered by the other -- the tiling sweep in tools/probes/dmma_variants.cu measured
// 34.3 TFLOP/s for this shape vs 31.6 for one 128 x 128 CTA per SM.  K inside a 16-block is
// visited in pairs so every thread fetches its two A (and B) fragment values with ONE 16-byte
// ld.shared; the pairing is the same for A and B, so each DMMA contracts matching k.  Shared
// rows are 128 B with 16-byte chunks XOR-swizzled by (row & 1) << 2 -> conflict-free LDS.128.
// All sizes are padded to multiples of 128 by the engine (zero padding), so the main loop has
// no bounds checks.  Each output element is produced by exactly one CTA with a fixed K order
// -> bit-reproducible and independent of the column-panel sharding.
#include "common.cuh"
#include "epilogue.cuh"

namespace ipr {

constexpr int DM_BM = 128, DM_BN = 64, DM_BK = 16, DM_ST = 4, DM_NT = 128;
constexpr int DM_GROUP_M = 16;
constexpr int DM_STAGE_DBL = DM_BM * DM_BK + DM_BN * DM_BK;     // doubles per stage
constexpr int DM_SMEM = DM_ST * DM_STAGE_DBL * 8;               // 98304 bytes

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ int swz(int row, int chunk) { return chunk ^ ((row & 1) << 2); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(DM_NT, 2) k_gemm_dmma(const GemmArgs g) {
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;              // 2 x 2 warps
  // grouped raster: consecutive CTAs sweep DM_GROUP_M tile-rows x all tile-columns, so the A and B
  // K-slices a wave touches are shared across many CTAs through L2 (DRAM re-reads / 3 vs row-major)
  int tm, tn;
  {
    const int tiles_m = (int)(g.M / DM_BM), tiles_n = (int)(g.N / DM_BN);
    const int per_group = DM_GROUP_M * tiles_n, bid = blockIdx.x;
    const int gidx = bid / per_group, first_m = gidx * DM_GROUP_M;
    const int gm = min(tiles_m - first_m, DM_GROUP_M);
    const int r = bid - gidx * per_group;
    tm = first_m + r % gm;
    tn = r / gm;
  }
  const int64_t m0 = (int64_t)tm * DM_BM, n0 = (int64_t)tn * DM_BN;
  if (g.tri && m0 > g.col0 + n0 + DM_BN - 1) {          // wholly below the diagonal (tri form)
    if (tid == 0 && (g.mode & EPI_RESID)) g.part[((g.col0 + n0) / DM_BN) * g.tiles_m + g.row0 / DM_BM + tm] = 0.0;
    return;
  }
  const double *A = (const double *)g.A, *B = (const double *)g.B;
  const int nkb = (int)(g.K / DM_BK);
  const int kb_per_panel = (int)(g.a_kp / DM_BK);
  const int kb_per_bpanel = (int)((g.b_kp ? g.b_kp : g.a_kp) / DM_BK);   // paneled B (2-D grid T panels)

  auto sA = [&](int s) { return smem + s * DM_STAGE_DBL; };
  auto sB = [&](int s) { return smem + s * DM_STAGE_DBL + DM_BM * DM_BK; };

  auto load_stage = [&](int s, int kb) {
    const int panel = kb / kb_per_panel, kin = (kb - panel * kb_per_panel) * DM_BK;
    const double *Ap = A + (int64_t)panel * g.a_pstride + kin + m0 * g.a_kp;
    const int bpanel = g.b_pstride ? kb / kb_per_bpanel : 0;
    const double *Bp = B + (int64_t)bpanel * g.b_pstride + n0 * g.ldb + (int64_t)(kb - bpanel * kb_per_bpanel) * DM_BK;
    double *a = sA(s), *b = sB(s);
    #pragma unroll
    for (int i = 0; i < 8; ++i) {            // A: 128 rows x 8 chunks
      const int idx = tid + i * DM_NT, r = idx >> 3, c = idx & 7;
      cp_async16(a + r * DM_BK + swz(r, c) * 2, Ap + r * g.a_kp + c * 2);
    }
    #pragma unroll
    for (int i = 0; i < 4; ++i) {            // B: 64 rows x 8 chunks
      const int idx = tid + i * DM_NT, r = idx >> 3, c = idx & 7;
      cp_async16(b + r * DM_BK + swz(r, c) * 2, Bp + r * g.ldb + c * 2);
    }
  };

  double acc[8][4][2];
  #pragma unroll
  for (int i = 0; i < 8; ++i)
    #pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  #pragma unroll
  for (int s = 0; s < DM_ST - 1; ++s) {
    if (s < nkb) load_stage(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int kb = 0; kb < nkb; ++kb) {
    cp_async_wait<DM_ST - 2>();
    __syncthreads();
    {
      const int nk = kb + DM_ST - 1;
      if (nk < nkb) load_stage(nk % DM_ST, nk);
      cp_async_commit();
    }
    const double *a = sA(kb % DM_ST), *b = sB(kb % DM_ST);
    #pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int chunk = kk * 4 + fk;
      double2 af[8], bf[4];
      #pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        const int r = wm * 64 + mi * 8 + fr;
        af[mi] = *(const double2 *)(a + r * DM_BK + swz(r, chunk) * 2);
      }
      #pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int r = wn * 32 + ni * 8 + fr;
        bf[ni] = *(const double2 *)(b + r * DM_BK + swz(r, chunk) * 2);
      }
      #pragma unroll
      for (int mi = 0; mi < 8; ++mi)
        #pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi].x, bf[ni].x);
      #pragma unroll
      for (int mi = 0; mi < 8; ++mi)
        #pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi].y, bf[ni].y);
    }
  }
  cp_async_wait<0>();

  // ---- fused epilogue (per element, fixed order) ----
  double scale = 1.0;
  if (g.sigA) scale = pow2(-(*g.sigA + *g.sigB));
  EpiAcc ea{0.0, 0.0, 0.0f};
  #pragma unroll
  for (int mi = 0; mi < 8; ++mi)
    #pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      #pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t row = g.row0 + m0 + wm * 64 + mi * 8 + fr;   // global row (2-D grid: row0)
        const int64_t col = n0 + wn * 32 + ni * 8 + fk * 2 + e;
        epi_element<MODE>(g, row, col, __dmul_rn(acc[mi][ni][e], scale), ea);
      }
  __shared__ double red[DM_NT / 32];
  __shared__ float redf[DM_NT / 32];
  const int mode = MODE >= 0 ? MODE : g.mode;
  const int64_t tile = ((g.col0 + n0) / DM_BN) * g.tiles_m + g.row0 / DM_BM + tm;
  if (mode & (EPI_RESID | EPI_UPDATE | EPI_NSUPDATE)) {
    const double s = block_sum_det<DM_NT>((mode & EPI_RESID) ? ea.r2 : ea.d2, red);
    if (tid == 0) g.part[tile] = s;
  }
  if (g.pmax) {
    const float s = block_max<DM_NT>(ea.mx, redf);
    if (tid == 0) g.pmax[tile] = s;
  }
}

template <int MODE>
static cudaError_t launch_mode(const GemmArgs &a, cudaStream_t s) {
  static DeviceOnce attr;
  if (!attr.done()) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_dmma<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, DM_SMEM);
    if (e != cudaSuccess) return e;
    attr.set();
  }
  dim3 grid((unsigned)((a.N / DM_BN) * (a.M / DM_BM)));
  k_gemm_dmma<MODE><<<grid, DM_NT, DM_SMEM, s>>>(a);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_gemm_dmma(const GemmArgs &a_in, cudaStream_t s) {
  GemmArgs a = a_in;
  if (!a.mout) { a.mout = a.tout; a.ldm = a.ldt; }   // tri mirror: in place at G = 1
  if (a.M % DM_BM || a.N % DM_BN || a.K % DM_BK || a.a_kp % DM_BK) return cudaErrorInvalidValue;
  // the hot-path modes get specialised kernels; anything else uses the runtime-mode build
  if (!a.pmax && a.prec == P_FP64) {
    if (a.mode == EPI_STORE_T) return launch_mode<EPI_STORE_T>(a, s);
    if (a.mode == EPI_STORE_N) return launch_mode<EPI_STORE_N>(a, s);
    if (a.mode == (EPI_STORE_T | EPI_STORE_N)) return launch_mode<EPI_STORE_T | EPI_STORE_N>(a, s);
    if (a.mode == (EPI_STORE_T | EPI_RESID)) return launch_mode<EPI_STORE_T | EPI_RESID>(a, s);
    if (a.mode == EPI_RESID) return launch_mode<EPI_RESID>(a, s);
    if (a.mode == (EPI_STORE_T | EPI_DIAG_MINUS | EPI_RESID))
      return launch_mode<EPI_STORE_T | EPI_DIAG_MINUS | EPI_RESID>(a, s);
    if (a.mode == EPI_WSTORE) return launch_mode<EPI_WSTORE>(a, s);
    if (a.mode == EPI_UPDATE && a.cont64 && !a.chat_new) return launch_mode<EPI_UPDATE>(a, s);
  }
  return launch_mode<-1>(a, s);
}

int dmma_tile_n() { return DM_BN; }

}  // namespace ipr
