// gemm_tc.cu -- tcgen05 GEMM of the hot path for the reduced-precision phases (BF16, FP16 and
// TF32 operands, FP32 accumulation in TMEM).  D = Chat * X, one of:
// T_j = Chat T_{j-1} (stored transposed in the operand format), the fused residual, or the
// fused FP64 update C_{k+1} = q_m(((p+1) C_k - P) / p)  (epilogue.cuh, readings R-1/R-2/R-4).
//
// Design (sm_100a): persistent kernel, clusters of 2 CTAs (a CTA pair on one TPC) computing
// 256 x 256 output tiles with tcgen05.mma.cta_group::2 (M = 256, N = 256):
//   warp 0     TMA producer (both CTAs): each CTA loads its 128 rows of A and its 128 rows of
//              B per 128-byte K-block (SWIZZLE_128B) into a 6-stage ring; completion bytes of
//              both CTAs land on the leader CTA's mbarrier
//   warp 1     MMA issuer (leader CTA, one thread): 4 x tcgen05.mma per K-block, commits
//              multicast to both CTAs' "stage empty" / "accumulator full" mbarriers
//   warps 2-9  epilogue (both CTAs): tcgen05.ld 32x32b.x32 (thread = accumulator row) ->
//              FP64 epilogue -> global; warp w reads TMEM lane quarter w % 4 and column
//              half (w - 2) / 4, so two warps share each quarter
// Each CTA keeps two 128 x 256 FP32 accumulators (all 512 TMEM columns), so the epilogue of
// tile i overlaps the MMAs of tile i+1.  Per SM and K-block the operands are 32 KB for 128 x 256
// outputs (a 1-CTA 128 x 256 tile needs 48 KB), which keeps the L2 -> SM traffic under the
// L2 bandwidth.  Pair tiles are visited in groups of 8 along M for L2 reuse.
// Each output element is produced by one CTA with a fixed K order (deterministic; identical
// for any column-panel sharding).
#include <cuda.h>
#include <cstdio>

#include "common.cuh"
#include "epilogue.cuh"

namespace ipr {

constexpr int TC_BM = 128;            // rows per CTA (256 per pair)
constexpr int TC_BN = 256;            // columns per pair tile
constexpr int TC_BKB = 128;           // K-block in bytes (one 128-B swizzle row)
constexpr int TC_ST = 6, TC_NT = 320;   // 2 control warps + 8 epilogue warps
constexpr int TC_A_BYTES = TC_BM * TC_BKB;          // 16 KB
constexpr int TC_B_BYTES = (TC_BN / 2) * TC_BKB;    // 16 KB (this CTA's half of N)
constexpr int TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;
constexpr int TC_SMEM = TC_ST * TC_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
#ifndef IPR_TC_GROUP_M
#define IPR_TC_GROUP_M 8
#endif
constexpr int TC_GROUP_M = IPR_TC_GROUP_M;   // pair-rows per scheduling group
// CRT modulus GEMMs: 16 pair-rows per group -- each B (residue) column block is streamed n / (16 x 256)
// times instead of n / (8 x 256) per modulus (DRAM traffic; the launches are tensor-bound either way)
#ifndef IPR_CRT_GROUP_M
#define IPR_CRT_GROUP_M 16
#endif

bool tc_supported(int prec) {
  return prec == P_BF16 || prec == P_FP16 || prec == P_TF32 || prec == P_FP8 || prec == P_INT8;
}
// partial-sum tile of the kernel that produces a format's GEMM epilogue (P_FP64_OZ finishes inside
// the grouped kind::i8 launch: the tcgen05 tile)
// tcgen05.mma kind of an operand format: 0 kind::f16 (BF16/FP16), 1 kind::tf32, 2 kind::f8f6f4
// (E4M3), 3 kind::i8 (signed).  Every kind consumes 32 bytes of K per instruction.
__host__ __device__ constexpr int tc_kind(int prec) {
  return prec == P_TF32 ? 1 : prec == P_FP8 ? 2 : prec == P_INT8 ? 3 : 0;
}
int gemm_tile_n(int prec) { return prec == P_FP64 ? dmma_tile_n() : TC_BN; }
int gemm_tile_m(int prec) { return 128; }

// ---------------------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// arrive on the mbarrier at the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *b, uint32_t rank) {
  asm volatile(
      "{\n.reg .b32 ra;\nmapa.shared::cluster.u32 ra, %0, %1;\n"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}\n" ::"r"(su32(b)),
      "r"(rank)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// cluster-scope acquire wait (barrier arrived from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// 2-CTA TMA: the transaction bytes complete on the LEADER CTA's barrier (peer bit cleared)
__device__ __forceinline__ void tma_load_3d_pair(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                                 int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];\n" ::"r"(su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n" ::"r"(su32(dst)),
      "l"((uint64_t)map), "r"(su32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// commit all prior MMAs of this thread; arrive on the barrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          su32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int KIND>  // 0: kind::f16 (bf16/fp16), 1: kind::tf32, 2: kind::f8f6f4, 3: kind::i8
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t acc) {
  if (KIND == 0)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  else if (KIND == 1)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  else if (KIND == 2)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row core-matrix groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);          // start address
  d |= (uint64_t)1 << 16;                          // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset
  d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
  return d;
}

// Instruction descriptor: K-major A and B, M = 256 (pair), N = 256.  D format (bits 4-5): F32 = 1,
// S32 = 2 (kind::i8).  A/B formats (bits 7-9 / 10-12): kind::f16 F16 = 0, BF16 = 1; kind::tf32
// TF32 = 2; kind::f8f6f4 E4M3 = 0; kind::i8 signed = 1.
__host__ __device__ constexpr uint32_t make_idesc(int prec, bool u8 = false) {   // u8: kind::i8 unsigned operands
  const uint32_t fmt = prec == P_BF16 ? 1u : prec == P_FP16 ? 0u : prec == P_TF32 ? 2u : prec == P_FP8 ? 0u
                       : u8 ? 0u : 1u;
  const uint32_t dfmt = prec == P_INT8 ? 2u : 1u;
  return (dfmt << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)((2 * TC_BM) >> 4) << 24);
}
// accumulator word -> FP64 (exact): FP32 bits, or INT32 for kind::i8
// (an integer-pipe FP32 -> FP64 conversion measured slower here: 291 -> 321 / 331 us for the FP8 tri GEMM, and
// 4.5 -> 8.5 ms per solve in k_sym_update, r02e/f/i -- the hardware F2F stays)
template <int KIND>
__device__ __forceinline__ double acc_to_f64(uint32_t w) {
  return KIND == 3 ? (double)(int32_t)w : (double)__uint_as_float(w);
}

struct TileSched {      // pair tiles: tiles_m pair-rows (256 rows) x tiles_n (256 columns)
  int tiles_m, tiles_n, tri;
  int coff;             // tri, column panel of a G > 1 rank: global 256-column tile of local tile 0 --
                        // the upper-triangle tiles are tm <= coff + tn (0 for a square single panel)
  int gm = TC_GROUP_M;  // pair-rows per L2 raster group (non-tri)
  // tri (square, symmetric-tri GEMM 2 / fused update): only the upper-triangle pair tiles tm <= tn, in
  // bands of TRI_GC pair-columns, row by row inside a band, so the CTA pairs in flight share their A
  // row blocks (TRI_GC tiles each) and B column blocks (the band) in L2 -- a column-by-column order
  // streamed ~8 GB per K = 2n fused-update GEMM from DRAM
  static constexpr int TRI_GC = 8;
  __host__ __device__ int count() const {
    return tri ? tiles_n * coff + tiles_n * (tiles_n + 1) / 2 : tiles_m * tiles_n;
  }
  __device__ void get(int t, int &tm, int &tn) const {
    if (tri) {
      // the tiles ON the diagonal first (their epilogue takes the slower mixed path): the last wave --
      // whose epilogue nothing overlaps -- then holds only strictly-upper tiles
      if (t < tiles_n) { tm = coff + t; tn = t; return; }
      t -= tiles_n;
      for (int c0 = 0;; c0 += TRI_GC) {                // band [c0, c1): (coff + c0) * w full-width rows, then its diagonal
        const int c1 = min(c0 + TRI_GC, tiles_n), w = c1 - c0, fr = coff + c0;
        const int nb = fr * w + w * (w - 1) / 2;       // (the diagonal tiles went first)
        if (t < nb) {
          if (t < fr * w) { tm = t / w; tn = c0 + t % w; return; }
          t -= fr * w;
          int r = 0;
          while (t >= w - r - 1) { t -= w - r - 1; ++r; }   // diagonal block: row fr + r has w - r - 1 tiles right of it
          tm = fr + r; tn = c0 + r + 1 + t;
          return;
        }
        t -= nb;
      }
    }
    const int per_group = this->gm * tiles_n;
    const int gidx = t / per_group, first_m = gidx * this->gm;
    const int gmm = min(tiles_m - first_m, this->gm);
    const int r = t - gidx * per_group;
    tm = first_m + r % gmm;
    tn = r / gmm;
  }
};

// Store of an updated iterate value to the container (FP32 / FP64) and to an operand (BF16 / TF32).
__device__ __forceinline__ void put_cont(void *base, int64_t idx, int cont64, double v) {
  if (cont64) ((double *)base)[idx] = v;
  else ((float *)base)[idx] = (float)v;
}
__device__ __forceinline__ void put_op(void *base, int64_t idx, int prec, double v) {
  if (prec == P_BF16) ((__nv_bfloat16 *)base)[idx] = __float2bfloat16_rn((float)v);
  else ((float *)base)[idx] = to_tf32((float)v);
}
// EPI_SYMUPD on one 32-column segment of row `row` (reading R-22 with the tri form): the accumulator
// is S_ij = (Chat Rhat + Rhat Chat)_ij (FP32, one accumulation over K = 2n); e = S/(2p) (exact
// reciprocal for p = 2^k), C_{k+1} = q_m(C_ij + e) -- the op order of k_sym_update with s = S -- stored
// at (i,j) and (j,i) in the container and as the next operands, delta partials weighted 2 off the
// diagonal; elements below the diagonal are left to their mirror (bitwise symmetric iterates).
__device__ __forceinline__ void sym_update_chunk(const GemmArgs &g, int64_t row, int64_t col, const uint32_t (&r)[32],
                                                 EpiAcc &ea) {
  const bool pow2p = (g.p & (g.p - 1)) == 0;
  const double tp2 = (double)(2 * g.p), itp = 1.0 / tp2;
  const int64_t plane = g.M * g.ldh;
  const bool upper = row < g.col0 + col;              // the whole segment strictly above the diagonal
  #pragma unroll 1
  for (int j0 = 0; j0 < 32; j0 += 8) {                // not unrolled: compact code (instruction cache)
    double cv[8], cn[8];
    if (g.cont64) {
      const double2 *src = (const double2 *)((const double *)g.cold + row * g.ldc + col + j0);
      #pragma unroll
      for (int q = 0; q < 4; ++q) { const double2 t = src[q]; cv[2 * q] = t.x; cv[2 * q + 1] = t.y; }
    } else {
      const float4 *src = (const float4 *)((const float *)g.cold + row * g.ldc + col + j0);
      #pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float4 t = src[q];
        cv[4 * q] = t.x; cv[4 * q + 1] = t.y; cv[4 * q + 2] = t.z; cv[4 * q + 3] = t.w;
      }
    }
    #pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int64_t c = col + j0 + v, gc = g.col0 + c;
      const double s = (double)__uint_as_float(r[j0 + v]);
      const double e = pow2p ? __dmul_rn(s, itp) : __ddiv_rn(s, tp2);
      const double x = __dadd_rn(cv[v], e);
      cn[v] = g.cont64 ? q_e11(x, g.m, g.rtz) : (double)q_e8(x, g.m, g.rtz);
      if (!upper && row > gc) continue;                // lower triangle: the mirror element's value
      const double dd = __dsub_rn(cn[v], cv[v]);
      ea.d2 = __fma_rn(row != gc ? 2.0 * dd : dd, dd, ea.d2);
      if (row != gc) {                                 // mirror (j, i): coalesced across the warp's rows
        put_cont(g.cnew, c * g.ldc + row, g.cont64, cn[v]);
        if (g.chat_new) put_op(g.chat_new, c * g.ldc + row, g.hprec, cn[v]);
        put_op(g.qnext, c * g.ldh + row, g.tprec, cn[v]);
        put_op(g.qnext, 2 * plane + c * g.ldh + row, g.tprec, cn[v]);
      }
      if (!upper) {                                    // diagonal segment: per-element direct stores
        put_cont(g.cnew, row * g.ldc + c, g.cont64, cn[v]);
        if (g.chat_new) put_op(g.chat_new, row * g.ldc + c, g.hprec, cn[v]);
        put_op(g.qnext, row * g.ldh + c, g.tprec, cn[v]);
        put_op(g.qnext, 2 * plane + row * g.ldh + c, g.tprec, cn[v]);
      }
    }
    if (upper) {                                       // direct (i, j): vector stores of the 8 values
      if (g.cont64) {
        double2 *d = (double2 *)((double *)g.cnew + row * g.ldc + col + j0);
        #pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = make_double2(cn[2 * q], cn[2 * q + 1]);
      } else {
        float4 *d = (float4 *)((float *)g.cnew + row * g.ldc + col + j0);
        #pragma unroll
        for (int q = 0; q < 2; ++q)
          d[q] = make_float4((float)cn[4 * q], (float)cn[4 * q + 1], (float)cn[4 * q + 2], (float)cn[4 * q + 3]);
      }
      #pragma unroll
      for (int o = 0; o < 3; ++o) {                    // chat_new (prec), qnext planes 0 and 2 (tprec)
        void *base = o == 0 ? g.chat_new : g.qnext;
        if (!base) continue;
        const int pr = o == 0 ? g.hprec : g.tprec;
        const int64_t idx = (o == 0 ? row * g.ldc : (o == 2 ? 2 * plane : 0) + row * g.ldh) + col + j0;
        if (pr == P_BF16) {
          uint32_t w[4];
          #pragma unroll
          for (int q = 0; q < 4; ++q) {
            const __nv_bfloat162 b2 = __floats2bfloat162_rn((float)cn[2 * q], (float)cn[2 * q + 1]);
            w[q] = *(const uint32_t *)&b2;
          }
          *(uint4 *)((__nv_bfloat16 *)base + idx) = make_uint4(w[0], w[1], w[2], w[3]);
        } else {
          float4 *d = (float4 *)((float *)base + idx);
          d[0] = make_float4(to_tf32((float)cn[0]), to_tf32((float)cn[1]), to_tf32((float)cn[2]), to_tf32((float)cn[3]));
          d[1] = make_float4(to_tf32((float)cn[4]), to_tf32((float)cn[5]), to_tf32((float)cn[6]), to_tf32((float)cn[7]));
        }
      }
    }
  }
}

// Residual partials inside the tcgen05 epilogue without FP64 arithmetic.  On sm_100a the FP64 pipe
// stalls while tcgen05.mma streams (ncu r02: the tri GEMM's DMUL / DADD / DFMA drew 47 % of the
// epilogue's stall samples as math-pipe throttle, tensor pipe 50 % busy), so w d^2 (w = 1 or 2, exact)
// of an FP32 d is split exactly by one FMA into p + e and added to a float-float accumulator (TwoSum;
// hi + lo carries ~48 bits); a chunk's (hi, lo) joins the FP64 partial once per 32 elements.
__device__ __forceinline__ void ff_add_sq(float &hi, float &lo, float d, float w) {
  const float p = __fmul_rn(__fmul_rn(d, d), w);
  const float e = __fmul_rn(__fmaf_rn(d, d, -__fmul_rn(d, d)), w);   // d^2 - fl(d^2), exact
  const float sm = __fadd_rn(hi, p);
  const float bb = __fsub_rn(sm, hi);
  const float er = __fadd_rn(__fsub_rn(hi, __fsub_rn(sm, bb)), __fsub_rn(p, bb));
  lo = __fadd_rn(lo, __fadd_rn(er, e));
  hi = sm;
}
// the chunk's sum into the FP64 partial; false if it overflowed FP32 (the caller redoes it in FP64)
__device__ __forceinline__ bool ff_flush(float hi, float lo, double &r2) {
  if (!(fabsf(hi) <= 3.0e38f)) return false;
  r2 = __dadd_rn(r2, __dadd_rn((double)hi, (double)lo));
  return true;
}

// One 32-column chunk of one accumulator row: the fused epilogue with vectorised row access.
template <int KIND>
__device__ __forceinline__ void epi_chunk(const GemmArgs &g, int64_t row, int64_t col, const uint32_t (&r)[32],
                                          double scale, EpiAcc &ea) {
  const int mode = g.mode;
  if (KIND == 3 && mode == EPI_OZACC) {
    // Ozaki group g (reading R-23): the INT32 group sum is exact; 2^(rsig + csig - 7 g) scaling is
    // exact; the FP64 accumulation (smallest groups first) is the only rounding.  Transposed
    // layout: a warp's 32 rows are 256 contiguous bytes per column.
    const int rs = g.oz_rsig[row];
    double *z = g.ozacc + col * g.ldoz + row;
    #pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double v = __dmul_rn((double)(int32_t)r[j], pow2(rs + g.oz_csig[col + j] - 7 * g.oz_g));
      z[j * g.ldoz] = g.oz_first ? v : __dadd_rn(z[j * g.ldoz], v);
    }
    return;
  }
  if (mode & EPI_COUPLED) {           // coupled form: the generic per-element FP64 epilogue
    // a copy for the rolled loop: dynamic indexing of r itself would put every epilogue's accumulator
    // registers in local memory (a 128-byte stack frame and 8 STL.128 per chunk in all modes)
    uint32_t rl[32];
    #pragma unroll
    for (int j = 0; j < 32; ++j) rl[j] = r[j];
    #pragma unroll 1
    for (int j = 0; j < 32; ++j) epi_element<-1>(g, row, col + j, __dmul_rn(acc_to_f64<KIND>(rl[j]), scale), ea);
    return;
  }
  // ---- FP32 fast paths (no FP64 arithmetic; results identical to the general path below) ----
  // (a) plain chain store: qin(D) of an unscaled accumulator -- BF16 / TF32 are one RNE rounding
  //     of the FP32 value, exactly what the FP64 detour produced ((float)(double)f == f)
  if (mode == EPI_STORE_T && scale == 1.0 && !g.tri && KIND <= 1 && (g.tprec == P_BF16 || g.tprec == P_TF32)) {
    if (g.tprec == P_BF16) {
      __nv_bfloat16 *t = (__nv_bfloat16 *)g.tout + col * g.ldt + row;
      #pragma unroll
      for (int j = 0; j < 32; ++j) t[j * g.ldt] = __float2bfloat16_rn(__uint_as_float(r[j]));
    } else {
      float *t = (float *)g.tout + col * g.ldt + row;
      #pragma unroll
      for (int j = 0; j < 32; ++j) t[j * g.ldt] = to_tf32(__uint_as_float(r[j]));
    }
    return;
  }
  // (c) GEMM 2 of the symmetric-tri form with a BF16 / TF32 R: a row segment strictly above the
  //     diagonal stores every element twice -- K-major (coalesced across the warp's rows) and
  //     mirrored row-major with 16-byte vector stores (the generic path's per-element mirror stores
  //     were uncoalesced: 1.11 ms vs 0.76 ms for the full GEMM 1).  Same FP64 arithmetic and order.
  //     Also R-29's FP32 scratch of a scaled R (TSCRATCH instead of STORE_T, + the tile maximum).
  if (g.tri && row < g.col0 + col &&
      (((mode & EPI_STORE_T) && (mode & ~(EPI_STORE_T | EPI_DIAG_MINUS | EPI_RESID)) == 0 &&
        (g.tprec == P_BF16 || g.tprec == P_TF32)) ||
       ((mode & EPI_TSCRATCH) && (mode & ~(EPI_TSCRATCH | EPI_DIAG_MINUS | EPI_RESID)) == 0))) {
    const bool ts = (mode & EPI_TSCRATCH) != 0;
    const bool dm = (mode & EPI_DIAG_MINUS) != 0, rsd = (mode & EPI_RESID) != 0;
    if (!ts && g.tprec == P_BF16 && KIND != 3 && scale >= 0x1p-126 && scale <= 0x1p127) {
      // the R value 0 - v (v = acc * scale, a power of two) is an exact float: round it to BF16 from FP32
      // (the same single rounding as from FP64; no F2F per element), FP64 only for the residual sum
      __nv_bfloat16 *t = (__nv_bfloat16 *)g.tout;
      const float sf = (float)scale;
      uint32_t pk[16];
      float rh = 0.f, rlo = 0.f;
      #pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float fv = __fmul_rn(__uint_as_float(r[j]), sf);
        const float fw = dm ? __fsub_rn(0.0f, fv) : fv;       // row < gc: off the diagonal
        const __nv_bfloat16 b = __float2bfloat16_rn(fw);
        t[(col + j) * g.ldt + row] = b;
        const uint32_t bits = (uint32_t)__bfloat16_as_ushort(b);
        pk[j >> 1] = (j & 1) ? (pk[j >> 1] | (bits << 16)) : bits;
        if (rsd && row < g.n && g.col0 + col + j < g.n) ff_add_sq(rh, rlo, fv, 2.0f);   // 2 (0 - v)^2
      }
      if (rsd && !ff_flush(rh, rlo, ea.r2)) {
        #pragma unroll
        for (int j = 0; j < 32; ++j)
          if (row < g.n && g.col0 + col + j < g.n) {
            const double d = __dsub_rn(0.0, __dmul_rn(acc_to_f64<KIND>(r[j]), scale));
            ea.r2 = __fma_rn(2.0 * d, d, ea.r2);
          }
      }
      uint4 *m = (uint4 *)((__nv_bfloat16 *)g.mout + row * g.ldm + col);
      #pragma unroll
      for (int q = 0; q < 4; ++q) m[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    } else if (!ts && g.tprec == P_BF16) {
      __nv_bfloat16 *t = (__nv_bfloat16 *)g.tout;
      uint32_t pk[16];
      #pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double a = acc_to_f64<KIND>(r[j]);
        const double v = scale == 1.0 ? a : __dmul_rn(a, scale);   // scaled formats: exact 2^-(sigma)
        const double w = dm ? __dsub_rn(0.0, v) : v;          // row < gc: off the diagonal
        const __nv_bfloat16 b = __float2bfloat16_rn((float)w);
        t[(col + j) * g.ldt + row] = b;
        const uint32_t bits = (uint32_t)__bfloat16_as_ushort(b);
        pk[j >> 1] = (j & 1) ? (pk[j >> 1] | (bits << 16)) : bits;
        if (rsd && row < g.n && g.col0 + col + j < g.n) {
          const double d = __dsub_rn(0.0, v);
          ea.r2 = __fma_rn(2.0 * d, d, ea.r2);
        }
      }
      uint4 *m = (uint4 *)((__nv_bfloat16 *)g.mout + row * g.ldm + col);
      #pragma unroll
      for (int q = 0; q < 4; ++q) m[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    } else {
      float *t = (float *)g.tout;
      float4 *m = (float4 *)((float *)g.mout + row * g.ldm + col);
      if (ts) {
        // R-29 scratch: the stored float is one FP32 multiply by the power-of-two scale (the same
        // float as (float)(acc * scale) in FP64, as in (b)); FP64 only for the residual, from the
        // exact product -- the same values and order as below, fewer dependent FP64 operations
        const float sf = (float)scale;
        // FP32 residual terms need v = acc * scale exact in FP32: FP32 accumulators (not INT32) and a
        // normal-range scale (warp-uniform); otherwise the FP64 terms
        const bool f32r = KIND != 3 && scale >= 0x1p-126 && scale <= 0x1p127;
        float rh = 0.f, rlo = 0.f;
        #pragma unroll
        for (int q = 0; q < 8; ++q) {
          float f[4];
          #pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * q + u;
            const float a = KIND == 3 ? (float)(int32_t)r[j] : __uint_as_float(r[j]);
            const float fv = __fmul_rn(a, sf);
            f[u] = dm ? __fsub_rn(0.0f, fv) : fv;      // 0 - v as in FP64: +0 for v = 0
            ea.mx = fmaxf(ea.mx, fabsf(f[u]));
            if (!(g.diag_epi & 2)) t[(col + j) * g.ldt + row] = f[u];
            if (rsd && !(g.diag_epi & 1) && row < g.n && g.col0 + col + j < g.n) {
              if (f32r) {
                ff_add_sq(rh, rlo, fv, 2.0f);          // d = 0 - v: 2 d^2
              } else {
                const double v = scale == 1.0 ? acc_to_f64<KIND>(r[j]) : __dmul_rn(acc_to_f64<KIND>(r[j]), scale);
                ea.r2 = __fma_rn(-2.0 * v, -v, ea.r2);
              }
            }
          }
          if (!(g.diag_epi & 4)) m[q] = make_float4(f[0], f[1], f[2], f[3]);
        }
        if (rsd && f32r && !ff_flush(rh, rlo, ea.r2)) {
          #pragma unroll
          for (int j = 0; j < 32; ++j)
            if (row < g.n && g.col0 + col + j < g.n) {
              const double v = __dmul_rn(acc_to_f64<KIND>(r[j]), scale);
              ea.r2 = __fma_rn(-2.0 * v, -v, ea.r2);
            }
        }
        return;
      }
      #pragma unroll
      for (int q = 0; q < 8; ++q) {        // 4 at a time: the mirror float4 leaves as soon as it is complete
        float f[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * q + u;
          const double a = acc_to_f64<KIND>(r[j]);
          const double v = scale == 1.0 ? a : __dmul_rn(a, scale);
          const double w = dm ? __dsub_rn(0.0, v) : v;
          f[u] = ts ? (float)w : to_tf32((float)w);
          if (ts) ea.mx = fmaxf(ea.mx, fabsf(f[u]));
          t[(col + j) * g.ldt + row] = f[u];
          if (rsd && row < g.n && g.col0 + col + j < g.n) {
            const double d = __dsub_rn(0.0, v);
            ea.r2 = __fma_rn(2.0 * d, d, ea.r2);
          }
        }
        m[q] = make_float4(f[0], f[1], f[2], f[3]);
      }
    }
    return;
  }
  // (b) FP32 scratch of a scaled format: the scale is an exact power of two, so one FP32
  //     multiply gives the same float as (float)(acc * scale) in FP64 (one rounding for INT32).
  //     Not for tri (R-36's GEMM 1): its segments on / below the diagonal take (d), whose lower elements
  //     come from the mirror -- stored here too, they raced with the mirror stores of the upper ones
  if (mode == EPI_TSCRATCH && !g.tri) {
    const float sf = (float)scale;
    float *t = (float *)g.tout + col * g.ldt + row;
    #pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float a = KIND == 3 ? (float)(int32_t)r[j] : __uint_as_float(r[j]);
      const float w = __fmul_rn(a, sf);
      t[j * g.ldt] = w;
      ea.mx = fmaxf(ea.mx, fabsf(w));
    }
    return;
  }
  // (d) the (c) modes with an FP32 / TF32 R on a segment that is not strictly above the diagonal
  //     (the diagonal tiles of the tri GEMM): the generic path's arithmetic and order, but the mirror
  //     row segment leaves as float4 stores where all four elements are strictly upper -- the
  //     generic path's scalar mirror stores (32 rows per warp store) made a diagonal tile cost ~2
  //     mainloops, and the CTA pairs that drew one set the tri kernel's makespan
  if (g.tri && row >= g.col0 + col &&
      (((mode & EPI_STORE_T) && (mode & ~(EPI_STORE_T | EPI_DIAG_MINUS | EPI_RESID)) == 0 && g.tprec == P_TF32) ||
       ((mode & EPI_TSCRATCH) && (mode & ~(EPI_TSCRATCH | EPI_DIAG_MINUS | EPI_RESID)) == 0))) {
    const int64_t gc0 = g.col0 + col;
    if (row > gc0 + 31) return;                      // the whole segment comes from the mirror
    const bool ts = (mode & EPI_TSCRATCH) != 0, dm = (mode & EPI_DIAG_MINUS) != 0, rsd = (mode & EPI_RESID) != 0;
    float *t = (float *)g.tout;
    float f[32];
    // off-diagonal elements in FP32 (exact v = acc * scale: FP32 accumulators, normal-range scale;
    // (float)(0 - v) then equals 0 - fv), the one diagonal element of the row in FP64 as before
    const bool f32r = KIND != 3 && scale >= 0x1p-126 && scale <= 0x1p127;
    const float sf = (float)scale;
    float rh = 0.f, rlo = 0.f;
    #pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t gc = gc0 + j;
      f[j] = 0.f;
      if (row > gc) continue;                        // lower triangle: from the mirror
      if (f32r && row != gc) {
        const float fv = __fmul_rn(__uint_as_float(r[j]), sf);
        const float fw = dm ? __fsub_rn(0.0f, fv) : fv;
        f[j] = ts ? fw : to_tf32(fw);
        t[(col + j) * g.ldt + row] = f[j];
        if (ts) ea.mx = fmaxf(ea.mx, fabsf(f[j]));
        if (rsd && row < g.n && gc < g.n) ff_add_sq(rh, rlo, fv, 2.0f);
        continue;
      }
      const double a = acc_to_f64<KIND>(r[j]);
      const double v = scale == 1.0 ? a : __dmul_rn(a, scale);
      const double w = dm ? __dsub_rn((row == gc && row < g.n) ? g.diag : 0.0, v) : v;
      f[j] = ts ? (float)w : to_tf32((float)w);
      t[(col + j) * g.ldt + row] = f[j];             // K-major: coalesced across the warp's rows
      if (ts) ea.mx = fmaxf(ea.mx, fabsf(f[j]));
      if (rsd && row < g.n && gc < g.n) {
        const double d = __dsub_rn(row == gc ? 1.0 : 0.0, v);
        ea.r2 = __fma_rn(row != gc ? 2.0 * d : d, d, ea.r2);
      }
    }
    if (rsd && f32r && !ff_flush(rh, rlo, ea.r2)) {
      #pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int64_t gc = gc0 + j;
        if (row >= gc || row >= g.n || gc >= g.n) continue;
        const double v = __dmul_rn(acc_to_f64<KIND>(r[j]), scale);
        ea.r2 = __fma_rn(-2.0 * v, -v, ea.r2);
      }
    }
    float *mr = (float *)g.mout + row * g.ldm + col;   // mirror (row, c), c > row
    #pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t c4 = gc0 + 4 * q;
      if (c4 > row) {
        *(float4 *)(mr + 4 * q) = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
      } else if (c4 + 3 > row) {
        #pragma unroll
        for (int u = 1; u < 4; ++u)
          if (c4 + u > row) mr[4 * q + u] = f[4 * q + u];
      }
    }
    return;
  }
  if (mode & (EPI_STORE_T | EPI_TSCRATCH | EPI_RESID | EPI_F64)) {
    #pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double a = acc_to_f64<KIND>(r[j]);
      const double v = scale == 1.0 ? a : __dmul_rn(a, scale);
      const int64_t c = col + j;
      if (g.tri && row > g.col0 + c) continue;         // tri: lower triangle comes from the mirror
      const bool mirror = g.tri && row != g.col0 + c;
      double w = v;
      if (mode & EPI_DIAG_MINUS) {    // diag*I - D: NS What = 2I - A X, symmetric R = I - Z_p
        const int64_t gc = g.col0 + c;
        w = __dsub_rn((row == gc && row < g.n) ? g.diag : 0.0, v);
      }
      if (mode & EPI_STORE_T) {
        store_operand(g.tout, c * g.ldt + row, g.tprec, w, 0);
        if (mirror) store_operand(g.mout, row * g.ldm + c, g.tprec, w, 0);
      }
      if (mode & EPI_TSCRATCH) {
        ((float *)g.tout)[c * g.ldt + row] = (float)w;
        if (mirror) ((float *)g.mout)[row * g.ldm + c] = (float)w;
        ea.mx = fmaxf(ea.mx, fabsf((float)w));
      }
      if (mode & EPI_RESID) {
        const int64_t gc = g.col0 + c;
        if (row < g.n && gc < g.n) {
          const double d = __dsub_rn(row == gc ? 1.0 : 0.0, v);
          ea.r2 = __fma_rn(mirror ? 2.0 * d : d, d, ea.r2);
        }
      }
      if (mode & EPI_F64) g.zout[row * g.ldz + c] = v;
    }
  }
  if (mode & EPI_WSTORE) {
    // symmetric form: W row segment [row][col .. col+31], 16-byte stores.  An unscaled BF16 / TF32
    // correction has scale == 1 (raw FP32 accumulators); R-29's scaled correction (FP8 / FP16 / INT8 =
    // the phase's format) unscales by scale = 2^-(sigma_C + sigma_R) -- one FP32 multiply while that
    // power of two is a normal float (then exactly (float)(acc * scale)), else (sigma_C + sigma_R > 126:
    // a residual far below the phase's floor) the product in FP64 and one rounding, so W never
    // underflows to 0 through the scale itself
    float4 *dst = (float4 *)((float *)g.wout + row * g.ldw + col);
    if (scale >= 0x1p-126 && scale <= 0x1p127) {       // warp-uniform: one loop or the other
      const float sf = (float)scale;
      #pragma unroll
      for (int q = 0; q < 8; ++q) {
        float w[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float a = KIND == 3 ? (float)(int32_t)r[4 * q + u] : __uint_as_float(r[4 * q + u]);
          w[u] = __fmul_rn(a, sf);
        }
        dst[q] = make_float4(w[0], w[1], w[2], w[3]);
      }
    } else {
      #pragma unroll
      for (int q = 0; q < 8; ++q) {
        float w[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = (float)__dmul_rn(acc_to_f64<KIND>(r[4 * q + u]), scale);
        dst[q] = make_float4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  if (mode & (EPI_UPDATE | EPI_NSUPDATE)) {
    // container row segment [row][col .. col+31]: 128 B (FP32) per thread, 16-byte accesses
    const bool ns = (mode & EPI_NSUPDATE) != 0;   // Newton-Schulz: X_{k+1} = q_m(D)
    const double pp1 = (double)(g.p + 1), pd = (double)g.p, invp = 1.0 / (double)g.p;
    const bool p2 = (g.p & (g.p - 1)) == 0;   // d/p == d*(1/p) exactly for p = 2^k
    const float4 *src = (const float4 *)((const float *)g.cold + row * g.ldc + col);
    float4 *dst = (float4 *)((float *)g.cnew + row * g.ldc + col);
    float cn[32];
    #pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 c4 = src[q];
      const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
      #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = q * 4 + u;
        const double v = __dmul_rn(acc_to_f64<KIND>(r[j]), scale);
        const double c = (double)cc[u];
        double e = v;
        if (!ns) {
          const double a = __dmul_rn(pp1, c);
          const double d = __dsub_rn(a, v);
          e = p2 ? __dmul_rn(d, invp) : __ddiv_rn(d, pd);
        }
        const float f = q_e8(e, g.m, g.rtz);
        cn[j] = f;
        const double dd = __dsub_rn((double)f, c);
        ea.d2 = __fma_rn(dd, dd, ea.d2);
        ea.mx = fmaxf(ea.mx, fabsf(f));
      }
      dst[q] = make_float4(cn[q * 4], cn[q * 4 + 1], cn[q * 4 + 2], cn[q * 4 + 3]);
    }
    if (g.chat_new && !is_scaled(g.prec)) {
      if (g.prec == P_TF32) {
        float4 *h = (float4 *)((float *)g.chat_new + row * g.ldh + col);
        #pragma unroll
        for (int q = 0; q < 8; ++q)
          h[q] = make_float4(to_tf32(cn[q * 4]), to_tf32(cn[q * 4 + 1]), to_tf32(cn[q * 4 + 2]), to_tf32(cn[q * 4 + 3]));
      } else {
        uint4 *h = (uint4 *)((__nv_bfloat16 *)g.chat_new + row * g.ldh + col);
        #pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t w[4];
          #pragma unroll
          for (int u = 0; u < 4; ++u) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(cn[q * 8 + 2 * u], cn[q * 8 + 2 * u + 1]);
            w[u] = *(uint32_t *)&b2;
          }
          h[q] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
  }
}

// The hot path's FP64 epilogue on 32 completed FP64 values of one row (the group-2 finish of an
// Ozaki product): STORE_T (+ mirror for tri), STORE_N, DIAG_MINUS, RESID, F64 -- the modes the
// FP64_OZ GEMMs use.  The store format and the DIAG/RESID/tri path are template parameters: with
// run-time switches per element the finish was instruction-bound (~1 ms per n = 8192 product).
template <int TP>   // 0: FP64, 1: BF16, 2: TF32 (tprec of the STORE_T output)
__device__ __forceinline__ void st_t(void *base, int64_t idx, double w) {
  if (TP == 0) ((double *)base)[idx] = w;
  else if (TP == 1) ((__nv_bfloat16 *)base)[idx] = __float2bfloat16_rn((float)w);
  else ((float *)base)[idx] = to_tf32((float)w);
}
template <int TP, bool DR, int W>
__device__ __forceinline__ void epi_row_t(const GemmArgs &g, int64_t row, int64_t col, const double (&v)[W], EpiAcc &ea) {
  const int mode = g.mode;
  if (!DR) {                                    // plain STORE_T
    if (mode & EPI_STORE_T) {
      #pragma unroll
      for (int j = 0; j < W; ++j) st_t<TP>(g.tout, (col + j) * g.ldt + row, v[j]);
    }
    return;
  }
  const bool diag = (mode & EPI_DIAG_MINUS) != 0, st = (mode & EPI_STORE_T) != 0, rs = (mode & EPI_RESID) != 0;
  #pragma unroll
  for (int j = 0; j < W; ++j) {
    const int64_t c = col + j, gc = g.col0 + c;
    if (g.tri && row > gc) continue;
    const bool mirror = g.tri && row != gc;
    const double dv = (row == gc && row < g.n) ? 1.0 : 0.0;
    const double w = diag ? __dsub_rn(dv * g.diag, v[j]) : v[j];
    if (st) {
      st_t<TP>(g.tout, c * g.ldt + row, w);
      if (mirror) st_t<TP>(g.mout, row * g.ldm + c, w);
    }
    if (rs && row < g.n && gc < g.n) {
      const double d = __dsub_rn(row == gc ? 1.0 : 0.0, v[j]);
      ea.r2 = __fma_rn(mirror ? 2.0 * d : d, d, ea.r2);
    }
  }
}
template <int W = 32>   // W consecutive columns (even)
__device__ __forceinline__ void epi_row_f64(const GemmArgs &g, int64_t row, int64_t col, const double (&v)[W],
                                            EpiAcc &ea) {
  const int mode = g.mode;
  if (mode & EPI_STORE_N) {
    double2 *dn = (double2 *)((double *)g.nout + row * g.ldn + col);
    #pragma unroll
    for (int j = 0; j < W / 2; ++j) dn[j] = make_double2(v[2 * j], v[2 * j + 1]);
  }
  if (mode & EPI_F64) {
    double2 *dz = (double2 *)(g.zout + row * g.ldz + col);
    #pragma unroll
    for (int j = 0; j < W / 2; ++j) dz[j] = make_double2(v[2 * j], v[2 * j + 1]);
  }
  if (!(mode & (EPI_STORE_T | EPI_RESID))) return;
  const bool dr = (mode & (EPI_DIAG_MINUS | EPI_RESID)) || g.tri;
  const int tp = is_f64(g.tprec) ? 0 : g.tprec == P_BF16 ? 1 : 2;
  if (dr) {
    if (tp == 0) epi_row_t<0, true, W>(g, row, col, v, ea);
    else if (tp == 1) epi_row_t<1, true, W>(g, row, col, v, ea);
    else epi_row_t<2, true, W>(g, row, col, v, ea);
  } else {
    if (tp == 0) epi_row_t<0, false, W>(g, row, col, v, ea);
    else if (tp == 1) epi_row_t<1, false, W>(g, row, col, v, ea);
    else epi_row_t<2, false, W>(g, row, col, v, ea);
  }
}

// ---- Ozaki scheme II (CRT, reading R-28; ozaki.cu) ----
__constant__ CrtTab c_crt;
cudaError_t tc_set_crt_table(const CrtTab &t) { return cudaMemcpyToSymbol(c_crt, &t, sizeof t); }

// One 32-column chunk of one accumulator row of modulus product l (INT32, exact): the bytes
// v = ((U mod m_l) inv_l) mod m_l to the crt_v scratch (k_crt_finish reconstructs).  Integer ALU
// only: x mod m = x - m umulhi(x, ceil(2^32 / m)), exact or one m too far for x < 2^31.
__device__ __forceinline__ void crt_chunk(const GemmArgs &g, int l, int64_t row, int64_t c0, const uint32_t (&r)[32]) {
  const int nm = g.crt_n;
  // unsigned residues (g.crt_u8): U = sum of byte products < 2^31, no offset needed
  const int m = c_crt.m[l], off = g.crt_u8 ? 0 : c_crt.off[l], iv = c_crt.inv[nm][l];
  const uint32_t mag = c_crt.mag[l];
  uint32_t pk[8];
  #pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t w = 0;
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t x = (uint32_t)((int)r[4 * q + u] + off);     // |U| <= 2^14 n <= 2^30 < off
      int a = (int)(x - __umulhi(x, mag) * (uint32_t)m);
      a += a < 0 ? m : 0;
      const uint32_t y = (uint32_t)(a * iv);                        // < 2^16
      int b = (int)(y - __umulhi(y, mag) * (uint32_t)m);
      b += b < 0 ? m : 0;
      w |= (uint32_t)b << (8 * u);
    }
    pk[q] = w;
  }
  uint4 *dst = (uint4 *)(g.crt_v + ((int64_t)l * g.M + row) * g.ldv + c0);
  dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
}

// CRT reconstruction + the hot path's FP64 finish epilogue (reading R-28): one block per 128 x 256
// output tile of the GEMM (tri: the upper-triangle pair tiles only), in two 128-column halves.
// Lane = 4 consecutive columns (the warp reads 128 contiguous residue bytes per modulus and row),
// warp = 4 rows of a 32-row slab: Pbar = sum_l v_l W_l - q M_N in two FP64 slices (H exact, Lo rounded),
// Z = 2^-(e_i + f_j) Pbar, then the epilogue of epi_row_f64: row-major stores directly, the K-major
// (transposed) store of the slab through shared memory (row r, column c at r * 161 + c + c / 4:
// conflict-free both ways).
constexpr int CRT_FIN_LD = 161;
// 3 resident blocks per SM (80 registers, a few spills): 5.86 -> 5.67 ms of finishes per solve against 2 (r02b)
template <int NM>   // the modulus count: the loops over moduli unroll exactly, constants come from c[] directly
__global__ void __launch_bounds__(256, 3) k_crt_finish(const GemmArgs g) {
  extern __shared__ double sm_slab[];          // [32][CRT_FIN_LD]
  __shared__ double red[8];
  const TileSched sch{(int)(g.M / (2 * TC_BM)), (int)(g.N / TC_BN), g.tri, (int)(g.col0 / TC_BN)};
  int tm, tn;
  sch.get((int)(blockIdx.x >> 1), tm, tn);
  const int tile_m = tm * 2 + (int)(blockIdx.x & 1);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nm = NM;
  const int mode = g.mode;
  const bool diag = (mode & EPI_DIAG_MINUS) != 0, st = (mode & EPI_STORE_T) != 0, rsd = (mode & EPI_RESID) != 0;
  const int tp = is_f64(g.tprec) ? 0 : g.tprec == P_BF16 ? 1 : 2;
  const double p1 = c_crt.p2s1[nm], iM = c_crt.invM[nm];
  const double MH = c_crt.MH[nm], MLo = c_crt.MLo[nm], CH = c_crt.CH[nm], CL = c_crt.CL[nm];
  double r2 = 0.0;
  // block-uniform tile class: a tile that touches neither the diagonal nor the padding takes the
  // branch-free path (tri: strictly above the diagonal, every element mirrored)
  const int64_t r0 = (int64_t)tile_m * TC_BM, gcb = g.col0 + (int64_t)tn * TC_BN;
  const bool clean = (r0 + TC_BM <= g.n) && (gcb + TC_BN <= g.n) && (r0 + TC_BM <= gcb || gcb + TC_BN <= r0);
  const bool mir = g.tri != 0;                       // clean + tri => strictly upper
  #pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    const int64_t colb = (int64_t)tn * TC_BN + 128 * half, c0 = colb + 4 * lane;
    double scol[4];
    int csg[4];
    bool cok = true;                              // |f_j| < 500: two scalings never leave the normal range
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
      csg[u] = g.oz_csig[c0 + u];
      cok = cok && csg[u] > -500 && csg[u] < 500;
      scol[u] = cok ? pow2(-csg[u]) : 1.0;
    }
    #pragma unroll 1
    for (int slab = 0; slab < 4; ++slab) {
      #pragma unroll 1
      for (int i2 = 0; i2 < 4; i2 += 2) {            // two rows at a time: 16 independent FMA chains
        uint32_t bv[2][NM];
        #pragma unroll
        for (int ii = 0; ii < 2; ++ii) {
          const int64_t row = r0 + slab * 32 + 4 * w + i2 + ii;
          const uint8_t *src = g.crt_v + row * g.ldv + c0;
          const int64_t plane = g.M * g.ldv;
          #pragma unroll
          for (int l = 0; l < NM; ++l) bv[ii][l] = *(const uint32_t *)(src + l * plane);
        }
        // two slices: sh = sum v_l H_l exact (< 2^53), so = sum v_l Lo_l (Lo_l = (W_l mod 2^s1) 2^-s1,
        // rounded: absolute error ~2^(s1 - 45) in Pbar, far below its own last bit at these sizes)
        double sh[2][4], so[2][4];
        #pragma unroll
        for (int ii = 0; ii < 2; ++ii)
          #pragma unroll
          for (int u = 0; u < 4; ++u) { sh[ii][u] = 0.0; so[ii][u] = 0.0; }
        #pragma unroll
        for (int l = 0; l < NM; ++l) {
          const double hh = c_crt.H[nm][l], lo = c_crt.Lo[nm][l];
          #pragma unroll
          for (int ii = 0; ii < 2; ++ii)
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
              // 256 + v as an FP64 bit pattern (exponent 8, v in the top mantissa bits): no conversion,
              // no FP64 add; the bias 256 sum_l H_l (exact) / 256 sum_l Lo_l is removed below
              const uint32_t f = u == 0 ? (bv[ii][l] << 12) : u == 1 ? (bv[ii][l] << 4)
                               : u == 2 ? (bv[ii][l] >> 4) : (bv[ii][l] >> 12);
              const double d = __hiloint2double((int)((f & 0xff000u) | 0x40700000u), 0);
              sh[ii][u] = __fma_rn(d, hh, sh[ii][u]);   // integers < 2^53: exact
              so[ii][u] = __fma_rn(d, lo, so[ii][u]);
            }
        }
        #pragma unroll
        for (int ii = 0; ii < 2; ++ii) {
          const int rl = 4 * w + i2 + ii;
          const int64_t row = r0 + slab * 32 + rl;
          const int rsg = g.oz_rsig[row];
          const bool fast = __all_sync(0xffffffffu, cok && rsg > -500 && rsg < 500);   // warp-uniform
          const double srow = fast ? pow2(-rsg) : 1.0;
          double vv[4], wv[4];
          #pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double shu = __dsub_rn(sh[ii][u], CH), sou = __dsub_rn(so[ii][u], CL);   // exact / ~2^-40
            const double q = rint(__dmul_rn(__fma_rn(shu, p1, __dmul_rn(sou, p1)), iM));  // within 0.493 of an integer
            const double dh = __fma_rn(-q, MH, shu);                    // exact
            const double dlo = __fma_rn(-q, MLo, sou);
            vv[u] = __dmul_rn(__dadd_rn(dh, dlo), p1);                  // Pbar = (dh + dlo) 2^s1
          }
          // 2^-(e_i + f_j) Pbar: two exact scalings; one scalbn where the exponents are extreme
          if (fast) {
            #pragma unroll
            for (int u = 0; u < 4; ++u) vv[u] = __dmul_rn(__dmul_rn(vv[u], srow), scol[u]);
          } else {
            #pragma unroll
            for (int u = 0; u < 4; ++u) vv[u] = scalbn(vv[u], -(rsg + csg[u]));
          }
          if (mode & EPI_STORE_N) {
            double2 *dn = (double2 *)((double *)g.nout + row * g.ldn + c0);
            dn[0] = make_double2(vv[0], vv[1]); dn[1] = make_double2(vv[2], vv[3]);
          }
          if (mode & EPI_F64) {
            double2 *dz = (double2 *)(g.zout + row * g.ldz + c0);
            dz[0] = make_double2(vv[0], vv[1]); dz[1] = make_double2(vv[2], vv[3]);
          }
          if (clean) {                                   // off the diagonal, inside n
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double d = __dsub_rn(0.0, vv[u]);
              wv[u] = diag ? d : vv[u];
              if (rsd) r2 = __fma_rn(mir ? 2.0 * d : d, d, r2);
            }
            if (st && mir) {                             // (j, i): row-major in T, one vector store
              if (tp == 0) {
                double2 *m = (double2 *)((double *)g.mout + row * g.ldm + c0);
                m[0] = make_double2(wv[0], wv[1]); m[1] = make_double2(wv[2], wv[3]);
              } else if (tp == 1) {
                const __nv_bfloat162 a = __floats2bfloat162_rn((float)wv[0], (float)wv[1]);
                const __nv_bfloat162 b = __floats2bfloat162_rn((float)wv[2], (float)wv[3]);
                *(uint2 *)((__nv_bfloat16 *)g.mout + row * g.ldm + c0) = make_uint2(*(const uint32_t *)&a, *(const uint32_t *)&b);
              } else {
                *(float4 *)((float *)g.mout + row * g.ldm + c0) =
                    make_float4(to_tf32((float)wv[0]), to_tf32((float)wv[1]), to_tf32((float)wv[2]), to_tf32((float)wv[3]));
              }
            }
          } else {
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int64_t c = c0 + u, gc = g.col0 + c;
              const bool skip = g.tri && row > gc;            // tri: the lower triangle comes from the mirror
              const bool mirror = g.tri && row < gc;
              wv[u] = diag ? __dsub_rn((row == gc && row < g.n) ? g.diag : 0.0, vv[u]) : vv[u];
              if (rsd && !skip && row < g.n && gc < g.n) {
                const double d = __dsub_rn(row == gc ? 1.0 : 0.0, vv[u]);
                r2 = __fma_rn(mirror ? 2.0 * d : d, d, r2);
              }
              if (st && mirror) {                              // (j, i) of a tri element: row-major in T
                if (tp == 0) st_t<0>(g.mout, row * g.ldm + c, wv[u]);
                else if (tp == 1) st_t<1>(g.mout, row * g.ldm + c, wv[u]);
                else st_t<2>(g.mout, row * g.ldm + c, wv[u]);
              }
            }
          }
          #pragma unroll
          for (int u = 0; u < 4; ++u) sm_slab[rl * CRT_FIN_LD + 5 * lane + u] = wv[u];   // column 4 lane + u, + lane
        }
      }
      __syncthreads();
      if (st) {                                            // K-major store: 32 consecutive rows per warp
        const int64_t row = r0 + slab * 32 + lane;
        const bool chk = g.tri && !clean;
        if (tp == 0) {
          #pragma unroll 4
          for (int j = 0; j < 16; ++j) {
            const int cl = w * 16 + j;
            const int64_t c = colb + cl;
            if (!(chk && row > g.col0 + c)) st_t<0>(g.tout, c * g.ldt + row, sm_slab[lane * CRT_FIN_LD + cl + (cl >> 2)]);
          }
        } else if (tp == 1) {
          #pragma unroll 4
          for (int j = 0; j < 16; ++j) {
            const int cl = w * 16 + j;
            const int64_t c = colb + cl;
            if (!(chk && row > g.col0 + c)) st_t<1>(g.tout, c * g.ldt + row, sm_slab[lane * CRT_FIN_LD + cl + (cl >> 2)]);
          }
        } else {
          #pragma unroll 4
          for (int j = 0; j < 16; ++j) {
            const int cl = w * 16 + j;
            const int64_t c = colb + cl;
            if (!(chk && row > g.col0 + c)) st_t<2>(g.tout, c * g.ldt + row, sm_slab[lane * CRT_FIN_LD + cl + (cl >> 2)]);
          }
        }
      }
      __syncthreads();
    }
  }
  if (rsd) {
    const double sum = block_sum_det<256>(r2, red);
    if (threadIdx.x == 0) g.part[((g.col0 + (int64_t)tn * TC_BN) / TC_BN) * g.tiles_m + tile_m] = sum;
  }
}

cudaError_t launch_crt_finish(const GemmArgs &a_in, cudaStream_t s) {
  GemmArgs a = a_in;
  if (!a.mout) { a.mout = a.tout; a.ldm = a.ldt; }   // tri mirror: in place at G = 1
  const TileSched hs{(int)(a.M / (2 * TC_BM)), (int)(a.N / TC_BN), a.tri, (int)(a.col0 / TC_BN)};
  if (a.tri && (a.mode & EPI_RESID)) {   // the tiles below the diagonal are not visited: zero partials
    cudaError_t z = cudaMemsetAsync(a.part + (a.col0 / TC_BN) * a.tiles_m, 0, (size_t)(a.N / TC_BN) * a.tiles_m * sizeof(double), s);
    if (z != cudaSuccess) return z;
  }
  const int smem = 32 * CRT_FIN_LD * 8;
  switch (a.crt_n) {
#define CRT_FIN(N)                                                                                       \
    case N: {                                                                                            \
      static DeviceOnce attr;                                                                            \
      if (!attr.done()) {                                                                                \
        cudaError_t e = cudaFuncSetAttribute(k_crt_finish<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        if (e != cudaSuccess) return e;                                                                  \
        attr.set();                                                                                      \
      }                                                                                                  \
      k_crt_finish<N><<<2 * hs.count(), 256, smem, s>>>(a);                                              \
    } break;
    CRT_FIN(2) CRT_FIN(3) CRT_FIN(4) CRT_FIN(5) CRT_FIN(6) CRT_FIN(7) CRT_FIN(8) CRT_FIN(9) CRT_FIN(10)
    CRT_FIN(11) CRT_FIN(12) CRT_FIN(13) CRT_FIN(14) CRT_FIN(15) CRT_FIN(16) CRT_FIN(17) CRT_FIN(18)
#undef CRT_FIN
    default: return cudaErrorInvalidValue;
  }
  ++g_launches;
  return cudaGetLastError();
}

// CRT reconstruction for the certificate (reading R-35): the EXACT integer Pbar of every element,
// returned as a double-double.  W_l = H 2^s1 + L 2^s2 + X3 2^s3 + X4 with integer slices < 2^39, so each
// slice sum S_k = sum_l (256 + v_l) slice_l is an exact FP64 integer (< 2^53); q = rint(X / M) is
// exact (X / M within 0.493 of an integer, evaluated to ~2^-40), D_k = S_k - bias_k - q M_k exact, and
// Pbar = D_1 2^s1 + D_2 2^s2 + D_3 2^s3 + D_4 by an error-free two-sum cascade: hi + lo = Pbar within
// 6 u^2 sum_k |D_k 2^sk| <= 2^(s1 - 48) (engine.cu certify_crt bounds it), scaled by 2^-(e_i + f_j)
// exactly.  MODE 0: hi -> nout, lo -> zout (tri: the upper elements and their mirrors, K-major through
// two shared-memory slabs as in k_crt_finish); MODE 2: the same, K-major only ([local col][row]: the
// rows of a symmetric product's column panel, G > 1); MODE 1: per-tile partials of R_ij^2, R_ij = (delta_ij -
// hi) - lo over i, j < n (tri weight 2 off the diagonal).  Exponents are in (-400, 400) (the
// certificate's splits flag anything else), so every scaling is exact.
__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
template <int NM, int MODE>
__global__ void __launch_bounds__(256, MODE == 1 ? 3 : 2) k_crt_finish_dd(const GemmArgs g) {
  extern __shared__ double sm_dd[];            // MODE 0: [2][32][CRT_FIN_LD]
  __shared__ double red[8];
  const TileSched sch{(int)(g.M / (2 * TC_BM)), (int)(g.N / TC_BN), g.tri, (int)(g.col0 / TC_BN)};
  int tm, tn;
  sch.get((int)(blockIdx.x >> 1), tm, tn);
  const int tile_m = tm * 2 + (int)(blockIdx.x & 1);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nm = NM;
  const double p1 = c_crt.p2s1[nm], p2 = c_crt.p2s2[nm], p3 = c_crt.p2s3[nm], iM = c_crt.invM[nm];
  const double MH = c_crt.MH[nm], ML = c_crt.ML[nm], M3 = c_crt.MX3[nm], M4 = c_crt.MX4[nm];
  const double B1 = c_crt.CH[nm], B2 = c_crt.CB2[nm], B3 = c_crt.CB3[nm], B4 = c_crt.CB4[nm];
  double r2 = 0.0;
  const int64_t r0 = (int64_t)tile_m * TC_BM;
  double *slh = sm_dd, *sll = sm_dd + 32 * CRT_FIN_LD;
  #pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    const int64_t colb = (int64_t)tn * TC_BN + 128 * half, c0 = colb + 4 * lane;
    double scol[4];
    #pragma unroll
    for (int u = 0; u < 4; ++u) scol[u] = pow2(-g.oz_csig[c0 + u]);
    #pragma unroll 1
    for (int slab = 0; slab < 4; ++slab) {
      #pragma unroll 1
      for (int i2 = 0; i2 < 4; ++i2) {
        const int rl = 4 * w + i2;
        const int64_t row = r0 + slab * 32 + rl;
        uint32_t bv[NM];
        {
          const uint8_t *src = g.crt_v + row * g.ldv + c0;
          const int64_t plane = g.M * g.ldv;
          #pragma unroll
          for (int l = 0; l < NM; ++l) bv[l] = *(const uint32_t *)(src + l * plane);
        }
        double s1[4], s2[4], s3[4], s4[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) { s1[u] = 0.0; s2[u] = 0.0; s3[u] = 0.0; s4[u] = 0.0; }
        #pragma unroll
        for (int l = 0; l < NM; ++l) {
          const double h1 = c_crt.H[nm][l], h2 = c_crt.L[nm][l], h3 = c_crt.X3[nm][l], h4 = c_crt.X4[nm][l];
          #pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t f = u == 0 ? (bv[l] << 12) : u == 1 ? (bv[l] << 4) : u == 2 ? (bv[l] >> 4) : (bv[l] >> 12);
            const double d = __hiloint2double((int)((f & 0xff000u) | 0x40700000u), 0);   // 256 + v_l
            s1[u] = __fma_rn(d, h1, s1[u]);            // integers < 2^53: exact
            s2[u] = __fma_rn(d, h2, s2[u]);
            s3[u] = __fma_rn(d, h3, s3[u]);
            s4[u] = __fma_rn(d, h4, s4[u]);
          }
        }
        const double srow = pow2(-g.oz_rsig[row]);
        double vh[4], vl[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double t1 = __dsub_rn(s1[u], B1), t2 = __dsub_rn(s2[u], B2);   // exact
          const double t3 = __dsub_rn(s3[u], B3), t4 = __dsub_rn(s4[u], B4);
          const double q = rint(__dmul_rn(__fma_rn(t1, p1, __dmul_rn(t2, p2)), iM));
          const double a = __dmul_rn(__fma_rn(-q, MH, t1), p1);          // D_1 2^s1 (exact)
          const double b = __dmul_rn(__fma_rn(-q, ML, t2), p2);
          const double c = __dmul_rn(__fma_rn(-q, M3, t3), p3);
          const double d = __fma_rn(-q, M4, t4);
          double sA, e1, sB, e2, sC, e3, hi, lo;
          two_sum(a, b, sA, e1);
          two_sum(sA, c, sB, e2);
          two_sum(sB, d, sC, e3);
          two_sum(sC, __dadd_rn(__dadd_rn(e1, e2), e3), hi, lo);
          const double sc = __dmul_rn(srow, scol[u]);                      // 2^-(e_i + f_j): exact
          vh[u] = __dmul_rn(hi, sc);
          vl[u] = __dmul_rn(lo, sc);
        }
        if (MODE != 1) {
          #pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t gc = g.col0 + c0 + u;
            if (MODE == 0 && (!g.tri || row <= gc)) {
              ((double *)g.nout)[row * g.ldn + c0 + u] = vh[u];
              g.zout[row * g.ldz + c0 + u] = vl[u];
            }
            slh[rl * CRT_FIN_LD + 5 * lane + u] = vh[u];
            sll[rl * CRT_FIN_LD + 5 * lane + u] = vl[u];
          }
        } else {
          #pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t gc = g.col0 + c0 + u;
            if (row < g.n && gc < g.n && (!g.tri || row <= gc)) {
              const double rr = __dsub_rn(__dsub_rn(row == gc ? 1.0 : 0.0, vh[u]), vl[u]);
              r2 = __fma_rn((g.tri && row < gc) ? 2.0 * rr : rr, rr, r2);
            }
          }
        }
      }
      if (MODE != 1) {
        __syncthreads();
        if (MODE == 2 || g.tri) {                        // (row, c) -> [c][row], 32 rows per warp: the tri
          const int64_t row = r0 + slab * 32 + lane;     // mirrors (MODE 0), or the whole tile K-major (MODE 2)
          #pragma unroll 4
          for (int j = 0; j < 16; ++j) {
            const int cl = w * 16 + j;
            const int64_t c = colb + cl;
            if (MODE == 2 || row < g.col0 + c) {
              ((double *)g.nout)[c * g.ldn + row] = slh[lane * CRT_FIN_LD + cl + (cl >> 2)];
              g.zout[c * g.ldz + row] = sll[lane * CRT_FIN_LD + cl + (cl >> 2)];
            }
          }
        }
        __syncthreads();
      }
    }
  }
  if (MODE == 1) {
    const double sum = block_sum_det<256>(r2, red);
    if (threadIdx.x == 0) g.part[((g.col0 + (int64_t)tn * TC_BN) / TC_BN) * g.tiles_m + tile_m] = sum;
  }
}

cudaError_t launch_crt_finish_dd(const GemmArgs &a, cudaStream_t s) {
  const TileSched hs{(int)(a.M / (2 * TC_BM)), (int)(a.N / TC_BN), a.tri, (int)(a.col0 / TC_BN)};
  const int mode = (a.mode & EPI_RESID) ? 1 : (a.mode & EPI_STORE_T) ? 2 : 0;
  if (mode != 1 && (!a.nout || !a.zout)) return cudaErrorInvalidValue;
  if (mode == 1 && a.tri) {   // the tiles below the diagonal are not visited: zero partials
    cudaError_t z = cudaMemsetAsync(a.part + (a.col0 / TC_BN) * a.tiles_m, 0, (size_t)(a.N / TC_BN) * a.tiles_m * sizeof(double), s);
    if (z != cudaSuccess) return z;
  }
  const int smem = mode != 1 ? 2 * 32 * CRT_FIN_LD * 8 : 0;
#define CRT_FIN_DD(N)                                                                                     \
  case N: {                                                                                               \
    static DeviceOnce attr;                                                                               \
    if (!attr.done()) {                                                                                   \
      cudaError_t e = cudaFuncSetAttribute(k_crt_finish_dd<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32 * CRT_FIN_LD * 8); \
      if (e == cudaSuccess)                                                                               \
        e = cudaFuncSetAttribute(k_crt_finish_dd<N, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 32 * CRT_FIN_LD * 8); \
      if (e != cudaSuccess) return e;                                                                     \
      attr.set();                                                                                         \
    }                                                                                                     \
    if (mode == 0) k_crt_finish_dd<N, 0><<<2 * hs.count(), 256, smem, s>>>(a);                            \
    else if (mode == 2) k_crt_finish_dd<N, 2><<<2 * hs.count(), 256, smem, s>>>(a);                       \
    else k_crt_finish_dd<N, 1><<<2 * hs.count(), 256, 0, s>>>(a);                                         \
  } break;
  switch (a.crt_n) {
    CRT_FIN_DD(16) CRT_FIN_DD(17) CRT_FIN_DD(18)
    default: return cudaErrorInvalidValue;
  }
#undef CRT_FIN_DD
  ++g_launches;
  return cudaGetLastError();
}

// EF = 1: the fused symmetric update (EPI_SYMUPD) is the only epilogue of this instance -- with the
// general epilogue's code in the same kernel the instruction cache thrashed (tensor pipe 30 % busy,
// "no instruction" the top stall)
// EF: 0 the hot path's epilogues, 1 EPI_SYMUPD, 2 Ozaki-I digit groups (kind::i8), 3 CRT moduli
// (kind::i8) -- each its own instance, so the plain and CRT INT8 kernels carry no Ozaki-I code
template <int KIND, int EF = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_NT, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, const GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + TC_ST * TC_STAGE_BYTES);
  uint64_t *empty = full + TC_ST;
  uint64_t *tfull = empty + TC_ST;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = (uint32_t *)(tempty + 2);
  __shared__ double red[2][8];
  __shared__ float redm[2][8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  if (KIND == 3 && EF == 3) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");   // next modulus launch
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr bool crt = KIND == 3 && EF == 3, ozg = KIND == 3 && EF == 2;
  TileSched sch{(int)(g.M / (2 * TC_BM)), (int)(g.N / TC_BN), g.tri, (int)(g.col0 / TC_BN)};
  if (crt) sch.gm = IPR_CRT_GROUP_M;
  const int ntiles = sch.count();
  // CRT (oz_grouped == 3): moduli [crt_l0, crt_l1) of every tile, modulus-major (all CTA pairs
  // stream the same residue planes at a time, as in one plain GEMM)
  const int nitems = crt ? (g.crt_l1 - g.crt_l0) * ntiles : ntiles;
  // Ozaki grouped launch: groups S+1 .. 2 per tile; otherwise one pass (g0 == g1)
  // oz_grouped == 2: the single group g.oz_g (one launch per group keeps each group's digit planes
  // L2-hot across all CTAs -- measured faster than all groups per tile in one launch)
  const int g0 = !ozg ? 0 : g.oz_grouped == 1 ? g.oz_S + 1 : g.oz_g;
  const int g1 = !ozg ? 0 : g.oz_grouped == 1 ? 2 : g.oz_g;
  const int gfirst = g.oz_S + 1;                 // the group that initialises the FP64 accumulator
  const int nsub = crt ? 1 : g0 - g1 + 1;
  const int esz = elt_size(g.prec);
  const int64_t bkp = g.b_kp ? g.b_kp : g.a_kp;       // K-panel length of a paneled B operand
  const int nkb = (int)(g.K * esz / TC_BKB);
  const int bke = TC_BKB / esz;                       // K elements per block

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 16); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer (both CTAs) =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < nitems; t += npairs) {
        const int lmod = crt ? g.crt_l0 + t / ntiles : 0;
        int tm, tn;
        sch.get(crt ? t % ntiles : t, tm, tn);
        const int arow = tm * 2 * TC_BM + (int)rank * TC_BM;
        const int brow = tn * TC_BN + (int)rank * (TC_BN / 2);
        for (int si = 0; si < nsub; ++si) {      // Ozaki groups / CRT moduli (one pass otherwise)
          const int gi = g0 - si;
          const int nk = crt ? (int)(g.a_kp * esz / TC_BKB)
                             : ozg ? (int)((int64_t)(gi - 1) * g.a_kp * esz / TC_BKB) : nkb;
          const int64_t boff = ozg ? (int64_t)(OZ_S - gi + 1) * g.a_kp : 0;
          const int64_t kpl = crt ? (int64_t)lmod * g.a_kp : 0;      // CRT: residue plane lmod
          const int brow2 = crt ? lmod * (int)g.N + brow : brow;
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t *sa = smem + stage * TC_STAGE_BYTES, *sb = sa + TC_A_BYTES;
            if (leader) mbar_expect_tx(&full[stage], 2 * TC_STAGE_BYTES);
            const int64_t k0 = (int64_t)kb * bke;
            tma_load_3d_pair(sa, &mapA, &full[stage], (int)((kpl + k0) % g.a_kp), arow, (int)((kpl + k0) / g.a_kp));
            if (g.b_pstride) tma_load_3d_pair(sb, &mapB, &full[stage], (int)(k0 % bkp), brow2, (int)(k0 / bkp));
            else tma_load_2d_pair(sb, &mapB, &full[stage], (int)(boff + k0), brow2);
            if (++stage == TC_ST) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA, single thread) =====
    if (leader && lane == 0) {
      const uint32_t idesc = make_idesc(g.prec, crt && g.crt_u8);   // CRT: residues in [0, m) (u8 x u8)
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < nitems; t += npairs) {
        for (int si = 0; si < nsub; ++si) {
          const int gi = g0 - si;
          const int nk = crt ? (int)(g.a_kp * esz / TC_BKB)
                             : ozg ? (int)((int64_t)(gi - 1) * g.a_kp * esz / TC_BKB) : nkb;
          const int buf = it & 1;
          mbar_wait_cluster(&tempty[buf], ((it >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dcol = tmem + buf * TC_BN;
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = su32(smem + stage * TC_STAGE_BYTES), sb = sa + TC_A_BYTES;
            #pragma unroll
            for (int k = 0; k < TC_BKB / 32; ++k)
              tc_mma_pair<KIND>(dcol, smem_desc_sw128(sa + k * 32), smem_desc_sw128(sb + k * 32), idesc, (kb | k) != 0);
            tc_commit_pair(&empty[stage]);
            if (++stage == TC_ST) { stage = 0; phase ^= 1; }
          }
          tc_commit_pair(&tfull[buf]);
          ++it;
        }
      }
    }
  } else {
    // ===== epilogue warps 2..5 (both CTAs): TMEM lane quarter q = warp % 4 =====
    const int q = warp & 3;             // TMEM lane quarter
    const int hh = (warp - 2) >> 2;     // column half: chunks [4 hh, 4 hh + 4)
    const int et = threadIdx.x - 64;    // 0..255
    double scale = 1.0;
    if (g.sigA) scale = pow2(-(*g.sigA + *g.sigB));
    int it = 0;
    for (int t = pair; t < nitems; t += npairs)
    for (int si = 0; si < nsub; ++si) {
      const int gi = g0 - si;
      const int lmod = crt ? g.crt_l0 + t / ntiles : 0;
      int tm, tn;
      sch.get(crt ? t % ntiles : t, tm, tn);
      const int buf = it & 1;
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      tc_fence_after();
      const int tile_m = tm * 2 + (int)rank;             // 128-row tile index
      const int64_t row = g.row0 + (int64_t)tile_m * TC_BM + q * 32 + lane;   // global row (2-D grid: row0)
      const int64_t colb = (int64_t)tn * TC_BN;
      EpiAcc ea{0.0, 0.0, 0.0f};
      #pragma unroll 1
      for (int ch = hh * 4; ch < hh * 4 + 4; ++ch) {
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + buf * TC_BN + ch * 32, r);
        if (EF == 1) {
          sym_update_chunk(g, row, colb + ch * 32, r, ea);
        } else if (crt) {
          crt_chunk(g, lmod, row, colb + ch * 32, r);
        } else if (ozg) {
          // the 32 accumulator values of this row segment are loaded up front (independent loads in
          // flight; a load-add-store chain per element serialised on memory latency)
          const int rs = g.oz_rsig[row];
          const int64_t c0 = colb + ch * 32;
          double *z = g.ozacc + c0 * g.ldoz + row;
          double zo[32];
          if (gi != gfirst) {
            #pragma unroll
            for (int j = 0; j < 32; ++j) zo[j] = z[j * g.ldoz];
          }
          if (gi > 2) {                                  // Ozaki group: FP64 accumulate
            #pragma unroll
            for (int j = 0; j < 32; ++j) {
              const double v = __dmul_rn((double)(int32_t)r[j], pow2(rs + g.oz_csig[c0 + j] - 7 * gi));
              z[j * g.ldoz] = gi == gfirst ? v : __dadd_rn(zo[j], v);
            }
          } else {                                       // group 2: complete Z, then the finish epilogue
            #pragma unroll
            for (int j = 0; j < 32; ++j) {
              const double pv = __dmul_rn((double)(int32_t)r[j], pow2(rs + g.oz_csig[c0 + j] - 14));
              zo[j] = gfirst > 2 ? __dadd_rn(zo[j], pv) : pv;
            }
            epi_row_f64(g, row, c0, zo, ea);
          }
        } else {
          epi_chunk<KIND>(g, row, colb + ch * 32, r, scale, ea);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty[buf], 0);
      if (crt || (ozg && gi > 2)) { ++it; continue; }   // partials after the finish only
      // per-tile partials: deterministic (fixed shuffle tree, warps summed in order 0..3)
      const bool need_s = (g.mode & (EPI_RESID | EPI_UPDATE | EPI_NSUPDATE | EPI_SYMUPD)) != 0;
      if (need_s || g.pmax) {
        double s = (g.mode & EPI_RESID) ? ea.r2 : ea.d2;
        float mx = ea.mx;
        if (need_s) {                                    // FP64 only when a sum partial is wanted
          #pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) { red[it & 1][hh * 4 + q] = s; redm[it & 1][hh * 4 + q] = mx; }
        asm volatile("bar.sync 1, 256;\n" ::: "memory");
        if (et == 0) {
          const int64_t tile = ((g.col0 + colb) / TC_BN) * g.tiles_m + g.row0 / TC_BM + tile_m;
          if (need_s)
          {
            const double *rr = red[it & 1];
            double acc = 0.0;
            #pragma unroll
            for (int w = 0; w < 8; ++w) acc += rr[w];
            g.part[tile] = acc;
          }
          if (g.pmax)
          {
            float m8 = 0.f;
            #pragma unroll
            for (int w = 0; w < 8; ++w) m8 = fmaxf(m8, redm[it & 1][w]);
            g.pmax[tile] = m8;
          }
        }
      }
      ++it;
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
  if (KIND == 3 && EF == 3 && g.pdl) asm volatile("griddepcontrol.wait;\n" ::: "memory");   // predecessor done
}

// ---------------------------------------------------------------------------------------
// host side: tensor maps through the driver entry point (no -lcuda link dependency)
// ---------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

char g_tc_err[256] = "";
const char *tc_last_error() { return g_tc_err; }

static int num_sms() {            // per device ordinal (cached)
  static int cache[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev];
}

cudaError_t launch_gemm_tc(const GemmArgs &a_in, cudaStream_t s) {
  GemmArgs a = a_in;
  if (!a.mout) { a.mout = a.tout; a.ldm = a.ldt; }   // tri mirror: in place at G = 1
  if (!tc_supported(a.prec)) return cudaErrorNotSupported;
  if (a.M % (2 * TC_BM) || a.N % TC_BN || a.K % 128 || a.a_kp % 128) {
    snprintf(g_tc_err, sizeof g_tc_err, "tcgen05 GEMM: sizes M=%lld N=%lld K=%lld kp=%lld not tile multiples",
             (long long)a.M, (long long)a.N, (long long)a.K, (long long)a.a_kp);
    return cudaErrorInvalidValue;
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) {
    snprintf(g_tc_err, sizeof g_tc_err, "cuTensorMapEncodeTiled entry point unavailable");
    return cudaErrorNotSupported;
  }
  const int esz = elt_size(a.prec);
  const CUtensorMapDataType dt = a.prec == P_BF16   ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                 : a.prec == P_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                 : (a.prec == P_FP8 || a.prec == P_INT8) ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const cuuint32_t bke = TC_BKB / esz;
  CUtensorMap ma, mb;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)a.a_kp, (cuuint64_t)a.M, (cuuint64_t)(a.K / a.a_kp)};
    const cuuint64_t strides[2] = {(cuuint64_t)(a.a_kp * esz), (cuuint64_t)(a.a_pstride * esz)};
    const cuuint32_t box[3] = {bke, (cuuint32_t)TC_BM, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&ma, dt, 3, (void *)a.A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      snprintf(g_tc_err, sizeof g_tc_err, "cuTensorMapEncodeTiled(A) failed");
      return cudaErrorInvalidValue;
    }
  }
  if (a.b_pstride) {   // K-concatenated B planes (fused symmetric update; 2-D grid T panels): [K / b_kp][N][b_kp]
    const int64_t bkp = a.b_kp ? a.b_kp : a.a_kp;
    const cuuint64_t dims[3] = {(cuuint64_t)bkp, (cuuint64_t)a.N, (cuuint64_t)(a.K / bkp)};
    const cuuint64_t strides[2] = {(cuuint64_t)(a.ldb * esz), (cuuint64_t)(a.b_pstride * esz)};
    const cuuint32_t box[3] = {bke, (cuuint32_t)(TC_BN / 2), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&mb, dt, 3, (void *)a.B, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      snprintf(g_tc_err, sizeof g_tc_err, "cuTensorMapEncodeTiled(B, 3-D) failed");
      return cudaErrorInvalidValue;
    }
  } else {
    // CRT: the residue planes of the B operand stacked along N ([crt_n][N][a_kp])
    const cuuint64_t dims[2] = {(cuuint64_t)(a.oz_grouped == 3 ? a.a_kp : a.K),
                                (cuuint64_t)(a.oz_grouped == 3 ? a.N * a.crt_n : a.N)};
    const cuuint64_t strides[1] = {(cuuint64_t)(a.ldb * esz)};
    const cuuint32_t box[2] = {bke, (cuuint32_t)(TC_BN / 2)};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&mb, dt, 2, (void *)a.B, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      snprintf(g_tc_err, sizeof g_tc_err, "cuTensorMapEncodeTiled(B) failed");
      return cudaErrorInvalidValue;
    }
  }
  if (a.tri && a.col0 + a.N > a.M) {   // (K is crt_n npad for the CRT moduli products)
    snprintf(g_tc_err, sizeof g_tc_err, "tcgen05 GEMM: tri needs a square product (or a column panel of one)");
    return cudaErrorInvalidValue;
  }
  const TileSched hs{(int)(a.M / (2 * TC_BM)), (int)(a.N / TC_BN), a.tri, (int)(a.col0 / TC_BN)};
  const int ntiles = hs.count() * (a.oz_grouped == 3 ? a.crt_l1 - a.crt_l0 : 1);
  if (a.tri && (a.mode & (EPI_RESID | EPI_SYMUPD)) && a.oz_grouped != 3) {   // the tiles below the diagonal are not visited: zero partials
    cudaError_t z = cudaMemsetAsync(a.part + (a.col0 / TC_BN) * a.tiles_m, 0, (size_t)(a.N / TC_BN) * a.tiles_m * sizeof(double), s);
    if (z != cudaSuccess) return z;
  }
  {
    static int diag = -1;
    if (diag < 0) { const char *v = getenv("IPR_DIAG_EPI"); diag = v ? atoi(v) : 0; }
    a.diag_epi = diag;
  }
  const int maxpairs = num_sms() / 2;
  const int grid = 2 * (ntiles < maxpairs ? ntiles : maxpairs);
  cudaError_t e = cudaSuccess;
  const bool symupd = (a.mode & EPI_SYMUPD) != 0;
  if (symupd && tc_kind(a.prec) > 1) return cudaErrorNotSupported;
  const int sel = tc_kind(a.prec) != 3 || !a.oz_grouped ? tc_kind(a.prec) + (symupd ? 4 : 0)
                  : a.oz_grouped == 3 ? 7 : 6;
  switch (sel) {
#define TC_LAUNCH(C, K, EF)                                                                              \
    case C: {                                                                                            \
      static DeviceOnce attr;                                                                            \
      if (!attr.done()) {                                                                                \
        e = cudaFuncSetAttribute(k_gemm_tc<K, EF>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM); \
        if (e != cudaSuccess) return e;                                                                  \
        attr.set();                                                                                      \
      }                                                                                                  \
      if (a.pdl) {                                                                                       \
        cudaLaunchConfig_t cfg = {};                                                                     \
        cudaLaunchAttribute at[1];                                                                       \
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                   \
        at[0].val.programmaticStreamSerializationAllowed = 1;                                            \
        cfg.gridDim = dim3((unsigned)grid); cfg.blockDim = dim3(TC_NT); cfg.dynamicSmemBytes = TC_SMEM;  \
        cfg.stream = s; cfg.attrs = at; cfg.numAttrs = 1;                                                \
        e = cudaLaunchKernelEx(&cfg, k_gemm_tc<K, EF>, ma, mb, a);                                       \
        if (e != cudaSuccess) return e;                                                                  \
      } else {                                                                                           \
        k_gemm_tc<K, EF><<<grid, TC_NT, TC_SMEM, s>>>(ma, mb, a);                                        \
      }                                                                                                  \
    } break;
    TC_LAUNCH(0, 0, 0)
    TC_LAUNCH(1, 1, 0)
    TC_LAUNCH(2, 2, 0)
    TC_LAUNCH(3, 3, 0)
    TC_LAUNCH(4, 0, 1)
    TC_LAUNCH(5, 1, 1)
    TC_LAUNCH(6, 3, 2)
    TC_LAUNCH(7, 3, 3)
#undef TC_LAUNCH
  }
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace ipr
