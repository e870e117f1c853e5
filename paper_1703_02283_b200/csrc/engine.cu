// engine.cu -- the C-ABI (include/ipr.h), iteration engine and host precision-switch
// controller of libipr.
//
// Per iteration k in phase phi:
//   p GEMMs  T_1 = Chat Ahat, T_j = Chat qin(T_{j-1})     (R-1, Eq. (1))
//            the p-th with the fused residual partials      (R-4)
//   deterministic reduction -> rho; ONE 16-byte D2H + stream sync (the only host round trip)
//   controller (R-5) -> continue / switch / stop
//   GEMM p+1 with the fused FP64 update C_{k+1} = q_m(((p+1)C_k - P)/p)   (R-2)
//   world > 1: NCCL all-gather of Chat_{k+1} panels in the operand format
//
// Multi-GPU layout ("1 x G" column panels): rank g owns columns
// S_g = [g*kp, (g+1)*kp) of A, T_j and C_{k+1}; Chat is replicated in a panel-major buffer
// [G][npad][kp] so one in-place ncclAllGather assembles it; every per-tile partial has a
// global slot so rho / delta are reduced in the same fixed order for any G.
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <dlfcn.h>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ipr.h"
#include "../../include/ipr_testing.h"
#include "common.cuh"
#include "kernels.h"
#include "nccl_dl.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a tool (nsys) injects

using namespace ipr;

namespace {

thread_local std::string t_err;

// NVTX range per hot-path step (chain / update / certificate / phase entry / exchanges), named by format
struct Nvtx {
  explicit Nvtx(const char *fmt, ...) {
    char b[96];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(b, sizeof b, fmt, ap);
    va_end(ap);
    nvtxRangePushA(b);
  }
  ~Nvtx() { nvtxRangePop(); }
};
const char *pname(int prec) {
  static const char *nm[] = {"fp64", "tf32", "bf16", "fp16", "fp8", "int8", "fp64oz", "fp64crt"};
  return prec >= 0 && prec < 8 ? nm[prec] : "?";
}

struct PhaseC {
  int prec, m, rtz, cont64;
  int adaptive;                // FP64_OZ with mant_bits = IPR_MANT_ADAPTIVE (reading R-26)
  int corr;                    // symmetric form: operand format of the correction GEMM
  double switch_tol, plateau_ratio, plateau_arm;
  int max_iters;
};

}  // namespace

struct ipr_ctx {
  int64_t n = 0, lda = 0, npad = 0, kp = 0, col0 = 0;
  int world = 1, rank = 0;
  // grid: grows x gcols ranks, this rank at (grow, gcol); it owns rows [row0, row0 + mr)
  // and columns [col0, col0 + kp).  The default 1 x world grid: mr = npad, row0 = 0, gcol = rank.
  int grows = 1, gcols = 1, grow = 0, gcol = 0;
  int64_t mr = 0, row0 = 0;
  Transport *rowt = nullptr, *colt = nullptr;   // 2-D grid: the rank's grid row / grid column
  void *Tcol = nullptr;                 // 2-D grid: gathered T column panel [grows][kp][mr] (B operand)
  double *partg = nullptr;              // 2-D grid: every rank's full partial array [world][npart]
  cudaStream_t st = nullptr;
  const double *A = nullptr;
  double *Aown = nullptr;               // host A at ipr_init: the library's device copy (pool block)
  // ipr_set_output: the destination of ipr_finalize, where the certified candidate is streamed while
  // its FP64 certificate runs (G = 1, FP64 container); valid once the solve converged on that buffer
  double *out_ptr = nullptr;
  int64_t out_ld = 0;
  cudaStream_t ost = nullptr;
  cudaEvent_t oev = nullptr, orev = nullptr;
  int out_buf = -1;                     // iterate buffer whose copy is in flight / done (-1: none)
  bool out_valid = false;
  double norms[4] = {0, 0, 0, 0};
  std::string err;
  Transport *comm = nullptr;           // world > 1: NCCL (ipr_init) or an in-process local group (ipr_testing.h)
  cudaStream_t cst = nullptr;           // world > 1: side stream of the Chat all-gathers that overlap GEMM 1
  cudaEvent_t gev[2] = {nullptr, nullptr};
  bool gpend = false;                   // an all-gather on cst that the compute stream has not joined yet
  void *chat_rm = nullptr;              // world > 1, CRT phases: row-major FP64 Chat (the A-role residue split)
  void *msend = nullptr, *mrecv = nullptr;   // world > 1, tri form: packed [G][kp][kp] mirror exchange buffers
  // schedule
  int p = 0;
  std::vector<PhaseC> ph;
  double final_tol = 0.0;
  bool scheduled = false, started = false, done = false;
  int outcome = IPR_RUNNING;
  // controller state (reading R-5)
  int phase = 0, it_in_phase = 0;
  double rho_prev = NAN, rho_best = INFINITY, rhohat_min = INFINITY, last_rho = NAN;
  // device buffers
  void *chat[2] = {nullptr, nullptr};   // operand Chat, panel-major [G][npad][kp], 8 B slots
  void *cont[2] = {nullptr, nullptr};   // container local panel [npad][kp]
  double *best = nullptr;                // FP64 local panel
  void *T[2] = {nullptr, nullptr};      // chain intermediates, K-major [kp][npad]
  void *Aop = nullptr;                  // stage-A operand of the current phase [kp][npad]
  void *Afull = nullptr;                // NS / symmetric, world > 1: full row-major Ahat (A operand)
  void *chatc[2] = {nullptr, nullptr};  // symmetric form: Chat in the correction format (panel-major)
  void *wbuf = nullptr;                 // symmetric form: W = qc(C) Rhat, full panel-major
  int wbytes = 4;                       // allocated element size of wbuf (8 if any FP64 correction)
  void *Zr = nullptr;                   // symmetric form, G = 1: Z_1 = A C row-major (FP64 phases)
  // FP64 via Ozaki on INT8 tensor cores (IPR_FP64_OZ phases, reading R-23): digit planes (A role)
  // and per-column digit rows (B role) of Ahat, of Chat (one set per iterate buffer) and of the
  // current B operand, their scale exponents, and the FP64 accumulator (transposed)
  int8_t *ozA = nullptr, *ozC[2] = {nullptr, nullptr}, *ozCb[2] = {nullptr, nullptr}, *ozB = nullptr;
  int *ozA_sig = nullptr, *ozC_sig[2] = {nullptr, nullptr}, *ozB_sig = nullptr;
  double *ozacc = nullptr;
  // FP64 via the Ozaki scheme II (IPR_FP64_CRT phases, reading R-28): residue planes [CRT_MAX][npad]
  // [npad] of Ahat, of Chat (per iterate buffer; symmetric, so one set serves both roles) and of the
  // current B operand, their exponents, the bits b each set was split with (-1: stale), and the
  // byte scratch of the modulus products
  // ONE Chat set (keyed by iterate buffer and bits; re-split lazily -- at n = 32768 a set is 19 GB)
  int8_t *crA = nullptr, *crC = nullptr, *crB = nullptr;
  int *crA_sig = nullptr, *crC_sig = nullptr, *crB_sig = nullptr;
  int crA_b = -1, crC_for = -1, crC_b = -1;
  uint8_t *crV = nullptr;
  // symmetric-tri form, fused update (EPI_SYMUPD): per iterate buffer [Chat | Rhat | Chat] in the
  // correction format -- the A operand [Chat | Rhat] is planes 0-1, the B operand [Rhat ; Chat] planes 1-2
  void *qbuf[2] = {nullptr, nullptr};
  // coupled form (R-27): Mhat and Nhat K-major local panels (ping-pong), Nhat as the replicated A
  // operand (panel-major), which set is current, and whether the next chain must re-anchor M
  void *cM[2] = {nullptr, nullptr}, *cNk[2] = {nullptr, nullptr}, *cNf = nullptr;
  int cmi = 0;
  bool c_anchor = true;
  int zr_for = -1;                      // iterate buffer whose chain wrote Zr (-1: none)
  // dynamic precision inside an FP64_OZ phase (R-26): digits of this chain, stored bits of the
  // next iterate and of the current one, the last two in-phase residuals
  int oz_S_cur = OZ_S, oz_m_next = 52, m_of_cur = 52, last_chain_S = 0;
  int last_chain_ztri = 0;              // R-37: the last chain took Z_1 from its upper tiles (record.ztri)
  double ph_r1 = NAN, ph_r2 = NAN;
  bool triz = false;                    // IPR_FORM_SYMMETRIC_TRIZ (reading R-37): form = SYMMETRIC_TRI + the Z_1 rule
  bool z_ok = true;                     // R-37: no in-phase ratio rho_k / rho_{k-1} above kZtriRatio so far
  int form = IPR_FORM_LITERAL;          // iteration form (ipr_set_form)
  float *tscr = nullptr;                // FP16 phase T scratch (FP32)
  double *full64 = nullptr;             // FP64 npad x npad scratch (copy-out / certify)
  void *Acert = nullptr;                // FP64 Ahat for certify
  double *part = nullptr; float *pmax = nullptr; int64_t npart = 0;
  double *dscal = nullptr; double *hscal = nullptr;   // [0] rho^2 [1] delta^2 [2] max
  int *dsig = nullptr;                  // [0] sigma_A(phase) [1,2] sigma_C ping-pong [3,4] sigma_T
  double *colsum = nullptr; int *dflag = nullptr;
  double kern_ms = 0.0;                 // CRT: device time of the last chain's kind::i8 GEMM launches
  int cur = 0;
  int best_loc = -1;                    // 0/1: cont[best_loc] holds the best; 2: `best`; -1 none
  int best_cont64 = 1;
  int64_t pending_delta = -1;           // trace record whose delta is in flight
  std::vector<ipr_record> trace;
  void *arena = nullptr;                // every O(n^2) buffer: ONE pool allocation at the first ipr_iterate
  void *aux = nullptr;                  // the small device buffers (flag, scalars, sigmas, colsum)
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // [4]: chain's results ready
  cudaEvent_t kev[16] = {};             // CRT: event pairs around the kind::i8 GEMM launches of a chain
  CrtTimer ktimer{kev, 8, 0};
  bool upd_timed = false;
  int cert = IPR_CERT_FP64;             // convergence certificate of the symmetric / coupled forms (ipr_set_cert)
  bool cert_pending = false;            // R-33: certify the next iterate before (instead of) its chain
  // IPR_TIMELINE=1 (diagnostics): CUDA events at the start of every activity of the solve; the device
  // time per activity (and the idle gaps between them) is printed to stderr at ipr_finalize
  bool tl_on = false;
  std::vector<std::pair<const char *, cudaEvent_t>> tl;
  double cert_prev = NAN;               // R-33: that certificate missed: its value, for the chain's record
  // IPR_CERT_CRT (reading R-35): per-row quantities of the certificate's splits [8][npad], the pinned
  // host copy of its reductions, and the last certificate's components (ipr_test_cert_info)
  double *certv = nullptr;
  double *hcert = nullptr;
  double cert_info[10] = {NAN, NAN, NAN, NAN, NAN, NAN, NAN, NAN, NAN, NAN};
  std::vector<size_t> guards;           // ipr_test_set_guards: arena offsets of the guard bands
};

namespace {

// Process-wide pinned slab for the per-context 8-double D2H scalars (cudaMallocHost /
// cudaFreeHost synchronise the device and can stall for 100+ ms: never on the solve path).
constexpr int kPinnedSlots = 1024;
std::mutex g_pin_mu;
double *g_pin_base = nullptr;
bool g_pin_used[kPinnedSlots] = {};
double *pinned_acquire() {
  std::lock_guard<std::mutex> lock(g_pin_mu);
  if (!g_pin_base && cudaMallocHost((void **)&g_pin_base, (size_t)kPinnedSlots * 64) != cudaSuccess) {
    cudaGetLastError();
    g_pin_base = nullptr;
    return nullptr;
  }
  for (int i = 0; i < kPinnedSlots; ++i)
    if (!g_pin_used[i]) { g_pin_used[i] = true; return g_pin_base + 8 * i; }
  return nullptr;
}
void pinned_release(double *p) {
  std::lock_guard<std::mutex> lock(g_pin_mu);
  const int64_t i = (p - g_pin_base) / 8;
  if (g_pin_base && i >= 0 && i < kPinnedSlots) g_pin_used[i] = false;
}

void tl_mark(ipr_ctx *c, const char *what) {
  if (!c->tl_on) return;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess || cudaEventRecord(e, c->st) != cudaSuccess) { cudaGetLastError(); return; }
  c->tl.push_back({what, e});
}
void tl_report(ipr_ctx *c) {
  if (!c->tl_on || c->tl.size() < 2) return;
  cudaStreamSynchronize(c->st);
  std::vector<std::pair<std::string, double>> acc;
  double total = 0.0;
  for (size_t i = 0; i + 1 < c->tl.size(); ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->tl[i].second, c->tl[i + 1].second) != cudaSuccess) { cudaGetLastError(); continue; }
    total += ms;
    bool found = false;
    for (auto &a : acc) if (a.first == c->tl[i].first) { a.second += ms; found = true; }
    if (!found) acc.push_back({c->tl[i].first, (double)ms});
  }
  fprintf(stderr, "ipr timeline (device ms): total %.3f", total);
  for (auto &a : acc) fprintf(stderr, " | %s %.3f", a.first.c_str(), a.second);
  fprintf(stderr, "\n");
  for (auto &m : c->tl) cudaEventDestroy(m.second);
  c->tl.clear();
}

// host memory (pinned, or pageable / unknown to CUDA) rather than device or managed memory
bool is_host_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return true; }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

// One retained stream-ordered memory pool per device (release threshold = unlimited): the
// arenas of back-to-back solves are recycled without driver (un)mapping.
cudaMemPool_t arena_pool() {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!pools[dev]) {
    cudaMemPoolProps props;
    memset(&props, 0, sizeof props);
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) { cudaGetLastError(); return nullptr; }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[dev] = p;
  }
  return pools[dev];
}

ipr_status fail(ipr_ctx *c, ipr_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  if (c) c->err = buf;
  return s;
}

#define CK(expr)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return fail(c, IPR_E_CUDA, "%s:%d %s: %s %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e), tc_last_error()); \
  } while (0)
#define CKS(expr)                                                                             \
  do {                                                                                        \
    ipr_status _s = (expr);                                                                   \
    if (_s != IPR_OK) return _s;                                                              \
  } while (0)

int native_m(int prec) {
  return is_f64(prec) ? 52 : (prec == IPR_BF16 || prec == IPR_INT8) ? 7 : prec == IPR_FP8 ? 3 : 10;
}

// padded order: whole 256-wide tiles per rank (tcgen05 tile N), zero padding
int64_t padded_order(int64_t n, int world) {
  const int64_t unit = 256 * (int64_t)world;
  return (n + unit - 1) / unit * unit;
}
int operand_bits(int prec) { return native_m(prec); }

template <typename T>
ipr_status dalloc(ipr_ctx *c, T **p, size_t bytes) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc((void **)p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, IPR_E_OOM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
  }
  return IPR_OK;
}

// elements of this rank's block (1 x G: the column panel npad x kp; 2-D: mr x kp)
inline int64_t blk(const ipr_ctx *c) { return c->mr * c->kp; }
inline size_t slot_bytes(const ipr_ctx *c) { return (size_t)blk(c) * 8; }

// container of iterate buffer i in the current phase (FP64 phases alias the operand slot).  The operand
// Chat is replicated along the rank's grid row: [gcols][mr][kp], this rank's block at slot gcol.
void *cont_ptr(ipr_ctx *c, int i, const PhaseC &P) {
  if (is_f64(P.prec)) return (char *)c->chat[i] + (size_t)c->gcol * slot_bytes(c);
  return c->cont[i];
}
void *chat_slot(ipr_ctx *c, int i, int prec) {
  return (char *)c->chat[i] + (size_t)c->gcol * (size_t)blk(c) * elt_size(prec);
}
// the transport of the Chat / W / partial-panel exchanges: the grid row (all ranks for 1 x G)
inline Transport *row_transport(ipr_ctx *c) { return c->rowt ? c->rowt : c->comm; }

ipr_status gather_chat(ipr_ctx *c, int i, int prec) {
  if (c->gcols == 1) return IPR_OK;
  // packed panel-major layout for this precision: grid-row slot r at r * mr * kp * esz
  const size_t bytes = (size_t)blk(c) * elt_size(prec);
  char *base = (char *)c->chat[i];
  Transport *t = row_transport(c);
  if (!t->allgather(base + c->gcol * bytes, base, bytes, c->st))
    return fail(c, IPR_E_NCCL, "ncclAllGather(Chat) failed: %s", t->last_error());
  return IPR_OK;
}

// world > 1, symmetric forms: the all-gather of Chat_{k+1} (and its correction-format copy) runs on the
// side stream cst while GEMM 1 of the next chain (Z_1 = Ahat Chat[:, S_g]: the LOCAL panel only) runs on
// the compute stream; join_gather() before the first GEMM that reads the whole Chat (SURVEY 8(e)
// overlap; PAPER.md:138-141 data exchange)
ipr_status gather_bytes_async(ipr_ctx *c, void *base, size_t per_rank, const char *what) {
  if (c->world == 1) return IPR_OK;
  if (!c->gpend) {
    CK(cudaEventRecord(c->gev[0], c->st));
    CK(cudaStreamWaitEvent(c->cst, c->gev[0], 0));
  }
  if (!c->comm->allgather((char *)base + c->rank * per_rank, base, per_rank, c->cst))
    return fail(c, IPR_E_NCCL, "all-gather(%s) failed: %s", what, c->comm->last_error());
  CK(cudaEventRecord(c->gev[1], c->cst));
  c->gpend = true;
  return IPR_OK;
}
ipr_status join_gather(ipr_ctx *c) {
  if (!c->gpend) return IPR_OK;
  CK(cudaStreamWaitEvent(c->st, c->gev[1], 0));
  c->gpend = false;
  return IPR_OK;
}

// A-operand view of Chat for the GEMMs: element (i,k) at (k/kp)*pstride + i*kp + k%kp
void chat_view(ipr_ctx *c, int i, int prec, const void **A, int64_t *akp, int64_t *pstride) {
  *A = c->chat[i];
  *akp = c->kp;
  *pstride = blk(c);
  (void)prec;
}

// per-tile partials: every GEMM writes its tiles' sums at GLOBAL slots [tile_n][tile_m], so the reduction
// order is the same for any decomposition.  1 x G: a rank's tiles are one contiguous chunk (per_rank
// slots at rank * per_rank).  2-D grid: a rank's slots are scattered -- every rank's whole array is
// gathered and each slot taken from its owner (tile sizes tmsz x tnsz of the kernel that wrote them).
ipr_status gather_partials(ipr_ctx *c, double *part, int64_t per_rank, int tmsz = 0, int tnsz = 0) {
  if (c->world == 1) return IPR_OK;
  if (c->grows == 1) {
    if (!c->comm->allgather(part + c->rank * per_rank, part, (size_t)per_rank * 8, c->st))
      return fail(c, IPR_E_NCCL, "ncclAllGather(partials) failed: %s", c->comm->last_error());
    return IPR_OK;
  }
  if (!tmsz || !tnsz) return fail(c, IPR_E_UNSUPPORTED, "2-D grid: partials without tile sizes");
  const int64_t total = per_rank * c->gcols;   // tiles_n_total * tiles_m
  if (!c->comm->allgather(part, c->partg, (size_t)total * 8, c->st))
    return fail(c, IPR_E_NCCL, "all-gather(2-D partials) failed: %s", c->comm->last_error());
  CK(launch_select_partials(c->partg, total, c->npad / tmsz, tmsz, tnsz, c->mr, c->kp, c->gcols, part, c->st));
  return IPR_OK;
}
ipr_status gather_pmax(ipr_ctx *c, float *pm, int64_t per_rank) {
  if (c->world == 1) return IPR_OK;
  if (!c->comm->allgather(pm + c->rank * per_rank, pm, (size_t)per_rank * 4, c->st))
    return fail(c, IPR_E_NCCL, "ncclAllGather(max partials) failed: %s", c->comm->last_error());
  return IPR_OK;
}

int64_t tiles_m(const ipr_ctx *c, int prec) { return c->npad / gemm_tile_m(prec); }
int64_t tiles_n_total(const ipr_ctx *c, int prec) { return c->npad / gemm_tile_n(prec); }

cudaError_t run_gemm(ipr_ctx *c, GemmArgs &g) {
  if (g.prec == IPR_FP64_OZ) return launch_gemm_ozaki(g, c->st);
  if (g.prec == IPR_FP64_CRT) return launch_gemm_crt(g, c->st);
  return g.prec == IPR_FP64 ? launch_gemm_dmma(g, c->st) : launch_gemm_tc(g, c->st);
}

GemmArgs base_args(ipr_ctx *c, int prec, const void *Bop) {
  GemmArgs g;
  memset(&g, 0, sizeof g);
  g.M = c->mr; g.N = c->kp; g.K = c->npad; g.n = c->n; g.col0 = c->col0; g.row0 = c->row0;
  g.B = Bop; g.ldb = c->npad; g.prec = prec; g.tprec = prec;
  g.tiles_m = tiles_m(c, prec);
  g.p = c->p;
  return g;
}

// ---- stage A for a phase (a1) ----
ipr_status stage_a(ipr_ctx *c, const PhaseC &P, void *dst, int *sig_dst) {
  const int *sig = nullptr;
  if (is_scaled(P.prec)) {
    const int nparts = 1024;
    CK(launch_maxabs_qA(c->A, c->lda, c->n, P.cont64, P.m, P.rtz, c->pmax, nparts, c->st));
    CK(launch_reduce_max(c->pmax, nparts, nullptr, sig_dst, P.prec, c->st));
    sig = sig_dst;
  }
  CK(launch_stage_a(c->A, c->lda, c->n, c->npad, c->col0, c->kp, P.prec, P.cont64, P.m, P.rtz, sig, dst, c->st));
  return IPR_OK;
}

// container cont(i) -> operand Chat(i) (+ FP16 sigma), then all-gather (a8 / a9)
// premax: the per-rank max |C| is already in pmax[rank] (k_sym_update's amax), one partial per rank
ipr_status make_operand(ipr_ctx *c, int i, const PhaseC &P, bool premax = false, bool async = false) {
  const int64_t cnt = blk(c);
  if (!is_f64(P.prec)) {
    const int *sig = nullptr;
    if (is_scaled(P.prec)) {
      const int nparts = premax ? 1 : 256;
      if (!premax) CK(launch_maxabs_cont(c->cont[i], P.cont64, cnt, c->pmax + c->rank * nparts, nparts, c->st));
      CKS(gather_pmax(c, c->pmax, nparts));
      CK(launch_reduce_max(c->pmax, (int64_t)nparts * c->world, nullptr, c->dsig + 1 + i, P.prec, c->st));
      sig = c->dsig + 1 + i;
    }
    CK(launch_make_operand(cont_ptr(c, i, P), P.cont64, cnt, P.prec, sig, chat_slot(c, i, P.prec), c->st));
  }
  if (async) return gather_bytes_async(c, c->chat[i], (size_t)cnt * elt_size(P.prec), "Chat");
  return gather_chat(c, i, P.prec);
}

// materialise the best iterate into c->best (FP64 local panel)
ipr_status save_best(ipr_ctx *c) {
  if (c->best_loc == 0 || c->best_loc == 1) {
    const PhaseC &P = c->ph[c->phase];
    (void)P;
    const int64_t cnt = blk(c);
    const void *src = c->best_cont64 ? (const void *)((char *)c->chat[c->best_loc] + (size_t)c->gcol * slot_bytes(c))
                                     : c->cont[c->best_loc];
    // FP64 phases keep the iterate in the operand slot; low phases in cont[]
    CK(launch_cont_to_f64(src, c->best_cont64, cnt, c->best, c->st));
    c->best_loc = 2;
  }
  return IPR_OK;
}

ipr_status make_xt(ipr_ctx *c, int i, const PhaseC &P);
ipr_status coupled_gather_n(ipr_ctx *c);
// Ozaki digits of the FP64 iterate in buffer i (exactly symmetric, G = 1: its columns are its rows)
// R-26: digits for a target RMS residual, and the stored bits that go with them
int oz_digits_for(double rho_hat_target, int64_t n) {
  if (!(rho_hat_target > 0.0) || !std::isfinite(rho_hat_target)) return OZ_S;
  const double b = std::log2(30.0 * std::sqrt((double)n)) - std::log2(rho_hat_target);
  int S = (int)std::ceil(b / 7.0);
  return S < 3 ? 3 : S > OZ_S ? OZ_S : S;
}
int oz_adaptive_m(int S) { return 7 * S - 4 < 52 ? 7 * S - 4 : 52; }
// digits of the current chain's products: fixed per phase (m), or per iteration (R-26)
int oz_S_now(const ipr_ctx *c) {
  const PhaseC &P = c->ph[c->phase];
  return P.adaptive ? c->oz_S_cur : oz_digits(P.m);
}
ipr_status oz_split_chat(ipr_ctx *c, int i) {   // always all OZ_S digits; a product uses the leading S
  CK(launch_oz_split((const double *)c->chat[i], c->npad, c->npad, c->npad, OZ_S, c->ozC[i], c->ozCb[i],
                     c->ozC_sig[i], c->st));
  return IPR_OK;
}
// Ozaki operands of a GEMM: A = the iterate buffer i's digits (or Ahat's if i < 0), B = digits of
// the rows of the K-major B operand Xt (npad x npad FP64), split now into the scratch set
ipr_status oz_operands(ipr_ctx *c, GemmArgs &g, int i, const void *Xt) {
  CK(launch_oz_split((const double *)Xt, c->npad, c->npad, c->npad, OZ_S, nullptr, c->ozB, c->ozB_sig, c->st));
  g.oz_S = oz_S_now(c);
  g.oz_a = i < 0 ? c->ozA : c->ozC[i];
  g.oz_rsig = i < 0 ? c->ozA_sig : c->ozC_sig[i];
  g.oz_b = c->ozB; g.oz_csig = c->ozB_sig;
  g.ozacc = c->ozacc; g.ldoz = c->npad;
  return IPR_OK;
}
// Ozaki scheme II (R-28): residues of Ahat / Chat(i) with the bits of the current chain (split only
// when stale), and of the K-major B operand Xt (split now)
int crt_bits_now(const ipr_ctx *c) { return crt_bits(oz_S_now(c), c->n); }
ipr_status crt_ensure_a(ipr_ctx *c, int b) {
  if (c->crA_b == b) return IPR_OK;
  // the A role needs every row of Ahat: G = 1 its K-major local panel is the whole (symmetric) Ahat;
  // G > 1 the full row-major copy the symmetric forms keep
  CK(launch_crt_split((const double *)(c->world > 1 ? c->Afull : c->Aop), c->npad, c->npad, c->npad, b,
                      crt_moduli(b, c->n), c->crA, c->crA_sig, c->st));
  c->crA_b = b;
  return IPR_OK;
}
ipr_status crt_ensure_c(ipr_ctx *c, int i, int b) {
  if (c->crC_for == i && c->crC_b == b) return IPR_OK;
  const double *src = (const double *)c->chat[i];
  if (c->world > 1) {   // panel-major [G][npad][kp] -> row-major (the split takes whole rows)
    CKS(join_gather(c));
    CK(launch_copy_out((const double *)c->chat[i], c->npad, c->kp, c->n, (double *)c->chat_rm, c->npad, c->st));
    src = (const double *)c->chat_rm;
  }
  CK(launch_crt_split(src, c->npad, c->npad, c->npad, b, crt_moduli(b, c->n), c->crC, c->crC_sig, c->st));
  c->crC_for = i; c->crC_b = b;
  return IPR_OK;
}
void crt_args(ipr_ctx *c, GemmArgs &g, int b) {
  g.crt_n = crt_moduli(b, c->n);
  g.crt_v = c->crV;
}
// A role: iterate buffer i (or Ahat if i < 0); B role: the rows of the K-major Xt
ipr_status crt_operands(ipr_ctx *c, GemmArgs &g, int i, const void *Xt) {
  const int b = crt_bits_now(c);
  if (i < 0) CKS(crt_ensure_a(c, b));
  else CKS(crt_ensure_c(c, i, b));
  // B role: the kp rows of the K-major local panel Xt (the columns of this rank)
  CK(launch_crt_split((const double *)Xt, c->npad, c->kp, c->npad, b, crt_moduli(b, c->n), c->crB, c->crB_sig, c->st));
  g.oz_a = i < 0 ? c->crA : c->crC;
  g.oz_rsig = i < 0 ? c->crA_sig : c->crC_sig;
  g.oz_b = c->crB; g.oz_csig = c->crB_sig;
  crt_args(c, g, b);
  return IPR_OK;
}
// fused symmetric update (EPI_SYMUPD) for this phase: tri form, one GPU, unscaled phase operands and a
// tcgen05 correction format
// Off by default (IPR_FUSED_SYMUPD=1 enables it): measured 1.39 ms per n = 8192 update against 1.08 ms
// for the W GEMM + k_sym_update pair -- with K = 2n a wave's operand blocks (~136 MB) exceed L2 and the
// epilogue's FP64 conversions and stores compete with the operand streams.
bool fused_sym_ok(const ipr_ctx *c, const PhaseC &P) {
  static int on = -1;
  if (on < 0) { const char *v = getenv("IPR_FUSED_SYMUPD"); on = v && atoi(v) ? 1 : 0; }
  return on && c->world == 1 && c->form == IPR_FORM_SYMMETRIC_TRI && !is_scaled(P.prec) &&
         (P.corr == IPR_BF16 || P.corr == IPR_TF32) && tc_supported(P.corr);
}
void *qplane(ipr_ctx *c, int i, int prec, int plane) {
  return (char *)c->qbuf[i] + (size_t)plane * (size_t)(c->npad * c->npad) * elt_size(prec);
}
// operand formats that share storage (FP64 and FP64-by-Ozaki both keep Chat in FP64)
inline bool same_fmt(int a, int b) { return a == b || (is_f64(a) && is_f64(b)); }
// IPR_CERT_CRT (reading R-35): the certificate quantises its operands to 62 bits (18 moduli up to n = 86000)
constexpr int kCertBits = 62;
inline bool is_sym(const ipr_ctx *c) { return c->form == IPR_FORM_SYMMETRIC || c->form == IPR_FORM_SYMMETRIC_TRI; }
// Reading R-36: the symmetric forms in a phase below the FP64 range (FP8 / INT8 / FP16 / BF16 / TF32) take
// every product from its upper triangle -- each chain GEMM Z_j and the W GEMM run on their upper tiles, the
// Z_j are mirrored, and S_ij = 2 W_{min(i,j), max(i,j)} replaces W_ij + W_ji: each differs from the full
// product by a commutator ([A, C], [C, Z_j], [C, R]) at the phase's own rounding level there.  FP64-range
// phases keep the full products (the symmetrisation of W + W^T sets R-22's linear rate), except the tri
// form's Z_2.  IPR_TRI_W=0: off (A/B only).
// Reading R-37 (IPR_FORM_SYMMETRIC_TRIZ, p = 2): in an IPR_FP64_CRT phase Z_1 = Ahat Chat is taken from its upper
// tiles as well (2/3 of the chain's modulus GEMM work) from the third chain of the phase on, while every in-phase
// ratio rho_k / rho_{k-1} so far was <= kZtriRatio -- sticky: one slower step and the phase keeps the full Z_1
// (the mirror feeds the commutator [A, C] back into R; that only pays while the update removes it much faster).
constexpr double kZtriRatio = 0.1;
inline bool ztri_chain(const ipr_ctx *c, const PhaseC &P) {
  return c->triz && P.prec == IPR_FP64_CRT && c->z_ok && std::isfinite(c->ph_r1) && std::isfinite(c->ph_r2);
}
int wtri_phase(const ipr_ctx *c, const PhaseC &P) {
  static int on = -1;
  if (on < 0) { const char *v = getenv("IPR_TRI_W"); on = v ? atoi(v) != 0 : 1; }
  return on && is_sym(c) && !is_f64(P.prec) ? 1 : 0;
}
void *chatc_slot(ipr_ctx *c, int i, int prec) {
  return (char *)c->chatc[i] + (size_t)c->rank * (size_t)(c->npad * c->kp) * elt_size(prec);
}
ipr_status gather_bytes(ipr_ctx *c, void *base, size_t per_rank, const char *what) {
  if (c->world == 1) return IPR_OK;
  if (!c->comm->allgather((char *)base + c->rank * per_rank, base, per_rank, c->st))
    return fail(c, IPR_E_NCCL, "ncclAllGather(%s) failed: %s", what, c->comm->last_error());
  return IPR_OK;
}
// symmetric form: Chat of iterate buffer i in the correction format (if it differs from prec)
ipr_status make_corr_operand(ipr_ctx *c, int i, const PhaseC &P) {
  if (same_fmt(P.corr, P.prec)) return IPR_OK;
  const int64_t cnt = c->npad * c->kp;
  CK(launch_make_operand(cont_ptr(c, i, P), P.cont64, cnt, P.corr, nullptr, chatc_slot(c, i, P.corr), c->st));
  return gather_bytes(c, c->chatc[i], (size_t)cnt * elt_size(P.corr), "Chat corr");
}

ipr_status begin_phase(ipr_ctx *c, bool first) {
  const PhaseC &P = c->ph[c->phase];
  Nvtx nv("phase %d %s", c->phase, pname(P.prec));
  CKS(stage_a(c, P, c->Aop, c->dsig + 0));
  if (c->form != IPR_FORM_LITERAL && c->world > 1) {   // full row-major Ahat (A operand)
    CK(launch_stage_a(c->A, c->lda, c->n, c->npad, 0, c->npad, P.prec, P.cont64, P.m, P.rtz,
                      is_scaled(P.prec) ? c->dsig + 0 : nullptr, c->Afull, c->st));
  }
  // stored bits of the entering iterate; R-26: those of the digits its first chain will use
  int m_in = P.m;
  if (P.adaptive && !first) m_in = oz_adaptive_m(oz_digits_for(c->last_rho / std::sqrt((double)c->n) * 0.03 * 0.03, c->n));
  c->m_of_cur = m_in;
  c->ph_r1 = NAN; c->ph_r2 = NAN; c->z_ok = true;
  if (first) {
    CK(launch_c0(c->A, c->lda, c->n, c->mr, c->row0, c->col0, c->kp, c->norms[3], P.cont64, m_in, P.rtz,
                 cont_ptr(c, c->cur, P), c->st));
  } else {
    CKS(save_best(c));
    if (c->best_loc == 2) {
      CK(launch_f64_to_cont(c->best, blk(c), P.cont64, m_in, P.rtz, cont_ptr(c, c->cur, P), c->st));
    }
  }
  CKS(make_operand(c, c->cur, P));
  c->c_anchor = true;                // coupled form: re-anchor M = X^p A in this phase
  c->crA_b = -1; c->crC_for = -1; c->crC_b = -1;     // CRT residues: split lazily per chain
  if (P.prec == IPR_FP64_OZ) {   // digits of Ahat (A role) and of Chat (both roles; G = 1, symmetric)
    CK(launch_oz_split((const double *)c->Aop, c->npad, c->npad, c->npad, OZ_S, c->ozA, nullptr, c->ozA_sig, c->st));
    CKS(oz_split_chat(c, c->cur));
  }
  if (c->form == IPR_FORM_NEWTON_SCHULZ) CKS(make_xt(c, c->cur, P));
  if (fused_sym_ok(c, P)) {        // [Chat | . | Chat] of the entering iterate in the correction format
    const int64_t cnt = c->npad * c->npad;
    CK(launch_make_operand(cont_ptr(c, c->cur, P), P.cont64, cnt, P.corr, nullptr, qplane(c, c->cur, P.corr, 0), c->st));
    CK(launch_make_operand(cont_ptr(c, c->cur, P), P.cont64, cnt, P.corr, nullptr, qplane(c, c->cur, P.corr, 2), c->st));
  }
  if (is_sym(c)) {
    CKS(make_corr_operand(c, c->cur, P));
    if (c->world > 1) CKS(make_xt(c, c->cur, P));
  }
  return IPR_OK;
}

// Newton-Schulz form (NEXT-1): the transposed operand X^T of the local column panel (the B operand
// of T = Ahat Xhat) from the row-major local slot of Chat(i).
ipr_status make_xt(ipr_ctx *c, int i, const PhaseC &P) {
  CK(launch_transpose(chat_slot(c, i, P.prec), c->npad, c->kp, elt_size(P.prec), c->T[0], c->st));
  return IPR_OK;
}

// tri form, G > 1: GEMM 2 computed the upper-triangle tiles of this rank's columns S_g; their mirrors
// (j, i), i < j, belong to the columns S_h of the ranks owning row i and were written packed into msend
// [h][i - col0_h][j - col0_g].  One all-to-all delivers each block to its owner, which copies the
// strictly-lower elements of its columns into its K-major panel T (the same values, so every element
// is bit-identical to G = 1 -- DESIGN.md section 7).
ipr_status mirror_exchange(ipr_ctx *c, void *T, int esz) {
  Nvtx nv("tri mirror all-to-all");
  const size_t blk = (size_t)(c->kp * c->kp) * esz;
  if (!c->comm->alltoall(c->msend, c->mrecv, blk, c->st))
    return fail(c, IPR_E_NCCL, "all-to-all(tri mirror) failed: %s", c->comm->last_error());
  CK(launch_mirror_unpack(c->mrecv, esz, c->kp, c->npad, c->rank, c->world, T, c->st));
  return IPR_OK;
}

// ---- one chain: p GEMMs + fused residual; returns rho (host sync) ----
ipr_status chain(ipr_ctx *c, double *rho_out, float *ms) {
  const PhaseC &P = c->ph[c->phase];
  Nvtx nv("chain k=%zu %s", c->trace.size(), pname(P.prec));
  const int prec = P.prec;
  const void *X = c->Aop;
  const bool scaled = is_scaled(prec);
  const int *sigX = scaled ? c->dsig + 0 : nullptr;
  const int64_t tm = tiles_m(c, prec), tn_loc = c->kp / gemm_tile_n(prec);
  double *part = c->part;
  c->ktimer.used = 0;
  crt_set_timer(prec == IPR_FP64_CRT ? &c->ktimer : nullptr);
  struct TimerOff { ~TimerOff() { crt_set_timer(nullptr); } } timer_off;
  CK(cudaEventRecord(c->ev[0], c->st));
  if (c->form == IPR_FORM_NEWTON_SCHULZ) {
    // T = Ahat Xhat (A operand: full row-major Ahat; B: X^T panel), epilogue: residual partials
    // and What = qin(2I - T) stored K-major for the update GEMM
    GemmArgs g = base_args(c, prec, c->T[0]);
    g.A = c->world == 1 ? c->Aop : c->Afull;
    g.a_kp = c->npad; g.a_pstride = c->npad * c->npad;
    if (scaled) { g.sigA = c->dsig + 0; g.sigB = c->dsig + 1 + c->cur; g.pmax = c->pmax; }
    g.mode = (scaled ? EPI_TSCRATCH : EPI_STORE_T) | EPI_DIAG_MINUS | EPI_RESID;
    g.diag = 2.0;
    g.tout = scaled ? (void *)c->tscr : c->T[1];
    g.ldt = c->npad;
    g.part = part;
    CK(run_gemm(c, g));
    if (scaled) {
      CKS(gather_pmax(c, c->pmax, tn_loc * tm));
      CK(launch_reduce_max(c->pmax, tiles_n_total(c, prec) * tm, nullptr, c->dsig + 4, prec, c->st));
      CK(launch_scale_op(c->tscr, c->kp * c->npad, c->dsig + 4, prec, c->T[1], c->st));
    }
  }
  if (is_sym(c) && P.adaptive) {   // R-26: this chain's digits and the next iterate's stored bits
    const double q = (std::isfinite(c->ph_r1) && std::isfinite(c->ph_r2) && c->ph_r2 > 0.0)
                         ? std::fmin(std::fmax(c->ph_r1 / c->ph_r2, 1e-3), 1.0) : 0.03;
    c->oz_S_cur = c->trace.empty() ? OZ_S : oz_digits_for(c->last_rho / std::sqrt((double)c->n) * q * q, c->n);
    c->oz_m_next = oz_adaptive_m(c->oz_S_cur);
  }
  c->last_chain_S = is_emu(prec) ? oz_S_now(c) : 0;
  c->last_chain_ztri = ztri_chain(c, P) ? 1 : 0;
  if (is_sym(c)) {
    // Z_1 = Ahat Chat (A operand: Ahat row-major; B: Chat itself for G = 1 -- exactly symmetric --
    // else the transposed local panel), Z_j = Chat qin(Z_{j-1}); GEMM p: R = I - Z_p in the
    // correction format (K-major for the W GEMM) + residual partials.  Z_j -> T[j & 1].
    for (int j = 1; j <= c->p; ++j) {
      if (j == 2) CKS(join_gather(c));   // GEMM 1 needed only the local panel; from here on the whole Chat
      GemmArgs g = base_args(c, prec, j == 1 ? (c->world == 1 ? c->chat[c->cur] : c->T[0]) : c->T[(j - 1) & 1]);
      if (j == 1) {
        g.A = c->world == 1 ? c->Aop : c->Afull;
        g.a_kp = c->npad; g.a_pstride = c->npad * c->npad;
      } else {
        chat_view(c, c->cur, prec, &g.A, &g.a_kp, &g.a_pstride);
      }
      // scaled formats (FP16/FP8/INT8): unscale by 2^-(sigma_X + sigma_C); Z_j (j < p) goes through
      // the FP32 scratch + per-tile max so its own sigma is known before it becomes an operand
      if (scaled) { g.sigA = c->dsig + 1 + c->cur; g.sigB = sigX; }
      g.mode = (scaled && j < c->p) ? EPI_TSCRATCH : EPI_STORE_T;
      if (scaled && j < c->p) { g.pmax = c->pmax; }
      if (j == 1) {
        // IPR_CERT_PHASE, FP64 last phase (G = 1): also keep Z_1 = A C row-major -- the B operand of
        // C (C A), so the phase-product estimate of ||I - C^p A||_F costs p - 1 GEMMs instead of p
        c->zr_for = -1;
        const bool full = P.adaptive ? c->oz_S_cur == OZ_S : P.m == 52;
        // (not for a chain whose Z_1 comes from its upper tiles only, R-37: the estimate then takes its own Z_1)
        if (c->Zr && c->cert == IPR_CERT_PHASE && is_f64(prec) && full && c->phase == (int)c->ph.size() - 1 &&
            !ztri_chain(c, P)) {
          g.mode |= EPI_STORE_N; g.nout = c->Zr; g.ldn = c->npad; c->zr_for = c->cur;
        }
      }
      // R-36: below the FP64 range the symmetric forms compute every Z_j on its upper tiles and mirror them
      const bool z1tri = j < c->p && (wtri_phase(c, P) || ztri_chain(c, P));
      if (z1tri) {
        g.tri = 1;
        // tiles below the diagonal are not visited -- their partial maxima must not be stale
        if (g.mode & EPI_TSCRATCH) CK(cudaMemsetAsync(c->pmax, 0, sizeof(float) * tiles_n_total(c, prec) * tm, c->st));
      }
      // R-29: a scaled correction (= prec) takes R = I - Z_p through the FP32 scratch + per-tile max
      const bool rscr = j == c->p && is_scaled(P.corr);
      if (j == c->p) {
        g.mode |= EPI_DIAG_MINUS | EPI_RESID; g.diag = 1.0; g.tprec = P.corr;
        g.tri = c->form == IPR_FORM_SYMMETRIC_TRI || wtri_phase(c, P);   // Z_2 = C A C / R-36: upper + mirror
        if (rscr) {
          g.mode = (g.mode & ~EPI_STORE_T) | EPI_TSCRATCH; g.pmax = c->pmax;
          // tri: tiles below the diagonal are not visited -- their partial maxima must not be stale
          if (g.tri) CK(cudaMemsetAsync(c->pmax, 0, sizeof(float) * tiles_n_total(c, prec) * tm, c->st));
        }
      }
      g.tout = ((scaled && j < c->p) || rscr) ? (void *)c->tscr : c->T[j & 1];
      if (j == c->p && fused_sym_ok(c, P)) g.tout = qplane(c, c->cur, P.corr, 1);   // Rhat into [Chat | Rhat | Chat]
      g.ldt = c->npad;
      g.part = part;
      if (prec == IPR_FP64_OZ) {
        if (j == 1) {   // Ahat (A role) x Chat (B role: its rows, by symmetry)
          g.oz_a = c->ozA; g.oz_rsig = c->ozA_sig; g.oz_b = c->ozCb[c->cur]; g.oz_csig = c->ozC_sig[c->cur];
          g.ozacc = c->ozacc; g.ldoz = c->npad; g.oz_S = oz_S_now(c);
        } else {
          CKS(oz_operands(c, g, c->cur, c->T[(j - 1) & 1]));
        }
      } else if (prec == IPR_FP64_CRT) {
        if (j == 1 && c->world > 1) {   // Ahat (A role) x the transposed local panel of Chat (B role)
          CKS(crt_operands(c, g, -1, c->T[0]));
        } else if (j == 1) {   // Ahat (A role) x Chat (B role: its rows, by symmetry)
          const int b = crt_bits_now(c);
          CKS(crt_ensure_a(c, b));
          CKS(crt_ensure_c(c, c->cur, b));
          g.oz_a = c->crA; g.oz_rsig = c->crA_sig; g.oz_b = c->crC; g.oz_csig = c->crC_sig;
          crt_args(c, g, b);
        } else {
          CKS(crt_operands(c, g, c->cur, c->T[(j - 1) & 1]));
        }
      }
      const bool mx = (j == c->p || z1tri) && g.tri && c->world > 1;   // tri, G > 1: mirror tiles cross panels
      if (mx) { g.mout = c->msend; g.ldm = c->kp; }
      CK(run_gemm(c, g));
      if (mx) CKS(mirror_exchange(c, g.tout, (rscr || (scaled && j < c->p)) ? 4 : elt_size(g.tprec)));
      if (rscr) {   // sigma_R -> dsig[3 + (p & 1)] (not the slot GEMM p read), Rhat -> T[p & 1]
        CKS(gather_pmax(c, c->pmax, tn_loc * tm));
        CK(launch_reduce_max(c->pmax, tiles_n_total(c, prec) * tm, nullptr, c->dsig + 3 + (j & 1), prec, c->st));
        CK(launch_scale_op(c->tscr, c->kp * c->npad, c->dsig + 3 + (j & 1), prec, c->T[j & 1], c->st));
      }
      if (scaled && j < c->p) {
        CKS(gather_pmax(c, c->pmax, tn_loc * tm));
        CK(launch_reduce_max(c->pmax, tiles_n_total(c, prec) * tm, nullptr, c->dsig + 3 + (j & 1), prec, c->st));
        CK(launch_scale_op(c->tscr, c->kp * c->npad, c->dsig + 3 + (j & 1), prec, c->T[j & 1], c->st));
        sigX = c->dsig + 3 + (j & 1);
      }
    }
  }
  const bool coupled_cached = c->form == IPR_FORM_COUPLED && !c->c_anchor;   // rho from the last step
  if (c->form == IPR_FORM_COUPLED && c->c_anchor) {
    // anchor: the literal chain T_j = Xhat qin(T_{j-1}) (T_0 = Ahat); the last GEMM stores
    // Mhat = qin(q_m(T_p)) and Nhat = qin(((p+1)I - q_m(T_p))/p) K-major + residual partials
    const void *Xb = c->Aop;
    for (int j = 1; j <= c->p; ++j) {
      GemmArgs g = base_args(c, prec, Xb);
      chat_view(c, c->cur, prec, &g.A, &g.a_kp, &g.a_pstride);
      g.ldt = c->npad; g.part = part;
      if (j < c->p) { g.mode = EPI_STORE_T; g.tout = c->T[j & 1]; }
      else {
        g.mode = EPI_COUPLED | EPI_RESID; g.tout = c->cM[c->cmi]; g.nkout = c->cNk[c->cmi];
        g.m = P.m; g.rtz = P.rtz; g.cont64 = P.cont64;
      }
      CK(run_gemm(c, g));
      Xb = c->T[j & 1];
    }
    CKS(coupled_gather_n(c));
    c->c_anchor = false;
  }
  for (int j = 1; c->form == IPR_FORM_LITERAL && j <= c->p; ++j) {
    GemmArgs g = base_args(c, prec, X);
    chat_view(c, c->cur, prec, &g.A, &g.a_kp, &g.a_pstride);
    if (j > 1 && c->grows > 1) {   // 2-D grid: B = the gathered T_{j-1} column panel [grows][kp][mr]
      g.ldb = c->mr; g.b_kp = c->mr; g.b_pstride = c->kp * c->mr;
    }
    if (scaled) { g.sigA = c->dsig + 1 + c->cur; g.sigB = sigX; }
    g.mode = (scaled ? EPI_TSCRATCH : EPI_STORE_T) | (j == c->p ? EPI_RESID : 0);
    g.tout = scaled ? (void *)c->tscr : c->T[j & 1];
    // the rank's output block is rows [row0, row0 + mr): K-major [kp][mr]; epilogues index global rows
    g.ldt = c->mr;
    g.tout = (char *)g.tout - c->row0 * elt_size(scaled ? IPR_TF32 : g.tprec);
    g.part = part;
    if (scaled) g.pmax = c->pmax;
    CK(run_gemm(c, g));
    if (c->grows > 1) {            // 2-D grid: the T_j column panel along the grid column (SUMMA-like)
      if (!c->colt->allgather(c->T[j & 1], c->Tcol, (size_t)blk(c) * elt_size(g.tprec), c->st))
        return fail(c, IPR_E_NCCL, "all-gather(T column panel) failed: %s", c->colt->last_error());
    }
    if (scaled) {
      CKS(gather_pmax(c, c->pmax, tn_loc * tm));
      CK(launch_reduce_max(c->pmax, tiles_n_total(c, prec) * tm, nullptr, c->dsig + 3 + (j & 1), prec, c->st));
      CK(launch_scale_op(c->tscr, c->kp * c->npad, c->dsig + 3 + (j & 1), prec, c->T[j & 1], c->st));
      sigX = c->dsig + 3 + (j & 1);
    }
    X = c->grows > 1 ? c->Tcol : c->T[j & 1];
  }
  CK(cudaEventRecord(c->ev[1], c->st));
  if (!coupled_cached) {
    CKS(gather_partials(c, part, tn_loc * tm, (int)gemm_tile_m(prec), (int)gemm_tile_n(prec)));
    CK(launch_reduce_sum(part, tiles_n_total(c, prec) * tm, c->dscal + 0, c->st));
  }
  CK(cudaEventRecord(c->ev[4], c->st));      // the GPU has the chain's residual: the decision's bubble starts
  CK(cudaMemcpyAsync(c->hscal, c->dscal, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  // only what the decision needs before the next enqueue: the chain's own timers (ev[0], ev[1], the CRT
  // kernel pairs) are read by chain_timers() after the update is on the stream -- every host microsecond
  // between this sync and the update's first launch is a GPU bubble (r02: ~28 per solve)
  float tu = 0.f, tg = 0.f;
  if (c->upd_timed) {
    CK(cudaEventElapsedTime(&tu, c->ev[2], c->ev[3]));
    CK(cudaEventElapsedTime(&tg, c->ev[5], c->ev[2]));   // device idle from the last chain's end to the update
    c->upd_timed = false;
  }
  if (c->pending_delta >= 0) {
    c->trace[c->pending_delta].delta = std::sqrt(c->hscal[1]);
    c->trace[c->pending_delta].gemm_ms += tu;
    c->trace[c->pending_delta].upd_ms = tu;
    c->trace[c->pending_delta].gap_ms = tg;
    c->pending_delta = -1;
  }
  // keep this chain's "results ready" timestamp for the gap to its update (ev[4] is re-recorded per chain)
  std::swap(c->ev[4], c->ev[5]);
  *rho_out = std::sqrt(c->hscal[0]);
  *ms = 0.f;
  return IPR_OK;
}

// the last chain's device times (its events are not re-recorded before the next chain)
ipr_status chain_timers(ipr_ctx *c, ipr_record &r) {
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, c->ev[0], c->ev[1]));
  double km = 0.0;
  for (int i = 0; i < c->ktimer.used; ++i) {
    float tk = 0.f;
    CK(cudaEventElapsedTime(&tk, c->kev[2 * i], c->kev[2 * i + 1]));
    km += tk;
  }
  r.gemm_ms += t;
  if (r.prec == IPR_FP64_CRT) r.kern_ms = km;
  return IPR_OK;
}

// ---- GEMM p+1 with the fused update (a6) ----
ipr_status update(ipr_ctx *c) {
  const PhaseC &P = c->ph[c->phase];
  Nvtx nv("update %s", pname(P.prec));
  const int prec = P.prec, nx = 1 - c->cur;
  // the update overwrites buffer nx: keep the best iterate if it lives there
  if (c->best_loc == nx) CKS(save_best(c));
  const int64_t tm = tiles_m(c, prec), tn_loc = c->kp / gemm_tile_n(prec);
  const bool ns = c->form == IPR_FORM_NEWTON_SCHULZ;
  // literal: P = Chat qin(T_p); Newton-Schulz: X_{k+1} = Xhat What (What in T[1])
  const int tb = ns ? 1 : (c->p & 1);
  GemmArgs g = base_args(c, prec, c->grows > 1 ? c->Tcol : c->T[tb]);
  chat_view(c, c->cur, prec, &g.A, &g.a_kp, &g.a_pstride);
  if (c->grows > 1) { g.ldb = c->mr; g.b_kp = c->mr; g.b_pstride = c->kp * c->mr; }
  if (is_scaled(prec)) { g.sigA = c->dsig + 1 + c->cur; g.sigB = c->dsig + 3 + tb; g.pmax = c->pmax; }
  g.mode = ns ? EPI_NSUPDATE : EPI_UPDATE;
  // the rank's block rows [row0, row0 + mr) (global-row epilogue: pointers offset by -row0 rows)
  const size_t cb = P.cont64 ? 8 : 4;
  g.cold = (char *)cont_ptr(c, c->cur, P) - (size_t)c->row0 * c->kp * cb;
  g.cnew = (char *)cont_ptr(c, nx, P) - (size_t)c->row0 * c->kp * cb;
  g.ldc = c->kp;
  g.chat_new = is_f64(prec) ? nullptr : (char *)chat_slot(c, nx, prec) - (size_t)c->row0 * c->kp * elt_size(prec);
  g.ldh = c->kp;
  g.m = P.m; g.rtz = P.rtz; g.cont64 = P.cont64;
  g.part = c->part;
  CK(cudaEventRecord(c->ev[2], c->st));
  CK(run_gemm(c, g));
  CK(cudaEventRecord(c->ev[3], c->st));
  c->upd_timed = true;
  CKS(gather_partials(c, c->part, tn_loc * tm, (int)gemm_tile_m(prec), (int)gemm_tile_n(prec)));
  CK(launch_reduce_sum(c->part, tiles_n_total(c, prec) * tm, c->dscal + 1, c->st));
  if (is_scaled(prec)) {
    CKS(gather_pmax(c, c->pmax, tn_loc * tm));
    CK(launch_reduce_max(c->pmax, tiles_n_total(c, prec) * tm, nullptr, c->dsig + 1 + nx, prec, c->st));
    CK(launch_make_operand(c->cont[nx], 0, blk(c), prec, c->dsig + 1 + nx, chat_slot(c, nx, prec), c->st));
  }
  CKS(gather_chat(c, nx, prec));
  if (ns) CKS(make_xt(c, nx, P));
  c->cur = nx;
  return IPR_OK;
}

// ---- symmetric form (NEXT-2): W = qc(C) Rhat, then C_{k+1} = q_m(C + (W + W^T)/(2p)) ----
ipr_status update_sym(ipr_ctx *c) {
  const PhaseC &P = c->ph[c->phase];
  Nvtx nv("update sym corr=%s", pname(P.corr));
  const int nx = 1 - c->cur;
  if (c->best_loc == nx) CKS(save_best(c));
  if (fused_sym_ok(c, P)) {
    // S = Chat Rhat + Rhat Chat = W + W^T as ONE upper-triangle GEMM over K = 2n ([Chat | Rhat] x
    // [Rhat ; Chat], both symmetric), the update C_{k+1} = q_m(C + S/(2p)) and the next operands fused
    // into its epilogue (no W round trip, no k_sym_update pass)
    const int64_t np = c->npad;
    GemmArgs g = base_args(c, P.corr, qplane(c, c->cur, P.corr, 1));
    g.A = qplane(c, c->cur, P.corr, 0); g.a_kp = np; g.a_pstride = np * np;
    g.K = 2 * np; g.ldb = np; g.b_pstride = np * np;
    g.mode = EPI_SYMUPD; g.tri = 1; g.tprec = P.corr;
    g.cold = cont_ptr(c, c->cur, P); g.cnew = cont_ptr(c, nx, P); g.ldc = c->kp;
    g.chat_new = (is_f64(P.prec) || is_scaled(P.prec)) ? nullptr : chat_slot(c, nx, P.prec);
    g.hprec = P.prec;
    g.qnext = c->qbuf[nx]; g.ldh = np;
    g.m = P.adaptive ? c->oz_m_next : P.m; g.rtz = P.rtz; g.cont64 = P.cont64;
    g.part = c->part;
    CK(cudaEventRecord(c->ev[2], c->st));
    CK(run_gemm(c, g));
    CK(launch_reduce_sum(c->part, tiles_n_total(c, P.corr) * tiles_m(c, P.corr), c->dscal + 1, c->st));
    CK(cudaEventRecord(c->ev[3], c->st));
    c->upd_timed = true;
    if (P.prec == IPR_FP64_OZ) CKS(oz_split_chat(c, nx));
    if (c->crC_for == nx) c->crC_for = -1;
    c->m_of_cur = P.adaptive ? c->oz_m_next : P.m;
    c->cur = nx;
    return IPR_OK;
  }
  GemmArgs g = base_args(c, P.corr, c->T[c->p & 1]);
  if (same_fmt(P.corr, P.prec)) chat_view(c, c->cur, P.prec, &g.A, &g.a_kp, &g.a_pstride);
  else { g.A = c->chatc[c->cur]; g.a_kp = c->kp; g.a_pstride = c->npad * c->kp; }
  if (is_scaled(P.corr)) { g.sigA = c->dsig + 1 + c->cur; g.sigB = c->dsig + 3 + (c->p & 1); }   // R-29
  // W holds the exact accumulator values: FP64 for an FP64 (DMMA) correction, else FP32
  const int wb = P.corr == IPR_FP64 ? 8 : 4;
  // reading R-36: the tri form below the FP64 range computes only W's upper tiles (S = 2 W_{min, max})
  const int wtri = wtri_phase(c, P);
  g.tri = wtri;
  g.mode = EPI_WSTORE;
  g.w64 = wb == 8;
  g.wout = (char *)c->wbuf + (size_t)c->rank * (size_t)(c->npad * c->kp) * wb;
  g.ldw = c->kp;
  CK(cudaEventRecord(c->ev[2], c->st));
  CK(run_gemm(c, g));
  CKS(gather_bytes(c, c->wbuf, (size_t)(c->npad * c->kp) * wb, "W"));
  // scaled phases: the update also takes max |C_{k+1}| (this rank's slot of pmax) for the next sigma
  unsigned *amax = is_scaled(P.prec) ? (unsigned *)(c->pmax + c->rank) : nullptr;
  if (amax) CK(cudaMemsetAsync(amax, 0, sizeof(unsigned), c->st));
  CK(launch_sym_update(cont_ptr(c, c->cur, P), P.cont64, cont_ptr(c, nx, P), c->wbuf, wb == 8, c->npad,
                       c->kp, c->col0, c->p, P.adaptive ? c->oz_m_next : P.m, P.rtz, P.prec,
                       (is_f64(P.prec) || is_scaled(P.prec)) ? nullptr : chat_slot(c, nx, P.prec), P.corr,
                       same_fmt(P.corr, P.prec) ? nullptr : chatc_slot(c, nx, P.corr), c->part, amax, wtri, c->st));
  CK(cudaEventRecord(c->ev[3], c->st));
  c->upd_timed = true;
  const int64_t t64 = c->npad / 64;
  CKS(gather_partials(c, c->part, (c->kp / 64) * t64));
  CK(launch_reduce_sum(c->part, t64 * t64, c->dscal + 1, c->st));
  if (is_scaled(P.prec)) CKS(make_operand(c, nx, P, true, true));   // sigma from the update's max|C_{k+1}|
  else CKS(gather_bytes_async(c, c->chat[nx], (size_t)(c->npad * c->kp) * elt_size(P.prec), "Chat"));
  if (P.prec == IPR_FP64_OZ) CKS(oz_split_chat(c, nx));
  if (c->crC_for == nx) c->crC_for = -1;
  c->m_of_cur = P.adaptive ? c->oz_m_next : P.m;
  if (!same_fmt(P.corr, P.prec))
    CKS(gather_bytes_async(c, c->chatc[nx], (size_t)(c->npad * c->kp) * elt_size(P.corr), "Chat corr"));
  if (c->world > 1) CKS(make_xt(c, nx, P));
  c->cur = nx;
  return IPR_OK;
}

// ---- coupled form (NEXT-2 (ii), R-27) ----
// the current K-major Nhat panel -> row-major column panel (slot rank of cNf), all-gathered: the
// replicated A operand of the M chain
ipr_status coupled_gather_n(ipr_ctx *c) {
  const PhaseC &P = c->ph[c->phase];
  const size_t esz = elt_size(P.prec), slot = (size_t)(c->npad * c->kp) * esz;
  CK(launch_transpose(c->cNk[c->cmi], c->kp, c->npad, (int)esz, (char *)c->cNf + c->rank * slot, c->st));
  return gather_bytes(c, c->cNf, slot, "Nhat");
}

// X_{k+1} = q_m(Xhat Nhat) (+ Xhat_{k+1}, delta partials); T_1 = Nhat Mhat, T_j = Nhat qin(T_{j-1});
// the last GEMM stores the next Mhat / Nhat and the residual partials of M_{k+1}
ipr_status update_coupled(ipr_ctx *c) {
  const PhaseC &P = c->ph[c->phase];
  const int prec = P.prec, nx = 1 - c->cur;
  if (c->best_loc == nx) CKS(save_best(c));
  const int64_t tm = tiles_m(c, prec), tn_loc = c->kp / gemm_tile_n(prec);
  CK(cudaEventRecord(c->ev[2], c->st));
  GemmArgs g = base_args(c, prec, c->cNk[c->cmi]);
  chat_view(c, c->cur, prec, &g.A, &g.a_kp, &g.a_pstride);
  g.mode = EPI_NSUPDATE;
  g.cold = cont_ptr(c, c->cur, P); g.cnew = cont_ptr(c, nx, P); g.ldc = c->kp;
  g.chat_new = is_f64(prec) ? nullptr : chat_slot(c, nx, prec); g.ldh = c->kp;
  g.m = P.m; g.rtz = P.rtz; g.cont64 = P.cont64;
  g.part = c->part;
  CK(run_gemm(c, g));
  CKS(gather_partials(c, c->part, tn_loc * tm));
  CK(launch_reduce_sum(c->part, tiles_n_total(c, prec) * tm, c->dscal + 1, c->st));
  const void *Xb = c->cM[c->cmi];
  for (int j = 1; j <= c->p; ++j) {
    GemmArgs q = base_args(c, prec, Xb);
    q.A = c->cNf; q.a_kp = c->kp; q.a_pstride = c->npad * c->kp;
    q.ldt = c->npad; q.part = c->part;
    if (j < c->p) { q.mode = EPI_STORE_T; q.tout = c->T[j & 1]; }
    else {
      q.mode = EPI_COUPLED | EPI_RESID; q.tout = c->cM[1 - c->cmi]; q.nkout = c->cNk[1 - c->cmi];
      q.m = P.m; q.rtz = P.rtz; q.cont64 = P.cont64;
    }
    CK(run_gemm(c, q));
    Xb = c->T[j & 1];
  }
  CKS(gather_partials(c, c->part, tn_loc * tm));
  CK(launch_reduce_sum(c->part, tiles_n_total(c, prec) * tm, c->dscal + 0, c->st));
  c->cmi ^= 1;
  CKS(gather_chat(c, nx, prec));
  CKS(coupled_gather_n(c));
  CK(cudaEventRecord(c->ev[3], c->st));
  c->upd_timed = true;
  c->m_of_cur = P.m;
  c->cur = nx;
  return IPR_OK;
}

ipr_status step_update(ipr_ctx *c) {
  return is_sym(c) ? update_sym(c) : c->form == IPR_FORM_COUPLED ? update_coupled(c) : update(c);
}

// Controller, reading R-5 (independent implementation of the rules in DESIGN.md).
int decide(ipr_ctx *c, double rho, bool *best_new) {
  const PhaseC &P = c->ph[c->phase];
  const bool last = c->phase == (int)c->ph.size() - 1;
  const double rhohat = rho / std::sqrt((double)c->n);
  const bool fin = std::isfinite(rho);
  *best_new = fin && rho < c->rho_best;
  if (*best_new) c->rho_best = rho;
  int d;
  if (!fin) d = last ? IPR_DEC_NONFINITE : IPR_DEC_SWITCH;
  else if (last && rho <= c->final_tol) d = IPR_DEC_CONVERGED;
  else if (rhohat > 10.0 * c->rhohat_min && rhohat > 1.0) d = last ? IPR_DEC_DIVERGED : IPR_DEC_SWITCH;
  else if (!last && P.switch_tol > 0.0 && rho <= P.switch_tol) d = IPR_DEC_SWITCH;
  else if (!last && P.plateau_ratio > 0.0 && rhohat < P.plateau_arm && std::isfinite(c->rho_prev) &&
           rho > P.plateau_ratio * c->rho_prev)
    d = IPR_DEC_SWITCH;
  else if (P.max_iters > 0 && c->it_in_phase + 1 >= P.max_iters) d = last ? IPR_DEC_ITER_LIMIT : IPR_DEC_SWITCH;
  else d = IPR_DEC_CONTINUE;
  if (fin && rhohat < c->rhohat_min) c->rhohat_min = rhohat;
  c->rho_prev = rho;
  c->it_in_phase += 1;
  return d;
}

void free_ctx(ipr_ctx *c) {
  if (!c) return;
  if (c->arena) cudaFreeAsync(c->arena, c->st);   // back to the library's retained pool
  if (c->aux) cudaFreeAsync(c->aux, c->st);
  if (c->hscal) pinned_release(c->hscal);
  if (c->hcert) pinned_release(c->hcert);
  for (auto &e : c->ev) if (e) cudaEventDestroy(e);
  for (auto &e : c->kev) if (e) cudaEventDestroy(e);
  if (c->cst) { cudaStreamSynchronize(c->cst); cudaStreamDestroy(c->cst); }
  if (c->ost) { cudaStreamSynchronize(c->ost); cudaStreamDestroy(c->ost); }
  if (c->oev) cudaEventDestroy(c->oev);
  if (c->orev) cudaEventDestroy(c->orev);
  if (c->Aown) cudaFreeAsync(c->Aown, c->st);
  for (auto &e : c->gev) if (e) cudaEventDestroy(e);
  delete c->rowt;
  delete c->colt;
  delete c->comm;
  delete c;
}

// All O(n^2) buffers in one arena, sized once the schedule and the form are known (first
// ipr_iterate): one cudaMalloc / cudaFree per solve, and an OOM is reported before any work.
// test-only guard bands behind every arena buffer (compute-sanitizer is closed on the pool):
// ipr_test_set_guards(1) before ipr_iterate, ipr_test_check_guards after
constexpr size_t kGuard = 4096;
constexpr unsigned char kGuardByte = 0xA5;
int g_guards = 0;

ipr_status alloc_arena(ipr_ctx *c, bool need_corr) {
  const size_t full = (size_t)(c->npad * c->npad), panel = (size_t)(c->npad * c->kp);
  const bool cpl = c->form == IPR_FORM_COUPLED;
  bool fp16 = false, oz = false, cr = false;   // any scaled-format phase: FP32 T scratch; Ozaki I / II
  for (auto &P : c->ph) { fp16 |= is_scaled(P.prec); oz |= P.prec == IPR_FP64_OZ; cr |= P.prec == IPR_FP64_CRT; }
  const size_t crp = cr ? full * CRT_MAX : 0, crs = cr ? (size_t)c->npad * 4 : 0;
  bool fq = false;                      // any phase with the fused symmetric update: [Chat | Rhat | Chat] x 2
  for (auto &P : c->ph) fq |= fused_sym_ok(c, P);
  const size_t qb = fq ? 3 * full * 4 : 0;
  size_t cesz = 2;                      // correction-format copies of Chat: BF16 2 B, TF32 4 B
  for (auto &P : c->ph) if (!same_fmt(P.corr, P.prec) && elt_size(P.corr) > (int)cesz) cesz = elt_size(P.corr);
  struct Slot { void **p; size_t bytes; };
  const Slot slots[] = {
      {&c->chat[0], full * 8}, {&c->chat[1], full * 8}, {&c->cont[0], panel * 4}, {&c->cont[1], panel * 4},
      {(void **)&c->best, panel * 8}, {&c->T[0], panel * 8}, {&c->T[1], panel * 8}, {&c->Aop, panel * 8},
      {(void **)&c->part, (size_t)c->npart * 8}, {(void **)&c->pmax, (size_t)c->npart * 4},
      {(void **)&c->tscr, fp16 ? panel * 4 : 0},
      {&c->Afull, (c->world > 1 && c->form != IPR_FORM_LITERAL) ? full * 8 : 0},
      {&c->chatc[0], need_corr ? full * cesz : 0}, {&c->chatc[1], need_corr ? full * cesz : 0},
      {&c->wbuf, is_sym(c) ? full * c->wbytes : 0},
      {&c->Zr, (is_sym(c) && c->world == 1) ? panel * 8 : 0},
      {(void **)&c->ozA, oz ? full * OZ_S : 0}, {(void **)&c->ozC[0], oz ? full * OZ_S : 0},
      {(void **)&c->ozC[1], oz ? full * OZ_S : 0}, {(void **)&c->ozCb[0], oz ? full * OZ_S : 0},
      {(void **)&c->ozCb[1], oz ? full * OZ_S : 0}, {(void **)&c->ozB, oz ? full * OZ_S : 0},
      {(void **)&c->ozA_sig, oz ? (size_t)c->npad * 4 : 0}, {(void **)&c->ozC_sig[0], oz ? (size_t)c->npad * 4 : 0},
      {(void **)&c->ozC_sig[1], oz ? (size_t)c->npad * 4 : 0}, {(void **)&c->ozB_sig, oz ? (size_t)c->npad * 4 : 0},
      {(void **)&c->ozacc, oz ? full * 8 : 0},
      {(void **)&c->crA, crp}, {(void **)&c->crC, crp}, {(void **)&c->crB, crp},
      {(void **)&c->crA_sig, crs}, {(void **)&c->crC_sig, crs},
      {(void **)&c->crB_sig, crs}, {(void **)&c->crV, cr ? full * CRT_MAX : 0},
      {&c->qbuf[0], qb}, {&c->qbuf[1], qb},
      {&c->cM[0], cpl ? panel * 8 : 0}, {&c->cM[1], cpl ? panel * 8 : 0}, {&c->cNk[0], cpl ? panel * 8 : 0},
      {&c->cNk[1], cpl ? panel * 8 : 0}, {&c->cNf, cpl ? full * 8 : 0},
      // CRT arenas: the certify / copy-out scratch lives in the B-residue and v-byte scratch (dead
      // outside a CRT product; every product re-splits its B operand)
      {(void **)&c->full64, cr ? 0 : full * 8}, {&c->Acert, cr ? 0 : panel * 8},
      {&c->chat_rm, (cr && c->world > 1) ? full * 8 : 0},
      {&c->Tcol, c->grows > 1 ? panel * 8 : 0},
      {(void **)&c->certv, (cr && is_sym(c)) ? (size_t)c->npad * 12 * 8 : 0},
      {(void **)&c->partg, c->grows > 1 ? (size_t)c->world * c->npart * 8 : 0},
      {&c->msend, (c->world > 1 && is_sym(c)) ? panel * 8 : 0},     // tri mirror exchange (R-36: every sym form)
      {&c->mrecv, (c->world > 1 && is_sym(c)) ? panel * 8 : 0}};
  const size_t gb = g_guards ? kGuard : 0;
  size_t total = 0;
  for (const Slot &q : slots) total += (q.bytes + 255) / 256 * 256 + (q.bytes ? gb : 0);
  // stream-ordered allocation from a library-owned pool that retains its memory, so back-to-back
  // solves reuse the arena without driver (un)mapping: one context = one cudaMallocFromPoolAsync
  cudaMemPool_t pool = arena_pool();
  if (!pool) return fail(c, IPR_E_CUDA, "cudaMemPoolCreate failed");
  char *base = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync((void **)&base, total, pool, c->st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, IPR_E_OOM, "arena of %zu bytes: %s", total, cudaGetErrorString(e));
  }
  c->arena = base;
  size_t off = 0;
  c->guards.clear();
  for (const Slot &q : slots) {
    *q.p = q.bytes ? base + off : nullptr;
    off += (q.bytes + 255) / 256 * 256;
    if (q.bytes && gb) {
      c->guards.push_back(off);
      CK(cudaMemsetAsync(base + off, kGuardByte, gb, c->st));
      off += gb;
    }
  }
  if (cr) { c->full64 = (double *)c->crB; c->Acert = c->crV; }   // 8 B x npad^2 <= 18 B x npad^2
  CK(cudaMemsetAsync(c->chat[0], 0, full * 8, c->st));
  CK(cudaMemsetAsync(c->chat[1], 0, full * 8, c->st));
  if (c->chat_rm) CK(cudaMemsetAsync(c->chat_rm, 0, full * 8, c->st));   // padding rows / columns stay 0
  return IPR_OK;
}

// FP64 full matrix (panel-major [G][npad][kp]) of a local FP64 panel -> full64
ipr_status gather_f64(ipr_ctx *c, const double *local) {
  // block-major [world][mr][kp] (1 x G: panel-major [G][npad][kp])
  double *slot = c->full64 + (size_t)c->rank * blk(c);
  if (local != slot) CK(cudaMemcpyAsync(slot, local, (size_t)blk(c) * 8, cudaMemcpyDeviceToDevice, c->st));
  if (c->world > 1 && !c->comm->allgather(slot, c->full64, (size_t)blk(c) * 8, c->st))
    return fail(c, IPR_E_NCCL, "ncclAllGather(C) failed: %s", c->comm->last_error());
  return IPR_OK;
}

}  // namespace

// =========================================================================================
// C-ABI
// =========================================================================================
extern "C" {

static ipr_status certify_best(ipr_ctx *c, double *rho);
static ipr_status certify_iter(ipr_ctx *c, int i, double *rho);
static ipr_status certify_from_zr(ipr_ctx *c, int i, double *rho);
static ipr_status stream_candidate(ipr_ctx *c, int i);

const char *ipr_version(void) {
  return "ipr 0.4.0 (sm_100a: tcgen05 BF16/FP16/TF32/FP8/INT8, DMMA FP64, FP64 on INT8 tensor cores: Ozaki I / II-CRT; CRT certificate)";
}

const char *ipr_last_error(const ipr_ctx *c) { return c ? c->err.c_str() : t_err.c_str(); }

ipr_status ipr_nccl_unique_id(void *out128) {
  ipr_ctx *c = nullptr;
  if (!out128) return fail(c, IPR_E_INVALID_ARG, "ipr_nccl_unique_id: null output");
  std::string e;
  if (!NcclComm::unique_id(out128, &e)) return fail(c, IPR_E_NCCL, "%s", e.c_str());
  return IPR_OK;
}

// ipr_init / ipr_test_init_local: lg == nullptr -> NCCL from nccl_unique_id (world > 1)
static ipr_status init_ctx(ipr_ctx **out, int64_t n, const double *A_dev, int64_t lda, void *cuda_stream, int world,
                           int rank, const void *nccl_unique_id, LocalGroup *lg, int grid_rows, int grid_cols) {
  ipr_ctx *c = nullptr;
  if (!out || !A_dev) return fail(c, IPR_E_INVALID_ARG, "ipr_init: null pointer");
  *out = nullptr;
  if (n <= 0 || lda < n) return fail(c, IPR_E_INVALID_ARG, "ipr_init: need n > 0 and lda >= n (n=%lld lda=%lld)",
                                     (long long)n, (long long)lda);
  if (n > 65535) return fail(c, IPR_E_UNSUPPORTED, "ipr_init: n > 65535 not supported");
  if (world < 1 || rank < 0 || rank >= world) return fail(c, IPR_E_INVALID_ARG, "ipr_init: bad world/rank");
  if (grid_rows < 1 || grid_cols < 1 || grid_rows * grid_cols != world)
    return fail(c, IPR_E_INVALID_ARG, "ipr_init: grid_rows x grid_cols must equal world (%d x %d vs %d)", grid_rows,
                grid_cols, world);
  if (world > 1 && !nccl_unique_id && !lg) return fail(c, IPR_E_INVALID_ARG, "ipr_init: world > 1 needs an NCCL id");
  c = new ipr_ctx();
  c->n = n; c->lda = lda; c->A = A_dev; c->world = world; c->rank = rank;
  c->st = (cudaStream_t)cuda_stream;
  const bool a_host = is_host_ptr(A_dev);
  c->tl_on = getenv("IPR_TIMELINE") != nullptr;
  tl_mark(c, "init");
  c->npad = padded_order(n, world);          // a multiple of 256 grid_rows and of 256 grid_cols
  c->grows = grid_rows; c->gcols = grid_cols;
  c->grow = rank / grid_cols; c->gcol = rank % grid_cols;
  c->mr = c->npad / grid_rows; c->kp = c->npad / grid_cols;
  c->row0 = (int64_t)c->grow * c->mr;
  c->col0 = (int64_t)c->gcol * c->kp;
  ipr_status s;
#define TRY(x) do { s = (x); if (s != IPR_OK) { std::string m = c->err; free_ctx(c); t_err = m; return s; } } while (0)
#define TRYC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { TRY(fail(c, IPR_E_CUDA, "%s: %s", #x, cudaGetErrorString(_e))); } } while (0)
  // validate the stream / device early
  {
    cudaError_t q = cudaStreamQuery(c->st);
    if (q != cudaSuccess && q != cudaErrorNotReady) TRYC(q);
  }
  // small device buffers: one stream-ordered block from the retained pool (no synchronous
  // cudaMalloc / cudaFree on the solve path); 8 pinned doubles from a process-wide slab
  {
    cudaMemPool_t pool = arena_pool();
    if (!pool) TRY(fail(c, IPR_E_CUDA, "cudaMemPoolCreate failed"));
    const size_t cs = ((size_t)n * 8 + 255) / 256 * 256;
    char *b = nullptr;
    TRYC(cudaMallocFromPoolAsync((void **)&b, 256 * 3 + cs, pool, c->st));
    c->aux = b;
    c->dflag = (int *)b; c->dscal = (double *)(b + 256); c->dsig = (int *)(b + 512);
    c->colsum = (double *)(b + 768);
    c->hscal = pinned_acquire();
    if (!c->hscal) TRY(fail(c, IPR_E_OOM, "pinned host slab exhausted (too many live contexts)"));
    if (a_host) {   // host A (pinned: full link speed; pageable: staged by the runtime) -> compact device copy
      if (cudaMallocFromPoolAsync((void **)&c->Aown, (size_t)n * n * 8, pool, c->st) != cudaSuccess) {
        cudaGetLastError();
        c->Aown = nullptr;
        TRY(fail(c, IPR_E_OOM, "ipr_init: device copy of the host A (%lld x %lld)", (long long)n, (long long)n));
      }
      TRYC(cudaMemcpy2DAsync(c->Aown, (size_t)n * 8, A_dev, (size_t)lda * 8, (size_t)n * 8, (size_t)n,
                             cudaMemcpyHostToDevice, c->st));
      c->A = c->Aown; c->lda = n;
    }
  }
  A_dev = c->A; lda = c->lda;
  for (auto &e : c->ev) TRYC(cudaEventCreate(&e));
  for (auto &e : c->kev) TRYC(cudaEventCreate(&e));
  TRYC(cudaMemsetAsync(c->dflag, 0, 16, c->st));
  TRYC(cudaMemsetAsync(c->dsig, 0, 32, c->st));
  TRYC(launch_symcheck(A_dev, lda, n, c->dflag, c->st));
  TRYC(launch_norms(A_dev, lda, n, c->colsum, c->dscal, c->st));
  int flag = 0;
  TRYC(cudaMemcpyAsync(&flag, c->dflag, 4, cudaMemcpyDeviceToHost, c->st));
  TRYC(cudaMemcpyAsync(c->norms, c->dscal, 3 * 8, cudaMemcpyDeviceToHost, c->st));
  TRYC(cudaStreamSynchronize(c->st));
  if (flag) TRY(fail(c, IPR_E_NOT_SYMMETRIC, "ipr_init: A is not exactly symmetric (A[i][j] != A[j][i] bitwise)"));
  c->norms[3] = c->norms[0] * c->norms[1];   // s of Eq. (3)
  if (!(c->norms[3] > 0.0) || !std::isfinite(c->norms[3]))
    TRY(fail(c, IPR_E_INVALID_ARG, "ipr_init: ||A||_1 ||A||_inf = %g (zero or non-finite A)", c->norms[3]));
  // O(n^2) buffers (sized for the widest, FP64, phase): one arena at the first ipr_iterate
  c->npart = (c->npad / 64) * (c->npad / 64) + 1024;    // one slot per 64 x 64 tile (k_sym_update)
  if (world > 1) {
    std::string e;
    if (lg) {
      c->comm = local_transport(lg, rank, &e);
      if (!c->comm) TRY(fail(c, IPR_E_INVALID_ARG, "%s", e.c_str()));
    } else {
      NcclComm *nc = new NcclComm();
      c->comm = nc;
      if (!nc->init(world, rank, nccl_unique_id, &e)) TRY(fail(c, IPR_E_NCCL, "%s", e.c_str()));
    }
    if (grid_rows > 1) {   // 2-D grid: the rank's grid row (Chat panels) and grid column (T panels)
      c->rowt = c->comm->split(c->grow, c->gcol, &e);
      if (!c->rowt) TRY(fail(c, IPR_E_NCCL, "grid row split: %s", e.c_str()));
      c->colt = c->comm->split(c->gcol, c->grow, &e);
      if (!c->colt) TRY(fail(c, IPR_E_NCCL, "grid column split: %s", e.c_str()));
    }
    TRYC(cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking));
    for (auto &ev : c->gev) TRYC(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  TRYC(cudaStreamSynchronize(c->st));
#undef TRY
#undef TRYC
  *out = c;
  return IPR_OK;
}

ipr_status ipr_init(ipr_ctx **out, int64_t n, const double *A_dev, int64_t lda, void *cuda_stream, int world,
                    int rank, const void *nccl_unique_id, int grid_rows, int grid_cols) {
  return init_ctx(out, n, A_dev, lda, cuda_stream, world, rank, nccl_unique_id, nullptr, grid_rows, grid_cols);
}

ipr_status ipr_test_local_group_create(int world, ipr_local_group **out) {
  ipr_ctx *c = nullptr;
  if (!out) return fail(c, IPR_E_INVALID_ARG, "ipr_test_local_group_create: null output");
  std::string e;
  LocalGroup *g = local_group_create(world, &e);
  if (!g) return fail(c, IPR_E_INVALID_ARG, "%s", e.c_str());
  *out = (ipr_local_group *)g;
  return IPR_OK;
}

ipr_status ipr_test_local_group_destroy(ipr_local_group *g) {
  local_group_destroy((LocalGroup *)g);
  return IPR_OK;
}

ipr_status ipr_test_init_local(ipr_ctx **out, int64_t n, const double *A_dev, int64_t lda, void *cuda_stream,
                               ipr_local_group *group, int rank, int grid_rows, int grid_cols) {
  ipr_ctx *c = nullptr;
  if (!group) return fail(c, IPR_E_INVALID_ARG, "ipr_test_init_local: null group");
  LocalGroup *g = (LocalGroup *)group;
  return init_ctx(out, n, A_dev, lda, cuda_stream, local_group_world(g), rank, nullptr, g, grid_rows, grid_cols);
}

ipr_status ipr_set_schedule(ipr_ctx *c, int p, const ipr_phase *phases, int nphases, double final_tol) {
  if (!c) return fail(c, IPR_E_INVALID_ARG, "ipr_set_schedule: null context");
  if (c->started) return fail(c, IPR_E_STATE, "ipr_set_schedule: iteration already started");
  if (p < 1 || p > 64) return fail(c, IPR_E_INVALID_ARG, "ipr_set_schedule: p must be in [1, 64] (got %d)", p);
  if (!phases || nphases < 1 || nphases > 16) return fail(c, IPR_E_INVALID_ARG, "ipr_set_schedule: 1..16 phases");
  if (!(final_tol >= 0.0)) return fail(c, IPR_E_INVALID_ARG, "ipr_set_schedule: final_tol must be >= 0");
  std::vector<PhaseC> v;
  int prev_ob = -1, prev_m = -1;
  for (int i = 0; i < nphases; ++i) {
    const ipr_phase &q = phases[i];
    if (q.prec < IPR_FP64 || q.prec > IPR_FP64_CRT) return fail(c, IPR_E_INVALID_ARG, "phase %d: bad prec", i);
    PhaseC P;
    P.prec = q.prec;
    P.cont64 = is_f64(q.prec);
    const int mmax = P.cont64 ? 52 : 23;
    P.adaptive = is_emu(q.prec) && q.mant_bits == IPR_MANT_ADAPTIVE;
    if (q.mant_bits < -1 && !P.adaptive)
      return fail(c, IPR_E_INVALID_ARG, "phase %d: mant_bits %d (IPR_MANT_ADAPTIVE needs IPR_FP64_OZ / IPR_FP64_CRT)", i,
                  q.mant_bits);
    P.m = q.mant_bits < 0 ? native_m(q.prec) : q.mant_bits;
    if (P.m > mmax) return fail(c, IPR_E_INVALID_ARG, "phase %d: mant_bits %d > %d for this container", i, P.m, mmax);
    if (q.round != IPR_RNE && q.round != IPR_RTZ) return fail(c, IPR_E_INVALID_ARG, "phase %d: bad round", i);
    P.rtz = q.round == IPR_RTZ;
    if (!(q.switch_tol >= 0) || !(q.plateau_ratio >= 0) || q.max_iters < 0)
      return fail(c, IPR_E_INVALID_ARG, "phase %d: negative tolerance / cap", i);
    if (q.plateau_ratio > 0 && !(q.plateau_arm > 0))
      return fail(c, IPR_E_INVALID_ARG, "phase %d: plateau_ratio needs plateau_arm > 0", i);
    P.switch_tol = q.switch_tol; P.plateau_ratio = q.plateau_ratio; P.plateau_arm = q.plateau_arm;
    P.max_iters = q.max_iters;
    P.corr = q.corr_prec >= 0 ? q.corr_prec : is_scaled(q.prec) ? IPR_BF16 : q.prec;
    if (P.corr < IPR_FP64 || P.corr > IPR_FP64_CRT) return fail(c, IPR_E_INVALID_ARG, "phase %d: bad corr_prec", i);
    if (is_emu(P.corr)) P.corr = IPR_FP64;   // an FP64 correction runs on DMMA
    if (P.corr == IPR_FP64 && !is_f64(P.prec))
      return fail(c, IPR_E_INVALID_ARG, "phase %d: an FP64 correction needs an FP64 phase", i);
    const int ob = operand_bits(q.prec);
    if (ob < prev_ob || (ob == prev_ob && P.m < prev_m))
      return fail(c, IPR_E_INVALID_ARG, "phase %d: precision must be non-decreasing along the schedule", i);
    prev_ob = ob; prev_m = P.m;
    if (!is_f64(P.prec) && !tc_supported(P.prec))
      return fail(c, IPR_E_UNSUPPORTED, "phase %d: tcgen05 path for this precision is not built", i);
    v.push_back(P);
  }
  c->p = p; c->ph = v; c->final_tol = final_tol; c->scheduled = true;
  c->err.clear();
  if (p >= 2 && !(c->norms[2] > std::pow(2.0, -1.0 / (p - 1)))) {
    c->err = "warning: max diagonal <= 2^(-1/(p-1)): the sufficient condition for Eq. (2) (reading R-12) fails";
  }
  return IPR_OK;
}

ipr_status ipr_set_form(ipr_ctx *c, int form) {
  if (!c) return fail(c, IPR_E_INVALID_ARG, "ipr_set_form: null context");
  if (c->started) return fail(c, IPR_E_STATE, "ipr_set_form: iteration already started");
  if (form < IPR_FORM_LITERAL || form > IPR_FORM_SYMMETRIC_TRIZ)
    return fail(c, IPR_E_INVALID_ARG, "ipr_set_form: unknown form %d", form);
  c->triz = form == IPR_FORM_SYMMETRIC_TRIZ;   // R-37: the tri form + the Z_1 rule of ztri_chain()
  c->form = c->triz ? (int)IPR_FORM_SYMMETRIC_TRI : form;
  return IPR_OK;
}

ipr_status ipr_set_cert(ipr_ctx *c, int mode) {
  if (!c) return fail(c, IPR_E_INVALID_ARG, "ipr_set_cert: null context");
  if (c->started) return fail(c, IPR_E_STATE, "ipr_set_cert: iteration already started");
  if (mode != IPR_CERT_FP64 && mode != IPR_CERT_PHASE && mode != IPR_CERT_FP64_CHAIN && mode != IPR_CERT_CRT)
    return fail(c, IPR_E_INVALID_ARG, "ipr_set_cert: unknown mode %d", mode);
  c->cert = mode;
  return IPR_OK;
}

// Reading R-33: after an update in the last phase of a symmetric form, the in-phase linear rate
// q = rho_k / rho_{k-1} predicts rho_{k+1} ~ rho_k q.  When that is <= final_tol / 2 the next iterate is
// certified first (the FP64 residual the stop needs anyway); its chain -- computed only to trigger the
// certificate -- runs only if the certificate misses.  The oracle mirrors the rule (orc_solve_form).
// A missed certificate turns the decision into "continue" -- but the last phase's iteration cap still
// applies (without it an in-chain residual below final_tol over an FP64 floor above it, e.g. n = 32768,
// would certify and miss forever): the trace record becomes IPR_DEC_ITER_LIMIT and the solve ends.
static bool cert_cap(ipr_ctx *c) {
  const PhaseC &P = c->ph[c->phase];
  if (!(P.max_iters > 0 && c->it_in_phase >= P.max_iters)) return false;
  c->trace.back().decision = IPR_DEC_ITER_LIMIT;
  c->done = true;
  c->outcome = IPR_DEC_ITER_LIMIT;
  return true;
}

static bool predict_cert(const ipr_ctx *c) {
  if ((c->cert != IPR_CERT_FP64 && c->cert != IPR_CERT_CRT) || !is_sym(c) || c->phase != (int)c->ph.size() - 1)
    return false;
  if (!(std::isfinite(c->ph_r1) && std::isfinite(c->ph_r2) && c->ph_r2 > 0.0 && c->ph_r1 < c->ph_r2)) return false;
  return c->ph_r1 * (c->ph_r1 / c->ph_r2) <= 0.5 * c->final_tol;
}

ipr_status ipr_iterate(ipr_ctx *c, int max_iters, int *iters_done, ipr_outcome *outcome) {
  if (!c || !iters_done || !outcome) return fail(c, IPR_E_INVALID_ARG, "ipr_iterate: null pointer");
  if (!c->scheduled) return fail(c, IPR_E_STATE, "ipr_iterate: call ipr_set_schedule first");
  if (max_iters <= 0) return fail(c, IPR_E_INVALID_ARG, "ipr_iterate: max_iters must be > 0");
  *iters_done = 0;
  if (c->done) { *outcome = (ipr_outcome)c->outcome; return IPR_OK; }
  if (!c->started) {
    if (c->form == IPR_FORM_NEWTON_SCHULZ) {
      if (c->p != 1) return fail(c, IPR_E_INVALID_ARG, "ipr_iterate: the Newton-Schulz form needs p = 1");
    }
    bool need_c = false;
    for (auto &P : c->ph)
      if (c->form == IPR_FORM_COUPLED && (is_scaled(P.prec) || is_emu(P.prec)))
        return fail(c, IPR_E_UNSUPPORTED, "ipr_iterate: the coupled form takes FP64 / TF32 / BF16 phases");
    for (auto &P : c->ph)
      if (P.prec == IPR_FP64_OZ && c->npad > 47800)   // INT32 digit-group sums (ozaki.cu)
        return fail(c, IPR_E_UNSUPPORTED, "ipr_iterate: IPR_FP64_OZ needs n <= 47800 (exact INT32 group sums)");
    for (auto &P : c->ph) {
      if (is_emu(P.prec) && !is_sym(c))
        return fail(c, IPR_E_UNSUPPORTED, "ipr_iterate: IPR_FP64_OZ / IPR_FP64_CRT phases need a symmetric form");
      if (P.prec == IPR_FP64_OZ && c->world != 1)
        return fail(c, IPR_E_UNSUPPORTED, "ipr_iterate: IPR_FP64_OZ phases are single-GPU (IPR_FP64_CRT shards)");
    }
    if (c->cert == IPR_CERT_CRT) {   // reading R-35: where the CRT certificate is built
      bool crt = false;
      for (auto &P : c->ph) crt |= P.prec == IPR_FP64_CRT;
      const int nm = crt_moduli(kCertBits, c->n);
      if (!is_sym(c) || !(c->p == 2 || (c->p == 3 && c->world == 1)) || c->grows != 1 || !crt ||
          !c->ph.back().cont64 || nm < 16)
        return fail(c, IPR_E_UNSUPPORTED,
                    "ipr_iterate: IPR_CERT_CRT needs a symmetric form with p = 2 on a 1 x G grid or p = 3 on one GPU, "
                    "an IPR_FP64_CRT phase and an FP64 last phase, and n <= 65535");
    }
    if (c->grows > 1) {   // the 2-D grid option: Eq. (1) as printed, unscaled tensor-core / DMMA formats
      if (c->form != IPR_FORM_LITERAL)
        return fail(c, IPR_E_UNSUPPORTED, "ipr_iterate: 2-D grids (grid_rows > 1) run the literal form only");
      for (auto &P : c->ph)
        if (P.prec != IPR_FP64 && P.prec != IPR_TF32 && P.prec != IPR_BF16)
          return fail(c, IPR_E_UNSUPPORTED, "ipr_iterate: 2-D grids take FP64 / TF32 / BF16 phases");
    }
    if (is_sym(c)) {
      if (c->p < 2) return fail(c, IPR_E_INVALID_ARG, "ipr_iterate: the symmetric form needs p >= 2 (p = 1: Newton-Schulz)");
      if (c->form == IPR_FORM_SYMMETRIC_TRI && c->p != 2)
        return fail(c, IPR_E_INVALID_ARG, "ipr_iterate: the symmetric-tri form needs p = 2 (Z_2 = C A C symmetric)");
      c->wbytes = 4;
      for (auto &P : c->ph) {
        if (is_scaled(P.corr) && P.corr != P.prec)
          return fail(c, IPR_E_UNSUPPORTED,
                      "ipr_iterate: the symmetric form's correction must be BF16, TF32, FP64 or the phase's own scaled format");
        if (P.corr != IPR_FP64 && !tc_supported(P.corr))
          return fail(c, IPR_E_UNSUPPORTED, "ipr_iterate: tcgen05 path for the correction precision is not built");
        need_c |= !same_fmt(P.corr, P.prec);
        if (P.corr == IPR_FP64) c->wbytes = 8;
      }
    }
    if (!c->arena) CKS(alloc_arena(c, need_c));
    c->phase = 0; c->it_in_phase = 0; c->cur = 0;
    tl_mark(c, "entry");
    CKS(begin_phase(c, true));
    tl_mark(c, "gap");
    c->started = true;
  }
  for (int it = 0; it < max_iters; ++it) {
    if (c->cert_pending) {                 // R-33: the predicted-converged iterate, certificate first
      c->cert_pending = false;
      double rc = NAN;
      CKS(stream_candidate(c, c->cur));
      tl_mark(c, "cert");
      CKS(certify_iter(c, c->cur, &rc));
      tl_mark(c, "gap");
      if (rc <= c->final_tol) {
        c->out_valid = c->out_buf == c->cur;
        ipr_record r;
        memset(&r, 0, sizeof r);
        r.k = (int)c->trace.size(); r.phase = c->phase; r.prec = c->ph[c->phase].prec; r.mant_bits = c->m_of_cur;
        r.decision = IPR_DEC_CONVERGED; r.rho = NAN; r.rho_hat = NAN; r.delta = NAN; r.rho_cert = rc;
        r.gap_ms = NAN;
        c->trace.push_back(r);
        *iters_done += 1;
        c->best_loc = c->cur; c->best_cont64 = is_f64(c->ph[c->phase].prec);
        c->done = true;
        c->outcome = IPR_DEC_CONVERGED;
        break;
      }
      c->cert_prev = rc;                   // missed: the chain runs; its record carries this certificate
      if (c->out_buf >= 0) CK(cudaStreamWaitEvent(c->st, c->oev, 0));   // the copy reads C_k: done before reuse
      if (c->world > 1) CKS(make_xt(c, c->cur, c->ph[c->phase]));   // the certificate reused the T buffers
    }
    const double cert_pre = c->cert_prev;
    c->cert_prev = NAN;
    double rho = NAN;
    float ms = 0.f;
    tl_mark(c, "chain");
    CKS(chain(c, &rho, &ms));
    tl_mark(c, "gap");
    c->last_rho = rho;
    const int phase_now = c->phase;
    bool best_new = false;
    const int d = decide(c, rho, &best_new);
    c->ph_r2 = c->ph_r1; c->ph_r1 = rho;   // R-26 in-phase history (reset by begin_phase)
    if (std::isfinite(c->ph_r2) && !(c->ph_r1 <= kZtriRatio * c->ph_r2)) c->z_ok = false;   // R-37: sticky
    if (best_new) { c->best_loc = c->cur; c->best_cont64 = is_f64(c->ph[c->phase].prec); }
    ipr_record r;
    r.k = (int)c->trace.size(); r.phase = phase_now; r.prec = c->ph[phase_now].prec; r.mant_bits = c->m_of_cur;
    r.decision = d; r.rho = rho; r.rho_hat = rho / std::sqrt((double)c->n); r.delta = NAN; r.gemm_ms = ms;
    r.rho_cert = cert_pre; r.upd_ms = 0.0;
    r.kern_ms = 0.0;                           // chain_timers() fills gemm_ms / kern_ms
    r.gap_ms = NAN;
    r.digits = is_emu(c->ph[phase_now].prec) ? c->last_chain_S : 0;
    r.moduli = c->ph[phase_now].prec == IPR_FP64_CRT ? crt_moduli(crt_bits(c->last_chain_S, c->n), c->n) : 0;
    r.ztri = c->last_chain_ztri;
    c->trace.push_back(r);
    *iters_done += 1;
    if (d != IPR_DEC_CONTINUE) CKS(chain_timers(c, c->trace.back()));
    if (d == IPR_DEC_CONVERGED && c->form == IPR_FORM_COUPLED) {
      // rho = ||I - M_k||_F tracks ||I - X_k^p A||_F only up to drift: certify X_k itself with the
      // FP64 literal chain on DMMA (R-3, R-27; the computation ipr_residual(certify = 1) runs); if it
      // misses, take the step and continue.  A certified X_k is the answer (best := X_k).
      double rc = NAN;
      CKS(certify_iter(c, c->cur, &rc));
      c->trace.back().rho_cert = rc;
      if (!(rc <= c->final_tol)) {
        c->trace.back().decision = IPR_DEC_CONTINUE;
        CKS(update_coupled(c));
        c->pending_delta = (int64_t)c->trace.size() - 1;
        if (cert_cap(c)) break;
        continue;
      }
      c->best_loc = c->cur; c->best_cont64 = is_f64(c->ph[c->phase].prec);
      c->done = true;
      c->outcome = d;
      break;
    }
    if (d == IPR_DEC_CONVERGED && is_sym(c)) {
      // rho_s = ||I - C^{p-1}AC||_F met final_tol: certify ||I - C_k^p A||_F (R-3, R-30).
      //  IPR_CERT_FP64 (default): ||I - C^p A||_F on the FP64 DMMA pipe (p = 2: (C C) A with C C on its
      //    upper tiles, reading R-32; else the literal chain C (C A)) -- the same function
      //    ipr_residual(certify = 1) runs, so a converged solve's re-check equals its certificate bit
      //    for bit.  p = 2: the certification stores only T_1 (T[1]); R (T[p & 1] = T[0]) survives, so
      //    the update runs only if the certification misses.
      //  IPR_CERT_PHASE: the phase's own product from the Z_1 = A C its chain kept (an FP64-range
      //    estimate: the CRT / Ozaki quantisation error is not bounded here -- see ipr.h).
      // A certified C_k is the answer (best := C_k); on a miss the iteration continues from C_{k+1}.
      const int ck = c->cur;
      const bool phase_cert = c->cert == IPR_CERT_PHASE && c->zr_for == ck && c->best_loc == ck;
      const bool cert_first = c->p == 2;
      if (!cert_first) {
        CKS(update_sym(c));
        c->pending_delta = (int64_t)c->trace.size() - 1;
      }
      double rc = NAN;
      if (std::isfinite(cert_pre)) rc = cert_pre;      // certified before the chain (R-33) and missed
      else {
        CKS(stream_candidate(c, ck));
        tl_mark(c, "cert");
        if (phase_cert) CKS(certify_from_zr(c, ck, &rc));
        else CKS(certify_iter(c, ck, &rc));
        tl_mark(c, "gap");
      }
      c->trace.back().rho_cert = rc;
      if (!(rc <= c->final_tol)) {
        c->out_valid = false;
        if (c->out_buf >= 0) CK(cudaStreamWaitEvent(c->st, c->oev, 0));
        c->trace.back().decision = IPR_DEC_CONTINUE;
        if (cert_first) {
          tl_mark(c, "update");
          CKS(update_sym(c));
          tl_mark(c, "gap");
          c->pending_delta = (int64_t)c->trace.size() - 1;
        }
        if (c->world > 1) CKS(make_xt(c, c->cur, c->ph[c->phase]));
        if (cert_cap(c)) break;
        c->cert_pending = predict_cert(c);
        continue;
      }
      c->best_loc = ck; c->best_cont64 = is_f64(c->ph[c->phase].prec);
      c->out_valid = c->out_buf == ck;
      c->done = true;
      c->outcome = d;
      break;
    }
    if (d == IPR_DEC_CONTINUE) {
      tl_mark(c, "update");
      CKS(step_update(c));
      tl_mark(c, "gap");
      c->pending_delta = (int64_t)c->trace.size() - 1;
      c->cert_pending = predict_cert(c);
      CKS(chain_timers(c, c->trace.back()));   // after the update is enqueued: no bubble
    } else if (d == IPR_DEC_SWITCH) {
      if (c->best_loc < 0) { c->best_loc = c->cur; c->best_cont64 = is_f64(c->ph[c->phase].prec); }
      CKS(save_best(c));
      c->phase += 1; c->it_in_phase = 0; c->rho_prev = NAN;
      c->cur = 0;
      tl_mark(c, "entry");
      CKS(begin_phase(c, false));
      tl_mark(c, "gap");
    } else {
      c->done = true;
      c->outcome = d;   // IPR_DEC_* terminal values equal the ipr_outcome values
      break;
    }
  }
  CKS(join_gather(c));   // no side-stream exchange outlives the call
  *outcome = c->done ? (ipr_outcome)c->outcome : IPR_RUNNING;
  return IPR_OK;
}

ipr_status ipr_get_trace(ipr_ctx *c, ipr_record *buf, int cap, int *count) {
  if (!c || !count) return fail(c, IPR_E_INVALID_ARG, "ipr_get_trace: null pointer");
  if (c->pending_delta >= 0) {
    CK(cudaMemcpyAsync(c->hscal + 1, c->dscal + 1, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    float tu = 0.f;
    float tg = 0.f;
    if (c->upd_timed) {
      CK(cudaEventElapsedTime(&tu, c->ev[2], c->ev[3]));
      CK(cudaEventElapsedTime(&tg, c->ev[5], c->ev[2]));
      c->upd_timed = false;
    }
    c->trace[c->pending_delta].delta = std::sqrt(c->hscal[1]);
    c->trace[c->pending_delta].gemm_ms += tu;
    c->trace[c->pending_delta].upd_ms = tu;
    c->trace[c->pending_delta].gap_ms = tg;
    c->pending_delta = -1;
  }
  *count = (int)c->trace.size();
  if (buf && cap > 0) {
    const int k = cap < *count ? cap : *count;
    memcpy(buf, c->trace.data(), sizeof(ipr_record) * (size_t)k);
  }
  return IPR_OK;
}

ipr_status ipr_get_norms(ipr_ctx *c, double *out4) {
  if (!c || !out4) return fail(c, IPR_E_INVALID_ARG, "ipr_get_norms: null pointer");
  memcpy(out4, c->norms, sizeof c->norms);
  return IPR_OK;
}

static ipr_status copy_iterate(ipr_ctx *c, int which, double *dst, int64_t ldc) {
  const int64_t cnt = blk(c);
  double *slot = c->full64 + (size_t)c->rank * cnt;
  if (which == 0) {
    const PhaseC &P = c->ph[c->phase];
    CK(launch_cont_to_f64(cont_ptr(c, c->cur, P), P.cont64, cnt, slot, c->st));
  } else {
    if (c->best_loc < 0) return fail(c, IPR_E_STATE, "no iterate evaluated yet");
    CKS(save_best(c));
    CK(cudaMemcpyAsync(slot, c->best, (size_t)cnt * 8, cudaMemcpyDeviceToDevice, c->st));
  }
  CKS(gather_f64(c, slot));
  if (dst && is_host_ptr(dst)) {
    // host destination: one 2-D copy per (row, column) block of the block-major [world][mr][kp] layout
    for (int b = 0; b < c->world; ++b) {
      const int64_t r0 = (int64_t)(b / c->gcols) * c->mr, c0 = (int64_t)(b % c->gcols) * c->kp;
      const int64_t nr = std::min(c->mr, c->n - r0), nc = std::min(c->kp, c->n - c0);
      if (nr <= 0 || nc <= 0) continue;
      CK(cudaMemcpy2DAsync(dst + r0 * ldc + c0, (size_t)ldc * 8, c->full64 + (size_t)b * blk(c), (size_t)c->kp * 8,
                           (size_t)nc * 8, (size_t)nr, cudaMemcpyDeviceToHost, c->st));
    }
  } else if (dst) {
    CK(launch_copy_out_blocks(c->full64, c->mr, c->kp, c->gcols, c->n, dst, ldc, c->st));
  }
  CK(cudaStreamSynchronize(c->st));
  return IPR_OK;
}

// ipr_set_output: stream the candidate C_k (FP64 container, G = 1) to the caller's destination on a copy
// stream while its certificate runs; finalize then only waits for it if C_k is the answer
static ipr_status stream_candidate(ipr_ctx *c, int i) {
  c->out_valid = false;
  if (c->cert == IPR_CERT_CRT) return IPR_OK;   // certify_crt streams the certified matrix Ct itself
  const PhaseC &P = c->ph[c->phase];
  if (!c->out_ptr || c->world != 1 || !P.cont64) return IPR_OK;
  if (!c->ost) {
    CK(cudaStreamCreateWithFlags(&c->ost, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->oev, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->orev, cudaEventDisableTiming));
  }
  if (c->out_buf >= 0) CK(cudaStreamWaitEvent(c->st, c->oev, 0));   // a previous copy reads a live buffer
  CK(cudaEventRecord(c->orev, c->st));
  CK(cudaStreamWaitEvent(c->ost, c->orev, 0));
  CK(cudaMemcpy2DAsync(c->out_ptr, (size_t)c->out_ld * 8, cont_ptr(c, i, P), (size_t)c->kp * 8, (size_t)c->n * 8,
                       (size_t)c->n, cudaMemcpyDefault, c->ost));
  CK(cudaEventRecord(c->oev, c->ost));
  c->out_buf = i;
  return IPR_OK;
}

ipr_status ipr_get_iterate(ipr_ctx *c, int which, double *C_dev_out, int64_t ldc) {
  if (!c || !C_dev_out) return fail(c, IPR_E_INVALID_ARG, "ipr_get_iterate: null pointer");
  if (ldc < c->n) return fail(c, IPR_E_INVALID_ARG, "ipr_get_iterate: ldc < n");
  if (which != 0 && which != 1) return fail(c, IPR_E_INVALID_ARG, "ipr_get_iterate: which must be 0 or 1");
  if (!c->started) return fail(c, IPR_E_STATE, "ipr_get_iterate: no iterate yet (call ipr_iterate)");
  return copy_iterate(c, which, C_dev_out, ldc);
}

// ||I - C^p A||_F of the iterate in buffer i (FP64, exact operand) from the Zr = A C kept by its
// chain: X_1 = C (C A) [B = Zr row-major], X_j = C X_{j-1}; p - 1 DMMA GEMMs, the last with the
// residual partials (reading R-3; same arithmetic class as certify_best).
static ipr_status certify_from_zr(ipr_ctx *c, int i, double *rho) {
  // in an IPR_FP64_OZ phase the certifying product runs on the same FP64-accurate Ozaki GEMM
  // (9 digits); ipr_residual(certify = 1) recomputes the whole chain on the DMMA pipe
  const void *X = c->Zr;
  const int prec = is_emu(c->ph[c->phase].prec) ? c->ph[c->phase].prec : IPR_FP64;
  for (int j = 2; j <= c->p; ++j) {
    GemmArgs g = base_args(c, prec, X);
    chat_view(c, i, prec, &g.A, &g.a_kp, &g.a_pstride);
    g.mode = j == c->p ? EPI_RESID : EPI_STORE_T;     // the last product: residual partials only
    g.tout = c->T[j & 1]; g.ldt = c->npad; g.part = c->part;
    if (prec == IPR_FP64_OZ) CKS(oz_operands(c, g, i, X));
    if (prec == IPR_FP64_CRT) CKS(crt_operands(c, g, i, X));
    CK(run_gemm(c, g));
    X = c->T[j & 1];
  }
  CK(launch_reduce_sum(c->part, tiles_n_total(c, prec) * tiles_m(c, prec), c->dscal + 2, c->st));
  CK(cudaMemcpyAsync(c->hscal + 2, c->dscal + 2, 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  *rho = std::sqrt(c->hscal[2]);
  return IPR_OK;
}

// ||I - C^p A||_F of the FP64 iterate in full64 (panel-major, every rank) with the literal chain on the
// FP64 DMMA pipe: T_1 = C A, T_j = C T_{j-1}; the last GEMM keeps only its residual partials, so T[p & 1]
// is not written for p = 2 (reading R-3).  Deterministic: the same iterate gives the same bits.
static ipr_status certify_full64(ipr_ctx *c, double *rho) {
  Nvtx nv("certify fp64 dmma");
  PhaseC P64{IPR_FP64, 52, 0, 1, 0, 0, 0, 0};
  CKS(stage_a(c, P64, c->Acert, c->dsig + 0));
  if (c->p == 2 && c->form != IPR_FORM_LITERAL) {
    // reading R-32: ||I - Y A||_F with Y = C C.  C is bitwise symmetric, so the DMMA product Y is too
    // (each Y_ij and Y_ji is the same K-ordered sum of the same products; tests/test_gpu_certify.py):
    // G = 1 computes only its upper tiles and mirrors them (tri), a G > 1 rank its full column panel,
    // then all-gathers Y -- the same bits.  1.5 DMMA GEMMs instead of the chain's 2.  The literal
    // form keeps the chain C (C A): its FP64 phase's in-chain rho is that chain and IS its certificate.
    GemmArgs g = base_args(c, IPR_FP64, c->full64);   // G = 1: C is its own K-major form
    g.A = c->full64; g.a_kp = c->kp; g.a_pstride = c->npad * c->kp;
    double *Y = (double *)c->T[1];
    if (c->world == 1) {
      g.tri = 1; g.mode = EPI_STORE_T; g.tout = Y; g.ldt = c->npad;   // Y row-major (= its transpose)
    } else {
      // B(k, j) = C[col0 + j][k]: row col0 + j of the gathered panel-major C, a paneled B view (T[0]
      // holds R, which the update needs if the certificate misses)
      g.B = c->full64 + (size_t)c->col0 * c->kp; g.ldb = c->kp; g.b_kp = c->kp; g.b_pstride = c->npad * c->kp;
      g.mode = EPI_STORE_N; g.nout = Y; g.ldn = c->kp; // Y[:, S_g] as a [npad][kp] panel
    }
    CK(run_gemm(c, g));
    if (c->world > 1) CKS(gather_f64(c, Y));           // full64 := Y, panel-major
    GemmArgs h = base_args(c, IPR_FP64, c->Acert);
    h.A = c->world == 1 ? (const void *)Y : (const void *)c->full64;
    h.a_kp = c->kp; h.a_pstride = c->npad * c->kp;
    h.mode = EPI_RESID; h.part = c->part;
    CK(run_gemm(c, h));
  } else {
    const void *X = c->Acert;
    for (int j = 1; j <= c->p; ++j) {
      GemmArgs g = base_args(c, IPR_FP64, X);
      g.A = c->full64; g.a_kp = c->kp; g.a_pstride = c->npad * c->kp;
      g.mode = j == c->p ? EPI_RESID : EPI_STORE_T;
      g.tout = c->T[j & 1]; g.ldt = c->npad; g.part = c->part;
      CK(run_gemm(c, g));
      X = c->T[j & 1];
    }
  }
  const int64_t tm = tiles_m(c, IPR_FP64), tn_loc = c->kp / gemm_tile_n(IPR_FP64);
  CKS(gather_partials(c, c->part, tn_loc * tm));
  CK(launch_reduce_sum(c->part, tiles_n_total(c, IPR_FP64) * tm, c->dscal + 2, c->st));
  CK(cudaMemcpyAsync(c->hscal + 2, c->dscal + 2, 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  *rho = std::sqrt(c->hscal[2]);
  return IPR_OK;
}

// Reading R-35 (IPR_CERT_CRT; symmetric forms, p = 2, one GPU): a PROVEN upper bound on ||I - Ct^2 A||_F
// for the certified matrix Ct -- the candidate C in full64 rounded to the coarser of its row's and its
// column's b-bit grids (b = 62; |Ct - C| <= 2^-62 relative to the row / column maximum) -- from exact
// integer products on the INT8 tensor cores (Ozaki scheme II, R-28) instead of FP64 DMMA GEMMs:
//   1. e_i from C's rows; Ct in place (full64); the residues of 2^e_i Ct_ij -- EXACT, so the one residue
//      set is both operands of Y = Ct Ct (Ct is symmetric; checked bitwise)
//   2. A staged in FP64 (T[1]) and split at b bits: Atilde, ||Atilde - A||_F
//   3. Y = Ct Ct on the upper tiles (mirrored), reconstructed exactly as hi (T[1]) + lo (Zr)
//   4. Y split from hi + lo: Ytilde, ||Ytilde - Yh||_F, the row sums of |hi| + |lo|
//   5. P = Ytilde Atilde exact; the partials of (delta_ij - hi) - lo
// Since I - Ct^2 A = (I - P) + (Ytilde - Y) Atilde + Y (Atilde - A) (Y = Ct^2 exact),
//   ||I - Ct^2 A||_F <= ||I - P||_F + (dY + eY)(||A||_2 + dA) + ||Y||_2 dA,
// with ||A||_2 <= ||A||_1 and ||Y||_2 <= ||Y||_inf (both symmetric), dY / dA the measured quantisation
// errors, eY / eP the reconstruction bounds (n 2^(s1-48) max 2^-(e_i+f_j)), every FP64 sum inflated by
// 1 + 1e-10 (>= n u for n <= 9e5).  *rho = that bound; c->cert_info keeps its terms.
// i >= 0: the candidate came from iterate buffer i -- with ipr_set_output the certified Ct streams to the
// caller during the products, and a passing Ct replaces C_i in its (FP64) container: Ct is the answer.
static ipr_status certify_crt(ipr_ctx *c, int i, double *rho, const double *cand = nullptr) {
  Nvtx nv("certify crt");
  cudaStream_t st = c->st;
  const int b = kCertBits, nm = crt_moduli(b, c->n);
  const int64_t np = c->npad, kp = c->kp, col0 = c->col0;
  const bool sh = c->world > 1;                    // 1 x G column panels: rank g owns the columns S_g
  const bool p3 = c->p == 3;                       // p = 3 (G = 1): T = Ct Ytilde between Y and the residual
  double *err2Y = c->certv, *asumY = c->certv + np, *scY = c->certv + 2 * np, *err2A = c->certv + 3 * np;
  double *asumA = c->certv + 4 * np, *scA = c->certv + 5 * np, *scC = c->certv + 6 * np;
  double *err2T = c->certv + 7 * np, *asumT = c->certv + 8 * np, *scT = c->certv + 9 * np;
  double *asumC = c->certv + 10 * np;
  if (!c->hcert && !(c->hcert = pinned_acquire())) return fail(c, IPR_E_OOM, "pinned host slab exhausted");
  // G > 1: the gathered C (panel-major in full64) row-major in chat_rm; every rank rounds and splits all
  // of it (the A role of Y = Ct Ct needs every row), the B role takes the rows S_g of the same residues
  double *Ct = sh ? (double *)c->chat_rm : c->full64;
  if (sh) CK(launch_copy_out(c->full64, np, kp, c->n, Ct, np, st));
  // cand (G = 1, FP64 container): the candidate is read in place from its container; Ct goes to full64
  const double *Cin = cand ? cand : Ct;
  // 1. the certified matrix and its residues
  CK(launch_cert_rowexp(Cin, np, np, np, b, c->crC_sig, scC, st));
  CK(launch_cert_round_split(Cin, Ct, np, np, np, nm, c->crC_sig, c->crC, p3 ? asumC : nullptr, st));
  c->crC_for = -1;
  CK(cudaMemsetAsync(c->dflag + 2, 0, 4, st));
  CK(launch_symcheck(Ct, np, c->n, c->dflag + 2, st));
  if (i >= 0 && c->out_ptr && !sh) {               // ipr_set_output: stream Ct while the products run
    if (!c->ost) {
      CK(cudaStreamCreateWithFlags(&c->ost, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->oev, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->orev, cudaEventDisableTiming));
    }
    if (c->out_buf >= 0) CK(cudaStreamWaitEvent(st, c->oev, 0));
    CK(cudaEventRecord(c->orev, st));
    CK(cudaStreamWaitEvent(c->ost, c->orev, 0));
    CK(cudaMemcpy2DAsync(c->out_ptr, (size_t)c->out_ld * 8, Ct, (size_t)np * 8, (size_t)c->n * 8, (size_t)c->n,
                         cudaMemcpyDefault, c->ost));
    CK(cudaEventRecord(c->oev, c->ost));
    c->out_buf = i;
  }
  const int8_t *ctB = c->crC;                      // B role of Ct: its rows S_g (G > 1: compact copy in crB)
  double *ylo = (double *)c->Zr;
  if (sh) {
    CK(cudaMemcpy2DAsync(c->crB, (size_t)(kp * np), c->crC + col0 * np, (size_t)(np * np), (size_t)(kp * np), (size_t)nm,
                         cudaMemcpyDeviceToDevice, st));
    ctB = c->crB;
    ylo = (double *)(c->crB + ((size_t)nm * kp * np + 255) / 256 * 256);   // 18/G + 8/G <= 18 bytes per n^2
  }
  PhaseC P64{IPR_FP64, 52, 0, 1, 0, 0, 0, 0};
  // A in FP64 (m = 52; its local K-major panel = the rows S_g): an FP64-range phase with m = 52 staged exactly
  // that as its operand (Aop), else stage it now
  const PhaseC &Pc = c->ph[c->phase];
  const bool aop_exact = is_f64(Pc.prec) && Pc.m == 52 && !Pc.rtz;
  auto a_f64 = [&](ipr_ctx *cc) -> const double * {
    if (aop_exact) return (const double *)cc->Aop;
    if (stage_a(cc, P64, cc->T[1], cc->dsig + 0) != IPR_OK) return nullptr;
    return (const double *)cc->T[1];
  };
  // 2. (p = 2) A's residues
  if (!p3) {
    const double *Af = a_f64(c);
    if (!Af) return IPR_E_CUDA;
    CK(launch_cert_split(Af, nullptr, np, kp, np, b, nm, c->crA, 0, c->crA_sig, scA + col0, err2A + col0,
                         asumA + col0, st));
  }
  c->crA_b = -1;
  // 3. Y = Ct Ct exact, hi + lo: G = 1 its upper tiles mirrored (row-major); G > 1 the column panel
  //    Y[:, S_g] stored K-major, i.e. the rows S_g of the symmetric Y
  GemmArgs g = base_args(c, IPR_FP64_CRT, nullptr);
  g.oz_a = c->crC; g.oz_rsig = c->crC_sig; g.oz_b = ctB; g.oz_csig = c->crC_sig + col0;
  g.crt_n = nm; g.crt_v = c->crV; g.crt_dd = 1;
  g.nout = c->T[1]; g.ldn = np; g.zout = ylo; g.ldz = np;
  if (sh) g.mode = EPI_STORE_T;
  else { g.tri = 1; g.mode = EPI_STORE_N; }
  CK(launch_gemm_crt(g, st));
  c->zr_for = -1;
  if (p3) {
    // p = 3: Y's rows -> crA (Y is exactly symmetric, so its row quantisation read as columns is the B
    // role of T = Ct Ytilde); T exact (full) -> hi + lo; T's rows -> crC; then A -> crA
    int *ysig = c->crA_sig;
    CK(launch_cert_split((const double *)c->T[1], ylo, np, np, np, b, nm, c->crA, 0, ysig, scY, err2Y, asumY, st));
    GemmArgs t = base_args(c, IPR_FP64_CRT, nullptr);
    t.oz_a = c->crC; t.oz_rsig = c->crC_sig; t.oz_b = c->crA; t.oz_csig = ysig;
    t.crt_n = nm; t.crt_v = c->crV; t.crt_dd = 1;
    t.nout = c->T[1]; t.ldn = np; t.zout = ylo; t.ldz = np; t.mode = EPI_STORE_N;
    CK(launch_gemm_crt(t, st));
    CK(launch_cert_split((const double *)c->T[1], ylo, np, np, np, b, nm, c->crC, 0, c->crC_sig, scT, err2T, asumT, st));
    const double *Af = a_f64(c);
    if (!Af) return IPR_E_CUDA;
    CK(launch_cert_split(Af, nullptr, np, np, np, b, nm, c->crA, 0, c->crA_sig, scA, err2A, asumA, st));
  } else {
    // 4. residues of Y's rows (G > 1: the rows S_g into their global slots, then all-gathered)
    CK(launch_cert_split((const double *)c->T[1], ylo, np, kp, np, b, nm, c->crC + col0 * np, np * np, c->crC_sig + col0,
                         scY + col0, err2Y + col0, asumY + col0, st));
    if (sh) {
      for (int l = 0; l < nm; ++l) {
        int8_t *pl = c->crC + (size_t)l * np * np;
        if (!c->comm->allgather(pl + col0 * np, pl, (size_t)(kp * np), st))
          return fail(c, IPR_E_NCCL, "all-gather(Y residues) failed: %s", c->comm->last_error());
      }
      bool ok = c->comm->allgather(c->crC_sig + col0, c->crC_sig, (size_t)kp * 4, st);
      for (double *v : {scY, err2Y, asumY, scA, err2A})
        ok = ok && c->comm->allgather(v + col0, v, (size_t)kp * 8, st);
      if (!ok) return fail(c, IPR_E_NCCL, "all-gather(certificate rows) failed: %s", c->comm->last_error());
    }
  }
  // 5. P = Ltilde Atilde (L = Y for p = 2, T for p = 3; the local columns): residual partials in their global slots
  GemmArgs h = base_args(c, IPR_FP64_CRT, nullptr);
  h.oz_a = c->crC; h.oz_rsig = c->crC_sig; h.oz_b = c->crA; h.oz_csig = c->crA_sig;
  h.crt_n = nm; h.crt_v = c->crV; h.crt_dd = 1; h.mode = EPI_RESID; h.part = c->part;
  CK(launch_gemm_crt(h, st));
  const int64_t tm = tiles_m(c, IPR_FP64_CRT);
  CKS(gather_partials(c, c->part, kp / gemm_tile_n(IPR_FP64_CRT) * tm));
  CK(launch_reduce_sum(c->part, tiles_n_total(c, IPR_FP64_CRT) * tm, c->dscal + 16, st));
  const double *vv[6] = {err2Y, err2A, asumY, scY, scA, scC};
  const int ops[6] = {0, 0, 1, 1, 1, 1};
  CK(launch_cert_stats(vv, ops, 6, np, c->dscal + 17, st));
  if (p3) {
    const double *vt[4] = {err2T, asumT, scT, asumC};
    const int ot[4] = {0, 1, 1, 1};
    CK(launch_cert_stats(vt, ot, 4, np, c->dscal + 24, st));
  }
  CK(cudaMemcpyAsync(c->hcert, c->dscal + 16, 7 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(c->hcert + 7, c->dflag + 2, 4, cudaMemcpyDeviceToHost, st));
  double ht[4] = {0, 0, 0, 0};
  if (p3) CK(cudaMemcpyAsync(ht, c->dscal + 24, 4 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double SR = c->hcert[0], SY = c->hcert[1], SA = c->hcert[2], Yinf = c->hcert[3];
  const double scYm = c->hcert[4], scAm = c->hcert[5], scCm = c->hcert[6];
  int asym = 0;
  memcpy(&asym, c->hcert + 7, 4);
  const double infl = 1.0 + 1e-10, nd = (double)c->n, rec = ldexp(crt_table().p2s1[nm], -48);
  const double eY = nd * rec * scCm * scCm;        // ||Yh - Ct Ct||_F (reconstruction, >= its inf-norm too)
  const double dY = std::sqrt(SY) * infl, dA = std::sqrt(SA) * infl;
  const double A2 = c->norms[0] * infl;
  const double est = std::sqrt(SR);
  double beta, Y2, eP;
  if (!p3) {
    // I - Ct^2 A = (I - P) + (Ytilde - Ct^2) Atilde + Ct^2 (Atilde - A)
    eP = nd * rec * scYm * scAm;
    Y2 = Yinf * infl + eY;                         // ||Ct^2||_2 <= ||Ct^2||_inf (symmetric)
    beta = (dY + eY) * (A2 + dA) + Y2 * dA + eP;
  } else {
    // I - Ct^3 A = (I - P) + (Ttilde - Ct^3) Atilde + Ct^3 (Atilde - A), with Ttilde - Ct^3 =
    // (Ttilde - Th) + (Th - Ct Ytilde) + Ct (Ytilde - Ct^2): E3 = dT + eT + ||Ct||_2 (dY + eY)
    const double dT = std::sqrt(ht[0]) * infl, Tinf = ht[1], scTm = ht[2], C2 = ht[3] * infl;
    const double eT = nd * rec * scCm * scYm;
    eP = nd * rec * scTm * scAm;
    const double E3 = dT + eT + C2 * (dY + eY);
    Y2 = Tinf * infl + std::sqrt(nd) * E3;         // ||Ct^3||_2 <= ||Ct^3||_inf <= ||Th||_inf + sqrt(n) ||T - Ct^3||_F
    beta = E3 * (A2 + dA) + Y2 * dA + eP;
  }
  double bound = (est * infl + beta) * infl;
  if (asym || !std::isfinite(bound)) bound = NAN;   // exponents out of range / an asymmetric candidate
  const double info[10] = {bound, est, beta, dY, dA, A2, Y2, eY, eP, (double)nm};
  memcpy(c->cert_info, info, sizeof info);
  if (std::isnan(bound)) {                         // outside what the bound covers: the FP64 DMMA certificate
    if (sh) {                                      // full64 must hold Ct panel-major again (the gathered C)
      CK(cudaMemcpy2DAsync(c->full64 + (size_t)c->rank * np * kp, (size_t)kp * 8, Ct + col0, (size_t)np * 8,
                           (size_t)kp * 8, (size_t)np, cudaMemcpyDeviceToDevice, st));
      CKS(gather_f64(c, c->full64 + (size_t)c->rank * np * kp));
    }
    CKS(certify_full64(c, rho));
    c->cert_info[0] = *rho;
    return IPR_OK;
  }
  *rho = bound;
  if (i >= 0 && bound <= c->final_tol) {           // the certified Ct is the answer (its local columns)
    CK(cudaMemcpy2DAsync(cont_ptr(c, i, c->ph[c->phase]), (size_t)kp * 8, Ct + col0, (size_t)np * 8, (size_t)kp * 8,
                         (size_t)np, cudaMemcpyDeviceToDevice, st));
  }
  return IPR_OK;
}

// the iterate in buffer i (the candidate C_k), FP64, gathered into full64
static ipr_status certify_iter(ipr_ctx *c, int i, double *rho) {
  const PhaseC &P = c->ph[c->phase];
  if (c->cert == IPR_CERT_CRT && c->world == 1 && P.cont64)   // the FP64 container is already row-major FP64
    return certify_crt(c, i, rho, (const double *)cont_ptr(c, i, P));
  double *slot = c->full64 + (size_t)c->rank * c->npad * c->kp;
  CK(launch_cont_to_f64(cont_ptr(c, i, P), P.cont64, c->npad * c->kp, slot, c->st));
  CKS(gather_f64(c, slot));
  if (c->cert == IPR_CERT_CRT) return certify_crt(c, i, rho);
  return certify_full64(c, rho);
}

static ipr_status certify_best(ipr_ctx *c, double *rho) {
  CKS(copy_iterate(c, 1, nullptr, 0));              // full64 = best (FP64, panel-major)
  if (c->cert == IPR_CERT_CRT) return certify_crt(c, -1, rho);
  return certify_full64(c, rho);
}

ipr_status ipr_residual(ipr_ctx *c, int certify, double *rho) {
  if (!c || !rho) return fail(c, IPR_E_INVALID_ARG, "ipr_residual: null pointer");
  if (!c->started || c->trace.empty()) return fail(c, IPR_E_STATE, "ipr_residual: no iterate evaluated yet");
  if (!certify) { *rho = c->last_rho; return IPR_OK; }
  if (c->grows > 1)   // the literal form's FP64 in-chain residual is already the DMMA literal chain
    return fail(c, IPR_E_UNSUPPORTED, "ipr_residual: certify = 1 on a 2-D grid (use the FP64 phase's in-chain rho)");
  if (certify == 2) {                              // the FP64 DMMA evaluation whatever the mode (R-30)
    CKS(copy_iterate(c, 1, nullptr, 0));
    CKS(certify_full64(c, rho));
  } else {
    CKS(certify_best(c, rho));
  }
  // the certification chain reuses the T buffers: restore the transposed operand it clobbered
  if (c->world > 1 && c->form != IPR_FORM_LITERAL && !c->done) CKS(make_xt(c, c->cur, c->ph[c->phase]));
  return IPR_OK;
}

ipr_status ipr_set_output(ipr_ctx *c, double *C_out, int64_t ldc) {
  if (!c) return fail(c, IPR_E_INVALID_ARG, "ipr_set_output: null context");
  if (C_out && ldc < c->n) return fail(c, IPR_E_INVALID_ARG, "ipr_set_output: ldc < n");
  if (c->out_buf >= 0) CK(cudaStreamSynchronize(c->ost));
  c->out_ptr = C_out; c->out_ld = ldc; c->out_buf = -1; c->out_valid = false;
  return IPR_OK;
}

ipr_status ipr_finalize(ipr_ctx *c, double *C_dev_out, int64_t ldc) {
  if (!c) return fail(c, IPR_E_INVALID_ARG, "ipr_finalize: null context");
  ipr_status s = IPR_OK;
  tl_mark(c, "finalize");
  if (C_dev_out) {
    if (ldc < c->n) s = fail(c, IPR_E_INVALID_ARG, "ipr_finalize: ldc < n");
    else if (!c->started || c->best_loc < 0) s = fail(c, IPR_E_STATE, "ipr_finalize: no iterate evaluated");
    else if (c->out_valid && C_dev_out == c->out_ptr && ldc == c->out_ld) {
      // the certified answer already streamed there during its certificate (ipr_set_output)
      cudaError_t e = cudaStreamWaitEvent(c->st, c->oev, 0);
      if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
      if (e != cudaSuccess) s = fail(c, IPR_E_CUDA, "ipr_finalize: %s", cudaGetErrorString(e));
    } else {
      s = copy_iterate(c, 1, C_dev_out, ldc);
    }
  }
  tl_mark(c, "end");
  tl_report(c);
  if (s != IPR_OK) t_err = c->err;
  free_ctx(c);
  return s;
}

// ---- test hooks (include/ipr_testing.h) ----
int64_t ipr_launch_count(void) { return g_launches; }

ipr_status ipr_test_cert_info(ipr_ctx *c, double *out10) {
  if (!c || !out10) return fail(c, IPR_E_INVALID_ARG, "ipr_test_cert_info: null pointer");
  memcpy(out10, c->cert_info, sizeof c->cert_info);
  return IPR_OK;
}

ipr_status ipr_test_set_guards(int on) {
  g_guards = on ? 1 : 0;
  return IPR_OK;
}

ipr_status ipr_test_check_guards(ipr_ctx *c, int corrupt_first, int *bad) {
  if (!c || !bad) return fail(c, IPR_E_INVALID_ARG, "ipr_test_check_guards: null pointer");
  *bad = -1;
  if (!c->arena || c->guards.empty()) return fail(c, IPR_E_STATE, "ipr_test_check_guards: no guarded arena");
  if (corrupt_first) CK(cudaMemsetAsync((char *)c->arena + c->guards[0] + 17, 0x5A, 1, c->st));   // the control
  std::vector<unsigned char> h(kGuard);
  for (size_t i = 0; i < c->guards.size() && *bad < 0; ++i) {
    CK(cudaMemcpyAsync(h.data(), (char *)c->arena + c->guards[i], kGuard, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (size_t k = 0; k < kGuard; ++k)
      if (h[k] != kGuardByte) { *bad = (int)i; break; }
  }
  return IPR_OK;
}

ipr_status ipr_test_peek(ipr_ctx *c, int what, double *dst, int64_t *npad_out) {
  if (!c || !dst || !npad_out || what < IPR_PEEK_AHAT || what > IPR_PEEK_CHATC)
    return fail(c, IPR_E_INVALID_ARG, "ipr_test_peek: bad arguments");
  if (!c->started || c->trace.empty()) return fail(c, IPR_E_STATE, "ipr_test_peek: no iteration yet");
  const PhaseC &P = c->ph[c->phase];
  if (!is_sym(c) || c->world != 1 || P.prec == IPR_FP64_OZ || fused_sym_ok(c, P))
    return fail(c, IPR_E_UNSUPPORTED, "ipr_test_peek: symmetric forms, G = 1, non-Ozaki-I phases");
  const int prev = 1 - c->cur;              // C_k: the update wrote C_{k+1} into buffer cur
  const int64_t cnt = c->npad * c->npad;
  const void *src = nullptr;
  int prec = P.prec;
  const int *sig = nullptr;
  const bool sc = is_scaled(P.prec), scc = is_scaled(P.corr);
  switch (what) {
    case IPR_PEEK_AHAT: src = c->Aop; sig = sc ? c->dsig + 0 : nullptr; break;
    case IPR_PEEK_CHAT: src = c->chat[prev]; sig = sc ? c->dsig + 1 + prev : nullptr; break;
    case IPR_PEEK_Z1: src = c->T[1]; sig = sc ? c->dsig + 4 : nullptr; break;
    case IPR_PEEK_RHAT: src = c->T[c->p & 1]; prec = P.corr; sig = scc ? c->dsig + 3 + (c->p & 1) : nullptr; break;
    case IPR_PEEK_W: src = c->wbuf; prec = c->wbytes == 8 && P.corr == IPR_FP64 ? IPR_FP64 : -1; break;
    case IPR_PEEK_CHATC:
      if (same_fmt(P.corr, P.prec)) { src = c->chat[prev]; sig = sc ? c->dsig + 1 + prev : nullptr; }
      else { src = c->chatc[prev]; prec = P.corr; }
      break;
  }
  if (is_f64(prec)) prec = IPR_FP64;
  if (c->p != 2 && what == IPR_PEEK_Z1) return fail(c, IPR_E_UNSUPPORTED, "ipr_test_peek: Z1 for p = 2 only");
  CK(launch_peek(src, prec, sig, cnt, dst, c->st));
  CK(cudaStreamSynchronize(c->st));
  *npad_out = c->npad;
  return IPR_OK;
}

ipr_status ipr_plan(int64_t n, int world, int rank, int prec, int64_t *out8) {
  ipr_ctx *c = nullptr;
  if (n <= 0 || world < 1 || rank < 0 || rank >= world || prec < 0 || prec > IPR_INT8 || !out8)
    return fail(c, IPR_E_INVALID_ARG, "ipr_plan: bad arguments");
  const int64_t npad = padded_order(n, world), kp = npad / world, col0 = (int64_t)rank * kp;
  const int64_t tm = gemm_tile_m(prec), tn = gemm_tile_n(prec);
  out8[0] = npad; out8[1] = kp; out8[2] = col0; out8[3] = tm; out8[4] = tn;
  out8[5] = npad / tm; out8[6] = npad / tn; out8[7] = (col0 / tn) * (npad / tm);
  return IPR_OK;
}

ipr_status ipr_test_quantize(int mode, const void *in_dev, void *out_dev, int64_t len, int m, int round, int sigma,
                             void *stream) {
  ipr_ctx *c = nullptr;
  if (mode < 0 || mode > 8 || len < 0 || (len > 0 && (!in_dev || !out_dev)))
    return fail(c, IPR_E_INVALID_ARG, "ipr_test_quantize: bad arguments");
  if ((mode == 0 && (m < 0 || m > 23)) || (mode == 1 && (m < 0 || m > 52)))
    return fail(c, IPR_E_INVALID_ARG, "ipr_test_quantize: bad m");
  cudaStream_t s = (cudaStream_t)stream;
  CK(launch_test_quant(mode, in_dev, out_dev, len, m, round == IPR_RTZ, sigma, s));
  CK(cudaStreamSynchronize(s));
  return IPR_OK;
}

static int g_test_digits = OZ_S;
ipr_status ipr_test_nccl_selftest(void) {
  // the NCCL transport's plumbing on one GPU (NCCL refuses two ranks on one device): dlopen + symbol
  // binding, a 1-rank communicator, in-place all-gather, grouped send / recv all-to-all, split
  ipr_ctx *c = nullptr;
  std::string e;
  unsigned char uid[128];
  if (!NcclComm::unique_id(uid, &e)) return fail(c, IPR_E_NCCL, "nccl selftest: unique id: %s", e.c_str());
  NcclComm comm;
  if (!comm.init(1, 0, uid, &e)) return fail(c, IPR_E_NCCL, "nccl selftest: %s", e.c_str());
  const size_t nb = 1 << 16;
  std::vector<unsigned char> h(3 * nb), back(3 * nb);
  for (size_t i = 0; i < nb; ++i) h[i] = (unsigned char)(i * 131 + 7);
  unsigned char *d = nullptr;
  cudaStream_t st = nullptr;
  if (cudaMalloc((void **)&d, 3 * nb) != cudaSuccess || cudaStreamCreate(&st) != cudaSuccess)
    return fail(c, IPR_E_CUDA, "nccl selftest: %s", cudaGetErrorString(cudaGetLastError()));
  ipr_status s = IPR_OK;
  cudaMemset(d, 0, 3 * nb);
  cudaMemcpy(d, h.data(), nb, cudaMemcpyHostToDevice);
  Transport *sub = nullptr;
  if (!comm.allgather(d, d, nb, st)) s = fail(c, IPR_E_NCCL, "nccl selftest: all-gather: %s", comm.last_error());
  else if (!comm.alltoall(d, d + nb, nb, st)) s = fail(c, IPR_E_NCCL, "nccl selftest: all-to-all: %s", comm.last_error());
  else if (!(sub = comm.split(0, 0, &e))) s = fail(c, IPR_E_NCCL, "nccl selftest: split: %s", e.c_str());
  else if (!sub->allgather(d + nb, d + 2 * nb, nb, st))
    s = fail(c, IPR_E_NCCL, "nccl selftest: split all-gather: %s", sub->last_error());
  if (s == IPR_OK && cudaStreamSynchronize(st) == cudaSuccess &&
      cudaMemcpy(back.data(), d, 3 * nb, cudaMemcpyDeviceToHost) == cudaSuccess) {
    for (size_t i = 0; i < 3 * nb && s == IPR_OK; ++i)
      if (back[i] != h[i % nb]) s = fail(c, IPR_E_NCCL, "nccl selftest: byte %zu is %d, expected %d", i, back[i], h[i % nb]);
  } else if (s == IPR_OK) {
    s = fail(c, IPR_E_CUDA, "nccl selftest: %s", cudaGetErrorString(cudaGetLastError()));
  }
  delete sub;
  cudaStreamDestroy(st);
  cudaFree(d);
  return s;
}

ipr_status ipr_test_crt_signed(int on) {
  crt_force_signed(on);
  return IPR_OK;
}

ipr_status ipr_test_set_digits(int digits) {
  ipr_ctx *c = nullptr;
  if (digits < 2 || digits > OZ_S) return fail(c, IPR_E_INVALID_ARG, "ipr_test_set_digits: digits in [2, 9]");
  g_test_digits = digits;
  return IPR_OK;
}

ipr_status ipr_test_crt_table(int N, int b, int64_t n, int *out40, double *dout64, int *n_for, int *b_for) {
  ipr_ctx *c = nullptr;
  if (N < 1 || N > CRT_MAX || !out40 || !dout64 || !n_for || !b_for)
    return fail(c, IPR_E_INVALID_ARG, "ipr_test_crt_table: bad arguments");
  const CrtTab &t = crt_table();
  for (int l = 0; l < CRT_MAX; ++l) {
    out40[l] = l < N ? t.m[l] : 0;
    out40[20 + l] = l < N ? t.inv[N][l] : 0;
    dout64[3 * l] = l < N ? t.H[N][l] : 0.0;
    dout64[3 * l + 1] = l < N ? t.L[N][l] : 0.0;
    dout64[3 * l + 2] = l < N ? t.R[N][l] : 0.0;
  }
  dout64[54] = t.MH[N]; dout64[55] = t.ML[N]; dout64[56] = t.MR[N];
  dout64[57] = t.p2s1[N]; dout64[58] = t.p2s2[N];
  *n_for = (b >= 2 && b <= CRT_BMAX && n >= 1) ? crt_moduli(b, n) : -1;
  *b_for = (b >= 2 && b <= OZ_S && n >= 1) ? crt_bits(b, n) : 0;
  return IPR_OK;
}

// CRT operands of a test / bench product: residue planes of X (rows) and of Yt's rows
static cudaError_t crt_test_setup(GemmArgs &g, const void *X, const void *Y, int64_t np, int64_t n, int8_t **oa,
                                  int8_t **ob, int **sig, uint8_t **v, cudaStream_t s, bool split_y) {
  const int b = crt_bits(g_test_digits, n), nm = crt_moduli(b, n);
  if (nm < 0) return cudaErrorInvalidValue;
  cudaError_t e = cudaMalloc((void **)oa, (size_t)(np * np) * nm);
  if (e == cudaSuccess) e = cudaMalloc((void **)ob, (size_t)(np * np) * nm);
  if (e == cudaSuccess) e = cudaMalloc((void **)sig, (size_t)np * 8);
  if (e == cudaSuccess) e = cudaMalloc((void **)v, (size_t)(np * np) * nm);
  if (e == cudaSuccess) e = launch_crt_split((const double *)X, np, np, np, b, nm, *oa, *sig, s);
  if (e == cudaSuccess && split_y) e = launch_crt_split((const double *)Y, np, np, np, b, nm, *ob, *sig + np, s);
  g.oz_a = *oa; g.oz_rsig = *sig; g.oz_b = *ob; g.oz_csig = *sig + np; g.crt_n = nm; g.crt_v = *v;
  g.oz_S = g_test_digits;
  return e;
}

ipr_status ipr_test_gemm(int prec, int64_t n, const void *X_dev, const void *Yt_dev, double *Z_dev, void *stream) {
  ipr_ctx *c = nullptr;
  if (n <= 0 || !X_dev || !Yt_dev || !Z_dev || prec < 0 || prec > IPR_FP64_CRT)
    return fail(c, IPR_E_INVALID_ARG, "ipr_test_gemm: bad arguments");
  if (!is_f64(prec) && !tc_supported(prec))
    return fail(c, IPR_E_UNSUPPORTED, "ipr_test_gemm: tcgen05 path for this precision is not built");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t unit = prec == IPR_FP64 ? 128 : 256;
  const int64_t np = (n + unit - 1) / unit * unit;
  const int esz = elt_size(prec);
  void *X = nullptr, *Y = nullptr;
  double *Z = nullptr;
  CK(cudaMalloc(&X, (size_t)(np * np) * esz));
  CK(cudaMalloc(&Y, (size_t)(np * np) * esz));
  CK(cudaMalloc(&Z, (size_t)(np * np) * 8));
  CK(launch_pad_copy(X_dev, n, np, esz, X, s));
  CK(launch_pad_copy(Yt_dev, n, np, esz, Y, s));
  GemmArgs g;
  memset(&g, 0, sizeof g);
  g.M = np; g.N = np; g.K = np; g.n = n; g.col0 = 0;
  g.A = X; g.a_kp = np; g.a_pstride = np * np;
  g.B = Y; g.ldb = np; g.prec = prec; g.mode = EPI_F64;
  g.zout = Z; g.ldz = np; g.tiles_m = np / gemm_tile_m(prec);
  cudaError_t e = cudaSuccess;
  int8_t *oa = nullptr, *ob = nullptr;
  int *sig = nullptr;
  double *acc = nullptr;
  uint8_t *cv = nullptr;
  if (prec == IPR_FP64_OZ) {   // Ozaki digits of X (A role, rows) and of Yt's rows (B role)
    e = cudaMalloc(&oa, (size_t)(np * np) * OZ_S);
    if (e == cudaSuccess) e = cudaMalloc(&ob, (size_t)(np * np) * OZ_S);
    if (e == cudaSuccess) e = cudaMalloc(&sig, (size_t)np * 8);
    if (e == cudaSuccess) e = cudaMalloc(&acc, (size_t)(np * np) * 8);
    if (e == cudaSuccess) e = launch_oz_split((const double *)X, np, np, np, OZ_S, oa, nullptr, sig, s);
    if (e == cudaSuccess) e = launch_oz_split((const double *)Y, np, np, np, OZ_S, nullptr, ob, sig + np, s);
    g.oz_a = oa; g.oz_rsig = sig; g.oz_b = ob; g.oz_csig = sig + np; g.ozacc = acc; g.ldoz = np; g.oz_S = g_test_digits;
    if (e == cudaSuccess) e = launch_gemm_ozaki(g, s);
  } else if (prec == IPR_FP64_CRT) {
    e = crt_test_setup(g, X, Y, np, n, &oa, &ob, &sig, &cv, s, true);
    if (e == cudaSuccess) e = launch_gemm_crt(g, s);
  } else {
    e = prec == IPR_FP64 ? launch_gemm_dmma(g, s) : launch_gemm_tc(g, s);
  }
  if (e == cudaSuccess) e = launch_unpad_f64(Z, n, np, Z_dev, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(X); cudaFree(Y); cudaFree(Z); cudaFree(oa); cudaFree(ob); cudaFree(sig); cudaFree(acc); cudaFree(cv);
  if (e != cudaSuccess) return fail(c, IPR_E_CUDA, "ipr_test_gemm: %s %s", cudaGetErrorString(e), tc_last_error());
  return IPR_OK;
}

ipr_status ipr_bench_gemm(int prec, int64_t n, int warmup, int iters, void *stream, double *ms) {
  return ipr_bench_gemm_epi(prec, n, warmup, iters, 0, stream, ms);
}

ipr_status ipr_bench_gemm_epi(int prec, int64_t n, int warmup, int iters, int epi, void *stream, double *ms) {
  ipr_ctx *c = nullptr;
  if (n <= 0 || prec < 0 || prec > IPR_FP64_CRT || warmup < 0 || iters <= 0 || !ms || epi < 0 || epi > 3)
    return fail(c, IPR_E_INVALID_ARG, "ipr_bench_gemm: bad arguments");
  if (!is_f64(prec) && !tc_supported(prec))
    return fail(c, IPR_E_UNSUPPORTED, "ipr_bench_gemm: tcgen05 path for this precision is not built");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t unit = prec == IPR_FP64 ? 128 : 256;
  const int64_t np = (n + unit - 1) / unit * unit;
  const size_t bytes = (size_t)(np * np) * elt_size(prec);
  void *X = nullptr, *Y = nullptr, *T = nullptr;
  float *pm = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // scaled formats: the chain GEMM's epilogue is the FP32 scratch + per-tile max (EPI_TSCRATCH)
  const bool scaled = is_scaled(prec);
  cudaError_t e = cudaMalloc(&X, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&Y, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&T, (size_t)(np * np) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&pm, (size_t)(np / 128) * (np / 64) * 4 + 4096);
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  if (e == cudaSuccess) e = launch_fill_operand(X, np * np, prec, 0x1234u, s);
  if (e == cudaSuccess) e = launch_fill_operand(Y, np * np, prec, 0x9876u, s);
  GemmArgs g;
  memset(&g, 0, sizeof g);
  g.M = np; g.N = np; g.K = np; g.n = n; g.col0 = 0;
  g.A = X; g.a_kp = np; g.a_pstride = np * np;
  const int mode = epi == 1 ? 0 : epi == 2 ? EPI_STORE_T : epi == 3 ? EPI_TSCRATCH : scaled ? EPI_TSCRATCH : EPI_STORE_T;
  g.B = Y; g.ldb = np; g.prec = prec; g.tprec = prec; g.mode = mode;
  g.tout = T; g.ldt = np; g.tiles_m = np / gemm_tile_m(prec);
  if (mode == EPI_TSCRATCH) g.pmax = pm;
  // Ozaki: the left operand's digits once (amortised over an iteration's GEMMs), the right
  // operand's split inside every timed launch (one split per GEMM, as in the hot path)
  int8_t *oa = nullptr, *ob = nullptr;
  int *sig = nullptr;
  double *acc = nullptr;
  uint8_t *cv = nullptr;
  if (prec == IPR_FP64_CRT) {
    if (e == cudaSuccess) e = crt_test_setup(g, X, Y, np, n, &oa, &ob, &sig, &cv, s, false);
    g.mode = mode ? EPI_STORE_T : 0;
  }
  if (prec == IPR_FP64_OZ) {
    if (e == cudaSuccess) e = cudaMalloc(&oa, (size_t)(np * np) * OZ_S);
    if (e == cudaSuccess) e = cudaMalloc(&ob, (size_t)(np * np) * OZ_S);
    if (e == cudaSuccess) e = cudaMalloc(&sig, (size_t)np * 8);
    if (e == cudaSuccess) e = cudaMalloc(&acc, (size_t)(np * np) * 8);
    if (e == cudaSuccess) e = launch_oz_split((const double *)X, np, np, np, OZ_S, oa, nullptr, sig, s);
    g.oz_a = oa; g.oz_rsig = sig; g.oz_b = ob; g.oz_csig = sig + np; g.ozacc = acc; g.ldoz = np; g.oz_S = g_test_digits;
    g.mode = mode ? EPI_STORE_T : 0;
  }
  auto run = [&]() {
    if (prec == IPR_FP64_OZ) {
      cudaError_t r = launch_oz_split((const double *)Y, np, np, np, OZ_S, nullptr, ob, sig + np, s);
      return r == cudaSuccess ? launch_gemm_ozaki(g, s) : r;
    }
    if (prec == IPR_FP64_CRT) {
      cudaError_t r = launch_crt_split((const double *)Y, np, np, np, crt_bits(g_test_digits, n), g.crt_n, ob, sig + np, s);
      return r == cudaSuccess ? launch_gemm_crt(g, s) : r;
    }
    return prec == IPR_FP64 ? launch_gemm_dmma(g, s) : launch_gemm_tc(g, s);
  };
  for (int i = 0; i < warmup && e == cudaSuccess; ++i) e = run();
  if (e == cudaSuccess) e = cudaEventRecord(e0, s);
  for (int i = 0; i < iters && e == cudaSuccess; ++i) e = run();
  if (e == cudaSuccess) e = cudaEventRecord(e1, s);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float t = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&t, e0, e1);
  if (e == cudaSuccess) *ms = (double)t / iters;
  cudaFree(X); cudaFree(Y); cudaFree(T); cudaFree(pm); cudaFree(oa); cudaFree(ob); cudaFree(sig); cudaFree(acc); cudaFree(cv);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e != cudaSuccess) return fail(c, IPR_E_CUDA, "ipr_bench_gemm: %s %s", cudaGetErrorString(e), tc_last_error());
  return IPR_OK;
}

}  // extern "C"
