// gemm_tc.cu -- tcgen05 (TMEM/TMA) GEMM for BF16 / FP16 / TF32 phases.  (placeholder until the
// tcgen05 kernel lands: every low-precision phase returns IPR_E_UNSUPPORTED, never a CPU path)
#include "common.cuh"
namespace ipr {
bool tc_supported(int) { return false; }
int gemm_tile_n(int prec) { return 128; }
int gemm_tile_m(int prec) { return 128; }
cudaError_t launch_gemm_tc(const GemmArgs &, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace ipr
