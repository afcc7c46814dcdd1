// tt_launch_l2.cu — GEMM launchers for operand layout (A M-contiguous, B K-contiguous).
#include "tt_launch_tpl.cuh"

namespace ttint {
template cudaError_t launch_layout<false, true>(const GemmParams&, cudaStream_t);
}  // namespace ttint
