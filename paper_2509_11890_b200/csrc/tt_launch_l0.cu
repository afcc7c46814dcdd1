// tt_launch_l0.cu — GEMM launchers for operand layout (A K-contiguous, B K-contiguous).
#include "tt_launch_tpl.cuh"

namespace ttint {
template cudaError_t launch_layout<true, true>(const GemmParams&, cudaStream_t);
}  // namespace ttint
