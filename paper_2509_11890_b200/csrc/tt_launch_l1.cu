// tt_launch_l1.cu — GEMM launchers for operand layout (A K-contiguous, B N-contiguous).
#include "tt_launch_tpl.cuh"

namespace ttint {
template cudaError_t launch_layout<true, false>(const GemmParams&, cudaStream_t);
}  // namespace ttint
