// tt_launch_l3.cu — GEMM launchers for operand layout (A M-contiguous, B N-contiguous).
#include "tt_launch_tpl.cuh"

namespace ttint {
template cudaError_t launch_layout<false, false>(const GemmParams&, cudaStream_t);
}  // namespace ttint
