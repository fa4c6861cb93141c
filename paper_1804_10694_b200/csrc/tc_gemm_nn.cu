// tc_gemm_nn.cu -- instantiates the 3xTF32 tensor-core GEMM for op(A) = A, op(B) = B.
#include "tc_gemm.cuh"

namespace tmk {
template tm_status launch_tc_op<false, false>(const GemmArgs&, const TcChoice&, int, cudaStream_t);
}  // namespace tmk
