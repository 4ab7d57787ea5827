// gemm_tc.cu -- tcgen05 (kind::tf32, 3xTF32) grouped GEMM.  Placeholder until the tensor-core
// path lands: no descriptor is routed here yet.
#include "internal.cuh"

namespace kfac {

bool gemm_tc_supported(const GemmDesc &) { return false; }

kfac_status_t gemm_tc_grouped(const GemmDesc *, int, float, cudaStream_t) {
    set_error("tcgen05 GEMM not built");
    return KFAC_ERR_UNSUPPORTED;
}

}  // namespace kfac
