// tcgen05 3xTF32 engine (placeholder until the kernel lands; never selected).
#include "gemm.cuh"

namespace enks {

bool tc_gemm_applicable(int, int, int64_t, int64_t, int64_t, const float*, int64_t, const float*,
                        int64_t, int64_t) {
    return false;
}

int gemm_tc(int64_t, int64_t, int64_t, float, const float*, int64_t, const float*, int64_t, float,
            const float*, int64_t, const float*, int64_t, int, float*, int64_t, int, void*,
            cudaStream_t) {
    set_error("enks_gemm: tcgen05 engine not available in this build");
    return ENKS_E_UNSUPPORTED;
}

}  // namespace enks
