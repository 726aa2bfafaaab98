// K8: gain solve.  Sy = scale * sym(S); Cholesky with the reference's jitter
// fallback; Sy^{-1} = L^{-T} L^{-1} written densely for the gain GEMM.
//
// Reference: enks.py:234-235 (symmetrize), 238-244 (cho_factor, jitter
// 1e-9 * tr/p + 1e-30 on LinAlgError, jitter_events += 1), 246 (cho_solve).
// LAPACK dpotrf reports failure when a pivot is <= 0 or NaN; the same test
// is applied here.  One CTA of 1024 threads holds the packed lower triangle
// in shared memory (p(p+1)/2 floats; p <= 336 fits the 227 KB opt-in), so the
// factorisation, the in-place triangular inverse and L^{-T} L^{-1} never
// leave the SM and no host synchronisation is needed: failure is reported
// through device-side status / jitter counters.
#include "common.cuh"
#include "gemm.cuh"

namespace enks {
namespace {

constexpr int kThreads = 1024;
constexpr int kMaxP = 336;

__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }

__global__ void __launch_bounds__(kThreads)
    spd_inverse_kernel(const float* __restrict__ S, int64_t lds, int p, float scale,
                       float* __restrict__ linv, int* status, int* jitter_events) {
    extern __shared__ float L[];
    __shared__ float s_inv_piv;
    __shared__ int s_fail;
    __shared__ double s_trace;
    __shared__ float s_x[kMaxP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kThreads / 32;

    if (tid == 0) {
        double tr = 0.0;
        for (int i = 0; i < p; ++i) tr += (double)(scale * S[(int64_t)i * lds + i]);
        s_trace = tr;
    }
    __syncthreads();

    int failed = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const float jitter =
            attempt == 0 ? 0.f : (float)(1e-9 * s_trace / (double)p + 1e-30);
        for (int e = tid; e < p * p; e += kThreads) {
            const int i = e / p, j = e - i * p;
            if (j <= i) {
                float v = scale * (0.5f * (S[(int64_t)i * lds + j] + S[(int64_t)j * lds + i]));
                if (i == j) v += jitter;
                L[pk(i, j)] = v;
            }
        }
        if (tid == 0) s_fail = 0;
        __syncthreads();
        for (int k = 0; k < p; ++k) {
            if (tid == 0) {
                const float a = L[pk(k, k)];
                if (!(a > 0.f)) {
                    s_fail = 1;
                } else {
                    const float d = sqrtf(a);
                    L[pk(k, k)] = d;
                    s_inv_piv = 1.f / d;
                }
            }
            __syncthreads();
            if (s_fail) break;
            const float ip = s_inv_piv;
            for (int i = k + 1 + tid; i < p; i += kThreads) L[pk(i, k)] *= ip;
            __syncthreads();
            for (int i = k + 1 + warp; i < p; i += nwarps) {
                const float lik = L[pk(i, k)];
                const int base_i = pk(i, 0);
                for (int j = k + 1 + lane; j <= i; j += 32) L[base_i + j] -= lik * L[pk(j, k)];
            }
            __syncthreads();
        }
        failed = s_fail;
        __syncthreads();
        if (!failed) break;
        if (attempt == 0 && tid == 0) atomicAdd(jitter_events, 1);
    }
    if (failed) {
        if (tid == 0) *status = 1;
        const float nan = __int_as_float(0x7fc00000);
        for (int e = tid; e < p * p; e += kThreads) linv[e] = nan;
        return;
    }

    // in-place inverse of the lower-triangular factor (LAPACK dtrti2, lower, non-unit)
    for (int j = p - 1; j >= 0; --j) {
        if (tid == 0) {
            const float d = 1.f / L[pk(j, j)];
            L[pk(j, j)] = d;
            s_inv_piv = -d;
        }
        for (int i = j + 1 + tid; i < p; i += kThreads) s_x[i] = L[pk(i, j)];
        __syncthreads();
        // L[j+1:, j] = -Linv_jj * (Linv[j+1:, j+1:] @ x)
        const float aj = s_inv_piv;
        for (int i = j + 1 + warp; i < p; i += nwarps) {
            float acc = 0.f;
            const int base_i = pk(i, 0);
            for (int k = j + 1 + lane; k <= i; k += 32) acc += L[base_i + k] * s_x[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) L[pk(i, j)] = aj * acc;
        }
        __syncthreads();
    }
    // dense L^{-1} (zeros above the diagonal) for the L^{-T} L^{-1} product (enks_gemm)
    for (int e = tid; e < p * p; e += kThreads) {
        const int i = e / p, j = e - i * p;
        linv[e] = j <= i ? L[pk(i, j)] : 0.f;
    }
}

}  // namespace
}  // namespace enks

extern "C" {

int enks_spd_max_p(void) { return enks::kMaxP; }

int enks_spd_inverse(const float* S, int64_t lds, int p, float scale, float* inv, float* ws,
                     int* status, int* jitter_events, void* stream) {
    ENKS_REQUIRE(S && inv && ws && status && jitter_events, "enks_spd_inverse: null pointer");
    ENKS_REQUIRE(p >= 1 && p <= enks::kMaxP, "enks_spd_inverse: p=%d outside [1, %d]", p,
                 enks::kMaxP);
    const size_t smem = (size_t)p * (p + 1) / 2 * sizeof(float);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(enks::spd_inverse_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) {
            enks::set_error("enks_spd_inverse: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = smem;
    }
    cudaStream_t st = enks::as_stream(stream);
    enks::spd_inverse_kernel<<<1, enks::kThreads, smem, st>>>(S, lds, p, scale, ws, status,
                                                              jitter_events);
    int rc = enks::check_launch("enks_spd_inverse");
    if (rc) return rc;
    // Sy^{-1} = L^{-T} L^{-1}: one small GEMM (A = L^{-1} read transposed)
    return enks::gemm_simt(1, 0, p, p, p, 1.f, ws, p, ws, p, 0.f, nullptr, 0, nullptr, 0, 1, inv,
                           p, 0, 0, 1, nullptr, st);
}

}  // extern "C"
