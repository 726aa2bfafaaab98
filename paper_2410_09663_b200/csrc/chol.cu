// K8: gain solve.  Sy = scale * sym(S); Cholesky with the reference's jitter
// fallback; Sy^{-1} = L^{-T} L^{-1} written densely for the gain GEMM.
//
// Reference: enks.py:234-235 (symmetrize), 238-244 (cho_factor, jitter
// 1e-9 * tr/p + 1e-30 on LinAlgError, jitter_events += 1), 246 (cho_solve).
// LAPACK dpotrf reports failure when a pivot is <= 0 or NaN; the same test is
// applied here, and failure is reported through device-side status / jitter
// counters (no host synchronisation).
//
// One CTA of 1024 threads keeps the lower tile-triangle of the matrix in
// shared memory as 32x33 fp32 tiles (p <= 288).  Right-looking blocked
// Cholesky: one warp factors the diagonal tile in registers with shuffles,
// warps solve the panel tiles (lane = row), and the trailing SYRK/GEMM tile
// updates run one warp per tile (lane = column, conflict-free 33-float
// stride).  L^{-1} is formed tile-row by tile-row the same way and stored
// densely; L^{-T} L^{-1} is one small GEMM.
#include "common.cuh"
#include "gemm.cuh"

namespace enks {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kTS = 32;              // tile size
constexpr int kLd = 33;              // padded tile row stride (floats)
constexpr int kTile = kTS * kLd;     // floats per tile
constexpr int kMaxNB = 9;            // p <= 288
constexpr int kMaxP = kMaxNB * kTS;

__device__ __forceinline__ int tix(int I, int J) { return I * (I + 1) / 2 + J; }

// warp-level Cholesky of one 32x32 SPD tile in place; returns false on a bad pivot
__device__ bool factor_diag(float* T, int lane) {
    float a[kTS];
#pragma unroll
    for (int j = 0; j < kTS; ++j) a[j] = T[lane * kLd + j];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < kTS; ++k) {
        const float piv = __shfl_sync(0xffffffffu, a[k], k);
        if (!(piv > 0.f)) ok = false;
        const float d = sqrtf(piv);
        const float inv = 1.f / d;
        if (lane == k) a[k] = d;
        if (lane > k) a[k] *= inv;
        // trailing: a[i][j] -= l_ik l_jk for k < j <= i
#pragma unroll
        for (int j = k + 1; j < kTS; ++j) {
            const float ljk = __shfl_sync(0xffffffffu, a[k], j);
            if (lane >= j) a[j] = fmaf(-a[k], ljk, a[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < kTS; ++j) T[lane * kLd + j] = (j <= lane) ? a[j] : 0.f;
    return ok;
}

// X <- X L^{-T} for a 32x32 panel tile X and lower-triangular tile L (lane = row of X)
__device__ void panel_solve(float* X, const float* L, int lane) {
    float x[kTS];
#pragma unroll
    for (int j = 0; j < kTS; ++j) x[j] = X[lane * kLd + j];
#pragma unroll
    for (int j = 0; j < kTS; ++j) {
        float v = x[j];
#pragma unroll
        for (int k = 0; k < j; ++k) v = fmaf(-x[k], L[j * kLd + k], v);
        x[j] = v / L[j * kLd + j];
    }
#pragma unroll
    for (int j = 0; j < kTS; ++j) X[lane * kLd + j] = x[j];
}

// C <- C - A B^T (32x32x32), lane = column of C
__device__ void tile_syrk_sub(float* C, const float* A, const float* B, int lane) {
    float b[kTS];
#pragma unroll
    for (int k = 0; k < kTS; ++k) b[k] = B[lane * kLd + k];
    for (int r = 0; r < kTS; ++r) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < kTS; ++k) acc = fmaf(A[r * kLd + k], b[k], acc);
        C[r * kLd + lane] -= acc;
    }
}

// in-place inverse of a lower-triangular 32x32 tile (warp; lane = column of the inverse)
__device__ void invert_diag(float* T, int lane) {
    // column `lane` of L^{-1}: forward substitution L y = e_lane
    float y[kTS];
#pragma unroll
    for (int i = 0; i < kTS; ++i) {
        float v = (i == lane) ? 1.f : 0.f;
#pragma unroll
        for (int k = 0; k < i; ++k) v = fmaf(-T[i * kLd + k], y[k], v);
        y[i] = (i < lane) ? 0.f : v / T[i * kLd + i];
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kTS; ++i) T[i * kLd + lane] = y[i];
    __syncwarp();
}

__global__ void __launch_bounds__(kThreads)
    spd_inverse_kernel(const float* __restrict__ S, int64_t lds, int p, float scale,
                       float* __restrict__ linv, int* status, int* jitter_events) {
    extern __shared__ float sm[];
    float* Lt = sm;                           // lower tile-triangle of L
    __shared__ int s_fail;
    __shared__ double s_trace_part[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = (p + kTS - 1) / kTS;
    const int P = nb * kTS;
    const int n_tiles = nb * (nb + 1) / 2;

    {   // trace (parallel, fp64)
        double t = 0.0;
        for (int i = tid; i < p; i += kThreads) t += (double)(scale * S[(int64_t)i * lds + i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) s_trace_part[warp] = t;
    }
    __syncthreads();
    double trace = 0.0;
    for (int w = 0; w < kWarps; ++w) trace += s_trace_part[w];

    int failed = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const float jitter = attempt == 0 ? 0.f : (float)(1e-9 * trace / (double)p + 1e-30);
        // load sym(S) (+ jitter I); padding rows/cols = identity
        for (int e = tid; e < P * P; e += kThreads) {
            const int i = e / P, j = e - i * P;
            if (j > i) continue;
            float v;
            if (i < p && j < p)
                v = scale * (0.5f * (S[(int64_t)i * lds + j] + S[(int64_t)j * lds + i])) +
                    (i == j ? jitter : 0.f);
            else
                v = (i == j) ? 1.f : 0.f;
            Lt[tix(i / kTS, j / kTS) * kTile + (i % kTS) * kLd + (j % kTS)] = v;
        }
        if (tid == 0) s_fail = 0;
        __syncthreads();
        for (int K = 0; K < nb; ++K) {
            if (warp == 0) {
                const bool ok = factor_diag(Lt + tix(K, K) * kTile, lane);
                if (lane == 0 && !ok) s_fail = 1;
            }
            __syncthreads();
            if (s_fail) break;
            for (int I = K + 1 + warp; I < nb; I += kWarps)
                panel_solve(Lt + tix(I, K) * kTile, Lt + tix(K, K) * kTile, lane);
            __syncthreads();
            // trailing update of tiles (I, J), K < J <= I
            const int m = nb - K - 1;
            for (int q = warp; q < m * (m + 1) / 2; q += kWarps) {
                int I = 0;
                while ((I + 1) * (I + 2) / 2 <= q) ++I;
                const int J = q - I * (I + 1) / 2;
                const int gI = K + 1 + I, gJ = K + 1 + J;
                tile_syrk_sub(Lt + tix(gI, gJ) * kTile, Lt + tix(gI, K) * kTile,
                              Lt + tix(gJ, K) * kTile, lane);
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

    // L^{-1}, tile row by tile row: Linv_II = L_II^{-1};
    // Linv_IJ = -Linv_II * sum_{K=J}^{I-1} L_IK Linv_KJ   (J < I), written over L_IJ.
    // Row I needs Linv tiles of rows < I (already inverted) and L_IK (K < I, still L).
    for (int I = 0; I < nb; ++I) {
        if (warp == 0) invert_diag(Lt + tix(I, I) * kTile, lane);
        __syncthreads();
        // for each J < I (one warp per J): acc = sum_K L_IK Linv_KJ, then Linv_IJ = -Linv_II acc.
        // L_IK for K >= J are read before any warp overwrites them?  Warp J writes tile (I, J)
        // only, and reads (I, K) for K >= J: tiles (I, K > J) are written by other warps, so
        // stage the products in registers and write after a barrier.
        float res[kTS];
        const bool active = warp < I;
        if (active) {
            const int J = warp;
#pragma unroll
            for (int r = 0; r < kTS; ++r) res[r] = 0.f;
            for (int K = J; K < I; ++K) {
                const float* A = Lt + tix(I, K) * kTile;  // L_IK
                const float* B = Lt + tix(K, J) * kTile;  // Linv_KJ (K == J: Linv_JJ)
                float b[kTS];  // column `lane` of B
#pragma unroll
                for (int k = 0; k < kTS; ++k) b[k] = B[k * kLd + lane];
#pragma unroll 4
                for (int r = 0; r < kTS; ++r) {
                    float acc = 0.f;
#pragma unroll
                    for (int k = 0; k < kTS; ++k) acc = fmaf(A[r * kLd + k], b[k], acc);
                    res[r] += acc;
                }
            }
        }
        __syncthreads();
        if (active) {
            const int J = warp;
            float* out = Lt + tix(I, J) * kTile;
            const float* D = Lt + tix(I, I) * kTile;  // Linv_II
#pragma unroll
            for (int r = 0; r < kTS; ++r) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k <= r; ++k) acc = fmaf(D[r * kLd + k], res[k], acc);
                out[r * kLd + lane] = -acc;
            }
        }
        __syncthreads();
    }
    // dense L^{-1} (zeros above the diagonal, p x p)
    for (int e = tid; e < p * p; e += kThreads) {
        const int i = e / p, j = e - i * p;
        linv[e] = (j <= i) ? Lt[tix(i / kTS, j / kTS) * kTile + (i % kTS) * kLd + (j % kTS)] : 0.f;
    }
    (void)n_tiles;
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
    const int nb = (p + enks::kTS - 1) / enks::kTS;
    const size_t smem = (size_t)nb * (nb + 1) / 2 * enks::kTile * sizeof(float);
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
