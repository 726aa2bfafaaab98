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
#include <stdlib.h>

#include "common.cuh"
#include "gemm.cuh"

namespace enks {
namespace {

constexpr int kThreads = 512;
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
        for (int j = 1; j < kTS; ++j) {
            if (j > k) {  // constant trip count: full unroll keeps a[] in registers
                const float ljk = __shfl_sync(0xffffffffu, a[k], j);
                if (lane >= j) a[j] = fmaf(-a[k], ljk, a[j]);
            }
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
                       float* __restrict__ linv, int* status, int* jitter_events, int debug) {
    extern __shared__ float sm[];
    float* Lt = sm;                           // lower tile-triangle of L
    __shared__ int s_fail;
    __shared__ double s_trace_part[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = (p + kTS - 1) / kTS;
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
        // load sym(S) (+ jitter I) tile by tile with coalesced rows: tile (I, J) gets
        // 0.5 scale S[I-block][J-block] row-wise, then += 0.5 scale S[J-block][I-block]^T
        // (also read row-wise, written transposed: stride 33 keeps it conflict-free);
        // padding rows/cols = identity
        for (int q = warp; q < n_tiles; q += kWarps) {
            int I = 0;
            while ((I + 1) * (I + 2) / 2 <= q) ++I;
            const int J = q - I * (I + 1) / 2;
            float* T = Lt + q * kTile;
            const float hs = 0.5f * scale;
            const int cj = J * kTS + lane, ci = I * kTS + lane;
            for (int r = 0; r < kTS; ++r) {
                const int ri = I * kTS + r;
                T[r * kLd + lane] = (ri < p && cj < p) ? hs * S[(int64_t)ri * lds + cj] : 0.f;
            }
            __syncwarp();
            for (int r = 0; r < kTS; ++r) {
                const int rj = J * kTS + r;
                const float v = (rj < p && ci < p) ? hs * S[(int64_t)rj * lds + ci] : 0.f;
                T[lane * kLd + r] += v;  // element (I*32 + lane, J*32 + r)
            }
            __syncwarp();
            if (I == J) {
                const int gi = I * kTS + lane;
                T[lane * kLd + lane] = gi < p ? T[lane * kLd + lane] + jitter : 1.f;
            }
        }
        __syncthreads();
        if (tid == 0) s_fail = 0;
        __syncthreads();
        for (int K = 0; K < ((debug & 2) ? 0 : nb); ++K) {
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
    for (int I = 0; I < ((debug & 1) ? 0 : nb); ++I) {
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
#pragma unroll
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
    // dense L^{-1} (zeros above the diagonal, p x p), tile rows written coalesced
    for (int q = warp; q < nb * nb; q += kWarps) {
        const int I = q / nb, J = q - (q / nb) * nb;
        const int c = J * kTS + lane;
        for (int r = 0; r < kTS; ++r) {
            const int i = I * kTS + r;
            if (i >= p || c >= p) continue;
            linv[(int64_t)i * p + c] = (J < I || (J == I && lane <= r))
                                           ? Lt[tix(I, J) * kTile + r * kLd + lane] : 0.f;
        }
    }
    (void)n_tiles;
}

// inv = L^{-T} L^{-1}: inv[i][j] = sum_{k >= max(i, j)} Linv[k][i] Linv[k][j]; one CTA per
// 32 x 32 output tile, K staged through shared memory in 32-row slabs (coalesced rows)
__global__ void __launch_bounds__(256) ltl_kernel(const float* __restrict__ linv, int p,
                                                  float* __restrict__ inv) {
    __shared__ float a[kTS][kTS + 1], b[kTS][kTS + 1];
    const int I = blockIdx.y, J = blockIdx.x;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 4 outputs per thread
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int k0 = max(I, J) * kTS;
    for (int kb = k0; kb < p; kb += kTS) {
        for (int r = ty; r < kTS; r += 8) {
            const int k = kb + r;
            a[r][tx] = (k < p && I * kTS + tx < p) ? linv[(int64_t)k * p + I * kTS + tx] : 0.f;
            b[r][tx] = (k < p && J * kTS + tx < p) ? linv[(int64_t)k * p + J * kTS + tx] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < kTS; ++k) {
            const float bv = b[k][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fmaf(a[k][ty * 4 + q], bv, acc[q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = I * kTS + ty * 4 + q, j = J * kTS + tx;
        if (i < p && j < p) inv[(int64_t)i * p + j] = acc[q];
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
    static int debug = -1;
    if (debug < 0) {
        const char* e = getenv("ENKS_SPD_DEBUG");
        debug = e ? atoi(e) : 0;
    }
    enks::spd_inverse_kernel<<<1, enks::kThreads, smem, st>>>(S, lds, p, scale, ws, status,
                                                              jitter_events, debug);
    int rc = enks::check_launch("enks_spd_inverse");
    if (rc || (debug & 4)) return rc;
    // Sy^{-1} = L^{-T} L^{-1}: one CTA per 32 x 32 output tile
    const dim3 grid((unsigned)nb, (unsigned)nb);
    enks::ltl_kernel<<<grid, 256, 0, st>>>(ws, p, inv);
    return enks::check_launch("enks_spd_inverse(ltl)");
}

}  // extern "C"
