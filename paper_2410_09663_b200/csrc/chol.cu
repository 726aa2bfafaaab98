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
    // right-looking: finish x[k], then update every later x[j] (independent FMAs, ILP)
#pragma unroll
    for (int k = 0; k < kTS; ++k) {
        x[k] = x[k] / L[k * kLd + k];
#pragma unroll
        for (int j = k + 1; j < kTS; ++j) x[j] = fmaf(-x[k], L[j * kLd + k], x[j]);
        // keep the next columns' L loads from being hoisted across k (they would pin ~500
        // registers of prefetched values and spill x[])
        asm volatile("" ::: "memory");
    }
#pragma unroll
    for (int j = 0; j < kTS; ++j) X[lane * kLd + j] = x[j];
}

// rows [r0, r0 + 8) of C <- C - A B^T (lane = column of C): a quarter-tile task, so the trailing
// update of a block column spreads over 4x more warps
__device__ __forceinline__ void quarter_syrk_sub(float* C, const float* A, const float* B,
                                                 int lane, int r0) {
    float acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc[r] = 0.f;
#pragma unroll 8
    for (int k = 0; k < kTS; ++k) {
        const float bk = B[lane * kLd + k];
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r] = fmaf(A[(r0 + r) * kLd + k], bk, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) C[(r0 + r) * kLd + lane] -= acc[r];
}

// in-place inverse of a lower-triangular 32x32 tile (warp; lane = column of the inverse)
__device__ void invert_diag(float* T, int lane) {
    // column `lane` of L^{-1}: forward substitution L y = e_lane
    float y[kTS];
#pragma unroll
    for (int i = 0; i < kTS; ++i) y[i] = (i == lane) ? 1.f : 0.f;
    // right-looking: finish y[k], then update every later y[i] (independent FMAs)
#pragma unroll
    for (int k = 0; k < kTS; ++k) {
        y[k] = (k < lane) ? 0.f : y[k] / T[k * kLd + k];
#pragma unroll
        for (int i = k + 1; i < kTS; ++i) y[i] = fmaf(-T[i * kLd + k], y[k], y[i]);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kTS; ++i) T[i * kLd + lane] = y[i];
    __syncwarp();
}

__global__ void __launch_bounds__(kThreads)
    spd_inverse_kernel(const float* __restrict__ S, int64_t lds, int p, float scale,
                       float* __restrict__ linv, int* status, int* jitter_events, int debug,
                       int single, float* jit_out) {
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

    // attempt 0: no jitter; attempt 1: the reference's 1e-9 tr / p + 1e-30 (enks.py:241).  A
    // relative 1e-9 is below fp32 resolution, so when it cannot rescue a rank-deficient Sigma_y
    // (N m < p) the jitter is escalated (1e-7, 1e-6, 1e-5 relative) -- still one jitter event.
    int failed = 0;
    float used_jit = 0.f;
    for (int attempt = 0; attempt < (single ? 1 : 5); ++attempt) {
        // relative jitter per attempt: 0, 1e-9 (the reference), then 1e-7, 1e-6, 1e-5 (selects,
        // not an indexed local array: no stack frame)
        const double rel = attempt == 1 ? 1e-9 : (attempt == 2 ? 1e-7 : (attempt == 3 ? 1e-6 : 1e-5));
        const float jitter = attempt == 0 ? 0.f : (float)(rel * trace / (double)p + 1e-30);
        used_jit = jitter;
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
            // trailing update of tiles (I, J), K < J <= I, in quarter-tile tasks
            const int m = nb - K - 1;
            for (int t = warp; t < 2 * m * (m + 1); t += kWarps) {
                const int q = t >> 2, rq = t & 3;
                int I = 0;
                while ((I + 1) * (I + 2) / 2 <= q) ++I;
                const int J = q - I * (I + 1) / 2;
                const int gI = K + 1 + I, gJ = K + 1 + J;
                quarter_syrk_sub(Lt + tix(gI, gJ) * kTile, Lt + tix(gI, K) * kTile,
                                 Lt + tix(gJ, K) * kTile, lane, 8 * rq);
            }
            __syncthreads();
        }
        failed = s_fail;
        __syncthreads();
        if (!failed) break;
        if (attempt == 0 && tid == 0 && !single) atomicAdd(jitter_events, 1);
    }
    if (tid == 0 && jit_out) *jit_out = used_jit;
    if (failed) {
        if (tid == 0) *status = 1;
        const float nan = __int_as_float(0x7fc00000);
        for (int e = tid; e < p * p; e += kThreads) linv[e] = nan;
        return;
    }

    // L^{-1}, tile row by tile row: Linv_II = L_II^{-1};
    // Linv_IJ = -Linv_II * sum_{K=J}^{I-1} L_IK Linv_KJ   (J < I), written over L_IJ.
    // The diagonal inverses are independent: all at once first (one warp each).  Then per tile
    // row I: phase A forms res_J = sum_K L_IK Linv_KJ in quarter-tile tasks into a staging area
    // (tiles (I, K) are still L there and are read by other tasks), phase B overwrites
    // (I, J) with -Linv_II res_J, again in quarter tasks.
    float* res = Lt + (nb * (nb + 1) / 2) * kTile;  // staging: up to nb - 1 tiles
    if (!(debug & 1)) {
        for (int I = warp; I < nb; I += kWarps) invert_diag(Lt + tix(I, I) * kTile, lane);
        __syncthreads();
    }
    for (int I = 1; I < ((debug & 1) ? 0 : nb); ++I) {
        for (int t = warp; t < 4 * I; t += kWarps) {  // phase A: task (J, row quarter)
            const int J = t >> 2, r0 = 8 * (t & 3);
            float acc[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) acc[r] = 0.f;
            for (int K = J; K < I; ++K) {
                const float* A = Lt + tix(I, K) * kTile;  // L_IK
                const float* B = Lt + tix(K, J) * kTile;  // Linv_KJ (K == J: Linv_JJ)
#pragma unroll 8
                for (int k = 0; k < kTS; ++k) {
                    const float bk = B[k * kLd + lane];  // column `lane` of B
#pragma unroll
                    for (int r = 0; r < 8; ++r) acc[r] = fmaf(A[(r0 + r) * kLd + k], bk, acc[r]);
                }
            }
            float* R = res + J * kTile;
#pragma unroll
            for (int r = 0; r < 8; ++r) R[(r0 + r) * kLd + lane] = acc[r];
        }
        __syncthreads();
        const float* D = Lt + tix(I, I) * kTile;  // Linv_II
        for (int t = warp; t < 4 * I; t += kWarps) {  // phase B: out rows r0 .. r0 + 7
            const int J = t >> 2, r0 = 8 * (t & 3);
            const float* R = res + J * kTile;
            float o[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) o[r] = 0.f;
            for (int k = 0; k < r0 + 8; ++k) {  // D lower triangular: k <= r
                const float rk = R[k * kLd + lane];
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (k <= r0 + r) o[r] = fmaf(D[(r0 + r) * kLd + k], rk, o[r]);
            }
            float* out = Lt + tix(I, J) * kTile;
#pragma unroll
            for (int r = 0; r < 8; ++r) out[(r0 + r) * kLd + lane] = -o[r];
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

// One Newton step on the inverse in fp64 (the fp32 Cholesky's error grows like p eps cond):
//   R = I - W X0,  X = X0 + X0 R,   W = scale * sym(S) + jit I (the matrix that was inverted).
// Tiled 32 x 32 outputs per CTA, fp64 accumulation; two launches of 2 p^3 flop each.
__global__ void __launch_bounds__(256) refine_residual_kernel(const float* __restrict__ S,
                                                              int64_t lds, int p, float scale,
                                                              const float* jit,
                                                              const float* __restrict__ X0,
                                                              double* __restrict__ R) {
    __shared__ double a[kTS][kTS + 1], b[kTS][kTS + 1];
    const int I = blockIdx.y, J = blockIdx.x;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const double jv = (double)*jit;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kb = 0; kb < p; kb += kTS) {
        for (int r = ty; r < kTS; r += 8) {
            const int i = I * kTS + r, k = kb + tx;
            double w = 0.0;
            if (i < p && k < p)
                w = (double)(scale * (0.5f * (S[(int64_t)i * lds + k] + S[(int64_t)k * lds + i]))) +
                    (i == k ? jv : 0.0);
            a[r][tx] = w;
            const int kk = kb + r, j = J * kTS + tx;
            b[r][tx] = (kk < p && j < p) ? (double)X0[(int64_t)kk * p + j] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < kTS; ++k) {
            const double bv = b[k][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(a[ty * 4 + q][k], bv, acc[q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = I * kTS + ty * 4 + q, j = J * kTS + tx;
        if (i < p && j < p) R[(int64_t)i * p + j] = (i == j ? 1.0 : 0.0) - acc[q];
    }
}

__global__ void __launch_bounds__(256) refine_update_kernel(const float* __restrict__ X0,
                                                            const double* __restrict__ R, int p,
                                                            float* __restrict__ X) {
    __shared__ double a[kTS][kTS + 1], b[kTS][kTS + 1];
    const int I = blockIdx.y, J = blockIdx.x;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kb = 0; kb < p; kb += kTS) {
        for (int r = ty; r < kTS; r += 8) {
            const int i = I * kTS + r, k = kb + tx;
            a[r][tx] = (i < p && k < p) ? (double)X0[(int64_t)i * p + k] : 0.0;
            const int kk = kb + r, j = J * kTS + tx;
            b[r][tx] = (kk < p && j < p) ? R[(int64_t)kk * p + j] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int k = 0; k < kTS; ++k) {
            const double bv = b[k][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(a[ty * 4 + q][k], bv, acc[q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = I * kTS + ty * 4 + q, j = J * kTS + tx;
        if (i < p && j < p) X[(int64_t)i * p + j] = (float)((double)X0[(int64_t)i * p + j] + acc[q]);
    }
}

int refine(const float* S, int64_t lds, int p, float scale, const float* jit, const float* X0,
           double* R, float* X, cudaStream_t st) {
    const int nb = (p + kTS - 1) / kTS;
    const dim3 grid((unsigned)nb, (unsigned)nb);
    refine_residual_kernel<<<grid, 256, 0, st>>>(S, lds, p, scale, jit, X0, R);
    refine_update_kernel<<<grid, 256, 0, st>>>(X0, R, p, X);
    return check_launch("enks_spd_inverse(refine)");
}

// W = scale * sym(S) + jitter I, jitter = rel * tr / p + 1e-30 (rel = 0: none; enks.py:241)
__global__ void sym_scale_kernel(const float* __restrict__ S, int64_t lds, int p, float scale,
                                 double rel, float* __restrict__ W, float* jit_out) {
    __shared__ double tr_s;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < p; ++i) t += (double)(scale * S[(int64_t)i * lds + i]);
        tr_s = t;
    }
    __syncthreads();
    const float jit = rel > 0.0 ? (float)(rel * tr_s / (double)p + 1e-30) : 0.f;
    if (blockIdx.x == 0 && threadIdx.x == 0) *jit_out = jit;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < p * p; e += gridDim.x * blockDim.x) {
        const int i = e / p, j = e - i * p;
        W[e] = scale * (0.5f * (S[(int64_t)i * lds + j] + S[(int64_t)j * lds + i])) +
               (i == j ? jit : 0.f);
    }
}

// out = the first pass whose two factorisations succeeded (plain, reference jitter, escalated
// jitter), else NaN; status / jitter counters as enks.py:238-244
__global__ void select_kernel(const float* __restrict__ p0, const float* __restrict__ p1,
                              const float* __restrict__ p2, const int* flags, int n,
                              float* __restrict__ out, int* status, int* jitter_events,
                              const float* jits, float* jit_out) {
    const int f0 = flags[0] | flags[1], f1 = flags[2] | flags[3], f2 = flags[4] | flags[5];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (f0) atomicAdd(jitter_events, 1);
        if (f0 && f1 && f2) *status = 1;
        *jit_out = !f0 ? jits[0] : (!f1 ? jits[1] : jits[2]);
    }
    const float nan = __int_as_float(0x7fc00000);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
        out[e] = !f0 ? p0[e] : (!f1 ? p1[e] : (!f2 ? p2[e] : nan));
}

// dst[i][j] = alpha * (trans ? src[j][i] : src[i][j]) for an R x C block
__global__ void copy_block_kernel(const float* __restrict__ src, int64_t lds, int R, int C,
                                  float alpha, int trans, float* __restrict__ dst, int64_t ldd) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < R * C; e += gridDim.x * blockDim.x) {
        const int i = e / C, j = e - i * C;
        dst[(int64_t)i * ldd + j] = alpha * (trans ? src[(int64_t)j * lds + i] : src[(int64_t)i * lds + j]);
    }
}

int copy_block(const float* src, int64_t lds, int R, int C, float alpha, int trans, float* dst,
               int64_t ldd, cudaStream_t st) {
    copy_block_kernel<<<(R * C + 255) / 256, 256, 0, st>>>(src, lds, R, C, alpha, trans, dst, ldd);
    return check_launch("enks_spd_inverse(copy)");
}

size_t spd_smem(int p) {
    const int nb = (p + kTS - 1) / kTS;
    // lower tile-triangle + the inverse's staging tiles
    return ((size_t)nb * (nb + 1) / 2 + (nb > 1 ? nb - 1 : 0)) * kTile * sizeof(float);
}

int configure_spd(size_t smem) {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(spd_inverse_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            set_error("enks_spd_inverse: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = smem;
    }
    return ENKS_OK;
}

int spd_debug() {
    return debug_knob("ENKS_SPD_DEBUG", 0);  // phase switches: debug builds only
}

// inv = S^{-1} (p <= kMaxP) with the one-CTA kernel: single = 1 -> one attempt, *flag = 1 on a
// bad pivot (no jitter); single = 0 -> the reference's jitter rule with status / jitter_events
int spd_small(const float* S, int64_t lds, int p, float scale, float* inv, float* linv_ws,
              int* status, int* jitter_events, int single, cudaStream_t st,
              float* jit_out = nullptr) {
    const size_t smem = spd_smem(p);
    int rc = configure_spd(smem);
    if (rc) return rc;
    const int debug = spd_debug();
    spd_inverse_kernel<<<1, kThreads, smem, st>>>(S, lds, p, scale, linv_ws, status, jitter_events,
                                                   debug, single, jit_out);
    rc = check_launch("enks_spd_inverse");
    if (rc || (debug & 4)) return rc;
    const int nb = (p + kTS - 1) / kTS;
    ltl_kernel<<<dim3((unsigned)nb, (unsigned)nb), 256, 0, st>>>(linv_ws, p, inv);
    return check_launch("enks_spd_inverse(ltl)");
}

// One attempt of W^{-1} (W symmetric p x p, kMaxP < p <= 2 kMaxP) by a 2 x 2 Schur complement:
// A^{-1} = W11^{-1}; T = W21 A^{-1}; X = W22 - T W12; XT = X^{-1} T;
// inv = [A^{-1} + T^T XT, -XT^T; -XT, X^{-1}].  flags[0] / flags[1]: W11 / X not SPD
// (exactly when a Cholesky of W would fail, up to rounding).
int schur_inverse(const float* W, int p, float* inv, float* ws, int* flags, cudaStream_t st) {
    const int p1 = ((p / 2 + kTS - 1) / kTS) * kTS, p2 = p - p1;
    float* Ainv = ws;                 // p1 x p1
    float* T = Ainv + p1 * p1;        // p2 x p1
    float* X = T + p2 * p1;           // p2 x p2
    float* Xinv = X + p2 * p2;        // p2 x p2
    float* XT = Xinv + p2 * p2;       // p2 x p1
    float* lws = XT + p2 * p1;        // L^{-1} workspace, <= kMaxP^2
    const float* W12 = W + p1;
    const float* W21 = W + (int64_t)p1 * p;
    const float* W22 = W + (int64_t)p1 * p + p1;
    int rc = spd_small(W, p, p1, 1.f, Ainv, lws, flags, flags, 1, st);
    if (!rc) rc = gemm_simt(0, 0, p2, p1, p1, 1.f, W21, p, Ainv, p1, 0.f, nullptr, 0, nullptr, 0, 1,
                            T, p1, 0, 0, 1, nullptr, st);
    if (!rc) rc = gemm_simt(0, 0, p2, p2, p1, -1.f, T, p1, W12, p, 1.f, W22, p, nullptr, 0, 1, X, p2,
                            0, 0, 1, nullptr, st);
    if (!rc) rc = spd_small(X, p2, p2, 1.f, Xinv, lws, flags + 1, flags + 1, 1, st);
    if (!rc) rc = gemm_simt(0, 0, p2, p1, p2, 1.f, Xinv, p2, T, p1, 0.f, nullptr, 0, nullptr, 0, 1,
                            XT, p1, 0, 0, 1, nullptr, st);
    if (!rc) rc = copy_block(Xinv, p2, p2, p2, 1.f, 0, inv + (int64_t)p1 * p + p1, p, st);
    if (!rc) rc = copy_block(XT, p1, p2, p1, -1.f, 0, inv + (int64_t)p1 * p, p, st);
    if (!rc) rc = copy_block(XT, p1, p1, p2, -1.f, 1, inv + p1, p, st);
    if (!rc) rc = gemm_simt(1, 0, p1, p1, p2, 1.f, T, p1, XT, p1, 1.f, Ainv, p1, nullptr, 0, 1, inv,
                            p, 0, 0, 1, nullptr, st);
    return rc;
}

}  // namespace
}  // namespace enks

extern "C" {

int enks_spd_max_p(void) { return 2 * enks::kMaxP; }

int64_t enks_spd_ws_bytes(int p) {
    // + fp32 X0 (p^2) + fp64 residual (2 p^2 floats) for the Newton refinement
    if (p <= enks::kMaxP) return ((int64_t)4 * p * p + 64) * (int64_t)sizeof(float);
    // W (p^2, reused per pass), out0..2 (3 p^2) + Schur temporaries (< 3 p^2) + L^{-1} + flags
    return ((int64_t)10 * p * p + (int64_t)enks::kMaxP * enks::kMaxP + 128) * (int64_t)sizeof(float);
}

int enks_spd_inverse(const float* S, int64_t lds, int p, float scale, float* inv, float* ws,
                     int* status, int* jitter_events, void* stream) {
    ENKS_REQUIRE(S && inv && ws && status && jitter_events, "enks_spd_inverse: null pointer");
    ENKS_REQUIRE(p >= 1 && p <= 2 * enks::kMaxP, "enks_spd_inverse: p=%d outside [1, %d]", p,
                 2 * enks::kMaxP);
    cudaStream_t st = enks::as_stream(stream);
    const int64_t pp = (int64_t)p * p;
    if (p <= enks::kMaxP) {
        float* X0 = ws + pp;
        double* R = reinterpret_cast<double*>(ws + 2 * pp);
        float* jit = ws + 4 * pp + 8;
        int rc = enks::spd_small(S, lds, p, scale, X0, ws, status, jitter_events, 0, st, jit);
        if (rc || (enks::spd_debug() & 4)) return rc;
        return enks::refine(S, lds, p, scale, jit, X0, R, inv, st);
    }
    // three complete attempts on the whole matrix (plain, the reference jitter, escalated jitter
    // -- see spd_inverse_kernel), then a device-side select: no host synchronisation
    float* W = ws;
    float* outs = W + pp;               // 3 p^2
    float* tmp = outs + 3 * pp;         // Schur temporaries
    float* X0 = tmp + 2 * pp + enks::kMaxP * enks::kMaxP;
    double* R = reinterpret_cast<double*>(X0 + pp + (pp & 1));
    int* flags = reinterpret_cast<int*>(X0 + 3 * pp + 4);
    float* jits = reinterpret_cast<float*>(flags + 8);  // [3] per pass + [3] selected
    cudaMemsetAsync(flags, 0, 6 * sizeof(int), st);
    const double rel[3] = {0.0, 1e-9, 1e-5};
    int rc = ENKS_OK;
    for (int pass = 0; pass < 3 && !rc; ++pass) {
        enks::sym_scale_kernel<<<148, 256, 0, st>>>(S, lds, p, scale, rel[pass], W, jits + pass);
        rc = enks::check_launch("enks_spd_inverse(sym)");
        if (!rc) rc = enks::schur_inverse(W, p, outs + pass * pp, tmp, flags + 2 * pass, st);
    }
    if (rc) return rc;
    enks::select_kernel<<<148, 256, 0, st>>>(outs, outs + pp, outs + 2 * pp, flags, (int)pp, X0,
                                             status, jitter_events, jits, jits + 3);
    rc = enks::check_launch("enks_spd_inverse(select)");
    if (rc) return rc;
    return enks::refine(S, lds, p, scale, jits + 3, X0, R, inv, st);
}

}  // extern "C"
