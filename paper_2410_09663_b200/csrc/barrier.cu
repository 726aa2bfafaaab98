// Constraint barrier observation row.
//
// Reference: enks.py:201-208 (_observe_members: one extra observation row per member,
// filled with the scalar barrier reading) and virtualsys.py:289-302 (softplus_barrier,
// barrier_observe).  For member i of the predicted slice S_i = [X; U; dU] (d x m):
//     g_i = <C, S_i> + c0                       (kind 0: linear functional)
//     g_i = max_{r0 <= r < r1} |S_i[r, :]| + c0  (kind 1: box, c0 = -bound)
//     z   = beta g_i;  b_i = z > 30 ? z / alpha : log1p(exp(z)) / alpha
//     row[i*m + j] = b_i + sqrt_var * eps_i     for every column j
// g and the softplus run in fp64; one CTA per member, fixed reduction order.
#include "common.cuh"

namespace enks {
namespace {

constexpr int kBarThreads = 256;

__global__ void __launch_bounds__(kBarThreads)
    barrier_row_kernel(const float* __restrict__ S, int64_t lds, int d, int m, int kind,
                       const float* __restrict__ coef, int64_t ldc, double c0, int r0, int r1,
                       double alpha, double beta, double sqrt_var, const float* __restrict__ eps,
                       float* __restrict__ out) {
    const int64_t col0 = (int64_t)blockIdx.x * m;
    double acc = 0.0;
    const int rows = r1 - r0;
    for (int e = threadIdx.x; e < rows * m; e += blockDim.x) {
        const int r = r0 + e / m, j = e - (e / m) * m;
        const double v = S[r * lds + col0 + j];
        if (kind == 0)
            acc += (double)coef[r * ldc + j] * v;
        else
            acc = fmax(acc, fabs(v));
    }
    __shared__ double red[kBarThreads / 32];
    __shared__ double b;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, acc, o);
        acc = kind == 0 ? acc + other : fmax(acc, other);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double g = red[0];
        for (int w = 1; w < kBarThreads / 32; ++w) g = kind == 0 ? g + red[w] : fmax(g, red[w]);
        g += c0;
        const double z = beta * g;
        const double clean = z > 30.0 ? z / alpha : log1p(exp(z)) / alpha;
        b = clean + sqrt_var * (double)eps[blockIdx.x];
    }
    __syncthreads();
    const float bv = (float)b;
    for (int j = threadIdx.x; j < m; j += blockDim.x) out[col0 + j] = bv;
}

}  // namespace
}  // namespace enks

extern "C" int enks_barrier_row(const float* S, int64_t lds, int d, int m, int64_t n_members,
                                int kind, const float* coef, int64_t ldc, double c0, int r0, int r1,
                                double alpha, double beta, double sqrt_var, const float* eps,
                                float* out, void* stream) {
    ENKS_REQUIRE(S && eps && out, "enks_barrier_row: null pointer");
    ENKS_REQUIRE(kind == 0 || kind == 1, "enks_barrier_row: kind must be 0 (linear) or 1 (box)");
    ENKS_REQUIRE(kind == 1 || coef, "enks_barrier_row: linear kind needs coefficients");
    ENKS_REQUIRE(0 <= r0 && r0 < r1 && r1 <= d, "enks_barrier_row: bad row block");
    ENKS_REQUIRE(alpha > 0 && beta > 0, "enks_barrier_row: alpha, beta must be positive");
    if (n_members <= 0) return ENKS_OK;
    ENKS_REQUIRE(n_members <= 0x7fffffff, "enks_barrier_row: too many members");
    enks::barrier_row_kernel<<<(unsigned)n_members, enks::kBarThreads, 0,
                               enks::as_stream(stream)>>>(S, lds, d, m, kind, coef, ldc, c0, r0, r1,
                                                          alpha, beta, sqrt_var, eps, out);
    return enks::check_launch("enks_barrier_row");
}
