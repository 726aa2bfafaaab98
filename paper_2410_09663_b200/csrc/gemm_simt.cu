// Dense fp32 GEMM on the CUDA cores (FFMA), used for every contraction of the
// path that is not routed to the tcgen05 engine (gemm_tc.cu):
//   C = alpha * op(A) op(B) + beta * C0 + bias[i, n % bias_cols]
// 128x128x16 block tile, 256 threads, 8x8 outputs per thread, register
// prefetch of the next k-tile, deterministic split-K (partials in a fixed
// order).  Reference sites: enks.py:153 (_pair_covariance), 247 (member
// shift), matvar.py:188 (colouring), dynamics.py:63 (linear step).
#include "common.cuh"
#include "gemm.cuh"

namespace enks {
namespace {

constexpr int BM = 128, BN = 128, BK = 16, kThreads = 256;

struct GemmParams {
    int64_t M, N, K;
    float alpha, beta;
    const float* A;
    int64_t lda;
    const float* B;
    int64_t ldb;
    const float* C0;
    int64_t ldc0;
    const float* bias;
    int64_t ld_bias;
    int bias_cols;
    float* C;
    int64_t ldc;
    int64_t tri_rows, tri_k;
    int split;
    float* ws;
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(kThreads) sgemm_kernel(const GemmParams p) {
    __shared__ __align__(16) float As[BK][BM + 4];
    __shared__ __align__(16) float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;
    const int z = blockIdx.z;

    int64_t kbeg = 0;
    if (p.tri_rows > 0) kbeg = (row0 / p.tri_rows) * p.tri_k;
    if (kbeg > p.K) kbeg = p.K;
    const int64_t span = p.K - kbeg;
    int64_t chunk = (span + p.split - 1) / p.split;
    chunk = (chunk + BK - 1) / BK * BK;
    const int64_t k_lo = min(p.K, kbeg + z * chunk), k_hi = min(p.K, k_lo + chunk);

    // load mapping
    // "row-contiguous-k" operands (A !TA, B TB): thread -> (mn = tid/2, k = (tid&1)*8 .. +8)
    // "k-row" operands (A TA, B !TB): thread -> (k = tid/16, mn = (tid&15)*8 .. +8)
    float ra[8], rb[8];
    auto load_a = [&](int64_t k0) {
        if (!TA) {
            const int64_t r = row0 + (tid >> 1);
            const int64_t kb = k0 + (tid & 1) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int64_t k = kb + q;
                ra[q] = (r < p.M && k < k_hi) ? p.A[r * p.lda + k] : 0.f;
            }
        } else {
            const int64_t k = k0 + (tid >> 4);
            const int64_t rb0 = row0 + (tid & 15) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int64_t r = rb0 + q;
                ra[q] = (r < p.M && k < k_hi) ? p.A[k * p.lda + r] : 0.f;
            }
        }
    };
    auto load_b = [&](int64_t k0) {
        if (TB) {
            const int64_t c = col0 + (tid >> 1);
            const int64_t kb = k0 + (tid & 1) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int64_t k = kb + q;
                rb[q] = (c < p.N && k < k_hi) ? p.B[c * p.ldb + k] : 0.f;
            }
        } else {
            const int64_t k = k0 + (tid >> 4);
            const int64_t cb = col0 + (tid & 15) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int64_t c = cb + q;
                rb[q] = (c < p.N && k < k_hi) ? p.B[k * p.ldb + c] : 0.f;
            }
        }
    };
    auto store_tiles = [&]() {
        if (!TA) {
            const int m = tid >> 1, kb = (tid & 1) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) As[kb + q][m] = ra[q];
        } else {
            const int k = tid >> 4, mb = (tid & 15) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) As[k][mb + q] = ra[q];
        }
        if (TB) {
            const int n = tid >> 1, kb = (tid & 1) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) Bs[kb + q][n] = rb[q];
        } else {
            const int k = tid >> 4, nb = (tid & 15) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) Bs[k][nb + q] = rb[q];
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    if (k_lo < k_hi) {
        load_a(k_lo);
        load_b(k_lo);
        for (int64_t k0 = k_lo; k0 < k_hi; k0 += BK) {
            __syncthreads();
            store_tiles();
            __syncthreads();
            if (k0 + BK < k_hi) {
                load_a(k0 + BK);
                load_b(k0 + BK);
            }
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float a[8], b[8];
                const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
                const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
                const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 8]);
                const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 8 + 4]);
                a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
                a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
                b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
                b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
        }
    }

    // epilogue
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t r = row0 + ty * 8 + i;
        if (r >= p.M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t c = col0 + tx * 8 + j;
            if (c >= p.N) continue;
            float v = p.alpha * acc[i][j];
            if (p.split > 1) {
                p.ws[(int64_t)z * p.M * p.N + r * p.N + c] = v;
            } else {
                if (p.C0) v += p.beta * p.C0[r * p.ldc0 + c];
                if (p.bias) v += p.bias[r * p.ld_bias + (c % p.bias_cols)];
                p.C[r * p.ldc + c] = v;
            }
        }
    }
}

__global__ void split_reduce_kernel(const GemmParams p) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= p.M * p.N) return;
    const int64_t r = e / p.N, c = e - r * p.N;
    float v = 0.f;
    for (int z = 0; z < p.split; ++z) v += p.ws[(int64_t)z * p.M * p.N + e];
    if (p.C0) v += p.beta * p.C0[r * p.ldc0 + c];
    if (p.bias) v += p.bias[r * p.ld_bias + (c % p.bias_cols)];
    p.C[r * p.ldc + c] = v;
}

}  // namespace

int gemm_simt(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, float alpha,
              const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
              const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias, int bias_cols,
              float* C, int64_t ldc, int64_t tri_rows, int64_t tri_k, int split_k, void* ws,
              cudaStream_t st) {
    GemmParams p;
    p.M = M; p.N = N; p.K = K;
    p.alpha = alpha; p.beta = beta;
    p.A = A; p.lda = lda; p.B = B; p.ldb = ldb;
    p.C0 = C0; p.ldc0 = ldc0;
    p.bias = bias; p.ld_bias = ld_bias; p.bias_cols = bias_cols > 0 ? bias_cols : 1;
    p.C = C; p.ldc = ldc;
    p.tri_rows = tri_rows; p.tri_k = tri_k;
    p.split = split_k < 1 ? 1 : split_k;
    p.ws = static_cast<float*>(ws);
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)p.split);
    if (!trans_a && !trans_b) sgemm_kernel<false, false><<<grid, kThreads, 0, st>>>(p);
    else if (!trans_a && trans_b) sgemm_kernel<false, true><<<grid, kThreads, 0, st>>>(p);
    else if (trans_a && !trans_b) sgemm_kernel<true, false><<<grid, kThreads, 0, st>>>(p);
    else sgemm_kernel<true, true><<<grid, kThreads, 0, st>>>(p);
    int rc = check_launch("enks_gemm(simt)");
    if (rc || p.split == 1) return rc;
    const int64_t total = M * N;
    split_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(p);
    return check_launch("enks_gemm(split reduce)");
}

}  // namespace enks

extern "C" {

int64_t enks_gemm_ws_bytes(int64_t M, int64_t N, int split_k) {
    if (split_k <= 1) return 0;
    return (int64_t)split_k * M * N * (int64_t)sizeof(float);
}

int enks_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, float alpha,
              const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
              const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias, int bias_cols,
              float* C, int64_t ldc, int64_t tri_rows, int64_t tri_k, int split_k, void* ws,
              int engine, void* stream) {
    ENKS_REQUIRE(C != nullptr, "enks_gemm: null C");
    ENKS_REQUIRE(M >= 0 && N >= 0 && K >= 0, "enks_gemm: negative size");
    if (M == 0 || N == 0) return ENKS_OK;
    ENKS_REQUIRE(K == 0 || (A && B), "enks_gemm: null operand");
    ENKS_REQUIRE(split_k <= 1 || ws, "enks_gemm: split_k > 1 needs workspace");
    ENKS_REQUIRE(split_k <= 1024, "enks_gemm: split_k too large");
    cudaStream_t st = enks::as_stream(stream);
    if (engine == 2) {
        ENKS_REQUIRE(enks::tc_gemm_applicable(trans_a, trans_b, M, N, K, A, lda, B, ldb, tri_rows),
                     "enks_gemm: tcgen05 engine needs NT, N<=256, K>=128, 16B-aligned operands");
        return enks::gemm_tc(M, N, K, alpha, A, lda, B, ldb, beta, C0, ldc0, bias, ld_bias,
                             bias_cols, C, ldc, split_k, ws, st);
    }
    return enks::gemm_simt(trans_a, trans_b, M, N, K, alpha, A, lda, B, ldb, beta, C0, ldc0, bias,
                           ld_bias, bias_cols, C, ldc, tri_rows, tri_k, split_k, ws, st);
}

}  // extern "C"
