// K4/K5: member means and anomalies in the member-column layout.
//
// Reference: enks.py:171 / 248 (members.mean(axis=0)), enks.py:231-233
// (obs mean, dev_y, dev_traj).  Sums run over the member axis for every
// (row, col) pair; the shift z0 (global member 0) makes identical members
// produce exactly zero anomalies (the scale=0 degenerate case,
// test_enks.py:106-117, 244-251).
//
// enks_member_sum is a two-stage deterministic reduction: stage 1 splits the
// member axis into chunks (fp64 partials, fixed order), stage 2 adds the
// chunks in order.  enks_member_center is a flat, float4-vectorised pass.
#include "common.cuh"

namespace enks {
namespace {

constexpr int kSumThreads = 128;

__global__ void __launch_bounds__(kSumThreads)
    member_partial_kernel(const float* __restrict__ src, int64_t ld, int rows, int64_t n, int cols,
                          const float* __restrict__ z0, double* __restrict__ part, int64_t chunk) {
    const int64_t rc = (int64_t)rows * cols;
    const int64_t e = blockIdx.x * (int64_t)kSumThreads + threadIdx.x;
    if (e >= rc) return;
    const int r = (int)(e / cols), j = (int)(e - (int64_t)r * cols);
    const float* p = src + r * ld + j;
    const float s = z0 ? z0[e] : p[0];
    const int64_t i0 = blockIdx.y * chunk, i1 = min(n, i0 + chunk);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    int64_t i = i0;
    for (; i + 4 <= i1; i += 4) {
        float v0 = p[(i + 0) * cols], v1 = p[(i + 1) * cols];
        float v2 = p[(i + 2) * cols], v3 = p[(i + 3) * cols];
        acc0 += (double)(v0 - s);
        acc1 += (double)(v1 - s);
        acc2 += (double)(v2 - s);
        acc3 += (double)(v3 - s);
    }
    for (; i < i1; ++i) acc0 += (double)(p[i * cols] - s);
    part[blockIdx.y * rc + e] = (acc0 + acc1) + (acc2 + acc3);
}

__global__ void chunk_reduce_kernel(const double* __restrict__ part, int nchunks, int64_t rc,
                                    double* __restrict__ acc) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= rc) return;
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += part[c * rc + e];
    acc[e] = s;
}

// mean[r, j] = z0 + mu_sh; anom[r, i*cols + j] = (src - z0) - mu_sh
__global__ void center_kernel(const float* __restrict__ src, int64_t ld, int rows, int64_t n,
                              int cols, const float* __restrict__ z0,
                              const double* __restrict__ acc, double inv_n, float* __restrict__ mean,
                              float* anom, int64_t lda) {
    const int64_t K = n * cols;
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)rows * K) return;
    const int64_t r = e / K, k = e - r * K;
    const int j = (int)(k % cols);
    const float s = z0 ? z0[r * cols + j] : src[r * ld + j];
    const float mu = (float)(acc[r * cols + j] * inv_n);
    if (mean && k < cols) mean[r * cols + j] = s + mu;
    if (anom) anom[r * lda + k] = (src[r * ld + k] - s) - mu;
}

int64_t member_chunks(int rows, int64_t n, int cols) {
    const int64_t rc = (int64_t)rows * cols;
    const int64_t blocks = (rc + kSumThreads - 1) / kSumThreads;
    // aim for ~8 blocks per SM in flight
    int64_t want = (8LL * kNumSMs + blocks - 1) / blocks;
    if (want > 64) want = 64;
    if (want > n) want = n;
    if (want < 1) want = 1;
    return want;
}

}  // namespace
}  // namespace enks

extern "C" {

int64_t enks_member_sum_ws_bytes(int rows, int64_t n_members, int cols) {
    return enks::member_chunks(rows, n_members, cols) * (int64_t)rows * cols * (int64_t)sizeof(double);
}

int enks_member_sum(const float* src, int64_t ld_src, int rows, int64_t n_members, int cols,
                    const float* z0, double* acc, void* ws, void* stream) {
    ENKS_REQUIRE(src && acc && ws, "enks_member_sum: null pointer");
    if (rows <= 0 || cols <= 0) return ENKS_OK;
    const int64_t rc = (int64_t)rows * cols;
    cudaStream_t st = enks::as_stream(stream);
    if (n_members <= 0) {
        cudaMemsetAsync(acc, 0, rc * sizeof(double), st);
        return enks::check_launch("enks_member_sum(memset)");
    }
    const int64_t nch = enks::member_chunks(rows, n_members, cols);
    const int64_t chunk = (n_members + nch - 1) / nch;
    const int64_t nch_eff = (n_members + chunk - 1) / chunk;
    dim3 grid((unsigned)((rc + enks::kSumThreads - 1) / enks::kSumThreads), (unsigned)nch_eff);
    double* part = static_cast<double*>(ws);
    enks::member_partial_kernel<<<grid, enks::kSumThreads, 0, st>>>(src, ld_src, rows, n_members,
                                                                   cols, z0, part, chunk);
    int rc_ = enks::check_launch("enks_member_sum(partial)");
    if (rc_) return rc_;
    enks::chunk_reduce_kernel<<<(unsigned)((rc + 255) / 256), 256, 0, st>>>(part, (int)nch_eff, rc,
                                                                           acc);
    return enks::check_launch("enks_member_sum(reduce)");
}

int enks_member_center(const float* src, int64_t ld_src, int rows, int64_t n_members, int cols,
                       const float* z0, const double* acc, int64_t n_total, float* mean,
                       float* anom, int64_t ld_anom, void* stream) {
    ENKS_REQUIRE(src && acc && n_total > 0, "enks_member_center: bad arguments");
    ENKS_REQUIRE(!(anom == src && z0 == nullptr),
                 "enks_member_center: in-place centring needs an explicit z0");
    if (rows <= 0 || cols <= 0 || n_members <= 0) return ENKS_OK;
    const int64_t total = (int64_t)rows * n_members * cols;
    enks::center_kernel<<<(unsigned)((total + 255) / 256), 256, 0, enks::as_stream(stream)>>>(
        src, ld_src, rows, n_members, cols, z0, acc, 1.0 / (double)n_total, mean, anom, ld_anom);
    return enks::check_launch("enks_member_center");
}

}  // extern "C"
