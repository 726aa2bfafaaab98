// K1+K2: bit-exact device noise substreams.
//
// Reference call sites: enks.py:131-145 (_member_noise loop over members),
// matvar.py:149-151 (NoiseStreams.substream -> numpy SeedSequence/Philox),
// matvar.py:183-188 (colouring mean + L z I_m; col_chol = I_m in every
// reference virtual system, virtualsys.py:199-208).
//
// One warp owns one (member, t, channel) substream (noise_dev.cuh: run_stream).  The 32 lanes
// evaluate Philox4x64-10 blocks by counter in parallel (two per lane, 256 words per refill,
// staged in shared memory), classify 32 consecutive words at once against the ziggurat fast
// accept, resolve numpy's sequential parse on bitmasks (speculative wedge tests in parallel,
// tails warp-uniformly) and stage whole rows for float4 stores.  The word consumption is
// exactly numpy's sequential order.
#include "noise_dev.cuh"

namespace enks {
namespace {

constexpr int kWarps = 4;          // warps (streams) per block

template <bool RB>
__global__ void __launch_bounds__(kWarps * 32, 6) noise_kernel(const Args args) {
    const Job a = args.job[blockIdx.y];  // by value: fields live in registers, not re-read
    __shared__ __align__(16) float s_row[RB ? kWarps : 1][RB ? 2 * kMaxRowCols : 1];
    __shared__ uint64_t s_ki[256];
    __shared__ double s_wi[256];
    __shared__ uint64_t s_buf[kWarps][kBufWords];
    load_tables(s_ki, s_wi, threadIdx.x, blockDim.x);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t local = (int64_t)blockIdx.x * kWarps + warp;
    if (local >= args.n_members) return;
    run_stream<RB>(args, a, local, lane, &s_row[RB ? warp : 0][0], s_buf[warp], s_ki, s_wi);
}

}  // namespace
}  // namespace enks

namespace enks {
namespace {
int launch_noise(const uint32_t* head, int n_head, int64_t member0, int64_t n_members, int cols,
                 const Job* jobs, int n_jobs, cudaStream_t st, const uint32_t* head_dev = nullptr) {
    NoiseLaunch L;
    int rc = make_noise_launch(head, n_head, head_dev, member0, n_members, cols, jobs, n_jobs, L);
    if (rc || n_members <= 0 || cols <= 0) return rc;
    int64_t blocks = (n_members + kWarps - 1) / kWarps;
    if (L.rb)
        noise_kernel<true><<<dim3((unsigned)blocks, (unsigned)n_jobs), kWarps * 32, 0, st>>>(L.args);
    else
        noise_kernel<false><<<dim3((unsigned)blocks, (unsigned)n_jobs), kWarps * 32, 0, st>>>(L.args);
    return check_launch("enks_noise_fill");
}
}  // namespace
}  // namespace enks

extern "C" int enks_noise_fill(const uint32_t* head, int n_head, uint32_t t, uint32_t channel,
                               int64_t member0, int64_t n_members, int rows, int cols,
                               const double* diag, float* out, int64_t ld_out, const float* base,
                               int64_t ld_base, float* out_plus, int64_t ld_plus, void* stream) {
    if (rows <= 0) return ENKS_OK;
    enks::Job j{t, channel, rows, diag, out, ld_out, base, ld_base, out_plus, ld_plus};
    return enks::launch_noise(head, n_head, member0, n_members, cols, &j, 1,
                              enks::as_stream(stream));
}

extern "C" int enks_noise_fill_multi(const uint32_t* head, int n_head, int64_t member0,
                                     int64_t n_members, int cols, int n_jobs,
                                     const uint32_t* t, const uint32_t* channel, const int* rows,
                                     const double* const* diag, float* const* out,
                                     const int64_t* ld_out, const float* const* base,
                                     const int64_t* ld_base, float* const* out_plus,
                                     const int64_t* ld_plus, void* stream) {
    ENKS_REQUIRE(n_jobs >= 1 && n_jobs <= enks::kMaxJobs, "enks_noise_fill_multi: 1..%d jobs",
                 enks::kMaxJobs);
    enks::Job jobs[enks::kMaxJobs];
    for (int q = 0; q < n_jobs; ++q)
        jobs[q] = enks::Job{t[q], channel[q], rows[q], diag[q], out[q], ld_out[q],
                            base[q], ld_base[q], out_plus[q], ld_plus[q]};
    return enks::launch_noise(head, n_head, member0, n_members, cols, jobs, n_jobs,
                              enks::as_stream(stream));
}

extern "C" int enks_noise_fill_multi_dev(const uint32_t* head_dev, int n_head, int64_t member0,
                                         int64_t n_members, int cols, int n_jobs,
                                         const uint32_t* t, const uint32_t* channel,
                                         const int* rows, const double* const* diag,
                                         float* const* out, const int64_t* ld_out,
                                         const float* const* base, const int64_t* ld_base,
                                         float* const* out_plus, const int64_t* ld_plus,
                                         void* stream) {
    ENKS_REQUIRE(head_dev, "enks_noise_fill_multi_dev: null head");
    ENKS_REQUIRE(n_jobs >= 1 && n_jobs <= enks::kMaxJobs, "enks_noise_fill_multi_dev: 1..%d jobs",
                 enks::kMaxJobs);
    enks::Job jobs[enks::kMaxJobs];
    for (int q = 0; q < n_jobs; ++q)
        jobs[q] = enks::Job{t[q], channel[q], rows[q], diag[q], out[q], ld_out[q],
                            base[q], ld_base[q], out_plus[q], ld_plus[q]};
    return enks::launch_noise(nullptr, n_head, member0, n_members, cols, jobs, n_jobs,
                              enks::as_stream(stream), head_dev);
}
