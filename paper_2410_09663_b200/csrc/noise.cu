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
#include <climits>

#include "noise_dev.cuh"

namespace enks {
namespace {

constexpr int kWarps = 4;          // warps (streams) per block

template <bool RB>
#ifndef ENKS_NOISE_MINB
#define ENKS_NOISE_MINB 6  // blocks per SM: 3072 C3 substreams = 768 blocks fit one wave of 6 x 148
#endif
__global__ void __launch_bounds__(kWarps * 32, ENKS_NOISE_MINB) noise_kernel(const Args args) {
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


__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_int(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ long long ld_volatile_ll(const long long* p) {
    return *(const volatile long long*)p;
}

// ---------------------------------------------------------------------------------------------
// Segmented substreams for latency-bound launches (few substreams: small ensembles, or one rank's
// shard).  A substream's word sequence is cut into chunks of G groups (32 words each); one warp
// per (substream, chunk), taken in ticket order (chunk-major) so every chunk's predecessor is
// already running or done.  Phase A counts the normals started inside the chunk (speculating that
// the parse enters at the chunk's first word), then the warp waits for its predecessor's record
// (words of this chunk consumed by the previous normal = entry carry, normals before the chunk =
// prefix), recounts in the rare case the entry differs (~1.5 % of chunks), publishes its own
// record, and phase B re-parses the chunk emitting normals prefix, prefix + 1, ... -- numpy's
// order exactly, each chunk's words generated twice.  The last chunk runs on until the
// substream has all its normals (the chunk count is an estimate of the words needed).
struct SegRec {
    int carry;
    int flag;
    long long prefix;  // normals started before the next chunk (inclusive of this one)
};

constexpr int kSegWarps = 4;

// rec_x / rec_o: phase A records each group's emitted values (x per lane) and emit mask, so that
// phase B of an exactly speculated chunk (entry carry 0: ~98.5 %) replays them -- no second
// Philox / ziggurat pass (G groups per unit, unit = chunk-major ticket index).  The launch stays
// latency-bound either way; the saved instructions are issue slots the concurrent forecast gets.
__global__ void __launch_bounds__(kSegWarps * 32) noise_seg_kernel(const Args args, int n_jobs,
                                                                   int n_chunks, int G,
                                                                   SegRec* recs,
                                                                   unsigned* ticket,
                                                                   double* rec_x, unsigned* rec_o) {
    __shared__ uint64_t s_ki[256];
    __shared__ double s_wi[256];
    __shared__ uint64_t s_buf[kSegWarps][kBufWords];
    load_tables(s_ki, s_wi, threadIdx.x, blockDim.x);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* buf = s_buf[warp];
    const int64_t nm = args.n_members;
    const int64_t n_streams = nm * n_jobs;
    const int64_t n_units = n_streams * n_chunks;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int cols = args.cols;
    for (;;) {
        unsigned t0 = 0;
        if (lane == 0) t0 = atomicAdd(ticket, 1u);
        const int64_t t = (int64_t)__shfl_sync(0xffffffffu, t0, 0);
        if (t >= n_units) break;
        const int c = (int)(t / n_streams);
        const int64_t sidx = t - (int64_t)c * n_streams;
        const int j = (int)(sidx / nm);
        const int64_t local = sidx - (int64_t)j * nm;
        const Job a = j == 0 ? args.job[0] : (j == 1 ? args.job[1] : (j == 2 ? args.job[2] : args.job[3]));
        uint64_t k0, k1;
        if (args.head_dev) {
            Head hd;
            hd.n = args.head.n;
#pragma unroll
            for (int q = 0; q < 32; ++q) hd.w[q] = q < hd.n ? __ldg(args.head_dev + q) : 0u;
            seed_key(hd, (uint32_t)(args.member0 + local), a.t, a.ch, k0, k1);
        } else {
            seed_key(args.head, (uint32_t)(args.member0 + local), a.t, a.ch, k0, k1);
        }
        const int total = a.rows * cols;
        const int64_t col0 = local * cols;
        const bool last = c == n_chunks - 1;
        const int g_begin = c * G, g_end = last ? INT_MAX : (c + 1) * G;
        int base_w = -(1 << 30);
        auto word = [&](int ww) -> uint64_t {
            if (ww >= base_w && ww < base_w + kBufWords) return buf[ww - base_w];
            Block4 b = philox(k0, k1, (uint64_t)(ww >> 2) + 1);
            int s = (int)(ww & 3);
            return s == 0 ? b.v0 : (s == 1 ? b.v1 : (s == 2 ? b.v2 : b.v3));
        };
        double* ux = rec_x + t * (int64_t)G * 32;
        unsigned* uo = rec_o + t * (int64_t)G;
        auto emit1 = [&](long long q, double x) {
            const int r = (int)(q / cols), jj = (int)(q - (long long)r * cols);
            const double v = a.diag ? x * a.diag[r] : x;
            const float f = (float)v;
            if (a.out) a.out[r * a.ld_out + col0 + jj] = f;
            if (a.out_plus)
                a.out_plus[r * a.ld_plus + col0 + jj] = a.base[r * a.ld_base + col0 + jj] + f;
        };
        // parse groups [g_begin, g_end) entering with `carry`; EMIT: write normals q0, q0 + 1, ...
        // (< total); RECORD: keep each group's x / emit mask for replay (not the last chunk);
        // returns the count of normals started in the range, carry out in `carry`
        auto parse = [&](bool emit, bool record, int& carry, long long q0) -> long long {
            long long cnt = 0;
            base_w = -(1 << 30);
            for (int g = g_begin; g < g_end; ++g) {
                const int w = g * 32;
                if (last && q0 + cnt >= total) break;
                if (w >= base_w + kBufWords) {
                    base_w = w;
                    __syncwarp();
#pragma unroll
                    for (int bq = 0; bq < kBufWords / 128; ++bq) {
                        const Block4 b = philox(k0, k1, (uint64_t)((base_w >> 2) + bq * 32 + lane) + 1);
                        buf[bq * 128 + 4 * lane + 0] = b.v0;
                        buf[bq * 128 + 4 * lane + 1] = b.v1;
                        buf[bq * 128 + 4 * lane + 2] = b.v2;
                        buf[bq * 128 + 4 * lane + 3] = b.v3;
                    }
                    __syncwarp();
                }
                const uint64_t raw = buf[w - base_w + lane];
                double x;
                unsigned O;
                int next_carry;
                resolve_group(raw, w, carry, lane, s_ki, s_wi, word, x, O, next_carry);
                carry = next_carry;
                if (record) {
                    ux[(g - g_begin) * 32 + lane] = x;
                    if (lane == 0) uo[g - g_begin] = O;
                }
                if (emit && ((O >> lane) & 1u)) {
                    const long long q = q0 + cnt + __popc(O & lt_mask);
                    if (q < total) emit1(q, x);
                }
                cnt += __popc(O);
            }
            return cnt;
        };
        // phase B from the records of phase A (this chunk's groups, entry carry 0)
        auto replay = [&](long long q0) {
            long long cnt = 0;
            for (int g = g_begin; g < g_end; ++g) {
                const unsigned O = uo[g - g_begin];
                if ((O >> lane) & 1u) {
                    const long long q = q0 + cnt + __popc(O & lt_mask);
                    if (q < total) emit1(q, ux[(g - g_begin) * 32 + lane]);
                }
                cnt += __popc(O);
            }
        };
        int carry_in = 0;
        long long prefix = 0;
        long long cnt = 0;
        int carry_out = 0;
        if (!last) {  // phase A (speculative entry carry 0), recorded
            carry_out = 0;
            cnt = parse(false, true, carry_out, 0);
        }
        if (c > 0) {  // predecessor's record
            const SegRec* pr = recs + (int64_t)(c - 1) * n_streams + sidx;
            if (lane == 0) {
                while (ld_acquire(&pr->flag) == 0) {
                }
            }
            __syncwarp();
            carry_in = ld_volatile_int(&pr->carry);
            prefix = ld_volatile_ll(&pr->prefix) - 0;
        }
        if (!last) {
            if (carry_in != 0) {  // the entry differs from the speculation: recount
                carry_out = carry_in;
                cnt = parse(false, false, carry_out, 0);
            }
            SegRec* me = recs + (int64_t)c * n_streams + sidx;
            if (lane == 0) {
                me->carry = carry_out;
                me->prefix = prefix + cnt;
                __threadfence();
                st_release(&me->flag, 1);
            }
        }
        // phase B: emit this chunk's normals from index prefix -- replayed from phase A's records
        // when the speculated entry was right, parsed again otherwise (and for the last chunk)
        if (prefix < total) {
            __syncwarp();  // phase A's records visible to every lane
            if (!last && carry_in == 0) {
                replay(prefix);
            } else {
                int cb = carry_in;
                parse(true, false, cb, prefix);
            }
        }
        __syncwarp();
    }
}
}  // namespace
}  // namespace enks

namespace enks {
namespace {
// segmented plan: (n_chunks, G) for n_streams substreams of up to max_normals normals, or
// n_chunks = 0 when one warp per substream already fills the GPU
struct SegPlan {
    int n_chunks = 0, G = 0;
};
SegPlan seg_plan(int64_t n_streams, int64_t max_normals) {
    SegPlan P;
    // target resident warps per SM (tuning; ENKS_NOISE_WARPS, read once): below half of it the
    // substreams are cut into chunks so that the latency-bound per-warp parse has company
    const int64_t target = env_knob("ENKS_NOISE_WARPS", 16);
    if (n_streams <= 0 || 2 * n_streams >= target * kNumSMs) return P;
    const int64_t groups = (max_normals * 104 / 100 + 64 + 31) / 32;  // ~1.5 % rejected starts
    int64_t chunks = (target * kNumSMs + n_streams - 1) / n_streams;
    if (chunks > groups / 8) chunks = groups / 8;  // >= 8 groups per chunk
    if (chunks < 2) return P;
    P.n_chunks = (int)chunks;
    P.G = (int)((groups + chunks - 1) / chunks);
    return P;
}

// workspace: [ticket (256 B) | records (zeroed per launch) | replay records x, emit masks]
int64_t seg_rec_bytes(int64_t n_streams, const SegPlan& P) {
    return ((int64_t)P.n_chunks * n_streams * (int64_t)sizeof(SegRec) + 256 + 255) / 256 * 256;
}
int64_t seg_ws_bytes(int64_t n_streams, int64_t max_normals) {
    const SegPlan P = seg_plan(n_streams, max_normals);
    if (!P.n_chunks) return 0;
    const int64_t groups = (int64_t)P.n_chunks * n_streams * P.G;
    return seg_rec_bytes(n_streams, P) + groups * 32 * (int64_t)sizeof(double) +
           groups * (int64_t)sizeof(unsigned);
}

int launch_noise(const uint32_t* head, int n_head, int64_t member0, int64_t n_members, int cols,
                 const Job* jobs, int n_jobs, cudaStream_t st, const uint32_t* head_dev = nullptr,
                 void* ws = nullptr, int64_t ws_bytes = 0) {
    NoiseLaunch L;
    int rc = make_noise_launch(head, n_head, head_dev, member0, n_members, cols, jobs, n_jobs, L);
    if (rc || n_members <= 0 || cols <= 0) return rc;
    int max_rows = 0;
    for (int j = 0; j < n_jobs; ++j) max_rows = max_rows > jobs[j].rows ? max_rows : jobs[j].rows;
    const int64_t n_streams = n_members * n_jobs;
    const SegPlan P = seg_plan(n_streams, (int64_t)max_rows * cols);
    if (ws && P.n_chunks && env_knob("ENKS_NOISE_SEG", 1) != 0 &&
        ws_bytes >= seg_ws_bytes(n_streams, (int64_t)max_rows * cols)) {
        // records + ticket, zeroed in stream order (capture-safe); the replay records need no reset
        unsigned* ticket = static_cast<unsigned*>(ws);
        SegRec* recs = reinterpret_cast<SegRec*>(static_cast<char*>(ws) + 256);
        const int64_t rec_bytes = seg_rec_bytes(n_streams, P);
        cudaMemsetAsync(ws, 0, rec_bytes, st);
        const int64_t units = n_streams * P.n_chunks;
        double* rec_x = reinterpret_cast<double*>(static_cast<char*>(ws) + rec_bytes);
        unsigned* rec_o = reinterpret_cast<unsigned*>(rec_x + units * P.G * 32);
        const int64_t want = (units + kSegWarps - 1) / kSegWarps;
        const int blocks = (int)(want < 16LL * kNumSMs ? want : 16LL * kNumSMs);
        noise_seg_kernel<<<blocks, kSegWarps * 32, 0, st>>>(L.args, n_jobs, P.n_chunks, P.G, recs,
                                                            ticket, rec_x, rec_o);
        return check_launch("enks_noise_fill(segmented)");
    }
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
                                     const int64_t* ld_plus, void* ws, int64_t ws_bytes,
                                     void* stream) {
    ENKS_REQUIRE(n_jobs >= 1 && n_jobs <= enks::kMaxJobs, "enks_noise_fill_multi: 1..%d jobs",
                 enks::kMaxJobs);
    enks::Job jobs[enks::kMaxJobs];
    for (int q = 0; q < n_jobs; ++q)
        jobs[q] = enks::Job{t[q], channel[q], rows[q], diag[q], out[q], ld_out[q],
                            base[q], ld_base[q], out_plus[q], ld_plus[q]};
    return enks::launch_noise(head, n_head, member0, n_members, cols, jobs, n_jobs,
                              enks::as_stream(stream), nullptr, ws, ws_bytes);
}

extern "C" int64_t enks_noise_ws_bytes(int64_t n_members, int n_jobs, int max_rows, int cols) {
    return enks::seg_ws_bytes(n_members * n_jobs, (int64_t)max_rows * cols);
}

extern "C" int enks_noise_fill_multi_dev(const uint32_t* head_dev, int n_head, int64_t member0,
                                         int64_t n_members, int cols, int n_jobs,
                                         const uint32_t* t, const uint32_t* channel,
                                         const int* rows, const double* const* diag,
                                         float* const* out, const int64_t* ld_out,
                                         const float* const* base, const int64_t* ld_base,
                                         float* const* out_plus, const int64_t* ld_plus,
                                         void* ws, int64_t ws_bytes, void* stream) {
    ENKS_REQUIRE(head_dev, "enks_noise_fill_multi_dev: null head");
    ENKS_REQUIRE(n_jobs >= 1 && n_jobs <= enks::kMaxJobs, "enks_noise_fill_multi_dev: 1..%d jobs",
                 enks::kMaxJobs);
    enks::Job jobs[enks::kMaxJobs];
    for (int q = 0; q < n_jobs; ++q)
        jobs[q] = enks::Job{t[q], channel[q], rows[q], diag[q], out[q], ld_out[q],
                            base[q], ld_base[q], out_plus[q], ld_plus[q]};
    return enks::launch_noise(nullptr, n_head, member0, n_members, cols, jobs, n_jobs,
                              enks::as_stream(stream), head_dev, ws, ws_bytes);
}
