// Bit-exact numpy noise substreams: the per-warp device routine shared by noise.cu (the
// stand-alone launch) and cnn_tc.cu (noise drawn by the fused forecast's idle warps).
// See noise.cu for the algorithm and the reference call sites.
#pragma once
#include <stdint.h>

#include "common.cuh"
#include "ziggurat_tables.h"

namespace enks {
namespace {

constexpr int kBufWords = 256;     // 64 Philox blocks per refill (two per lane: ILP)
constexpr int kMaxRowCols = 256;   // row-staged output path: cols % 4 == 0, 32 <= cols <= 256

__device__ const uint64_t g_ki[256] = NPY_ZIG_KI_DOUBLE_INIT;
__device__ const uint64_t g_wi[256] = NPY_ZIG_WI_DOUBLE_INIT;
__device__ const uint64_t g_fi[256] = NPY_ZIG_FI_DOUBLE_INIT;

struct Head {
    uint32_t w[32];
    int n;
};

// numpy SeedSequence (bit_generator.pyx): hashmix / mix / generate_state(2, uint64)
__device__ __forceinline__ uint32_t hashmix(uint32_t v, uint32_t& h) {
    v ^= h;
    h *= 0x931e8875u;
    v *= h;
    v ^= v >> 16;
    return v;
}
__device__ __forceinline__ uint32_t mixw(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
}

__device__ void seed_key(const Head& hd, uint32_t i, uint32_t t, uint32_t ch, uint64_t& k0,
                         uint64_t& k1) {
    // entropy = hd.w[0..n) ++ [i, t, ch];  n >= 4 (seed words are padded to the pool size)
    uint32_t pool[4];
    uint32_t h = 0x43b0d7e5u;
#pragma unroll
    for (int q = 0; q < 4; ++q) pool[q] = hashmix(hd.w[q], h);
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], h));
    for (int s = 4; s < hd.n + 3; ++s) {
        uint32_t e = s < hd.n ? hd.w[s] : (s == hd.n ? i : (s == hd.n + 1 ? t : ch));
#pragma unroll
        for (int d = 0; d < 4; ++d) pool[d] = mixw(pool[d], hashmix(e, h));
    }
    uint32_t hb = 0x8b51f9ddu, w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t v = pool[q] ^ hb;
        hb *= 0x58f38dedu;
        v *= hb;
        w[q] = v ^ (v >> 16);
    }
    k0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    k1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

// Philox4x64-10; numpy increments the 256-bit counter before each block, so
// uint64 word `w` of a fresh stream comes from counter (w/4 + 1, 0, 0, 0).
struct Block4 {
    uint64_t v0, v1, v2, v3;
};
__device__ __forceinline__ Block4 philox(uint64_t k0, uint64_t k1, uint64_t ctr) {
    uint64_t c0 = ctr, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        const uint64_t m0 = 0xD2E7470EE14C6C93ULL, m1 = 0xCA5A826395121157ULL;
        uint64_t hi0 = __umul64hi(m0, c0), lo0 = m0 * c0;
        uint64_t hi1 = __umul64hi(m1, c2), lo1 = m1 * c2;
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return {c0, c1, c2, c3};
}

struct Job {
    uint32_t t, ch;
    int rows;
    const double* diag;
    float* out;
    int64_t ld_out;
    const float* base;
    int64_t ld_base;
    float* out_plus;
    int64_t ld_plus;
};

constexpr int kMaxJobs = 4;

struct Args {
    Head head;
    const uint32_t* head_dev;  // non-null: head words read from device memory (graph replays)
    int64_t member0, n_members;
    int cols;
    Job job[kMaxJobs];
};

__device__ __forceinline__ double u64_to_unit(uint64_t r) {
    return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

// RB (row-staged): the normals of a row are collected in shared memory (two row slots) and
// written as float4 once the row is complete, with the row's `base` values and diagonal
// scale prefetched a row ahead -- the sequential stream never waits on a global load.
// Otherwise each batch of accepted normals is stored straight away (any cols / alignment).
//
// One warp draws the whole substream (member0 + local, a.t, a.ch) of job `a`.  Shared memory:
// s_row (2 kMaxRowCols floats, RB only) and buf (kBufWords words) private to the warp; s_ki /
// s_wi the ziggurat tables (load_tables).  Called by noise_kernel and by the fused CNN forecast
// (cnn_tc.cu), whose otherwise idle warps draw the step's noise next to the convolution.
__device__ __forceinline__ void load_tables(uint64_t* s_ki, double* s_wi, int tid, int nthreads) {
    for (int q = tid; q < 256; q += nthreads) {
        s_ki[q] = g_ki[q];
        s_wi[q] = __longlong_as_double((long long)g_wi[q]);
    }
}

// One group of 32 consecutive words w .. w+31 (lane = word): the ziggurat fast test of every
// word as if it started a normal, numpy's sequential parse resolved on bitmasks.  In: `carry`
// words at the group start already consumed by an earlier normal.  Out: O (words that emit a
// normal; lane's value in x), next_carry.  `word(ww)` returns any word of the stream (uniform).
template <typename WordFn>
__device__ __forceinline__ void resolve_group(uint64_t raw, int w, int carry, int lane,
                                              const uint64_t* s_ki, const double* s_wi,
                                              WordFn&& word, double& x, unsigned& O,
                                              int& next_carry) {
    const int idx = (int)(raw & 0xff);
    const uint64_t r = raw >> 8;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    x = (double)rabs * s_wi[idx];
    if (r & 1) x = -x;
    const bool ok = rabs < s_ki[idx];
    const unsigned bad = __ballot_sync(0xffffffffu, !ok);
    unsigned S = carry >= 32 ? 0u : (0xffffffffu << carry);  // words that start a normal
    next_carry = carry >= 32 ? carry - 32 : 0;
    O = S;  // words that emit a normal
    if (bad & S) {
        // speculative wedge test of every failing word with the following word as uniform
        uint64_t nxt = __shfl_down_sync(0xffffffffu, raw, 1);
        if (bad >> 31) {
            const uint64_t n31 = word(w + 32);
            if (lane == 31) nxt = n31;
        }
        bool acc = false;
        if (!ok && idx != 0) {
            const double fa = __longlong_as_double((long long)g_fi[idx - 1]);
            const double fb = __longlong_as_double((long long)g_fi[idx]);
            const double uu = u64_to_unit(nxt);
            // numpy: accept iff (fa - fb) uu + fb < exp(-x^2 / 2) in double.  Decide with a
            // single-precision exp (ex2.approx, ~2^-22 relative) when the margin is wide,
            // and fall back to the double exp only near the boundary: same decisions.
            const double lhs = (fa - fb) * uu + fb;
            const float ef = exp2f(-0.72134752044448170f * (float)(x * x));  // e^{-x^2/2}
            if (lhs < (double)ef * (1.0 - 4e-6))
                acc = true;
            else if (lhs > (double)ef * (1.0 + 4e-6))
                acc = false;
            else
                acc = lhs < exp(-0.5 * x * x);
        }
        unsigned accm = __ballot_sync(0xffffffffu, acc);
        unsigned todo = bad & S;
        while (todo) {  // warp-uniform walk over the failing starts, in word order
            const int b = __ffs(todo) - 1;
            todo &= todo - 1;
            const int idb = __shfl_sync(0xffffffffu, idx, b);
            int used;  // words consumed after word b
            if (idb != 0) {
                used = 1;
            } else {  // tail: pairs of uniforms until accepted (numpy's loop, uniform)
                const uint64_t rb_raw = __shfl_sync(0xffffffffu, raw, b);
                const uint64_t ra = ((rb_raw >> 8) >> 1) & 0x000fffffffffffffULL;
                int ww = w + b + 1;
                double val;
                for (;;) {
                    const double xx = -NPY_ZIG_NOR_INV_R * log1p(-u64_to_unit(word(ww)));
                    const double yy = -log1p(-u64_to_unit(word(ww + 1)));
                    ww += 2;
                    if (yy + yy > xx * xx) {
                        val = ((ra >> 8) & 1) ? -(NPY_ZIG_NOR_R + xx) : NPY_ZIG_NOR_R + xx;
                        break;
                    }
                }
                used = ww - (w + b + 1);
                if (lane == b) x = val;
                accm |= 1u << b;
            }
            // the consumed words start no normal
            const int e = b + 1 + used;  // first word after this normal (group-relative)
            const unsigned span = (e >= 32 ? 0xffffffffu : ((1u << e) - 1u)) & ~((2u << b) - 1u);
            S &= ~span;
            todo &= ~span;
            if (e > 32) next_carry = e - 32;
        }
        O = S & (~bad | accm);
    }
}

template <bool RB>
__device__ __forceinline__ void run_stream(const Args& args, const Job& a, int64_t local, int lane,
                                           float* s_row, uint64_t* buf, const uint64_t* s_ki,
                                           const double* s_wi) {
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
    const int cols = args.cols;

    // 32-bit stream positions: a stream holds rows * cols < 2^31 normals (checked on the host)
    const int total = a.rows * cols;
    const int64_t col0 = local * cols;
    int base_w = -(1 << 30);  // buffer holds words [base_w, base_w + kBufWords)
    int w = 0, q = 0;

    // (row, col) of normal q, tracked incrementally: (rb, jb) is the position of q (warp-uniform)
    int rb = 0, jb = 0;
    auto advance = [&](int k) {
        jb += k;
        while (jb >= cols) {
            jb -= cols;
            ++rb;
        }
    };
    auto emit = [&](int off, double x) {  // normal q + off
        int r = rb, j = jb + off;
        while (j >= cols) {
            j -= cols;
            ++r;
        }
        const double v = a.diag ? x * a.diag[r] : x;
        const float f = (float)v;
        if (a.out) a.out[r * a.ld_out + col0 + j] = f;
        if (a.out_plus) a.out_plus[r * a.ld_plus + col0 + j] = a.base[r * a.ld_base + col0 + j] + f;
    };
    // ---- row-staged output (RB)
    double dcur = 0.0, dnext = 0.0;
    float4 bpre[kMaxRowCols / 128];
    auto load_diag = [&](int r) { return (a.diag && r < a.rows) ? a.diag[r] : 1.0; };
    auto prefetch_base = [&](int r) {
        if constexpr (RB) {
            if (!a.out_plus || r >= a.rows) return;
#pragma unroll
            for (int i = 0; i < kMaxRowCols / 128; ++i) {
                const int c = lane * 4 + i * 128;
                if (c < cols)
                    bpre[i] = __ldg(reinterpret_cast<const float4*>(a.base + r * a.ld_base + col0 + c));
            }
        }
    };
    auto flush = [&](int r) {
        __syncwarp();
        const float* row = s_row + (r & 1) * kMaxRowCols;
#pragma unroll
        for (int i = 0; i < kMaxRowCols / 128; ++i) {
            const int c = lane * 4 + i * 128;
            if (c < cols) {
                const float4 v = *reinterpret_cast<const float4*>(row + c);
                if (a.out) *reinterpret_cast<float4*>(a.out + r * a.ld_out + col0 + c) = v;
                if (a.out_plus) {
                    const float4 b = bpre[i];
                    *reinterpret_cast<float4*>(a.out_plus + r * a.ld_plus + col0 + c) =
                        make_float4(b.x + v.x, b.y + v.y, b.z + v.z, b.w + v.w);
                }
            }
        }
        __syncwarp();
    };
    auto emit_rb = [&](int off, double x) {
        int j = jb + off, slot = rb & 1;
        double dg = dcur;
        if (j >= cols) {
            j -= cols;
            slot ^= 1;
            dg = dnext;
        }
        const double v = a.diag ? x * dg : x;
        s_row[slot * kMaxRowCols + j] = (float)v;
    };
    auto advance_rb = [&](int k) {
        jb += k;
        if (jb >= cols) {  // k <= 32 <= cols: at most one row completes
            jb -= cols;
            flush(rb);
            ++rb;
            dcur = dnext;
            dnext = load_diag(rb + 1);
            prefetch_base(rb);
        }
    };
    if (RB) {
        dcur = load_diag(0);
        dnext = load_diag(1);
        prefetch_base(0);
    }

    // warp-uniform access to word `ww` (slow path only)
    auto word = [&](int ww) -> uint64_t {
        if (ww >= base_w && ww < base_w + kBufWords) return buf[ww - base_w];
        Block4 b = philox(k0, k1, (uint64_t)(ww >> 2) + 1);
        int s = (int)(ww & 3);
        return s == 0 ? b.v0 : (s == 1 ? b.v1 : (s == 2 ? b.v2 : b.v3));
    };

    // Each iteration consumes a group of 32 consecutive words (w .. w+31) completely: every lane
    // classifies its word as if it started a normal (ziggurat fast accept), and the sequential
    // structure of numpy's parse is resolved on bitmasks.  A word that fails the fast test and
    // really starts a normal (bit set in S) either takes the next word as its wedge uniform (wedge:
    // that word is no start) or starts a tail loop that consumes 2k further words; `carry` counts
    // consumed words that spill into the next group.  All wedge tests are evaluated speculatively
    // in parallel (one lane per failing word); only tails (~1 in 10^4 words) run warp-uniformly.
    const unsigned lt_mask = (1u << lane) - 1u;
    int carry = 0;
    while (q < total) {
        if (w >= base_w + kBufWords) {  // w is a multiple of 32; windows of kBufWords words
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
        const int n_emit = min(__popc(O), total - q);
        const int pos = __popc(O & lt_mask);
        if ((O >> lane) & 1u) {
            if (pos < n_emit) {
                if (RB)
                    emit_rb(pos, x);
                else
                    emit(pos, x);
            }
        }
        q += n_emit;
        w += 32;
        if (RB)
            advance_rb(n_emit);
        else
            advance(n_emit);
    }
}


// Host: pack the launch arguments of n_jobs jobs and decide the row-staged (RB) path.
struct NoiseLaunch {
    Args args;
    int n_jobs = 0;
    bool rb = false;
};

inline int make_noise_launch(const uint32_t* head, int n_head, const uint32_t* head_dev,
                             int64_t member0, int64_t n_members, int cols, const Job* jobs,
                             int n_jobs, NoiseLaunch& L) {
    ENKS_REQUIRE((head != nullptr || head_dev != nullptr) && n_head >= 4 && n_head <= 32,
                 "enks_noise_fill: need 4..32 head words (seed padded to 4 + prefix), got %d",
                 n_head);
    ENKS_REQUIRE(n_jobs >= 1 && n_jobs <= kMaxJobs, "enks_noise_fill: 1..%d jobs", kMaxJobs);
    ENKS_REQUIRE(member0 >= 0 && member0 + n_members <= (1LL << 32),
                 "enks_noise_fill: member ids must fit in uint32");
    Args& a = L.args;
    for (int q = 0; q < 32; ++q) a.head.w[q] = (head && q < n_head) ? head[q] : 0u;
    a.head.n = n_head;
    a.head_dev = head_dev;
    a.member0 = member0;
    a.n_members = n_members;
    a.cols = cols;
    for (int j = 0; j < n_jobs; ++j) {
        ENKS_REQUIRE(jobs[j].out || jobs[j].out_plus, "enks_noise_fill: job %d has no output", j);
        ENKS_REQUIRE(!jobs[j].out_plus || jobs[j].base, "enks_noise_fill: out_plus needs base");
        ENKS_REQUIRE(jobs[j].rows > 0, "enks_noise_fill: job %d has no rows", j);
        ENKS_REQUIRE((int64_t)jobs[j].rows * cols < (1LL << 30),
                     "enks_noise_fill: rows * cols must be < 2^30 per stream");
        a.job[j] = jobs[j];
    }
    L.n_jobs = n_jobs;
    // row-staged path when every job's rows can be written as aligned float4 rows
    bool rb = cols % 4 == 0 && cols >= 32 && cols <= kMaxRowCols;
    auto al16 = [](const void* ptr) { return ((uintptr_t)ptr & 15) == 0; };
    for (int j = 0; j < n_jobs && rb; ++j) {
        const Job& q = a.job[j];
        rb = (!q.out || (al16(q.out) && q.ld_out % 4 == 0)) &&
             (!q.out_plus || (al16(q.out_plus) && q.ld_plus % 4 == 0 && al16(q.base) &&
                              q.ld_base % 4 == 0));
    }
    L.rb = rb;
    return ENKS_OK;
}

}  // namespace
}  // namespace enks
