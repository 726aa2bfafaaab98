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
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace enks {
namespace {

constexpr int kSumThreads = 128;

__global__ void __launch_bounds__(kSumThreads)
    member_partial_kernel(const float* __restrict__ src, int64_t ld, const float* __restrict__ src2,
                          int64_t ld2, int rows, int64_t n, int cols,
                          const float* __restrict__ z0, double* __restrict__ part,
                          float* __restrict__ partmax, int64_t chunk) {
    const int64_t rc = (int64_t)rows * cols;
    const int64_t e = blockIdx.x * (int64_t)kSumThreads + threadIdx.x;
    if (e >= rc) return;
    const int r = (int)(e / cols), j = (int)(e - (int64_t)r * cols);
    const float* p = src + r * ld + j;
    const float* p2 = src2 ? src2 + r * ld2 + j : nullptr;
    // element value: src (+ src2, the perturbed observation x + v formed on the fly)
    auto val = [&](int64_t i) { return p2 ? p[i * cols] + p2[i * cols] : p[i * cols]; };
    const float s = z0 ? z0[e] : val(0);
    const int64_t i0 = blockIdx.y * chunk, i1 = min(n, i0 + chunk);
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    float mx = 0.f;
    int64_t i = i0;
    for (; i + 4 <= i1; i += 4) {
        float v0 = val(i + 0) - s, v1 = val(i + 1) - s;
        float v2 = val(i + 2) - s, v3 = val(i + 3) - s;
        acc0 += (double)v0;
        acc1 += (double)v1;
        acc2 += (double)v2;
        acc3 += (double)v3;
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v0), fabsf(v1)), fmaxf(fabsf(v2), fabsf(v3))));
    }
    for (; i < i1; ++i) {
        const float v = val(i) - s;
        acc0 += (double)v;
        mx = fmaxf(mx, fabsf(v));
    }
    part[blockIdx.y * rc + e] = (acc0 + acc1) + (acc2 + acc3);
    partmax[blockIdx.y * rc + e] = mx;
}

// vectorised variant: 4 consecutive columns per thread (cols % 4 == 0, 16-B aligned rows), so a
// warp reads one 512-B member row per load and keeps 4 members (8 with src2) of loads in flight.
// Per element the member order and the four interleaved fp64 chains are those of the scalar
// kernel above (bit-identical partials).
__global__ void __launch_bounds__(kSumThreads)
    member_partial_v4_kernel(const float* __restrict__ src, int64_t ld, const float* __restrict__ src2,
                             int64_t ld2, int rows, int64_t n, int cols,
                             const float* __restrict__ z0, double* __restrict__ part,
                             float* __restrict__ partmax, int64_t chunk) {
    const int64_t rc = (int64_t)rows * cols;
    const int64_t e = (blockIdx.x * (int64_t)kSumThreads + threadIdx.x) * 4;
    if (e >= rc) return;
    const int r = (int)(e / cols), j = (int)(e - (int64_t)r * cols);
    const float* p = src + r * ld + j;
    const float* p2 = src2 ? src2 + r * ld2 + j : nullptr;
    auto val = [&](int64_t i) {
        float4 v = __ldg(reinterpret_cast<const float4*>(p + i * cols));
        if (p2) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(p2 + i * cols));
            v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
        }
        return v;
    };
    const float4 s = z0 ? __ldg(reinterpret_cast<const float4*>(z0 + e)) : val(0);
    const int64_t i0 = blockIdx.y * chunk, i1 = min(n, i0 + chunk);
    double acc[4][4] = {};
    float mx[4] = {0.f, 0.f, 0.f, 0.f};
    auto add = [&](int c, const float4& v) {
        const float d0 = v.x - s.x, d1 = v.y - s.y, d2 = v.z - s.z, d3 = v.w - s.w;
        acc[c][0] += (double)d0;
        acc[c][1] += (double)d1;
        acc[c][2] += (double)d2;
        acc[c][3] += (double)d3;
        mx[0] = fmaxf(mx[0], fabsf(d0));
        mx[1] = fmaxf(mx[1], fabsf(d1));
        mx[2] = fmaxf(mx[2], fabsf(d2));
        mx[3] = fmaxf(mx[3], fabsf(d3));
    };
    int64_t i = i0;
    for (; i + 4 <= i1; i += 4) {
        const float4 v0 = val(i + 0), v1 = val(i + 1), v2 = val(i + 2), v3 = val(i + 3);
        add(0, v0);
        add(1, v1);
        add(2, v2);
        add(3, v3);
    }
    for (; i < i1; ++i) add(0, val(i));
    double out[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = (acc[0][q] + acc[1][q]) + (acc[2][q] + acc[3][q]);
    double* po = part + blockIdx.y * rc + e;
    reinterpret_cast<double2*>(po)[0] = make_double2(out[0], out[1]);
    reinterpret_cast<double2*>(po)[1] = make_double2(out[2], out[3]);
    *reinterpret_cast<float4*>(partmax + blockIdx.y * rc + e) = make_float4(mx[0], mx[1], mx[2], mx[3]);
}

// Both member sums of one predict in one pass (4 columns per thread): the slice sums of src (all
// rows) and, for rows < rows2, the observation sums of src + src2 (the perturbed observation
// x + v formed on the fly) -- src's first rows2 rows are read once instead of twice.  Shifts are
// each quantity's first member (z0 = NULL semantics); per element the member order and the four
// interleaved fp64 chains are those of the kernels above.
__global__ void __launch_bounds__(kSumThreads)
    member_partial2_v4_kernel(const float* __restrict__ src, int64_t ld, int rows,
                              const float* __restrict__ src2, int64_t ld2, int rows2, int64_t n,
                              int cols, double* __restrict__ part, float* __restrict__ partmax,
                              double* __restrict__ part2, float* __restrict__ partmax2,
                              int64_t chunk) {
    const int64_t rc = (int64_t)rows * cols, rc2 = (int64_t)rows2 * cols;
    const int64_t e = (blockIdx.x * (int64_t)kSumThreads + threadIdx.x) * 4;
    if (e >= rc) return;
    const int r = (int)(e / cols), j = (int)(e - (int64_t)r * cols);
    const bool two = r < rows2;
    const float* p = src + r * ld + j;
    const float* p2 = two ? src2 + r * ld2 + j : nullptr;
    auto ld4 = [](const float* q) { return __ldg(reinterpret_cast<const float4*>(q)); };
    auto plus = [](float4 a, const float4& b) {
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        return a;
    };
    const float4 s = ld4(p);
    const float4 s2 = two ? plus(s, ld4(p2)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t i0 = blockIdx.y * chunk, i1 = min(n, i0 + chunk);
    double acc[4][4] = {}, acc2[4][4] = {};
    float mx[4] = {0.f, 0.f, 0.f, 0.f}, mx2[4] = {0.f, 0.f, 0.f, 0.f};
    auto add = [](double (&a)[4][4], float (&m)[4], int c, const float4& v, const float4& z) {
        const float d0 = v.x - z.x, d1 = v.y - z.y, d2 = v.z - z.z, d3 = v.w - z.w;
        a[c][0] += (double)d0;
        a[c][1] += (double)d1;
        a[c][2] += (double)d2;
        a[c][3] += (double)d3;
        m[0] = fmaxf(m[0], fabsf(d0));
        m[1] = fmaxf(m[1], fabsf(d1));
        m[2] = fmaxf(m[2], fabsf(d2));
        m[3] = fmaxf(m[3], fabsf(d3));
    };
    int64_t i = i0;
    if (two) {
        for (; i + 4 <= i1; i += 4) {
            float4 v[4], w[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                v[c] = ld4(p + (i + c) * cols);
                w[c] = ld4(p2 + (i + c) * cols);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                add(acc, mx, c, v[c], s);
                add(acc2, mx2, c, plus(v[c], w[c]), s2);
            }
        }
        for (; i < i1; ++i) {
            const float4 v = ld4(p + i * cols);
            add(acc, mx, 0, v, s);
            add(acc2, mx2, 0, plus(v, ld4(p2 + i * cols)), s2);
        }
    } else {
        for (; i + 4 <= i1; i += 4) {
            float4 v[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) v[c] = ld4(p + (i + c) * cols);
#pragma unroll
            for (int c = 0; c < 4; ++c) add(acc, mx, c, v[c], s);
        }
        for (; i < i1; ++i) add(acc, mx, 0, ld4(p + i * cols), s);
    }
    auto store = [&](double* pp, float* pm, int64_t n_el, double (&a)[4][4], float (&m)[4]) {
        double out[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q] = (a[0][q] + a[1][q]) + (a[2][q] + a[3][q]);
        double* po = pp + blockIdx.y * n_el + e;
        reinterpret_cast<double2*>(po)[0] = make_double2(out[0], out[1]);
        reinterpret_cast<double2*>(po)[1] = make_double2(out[2], out[3]);
        *reinterpret_cast<float4*>(pm + blockIdx.y * n_el + e) = make_float4(m[0], m[1], m[2], m[3]);
    };
    store(part, partmax, rc, acc, mx);
    if (two) store(part2, partmax2, rc2, acc2, mx2);
}

__global__ void chunk_reduce_kernel(const double* __restrict__ part, const float* __restrict__ pmax,
                                    int nchunks, int64_t rc, double* __restrict__ acc,
                                    float* __restrict__ amax) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= rc) return;
    double s = 0.0;
    float mx = 0.f;
    for (int c = 0; c < nchunks; ++c) {
        s += part[c * rc + e];
        mx = fmaxf(mx, pmax[c * rc + e]);
    }
    acc[e] = s;
    if (amax) amax[e] = mx;
}

// acc[r, j] += coef * s[r, j], s = src[r, j] (+ src2[r, j], summed in fp32 exactly as the member
// sums form their shift): converts shifted member sums to absolute ones and back (multi-rank)
__global__ void sum_rebase_kernel(const float* __restrict__ src, int64_t ld,
                                  const float* __restrict__ src2, int64_t ld2, int rows, int cols,
                                  double* __restrict__ acc, double coef) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= (int64_t)rows * cols) return;
    const int r = (int)(e / cols), j = (int)(e - (int64_t)r * cols);
    const float s = src2 ? src[r * ld + j] + src2[r * ld2 + j] : src[r * ld + j];
    acc[e] += coef * (double)s;
}

// basis row of source row r when rows [skip0, skip1) are not stored in the basis (-1: skipped)
__device__ __forceinline__ int basis_row(int r, int skip0, int skip1) {
    return r < skip0 ? r : (r >= skip1 ? r - (skip1 - skip0) : -1);
}

// per-row power-of-two scale for the fp16-pair basis from a guaranteed bound on the anomalies:
// |anom| = |(src - z0) - mu| <= max|src - z0| + |mu|.  scale = 2^e with bound * scale in [2^13, 2^14)
__global__ void row_scale_kernel(const double* __restrict__ acc, const float* __restrict__ amax,
                                 double inv_n, int cols, float* __restrict__ scale,
                                 float* __restrict__ inv_scale, int skip0, int skip1) {
    const int r = blockIdx.x;
    float b = 0.f;
    for (int j = threadIdx.x; j < cols; j += blockDim.x) {
        const float mu = (float)(acc[(int64_t)r * cols + j] * inv_n);
        b = fmaxf(b, amax[(int64_t)r * cols + j] + fabsf(mu));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
    __shared__ float red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) m = fmaxf(m, red[w]);
        int e = 0;
        if (m > 0.f && isfinite(m)) {
            int ex;
            frexpf(m * 1.0001f, &ex);
            e = max(-120, min(120, 14 - ex));
        }
        scale[r] = ldexpf(1.f, e);
        const int hr = basis_row(r, skip0, skip1);
        if (hr >= 0) inv_scale[hr] = ldexpf(1.f, -e);
    }
}

// anomalies straight into the fp16-pair basis (+ optional fp32 copy of the first rows_f32 rows)
__global__ void center_f16pair_kernel(const float* __restrict__ src, int64_t ld, int rows, int64_t n,
                                      int cols, const float* __restrict__ z0,
                                      const double* __restrict__ acc, double inv_n,
                                      float* __restrict__ mean, __half* __restrict__ h,
                                      __half* __restrict__ l, int64_t ldh,
                                      const float* __restrict__ scale, float* __restrict__ f32,
                                      int64_t ldf, int rows_f32, int skip0, int skip1) {
    const int64_t K = n * cols;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (k >= K) return;
    const int j = (int)((uint32_t)k % (uint32_t)cols);
    const float s = z0 ? z0[r * cols + j] : src[r * ld + j];
    const float mu = (float)(acc[r * cols + j] * inv_n);
    if (mean && k < cols) mean[r * cols + j] = s + mu;
    const float a = (src[r * ld + k] - s) - mu;
    if (f32 && r < rows_f32) f32[r * ldf + k] = a;
    const int64_t hr = basis_row((int)r, skip0, skip1);
    if (hr < 0) return;
    const float v = a * scale[r];
    const __half hv = __float2half_rn(v);
    h[hr * ldh + k] = hv;
    l[hr * ldh + k] = __float2half_rn(v - __half2float(hv));
}

// vectorised variant: 4 consecutive columns per thread (cols % 4 == 0, 16-B aligned rows)
// src2 (optional): the centred quantity is src + src2, formed on the fly (the perturbed
// observation [x; u] + [v_x; v_u]); the member-0 shift is then src + src2 of member 0 as well
__global__ void center_f16pair_v4_kernel(const float* __restrict__ src, int64_t ld, int rows,
                                         int64_t n, int cols, const float* __restrict__ z0,
                                         const double* __restrict__ acc, double inv_n,
                                         float* __restrict__ mean, __half* __restrict__ h,
                                         __half* __restrict__ l, int64_t ldh,
                                         const float* __restrict__ scale, float* __restrict__ f32,
                                         int64_t ldf, int rows_f32, int skip0, int skip1,
                                         const float* __restrict__ src2, int64_t ld2) {
    const int64_t K = n * cols;
    const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
    const int64_t r = blockIdx.y;
    if (k >= K) return;
    const int j = (int)((uint32_t)k % (uint32_t)cols);
    float4 x = __ldg(reinterpret_cast<const float4*>(src + r * ld + k));
    float4 zz = __ldg(reinterpret_cast<const float4*>(z0 ? z0 + r * cols + j : src + r * ld + j));
    if (src2) {
        const float4 x2 = __ldg(reinterpret_cast<const float4*>(src2 + r * ld2 + k));
        x = make_float4(x.x + x2.x, x.y + x2.y, x.z + x2.z, x.w + x2.w);
        if (!z0) {
            const float4 z2 = __ldg(reinterpret_cast<const float4*>(src2 + r * ld2 + j));
            zz = make_float4(zz.x + z2.x, zz.y + z2.y, zz.z + z2.z, zz.w + z2.w);
        }
    }
    const double2 a01 = __ldg(reinterpret_cast<const double2*>(acc + r * cols + j));
    const double2 a23 = __ldg(reinterpret_cast<const double2*>(acc + r * cols + j + 2));
    const float m0 = (float)(a01.x * inv_n), m1 = (float)(a01.y * inv_n);
    const float m2 = (float)(a23.x * inv_n), m3 = (float)(a23.y * inv_n);
    if (mean && k < cols)
        *reinterpret_cast<float4*>(mean + r * cols + j) =
            make_float4(zz.x + m0, zz.y + m1, zz.z + m2, zz.w + m3);
    const float4 an = make_float4((x.x - zz.x) - m0, (x.y - zz.y) - m1, (x.z - zz.z) - m2,
                                  (x.w - zz.w) - m3);
    if (f32 && r < rows_f32) *reinterpret_cast<float4*>(f32 + r * ldf + k) = an;
    const int64_t hr = basis_row((int)r, skip0, skip1);
    if (hr < 0) return;
    const float sc = scale[r];
    const float v[4] = {an.x * sc, an.y * sc, an.z * sc, an.w * sc};
    __half hv[4], lv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        hv[q] = __float2half_rn(v[q]);
        lv[q] = __float2half_rn(v[q] - __half2float(hv[q]));
    }
    *reinterpret_cast<uint2*>(h + hr * ldh + k) =
        make_uint2(__half_as_ushort(hv[0]) | ((uint32_t)__half_as_ushort(hv[1]) << 16),
                   __half_as_ushort(hv[2]) | ((uint32_t)__half_as_ushort(hv[3]) << 16));
    *reinterpret_cast<uint2*>(l + hr * ldh + k) =
        make_uint2(__half_as_ushort(lv[0]) | ((uint32_t)__half_as_ushort(lv[1]) << 16),
                   __half_as_ushort(lv[2]) | ((uint32_t)__half_as_ushort(lv[3]) << 16));
}

// mean[r, j] = z0 + mu_sh; anom[r, i*cols + j] = (src - z0) - mu_sh
__global__ void center_kernel(const float* __restrict__ src, int64_t ld, int rows, int64_t n,
                              int cols, const float* __restrict__ z0,
                              const double* __restrict__ acc, double inv_n, float* __restrict__ mean,
                              float* anom, int64_t lda) {
    const int64_t K = n * cols;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t r = blockIdx.y;
    if (k >= K) return;
    const int j = (int)((uint32_t)k % (uint32_t)cols);
    const float s = z0 ? z0[r * cols + j] : src[r * ld + j];
    const float mu = (float)(acc[r * cols + j] * inv_n);
    if (mean && k < cols) mean[r * cols + j] = s + mu;
    if (anom) anom[r * lda + k] = (src[r * ld + k] - s) - mu;
}

// Observation centring with the sum x + v formed on the fly (src + src2) that also writes the
// transposed fp16-pair planes of Yc_tau (K x rows, per-K-row scale) that the newest-slice shift
// consumes as its K-major B operand -- no materialised observation, no separate transpose pass.
// One CTA per 32 consecutive K columns: anomalies of all `rows` rows are kept in shared memory.
constexpr int kTMaxRows = 256;
__global__ void __launch_bounds__(256) center_f16pair_t_kernel(
    const float* __restrict__ src, int64_t ld, const float* __restrict__ src2, int64_t ld2, int rows,
    int64_t n, int cols, const float* __restrict__ z0, const double* __restrict__ acc, double inv_n,
    float* __restrict__ mean, __half* __restrict__ h, __half* __restrict__ l, int64_t ldh,
    const float* __restrict__ scale, __half* __restrict__ th, __half* __restrict__ tl, int64_t ldt,
    float* __restrict__ t_inv) {
    __shared__ float tile[kTMaxRows][33];
    __shared__ float red[8][33];
    __shared__ float sc[32];
    const int64_t K = n * cols;
    const int64_t c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t c = c0 + tx;
    const bool in = c < K;
    const int j = in ? (int)((uint64_t)c % (uint64_t)cols) : 0;
    float mx = 0.f;
    // rows in batches of kB per warp: all loads of a batch are issued before any use, so each warp
    // keeps kB (2 kB with src2) 128-B row segments in flight
    // rows in batches of kB per warp: every load of a batch is issued before any arithmetic (the
    // x + v and member-0 sums happen after the batch), so each warp keeps up to 4 kB 128-B row
    // segments in flight instead of waiting on each row
    constexpr int kB = 4;
    const float* s1 = z0 ? z0 : src;  // member-0 shift: z0[r, j], or src[r, j] (+ src2[r, j])
    const int64_t ld_s1 = z0 ? cols : ld;
    for (int r0 = ty; r0 < rows; r0 += 8 * kB) {
        float x1[kB], x2[kB], z1[kB], z2[kB];
        double av[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int r = r0 + 8 * b;
            const bool ok = in && r < rows;
            x1[b] = ok ? src[r * ld + c] : 0.f;
            x2[b] = ok && src2 ? src2[r * ld2 + c] : 0.f;
            z1[b] = ok ? s1[r * ld_s1 + j] : 0.f;
            z2[b] = ok && !z0 && src2 ? src2[r * ld2 + j] : 0.f;
            av[b] = ok ? __ldg(acc + (int64_t)r * cols + j) : 0.0;
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
            const int r = r0 + 8 * b;
            if (r >= rows) break;
            float a = 0.f;
            if (in) {
                const float x = x1[b] + x2[b], s = z1[b] + z2[b];
                const float mu = (float)(av[b] * inv_n);
                if (mean && c < cols) mean[(int64_t)r * cols + j] = s + mu;
                a = (x - s) - mu;
                const float v = a * scale[r];
                const __half hv = __float2half_rn(v);
                h[r * ldh + c] = hv;
                l[r * ldh + c] = __float2half_rn(v - __half2float(hv));
            }
            if (th) {
                tile[r][tx] = a;
                mx = fmaxf(mx, fabsf(a));
            }
        }
    }
    if (!th) return;  // no transposed planes (the shift reads Yc_tau MN-major)
    red[ty][tx] = mx;
    __syncthreads();
    if (ty == 0) {
        float m = red[0][tx];
        for (int q = 1; q < 8; ++q) m = fmaxf(m, red[q][tx]);
        int e = 0;
        if (m > 0.f && isfinite(m)) {
            int ex;
            frexpf(m, &ex);
            e = max(-120, min(120, 14 - ex));
        }
        sc[tx] = ldexpf(1.f, e);
        if (in) t_inv[c] = ldexpf(1.f, -e);
    }
    __syncthreads();
    for (int jj = ty; jj < 32; jj += 8) {  // transposed row c0 + jj, lanes over pairs of rows
        const int64_t oc = c0 + jj;
        if (oc >= K) break;
        const float s = sc[jj];
        for (int r = 2 * tx; r < rows; r += 64) {
            const float v0 = tile[r][jj] * s;
            const float v1 = r + 1 < rows ? tile[r + 1][jj] * s : 0.f;
            const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
            const __half l0 = __float2half_rn(v0 - __half2float(h0));
            const __half l1 = __float2half_rn(v1 - __half2float(h1));
            if (r + 1 < rows) {
                *reinterpret_cast<__half2*>(th + oc * ldt + r) = __halves2half2(h0, h1);
                *reinterpret_cast<__half2*>(tl + oc * ldt + r) = __halves2half2(l0, l1);
            } else {
                th[oc * ldt + r] = h0;
                tl[oc * ldt + r] = l0;
            }
        }
    }
}

// Derived-U chain (engine.py, "u-chain"): the slice rows [X; U; dU] satisfy U_s = U_{s-1} + dU_s
// member-wise (enks.py:168 appends u + w next to w, and every update is linear), so the basis keeps
// only [X; dU] (ds = n + l rows per slice) and U follows by prefix sums over slices.
// delta: compact mean increments G_{tau,.} (y_ref - y_bar), slices 1..ns (ds rows each, ld_delta);
// mean: full layout from slice 1 (d = n + 2l rows each, ld_mean).  Thread per (compact row, col).
__global__ void uchain_mean_kernel(const float* __restrict__ delta, int64_t ld_delta,
                                   float* __restrict__ mean, int64_t ld_mean, int ns, int n, int l,
                                   int m) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;  // 0 .. n + l - 1
    if (j >= m) return;
    const int ds = n + l, d = n + 2 * l;
    // slices in batches of kU with every load of a batch issued before its stores: the walk over
    // slices is a dependent chain of global latencies otherwise (~0.5 us per slice)
    constexpr int kU = 8;
    if (r < n) {
        for (int s0 = 0; s0 < ns; s0 += kU) {
            float dv[kU], mv[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int s = s0 + u;
                dv[u] = s < ns ? delta[(int64_t)(s * ds + r) * ld_delta + j] : 0.f;
                mv[u] = s < ns ? mean[(int64_t)(s * d + r) * ld_mean + j] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (s0 + u < ns) mean[(int64_t)((s0 + u) * d + r) * ld_mean + j] = mv[u] + dv[u];
        }
        return;
    }
    const int ru = r - n;
    float run = 0.f;
    for (int s0 = 0; s0 < ns; s0 += kU) {
        float dv[kU], mu[kU], md[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int s = s0 + u;
            const bool ok = s < ns;
            dv[u] = ok ? delta[(int64_t)(s * ds + n + ru) * ld_delta + j] : 0.f;
            mu[u] = ok ? mean[(int64_t)(s * d + n + ru) * ld_mean + j] : 0.f;
            md[u] = ok ? mean[(int64_t)(s * d + n + l + ru) * ld_mean + j] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int s = s0 + u;
            if (s >= ns) break;
            run += dv[u];
            mean[(int64_t)(s * d + n + l + ru) * ld_mean + j] = md[u] + dv[u];  // dU_s
            mean[(int64_t)(s * d + n + ru) * ld_mean + j] = mu[u] + run;        // U_s = sum dU
        }
    }
}

// Gain rows of the newest slice [X; U] (q x p): X rows copied from the compact gain column,
// U rows = sum over slices 1..ns of the dU rows (the gain of a prefix sum is the prefix sum of gains)
__global__ void uchain_gain_kernel(const float* __restrict__ g, int64_t ld_g, float* __restrict__ gtt,
                                   int64_t ld_gtt, int ns, int n, int l, int p) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;  // 0 .. n + l - 1
    if (c >= p) return;
    const int ds = n + l;
    float v;
    if (r < n) {
        v = g[(int64_t)((ns - 1) * ds + r) * ld_g + c];
    } else {
        v = 0.f;
        for (int s = 0; s < ns; ++s) v += g[(int64_t)(s * ds + r) * ld_g + c];
    }
    gtt[(int64_t)r * ld_gtt + c] = v;
}

// ENKS_SUM_SCALAR=1: the scalar member-sum kernel (A/B measurements, tools/stats_bench.py)
bool sum_scalar() {
    return env_knob("ENKS_SUM_SCALAR", 0) == 1;
}

// blocks per SM the one-pass member sums aim for (tuning; ENKS_SUM2_BPS, read once)
int sum2_blocks_per_sm() { return env_knob("ENKS_SUM2_BPS", 8); }

// per = columns per thread (4 for the vectorised partial kernel)
int64_t member_chunks(int rows, int64_t n, int cols, int per, int per_sm = 8) {
    const int64_t rc = (int64_t)rows * cols;
    const int64_t blocks = (rc / per + kSumThreads - 1) / kSumThreads;
    // aim for ~per_sm blocks per SM in flight
    int64_t want = ((int64_t)per_sm * kNumSMs + blocks - 1) / blocks;
    if (want > 64) want = 64;
    if (want > n) want = n;
    if (want < 1) want = 1;
    return want;
}

}  // namespace
}  // namespace enks

extern "C" {

int64_t enks_member_sum_ws_bytes(int rows, int64_t n_members, int cols) {
    const int64_t nch = std::max(enks::member_chunks(rows, n_members, cols, 1),
                                 enks::member_chunks(rows, n_members, cols, 4));
    return nch * (int64_t)rows * cols *
           (int64_t)(sizeof(double) + sizeof(float));
}

int64_t enks_member_sum2_ws_bytes(int rows, int rows2, int64_t n_members, int cols) {
    const int64_t nch = enks::member_chunks(rows, n_members, cols, 4, enks::sum2_blocks_per_sm());
    return nch * ((int64_t)rows + rows2) * cols * (int64_t)(sizeof(double) + sizeof(float));
}

int enks_member_sum2(const float* src, int64_t ld_src, int rows, const float* src2,
                     int64_t ld_src2, int rows2, int64_t n_members, int cols, double* acc,
                     float* amax, double* acc2, float* amax2, void* ws, void* stream) {
    ENKS_REQUIRE(src && src2 && acc && acc2 && ws, "enks_member_sum2: null pointer");
    ENKS_REQUIRE(rows2 >= 0 && rows2 <= rows, "enks_member_sum2: rows2 %d outside [0, %d]", rows2,
                 rows);
    auto a16 = [](const void* ptr) { return ((uintptr_t)ptr & 15) == 0; };
    ENKS_REQUIRE(cols % 4 == 0 && ld_src % 4 == 0 && ld_src2 % 4 == 0 && a16(src) && a16(src2),
                 "enks_member_sum2: needs cols %% 4 == 0 and 16-byte aligned rows");
    if (rows <= 0 || cols <= 0) return ENKS_OK;
    const int64_t rc = (int64_t)rows * cols, rc2 = (int64_t)rows2 * cols;
    cudaStream_t st = enks::as_stream(stream);
    if (n_members <= 0) {
        cudaMemsetAsync(acc, 0, rc * sizeof(double), st);
        if (amax) cudaMemsetAsync(amax, 0, rc * sizeof(float), st);
        if (rc2) cudaMemsetAsync(acc2, 0, rc2 * sizeof(double), st);
        if (rc2 && amax2) cudaMemsetAsync(amax2, 0, rc2 * sizeof(float), st);
        return enks::check_launch("enks_member_sum2(memset)");
    }
    const int64_t nch = enks::member_chunks(rows, n_members, cols, 4, enks::sum2_blocks_per_sm());
    const int64_t chunk = (n_members + nch - 1) / nch;
    const int64_t nch_eff = (n_members + chunk - 1) / chunk;
    double* part = static_cast<double*>(ws);
    double* part2 = part + nch * rc;
    float* pmax = reinterpret_cast<float*>(part2 + nch * rc2);
    float* pmax2 = pmax + nch * rc;
    dim3 grid((unsigned)((rc / 4 + enks::kSumThreads - 1) / enks::kSumThreads), (unsigned)nch_eff);
    enks::member_partial2_v4_kernel<<<grid, enks::kSumThreads, 0, st>>>(
        src, ld_src, rows, src2, ld_src2, rows2, n_members, cols, part, pmax, part2, pmax2, chunk);
    int rc_ = enks::check_launch("enks_member_sum2(partial)");
    if (rc_) return rc_;
    enks::chunk_reduce_kernel<<<(unsigned)((rc + 255) / 256), 256, 0, st>>>(part, pmax, (int)nch_eff,
                                                                           rc, acc, amax);
    if (rc2)
        enks::chunk_reduce_kernel<<<(unsigned)((rc2 + 255) / 256), 256, 0, st>>>(
            part2, pmax2, (int)nch_eff, rc2, acc2, amax2);
    return enks::check_launch("enks_member_sum2(reduce)");
}

int enks_member_sum_rebase(const float* src, int64_t ld_src, const float* src2, int64_t ld_src2,
                           int rows, int cols, double* acc, double coef, void* stream) {
    ENKS_REQUIRE(src && acc, "enks_member_sum_rebase: null pointer");
    const int64_t rc = (int64_t)rows * cols;
    if (rc <= 0) return ENKS_OK;
    enks::sum_rebase_kernel<<<(unsigned)((rc + 255) / 256), 256, 0, enks::as_stream(stream)>>>(
        src, ld_src, src2, ld_src2, rows, cols, acc, coef);
    return enks::check_launch("enks_member_sum_rebase");
}

int enks_member_sum(const float* src, int64_t ld_src, const float* src2, int64_t ld_src2, int rows,
                    int64_t n_members, int cols, const float* z0, double* acc, float* amax, void* ws,
                    void* stream) {
    ENKS_REQUIRE(src && acc && ws, "enks_member_sum: null pointer");
    if (rows <= 0 || cols <= 0) return ENKS_OK;
    const int64_t rc = (int64_t)rows * cols;
    cudaStream_t st = enks::as_stream(stream);
    if (n_members <= 0) {
        cudaMemsetAsync(acc, 0, rc * sizeof(double), st);
        if (amax) cudaMemsetAsync(amax, 0, rc * sizeof(float), st);
        return enks::check_launch("enks_member_sum(memset)");
    }
    // The vectorised kernel (4 columns per thread) wins with the on-the-fly sum x + v (two
    // streams: 62 vs 75 us at C3, tools/stats_bench.py); for a single stream the scalar kernel
    // (more resident warps, 52 vs 63 us) does.
    auto a16 = [](const void* ptr) { return ((uintptr_t)ptr & 15) == 0; };
    const bool v4 = !enks::sum_scalar() && src2 && cols % 4 == 0 && ld_src % 4 == 0 && a16(src) &&
                    ld_src2 % 4 == 0 && a16(src2) && (!z0 || a16(z0)) && rc % 4 == 0;
    const int64_t nch = enks::member_chunks(rows, n_members, cols, v4 ? 4 : 1);
    const int64_t chunk = (n_members + nch - 1) / nch;
    const int64_t nch_eff = (n_members + chunk - 1) / chunk;
    double* part = static_cast<double*>(ws);
    const int64_t nch_ws = std::max(enks::member_chunks(rows, n_members, cols, 1),
                                    enks::member_chunks(rows, n_members, cols, 4));
    float* pmax = reinterpret_cast<float*>(part + nch_ws * rc);
    if (v4) {
        dim3 grid((unsigned)((rc / 4 + enks::kSumThreads - 1) / enks::kSumThreads), (unsigned)nch_eff);
        enks::member_partial_v4_kernel<<<grid, enks::kSumThreads, 0, st>>>(
            src, ld_src, src2, ld_src2, rows, n_members, cols, z0, part, pmax, chunk);
    } else {
        dim3 grid((unsigned)((rc + enks::kSumThreads - 1) / enks::kSumThreads), (unsigned)nch_eff);
        enks::member_partial_kernel<<<grid, enks::kSumThreads, 0, st>>>(
            src, ld_src, src2, ld_src2, rows, n_members, cols, z0, part, pmax, chunk);
    }
    int rc_ = enks::check_launch("enks_member_sum(partial)");
    if (rc_) return rc_;
    enks::chunk_reduce_kernel<<<(unsigned)((rc + 255) / 256), 256, 0, st>>>(part, pmax, (int)nch_eff,
                                                                           rc, acc, amax);
    return enks::check_launch("enks_member_sum(reduce)");
}

int enks_member_center(const float* src, int64_t ld_src, int rows, int64_t n_members, int cols,
                       const float* z0, const double* acc, int64_t n_total, float* mean,
                       float* anom, int64_t ld_anom, void* stream) {
    ENKS_REQUIRE(src && acc && n_total > 0, "enks_member_center: bad arguments");
    ENKS_REQUIRE(rows <= 65535, "enks_member_center: rows > 65535");
    ENKS_REQUIRE(!(anom == src && z0 == nullptr),
                 "enks_member_center: in-place centring needs an explicit z0");
    if (rows <= 0 || cols <= 0 || n_members <= 0) return ENKS_OK;
    const int64_t K = n_members * cols;
    enks::center_kernel<<<dim3((unsigned)((K + 255) / 256), (unsigned)rows), 256, 0,
                          enks::as_stream(stream)>>>(
        src, ld_src, rows, n_members, cols, z0, acc, 1.0 / (double)n_total, mean, anom, ld_anom);
    return enks::check_launch("enks_member_center");
}

int enks_member_center_f16pair(const float* src, int64_t ld_src, int rows, int64_t n_members,
                               int cols, const float* z0, const double* acc, const float* amax,
                               int64_t n_total, float* mean, void* h, void* l, int64_t ldh,
                               float* inv_scale, float* scale_ws, float* f32, int64_t ld_f32,
                               int rows_f32, int skip0, int skip1, void* stream) {
    ENKS_REQUIRE(src && acc && amax && h && l && inv_scale && scale_ws && n_total > 0,
                 "enks_member_center_f16pair: bad arguments");
    ENKS_REQUIRE(rows <= 65535, "enks_member_center_f16pair: rows > 65535");
    if (skip1 <= skip0) skip0 = skip1 = rows;
    ENKS_REQUIRE(skip0 >= 0 && skip1 <= rows, "enks_member_center_f16pair: bad skipped rows");
    if (rows <= 0 || cols <= 0 || n_members <= 0) return ENKS_OK;
    cudaStream_t st = enks::as_stream(stream);
    const double inv_n = 1.0 / (double)n_total;
    enks::row_scale_kernel<<<rows, 128, 0, st>>>(acc, amax, inv_n, cols, scale_ws, inv_scale,
                                                   skip0, skip1);
    int rc = enks::check_launch("enks_member_center_f16pair(scale)");
    if (rc) return rc;
    const int64_t K = n_members * cols;
    auto a16 = [](const void* ptr) { return ((uintptr_t)ptr & 15) == 0; };
    const bool v4 = cols % 4 == 0 && ld_src % 4 == 0 && ldh % 4 == 0 && a16(src) &&
                    ((uintptr_t)h & 7) == 0 && ((uintptr_t)l & 7) == 0 && (!z0 || a16(z0)) &&
                    a16(acc) && (!mean || a16(mean)) && (!f32 || (a16(f32) && ld_f32 % 4 == 0));
    if (v4)
        enks::center_f16pair_v4_kernel<<<dim3((unsigned)((K / 4 + 255) / 256), (unsigned)rows), 256,
                                         0, st>>>(
            src, ld_src, rows, n_members, cols, z0, acc, inv_n, mean, static_cast<__half*>(h),
            static_cast<__half*>(l), ldh, scale_ws, f32, ld_f32, rows_f32, skip0, skip1, nullptr, 0);
    else
        enks::center_f16pair_kernel<<<dim3((unsigned)((K + 255) / 256), (unsigned)rows), 256, 0,
                                      st>>>(
            src, ld_src, rows, n_members, cols, z0, acc, inv_n, mean, static_cast<__half*>(h),
            static_cast<__half*>(l), ldh, scale_ws, f32, ld_f32, rows_f32, skip0, skip1);
    return enks::check_launch("enks_member_center_f16pair");
}

int enks_member_center_f16pair_t(const float* src, int64_t ld_src, const float* src2,
                                 int64_t ld_src2, int rows, int64_t n_members, int cols,
                                 const float* z0, const double* acc, const float* amax,
                                 int64_t n_total, float* mean, void* h, void* l, int64_t ldh,
                                 float* inv_scale, float* scale_ws, void* th, void* tl, int64_t ldt,
                                 float* t_inv, void* stream) {
    ENKS_REQUIRE(src && acc && amax && h && l && inv_scale && scale_ws && n_total > 0 &&
                     (!th) == (!tl) && (!th) == (!t_inv),
                 "enks_member_center_f16pair_t: bad arguments");
    ENKS_REQUIRE(rows <= enks::kTMaxRows && (!th || (ldt >= rows && ldt % 2 == 0)),
                 "enks_member_center_f16pair_t: rows > %d or bad ldt", enks::kTMaxRows);
    if (rows <= 0 || cols <= 0 || n_members <= 0) return ENKS_OK;
    cudaStream_t st = enks::as_stream(stream);
    const double inv_n = 1.0 / (double)n_total;
    enks::row_scale_kernel<<<rows, 128, 0, st>>>(acc, amax, inv_n, cols, scale_ws, inv_scale, rows,
                                                 rows);
    int rc = enks::check_launch("enks_member_center_f16pair_t(scale)");
    if (rc) return rc;
    const int64_t K = n_members * cols;
    auto a16 = [](const void* ptr) { return ((uintptr_t)ptr & 15) == 0; };
    if (!th && cols % 4 == 0 && ld_src % 4 == 0 && ldh % 4 == 0 && a16(src) &&
        (!src2 || (a16(src2) && ld_src2 % 4 == 0)) && ((uintptr_t)h & 7) == 0 &&
        ((uintptr_t)l & 7) == 0 && (!z0 || a16(z0)) && a16(acc) && (!mean || a16(mean))) {
        // no transposed planes: the vectorised centring with the second source on the fly
        enks::center_f16pair_v4_kernel<<<dim3((unsigned)((K / 4 + 255) / 256), (unsigned)rows), 256,
                                         0, st>>>(
            src, ld_src, rows, n_members, cols, z0, acc, inv_n, mean, static_cast<__half*>(h),
            static_cast<__half*>(l), ldh, scale_ws, nullptr, 0, 0, rows, rows, src2, ld_src2);
        return enks::check_launch("enks_member_center_f16pair_t(v4)");
    }
    enks::center_f16pair_t_kernel<<<(unsigned)((K + 31) / 32), 256, 0, st>>>(
        src, ld_src, src2, ld_src2, rows, n_members, cols, z0, acc, inv_n, mean,
        static_cast<__half*>(h), static_cast<__half*>(l), ldh, scale_ws, static_cast<__half*>(th),
        static_cast<__half*>(tl), ldt, t_inv);
    return enks::check_launch("enks_member_center_f16pair_t");
}

int enks_uchain_apply(const float* delta, int64_t ld_delta, float* mean, int64_t ld_mean,
                      const float* gcol, int64_t ld_g, float* gtt, int64_t ld_gtt, int n_slices,
                      int n, int l, int m, int p, void* stream) {
    ENKS_REQUIRE(n >= 0 && l > 0 && m > 0 && p > 0 && n_slices >= 0,
                 "enks_uchain_apply: bad sizes");
    ENKS_REQUIRE(n + l <= 65535, "enks_uchain_apply: rows > 65535");
    if (n_slices == 0) return ENKS_OK;
    cudaStream_t st = enks::as_stream(stream);
    if (delta && mean) {
        enks::uchain_mean_kernel<<<dim3((unsigned)((m + 127) / 128), (unsigned)(n + l)), 128, 0,
                                   st>>>(delta, ld_delta, mean, ld_mean, n_slices, n, l, m);
        int rc = enks::check_launch("enks_uchain_apply(mean)");
        if (rc) return rc;
    }
    if (gcol && gtt) {
        enks::uchain_gain_kernel<<<dim3((unsigned)((p + 127) / 128), (unsigned)(n + l)), 128, 0,
                                   st>>>(gcol, ld_g, gtt, ld_gtt, n_slices, n, l, p);
        return enks::check_launch("enks_uchain_apply(gain)");
    }
    return ENKS_OK;
}

}  // extern "C"

