// K3 on tcgen05: the 3-layer CNN forecast (widths 2-32-32-1, fields 32, 64 or 128 pixels wide)
//     X' = X + alpha * conv3(tanh(conv2(tanh(conv1([X, U])))))
// fused into one persistent kernel per SM: HBM sees X, U once and X' once.  Layer 1 (2 -> 32) on
// the CUDA cores, the 32 -> 32 layer (92 % of the FLOPs) as fp16-pair kind::f16 tcgen05 MMAs
// (three per K = 16 step: lo*hi + hi*lo + hi*hi, operands pre-scaled, see kF16 below), and for
// 128-pixel images the 32 -> 1 layer on the tensor core as well (kL3 below).
//
// Model seam: MatrixDynamics.step (reference dynamics.py:40-50) called at
// enks.py:168; the CNN itself is the paper's surrogate (not shipped by the
// reference) -- defined in dynamics.py::CNNDynamics, restated in
// fp64 by oracle/models.py.
//
// Formulation (one CTA streams member images -- or row units of them, see Unit -- one image row
// = one 128-row MMA tile, TMEM lane = pixel).  128-pixel images (SH): the layer-1 row r sits in
// shared memory one 128-B row per pixel with zero pad rows, and the three horizontal taps are
// three MMAs whose A operand starts 0 / 1 / 2 rows down; the three vertical taps are stacked in N
// (N = 96), so accumulator D_r holds row r's contributions to output rows r+1, r, r-1 and the
// epilogue sums three of them.  Narrow fields (32 / 64 pixels): a 128-pixel MMA row carries
// 128 / seg images side by side, the horizontal taps are stacked in N instead and folded in the
// epilogue with warp shuffles, cut at the image boundaries (which fall on warp boundaries), and
// layer 3 stays on the CUDA cores.
//
// Warp roles (512 threads): warp 0 = MMA issuer (whole warp converged, one elected lane issues:
// the descriptors stay in uniform registers), warp 2 = TMEM allocator, warps 1-3 idle or -- with
// the fused-noise entry point -- drawing the step's noise substreams with noise_dev.cuh's
// run_stream, warps 4-7 / 8-11 = layer-1 producers of the even / odd image rows (thread = pixel;
// two groups so that two rows of the latency-bound CUDA-core layer are in flight per SM),
// warps 12-15 = epilogue (thread = pixel = TMEM lane).
#include <cuda_fp16.h>
#include <stdlib.h>

#include "common.cuh"
#include "noise_dev.cuh"
#include "tc_ptx.cuh"

namespace enks {
namespace {

constexpr int W = 128;     // image width (== MMA M)
constexpr int C1 = 32;     // layer-1 width
constexpr int C2 = 32;     // layer-2 width
constexpr int NB = 3 * C2; // MMA N: (dx, co)
#ifndef ENKS_CNN_NA
#define ENKS_CNN_NA 3
#endif
constexpr int NA = ENKS_CNN_NA;      // layer-1 row slots
constexpr int NACC = 5;    // TMEM accumulators (ring over rows; 5 x 96 <= 512 columns)
constexpr int kThreads = 512;
constexpr int kRing = 8;   // input-row ring slots per producer group

// Layer-2 operand format.  fp16 pairs (default): one 128-B SWIZZLE_128B row holds a pixel's (or a
// weight row's) 32 channels as fp16 hi (bytes 0-63) and lo (bytes 64-127) -- one tile per operand,
// kind::f16 MMAs (K = 16) at twice the kind::tf32 rate, half the shared-memory stores of the
// producers.  Three products (lo*hi + hi*lo + hi*hi) keep the operands to ~2^-22 of their range,
// as 3xTF32 does, so both are pre-scaled by powers of two: the activations (|tanh| < 1) by 2^14
// and split on a fixed grid (split_grid: |error| <= 2^-10 at scale 2^14, i.e. 6e-8 absolute),
// W2 / W3 so that their largest |entry| lands in [2^14, 2^15) (exact split); the epilogue folds
// the inverse scale into the bias add (one FFMA in place of the FADD).  Build with -DENKS_CNN_TF32=1 for the previous 3xTF32 operands (separate fp32
// hi / lo tiles).
#ifndef ENKS_CNN_TF32
#define ENKS_CNN_TF32 0
#endif
constexpr bool kF16 = !ENKS_CNN_TF32;
constexpr int kPlanes = kF16 ? 1 : 2;  // tiles per operand (hi and lo share a row in fp16)
constexpr float kScaleA = 16384.f;    // activation pre-scale (fp16 pairs)

// Layer 3 (32 -> 1) on the tensor core (128-pixel whole images, fp16 pairs): the epilogue writes
// the layer-2 activations h2 of each row into a shared-memory tile laid out like the layer-1
// tiles, and the MMA warp contracts it with W3 -- for each horizontal tap kx one MMA group whose
// A operand starts kx rows down (the zero pad rows give the 'same' padding), N = 16 columns of
// which the first three are the vertical taps ky:  U_j[x][ky] = sum_kx sum_c h2[j][x+kx-1][c]
// W3[c][ky][kx].  Output row y = U_{y-1}[0] + U_y[1] + U_{y+1}[2], three TMEM columns.  The
// epilogue keeps tanh, the fp16 split and that three-term fold; the 288 FMAs per pixel and the
// cross-warp tap exchange of the CUDA-core layer 3 go away (the epilogue was the kernel's
// bottleneck: one warp per SM sub-partition, latency-bound).  -DENKS_CNN_L3=0: CUDA-core layer 3.
#ifndef ENKS_CNN_L3
#define ENKS_CNN_L3 1
#endif
constexpr bool kL3 = ENKS_CNN_L3 && kF16;
constexpr int NH = 3;       // h2 tiles (layer-3 A operand ring)
constexpr int NU = 8;       // layer-3 accumulators (16 TMEM columns each, after 4 x 96)
constexpr int kUCol0 = 4 * NB;
#ifndef ENKS_CNN_CONV_ISSUER
#define ENKS_CNN_CONV_ISSUER 1
#endif
constexpr bool kConvIssuer = ENKS_CNN_CONV_ISSUER;
constexpr float kGrid = 1.5f * 67108864.f;  // 1.5 * 2^26: (v + kGrid) - kGrid rounds v to a multiple of 8

constexpr int kInRow = W + 2;
constexpr int kW1Stride = 20;                        // float2 per channel pair (18 used)
constexpr int kW3Stride = 12;
constexpr int kXD = 2 * 4 * 32;                     // [parity][warp][32]
constexpr int kXV = 2 * 4 * 4;                      // [parity][warp][3 (+pad)]

// layer-1 weights / bias, layer-2 bias and layer-3 weights in constant memory: the producers and
// the epilogue read them as uniform-register operands (LDCU) instead of shared-memory loads (the
// kernel's shared-memory pipe is its limit; the layer-1 weights were 85 % of its wavefronts)
struct Cnn3Epi {
    alignas(16) float w1[C1 / 2][kW1Stride * 2];  // channel pair cp: (w[2cp][k], w[2cp+1][k]) per k
    float b1[C1];
    float b2[C2];
    float w3[C2][kW3Stride];  // [c][ky*3 + kx], padded to 12
    float b3;
};
__constant__ Cnn3Epi c_epi;

// Shared-memory / TMEM layout.  SH = false: the three horizontal taps are stacked in N
// (N = 96, one accumulator per OUTPUT row, horizontal taps folded in the epilogue with warp
// shuffles).  SH = true (128-pixel images): the three VERTICAL taps are stacked in N and the
// horizontal taps are three MMAs whose A operand is the layer-1 tile read from row dx (the tile
// keeps a zero pad row above and below the 128 pixels; a SWIZZLE_128B operand may start at
// any 128-B row -- tools/probes/tc_shift_probe.cu).  One accumulator per INPUT row r holds
// its contributions to output rows r+1, r, r-1, which the epilogue adds in registers: no
// shuffles, no cross-warp exchange for layer 2.
template <bool SH>
struct CL {
    static constexpr int kBRows = NB;                      // rows of one B tile
    static constexpr int kBTile = kBRows * 128;
    static constexpr int kNBT = 3;                         // B tiles: dx (SH) or dy
    static constexpr int kARows = SH ? 136 : W;            // SH: pixel x at row x + 1
    static constexpr int kATile = kARows * 128;
    static constexpr int kOffB = 0;                        // [tap][hi/lo] B tiles
    static constexpr int kOffA = kOffB + kNBT * kPlanes * kBTile;  // [slot][plane] A tiles
    static constexpr int kOffIn = kOffA + NA * kPlanes * kATile;   // rings [2][kRing][2][W + 2]
    static constexpr int kOffW1 = kOffIn + 2 * kRing * 2 * kInRow * 4;
    static constexpr int kOffB1 = kOffW1 + (C1 / 2) * kW1Stride * 8;
    static constexpr int kOffB2 = kOffB1 + C1 * 4;
    static constexpr int kOffW3 = kOffB2 + C2 * 4;
    static constexpr int kOffB3 = kOffW3 + C2 * kW3Stride * 4;  // b3, layer-2 inverse scale
    static constexpr int kOffX = kOffB3 + 16;
    static constexpr int kOffBar = kOffX + (2 * kXD + 2 * kXV) * 4;
    static constexpr int kOffNz = kOffBar + 64 * 8;
    static_assert(2 * NA + 2 * NACC + 1 + 4 + 2 * NH + 2 * NU <= 64, "mbarrier region");                       // noise: ki, wi tables
    static constexpr int kNzWarp = 2 * kMaxRowCols * 4 + kBufWords * 8;     // row slots + words
    static constexpr int kOffNzW = kOffNz + 256 * 16;                       // [3] per noise warp
    static constexpr int kEndNz = kOffNzW + 3 * kNzWarp;
    // layer 3 on the tensor core (SH): W3 B tiles [kx] (16 rows: ky 0..2, then zeros), h2 tiles
    static constexpr int kOffW3T = (kEndNz + 1023) / 1024 * 1024;
    static constexpr int kW3Tile = 16 * 128;
    static constexpr int kOffH2 = kOffW3T + 3 * kW3Tile;
    static constexpr int kSmem = (SH && kL3 ? kOffH2 + NH * kATile : kEndNz) + 1024;
    static constexpr int kAccCols = NB;                    // TMEM columns per accumulator
    static constexpr uint32_t kTmemAlloc = 512;
    static_assert(kSmem <= 232448, "shared memory budget");
    static_assert(kOffA % 1024 == 0 && kATile % 1024 == 0, "SW128 tiles need 1 KB alignment");
};

__device__ __forceinline__ float exp2f_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t sw128(int row, int byte) {
    return (uint32_t)(row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15)));
}

// tanh(x) = 1 - 2 / (1 + e^{2x}): ex2.approx and rcp.approx on the SFU (~2^-22 relative
// each), so |error| ~ 1e-7 absolute; ENKS_CNN_TANH=1 selects the FMA-pipe Newton reciprocal
// (one SFU op per tanh) instead -- the kernel is issue-bound, so fewer instructions win.
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
template <bool NEWTON>
__device__ __forceinline__ float tanh_fast_t(float x) {
    // no clamp: e^{2x} -> +inf gives rcp 0 (tanh 1), -> 0 gives tanh -1
    const float t = exp2f_approx(x * 2.8853900817779268f);  // e^{2x}
    const float d = 1.f + t;
    float r;
    if (NEWTON) {
        r = __int_as_float(0x7EF311C3 - __float_as_int(d));
        r = r * fmaf(-d, r, 2.f);
        r = r * fmaf(-d, r, 2.f);
        r = r * fmaf(-d, r, 2.f);
    } else {
        r = rcp_approx(d);
    }
    return fmaf(-2.f, r, 1.f);
}
#define tanh_fast tanh_fast_t<false>

// two tanh at once: the non-SFU steps as packed f32x2 instructions (FADD2 / FMUL2 / FFMA2)
__device__ __forceinline__ float2 tanh2_fast(float2 x) {
    const float2 e = __fmul2_rn(x, make_float2(2.8853900817779268f, 2.8853900817779268f));
    const float2 d = __fadd2_rn(make_float2(exp2f_approx(e.x), exp2f_approx(e.y)),
                                make_float2(1.f, 1.f));
    return __ffma2_rn(make_float2(-2.f, -2.f), make_float2(rcp_approx(d.x), rcp_approx(d.y)),
                      make_float2(1.f, 1.f));
}

// s * tanh(x) for two values: the scale folds into the last FFMA2
__device__ __forceinline__ float2 tanh2_fast_s(float2 x, float s) {
    const float2 e = __fmul2_rn(x, make_float2(2.8853900817779268f, 2.8853900817779268f));
    const float2 d = __fadd2_rn(make_float2(exp2f_approx(e.x), exp2f_approx(e.y)),
                                make_float2(1.f, 1.f));
    return __ffma2_rn(make_float2(-2.f * s, -2.f * s), make_float2(rcp_approx(d.x), rcp_approx(d.y)),
                      make_float2(s, s));
}

__device__ __forceinline__ uint32_t h2_bits(__half2 h) {
    return *reinterpret_cast<const uint32_t*>(&h);
}

// fp16 pair of two values |v| <= 2^14: hi = v rounded to a multiple of 8 (exact in fp16 there),
// lo = v - hi (|lo| <= 4, rounded to fp16: 2^-10 absolute)
__device__ __forceinline__ void split_grid(float2 v, uint32_t& hi, uint32_t& lo) {
    const float2 h = __fadd2_rn(__fadd2_rn(v, make_float2(kGrid, kGrid)), make_float2(-kGrid, -kGrid));
    hi = h2_bits(__float22half2_rn(h));
    lo = h2_bits(__float22half2_rn(__ffma2_rn(h, make_float2(-1.f, -1.f), v)));
}

// one B row entry of W2 (hi / lo) into a tile at (row, ci)
__device__ __forceinline__ void stage_w2(uint8_t* tile, int row, int ci, float v, float ws) {
    if constexpr (kF16) {
        const float vs = v * ws;
        const __half h = __float2half_rn(vs);
        *reinterpret_cast<__half*>(tile + sw128(row, ci * 2)) = h;
        *reinterpret_cast<__half*>(tile + sw128(row, 64 + ci * 2)) =
            __float2half_rn(vs - __half2float(h));
    } else {
        const float h = ptx::tf32_round(v);
        *reinterpret_cast<float*>(tile + sw128(row, ci * 4)) = h;
        *reinterpret_cast<float*>(tile + NB * 128 + sw128(row, ci * 4)) = v - h;
    }
}

struct Cnn3Args {
    const float* w1;  // (C1, 2, 3, 3)
    const float* b1;
    const float* w2;  // (C2, C1, 3, 3)
    const float* b2;
    const float* w3;  // (1, C2, 3, 3)
    const float* b3;
    float alpha;
    const float* x;
    int64_t ldx;
    const float* u;
    int64_t ldu;
    float* out;
    int64_t ldo;
    int rows;
    int64_t n_members;  // 128-pixel row groups ("virtual members")
    int64_t cols_total; // n_members_real * seg: columns beyond it are padding
    int seg;            // image width: 32, 64 or 128
    int debug;  // ENKS_CNN_DEBUG: 1 = no MMAs, 2 = no layer-1 math, 4 = no epilogue math
    int products;  // 3 (default): lo*hi + hi*lo + hi*hi; 2 (ENKS_CNN_PRODUCTS=2): hi*lo + hi*hi
    NoiseLaunch nz;  // nz.n_jobs > 0: warps 1-3 draw these noise jobs (member-column layout)
    int parts;       // 128-pixel images: each image's rows split into `parts` units (small N)
};

// A unit of work: output rows [o0, o1) of one image, which need layer-2 (h2) rows [e0, e1) and
// layer-1 rows [l0, l1) (the 3x3 layer-3 and layer-2 taps: a two-row halo of recomputation at an
// interior cut; image edges keep the zero 'same' padding).  parts == 1: the whole image.
struct Unit {
    int mem;
    int o0, o1, e0, e1, l0, l1;
};
// 32-bit arithmetic only: a 64-bit division here compiles to a helper call, and a call inside the
// MMA issuer's loop corrupts the uniform-register descriptors of the tcgen05.mma that follow
// (garbage accumulators in the first rows -- measured)
template <bool SPLIT>
__device__ __forceinline__ Unit unit_of(const Cnn3Args& a, int u) {
    Unit U;
    const int n = a.rows;
    if constexpr (!SPLIT) {  // whole images: the ranges fold to constants
        U.mem = u;
        U.o0 = U.e0 = U.l0 = 0;
        U.o1 = U.e1 = U.l1 = n;
        return U;
    }
    const int S = a.parts;
    U.mem = u / S;
    const int part = u - U.mem * S;
    U.o0 = part * n / S;
    U.o1 = (part + 1) * n / S;
    U.e0 = max(0, U.o0 - 1);
    U.e1 = min(n, U.o1 + 1);
    U.l0 = max(0, U.o0 - 2);
    U.l1 = min(n, U.o1 + 2);
    return U;
}

template <bool SH, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1) cnn3_tc_kernel(const Cnn3Args a) {
    using L = CL<SH>;
    extern __shared__ uint8_t smem_raw[];
    // align to 1024 B by offsetting the shared pointer itself, so the compiler keeps the
    // shared address space (LDS/STS rather than generic LD/ST)
    uint8_t* sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    float* in_ring = reinterpret_cast<float*>(sm + L::kOffIn);
    float* w1s = reinterpret_cast<float*>(sm + L::kOffW1);
    float* b1s = reinterpret_cast<float*>(sm + L::kOffB1);
    float* b2s = reinterpret_cast<float*>(sm + L::kOffB2);
    float* w3s = reinterpret_cast<float*>(sm + L::kOffW3);
    float* b3s = reinterpret_cast<float*>(sm + L::kOffB3);
    float* xd0 = reinterpret_cast<float*>(sm + L::kOffX);
    float* xd2 = xd0 + kXD;
    float* xv0 = xd2 + kXD;
    float* xv2 = xv0 + kXV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::kOffBar);
    uint64_t* a_full = bars;             // [NA]
    uint64_t* a_empty = bars + NA;       // [NA]
    uint64_t* acc_full = bars + 2 * NA;  // [NACC]
    uint64_t* acc_empty = bars + 2 * NA + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NA + 2 * NACC);
    uint64_t* xb_full = bars + 2 * NA + 2 * NACC + 1;  // [4] SH: row's boundary taps written
    uint64_t* h2_full = xb_full + 4;     // [NH] layer 3: h2 row written by the epilogue
    uint64_t* h2_empty = h2_full + NH;   // [NH] layer 3: its MMAs done
    uint64_t* u_full = h2_empty + NH;    // [NU] layer-3 accumulator complete
    uint64_t* u_empty = u_full + NU;     // [NU] layer-3 accumulator read
    // layer 3 on the tensor core (128-pixel images, whole or split into units); the layer-2 ring
    // then has 4 accumulators (4 x 96 + NU x 16 columns).
    // (One 32-column accumulator per output row instead -- 54 N = 32 MMAs per row in place of
    // 18 N = 96 -- ran at half the speed: the MMA cost is per instruction at these shapes.)
    constexpr bool L3 = SH && kL3;
    constexpr int kNAcc = L3 ? 4 : NACC;

    // warp index and TMEM base through a lane-0 shuffle: provably warp-uniform, so the MMA warp's
    // descriptor arithmetic can stay in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int n = a.rows;

    // ---- stage weights (all threads) -------------------------------------------------
    // fp16 pairs: W2 pre-scale ws = 2^(15 - e) for max |W2| = m 2^e (m in [0.5, 1)), from a
    // block-wide max (the input ring is free scratch until the producers start)
    // (the same for W3 when layer 3 runs on the tensor core)
    float ws = 1.f, inv2 = 1.f, ws3 = 1.f, inv3 = 1.f;
    if constexpr (kF16) {
        float mx = 0.f, mx3 = 0.f;
        for (int e = threadIdx.x; e < C2 * C1 * 9; e += kThreads) mx = fmaxf(mx, fabsf(a.w2[e]));
        for (int e = threadIdx.x; e < C2 * 9; e += kThreads) mx3 = fmaxf(mx3, fabsf(a.w3[e]));
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mx3 = fmaxf(mx3, __shfl_xor_sync(0xffffffffu, mx3, o));
        }
        if (lane_id() == 0) {
            in_ring[threadIdx.x >> 5] = mx;
            in_ring[kThreads / 32 + (threadIdx.x >> 5)] = mx3;
        }
        __syncthreads();
        mx = mx3 = 0.f;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
            mx = fmaxf(mx, in_ring[w]);
            mx3 = fmaxf(mx3, in_ring[kThreads / 32 + w]);
        }
        __syncthreads();
        if (mx > 0.f && mx < 3.0e38f) {
            int ex;
            frexpf(mx, &ex);
            ws = ldexpf(1.f, 15 - ex);
            inv2 = ldexpf(1.f, ex - 15 - 14);  // 1 / (ws * kScaleA)
        }
        if (mx3 > 0.f && mx3 < 3.0e38f) {
            int ex;
            frexpf(mx3, &ex);
            ws3 = ldexpf(1.f, 15 - ex);
            inv3 = ldexpf(1.f, ex - 15 - 14);
        }
    }
    if constexpr (SH && kL3) {
        // W3 B tiles: row ky (< 3) of tile kx holds W3[c][ky][kx] as (hi | lo); rows 3..15 zero
        for (int e = threadIdx.x; e < 3 * 16 * C2; e += kThreads) {
            const int kx = e / (16 * C2), rem = e - kx * 16 * C2;
            const int row = rem / C2, c = rem - row * C2;
            const float v = row < 3 ? a.w3[(c * 3 + row) * 3 + kx] : 0.f;
            stage_w2(sm + L::kOffW3T + kx * L::kW3Tile, row, c, v, ws3);
        }
        // zero pad rows (0 and 129..135) of the h2 tiles
        for (int e = threadIdx.x; e < NH * 8 * 32; e += kThreads) {
            const int tile = e / (8 * 32), rem = e - tile * 8 * 32;
            const int pr = rem >> 5, k = rem & 31;
            const int row = pr == 0 ? 0 : 128 + pr;
            *reinterpret_cast<float*>(sm + L::kOffH2 + tile * L::kATile + sw128(row, k * 4)) = 0.f;
        }
    }
    if constexpr (SH) {
        for (int e = threadIdx.x; e < 3 * NB * C1; e += kThreads) {
            // B[dx][row = dy*C2 + co][ci] = W2[co][ci][dy][dx]
            const int dx = e / (NB * C1), rem = e - dx * NB * C1;
            const int row = rem / C1, ci = rem - row * C1;
            const int dy = row / C2, co = row - dy * C2;
            stage_w2(sm + L::kOffB + dx * kPlanes * L::kBTile, row, ci,
                     a.w2[((co * C1 + ci) * 3 + dy) * 3 + dx], ws);
        }
        // zero pad rows (0 and 129..135) of every A slot; never written afterwards
        for (int e = threadIdx.x; e < NA * kPlanes * 8 * 32; e += kThreads) {
            const int tile = e / (8 * 32), rem = e - tile * 8 * 32;
            const int pr = rem >> 5, k = rem & 31;
            const int row = pr == 0 ? 0 : 128 + pr;
            *reinterpret_cast<float*>(sm + L::kOffA + tile * L::kATile + sw128(row, k * 4)) = 0.f;
        }
    } else {
        for (int e = threadIdx.x; e < 3 * NB * C1; e += kThreads) {
            // B[dy][row = dx*C2 + co][ci] = W2[co][ci][dy][dx]
            const int dy = e / (NB * C1), rem = e - dy * NB * C1;
            const int row = rem / C1, ci = rem - row * C1;
            const int dx = row / C2, co = row - dx * C2;
            stage_w2(sm + L::kOffB + dy * kPlanes * L::kBTile, row, ci,
                     a.w2[((co * C1 + ci) * 3 + dy) * 3 + dx], ws);
        }
    }
    for (int e = threadIdx.x; e < C1 * 18; e += kThreads) {
        const int c = e / 18, k = e - c * 18;  // k = ci*9 + ky*3 + kx
        w1s[((c >> 1) * kW1Stride + k) * 2 + (c & 1)] = a.w1[c * 18 + k];
    }
    for (int e = threadIdx.x; e < C1; e += kThreads) b1s[e] = a.b1[e];
    for (int e = threadIdx.x; e < C2; e += kThreads) b2s[e] = a.b2[e];
    for (int e = threadIdx.x; e < C2 * kW3Stride; e += kThreads) {
        const int c = e / kW3Stride, k = e - c * kW3Stride;  // w3s[c][ky*3+kx]
        w3s[e] = k < 9 ? a.w3[c * 9 + k] : 0.f;
    }
    if (threadIdx.x == 0) {
        b3s[0] = a.b3[0];
        b3s[1] = inv2;
        b3s[2] = inv3;
        for (int s = 0; s < NA; ++s) {
            ptx::mbar_init(&a_full[s], 128);
            ptx::mbar_init(&a_empty[s], 1);
        }
        for (int q = 0; q < NACC; ++q) {
            ptx::mbar_init(&acc_full[q], 1);
            ptx::mbar_init(&acc_empty[q], 4);
        }
        for (int q = 0; q < 4; ++q) ptx::mbar_init(&xb_full[q], 128);
        for (int q = 0; q < NH; ++q) {
            ptx::mbar_init(&h2_full[q], 128);
            ptx::mbar_init(&h2_empty[q], 1);
        }
        for (int q = 0; q < NU; ++q) {
            ptx::mbar_init(&u_full[q], 1);
            ptx::mbar_init(&u_empty[q], 4);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, L::kTmemAlloc);
    ptx::fence_proxy_async_smem();  // staged B tiles -> async proxy
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
    if (warp == 0) {
        // ================= MMA issuer =================
        // kConvIssuer: the whole warp runs the loop and an elected lane issues each MMA / commit
        // (see tc_ptx.cuh); otherwise lane 0 alone
        if (kConvIssuer || lane == 0) {
            constexpr uint32_t idesc = kF16 ? ptx::idesc_f16(W, L::kAccCols)
                                            : ptx::idesc_tf32(W, L::kAccCols);
            // one K step: 16 fp16 or 8 tf32 channels = 32 B of the 128-B row (+2 in the
            // descriptor's start field); fp16: the lo half is 64 B (+4) along the same row,
            // tf32: the lo plane is the next tile
            constexpr int kSteps = kF16 ? C1 / 16 : C1 / 8;
            auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t acc) {
                if constexpr (kF16 && kConvIssuer) ptx::mma_f16_ss_elect(d, ad, bd, idesc, acc);
                else if constexpr (kF16) ptx::mma_f16_ss(d, ad, bd, idesc, acc);
                else if constexpr (kConvIssuer) ptx::mma_tf32_ss_elect(d, ad, bd, idesc, acc);
                else ptx::mma_tf32_ss(d, ad, bd, idesc, acc);
            };
            auto commit = [&](uint64_t* bar) {
                if constexpr (kConvIssuer) ptx::mma_commit_elect(bar);
                else ptx::mma_commit(bar);
            };
            // descriptors are built once: the start-address field (addr >> 4, 14 bits) of a tile
            // at a byte offset o from a base is the base descriptor + (o >> 4)
            const uint64_t dA0 = ptx::desc_kmajor_sw128(sm + L::kOffA);
            const uint64_t dB0 = ptx::desc_kmajor_sw128(sm + L::kOffB);
            constexpr uint64_t kAT = L::kATile >> 4, kBT = L::kBTile >> 4;
            const bool do_mma = !(a.debug & 1), p3 = a.products == 3;
            // layer 3 of the h2 row with global index Jg (L3): three horizontal taps x 2 K steps
            // x 3 products into the 16-column accumulator U_Jg
            const uint64_t dH0 = ptx::desc_kmajor_sw128(sm + L::kOffH2);
            const uint64_t dW0 = ptx::desc_kmajor_sw128(sm + L::kOffW3T);
            auto mma3 = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t acc) {
                constexpr uint32_t idesc3 = ptx::idesc_f16(W, 16);
                if constexpr (kConvIssuer) ptx::mma_f16_ss_elect(d, ad, bd, idesc3, acc);
                else ptx::mma_f16_ss(d, ad, bd, idesc3, acc);
            };
            auto layer3 = [&](int Jg) {
                const int hs = Jg % NH, qu = Jg % NU;
                ptx::mbar_wait(&h2_full[hs], (uint32_t)((Jg / NH) & 1));
                ptx::mbar_wait(&u_empty[qu], (uint32_t)(((Jg / NU) & 1) ^ 1));
                ptx::tc_fence_after();
                const uint32_t du = tmem + (uint32_t)(kUCol0 + qu * 16);
                if (do_mma) {
                    const uint64_t dh = dH0 + (uint64_t)hs * kAT;
#pragma unroll
                    for (int kx = 0; kx < 3; ++kx) {
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            const uint64_t adh = dh + (uint64_t)(kx * 8 + 2 * k), adl = adh + 4;
                            const uint64_t bdh = dW0 + (uint64_t)(kx * (L::kW3Tile >> 4) + 2 * k);
                            const uint64_t bdl = bdh + 4;
                            mma3(du, adl, bdh, (kx == 0 && k == 0) ? 0u : 1u);
                            mma3(du, adh, bdl, 1u);
                            mma3(du, adh, bdh, 1u);
                        }
                    }
                }
                commit(&u_full[qu]);
                commit(&h2_empty[hs]);
            };
            int l3_next = 0;  // global index of the next h2 row for layer 3
            int Lbase = 0;  // layer-1 rows of this CTA's earlier units (ring / slot counter)
            int Hbase = 0;  // h2 rows of this CTA's earlier units (layer-3 ring counter)
            const int n_units = (int)(a.n_members * a.parts);
            for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
                const Unit U = unit_of<SPLIT>(a, u);
                const int Lb = Lbase - U.l0, Hb = Hbase - U.e0;
                Lbase += U.l1 - U.l0;
                Hbase += U.e1 - U.e0;
                for (int r = U.l0; r < U.l1; ++r) {
                    const int Rg = Lb + r;
                    const int slot = Rg % NA;
                    ptx::mbar_wait(&a_full[slot], (uint32_t)((Rg / NA) & 1));
                                        ptx::tc_fence_after();
                    const uint64_t dah0 = dA0 + (uint64_t)(slot * kPlanes) * kAT;
                    const uint64_t dal0 = dah0 + (kF16 ? 4 : kAT);
                    if constexpr (SH) {
                        // layer 3 runs three rows behind: h2 row j needs D_{j+1} (issued at
                        // iteration j + 1) and the epilogue's pass over it
                        if constexpr (L3) {
                            while (l3_next <= Hb + r - 3) layer3(l3_next++);
                        }
                        // D_r[x][(dy, co)] = sum_dx sum_ci h1[r][x + dx - 1][ci] W2[co][ci][dy][dx]
                        const int q = Rg % kNAcc;
                        ptx::mbar_wait(&acc_empty[q], (uint32_t)(((Rg / kNAcc) & 1) ^ 1));
                                                ptx::tc_fence_after();
                        const uint32_t d = tmem + (uint32_t)(q * L::kAccCols);
                        if (do_mma) {
#pragma unroll
                            for (int dx = 0; dx < 3; ++dx) {
                                const uint64_t bh0 = dB0 + (uint64_t)(dx * kPlanes) * kBT;
#pragma unroll
                                for (int k = 0; k < kSteps; ++k) {  // A starts dx 128-B rows down
                                    const uint64_t adh = dah0 + (uint64_t)(dx * 8 + 2 * k);
                                    const uint64_t adl = dal0 + (uint64_t)(dx * 8 + 2 * k);
                                    const uint64_t bdh = bh0 + (uint64_t)(2 * k);
                                    const uint64_t bdl = bdh + (kF16 ? 4 : kBT);
                                    const uint32_t acc0 = (dx == 0 && k == 0) ? 0u : 1u;
                                    if (p3) mma(d, adl, bdh, acc0);
                                    mma(d, adh, bdl, p3 ? 1u : acc0);
                                    mma(d, adh, bdh, 1u);
                                }
                            }
                        }
                        commit(&acc_full[q]);
                                            } else {
                        for (int dy = 0; dy < 3; ++dy) {
                            const int y = r - dy + 1;
                            if (y < 0 || y >= n) continue;
                            const int Yg = Lb + y;  // (parts == 1 off the SH path)
                            const int q = Yg % kNAcc;
                            const bool first = (dy == 0) || (r == 0 && dy == 1);
                            if (first) {
                                ptx::mbar_wait(&acc_empty[q], (uint32_t)(((Yg / kNAcc) & 1) ^ 1));
                                                                ptx::tc_fence_after();
                            }
                            const uint32_t d = tmem + (uint32_t)(q * L::kAccCols);
                            const uint64_t bh0 = dB0 + (uint64_t)(dy * kPlanes) * kBT;
                            if (do_mma) {
#pragma unroll
                                for (int k = 0; k < kSteps; ++k) {
                                    const uint64_t adh = dah0 + (uint64_t)(2 * k);
                                    const uint64_t adl = dal0 + (uint64_t)(2 * k);
                                    const uint64_t bdh = bh0 + (uint64_t)(2 * k);
                                    const uint64_t bdl = bdh + (kF16 ? 4 : kBT);
                                    const uint32_t acc0 = (first && k == 0) ? 0u : 1u;
                                    if (p3) mma(d, adl, bdh, acc0);
                                    mma(d, adh, bdl, p3 ? 1u : acc0);
                                    mma(d, adh, bdh, 1u);
                                }
                            }
                            // row y complete: after its dy=2 contribution, or the last row's dy=1
                            if (dy == 2 || (r == n - 1 && dy == 1)) commit(&acc_full[q]);
                                                    }
                    }
                    commit(&a_empty[slot]);
                                    }
            }
            if constexpr (L3) {
                while (l3_next < Hbase) layer3(l3_next++);  // the last rows
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ================= layer-1 producers: thread = pixel, group g = row parity ============
        const int g = (warp - 4) >> 2;
        const int x = threadIdx.x - 128 - 128 * g;
        const int xs = x & (a.seg - 1);  // pixel within its image
        float* ring = in_ring + g * kRing * 2 * kInRow;
        int Lbase = 0;
        const int n_units = (int)(a.n_members * a.parts);
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const Unit U = unit_of<SPLIT>(a, u);
            const int64_t mem = U.mem;
            const int Lb = Lbase - U.l0;
            Lbase += U.l1 - U.l0;
            const float* xm = a.x + mem * W;
            const float* um = a.u + mem * W;
            const bool col_ok = mem * W + x < a.cols_total;
            // each group keeps its own ring of input rows; output row r (r = g, g + 2, ...)
            // reads rows r - 1 .. r + 1 and brings in rows r, r + 1, which were prefetched into
            // registers one iteration earlier (the global-load latency overlaps a row of work)
            auto fetch = [&](int j, float& vx, float& vu) {
                vx = (j < n && col_ok) ? xm[(int64_t)j * a.ldx + x] : 0.f;
                vu = (j < n && col_ok) ? um[(int64_t)j * a.ldu + x] : 0.f;
            };
            auto put = [&](int j, float vx, float vu) {  // row j into ring slot j % kRing
                float* dst = ring + (j & (kRing - 1)) * 2 * kInRow;
                dst[x + 1] = vx;
                dst[kInRow + x + 1] = vu;
                if (x == 0) {
                    dst[0] = 0.f; dst[kInRow - 1] = 0.f;
                    dst[kInRow] = 0.f; dst[2 * kInRow - 1] = 0.f;
                }
            };
            float p0x, p0u, p1x, p1u;
            if (g == 1) {  // row l0 (the group's first row l0 + 1 reads it)
                fetch(U.l0, p0x, p0u);
                put(U.l0, p0x, p0u);
            } else if (U.l0 > 0) {  // interior cut: row l0 - 1 is data, not padding
                fetch(U.l0 - 1, p0x, p0u);
                put(U.l0 - 1, p0x, p0u);
            }
            fetch(U.l0 + g, p0x, p0u);
            fetch(U.l0 + g + 1, p1x, p1u);
            for (int r = U.l0 + g; r < U.l1; r += 2) {
                put(r, p0x, p0u);
                if (r + 1 < n) put(r + 1, p1x, p1u);
                fetch(r + 2, p0x, p0u);
                fetch(r + 3, p1x, p1u);
                asm volatile("bar.sync %0, 128;" ::"r"(1 + 2 * g) : "memory");
                float in[18];
#pragma unroll
                for (int ci = 0; ci < 2; ++ci)
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky) {
                        const int j = r + ky - 1;
                        const bool ok = j >= 0 && j < n;
                        const float* src = ring + (j & (kRing - 1)) * 2 * kInRow + ci * kInRow + x;
                        in[ci * 9 + ky * 3 + 0] = (ok && xs != 0) ? src[0] : 0.f;
                        in[ci * 9 + ky * 3 + 1] = ok ? src[1] : 0.f;
                        in[ci * 9 + ky * 3 + 2] = (ok && xs != a.seg - 1) ? src[2] : 0.f;
                    }
                const int Rg = Lb + r;
                const int slot = Rg % NA;
                ptx::mbar_wait(&a_empty[slot], (uint32_t)(((Rg / NA) & 1) ^ 1));
                if (a.debug & 16) {
                    ptx::mbar_arrive(&a_full[slot]);
                    continue;
                }
                uint8_t* ah_t = sm + L::kOffA + (slot * kPlanes + 0) * L::kATile;
                uint8_t* al_t = ah_t + (kF16 ? 0 : L::kATile);
                if constexpr (kF16) {
                    const int row = SH ? x + 1 : x;
#pragma unroll
                    for (int c8 = 0; c8 < ((a.debug & 2) ? 0 : C1 / 8); ++c8) {
                        uint32_t hw[4], lw[4];
#pragma unroll
                        for (int pr = 0; pr < 4; ++pr) {  // channel pair (c, c+1), packed FFMA2
                            const int cp = c8 * 4 + pr;
                            const float4* wr = reinterpret_cast<const float4*>(c_epi.w1[cp]);
                            float2 acc = make_float2(c_epi.b1[2 * cp], c_epi.b1[2 * cp + 1]);
#pragma unroll
                            for (int q = 0; q < 9; ++q) {
                                const float4 wv = wr[q];
                                acc = __ffma2_rn(make_float2(wv.x, wv.y),
                                                 make_float2(in[2 * q], in[2 * q]), acc);
                                acc = __ffma2_rn(make_float2(wv.z, wv.w),
                                                 make_float2(in[2 * q + 1], in[2 * q + 1]), acc);
                            }
                            split_grid(tanh2_fast_s(acc, kScaleA), hw[pr], lw[pr]);  // 2^14 tanh
                        }
                        *reinterpret_cast<uint4*>(ah_t + sw128(row, c8 * 16)) =
                            make_uint4(hw[0], hw[1], hw[2], hw[3]);
                        *reinterpret_cast<uint4*>(ah_t + sw128(row, 64 + c8 * 16)) =
                            make_uint4(lw[0], lw[1], lw[2], lw[3]);
                    }
                } else {
#pragma unroll 2
                for (int c4 = 0; c4 < ((a.debug & 2) ? 0 : C1 / 4); ++c4) {
                    float hv[4];
#pragma unroll
                    for (int pr = 0; pr < 2; ++pr) {  // channel pair (c, c+1), packed FFMA2
                        const int cp = c4 * 2 + pr;
                        const float4* wr = reinterpret_cast<const float4*>(w1s + cp * kW1Stride * 2);
                        float2 acc = make_float2(b1s[2 * cp], b1s[2 * cp + 1]);
#pragma unroll
                        for (int q = 0; q < 9; ++q) {
                            const float4 wv = wr[q];  // (k=2q: c, c+1), (k=2q+1: c, c+1)
                            acc = __ffma2_rn(make_float2(wv.x, wv.y), make_float2(in[2 * q], in[2 * q]), acc);
                            acc = __ffma2_rn(make_float2(wv.z, wv.w),
                                             make_float2(in[2 * q + 1], in[2 * q + 1]), acc);
                        }
                        const float2 t2 = tanh2_fast(acc);  // packed non-SFU steps
                        hv[2 * pr] = t2.x;
                        hv[2 * pr + 1] = t2.y;
                    }
                    float4 h4, l4;
                    h4.x = ptx::tf32_round(hv[0]); l4.x = hv[0] - h4.x;
                    h4.y = ptx::tf32_round(hv[1]); l4.y = hv[1] - h4.y;
                    h4.z = ptx::tf32_round(hv[2]); l4.z = hv[2] - h4.z;
                    h4.w = ptx::tf32_round(hv[3]); l4.w = hv[3] - h4.w;
                    const uint32_t off = sw128(SH ? x + 1 : x, c4 * 16);
                    *reinterpret_cast<float4*>(ah_t + off) = h4;
                    *reinterpret_cast<float4*>(al_t + off) = l4;
                }
                }
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&a_full[slot]);
            }
            asm volatile("bar.sync %0, 128;" ::"r"(1 + 2 * g) : "memory");  // ring reuse across units
        }
    } else if (warp >= 12) {
        // ================= epilogue: thread = pixel = TMEM lane =================
        const float inv2 = b3s[1];  // layer-2 accumulator -> pre-activation (operand pre-scales)
        const int ew = warp - 12;  // == warp & 3 -> TMEM lane quarter
        const int x = ew * 32 + lane;
        const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
        const float b3 = c_epi.b3;
        // cross-warp tap exchange only inside an image (seg = 32: never; 64: not across 63|64)
        const bool xl = ew > 0 && ((ew * 32) & (a.seg - 1)) != 0;
        const bool xr = ew < 3 && (((ew + 1) * 32) & (a.seg - 1)) != 0;
        // bias + tanh, layer 3 (32 -> 1, taps folded by shuffles), residual, for the finished
        // layer-2 pre-activation row y (s = 32 channels of this pixel)
        // xres_m = X[y - 1] (prefetched a row ahead by the caller), xres_0 = X[y] (last row only)
        auto layer3 = [&](int y, const float (&s)[32], int par, float (&acc3)[3], float xres_m,
                          float xres_0, float* om, bool col_ok) {
            // layer-2 activation and the layer-3 taps v[ky][kx] = sum_c w3 h
            // four independent partial sums (8 channels each) for ILP
            float2 v01[4], v23[4], v45[4], v67[4];
            float v8[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                v01[g] = v23[g] = v45[g] = v67[g] = make_float2(0.f, 0.f);
                v8[g] = 0.f;
            }
#pragma unroll
            for (int c = 0; c < ((a.debug & 4) ? 0 : 32); ++c) {
                const int g = c & 3;
                const float h = tanh_fast(fmaf(s[c], inv2, c_epi.b2[c]));
                const float2 hh = make_float2(h, h);
                const float4 w0 = *reinterpret_cast<const float4*>(&c_epi.w3[c][0]);
                const float4 w1 = *reinterpret_cast<const float4*>(&c_epi.w3[c][4]);
                v01[g] = __ffma2_rn(make_float2(w0.x, w0.y), hh, v01[g]);
                v23[g] = __ffma2_rn(make_float2(w0.z, w0.w), hh, v23[g]);
                v45[g] = __ffma2_rn(make_float2(w1.x, w1.y), hh, v45[g]);
                v67[g] = __ffma2_rn(make_float2(w1.z, w1.w), hh, v67[g]);
                v8[g] = fmaf(c_epi.w3[c][8], h, v8[g]);
            }
#pragma unroll
            for (int g = 1; g < 4; ++g) {
                v01[0].x += v01[g].x; v01[0].y += v01[g].y;
                v23[0].x += v23[g].x; v23[0].y += v23[g].y;
                v45[0].x += v45[g].x; v45[0].y += v45[g].y;
                v67[0].x += v67[g].x; v67[0].y += v67[g].y;
                v8[0] += v8[g];
            }
            const float vv[9] = {v01[0].x, v01[0].y, v23[0].x, v23[0].y, v45[0].x,
                                 v45[0].y, v67[0].x, v67[0].y, v8[0]};
            // fold horizontal taps: lane x3 takes v[ky][0] from x3-1, v[ky][2] from x3+1
            float tk[3];
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const float up = __shfl_up_sync(0xffffffffu, vv[ky * 3 + 0], 1);
                const float dn = __shfl_down_sync(0xffffffffu, vv[ky * 3 + 2], 1);
                tk[ky] = vv[ky * 3 + 1] + (lane == 0 ? 0.f : up) + (lane == 31 ? 0.f : dn);
                if (lane == 31) xv0[(par * 4 + ew) * 4 + ky] = vv[ky * 3 + 0];
                if (lane == 0) xv2[(par * 4 + ew) * 4 + ky] = vv[ky * 3 + 2];
            }
            asm volatile("bar.sync 2, 128;" ::: "memory");
            if (lane == 0 && xl) {
#pragma unroll
                for (int ky = 0; ky < 3; ++ky) tk[ky] += xv0[(par * 4 + ew - 1) * 4 + ky];
            }
            if (lane == 31 && xr) {
#pragma unroll
                for (int ky = 0; ky < 3; ++ky) tk[ky] += xv2[(par * 4 + ew + 1) * 4 + ky];
            }
            // h at row y feeds output rows y+1 (ky=0), y (ky=1), y-1 (ky=2)
            acc3[(y + 1) % 3] += tk[0];
            acc3[y % 3] += tk[1];
            if (y >= 1) {
                const int yo = y - 1;
                const float o = acc3[yo % 3] + tk[2];
                acc3[yo % 3] = 0.f;
                if (col_ok) om[(int64_t)yo * a.ldo + x] = xres_m + a.alpha * (b3 + o);
            }
            if (y == n - 1) {
                const float o = acc3[y % 3];
                acc3[y % 3] = 0.f;
                if (col_ok) om[(int64_t)y * a.ldo + x] = xres_0 + a.alpha * (b3 + o);
            }
        };
        // layer 3 on the tensor core, one unit (output rows [o0, o1) of an image; h2 rows
        // [e0, e1) from layer-2 accumulators [l0, l1); Lb / Hb: global ring index of row 0)
        // pass 1 (h2 row y): layer-2 pre-activation D_{y-1}[0] + D_y[1] + D_{y+1}[2] from TMEM,
        // h2 = tanh(. inv2 + b2) as a scaled fp16 pair into h2 tile (Hb + y) % NH (pixel x at
        // row x + 1); the MMA warp contracts it with W3 into U_{Hb + y}.
        // pass 2 (two rows behind): out[o] = X[o] + alpha (b3 + inv3 (U_{o-1}[0] + U_o[1] +
        // U_{o+1}[2])).
        auto l3_unit = [&](const Unit& U, int Lb, int Hb, const float* xm, float* om,
                           bool col_ok) {
            const float inv3 = b3s[2];
            auto acc_base = [&](int j) {
                return tmem + lane_base + (uint32_t)(((Lb + j) % kNAcc) * L::kAccCols);
            };
            auto wait_acc = [&](int j) {
                const int Jg = Lb + j;
                ptx::mbar_wait(&acc_full[Jg % kNAcc], (uint32_t)((Jg / kNAcc) & 1));
                ptx::tc_fence_after();
            };
            auto release = [&](int j) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&acc_empty[(Lb + j) % kNAcc]);
            };
            auto u_col = [&](int j, int col) {
                return tmem + lane_base + (uint32_t)(kUCol0 + ((Hb + j) % NU) * 16 + col);
            };
            float xnext = col_ok ? xm[(int64_t)U.o0 * a.ldx + x] : 0.f;  // X of the next output row
            auto out_row = [&](int o) {
                const int jw = o + 1 < n ? o + 1 : o;  // newest U the row needs
                const int Jg = Hb + jw;
                ptx::mbar_wait(&u_full[Jg % NU], (uint32_t)((Jg / NU) & 1));
                ptx::tc_fence_after();
                const uint32_t u1 = ptx::tmem_ld_32x32b_x1(u_col(o, 1));
                const uint32_t u0 = o >= 1 ? ptx::tmem_ld_32x32b_x1(u_col(o - 1, 0)) : 0u;
                const uint32_t u2 = o + 1 < n ? ptx::tmem_ld_32x32b_x1(u_col(o + 1, 2)) : 0u;
                ptx::tmem_ld_wait();
                // U_{o-1} is done after this row; the unit's last row also hands back U_o and
                // U_{o+1} (an interior cut's halo row)
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (o >= 1) ptx::mbar_arrive(&u_empty[(Hb + o - 1) % NU]);
                    if (o == U.o1 - 1) {
                        ptx::mbar_arrive(&u_empty[(Hb + o) % NU]);
                        if (o + 1 < U.e1) ptx::mbar_arrive(&u_empty[(Hb + o + 1) % NU]);
                    }
                }
                const float v = __uint_as_float(u1) + (o >= 1 ? __uint_as_float(u0) : 0.f) +
                                (o + 1 < n ? __uint_as_float(u2) : 0.f);
                const float xr = xnext;
                if (o + 1 < U.o1) xnext = col_ok ? xm[(int64_t)(o + 1) * a.ldx + x] : 0.f;
                if (col_ok) om[(int64_t)o * a.ldo + x] = xr + a.alpha * fmaf(v, inv3, b3);
            };
            // at an interior cut D_{e0 - 1} = D_{l0} is data (at the image top e0 = l0 = 0)
            wait_acc(U.e0);
            if (U.e0 - 1 >= U.l0) wait_acc(U.e0 - 1);
            for (int y = U.e0; y < U.e1; ++y) {
                if (y + 1 < U.l1) wait_acc(y + 1);
                float s[32];
                uint32_t v[32], w[32];
                auto add_into = [&]() {  // s += v, as packed f32x2 adds
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        const float2 t = __fadd2_rn(make_float2(s[c], s[c + 1]),
                                                    make_float2(__uint_as_float(v[c]),
                                                                __uint_as_float(v[c + 1])));
                        s[c] = t.x;
                        s[c + 1] = t.y;
                    }
                };
                // D_y[dy = 1] and D_{y-1}[dy = 0] in flight together (one TMEM round trip)
                const bool up = y - 1 >= U.l0;
                ptx::tmem_ld_32x32b_x32(acc_base(y) + C2, w);
                if (up) ptx::tmem_ld_32x32b_x32(acc_base(y - 1), v);
                ptx::tmem_ld_wait_regs(w);
#pragma unroll
                for (int c = 0; c < 32; ++c) s[c] = __uint_as_float(w[c]);
                if (up) {
                    ptx::tmem_ld_wait_regs(v);
                    add_into();
                }
                if (y + 1 < U.l1) {
                    ptx::tmem_ld_32x32b_x32(acc_base(y + 1) + 2 * C2, v);  // D_{y+1}[dy = 2]
                    ptx::tmem_ld_wait();
                    add_into();
                }
                // D_j's last reader is h2 row j + 1 (or the unit's last h2 row)
                if (y - 1 >= U.l0) release(y - 1);
                if (y == U.e1 - 1) {
                    release(y);
                    if (y + 1 < U.l1) release(y + 1);
                }
                const int Yg = Hb + y, hs = Yg % NH;
                ptx::mbar_wait(&h2_empty[hs], (uint32_t)(((Yg / NH) & 1) ^ 1));
                uint8_t* ht = sm + L::kOffH2 + hs * L::kATile;
#pragma unroll
                for (int c8 = 0; c8 < 4; ++c8) {
                    uint32_t hw[4], lw[4];
#pragma unroll
                    for (int pr = 0; pr < 4; ++pr) {
                        const int c = c8 * 8 + 2 * pr;
                        const float2 t2 = tanh2_fast_s(
                            __ffma2_rn(make_float2(s[c], s[c + 1]), make_float2(inv2, inv2),
                                       make_float2(c_epi.b2[c], c_epi.b2[c + 1])),
                            kScaleA);
                        split_grid(t2, hw[pr], lw[pr]);
                    }
                    *reinterpret_cast<uint4*>(ht + sw128(x + 1, c8 * 16)) =
                        make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    *reinterpret_cast<uint4*>(ht + sw128(x + 1, 64 + c8 * 16)) =
                        make_uint4(lw[0], lw[1], lw[2], lw[3]);
                }
                // the output row two behind while the stores drain, then publish h2 row y
                if (y - 2 >= U.o0 && y - 2 < U.o1) out_row(y - 2);
                ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&h2_full[hs]);
            }
            for (int o = max(U.o0, U.e1 - 2); o < U.o1; ++o) out_row(o);
        };
        if constexpr (!SPLIT) {  // whole images (the common case): the tuned loop as is
        int it = 0;
        for (int64_t mem = blockIdx.x; mem < a.n_members; mem += gridDim.x, ++it) {
            float acc3[3] = {0.f, 0.f, 0.f};  // layer-3 partial sums, ring over output rows
            const float* xm = a.x + mem * W;
            float* om = a.out + mem * W;
            const bool col_ok = mem * W + x < a.cols_total;
            if constexpr (L3) {
                l3_unit(Unit{(int)mem, 0, n, 0, n, 0, n}, it * n, it * n, xm, om, col_ok);
            } else if constexpr (SH) {
                // accumulator D_j (input row j) holds contributions to output rows j + 1 (dy = 0
                // block), j (dy = 1) and j - 1 (dy = 2): output row y = D_{y-1}[0] + D_y[1] +
                // D_{y+1}[2], read straight from TMEM (three live accumulators of the ring), so no
                // running sums are carried in registers; D_{y-1} is released after row y
                auto acc_base = [&](int j) {
                    return tmem + lane_base + (uint32_t)(((it * n + j) % kNAcc) * L::kAccCols);
                };
                auto wait_acc = [&](int j) {
                    const int Jg = it * n + j;
                    ptx::mbar_wait(&acc_full[Jg % kNAcc], (uint32_t)((Jg / kNAcc) & 1));
                    ptx::tc_fence_after();
                };
                auto release = [&](int j) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&acc_empty[(it * n + j) % kNAcc]);
                };
                // SH: the cross-warp boundary taps of row y are exchanged through 4 smem buffers
                // with an mbarrier each, and consumed one row later (phase B), so the four
                // epilogue warps never wait for each other within a row.  4 buffers: a warp
                // writing row Yg has passed phase B of row Yg - 2, so every warp has finished
                // phase A of Yg - 2 and hence phase B of Yg - 4 (the buffer's previous row)
                float* xvA = xd0;        // [4][4 warps][4]: v[ky][0] of lane 31
                float* xvB = xd0 + 64;   // [4][4 warps][4]: v[ky][2] of lane 0
                auto taps = [&](const float (&sv)[32], float (&vv)[9]) {
                    float2 v01[4], v23[4], v45[4], v67[4];
                    float v8[4];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        v01[g] = v23[g] = v45[g] = v67[g] = make_float2(0.f, 0.f);
                        v8[g] = 0.f;
                    }
#pragma unroll
                    for (int c = 0; c < ((a.debug & 4) ? 0 : 32); c += 2) {
                        const float2 h2 = tanh2_fast(__ffma2_rn(make_float2(sv[c], sv[c + 1]),
                                                                make_float2(inv2, inv2),
                                                                make_float2(c_epi.b2[c], c_epi.b2[c + 1])));
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int cc = c + u, g = cc & 3;
                            const float h = u ? h2.y : h2.x;
                            const float2 hh = make_float2(h, h);
                            const float4 w0 = *reinterpret_cast<const float4*>(&c_epi.w3[cc][0]);
                            const float4 w1 = *reinterpret_cast<const float4*>(&c_epi.w3[cc][4]);
                            v01[g] = __ffma2_rn(make_float2(w0.x, w0.y), hh, v01[g]);
                            v23[g] = __ffma2_rn(make_float2(w0.z, w0.w), hh, v23[g]);
                            v45[g] = __ffma2_rn(make_float2(w1.x, w1.y), hh, v45[g]);
                            v67[g] = __ffma2_rn(make_float2(w1.z, w1.w), hh, v67[g]);
                            v8[g] = fmaf(c_epi.w3[cc][8], h, v8[g]);
                        }
                    }
#pragma unroll
                    for (int g = 1; g < 4; ++g) {
                        v01[0].x += v01[g].x; v01[0].y += v01[g].y;
                        v23[0].x += v23[g].x; v23[0].y += v23[g].y;
                        v45[0].x += v45[g].x; v45[0].y += v45[g].y;
                        v67[0].x += v67[g].x; v67[0].y += v67[g].y;
                        v8[0] += v8[g];
                    }
                    vv[0] = v01[0].x; vv[1] = v01[0].y; vv[2] = v23[0].x; vv[3] = v23[0].y;
                    vv[4] = v45[0].x; vv[5] = v45[0].y; vv[6] = v67[0].x; vv[7] = v67[0].y;
                    vv[8] = v8[0];
                };
                struct Pend {
                    float t0, t1, t2;
                    int y, Yg;
                    float xr_m, xres0;
                };
                Pend pend{0.f, 0.f, 0.f, 0, 0, 0.f, 0.f};
                auto finish = [&](const Pend& P) {
                    const int b = P.Yg % 4;
                    ptx::mbar_wait(&xb_full[b], (uint32_t)((P.Yg / 4) & 1));
                    float tk[3] = {P.t0, P.t1, P.t2};
                    if (lane == 0 && xl) {
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky) tk[ky] += xvA[(b * 4 + ew - 1) * 4 + ky];
                    }
                    if (lane == 31 && xr) {
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky) tk[ky] += xvB[(b * 4 + ew + 1) * 4 + ky];
                    }
                    const int y = P.y;
                    acc3[(y + 1) % 3] += tk[0];
                    acc3[y % 3] += tk[1];
                    if (y >= 1) {
                        const int yo = y - 1;
                        const float o = acc3[yo % 3] + tk[2];
                        acc3[yo % 3] = 0.f;
                        if (col_ok) om[(int64_t)yo * a.ldo + x] = P.xr_m + a.alpha * (b3 + o);
                    }
                    if (y == n - 1) {
                        const float o = acc3[y % 3];
                        acc3[y % 3] = 0.f;
                        if (col_ok) om[(int64_t)y * a.ldo + x] = P.xres0 + a.alpha * (b3 + o);
                    }
                };
                float xpre = 0.f;
                wait_acc(0);
                for (int y = 0; y < n; ++y) {
                    if (y + 1 < n) wait_acc(y + 1);
                    float s[32];
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(acc_base(y) + C2, v);  // D_y[dy = 1]
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 32; ++c) s[c] = __uint_as_float(v[c]);
                    auto add_into = [&]() {  // s += v, as packed f32x2 adds
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            const float2 t = __fadd2_rn(make_float2(s[c], s[c + 1]),
                                                        make_float2(__uint_as_float(v[c]),
                                                                    __uint_as_float(v[c + 1])));
                            s[c] = t.x;
                            s[c + 1] = t.y;
                        }
                    };
                    if (y >= 1) {
                        ptx::tmem_ld_32x32b_x32(acc_base(y - 1), v);  // D_{y-1}[dy = 0]
                        ptx::tmem_ld_wait();
                        add_into();
                    }
                    if (y + 1 < n) {
                        ptx::tmem_ld_32x32b_x32(acc_base(y + 1) + 2 * C2, v);  // D_{y+1}[dy = 2]
                        ptx::tmem_ld_wait();
                        add_into();
                    }
                    if (y >= 1) release(y - 1);
                    if (y == n - 1) release(y);
                    const float xr_m = xpre;  // X[y - 1]
                    xpre = col_ok ? xm[(int64_t)y * a.ldx + x] : 0.f;  // X[y]: next row's X[y' - 1]
                    // phase A: layer-3 taps, fold inside the warp, publish the boundary taps
                    const int Yg = it * n + y, b = Yg % 4;
                    float vv[9];
                    taps(s, vv);
                    float tk[3];
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky) {
                        const float up = __shfl_up_sync(0xffffffffu, vv[ky * 3 + 0], 1);
                        const float dn = __shfl_down_sync(0xffffffffu, vv[ky * 3 + 2], 1);
                        tk[ky] = vv[ky * 3 + 1] + (lane == 0 ? 0.f : up) + (lane == 31 ? 0.f : dn);
                        if (lane == 31) xvA[(b * 4 + ew) * 4 + ky] = vv[ky * 3 + 0];
                        if (lane == 0) xvB[(b * 4 + ew) * 4 + ky] = vv[ky * 3 + 2];
                    }
                    __syncwarp();
                    ptx::mbar_arrive(&xb_full[b]);
                    // phase B of the previous row (its neighbours' taps are out by now)
                    if (y >= 1) finish(pend);
                    pend = Pend{tk[0], tk[1], tk[2], y, Yg, xr_m, y == n - 1 ? xpre : 0.f};
                }
                finish(pend);
            } else {
                float xpre = 0.f;
                for (int y = 0; y < n; ++y) {
                    const int Yg = it * n + y;
                    const int q = Yg % kNAcc;
                    const int par = Yg & 1;
                    ptx::mbar_wait(&acc_full[q], (uint32_t)((Yg / kNAcc) & 1));
                    ptx::tc_fence_after();
                    const uint32_t base = tmem + lane_base + (uint32_t)(q * L::kAccCols);
                    float s[32];
                    float t[32];
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(base + 0, v);  // dx = 0 block
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 32; ++c) t[c] = __uint_as_float(v[c]);
                    if (lane == 31) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4)
                            *reinterpret_cast<float4*>(xd0 + (par * 4 + ew) * 32 + c) =
                                make_float4(t[c], t[c + 1], t[c + 2], t[c + 3]);
                    }
#pragma unroll
                    for (int c = 0; c < 32; ++c) s[c] = __shfl_up_sync(0xffffffffu, t[c], 1);
                    ptx::tmem_ld_32x32b_x32(base + 32, v);  // dx = 1 block
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 32; ++c) s[c] = (lane == 0 ? 0.f : s[c]) + __uint_as_float(v[c]);
                    ptx::tmem_ld_32x32b_x32(base + 64, v);  // dx = 2 block
                    ptx::tmem_ld_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&acc_empty[q]);
#pragma unroll
                    for (int c = 0; c < 32; ++c) t[c] = __uint_as_float(v[c]);
                    if (lane == 0) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4)
                            *reinterpret_cast<float4*>(xd2 + (par * 4 + ew) * 32 + c) =
                                make_float4(t[c], t[c + 1], t[c + 2], t[c + 3]);
                    }
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const float dn = __shfl_down_sync(0xffffffffu, t[c], 1);
                        if (lane != 31) s[c] += dn;
                    }
                    asm volatile("bar.sync 2, 128;" ::: "memory");
                    if (lane == 0 && xl) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            const float4 e4 = *reinterpret_cast<const float4*>(xd0 + (par * 4 + ew - 1) * 32 + c);
                            s[c] += e4.x; s[c + 1] += e4.y; s[c + 2] += e4.z; s[c + 3] += e4.w;
                        }
                    }
                    if (lane == 31 && xr) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            const float4 e4 = *reinterpret_cast<const float4*>(xd2 + (par * 4 + ew + 1) * 32 + c);
                            s[c] += e4.x; s[c + 1] += e4.y; s[c + 2] += e4.z; s[c + 3] += e4.w;
                        }
                    }
                    const float xr_m = xpre;
                    xpre = col_ok ? xm[(int64_t)y * a.ldx + x] : 0.f;
                    layer3(y, s, par, acc3, xr_m, y == n - 1 ? xpre : 0.f, om, col_ok);
                }
            }
        }
        } else {  // split images: units with a halo (small ensembles)
        int Lbase = 0, Hbase = 0;  // layer-1 / layer-2 rows of this CTA's earlier units
        const int n_units = (int)(a.n_members * a.parts);
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            const Unit U = unit_of<SPLIT>(a, u);
            const int64_t mem = U.mem;
            const int Lb = Lbase - U.l0, Hb = Hbase - U.e0;
            Lbase += U.l1 - U.l0;
            Hbase += U.e1 - U.e0;
            const int o0 = U.o0, o1 = U.o1;
            float acc3[3] = {0.f, 0.f, 0.f};  // layer-3 partial sums, ring over output rows
            const float* xm = a.x + mem * W;
            float* om = a.out + mem * W;
            const bool col_ok = mem * W + x < a.cols_total;
            if constexpr (L3) {
                l3_unit(U, Lb, Hb, xm, om, col_ok);
            } else if constexpr (SH) {
                // accumulator D_j (input row j) holds contributions to output rows j + 1 (dy = 0
                // block), j (dy = 1) and j - 1 (dy = 2): output row y = D_{y-1}[0] + D_y[1] +
                // D_{y+1}[2], read straight from TMEM (three live accumulators of the ring), so no
                // running sums are carried in registers; D_{y-1} is released after row y
                auto acc_base = [&](int j) {
                    return tmem + lane_base + (uint32_t)(((Lb + j) % kNAcc) * L::kAccCols);
                };
                auto wait_acc = [&](int j) {
                    const int Jg = Lb + j;
                    ptx::mbar_wait(&acc_full[Jg % kNAcc], (uint32_t)((Jg / kNAcc) & 1));
                    ptx::tc_fence_after();
                };
                auto release = [&](int j) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&acc_empty[(Lb + j) % kNAcc]);
                };
                // SH: the cross-warp boundary taps of row y are exchanged through 4 smem buffers
                // with an mbarrier each, and consumed one row later (phase B), so the four
                // epilogue warps never wait for each other within a row.  4 buffers: a warp
                // writing row Yg has passed phase B of row Yg - 2, so every warp has finished
                // phase A of Yg - 2 and hence phase B of Yg - 4 (the buffer's previous row)
                float* xvA = xd0;        // [4][4 warps][4]: v[ky][0] of lane 31
                float* xvB = xd0 + 64;   // [4][4 warps][4]: v[ky][2] of lane 0
                auto taps = [&](const float (&sv)[32], float (&vv)[9]) {
                    float2 v01[4], v23[4], v45[4], v67[4];
                    float v8[4];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        v01[g] = v23[g] = v45[g] = v67[g] = make_float2(0.f, 0.f);
                        v8[g] = 0.f;
                    }
#pragma unroll
                    for (int c = 0; c < ((a.debug & 4) ? 0 : 32); c += 2) {
                        const float2 h2 = tanh2_fast(__ffma2_rn(make_float2(sv[c], sv[c + 1]),
                                                                make_float2(inv2, inv2),
                                                                make_float2(c_epi.b2[c], c_epi.b2[c + 1])));
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const int cc = c + u, g = cc & 3;
                            const float h = u ? h2.y : h2.x;
                            const float2 hh = make_float2(h, h);
                            const float4 w0 = *reinterpret_cast<const float4*>(&c_epi.w3[cc][0]);
                            const float4 w1 = *reinterpret_cast<const float4*>(&c_epi.w3[cc][4]);
                            v01[g] = __ffma2_rn(make_float2(w0.x, w0.y), hh, v01[g]);
                            v23[g] = __ffma2_rn(make_float2(w0.z, w0.w), hh, v23[g]);
                            v45[g] = __ffma2_rn(make_float2(w1.x, w1.y), hh, v45[g]);
                            v67[g] = __ffma2_rn(make_float2(w1.z, w1.w), hh, v67[g]);
                            v8[g] = fmaf(c_epi.w3[cc][8], h, v8[g]);
                        }
                    }
#pragma unroll
                    for (int g = 1; g < 4; ++g) {
                        v01[0].x += v01[g].x; v01[0].y += v01[g].y;
                        v23[0].x += v23[g].x; v23[0].y += v23[g].y;
                        v45[0].x += v45[g].x; v45[0].y += v45[g].y;
                        v67[0].x += v67[g].x; v67[0].y += v67[g].y;
                        v8[0] += v8[g];
                    }
                    vv[0] = v01[0].x; vv[1] = v01[0].y; vv[2] = v23[0].x; vv[3] = v23[0].y;
                    vv[4] = v45[0].x; vv[5] = v45[0].y; vv[6] = v67[0].x; vv[7] = v67[0].y;
                    vv[8] = v8[0];
                };
                struct Pend {
                    float t0, t1, t2;
                    int y, Yg;
                    float xr_m, xres0;
                };
                Pend pend{0.f, 0.f, 0.f, 0, 0, 0.f, 0.f};
                auto finish = [&](const Pend& P) {
                    const int b = P.Yg % 4;
                    ptx::mbar_wait(&xb_full[b], (uint32_t)((P.Yg / 4) & 1));
                    float tk[3] = {P.t0, P.t1, P.t2};
                    if (lane == 0 && xl) {
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky) tk[ky] += xvA[(b * 4 + ew - 1) * 4 + ky];
                    }
                    if (lane == 31 && xr) {
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky) tk[ky] += xvB[(b * 4 + ew + 1) * 4 + ky];
                    }
                    const int y = P.y;
                    acc3[(y + 1) % 3] += tk[0];
                    acc3[y % 3] += tk[1];
                    if (y >= 1) {  // output rows outside [o0, o1) are another unit's (halo rows)
                        const int yo = y - 1;
                        const float o = acc3[yo % 3] + tk[2];
                        acc3[yo % 3] = 0.f;
                        if (col_ok && yo >= o0 && yo < o1)
                            om[(int64_t)yo * a.ldo + x] = P.xr_m + a.alpha * (b3 + o);
                    }
                    if (y == n - 1) {
                        const float o = acc3[y % 3];
                        acc3[y % 3] = 0.f;
                        if (col_ok && y < o1)
                            om[(int64_t)y * a.ldo + x] = P.xres0 + a.alpha * (b3 + o);
                    }
                };
                float xpre = 0.f;
                // h2 rows [e0, e1) from D rows [l0, l1): at an interior cut D_{e0 - 1} = D_{l0} is
                // data (at the image top e0 = l0 = 0 and D_{-1} is padding)
                wait_acc(U.e0);
                if (U.e0 - 1 >= U.l0) wait_acc(U.e0 - 1);
                for (int y = U.e0; y < U.e1; ++y) {
                    if (y + 1 < U.l1) wait_acc(y + 1);
                    float s[32];
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(acc_base(y) + C2, v);  // D_y[dy = 1]
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 32; ++c) s[c] = __uint_as_float(v[c]);
                    auto add_into = [&]() {  // s += v, as packed f32x2 adds
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            const float2 t = __fadd2_rn(make_float2(s[c], s[c + 1]),
                                                        make_float2(__uint_as_float(v[c]),
                                                                    __uint_as_float(v[c + 1])));
                            s[c] = t.x;
                            s[c + 1] = t.y;
                        }
                    };
                    if (y - 1 >= U.l0) {
                        ptx::tmem_ld_32x32b_x32(acc_base(y - 1), v);  // D_{y-1}[dy = 0]
                        ptx::tmem_ld_wait();
                        add_into();
                    }
                    if (y + 1 < U.l1) {
                        ptx::tmem_ld_32x32b_x32(acc_base(y + 1) + 2 * C2, v);  // D_{y+1}[dy = 2]
                        ptx::tmem_ld_wait();
                        add_into();
                    }
                    // D_j's last reader is h2 row j + 1 (or the unit's last h2 row)
                    if (y - 1 >= U.l0) release(y - 1);
                    if (y == U.e1 - 1) {
                        release(y);
                        if (y + 1 < U.l1) release(y + 1);
                    }
                    const float xr_m = xpre;  // X[y - 1]
                    xpre = col_ok ? xm[(int64_t)y * a.ldx + x] : 0.f;  // X[y]: next row's X[y' - 1]
                    // phase A: layer-3 taps, fold inside the warp, publish the boundary taps
                    const int Yg = Hb + y, b = Yg % 4;
                    float vv[9];
                    taps(s, vv);
                    float tk[3];
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky) {
                        const float up = __shfl_up_sync(0xffffffffu, vv[ky * 3 + 0], 1);
                        const float dn = __shfl_down_sync(0xffffffffu, vv[ky * 3 + 2], 1);
                        tk[ky] = vv[ky * 3 + 1] + (lane == 0 ? 0.f : up) + (lane == 31 ? 0.f : dn);
                        if (lane == 31) xvA[(b * 4 + ew) * 4 + ky] = vv[ky * 3 + 0];
                        if (lane == 0) xvB[(b * 4 + ew) * 4 + ky] = vv[ky * 3 + 2];
                    }
                    __syncwarp();
                    ptx::mbar_arrive(&xb_full[b]);
                    // phase B of the previous row (its neighbours' taps are out by now)
                    if (y > U.e0) finish(pend);
                    pend = Pend{tk[0], tk[1], tk[2], y, Yg, xr_m, y == n - 1 ? xpre : 0.f};
                }
                finish(pend);
            } else {
                float xpre = 0.f;
                for (int y = 0; y < n; ++y) {
                    const int Yg = Lb + y;  // parts == 1 here: Lb = rows of earlier images
                    const int q = Yg % kNAcc;
                    const int par = Yg & 1;
                    ptx::mbar_wait(&acc_full[q], (uint32_t)((Yg / kNAcc) & 1));
                    ptx::tc_fence_after();
                    const uint32_t base = tmem + lane_base + (uint32_t)(q * L::kAccCols);
                    float s[32];
                    float t[32];
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(base + 0, v);  // dx = 0 block
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 32; ++c) t[c] = __uint_as_float(v[c]);
                    if (lane == 31) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4)
                            *reinterpret_cast<float4*>(xd0 + (par * 4 + ew) * 32 + c) =
                                make_float4(t[c], t[c + 1], t[c + 2], t[c + 3]);
                    }
#pragma unroll
                    for (int c = 0; c < 32; ++c) s[c] = __shfl_up_sync(0xffffffffu, t[c], 1);
                    ptx::tmem_ld_32x32b_x32(base + 32, v);  // dx = 1 block
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 32; ++c) s[c] = (lane == 0 ? 0.f : s[c]) + __uint_as_float(v[c]);
                    ptx::tmem_ld_32x32b_x32(base + 64, v);  // dx = 2 block
                    ptx::tmem_ld_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&acc_empty[q]);
#pragma unroll
                    for (int c = 0; c < 32; ++c) t[c] = __uint_as_float(v[c]);
                    if (lane == 0) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4)
                            *reinterpret_cast<float4*>(xd2 + (par * 4 + ew) * 32 + c) =
                                make_float4(t[c], t[c + 1], t[c + 2], t[c + 3]);
                    }
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const float dn = __shfl_down_sync(0xffffffffu, t[c], 1);
                        if (lane != 31) s[c] += dn;
                    }
                    asm volatile("bar.sync 2, 128;" ::: "memory");
                    if (lane == 0 && xl) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            const float4 e4 = *reinterpret_cast<const float4*>(xd0 + (par * 4 + ew - 1) * 32 + c);
                            s[c] += e4.x; s[c + 1] += e4.y; s[c + 2] += e4.z; s[c + 3] += e4.w;
                        }
                    }
                    if (lane == 31 && xr) {
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            const float4 e4 = *reinterpret_cast<const float4*>(xd2 + (par * 4 + ew + 1) * 32 + c);
                            s[c] += e4.x; s[c + 1] += e4.y; s[c + 2] += e4.z; s[c + 3] += e4.w;
                        }
                    }
                    const float xr_m = xpre;
                    xpre = col_ok ? xm[(int64_t)y * a.ldx + x] : 0.f;
                    layer3(y, s, par, acc3, xr_m, y == n - 1 ? xpre : 0.f, om, col_ok);
                }
            }
        }
        }
    } else if (warp >= 1 && warp <= 3 && a.nz.n_jobs > 0) {
        // ================= noise workers: one substream per warp at a time =================
        uint64_t* s_ki = reinterpret_cast<uint64_t*>(sm + L::kOffNz);
        double* s_wi = reinterpret_cast<double*>(sm + L::kOffNz + 256 * 8);
        load_tables(s_ki, s_wi, threadIdx.x - 32, 96);
        asm volatile("bar.sync 4, 96;" ::: "memory");
        uint8_t* mine = sm + L::kOffNzW + (warp - 1) * L::kNzWarp;
        float* s_row = reinterpret_cast<float*>(mine);
        uint64_t* buf = reinterpret_cast<uint64_t*>(mine + 2 * kMaxRowCols * 4);
        const int64_t nm = a.nz.args.n_members;
        const int64_t total = nm * a.nz.n_jobs;
        for (int64_t sidx = (int64_t)blockIdx.x * 3 + (warp - 1); sidx < total;
             sidx += (int64_t)gridDim.x * 3) {
            const int j = (int)(sidx / nm);
            const int64_t local = sidx - (int64_t)j * nm;
            const Job jb = j == 0 ? a.nz.args.job[0]
                                  : (j == 1 ? a.nz.args.job[1]
                                            : (j == 2 ? a.nz.args.job[2] : a.nz.args.job[3]));
            if (a.nz.rb)
                run_stream<true>(a.nz.args, jb, local, lane, s_row, buf, s_ki, s_wi);
            else
                run_stream<false>(a.nz.args, jb, local, lane, s_row, buf, s_ki, s_wi);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc(tmem, L::kTmemAlloc);
}

__global__ void cnn3_epi_pack_kernel(const float* __restrict__ w1, const float* __restrict__ b1,
                                     const float* __restrict__ b2, const float* __restrict__ w3,
                                     const float* __restrict__ b3, Cnn3Epi* __restrict__ out) {
    for (int e = threadIdx.x; e < C1 * 18; e += blockDim.x) {
        const int c = e / 18, k = e - c * 18;  // k = ci*9 + ky*3 + kx
        out->w1[c >> 1][k * 2 + (c & 1)] = w1[c * 18 + k];
    }
    for (int e = threadIdx.x; e < C1; e += blockDim.x) out->b1[e] = b1[e];
    for (int e = threadIdx.x; e < C2 * kW3Stride; e += blockDim.x) {
        const int c = e / kW3Stride, k = e - c * kW3Stride;
        out->w3[c][k] = k < 9 ? w3[c * 9 + k] : 0.f;
    }
    for (int e = threadIdx.x; e < C2; e += blockDim.x) out->b2[e] = b2[e];
    if (threadIdx.x == 0) out->b3 = b3[0];
}

Cnn3Epi* epi_scratch() {  // per device (one process drives one GPU, but stay per-device)
    static Cnn3Epi* buf[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!buf[dev] && cudaMalloc(&buf[dev], sizeof(Cnn3Epi)) != cudaSuccess) buf[dev] = nullptr;
    return buf[dev];
}

}  // namespace

bool cnn3_tc_applicable(int n_layers, const int* widths, int rows, int cols) {
    return n_layers == 3 && widths[0] == 2 && widths[1] == C1 && widths[2] == C2 &&
           widths[3] == 1 && (cols == 32 || cols == 64 || cols == W) && rows >= 2;
}

template <bool SH>
int launch_cnn3(const Cnn3Args& a, int grid, cudaStream_t st);

namespace {
int cnn3_tc_forward_nz(const float* weights, const float* biases, float alpha, const float* x,
                       int64_t ldx, const float* u, int64_t ldu, float* out, int64_t ldo, int rows,
                       int cols, int64_t n_members, cudaStream_t st, const NoiseLaunch* nz) {
    Cnn3Args a;
    if (nz) a.nz = *nz; else a.nz.n_jobs = 0;
    a.w1 = weights;
    a.w2 = weights + C1 * 2 * 9;
    a.w3 = a.w2 + C2 * C1 * 9;
    a.b1 = biases;
    a.b2 = biases + C1;
    a.b3 = biases + C1 + C2;
    a.alpha = alpha;
    a.x = x; a.ldx = ldx; a.u = u; a.ldu = ldu; a.out = out; a.ldo = ldo;
    a.rows = rows;
    a.seg = cols;
    a.cols_total = n_members * cols;
    a.n_members = (a.cols_total + W - 1) / W;
    n_members = a.n_members;
    // 128-pixel images, fewer images than SMs: split every image's rows into `parts` units (a
    // two-row halo recomputed per cut) so that up to one unit per SM runs -- the per-image row
    // pipeline, not the SM count, bounds small ensembles.  ENKS_CNN_PARTS (tuning): 0 = auto.
    a.parts = 1;
    if (cols == W && !(nz && nz->n_jobs > 0)) {
        const int want = env_knob("ENKS_CNN_PARTS", 0);
        int parts = want > 0 ? want : (int)(kNumSMs / (n_members > 0 ? n_members : 1));
        parts = parts < 1 ? 1 : parts;
        if (parts > rows / 16) parts = rows / 16 > 0 ? rows / 16 : 1;  // >= 16 output rows each
        if (parts > 8) parts = 8;
        a.parts = parts;
    }
    {
        a.debug = debug_knob("ENKS_CNN_DEBUG", 0);  // role switches: debug builds only
        a.products = debug_knob("ENKS_CNN_PRODUCTS", 3) == 2 ? 2 : 3;  // 2 breaks 1e-4
    }
    const int64_t n_units = n_members * a.parts;
    const int grid = (int)(n_units < kNumSMs ? n_units : kNumSMs);
    {   // stream-ordered refresh of the epilogue's constant bank
        Cnn3Epi* scr = epi_scratch();
        if (!scr) {
            set_error("cnn3_tc: constant scratch allocation failed");
            return ENKS_E_CUDA;
        }
        cnn3_epi_pack_kernel<<<1, 256, 0, st>>>(a.w1, a.b1, a.b2, a.w3, a.b3, scr);
        int rc = check_launch("enks_cnn_forward(epi pack)");
        if (rc) return rc;
        if (cudaMemcpyToSymbolAsync(c_epi, scr, sizeof(Cnn3Epi), 0, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess) {
            set_error("cnn3_tc: constant upload failed");
            return ENKS_E_CUDA;
        }
    }
    if (cols == W) return launch_cnn3<true>(a, grid, st);
    return launch_cnn3<false>(a, grid, st);
}
}  // namespace

int cnn3_tc_forward(const float* weights, const float* biases, float alpha, const float* x,
                    int64_t ldx, const float* u, int64_t ldu, float* out, int64_t ldo, int rows,
                    int cols, int64_t n_members, cudaStream_t st) {
    return cnn3_tc_forward_nz(weights, biases, alpha, x, ldx, u, ldu, out, ldo, rows, cols,
                              n_members, st, nullptr);
}

template <bool SH, bool SPLIT>
int launch_cnn3_v(const Cnn3Args& a, int grid, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(cnn3_tc_kernel<SH, SPLIT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             CL<SH>::kSmem);
        if (e != cudaSuccess) {
            set_error("cnn3_tc: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = true;
    }
    cnn3_tc_kernel<SH, SPLIT><<<grid, kThreads, CL<SH>::kSmem, st>>>(a);
    return check_launch("enks_cnn_forward(tcgen05)");
}

template <bool SH>
int launch_cnn3(const Cnn3Args& a, int grid, cudaStream_t st) {
    // split images (parts > 1) only for 128-pixel rows; whole images keep the simpler instance
    if (SH && a.parts > 1) return launch_cnn3_v<true, true>(a, grid, st);
    return launch_cnn3_v<SH, false>(a, grid, st);
}

}  // namespace enks

extern "C" {

int enks_cnn_noise_fusable(int n_layers, const int* widths, int rows, int cols) {
    return widths && enks::cnn3_tc_applicable(n_layers, widths, rows, cols) ? 1 : 0;
}

int enks_cnn_forward_noise(int n_layers, const int* widths, const float* weights,
                           const float* biases, float alpha, const float* x, int64_t ldx,
                           const float* u, int64_t ldu, float* out, int64_t ldo, int rows, int cols,
                           int64_t n_members, const uint32_t* head, const uint32_t* head_dev,
                           int n_head, int64_t member0, int n_jobs, const uint32_t* t,
                           const uint32_t* channel, const int* job_rows, const double* const* diag,
                           float* const* nout, const int64_t* ld_nout, const float* const* base,
                           const int64_t* ld_base, float* const* out_plus,
                           const int64_t* ld_plus, void* stream) {
    ENKS_REQUIRE(widths && weights && biases && x && u && out, "enks_cnn_forward_noise: null pointer");
    if (!enks::cnn3_tc_applicable(n_layers, widths, rows, cols)) {
        enks::set_error("enks_cnn_forward_noise: only the fused 2-32-32-1 forecast draws noise "
                        "(check enks_cnn_noise_fusable)");
        return ENKS_E_UNSUPPORTED;
    }
    ENKS_REQUIRE(n_jobs >= 1 && n_jobs <= enks::kMaxJobs, "enks_cnn_forward_noise: 1..%d jobs",
                 enks::kMaxJobs);
    if (n_members <= 0) return ENKS_OK;
    enks::Job jobs[enks::kMaxJobs];
    for (int q = 0; q < n_jobs; ++q)
        jobs[q] = enks::Job{t[q], channel[q], job_rows[q], diag[q], nout[q], ld_nout[q],
                            base[q], ld_base[q], out_plus[q], ld_plus[q]};
    enks::NoiseLaunch L;
    int rc = enks::make_noise_launch(head, n_head, head_dev, member0, n_members, cols, jobs,
                                     n_jobs, L);
    if (rc) return rc;
    return enks::cnn3_tc_forward_nz(weights, biases, alpha, x, ldx, u, ldu, out, ldo, rows, cols,
                                     n_members, enks::as_stream(stream), &L);
}

}  // extern "C"
