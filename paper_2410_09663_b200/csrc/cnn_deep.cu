// K3 for deep CNN surrogates (BASELINE config C4: widths 2-32-...-32-1, fields a multiple of 128
// pixels wide): one kernel per layer, activations through HBM as fp16 pairs, every 32 -> 32
// layer on tcgen05.
//
// Model seam: MatrixDynamics.step (reference dynamics.py:40-50) called at enks.py:168; the CNN
// is the paper's surrogate (dynamics.py::CNNDynamics, fp64 restatement in oracle/models.py).
//
//   layer 1 (2 -> 32, SIMT):   h1 = tanh(conv(W1, [X, U]) + b1)
//   hidden (32 -> 32, tensor): h_{k+1} = tanh(conv(W_k, h_k) + b_k)
//   last (32 -> 1, SIMT):      X' = X + alpha * (conv(W_L, h_{L-1}) + b_L)
//
// Activations: [member][row][col][32 channels] as two fp16 planes h = fp16(a), l = fp16(a - h)
// (tanh outputs lie in [-1, 1], so the pair carries ~22 bits without scaling); 64 B per pixel
// and plane, so a 128-pixel strip row is one TMA box (32 ch x 130 px incl. the left/right halo,
// zero-filled outside the image) in the 64-B-row SWIZZLE_64B K-major layout kind::f16 reads.
//
// Hidden layer (persistent, one 128-pixel strip of one member at a time, rows in order):
//   warp 0  TMA producer (h and l planes of input row r -> stage ring)
//   warp 1  MMA issuer: D_r[x][(dy, co)] = sum_dx sum_ci h[r][x + dx - 1][ci] W[co][ci][dy][dx],
//           N = 96 (three vertical taps stacked), the horizontal taps as three MMAs whose A
//           operand starts one 64-B row earlier / later in the 130-row tile
//           (tools/probes/tc_shift_probe_f16.cu); three kind::f16 products per K = 16 step
//   warp 2  TMEM allocator
//   warps 4-7  epilogue: D_r's three 32-column blocks complete output row r - 1 and advance
//           rows r, r + 1 in registers; bias + tanh + fp16-pair split; 128 B stores per pixel.
#include <cuda.h>
#include <cuda_fp16.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace enks {
namespace {

constexpr int DW = 128;       // strip width = MMA M
constexpr int DC = 32;        // channels
constexpr int DN = 3 * DC;    // MMA N (dy, co)
constexpr int kDThreads = 384;
constexpr int kDStages = 6;
constexpr int kDAcc = 4;
constexpr int kARowsT = 130;                      // TMA box rows (pixels x0 - 1 .. x0 + 128)
constexpr int kATileD = 9 * 1024;                 // 136 x 64 B rounded up to 1 KB
constexpr int kBTileD = DN * 64;                  // 96 rows x 64 B = 6 KB
constexpr int kOffBD = 0;                         // [dx][h/l]
constexpr int kOffAD = kOffBD + 3 * 2 * kBTileD;  // [stage][h/l]
constexpr int kOffBiasD = kOffAD + kDStages * 2 * kATileD;
constexpr int kOffBarD = kOffBiasD + DC * 4;
constexpr int kSmemD = kOffBarD + 64 * 8 + 1024;

__device__ __forceinline__ uint32_t sw64(int row, int byte) {
    const uint32_t addr = (uint32_t)(row * 64 + byte);
    return addr ^ (((addr >> 7) & 3) << 4);
}

__device__ __forceinline__ uint64_t desc_sw64d(const void* smem) {
    const uint64_t addr = ptx::smem_u32(smem);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;  // SWIZZLE_64B
    return d;
}

__device__ __forceinline__ float tanh_d(float x) {
    x = fminf(fmaxf(x, -15.f), 15.f);
    float t, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(x * 2.8853900817779268f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f + t));
    return fmaf(-2.f, r, 1.f);
}

// 32 channel values -> fp16 pairs, 64 B per plane at pixel offset px (in halves)
__device__ __forceinline__ void store_pair32(__half* oh, __half* ol, int64_t px, const float (&a)[32]) {
    uint4 hv[4], lv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const float v0 = a[q * 8 + 2 * t], v1 = a[q * 8 + 2 * t + 1];
            const __half h0 = __float2half_rn(v0), h1 = __float2half_rn(v1);
            const __half l0 = __float2half_rn(v0 - __half2float(h0));
            const __half l1 = __float2half_rn(v1 - __half2float(h1));
            hw[t] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
            lw[t] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
        }
        hv[q] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        lv[q] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
    uint4* ph = reinterpret_cast<uint4*>(oh + px);
    uint4* pl = reinterpret_cast<uint4*>(ol + px);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        ph[q] = hv[q];
        pl[q] = lv[q];
    }
}

struct DeepArgs {
    const float* w;   // this layer (C_out, C_in, 3, 3) fp32
    const float* b;   // (C_out)
    __half* out_h;    // next activation planes [m][r][c][32]
    __half* out_l;
    int H, W;
    int64_t n_members;
    int debug;
};

__global__ void __launch_bounds__(kDThreads, 1)
    deep_hidden_kernel(const __grid_constant__ CUtensorMap tH, const __grid_constant__ CUtensorMap tL,
                       const DeepArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    float* bias = reinterpret_cast<float*>(sm + kOffBiasD);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kOffBarD);
    uint64_t* full = bars;
    uint64_t* empty = bars + kDStages;
    uint64_t* acc_full = bars + 2 * kDStages;
    uint64_t* acc_empty = acc_full + kDAcc;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kDAcc);
    // warp index / TMEM base via a lane-0 shuffle (provably warp-uniform: the converged MMA warp
    // keeps its descriptors in uniform registers)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int H = a.H, strips_w = a.W / DW;
    const int64_t n_strips = a.n_members * strips_w;

    // B[dx][row = dy*32 + co][ci] = W[co][ci][dy][dx] as fp16 pairs, SWIZZLE_64B K-major
    for (int e = threadIdx.x; e < 3 * DN * DC; e += kDThreads) {
        const int dx = e / (DN * DC), rem = e - dx * DN * DC;
        const int row = rem / DC, ci = rem - row * DC;
        const int dy = row / DC, co = row - dy * DC;
        const float v = a.w[((co * DC + ci) * 3 + dy) * 3 + dx];
        const __half h = __float2half_rn(v);
        const __half l = __float2half_rn(v - __half2float(h));
        const uint32_t off = sw64(row, ci * 2);
        *reinterpret_cast<__half*>(sm + kOffBD + (dx * 2 + 0) * kBTileD + off) = h;
        *reinterpret_cast<__half*>(sm + kOffBD + (dx * 2 + 1) * kBTileD + off) = l;
    }
    for (int e = threadIdx.x; e < DC; e += kDThreads) bias[e] = a.b[e];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kDStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int q = 0; q < kDAcc; ++q) {
            ptx::mbar_init(&acc_full[q], 1);
            ptx::mbar_init(&acc_empty[q], 4);
        }
        ptx::fence_barrier_init();
        ptx::tma_prefetch_desc(&tH);
        ptx::tma_prefetch_desc(&tL);
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

    if (warp == 0) {
        if (lane == 0) {
            int64_t g = 0;
            for (int64_t s = blockIdx.x; s < n_strips; s += gridDim.x) {
                const int64_t m = s / strips_w;
                const int x0 = (int)(s - m * strips_w) * DW;
                for (int r = 0; r < H; ++r, ++g) {
                    const int st = (int)(g % kDStages);
                    ptx::mbar_wait(&empty[st], (uint32_t)(((g / kDStages) & 1) ^ 1));
                    ptx::mbar_arrive_expect_tx(&full[st], 2 * kARowsT * 64);
                    uint8_t* ah = sm + kOffAD + (st * 2 + 0) * kATileD;
                    const int32_t rowg = (int32_t)(m * H + r);
                    ptx::tma_load_3d(&tH, &full[st], ah, 0, x0 - 1, rowg);
                    ptx::tma_load_3d(&tL, &full[st], ah + kATileD, 0, x0 - 1, rowg);
                }
            }
        }
    } else if (warp == 1) {
        {  // converged: an elected lane issues
            constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(DN >> 3) << 17) |
                                       ((uint32_t)(DW >> 4) << 24);
            int64_t g = 0;
            for (int64_t s = blockIdx.x; s < n_strips; s += gridDim.x) {
                for (int r = 0; r < H; ++r, ++g) {
                    const int st = (int)(g % kDStages), q = (int)(g % kDAcc);
                    ptx::mbar_wait(&acc_empty[q], (uint32_t)(((g / kDAcc) & 1) ^ 1));
                    ptx::mbar_wait(&full[st], (uint32_t)((g / kDStages) & 1));
                    ptx::tc_fence_after();
                    const uint8_t* ah = sm + kOffAD + (st * 2 + 0) * kATileD;
                    const uint8_t* al = ah + kATileD;
                    const uint32_t d = tmem + (uint32_t)(q * DN);
#pragma unroll
                    for (int dx = 0; dx < 3; ++dx) {
                        const uint8_t* bh = sm + kOffBD + (dx * 2 + 0) * kBTileD;
                        const uint8_t* bl = bh + kBTileD;
#pragma unroll
                        for (int k = 0; k < ((a.debug & 1) ? 0 : DC / 16); ++k) {
                            const uint64_t dah = desc_sw64d(ah + dx * 64 + 32 * k);
                            const uint64_t dal = desc_sw64d(al + dx * 64 + 32 * k);
                            const uint64_t dbh = desc_sw64d(bh + 32 * k);
                            const uint64_t dbl = desc_sw64d(bl + 32 * k);
                            ptx::mma_f16_ss_elect(d, dal, dbh, idesc, (dx == 0 && k == 0) ? 0u : 1u);
                            ptx::mma_f16_ss_elect(d, dah, dbl, idesc, 1u);
                            ptx::mma_f16_ss_elect(d, dah, dbh, idesc, 1u);
                        }
                    }
                    ptx::mma_commit_elect(&empty[st]);
                    ptx::mma_commit_elect(&acc_full[q]);
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        const int ew = warp - 4;
        const int x = ew * 32 + lane;
        const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
        int64_t g = 0;
        for (int64_t s = blockIdx.x; s < n_strips; s += gridDim.x) {
            const int64_t m = s / strips_w;
            const int x0 = (int)(s - m * strips_w) * DW;
            auto emit = [&](int row, const float (&pre)[32]) {
                float act[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) act[c] = tanh_d(pre[c] + bias[c]);
                const int64_t px = ((m * H + row) * a.W + x0 + x) * (int64_t)DC;
                store_pair32(a.out_h, a.out_l, px, act);
            };
            float pp[32], pc[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) pp[c] = pc[c] = 0.f;
            for (int r = 0; r < H; ++r, ++g) {
                const int q = (int)(g % kDAcc);
                ptx::mbar_wait(&acc_full[q], (uint32_t)((g / kDAcc) & 1));
                ptx::tc_fence_after();
                const uint32_t base = tmem + lane_base + (uint32_t)(q * DN);
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(base + 2 * DC, v);  // dy = 2 -> output row r - 1
                ptx::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c) pp[c] += __uint_as_float(v[c]);
                ptx::tmem_ld_32x32b_x32(base + DC, v);      // dy = 1 -> output row r
                ptx::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 32; ++c) pc[c] += __uint_as_float(v[c]);
                ptx::tmem_ld_32x32b_x32(base, v);           // dy = 0 -> output row r + 1
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&acc_empty[q]);
                if (r >= 1) emit(r - 1, pp);
                if (r == H - 1) emit(r, pc);
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    pp[c] = pc[c];
                    pc[c] = __uint_as_float(v[c]);
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc(tmem, 512);
}

// layer 1: 2 -> 32 from the member-column [X; U] blocks, thread = pixel
__global__ void __launch_bounds__(128) deep_first_kernel(const float* __restrict__ x, int64_t ldx,
                                                         const float* __restrict__ u, int64_t ldu,
                                                         const float* __restrict__ w,
                                                         const float* __restrict__ b, int H, int W,
                                                         int64_t m0, __half* oh, __half* ol) {
    __shared__ float sw[DC * 18], sb[DC];
    for (int e = threadIdx.x; e < DC * 18; e += blockDim.x) sw[e] = w[e];
    for (int e = threadIdx.x; e < DC; e += blockDim.x) sb[e] = b[e];
    __syncthreads();
    const int strips = W / DW;
    const int r = blockIdx.x / strips, c = (blockIdx.x - r * strips) * DW + threadIdx.x;
    const int64_t m = blockIdx.y;  // member within the chunk
    const int64_t col = (m0 + m) * W;
    float in[18];
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
            const int rr = r + ky - 1, cc = c + kx - 1;
            const bool ok = rr >= 0 && rr < H && cc >= 0 && cc < W;
            in[ky * 3 + kx] = ok ? __ldg(x + rr * ldx + col + cc) : 0.f;
            in[9 + ky * 3 + kx] = ok ? __ldg(u + rr * ldu + col + cc) : 0.f;
        }
    float act[32];
#pragma unroll
    for (int co = 0; co < DC; ++co) {
        float acc = sb[co];
#pragma unroll
        for (int k = 0; k < 18; ++k) acc = fmaf(sw[co * 18 + k], in[k], acc);
        act[co] = tanh_d(acc);
    }
    store_pair32(oh, ol, ((m * H + r) * (int64_t)W + c) * DC, act);
}

// last layer: 32 -> 1 + residual, thread = pixel; reads the fp16-pair activation neighbourhood
__global__ void __launch_bounds__(128) deep_last_kernel(const __half* __restrict__ ah,
                                                        const __half* __restrict__ al,
                                                        const float* __restrict__ w,
                                                        const float* __restrict__ b, float alpha,
                                                        const float* __restrict__ x, int64_t ldx,
                                                        float* __restrict__ out, int64_t ldo, int H,
                                                        int W, int64_t m0) {
    __shared__ float sw[9 * DC];  // [ky*3+kx][ci]
    for (int e = threadIdx.x; e < 9 * DC; e += blockDim.x) {
        const int k = e / DC, ci = e - k * DC;
        sw[e] = w[ci * 9 + k];
    }
    __syncthreads();
    const int strips = W / DW;
    const int r = blockIdx.x / strips, c = (blockIdx.x - r * strips) * DW + threadIdx.x;
    const int64_t m = blockIdx.y;
    float acc = b[0];
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
            const int rr = r + ky - 1, cc = c + kx - 1;
            if (rr < 0 || rr >= H || cc < 0 || cc >= W) continue;
            const int64_t px = ((m * H + rr) * (int64_t)W + cc) * DC;
            const uint4* ph = reinterpret_cast<const uint4*>(ah + px);
            const uint4* pl = reinterpret_cast<const uint4*>(al + px);
            const float* wk = sw + (ky * 3 + kx) * DC;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 hv = __ldg(ph + q), lv = __ldg(pl + q);
                const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 h2 = __half22float2(*reinterpret_cast<const __half2*>(&hw[t]));
                    const float2 l2 = __half22float2(*reinterpret_cast<const __half2*>(&lw[t]));
                    acc = fmaf(wk[q * 8 + 2 * t], h2.x + l2.x, acc);
                    acc = fmaf(wk[q * 8 + 2 * t + 1], h2.y + l2.y, acc);
                }
            }
        }
    const int64_t col = (m0 + m) * W + c;
    out[r * ldo + col] = x[r * ldx + col] + alpha * acc;
}

// Row-streaming variant of the 32 -> 1 layer: one CTA per member image (a thread per column, all
// W <= 1024 columns, so horizontal neighbours never cross CTAs), each thread walking all rows.  Each activation is read ONCE (the gather form above reads every pixel
// nine times) and turned into its nine tap contributions v[ky][kx] = sum_ci w[ci][ky][kx] h[ci]
// (nine independent FMA chains instead of one 288-long chain); horizontal taps are folded with
// warp shuffles plus a per-row exchange between the strip's four warps, vertical taps through a
// 3-row register ring (output row r is complete after input row r + 1).
__global__ void __launch_bounds__(1024) deep_last_rows_kernel(const __half* __restrict__ ah,
                                                           const __half* __restrict__ al,
                                                           const float* __restrict__ w,
                                                           const float* __restrict__ b, float alpha,
                                                           const float* __restrict__ x, int64_t ldx,
                                                           float* __restrict__ out, int64_t ldo,
                                                           int H, int W, int64_t m0) {
    __shared__ float sw[DC * 12];        // [ci][ky*3+kx], padded to 12
    __shared__ float xa[2][32][4], xb[2][32][4];  // [parity][warp][ky]: boundary taps
    for (int e = threadIdx.x; e < DC * 12; e += blockDim.x) {
        const int ci = e / 12, k = e - ci * 12;
        sw[e] = k < 9 ? w[ci * 9 + k] : 0.f;
    }
    __syncthreads();
    const int c = threadIdx.x;  // blockDim.x == W
    const int64_t m = blockIdx.y;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const bool xl = c > 0 && lane == 0, xr = c < W - 1 && lane == 31;  // neighbour across warps
    const float bias = b[0];
    const int64_t col = (m0 + m) * W + c;
    float acc3[3] = {0.f, 0.f, 0.f};
    for (int rr = 0; rr < H; ++rr) {
        const int64_t px = ((m * H + rr) * (int64_t)W + c) * DC;
        const uint4* ph = reinterpret_cast<const uint4*>(ah + px);
        const uint4* pl = reinterpret_cast<const uint4*>(al + px);
        float v[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) v[k] = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 hv = __ldg(ph + q), lv = __ldg(pl + q);
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float2 h2 = __half22float2(*reinterpret_cast<const __half2*>(&hw[t]));
                const float2 l2 = __half22float2(*reinterpret_cast<const __half2*>(&lw[t]));
                const float a0 = h2.x + l2.x, a1 = h2.y + l2.y;
                const float* w0 = sw + (q * 8 + 2 * t) * 12;
                const float* w1 = w0 + 12;
#pragma unroll
                for (int k = 0; k < 9; ++k) v[k] = fmaf(w1[k], a1, fmaf(w0[k], a0, v[k]));
            }
        }
        // horizontal fold: column c takes v[ky][0] of c - 1 and v[ky][2] of c + 1
        float tk[3];
        const int par = rr & 1;
#pragma unroll
        for (int ky = 0; ky < 3; ++ky) {
            const float up = __shfl_up_sync(0xffffffffu, v[ky * 3 + 0], 1);
            const float dn = __shfl_down_sync(0xffffffffu, v[ky * 3 + 2], 1);
            tk[ky] = v[ky * 3 + 1] + (lane == 0 ? 0.f : up) + (lane == 31 ? 0.f : dn);
            if (lane == 31) xa[par][wp][ky] = v[ky * 3 + 0];
            if (lane == 0) xb[par][wp][ky] = v[ky * 3 + 2];
        }
        __syncthreads();
        if (xl) {
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) tk[ky] += xa[par][wp - 1][ky];
        }
        if (xr) {
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) tk[ky] += xb[par][wp + 1][ky];
        }
        // input row rr feeds output rows rr + 1 (ky = 0), rr (ky = 1), rr - 1 (ky = 2)
        acc3[(rr + 1) % 3] += tk[0];
        acc3[rr % 3] += tk[1];
        if (rr >= 1) {
            const int ro = rr - 1;
            const float o = acc3[ro % 3] + tk[2];
            acc3[ro % 3] = 0.f;
            out[ro * ldo + col] = x[ro * ldx + col] + alpha * (bias + o);
        }
        if (rr == H - 1) {
            const float o = acc3[rr % 3];
            acc3[rr % 3] = 0.f;
            out[rr * ldo + col] = x[rr * ldx + col] + alpha * (bias + o);
        }
    }
}

typedef CUresult (*EncodeTiledFnD)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool act_map(CUtensorMap* mp, const void* base, int64_t rows_total, int W) {
    static EncodeTiledFnD fn = nullptr;
    if (!fn) {
        void* q = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &qr) !=
                cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            return false;
        fn = reinterpret_cast<EncodeTiledFnD>(q);
    }
    cuuint64_t dims[3] = {(cuuint64_t)DC, (cuuint64_t)W, (cuuint64_t)rows_total};
    cuuint64_t strides[2] = {(cuuint64_t)DC * 2, (cuuint64_t)W * DC * 2};
    cuuint32_t box[3] = {(cuuint32_t)DC, (cuuint32_t)kARowsT, 1};
    cuuint32_t es[3] = {1, 1, 1};
    return fn(mp, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box,
              es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool cnn_deep_applicable(int n_layers, const int* widths, int rows, int cols) {
    if (n_layers < 3 || widths[0] != 2 || widths[n_layers] != 1 || cols % DW != 0 || rows < 2)
        return false;
    for (int l = 1; l < n_layers; ++l)
        if (widths[l] != DC) return false;
    return true;
}

int64_t cnn_deep_member_bytes(int rows, int cols) {
    return 2LL * 2 * (int64_t)rows * cols * DC * (int64_t)sizeof(__half);  // two tensors, h + l
}

int cnn_deep_forward(int n_layers, const float* weights, const float* biases, float alpha,
                     const float* x, int64_t ldx, const float* u, int64_t ldu, float* out,
                     int64_t ldo, int rows, int cols, int64_t n_members, void* ws, int64_t ws_bytes,
                     cudaStream_t st) {
    const int64_t per = cnn_deep_member_bytes(rows, cols);
    ENKS_REQUIRE(ws && ws_bytes >= per, "enks_cnn_forward: deep CNN needs >= %lld B of workspace",
                 (long long)per);
    const int64_t chunk_max = ws_bytes / per;
    const int64_t plane = (int64_t)rows * cols * DC;  // halves per member and plane
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(deep_hidden_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemD);
        if (e != cudaSuccess) {
            set_error("cnn_deep: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = true;
    }
    const int debug = debug_knob("ENKS_CNN_DEBUG", 0);
    // weight / bias offsets per layer
    int woff[16], boff[16];
    {
        int wo = 0, bo = 0;
        for (int l = 0; l < n_layers; ++l) {
            const int ci = l == 0 ? 2 : DC, co = l == n_layers - 1 ? 1 : DC;
            woff[l] = wo;
            boff[l] = bo;
            wo += co * ci * 9;
            bo += co;
        }
    }
    for (int64_t m0 = 0; m0 < n_members; m0 += chunk_max) {
        const int64_t cm = (n_members - m0 < chunk_max) ? n_members - m0 : chunk_max;
        __half* t0h = static_cast<__half*>(ws);
        __half* t0l = t0h + cm * plane;
        __half* t1h = t0l + cm * plane;
        __half* t1l = t1h + cm * plane;
        const dim3 pgrid((unsigned)(rows * (cols / DW)), (unsigned)cm);
        deep_first_kernel<<<pgrid, DW, 0, st>>>(x, ldx, u, ldu, weights + woff[0], biases + boff[0],
                                                rows, cols, m0, t0h, t0l);
        int rc = check_launch("enks_cnn_forward(deep layer 1)");
        if (rc) return rc;
        for (int l = 1; l < n_layers - 1; ++l) {
            CUtensorMap mh, ml;
            if (!act_map(&mh, t0h, cm * rows, cols) || !act_map(&ml, t0l, cm * rows, cols)) {
                set_error("cnn_deep: cuTensorMapEncodeTiled failed");
                return ENKS_E_UNSUPPORTED;
            }
            DeepArgs da{weights + woff[l], biases + boff[l], t1h, t1l, rows, cols, cm, debug};
            const int64_t strips = cm * (cols / DW);
            const int grid = (int)(strips < kNumSMs ? strips : kNumSMs);
            deep_hidden_kernel<<<grid, kDThreads, kSmemD, st>>>(mh, ml, da);
            rc = check_launch("enks_cnn_forward(deep hidden)");
            if (rc) return rc;
            __half* th = t0h;
            __half* tl = t0l;
            t0h = t1h;
            t0l = t1l;
            t1h = th;
            t1l = tl;
        }
        {
            if (env_knob("ENKS_DEEP_LAST", 1) == 0 || cols > 1024 || cols % 32)
                deep_last_kernel<<<pgrid, DW, 0, st>>>(t0h, t0l, weights + woff[n_layers - 1],
                                                       biases + boff[n_layers - 1], alpha, x, ldx,
                                                       out, ldo, rows, cols, m0);
            else
                deep_last_rows_kernel<<<dim3(1, (unsigned)cm), (unsigned)cols, 0, st>>>(
                    t0h, t0l, weights + woff[n_layers - 1], biases + boff[n_layers - 1], alpha, x,
                    ldx, out, ldo, rows, cols, m0);
        }
        rc = check_launch("enks_cnn_forward(deep last)");
        if (rc) return rc;
    }
    return ENKS_OK;
}

}  // namespace enks
