// K3: layer-fused CNN forecast X' = X + alpha * CNN([X, U]) on the CUDA cores.
//
// The model seam is MatrixDynamics.step (reference dynamics.py:40-50), called
// for the whole member batch at enks.py:168.  The CNN surrogate itself is not
// in the reference; its definition (3x3 kernels, zero 'same'
// padding per layer, tanh between layers, residual output) is fixed in
// paper_2410_09663_b200/dynamics.py::CNNDynamics and restated in fp64 by
// oracle/models.py.
//
// One CTA computes a TILE x TILE output patch of one member through all
// layers: the input halo (TILE + 2L)^2 x 2 and every intermediate activation
// stay in shared memory, so HBM sees X and U once and X' once.  Activations
// at positions outside the image are forced to zero (that is what 'same'
// zero padding of the next layer reads).
#include <stdlib.h>

#include "common.cuh"

namespace enks {

bool cnn3_tc_applicable(int n_layers, const int* widths, int rows, int cols);
bool cnn_deep_applicable(int n_layers, const int* widths, int rows, int cols);
int64_t cnn_deep_member_bytes(int rows, int cols);
int cnn_deep_forward(int n_layers, const float* weights, const float* biases, float alpha,
                     const float* x, int64_t ldx, const float* u, int64_t ldu, float* out,
                     int64_t ldo, int rows, int cols, int64_t n_members, void* ws, int64_t ws_bytes,
                     cudaStream_t st);
int cnn3_tc_forward(const float* weights, const float* biases, float alpha, const float* x,
                    int64_t ldx, const float* u, int64_t ldu, float* out, int64_t ldo, int rows,
                    int cols, int64_t n_members, cudaStream_t st);

namespace {

constexpr int kTile = 16;
constexpr int kThreads = 256;
constexpr int kMaxWidth = 32;
constexpr int kMaxLayers = 8;
constexpr int kCoGroup = 8;

struct CnnArgs {
    int n_layers;
    int widths[kMaxLayers + 1];
    int w_off[kMaxLayers];  // offsets into the packed weight array (floats)
    int b_off[kMaxLayers];
    const float* weights;
    const float* biases;
    float alpha;
    const float* x;
    int64_t ldx;
    const float* u;
    int64_t ldu;
    float* out;
    int64_t ldo;
    int rows, cols;
    int tiles_x;
    int in_floats;   // staged input halo (2 channels)
    int act_floats;  // per ping-pong activation buffer
    int w_floats;    // total weight floats (smem copy, layout [layer][ci][3][3][co])
    int w_global;    // 1: weights too large for shared memory -> read (L1-cached) from global
};

// WG: weights read from global memory (deep nets whose weights exceed shared memory); a template
// parameter, not a runtime flag, so the common shared-memory path keeps a branch-free FMA loop
template <bool WG>
__global__ void __launch_bounds__(kThreads) cnn_fused_kernel(const CnnArgs a) {
    extern __shared__ __align__(16) float sm[];
    float* sw = sm;                        // weights, transposed to [ci][ky][kx][co]
    float* sb = sw + a.w_floats;           // biases
    float* buf0 = sb + a.n_layers * kMaxWidth;  // staged [X, U] halo
    float* act0 = buf0 + a.in_floats;
    float* act1 = act0 + a.act_floats;

    const int L = a.n_layers;
    const int64_t member = blockIdx.y;
    const int ty0 = (blockIdx.x / a.tiles_x) * kTile, tx0 = (blockIdx.x % a.tiles_x) * kTile;

    // stage weights: global [co][ci][ky][kx] -> smem [ci][ky][kx][co]
    if (!WG) {
        int off = 0;
        for (int l = 0; l < L; ++l) {
            const int ci_n = a.widths[l], co_n = a.widths[l + 1];
            const int cnt = co_n * ci_n * 9;
            for (int e = threadIdx.x; e < cnt; e += kThreads) {
                const int co = e / (ci_n * 9), rem = e - co * ci_n * 9;
                sw[off + rem * co_n + co] = a.weights[a.w_off[l] + e];
            }
            off += cnt;
        }
    }
    for (int l = 0; l < L; ++l)
        for (int e = threadIdx.x; e < a.widths[l + 1]; e += kThreads)
            sb[l * kMaxWidth + e] = a.biases[a.b_off[l] + e];
    // stage the input halo: region (kTile + 2L)^2, channels [X, U], origin (ty0 - L, tx0 - L)
    const int R0 = kTile + 2 * L;
    {
        const float* xm = a.x + member * a.cols;
        const float* um = a.u + member * a.cols;
        for (int e = threadIdx.x; e < R0 * R0; e += kThreads) {
            const int yy = e / R0, xx = e - yy * R0;
            const int gy = ty0 - L + yy, gx = tx0 - L + xx;
            const bool in = gy >= 0 && gy < a.rows && gx >= 0 && gx < a.cols;
            buf0[e] = in ? xm[(int64_t)gy * a.ldx + gx] : 0.f;
            buf0[R0 * R0 + e] = in ? um[(int64_t)gy * a.ldu + gx] : 0.f;
        }
    }
    __syncthreads();

    float* in = buf0;
    float* outb = act0;
    int w_base = 0;
    for (int l = 0; l < L; ++l) {
        const int ci_n = a.widths[l], co_n = a.widths[l + 1];
        const int Rin = kTile + 2 * (L - l), Rout = Rin - 2;
        const int off = l + 1;  // output region origin = tile origin - (L - l - 1)
        const int n_pos = Rout * Rout;
        const int n_grp = (co_n + kCoGroup - 1) / kCoGroup;
        const bool last = (l == L - 1);
        for (int item = threadIdx.x; item < n_pos * n_grp; item += kThreads) {
            const int g = item / n_pos, pos = item - g * n_pos;
            const int oy = pos / Rout, ox = pos - oy * Rout;
            const int gy = ty0 - L + off + oy, gx = tx0 - L + off + ox;
            const bool inside = gy >= 0 && gy < a.rows && gx >= 0 && gx < a.cols;
            const int co0 = g * kCoGroup;
            float acc[kCoGroup];
#pragma unroll
            for (int c = 0; c < kCoGroup; ++c)
                acc[c] = (co0 + c < co_n) ? sb[l * kMaxWidth + co0 + c] : 0.f;
            if (inside) {
                for (int ci = 0; ci < ci_n; ++ci) {
                    const float* ip = in + ci * Rin * Rin + oy * Rin + ox;
                    const float* wp = sw + w_base + ci * 9 * co_n + co0;
                    // global layout [co][ci][ky][kx]: weight of (co0 + c, ci, k) at gw[c * 9 ci_n + k]
                    const float* gw = a.weights + a.w_off[l] + (int64_t)co0 * ci_n * 9 + ci * 9;
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                        for (int kx = 0; kx < 3; ++kx) {
                            const float v = ip[ky * Rin + kx];
                            const float* wk = wp + (ky * 3 + kx) * co_n;
#pragma unroll
                            for (int c = 0; c < kCoGroup; ++c)
                                if (co0 + c < co_n) {
                                    const float w = WG ? __ldg(gw + c * 9 * ci_n + ky * 3 + kx)
                                                       : wk[c];
                                    acc[c] = fmaf(w, v, acc[c]);
                                }
                        }
                }
            }
            if (!last) {
#pragma unroll
                for (int c = 0; c < kCoGroup; ++c)
                    if (co0 + c < co_n)
                        outb[(co0 + c) * Rout * Rout + pos] = inside ? tanhf(acc[c]) : 0.f;
            } else if (inside && g == 0) {
                // residual: X' = X + alpha * y  (X is channel 0 of the staged input)
                const float xin = buf0[(oy + L) * R0 + (ox + L)];
                a.out[(int64_t)gy * a.ldo + member * a.cols + gx] = xin + a.alpha * acc[0];
            }
        }
        __syncthreads();
        w_base += ci_n * 9 * co_n;
        if (!last) {
            // the staged input (buf0) must survive for the residual: ping-pong act0/act1
            in = outb;
            outb = (outb == act0) ? act1 : act0;
        }
    }
}

}  // namespace
}  // namespace enks

extern "C" {

int enks_cnn_max_width(void) { return enks::kMaxWidth; }

int64_t enks_cnn_ws_bytes(int n_layers, const int* widths, int rows, int cols, int64_t n_members) {
    if (!widths || n_layers < 1 || n_members <= 0) return 0;
    if (enks::env_knob("ENKS_CNN_FUSED", 1) != 0 &&
        enks::cnn3_tc_applicable(n_layers, widths, rows, cols))
        return 0;
    if (!enks::cnn_deep_applicable(n_layers, widths, rows, cols)) return 0;
    const int64_t per = enks::cnn_deep_member_bytes(rows, cols);
    const int64_t cap = (4LL << 30) / per;  // member chunks of <= 4 GiB of activations
    return per * (n_members < cap ? n_members : (cap > 0 ? cap : 1));
}

int enks_cnn_forward(int n_layers, const int* widths, const float* weights, const float* biases,
                     float alpha, const float* x, int64_t ldx, const float* u, int64_t ldu,
                     float* out, int64_t ldo, int rows, int cols, int64_t n_members, void* stream) {
    return enks_cnn_forward_ws(n_layers, widths, weights, biases, alpha, x, ldx, u, ldu, out, ldo,
                               rows, cols, n_members, nullptr, 0, stream);
}

int enks_cnn_forward_ws(int n_layers, const int* widths, const float* weights,
                        const float* biases, float alpha, const float* x, int64_t ldx,
                        const float* u, int64_t ldu, float* out, int64_t ldo, int rows, int cols,
                        int64_t n_members, void* ws, int64_t ws_bytes, void* stream) {
    using namespace enks;
    ENKS_REQUIRE(n_layers >= 1 && n_layers <= kMaxLayers, "enks_cnn_forward: 1..%d layers",
                 kMaxLayers);
    ENKS_REQUIRE(widths && weights && biases && x && u && out, "enks_cnn_forward: null pointer");
    ENKS_REQUIRE(widths[0] == 2 && widths[n_layers] == 1,
                 "enks_cnn_forward: widths must start at 2 ([X, U]) and end at 1");
    if (n_members <= 0 || rows <= 0 || cols <= 0) return ENKS_OK;
    {
        // tuning: tcgen05 kernels vs the SIMT one (same results to rounding), read once
        const bool allow = env_knob("ENKS_CNN_TC", 1) != 0;
        const bool fused_ok = env_knob("ENKS_CNN_FUSED", 1) != 0;
        if (allow && fused_ok && cnn3_tc_applicable(n_layers, widths, rows, cols))
            return cnn3_tc_forward(weights, biases, alpha, x, ldx, u, ldu, out, ldo, rows, cols, n_members,
                                   as_stream(stream));
        if (allow && ws && cnn_deep_applicable(n_layers, widths, rows, cols))
            return cnn_deep_forward(n_layers, weights, biases, alpha, x, ldx, u, ldu, out, ldo, rows,
                                    cols, n_members, ws, ws_bytes, as_stream(stream));
    }
    CnnArgs a;
    a.n_layers = n_layers;
    int woff = 0, boff = 0, max_act = 0;
    for (int l = 0; l <= n_layers; ++l) {
        ENKS_REQUIRE(widths[l] >= 1 && widths[l] <= kMaxWidth, "enks_cnn_forward: width %d > %d",
                     widths[l], kMaxWidth);
        a.widths[l] = widths[l];
    }
    for (int l = 0; l < n_layers; ++l) {
        a.w_off[l] = woff;
        a.b_off[l] = boff;
        woff += widths[l + 1] * widths[l] * 9;
        boff += widths[l + 1];
        const int rout = kTile + 2 * (n_layers - l - 1);
        if (l < n_layers - 1) max_act = max_act > rout * rout * widths[l + 1] ? max_act
                                                                             : rout * rout * widths[l + 1];
    }
    a.weights = weights;
    a.biases = biases;
    a.alpha = alpha;
    a.x = x; a.ldx = ldx; a.u = u; a.ldu = ldu; a.out = out; a.ldo = ldo;
    a.rows = rows; a.cols = cols;
    a.tiles_x = (cols + kTile - 1) / kTile;
    const int tiles_y = (rows + kTile - 1) / kTile;
    const int r0 = kTile + 2 * n_layers;
    a.in_floats = (2 * r0 * r0 + 3) & ~3;
    a.act_floats = (max_act + 3) & ~3;
    a.w_floats = (woff + 3) & ~3;
    size_t smem3 = sizeof(float) * ((size_t)a.w_floats + n_layers * kMaxWidth +
                                    (size_t)a.in_floats + 2 * (size_t)a.act_floats);
    a.w_global = 0;
    if (smem3 > 227 * 1024) {  // deep nets: keep the weights in global memory (L1-cached)
        a.w_global = 1;
        smem3 -= sizeof(float) * (size_t)a.w_floats;
        a.w_floats = 0;
    }
    ENKS_REQUIRE(smem3 <= 227 * 1024, "enks_cnn_forward: shared memory %zu B exceeds 227 KB", smem3);
    static size_t configured[2] = {0, 0};
    if (smem3 > 48 * 1024 && smem3 > configured[a.w_global]) {
        cudaError_t e = cudaFuncSetAttribute(
            a.w_global ? cnn_fused_kernel<true> : cnn_fused_kernel<false>,
            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
        if (e != cudaSuccess) {
            set_error("enks_cnn_forward: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured[a.w_global] = smem3;
    }
    dim3 grid((unsigned)(a.tiles_x * tiles_y), (unsigned)n_members);
    ENKS_REQUIRE(n_members < 65536, "enks_cnn_forward: n_members must be < 65536 per launch");
    if (a.w_global)
        cnn_fused_kernel<true><<<grid, kThreads, smem3, as_stream(stream)>>>(a);
    else
        cnn_fused_kernel<false><<<grid, kThreads, smem3, as_stream(stream)>>>(a);
    return check_launch("enks_cnn_forward");
}

}  // extern "C"
