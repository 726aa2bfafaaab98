// 2-D viscous Burgers forecast for every member.
//
// Reference: pkg/src/enksmpc/dynamics.py:156-216 (_neighbor_slices, _cfl_check,
// _step_packed) and 246-270 (BurgersDynamics.step: cfg.substeps solver steps with
// the force held constant), called for the whole member batch at enks.py:168.
//
// Layout (member-column, as the rest of the smoother): the packed field of member i
// is rows 0..2g-1 (phi_x above phi_y), columns i*g .. i*g+g-1 of a (2g x K) matrix.
// The control is (u_rows x K) with u_rows = 2 (boundary) or 2g (pointwise).
//
// Per point:  lap = (up + down + left + right - 4 q) / dx^2        (Neumann: edge copy)
//             ddx = (vx > 0 ? q - left : right - q) / dx           (upwind by local vx)
//             ddy = (vy > 0 ? q - up   : down  - q) / dx           (upwind by local vy)
//             q'  = q + dt (nu lap - vx ddx - vy ddy)   [+ dt f]
//
// Fused kernel: one CTA per member, the member's 2g x g field resident in shared
// memory (ping-pong) for all substeps, so the stencil's HBM traffic is one read of
// the field + force and one write per forecast regardless of cfg.substeps.  Fields
// that do not fit in shared memory run one global-memory launch per substep.
//
// CFL (dynamics.py:168-180): the reference checks max|phi| over the whole batch on
// the input of every substep and raises.  Here every CTA folds max|phi| of each
// substep input into `vmax` (atomicMax on the float bits; values are >= 0) and
// raises bit 1 of `flags` on a non-finite entry; the host reads both lazily and
// raises CflError (no synchronisation inside a horizon).
#include "common.cuh"

namespace enks {
namespace {

constexpr int kBurgersThreads = 512;
constexpr int kBurgersSmemMax = 200 * 1024;

struct BurgersArgs {
    const float* x;
    int64_t ldx;
    const float* u;
    int64_t ldu;
    float* out;
    int64_t ldo;
    int g;        // grid_n: field is 2g x g per member
    int u_rows;   // 2 (boundary) or 2g (pointwise); 0 = no force
    int n_members;
    int substeps;
    float nu, dt, inv_dx, inv_dx2;
    float* vmax;
    int* flags;
};

__device__ __forceinline__ float stencil(float q, float up, float down, float left, float right,
                                         float vx, float vy, const BurgersArgs& a) {
    const float lap = (up + down + left + right - 4.f * q) * a.inv_dx2;
    const float ddx = (vx > 0.f ? q - left : right - q) * a.inv_dx;
    const float ddy = (vy > 0.f ? q - up : down - q) * a.inv_dx;
    return q + a.dt * (a.nu * lap - vx * ddx - vy * ddy);
}

__device__ __forceinline__ float force_at(const BurgersArgs& a, int r, int64_t col) {
    if (a.u_rows == 0) return 0.f;
    const int g = a.g;
    if (a.u_rows == 2 * g) return a.dt * a.u[r * a.ldu + col];
    // boundary: rows g-1 (phi_x) and 2g-1 (phi_y) take force rows 0 and 1
    if (r == g - 1) return a.dt * a.u[col];
    if (r == 2 * g - 1) return a.dt * a.u[a.ldu + col];
    return 0.f;
}

__device__ __forceinline__ void block_fold(float mx, bool bad, const BurgersArgs& a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad = __any_sync(0xffffffffu, bad);
    if (lane_id() == 0) {
        atomicMax(reinterpret_cast<int*>(a.vmax), __float_as_int(mx));
        if (bad) atomicOr(a.flags, 1);
    }
}

// One CTA per member; substeps fused in shared memory.
__global__ void __launch_bounds__(kBurgersThreads) burgers_fused_kernel(BurgersArgs a) {
    extern __shared__ float sm[];
    const int g = a.g, R = 2 * g, cells = R * g;
    float* cur = sm;
    float* nxt = sm + cells;
    const int64_t col0 = (int64_t)blockIdx.x * g;
    for (int e = threadIdx.x; e < cells; e += blockDim.x) {
        const int r = e / g, j = e - r * g;
        cur[e] = a.x[r * a.ldx + col0 + j];
    }
    __syncthreads();
    float mx = 0.f;
    bool bad = false;
    for (int s = 0; s < a.substeps; ++s) {
        for (int e = threadIdx.x; e < g * g; e += blockDim.x) {
            const int r = e / g, j = e - r * g;
            const int ru = r > 0 ? r - 1 : 0, rd = r < g - 1 ? r + 1 : g - 1;
            const int jl = j > 0 ? j - 1 : 0, jr = j < g - 1 ? j + 1 : g - 1;
            const float vx = cur[r * g + j], vy = cur[(g + r) * g + j];
            mx = fmaxf(mx, fmaxf(fabsf(vx), fabsf(vy)));
            bad |= !(isfinite(vx) && isfinite(vy));
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const float* q = cur + c * g * g;
                const float v = stencil(q[r * g + j], q[ru * g + j], q[rd * g + j], q[r * g + jl],
                                        q[r * g + jr], vx, vy, a);
                nxt[(c * g + r) * g + j] = v + force_at(a, c * g + r, col0 + j);
            }
        }
        __syncthreads();
        float* t = cur;
        cur = nxt;
        nxt = t;
    }
    for (int e = threadIdx.x; e < cells; e += blockDim.x) {
        const int r = e / g, j = e - r * g;
        a.out[r * a.ldo + col0 + j] = cur[e];
    }
    block_fold(mx, bad, a);
}

// One substep from global memory: thread per (member, row < g, col), both channels.
__global__ void __launch_bounds__(256) burgers_global_kernel(BurgersArgs a, const float* __restrict__ src,
                                                             int64_t lds, float* __restrict__ dst,
                                                             int64_t ldd, int add_force) {
    const int g = a.g;
    const int64_t K = (int64_t)a.n_members * g;
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    float mx = 0.f;
    bool bad = false;
    if (k < K) {
        const int j = (int)((uint32_t)k % (uint32_t)g);
        const int64_t kl = j > 0 ? k - 1 : k, kr = j < g - 1 ? k + 1 : k;
        const int ru = r > 0 ? r - 1 : 0, rd = r < g - 1 ? r + 1 : g - 1;
        const float vx = src[r * lds + k], vy = src[(g + r) * lds + k];
        mx = fmaxf(fabsf(vx), fabsf(vy));
        bad = !(isfinite(vx) && isfinite(vy));
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const float* q = src + (int64_t)c * g * lds;
            const float v = stencil(q[r * lds + k], q[ru * lds + k], q[rd * lds + k], q[r * lds + kl],
                                    q[r * lds + kr], vx, vy, a);
            dst[(c * g + r) * ldd + k] = v + (add_force ? force_at(a, c * g + r, k) : 0.f);
        }
    }
    block_fold(mx, bad, a);
}

}  // namespace
}  // namespace enks

extern "C" {

int64_t enks_burgers_ws_bytes(int grid_n, int n_members, int substeps) {
    const int64_t cells = 2LL * grid_n * grid_n;
    if (substeps <= 1 || 2 * cells * (int64_t)sizeof(float) <= enks::kBurgersSmemMax) return 0;
    return cells * (int64_t)n_members * (int64_t)sizeof(float);
}

int enks_burgers_forward(const float* x, int64_t ldx, const float* u, int64_t ldu, int u_rows,
                         float* out, int64_t ldo, int grid_n, int n_members, int substeps,
                         double nu, double dt, double dx, float* vmax, int* flags, void* ws,
                         void* stream) {
    ENKS_REQUIRE(x && out && vmax && flags, "enks_burgers_forward: null pointer");
    ENKS_REQUIRE(grid_n >= 2 && substeps >= 1 && dx > 0 && dt > 0,
                 "enks_burgers_forward: bad grid/solver parameters");
    ENKS_REQUIRE(u_rows == 0 || u_rows == 2 || u_rows == 2 * grid_n,
                 "enks_burgers_forward: force must have 2 (boundary) or 2*grid_n (pointwise) rows");
    ENKS_REQUIRE(u_rows == 0 || u, "enks_burgers_forward: null force");
    ENKS_REQUIRE(out != x, "enks_burgers_forward: out must not alias x");
    if (n_members <= 0) return ENKS_OK;
    enks::BurgersArgs a{x, ldx, u, ldu, out, ldo, grid_n, u_rows, n_members, substeps,
                        (float)nu, (float)dt, (float)(1.0 / dx), (float)(1.0 / (dx * dx)), vmax,
                        flags};
    cudaStream_t st = enks::as_stream(stream);
    const int64_t cells = 2LL * grid_n * grid_n;
    const size_t smem = 2 * cells * sizeof(float);
    if ((int64_t)smem <= enks::kBurgersSmemMax) {
        static size_t configured = 48 * 1024;
        if (smem > configured) {
            cudaError_t e = cudaFuncSetAttribute(enks::burgers_fused_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)enks::kBurgersSmemMax);
            if (e != cudaSuccess) {
                enks::set_error("burgers: smem attribute: %s", cudaGetErrorString(e));
                return ENKS_E_CUDA;
            }
            configured = enks::kBurgersSmemMax;
        }
        enks::burgers_fused_kernel<<<n_members, enks::kBurgersThreads, smem, st>>>(a);
        return enks::check_launch("enks_burgers_forward(fused)");
    }
    ENKS_REQUIRE(grid_n <= 65535, "enks_burgers_forward: grid_n too large");
    ENKS_REQUIRE(substeps == 1 || ws, "enks_burgers_forward: workspace required for substeps");
    const int64_t K = (int64_t)n_members * grid_n;
    const dim3 grid((unsigned)((K + 255) / 256), (unsigned)grid_n);
    // ping-pong between ws and out so the last substep lands in out
    float* bufs[2] = {out, static_cast<float*>(ws)};
    const int64_t lds[2] = {ldo, K};
    const float* src = x;
    int64_t ls = ldx;
    for (int s = 0; s < substeps; ++s) {
        const int dst = (substeps - 1 - s) & 1;  // s == substeps-1 -> out
        enks::burgers_global_kernel<<<grid, 256, 0, st>>>(a, src, ls, bufs[dst], lds[dst], 1);
        int rc = enks::check_launch("enks_burgers_forward(global)");
        if (rc) return rc;
        src = bufs[dst];
        ls = lds[dst];
    }
    return ENKS_OK;
}

}  // extern "C"
