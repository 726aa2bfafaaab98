// tcgen05 3xTF32 engine for the cross-moment contraction (K6/K7):
//     C[M x N] = alpha * A[M x K] B[N x K]^T        (both operands K-major, fp32 in HBM)
// Reference: enks.py:148-153 (_pair_covariance) and 234-236 (Sigma_y, Sigma_xy), here
// applied to the append-only basis of engine.py (P = [A; Yc] Yc^T).
//
// Precision: fp32 operands are split x = hi + lo with hi = rna_tf32(x); the MMA
// accumulates hi*hi + hi*lo + lo*hi in fp32 (TMEM), which matches fp32 FFMA
// accuracy (the dropped lo*lo term is ~2^-22 relative).  1xTF32 misses the 1e-4
// parity bar.
//
// Structure (one 128 x BN output tile and one K range per CTA, 1 CTA / SM):
//   warp 0      TMA producer: A tile (128 x 32 fp32, SWIZZLE_128B) + pre-split B_hi, B_lo
//   warps 4..7  converters: split their A row into hi (in place) / lo (second buffer),
//               fence.proxy.async, arrive; later the epilogue (tcgen05.ld -> HBM)
//   warp 1      MMA issuer: 4 K-steps x 3 tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) per stage
//   warp 2      TMEM allocator
// mbarrier rings: full (TMA bytes), conv (128 converter arrivals), empty (tcgen05.commit).
// Split-K partials go to a workspace and are summed in a fixed order (deterministic).
#include <cuda.h>
#include <stdlib.h>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace enks {
namespace {

constexpr int BM = 128, BK = 32;
constexpr int kThreads = 384;        // 4 control warps + 8 converter/epilogue warps
constexpr int kSmemBudget = 200 * 1024;
constexpr int kChainChunks = 4;      // TMEM accumulation chain = 4 x 32 = 128 K-elements

struct TcParams {
    int64_t M, N, K;
    float alpha;
    float* out;   // split partial base (ws) or C
    int64_t ldo;
    int64_t split_stride;  // elements between split partials (0 if writing C directly)
    int chunks_per_split;
    int total_chunks;
    int stages;
    int products;  // bitmask: 1 = lo*hi, 2 = hi*lo, 4 = hi*hi (debug knob ENKS_TC_PRODUCTS; default 7)
};

template <int BN>
struct Layout {
    static constexpr int kA = BM * BK * 4;     // 16 KB (hi in place)
    static constexpr int kB = BN * BK * 4;     // BN x 128 B
    static constexpr int kStage = 2 * kA + 2 * kB;
    static constexpr int kSlotCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
    static constexpr int kEpiWG = BN > 128 ? 2 : 1;         // warpgroups holding the fp32 sums
    static constexpr int kColsPerWG = BN > 128 ? BN / 2 : BN;
};

// The tensor core accumulates into TMEM with truncation; over long K chains that
// bias reaches ~1e-6 relative (measured: tools/tc_acc_probe.py).  The MMA warp
// therefore restarts a fresh TMEM slot every kChainChunks chunks (two slots,
// ping-pong) and the epilogue warps fold each finished chain into fp32 registers
// with round-to-nearest adds while the other slot fills.
template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    tc_nt_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                 const __grid_constant__ CUtensorMap tmBl, const TcParams p) {
    using L = Layout<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * L::kStage);
    uint64_t* full = bars;
    uint64_t* conv = bars + S;
    uint64_t* empty = bars + 2 * S;
    uint64_t* tfull = bars + 3 * S;       // [2] chain finished in slot
    uint64_t* tempty = bars + 3 * S + 2;  // [2] slot drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int split = blockIdx.y;
    const int c_lo = split * p.chunks_per_split;
    const int c_hi = min(p.total_chunks, c_lo + p.chunks_per_split);
    const int n_chunks = max(0, c_hi - c_lo);
    const int n_groups = (n_chunks + kChainChunks - 1) / kChainChunks;
    constexpr uint32_t kTmemCols = 2 * L::kSlotCols;

    auto stage_a = [&](int s) { return smem + (size_t)s * L::kStage; };
    auto stage_alo = [&](int s) { return smem + (size_t)s * L::kStage + L::kA; };
    auto stage_bh = [&](int s) { return smem + (size_t)s * L::kStage + 2 * L::kA; };
    auto stage_bl = [&](int s) { return smem + (size_t)s * L::kStage + 2 * L::kA + L::kB; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&conv[s], 256);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int q = 0; q < 2; ++q) {
            ptx::mbar_init(&tfull[q], 1);
            ptx::mbar_init(&tempty[q], 4 * L::kEpiWG);
        }
        ptx::fence_barrier_init();
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmBh);
        ptx::tma_prefetch_desc(&tmBl);
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)((i / S) & 1);
                ptx::mbar_wait(&empty[s], ph ^ 1);
                ptx::mbar_arrive_expect_tx(&full[s], L::kA + 2 * L::kB);
                const int kc = (c_lo + i) * BK;
                ptx::tma_load_2d(&tmA, &full[s], stage_a(s), kc, (int32_t)row0);
                ptx::tma_load_2d(&tmBh, &full[s], stage_bh(s), kc, 0);
                ptx::tma_load_2d(&tmBl, &full[s], stage_bl(s), kc, 0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_tf32(BM, BN);
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)((i / S) & 1);
                const int g = i / kChainChunks, slot = g & 1;
                const bool first = (i % kChainChunks) == 0;
                const bool last = (i % kChainChunks) == kChainChunks - 1 || i == n_chunks - 1;
                if (first) {
                    ptx::mbar_wait(&tempty[slot], (uint32_t)(((g >> 1) & 1) ^ 1));
                    ptx::tc_fence_after();
                }
                ptx::mbar_wait(&conv[s], ph);
                ptx::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(slot * L::kSlotCols);
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {
                    const uint64_t ah = ptx::desc_kmajor_sw128(stage_a(s) + 32 * k);
                    const uint64_t al = ptx::desc_kmajor_sw128(stage_alo(s) + 32 * k);
                    const uint64_t bh = ptx::desc_kmajor_sw128(stage_bh(s) + 32 * k);
                    const uint64_t bl = ptx::desc_kmajor_sw128(stage_bl(s) + 32 * k);
                    uint32_t acc = (first && k == 0) ? 0u : 1u;
                    if (p.products & 1) { ptx::mma_tf32_ss(d, al, bh, idesc, acc); acc = 1u; }
                    if (p.products & 2) { ptx::mma_tf32_ss(d, ah, bl, idesc, acc); acc = 1u; }
                    if (p.products & 4) { ptx::mma_tf32_ss(d, ah, bh, idesc, acc); }
                }
                ptx::mma_commit(&empty[s]);
                if (last) ptx::mma_commit(&tfull[slot]);
            }
        }
    } else if (warp >= 4) {
        const int t = threadIdx.x - 128;          // 0..255
        const int crow = t & 127, chalf = t >> 7;  // converter: half a row (64 B) each
        const int wg = (warp - 4) >> 2;            // epilogue warpgroup
        const bool epi = wg < L::kEpiWG;
        const int erow = ((warp & 3) << 5) + lane;  // TMEM lane == tile row
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        float acc[L::kColsPerWG];
#pragma unroll
        for (int j = 0; j < L::kColsPerWG; ++j) acc[j] = 0.f;

        auto drain = [&](int g) {
            const int slot = g & 1;
            ptx::mbar_wait(&tfull[slot], (uint32_t)((g >> 1) & 1));
            ptx::tc_fence_after();
            const uint32_t base = tmem + lane_base + (uint32_t)(slot * L::kSlotCols + wg * L::kColsPerWG);
#pragma unroll
            for (int c0 = 0; c0 < L::kColsPerWG; c0 += 32) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(base + c0, v);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[c0 + j] += __uint_as_float(v[j]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[slot]);
        };

        int drained = 0;
        for (int i = 0; i < n_chunks; ++i) {
            const int s = i % S;
            const uint32_t ph = (uint32_t)((i / S) & 1);
            ptx::mbar_wait(&full[s], ph);
            // elementwise split: any chunk order works; XOR with the row's swizzle phase
            // spreads the 8 threads of each shared-memory phase over all 32 banks.
            float4* a = reinterpret_cast<float4*>(stage_a(s) + crow * 128);
            float4* alo = reinterpret_cast<float4*>(stage_alo(s) + crow * 128);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int qq = (chalf * 4 + q) ^ (crow & 7);
                const float4 v = a[qq];
                float4 h, l;
                h.x = ptx::tf32_round(v.x); l.x = v.x - h.x;
                h.y = ptx::tf32_round(v.y); l.y = v.y - h.y;
                h.z = ptx::tf32_round(v.z); l.z = v.z - h.z;
                h.w = ptx::tf32_round(v.w); l.w = v.w - h.w;
                a[qq] = h;
                alo[qq] = l;
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&conv[s]);
            // fold chain g-1 once chain g has been fully converted (its slot is reused by g+1)
            if (epi && (i % kChainChunks) == kChainChunks - 1) {
                const int g = i / kChainChunks;
                if (g >= 1) drain(g - 1), drained = g;
            }
        }
        if (epi) {
            for (int g = drained; g < n_groups; ++g) drain(g);
            const int64_t r = row0 + erow;
            if (r < p.M) {
                float* orow = p.out + (int64_t)split * p.split_stride + r * p.ldo + wg * L::kColsPerWG;
                const int ncol = (int)min((int64_t)L::kColsPerWG, p.N - (int64_t)wg * L::kColsPerWG);
                if (ncol == L::kColsPerWG && (p.ldo & 3) == 0) {
#pragma unroll
                    for (int j = 0; j < L::kColsPerWG; j += 4)
                        *reinterpret_cast<float4*>(orow + j) =
                            make_float4(p.alpha * acc[j], p.alpha * acc[j + 1], p.alpha * acc[j + 2],
                                        p.alpha * acc[j + 3]);
                } else {
#pragma unroll
                    for (int j = 0; j < L::kColsPerWG; ++j)
                        if (j < ncol) orow[j] = p.alpha * acc[j];
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc(tmem, kTmemCols);
}

__global__ void tf32_split_kernel(const float* __restrict__ src, int64_t ld, int64_t rows,
                                  int64_t cols, float* __restrict__ hi, float* __restrict__ lo) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= rows * cols) return;
    const int64_t r = e / cols, c = e - r * cols;
    const float v = src[r * ld + c];
    const float h = ptx::tf32_round(v);
    hi[e] = h;
    lo[e] = v - h;
}

__global__ void sum_splits_kernel(const float* __restrict__ ws, int split, int64_t M, int64_t N,
                                  float* __restrict__ C, int64_t ldc, const float* __restrict__ C0,
                                  int64_t ldc0, float beta) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    const int64_t r = e / N, c = e - r * N;
    float v = 0.f;
    for (int z = 0; z < split; ++z) v += ws[(int64_t)z * M * N + e];
    if (C0) v += beta * C0[r * ldc0 + c];
    C[r * ldc + c] = v;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld,
              int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int bn_for(int64_t N) { return N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256)); }

template <int BN>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mh, const CUtensorMap& ml, TcParams p,
              int tiles, int split, cudaStream_t st) {
    using L = Layout<BN>;
    int stages = kSmemBudget / L::kStage;
    if (stages > 4) stages = 4;
    if (stages < 2) {
        set_error("tc gemm: stage does not fit shared memory");
        return ENKS_E_UNSUPPORTED;
    }
    p.stages = stages;
    const size_t smem = (size_t)stages * L::kStage + 1024 + 512;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(tc_nt_kernel<BN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            set_error("tc gemm: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = true;
    }
    dim3 grid((unsigned)tiles, (unsigned)split);
    tc_nt_kernel<BN><<<grid, kThreads, smem, st>>>(ma, mh, ml, p);
    return check_launch("enks_gemm(tcgen05)");
}

}  // namespace

int tc_choose_split(int64_t M, int64_t K) {
    const int tiles = (int)((M + BM - 1) / BM);
    const int chunks = (int)((K + BK - 1) / BK);
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 64; ++s) {
        if (chunks / s < 8 && s > 1) break;
        const int units = tiles * s;
        const int waves = (units + kNumSMs - 1) / kNumSMs;
        const double eff = (double)units / (double)(waves * kNumSMs);
        if (eff > best_eff + 0.03) {
            best_eff = eff;
            best = s;
        }
        if (eff > 0.95) break;
    }
    return best;
}

bool tc_gemm_applicable(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
                        int64_t lda, const float* B, int64_t ldb, int64_t tri_rows) {
    if (trans_a || !trans_b || tri_rows > 0) return false;
    if (N < 1 || N > 256 || K < 4 * BK || M < 1) return false;
    if ((lda & 3) || (ldb & 3)) return false;
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return false;
    return encode_fn() != nullptr;
}

// A raw fp32 (M x K, lda); B pre-split (Bh, Bl: N x K, ldb).  Writes C = alpha A B^T (+ beta C0).
int gemm_tc_presplit(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                     const float* Bh, const float* Bl, int64_t ldb, float beta, const float* C0,
                     int64_t ldc0, float* C, int64_t ldc, int split, float* ws, cudaStream_t st) {
    const int BN = bn_for(N);
    CUtensorMap ma, mh, ml;
    if (!make_map(&ma, A, M, K, lda, BM) || !make_map(&mh, Bh, N, K, ldb, BN) ||
        !make_map(&ml, Bl, N, K, ldb, BN)) {
        set_error("tc gemm: cuTensorMapEncodeTiled failed");
        return ENKS_E_UNSUPPORTED;
    }
    const int tiles = (int)((M + BM - 1) / BM);
    const int total_chunks = (int)((K + BK - 1) / BK);
    if (split < 1) split = tc_choose_split(M, K);
    const int cps = (total_chunks + split - 1) / split;
    split = (total_chunks + cps - 1) / cps;
    TcParams p;
    p.M = M; p.N = N; p.K = K;
    p.alpha = alpha;
    p.chunks_per_split = cps;
    {
        const char* e = getenv("ENKS_TC_PRODUCTS");
        p.products = e ? atoi(e) : 7;
    }
    p.total_chunks = total_chunks;
    const bool direct = (split == 1 && C0 == nullptr);
    if (!direct && !ws) {
        set_error("tc gemm: split-K needs workspace");
        return ENKS_E_ARG;
    }
    p.out = direct ? C : ws;
    p.ldo = direct ? ldc : N;
    p.split_stride = direct ? 0 : M * N;
    int rc;
    switch (BN) {
        case 32: rc = launch_tc<32>(ma, mh, ml, p, tiles, split, st); break;
        case 64: rc = launch_tc<64>(ma, mh, ml, p, tiles, split, st); break;
        case 128: rc = launch_tc<128>(ma, mh, ml, p, tiles, split, st); break;
        default: rc = launch_tc<256>(ma, mh, ml, p, tiles, split, st); break;
    }
    if (rc || direct) return rc;
    const int64_t total = M * N;
    sum_splits_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(ws, split, M, N, C, ldc, C0,
                                                                      ldc0, beta);
    return check_launch("enks_gemm(tcgen05 split reduce)");
}

int tf32_split(const float* src, int64_t ld, int64_t rows, int64_t cols, float* hi, float* lo,
               cudaStream_t st) {
    const int64_t total = rows * cols;
    if (total == 0) return ENKS_OK;
    tf32_split_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(src, ld, rows, cols, hi, lo);
    return check_launch("enks_tf32_split");
}

int64_t tc_ws_bytes(int64_t M, int64_t N, int64_t K, int split) {
    if (split < 1) split = tc_choose_split(M, K);
    return ((int64_t)split * M * N + 2 * N * K) * (int64_t)sizeof(float) + 64;
}

int gemm_tc(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
            const float* B, int64_t ldb, float beta, const float* C0, int64_t ldc0,
            const float* bias, int64_t ld_bias, int bias_cols, float* C, int64_t ldc, int split_k,
            void* ws, cudaStream_t st) {
    (void)ld_bias;
    (void)bias_cols;
    if (bias) {
        set_error("tc gemm: bias epilogue not supported");
        return ENKS_E_UNSUPPORTED;
    }
    if (!ws) {
        set_error("tc gemm: needs workspace (enks_gemm_ws_bytes with engine 2)");
        return ENKS_E_ARG;
    }
    // workspace: [B_hi | B_lo | split partials]
    float* bh = static_cast<float*>(ws);
    float* bl = bh + N * K;
    float* part = bl + N * K;
    part = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(part) + 15) & ~uintptr_t(15));
    int rc = tf32_split(B, ldb, N, K, bh, bl, st);
    if (rc) return rc;
    return gemm_tc_presplit(M, N, K, alpha, A, lda, bh, bl, K, beta, C0, ldc0, C, ldc,
                            split_k > 0 ? split_k : 0, part, st);
}

}  // namespace enks

extern "C" {

int64_t enks_tc_gemm_ws_bytes(int64_t M, int64_t N, int64_t K, int split_k) {
    return enks::tc_ws_bytes(M, N, K, split_k);
}

int enks_tf32_split(const float* src, int64_t ld, int64_t rows, int64_t cols, float* hi, float* lo,
                    void* stream) {
    ENKS_REQUIRE(src && hi && lo, "enks_tf32_split: null pointer");
    return enks::tf32_split(src, ld, rows, cols, hi, lo, enks::as_stream(stream));
}

int enks_gemm_nt_tc(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                    const float* Bh, const float* Bl, int64_t ldb, float* C, int64_t ldc,
                    int split_k, void* ws, void* stream) {
    ENKS_REQUIRE(A && Bh && Bl && C, "enks_gemm_nt_tc: null pointer");
    ENKS_REQUIRE(enks::tc_gemm_applicable(0, 1, M, N, K, A, lda, Bh, ldb, 0) &&
                     !(reinterpret_cast<uintptr_t>(Bl) & 15),
                 "enks_gemm_nt_tc: unsupported shape/alignment (N<=256, K>=128, ld%%4==0)");
    if (M == 0 || N == 0) return ENKS_OK;
    return enks::gemm_tc_presplit(M, N, K, alpha, A, lda, Bh, Bl, ldb, 0.f, nullptr, 0, C, ldc,
                                  split_k, static_cast<float*>(ws), enks::as_stream(stream));
}

}  // extern "C"
