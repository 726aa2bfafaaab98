// tcgen05 3xTF32 GEMM engine for the path's contractions:
//   NT  C[M x N] = alpha * A[M x K] B[N x K]^T           (cross moments K6/K7: P = [A; Yc] Yc^T,
//                                                         enks.py:148-153, 234-236)
//   NN  C[M x N] = alpha * A[M x K] B[K x N] + beta C0 + bias[r, c % bias_cols]
//                                                        (member shift / correction / gain
//                                                         products, enks.py:246-247)
// A is fp32 row-major (K-major), split in-kernel; B arrives pre-split as (hi, lo)
// fp32 planes, K-major (NT) or MN-major (NN).
//
// Precision: x = hi + lo with hi = rna_tf32(x); the MMAs accumulate lo*hi + hi*lo + hi*hi,
// matching fp32 FFMA accuracy (the dropped lo*lo term is ~2^-22 relative).  The tensor core
// accumulates into TMEM with truncation; over long K chains that bias reaches ~1e-6 relative
// (tools/tc_acc_probe.py), so the MMA warp restarts a fresh TMEM slot every p.chain
// chunks (two slots, ping-pong) and the epilogue warps fold each finished chain into fp32
// registers with round-to-nearest adds while the other slot fills.
//
// Structure (one 128 x BN output tile and one K range per CTA, 1 CTA / SM, 384 threads):
//   warp 0      TMA producer: A tile (128 x 32 fp32, SWIZZLE_128B) + B_hi, B_lo tiles
//   warp 1      MMA issuer: 4 K-steps x 3 tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) per stage
//   warp 2      TMEM allocator
//   warps 4-11  converters (A -> hi in place / lo, fence.proxy.async), then the epilogue
// mbarrier rings: full (TMA bytes), conv (256 converter arrivals), empty (tcgen05.commit),
// tfull/tempty (TMEM chain slots).  Split-K partials are summed in a fixed order.
#include <cuda.h>
#include <stdlib.h>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace enks {
namespace {

constexpr int BM = 128, BK = 32;  // BK: widest K chunk (128 B rows, SWIZZLE_128B)
constexpr int kThreads = 384;        // 4 control warps + 8 converter/epilogue warps
constexpr int kSmemBudget = 210 * 1024;
constexpr int kChainChunksDefault = 8;  // TMEM accumulation chain (chunks)

struct TcParams {
    int64_t M, N, K;
    float alpha, beta;
    float* out;            // split partial base (ws) or C
    int64_t ldo;
    int64_t split_stride;  // elements between split partials (0 if writing C directly)
    const float* C0;       // direct mode only
    int64_t ldc0;
    const float* bias;     // direct mode only
    int64_t ld_bias;
    int bias_cols;
    int64_t tri_rows, tri_k;  // block-triangular A: row tile r0 starts at k = (r0/tri_rows)*tri_k
    int splits;
    int stages;
    int products;  // bitmask: 1 = lo*hi, 2 = hi*lo, 4 = hi*hi (debug knob ENKS_TC_PRODUCTS)
    uint32_t mn_lbo, mn_sbo;  // MN-major B descriptor strides (debug knob ENKS_TC_MN)
    int debug;                // ENKS_TC_DEBUG: 1 = skip A split math, 2 = skip B loads
    int chain;                // TMEM accumulation chain length in chunks (ENKS_TC_CHAIN)
};

template <int BN, int KB = BK>
struct Layout {
    static constexpr int kRowB = KB * 4;       // bytes per operand row in a stage
    static constexpr int kA = BM * KB * 4;     // A tile (hi in place)
    static constexpr int kB = BN * KB * 4;     // B tile
    static constexpr int kStage = 2 * kA + 2 * kB;
    static constexpr int kSlotCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
    static constexpr int kEpiWG = BN > 128 ? 2 : 1;         // warpgroups holding the fp32 sums
    static constexpr int kColsPerWG = BN > 128 ? BN / 2 : BN;
};

// UMMA descriptor, MN-major SWIZZLE_128B: 32-element (128 B) MN atoms LBO bytes apart,
// 8-row K groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_mnmajor_sw128(const void* smem, uint32_t lbo,
                                                       uint32_t sbo = 1024) {
    const uint64_t addr = ptx::smem_u32(smem);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// UMMA descriptor, K-major SWIZZLE_64B (8-row x 64 B atoms, SBO = 512 B)
__device__ __forceinline__ uint64_t desc_kmajor_sw64(const void* smem) {
    const uint64_t addr = ptx::smem_u32(smem);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;  // SWIZZLE_64B
    return d;
}

template <int KB>
__device__ __forceinline__ uint64_t desc_k(const void* smem) {
    if constexpr (KB == 32) return ptx::desc_kmajor_sw128(smem);
    else return desc_kmajor_sw64(smem);
}

template <int BN, bool BMN, int KB, int CL>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                   const __grid_constant__ CUtensorMap tmBl, const TcParams p) {
    using L = Layout<BN, KB>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // align to 1024 B by offsetting the shared pointer itself (keeps LDS/STS addressing)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * L::kStage);
    uint64_t* full = bars;
    uint64_t* conv = bars + S;
    uint64_t* empty = bars + 2 * S;
    uint64_t* tfull = bars + 3 * S;       // [2] chain finished in slot
    uint64_t* tempty = bars + 3 * S + 2;  // [2] slot drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

    // warp index / TMEM base via a lane-0 shuffle: provably warp-uniform, so the converged MMA
    // warp keeps its descriptors in uniform registers (tc_ptx.cuh, *_elect)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int64_t col0 = (int64_t)blockIdx.y * BN;
    // CL > 1: the CTAs of a cluster (consecutive row tiles, same K range) share the B tile:
    // each loads 1/CL of it and multicasts, and every CTA's MMA commit releases the stage in
    // all of them, so B crosses L2 -> SM once per cluster instead of once per CTA.
    const uint32_t cta_rank = CL > 1 ? ptx::cluster_ctarank() : 0u;
    constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
    const int split = blockIdx.z;
    // K range of this CTA: [kbeg, K) split evenly (in BK chunks) over the splits
    int64_t kbeg = 0;
    if (p.tri_rows > 0) kbeg = (row0 / p.tri_rows) * p.tri_k;
    kbeg = (kbeg / KB) * KB;
    if (kbeg > p.K) kbeg = p.K;
    const int total_chunks = (int)((p.K - kbeg + KB - 1) / KB);
    const int cps = (total_chunks + p.splits - 1) / p.splits;
    const int c_lo = min(total_chunks, split * cps);
    const int c_hi = min(total_chunks, c_lo + cps);
    const int n_chunks = c_hi - c_lo;
    const int n_groups = (n_chunks + p.chain - 1) / p.chain;
    constexpr uint32_t kTmemCols = 2 * L::kSlotCols;

    auto stage_a = [&](int s) { return smem + (size_t)s * L::kStage; };
    auto stage_alo = [&](int s) { return smem + (size_t)s * L::kStage + L::kA; };
    auto stage_bh = [&](int s) { return smem + (size_t)s * L::kStage + 2 * L::kA; };
    auto stage_bl = [&](int s) { return smem + (size_t)s * L::kStage + 2 * L::kA + L::kB; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&conv[s], 256);
            ptx::mbar_init(&empty[s], CL);
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
    if (CL > 1) ptx::cluster_sync();  // peers' barriers initialised before any multicast
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)((i / S) & 1);
                ptx::mbar_wait(&empty[s], ph ^ 1);
                ptx::mbar_arrive_expect_tx(&full[s], (p.debug & 2) ? L::kA : L::kA + 2 * L::kB);
                const int kc = (int)(kbeg + (int64_t)(c_lo + i) * KB);
                ptx::tma_load_2d(&tmA, &full[s], stage_a(s), kc, (int32_t)row0);
                if (p.debug & 2) {
                } else if (!BMN && CL == 1) {
                    ptx::tma_load_2d(&tmBh, &full[s], stage_bh(s), kc, (int32_t)col0);
                    ptx::tma_load_2d(&tmBl, &full[s], stage_bl(s), kc, (int32_t)col0);
                } else if (!BMN) {
                    constexpr int kPiece = BN / CL;  // B rows loaded (and multicast) by this CTA
                    const int off = (int)cta_rank * kPiece * L::kRowB;
                    ptx::tma_load_2d_mc(&tmBh, &full[s], stage_bh(s) + off, kc,
                                        (int32_t)(col0 + cta_rank * kPiece), kMask);
                    ptx::tma_load_2d_mc(&tmBl, &full[s], stage_bl(s) + off, kc,
                                        (int32_t)(col0 + cta_rank * kPiece), kMask);
                } else {
#pragma unroll
                    for (int j = 0; j < BN / 32; ++j) {
                        ptx::tma_load_2d(&tmBh, &full[s], stage_bh(s) + j * 4096,
                                         (int32_t)(col0 + 32 * j), kc);
                        ptx::tma_load_2d(&tmBl, &full[s], stage_bl(s) + j * 4096,
                                         (int32_t)(col0 + 32 * j), kc);
                    }
                }
            }
        }
    } else if (warp == 1) {
        {  // converged: an elected lane issues
            uint32_t idesc = ptx::idesc_tf32(BM, BN);
            if (BMN) idesc |= 1u << 16;  // B MN-major
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % S;
                const uint32_t ph = (uint32_t)((i / S) & 1);
                const int g = i / p.chain, slot = g & 1;
                const bool first = (i % p.chain) == 0;
                const bool last = (i % p.chain) == p.chain - 1 || i == n_chunks - 1;
                if (first) {
                    ptx::mbar_wait(&tempty[slot], (uint32_t)(((g >> 1) & 1) ^ 1));
                    ptx::tc_fence_after();
                }
                ptx::mbar_wait(&conv[s], ph);
                ptx::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(slot * L::kSlotCols);
#pragma unroll
                for (int k = 0; k < KB / 8; ++k) {
                    const uint64_t ah = desc_k<KB>(stage_a(s) + 32 * k);
                    const uint64_t al = desc_k<KB>(stage_alo(s) + 32 * k);
                    uint64_t bh, bl;
                    if (!BMN) {
                        bh = desc_k<KB>(stage_bh(s) + 32 * k);
                        bl = desc_k<KB>(stage_bl(s) + 32 * k);
                    } else {
                        bh = desc_mnmajor_sw128(stage_bh(s) + 1024 * k, p.mn_lbo, p.mn_sbo);
                        bl = desc_mnmajor_sw128(stage_bl(s) + 1024 * k, p.mn_lbo, p.mn_sbo);
                    }
                    uint32_t acc = (first && k == 0) ? 0u : 1u;
                    if (p.products & 1) { ptx::mma_tf32_ss_elect(d, al, bh, idesc, acc); acc = 1u; }
                    if (p.products & 2) { ptx::mma_tf32_ss_elect(d, ah, bl, idesc, acc); acc = 1u; }
                    if (p.products & 4) { ptx::mma_tf32_ss_elect(d, ah, bh, idesc, acc); }
                }
                if (CL > 1) ptx::mma_commit_mc_elect(&empty[s], kMask);
                else ptx::mma_commit_elect(&empty[s]);
                if (last) ptx::mma_commit_elect(&tfull[slot]);
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
            // spreads the threads of each shared-memory phase over all 32 banks.
            constexpr int kChunks = L::kRowB / 16;       // 16-B chunks per row (8 or 4)
            constexpr int kPer = kChunks / 2;            // per converter thread (half a row)
            float4* a = reinterpret_cast<float4*>(stage_a(s) + crow * L::kRowB);
            float4* alo = reinterpret_cast<float4*>(stage_alo(s) + crow * L::kRowB);
            const int phase = KB == 32 ? (crow & 7) : ((crow >> 1) & 3);
#pragma unroll
            for (int q = 0; q < ((p.debug & 1) ? 0 : kPer); ++q) {
                const int qq = (chalf * kPer + q) ^ phase;
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
            if (epi && (i % p.chain) == p.chain - 1) {
                const int g = i / p.chain;
                if (g >= 1) drain(g - 1), drained = g;
            }
        }
        if (epi) {
            for (int g = drained; g < n_groups; ++g) drain(g);
            const int64_t r = row0 + erow;
            const int64_t c_first = col0 + wg * L::kColsPerWG;
            if (r < p.M && c_first < p.N) {
                float* orow = p.out + (int64_t)split * p.split_stride + r * p.ldo + c_first;
                const int ncol = (int)min((int64_t)L::kColsPerWG, p.N - c_first);
                const bool direct = p.split_stride == 0;
                const float* c0row = (direct && p.C0) ? p.C0 + r * p.ldc0 + c_first : nullptr;
                const float* brow = (direct && p.bias) ? p.bias + r * p.ld_bias : nullptr;
                const bool vec = ncol == L::kColsPerWG && ((p.ldo & 3) == 0) &&
                                 ((reinterpret_cast<uintptr_t>(orow) & 15) == 0) &&
                                 (!c0row || (reinterpret_cast<uintptr_t>(c0row) & 15) == 0);
                if (vec) {
#pragma unroll
                    for (int j = 0; j < L::kColsPerWG; j += 4) {
                        float4 v = make_float4(p.alpha * acc[j], p.alpha * acc[j + 1],
                                               p.alpha * acc[j + 2], p.alpha * acc[j + 3]);
                        if (c0row) {
                            const float4 c = *reinterpret_cast<const float4*>(c0row + j);
                            v.x += p.beta * c.x; v.y += p.beta * c.y;
                            v.z += p.beta * c.z; v.w += p.beta * c.w;
                        }
                        if (brow) {
                            v.x += brow[(c_first + j) % p.bias_cols];
                            v.y += brow[(c_first + j + 1) % p.bias_cols];
                            v.z += brow[(c_first + j + 2) % p.bias_cols];
                            v.w += brow[(c_first + j + 3) % p.bias_cols];
                        }
                        *reinterpret_cast<float4*>(orow + j) = v;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < L::kColsPerWG; ++j) {
                        if (j < ncol) {
                            float v = p.alpha * acc[j];
                            if (c0row) v += p.beta * c0row[j];
                            if (brow) v += brow[(c_first + j) % p.bias_cols];
                            orow[j] = v;
                        }
                    }
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (CL > 1) ptx::cluster_sync();  // no CTA exits while peers may still signal it
    if (warp == 2) ptx::tmem_dealloc(tmem, kTmemCols);
}

__global__ void tf32_split_kernel(const float* __restrict__ src, int64_t ld, int64_t rows,
                                  int64_t cols, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t ldo) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= cols) return;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const float v = src[r * ld + c];
        const float h = ptx::tf32_round(v);
        hi[r * ldo + c] = h;
        lo[r * ldo + c] = v - h;
    }
}

// hi/lo split with transpose: src (rows x cols, ld) -> hi, lo (cols x rows, ldo); 32x32 smem tiles
__global__ void tf32_split_t_kernel(const float* __restrict__ src, int64_t ld, int64_t rows,
                                    int64_t cols, float* __restrict__ hi, float* __restrict__ lo,
                                    int64_t ldo) {
    __shared__ float tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int64_t r = r0 + ty + k, c = c0 + tx;
        tile[ty + k][tx] = (r < rows && c < cols) ? src[r * ld + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 8) {
        const int64_t c = c0 + ty + k, r = r0 + tx;  // output row c, column r
        if (c < cols && r < rows) {
            const float v = tile[tx][ty + k];
            const float h = ptx::tf32_round(v);
            hi[c * ldo + r] = h;
            lo[c * ldo + r] = v - h;
        }
    }
}

__global__ void sum_splits_kernel(const float* __restrict__ ws, int split, int64_t M, int64_t N,
                                  float* C, int64_t ldc, const float* C0, int64_t ldc0, float beta,
                                  const float* __restrict__ bias, int64_t ld_bias, int bias_cols) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    const int64_t r = e / N, c = e - r * N;
    float v = 0.f;
    for (int z = 0; z < split; ++z) v += ws[(int64_t)z * M * N + e];
    if (C0) v += beta * C0[r * ldc0 + c];
    if (bias) v += bias[r * ld_bias + (c % bias_cols)];
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

// 2-D fp32 tensor map over a row-major (rows x cols, ld) matrix; box = box_cols x box_rows
bool make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld,
              int box_cols, int box_rows, bool sw64 = false) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    sw64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

constexpr int kBK256 = 16;  // BN = 256: 16-wide K chunks (SWIZZLE_64B) -> 4 pipeline stages

int bn_for(int64_t N) { return N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256)); }

template <int BN, bool BMN, int KB, int CL>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& mh, const CUtensorMap& ml, TcParams p,
              dim3 grid, cudaStream_t st) {
    using L = Layout<BN, KB>;
    int stages = kSmemBudget / L::kStage;
    if (stages > 8) stages = 8;
    if (stages < 2) {
        set_error("tc gemm: stage does not fit shared memory");
        return ENKS_E_UNSUPPORTED;
    }
    p.stages = stages;
    const size_t smem = (size_t)stages * L::kStage + 1024 + 512;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, BMN, KB, CL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            set_error("tc gemm: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = true;
    }
    if (CL == 1) {
        tc_gemm_kernel<BN, BMN, KB, 1><<<grid, kThreads, smem, st>>>(ma, mh, ml, p);
        return check_launch("enks_gemm(tcgen05)");
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, BMN, KB, CL>, ma, mh, ml, p);
    if (e != cudaSuccess) {
        set_error("tc gemm: cluster launch: %s", cudaGetErrorString(e));
        return ENKS_E_CUDA;
    }
    return check_launch("enks_gemm(tcgen05 cluster)");
}

template <bool BMN, int CL>
int dispatch_bn(int BN, const CUtensorMap& ma, const CUtensorMap& mh, const CUtensorMap& ml,
                const TcParams& p, dim3 grid, cudaStream_t st) {
    switch (BN) {
        case 32: return launch_tc<32, BMN, 32, CL>(ma, mh, ml, p, grid, st);
        case 64: return launch_tc<64, BMN, 32, CL>(ma, mh, ml, p, grid, st);
        case 128: return launch_tc<128, BMN, 32, CL>(ma, mh, ml, p, grid, st);
        default: return launch_tc<256, BMN, BMN ? BK : kBK256, CL>(ma, mh, ml, p, grid, st);
    }
}

int choose_split(int tiles, int64_t chunks) {
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

}  // namespace

int tc_choose_split(int64_t M, int64_t K) {
    return choose_split((int)((M + BM - 1) / BM), (K + BK - 1) / BK);
}

bool tc_gemm_applicable(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
                        int64_t lda, const float* B, int64_t ldb, int64_t tri_rows) {
    if (trans_a || !trans_b || tri_rows > 0) return false;
    if (N < 1 || N > 256 || K < 4 * BK || M < 1) return false;
    if ((lda & 3) || (ldb & 3)) return false;
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return false;
    return encode_fn() != nullptr;
}

int gemm_tc_general(bool bmn, int64_t M, int64_t N, int64_t K, float alpha, const float* A,
                    int64_t lda, const float* Bh, const float* Bl, int64_t ldb, float beta,
                    const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias,
                    int bias_cols, float* C, int64_t ldc, int64_t tri_rows, int64_t tri_k,
                    int split, float* ws, cudaStream_t st) {
    if (M == 0 || N == 0) return ENKS_OK;
    const int bn_cap = env_knob("ENKS_TC_BN", 256);
    const int BN = bn_for(N < bn_cap ? N : bn_cap);
    CUtensorMap ma, mh, ml;
    const int kb = (BN == 256 && !bmn) ? kBK256 : BK;
    const bool sw64 = kb == 16;
    const int m_tiles0 = (int)((M + BM - 1) / BM);
    // cluster the row tiles sharing B (multicast) when there are several and no triangular skip
    const int want_cl = env_knob("ENKS_TC_CLUSTER", 1);
    const int cl = (!bmn && tri_rows == 0 && want_cl == 4 && m_tiles0 >= 4) ? 4
                 : ((!bmn && tri_rows == 0 && want_cl >= 2 && m_tiles0 >= 2) ? 2 : 1);
    bool ok = make_map(&ma, A, M, K, lda, kb, BM, sw64);
    if (!bmn) {
        ok = ok && make_map(&mh, Bh, N, K, ldb, kb, BN / cl, sw64) &&
             make_map(&ml, Bl, N, K, ldb, kb, BN / cl, sw64);
    } else {
        ok = ok && make_map(&mh, Bh, K, N, ldb, 32, BK) && make_map(&ml, Bl, K, N, ldb, 32, BK);
    }
    if (!ok) {
        set_error("tc gemm: cuTensorMapEncodeTiled failed (alignment / ld %% 4?)");
        return ENKS_E_UNSUPPORTED;
    }
    const int m_tiles = (m_tiles0 + cl - 1) / cl * cl;  // whole clusters (extra tiles idle)
    const int n_tiles = (int)((N + BN - 1) / BN);
    if (split < 1) split = choose_split(m_tiles * n_tiles, (K + kb - 1) / kb);
    TcParams p;
    p.M = M; p.N = N; p.K = K;
    p.alpha = alpha; p.beta = beta;
    p.tri_rows = tri_rows; p.tri_k = tri_k;
    p.splits = split;
    {
        p.products = debug_knob("ENKS_TC_PRODUCTS", 7);  // product mask: debug builds only
        const int mode = debug_knob("ENKS_TC_MN", 0);       // descriptor LBO/SBO probe: debug only
        p.mn_lbo = mode == 1 ? 1024 : (mode == 2 ? 4096 : (mode == 3 ? 1024 : 4096));
        p.mn_sbo = mode == 1 ? 4096 : (mode == 2 ? 4096 : (mode == 3 ? 1024 : 1024));
        p.debug = debug_knob("ENKS_TC_DEBUG", 0);
        p.chain = env_knob("ENKS_TC_CHAIN", kChainChunksDefault);
        if (p.chain < 1) p.chain = 1;
    }
    const bool direct = (split == 1);
    if (!direct && !ws) {
        set_error("tc gemm: split-K needs workspace");
        return ENKS_E_ARG;
    }
    p.out = direct ? C : ws;
    p.ldo = direct ? ldc : N;
    p.split_stride = direct ? 0 : M * N;
    p.C0 = direct ? C0 : nullptr;
    p.ldc0 = ldc0;
    p.bias = direct ? bias : nullptr;
    p.ld_bias = ld_bias;
    p.bias_cols = bias_cols > 0 ? bias_cols : 1;
    dim3 grid((unsigned)m_tiles, (unsigned)n_tiles, (unsigned)split);
    int rc = bmn ? dispatch_bn<true, 1>(BN, ma, mh, ml, p, grid, st)
         : (cl == 4 ? dispatch_bn<false, 4>(BN, ma, mh, ml, p, grid, st)
                    : (cl == 2 ? dispatch_bn<false, 2>(BN, ma, mh, ml, p, grid, st)
                               : dispatch_bn<false, 1>(BN, ma, mh, ml, p, grid, st)));
    if (rc || direct) return rc;
    const int64_t total = M * N;
    sum_splits_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        ws, split, M, N, C, ldc, C0, ldc0, beta, bias, ld_bias, bias_cols > 0 ? bias_cols : 1);
    return check_launch("enks_gemm(tcgen05 split reduce)");
}

int gemm_tc_presplit(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                     const float* Bh, const float* Bl, int64_t ldb, float beta, const float* C0,
                     int64_t ldc0, float* C, int64_t ldc, int split, float* ws, cudaStream_t st) {
    return gemm_tc_general(false, M, N, K, alpha, A, lda, Bh, Bl, ldb, beta, C0, ldc0, nullptr, 0,
                           1, C, ldc, 0, 0, split, ws, st);
}

int tf32_split(const float* src, int64_t ld, int64_t rows, int64_t cols, float* hi, float* lo,
               int64_t ldo, cudaStream_t st) {
    const int64_t total = rows * cols;
    if (total == 0) return ENKS_OK;
    tf32_split_kernel<<<dim3((unsigned)((cols + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535)), 256, 0, st>>>(
        src, ld, rows, cols, hi, lo, ldo);
    return check_launch("enks_tf32_split");
}

int tf32_split_t(const float* src, int64_t ld, int64_t rows, int64_t cols, float* hi, float* lo,
                 int64_t ldo, cudaStream_t st) {
    if (rows == 0 || cols == 0) return ENKS_OK;
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    tf32_split_t_kernel<<<grid, 256, 0, st>>>(src, ld, rows, cols, hi, lo, ldo);
    return check_launch("enks_tf32_split(transpose)");
}

int64_t tc_ws_bytes(int64_t M, int64_t N, int64_t K, int split) {
    if (split < 1) split = choose_split((int)((M + BM - 1) / BM) * (int)((N + 255) / 256),
                                       (K + BK - 1) / BK);
    return ((int64_t)split * M * N + 2 * N * K) * (int64_t)sizeof(float) + 64;
}

int gemm_tc(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
            const float* B, int64_t ldb, float beta, const float* C0, int64_t ldc0,
            const float* bias, int64_t ld_bias, int bias_cols, float* C, int64_t ldc, int split_k,
            void* ws, cudaStream_t st) {
    if (!ws) {
        set_error("tc gemm: needs workspace (enks_tc_gemm_ws_bytes with engine 2)");
        return ENKS_E_ARG;
    }
    // workspace: [B_hi | B_lo | split partials]
    float* bh = static_cast<float*>(ws);
    float* bl = bh + N * K;
    float* part = bl + N * K;
    part = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(part) + 15) & ~uintptr_t(15));
    int rc = tf32_split(B, ldb, N, K, bh, bl, K, st);
    if (rc) return rc;
    return gemm_tc_general(false, M, N, K, alpha, A, lda, bh, bl, K, beta, C0, ldc0, bias,
                           ld_bias, bias_cols, C, ldc, 0, 0, split_k > 0 ? split_k : 0, part, st);
}

}  // namespace enks

extern "C" {

int64_t enks_tc_gemm_ws_bytes(int64_t M, int64_t N, int64_t K, int split_k) {
    return enks::tc_ws_bytes(M, N, K, split_k);
}

int enks_tf32_split(const float* src, int64_t ld, int64_t rows, int64_t cols, float* hi, float* lo,
                    int transpose, void* stream) {
    ENKS_REQUIRE(src && hi && lo, "enks_tf32_split: null pointer");
    return transpose ? enks::tf32_split_t(src, ld, rows, cols, hi, lo, rows, enks::as_stream(stream))
                     : enks::tf32_split(src, ld, rows, cols, hi, lo, cols, enks::as_stream(stream));
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

int enks_gemm_tc(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                 const float* Bh, const float* Bl, int64_t ldb, int b_mn_major, float beta,
                 const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias, int bias_cols,
                 float* C, int64_t ldc, int64_t tri_rows, int64_t tri_k, int split_k, void* ws,
                 void* stream) {
    ENKS_REQUIRE(A && Bh && Bl && C, "enks_gemm_tc: null pointer");
    ENKS_REQUIRE(K >= 1 && (lda & 3) == 0 && (ldb & 3) == 0 &&
                     !(reinterpret_cast<uintptr_t>(A) & 15) &&
                     !(reinterpret_cast<uintptr_t>(Bh) & 15) &&
                     !(reinterpret_cast<uintptr_t>(Bl) & 15),
                 "enks_gemm_tc: operands need 16-B aligned rows (ld %% 4 == 0)");
    ENKS_REQUIRE(b_mn_major || N <= 1 << 30, "enks_gemm_tc: bad N");
    if (M == 0 || N == 0) return ENKS_OK;
    return enks::gemm_tc_general(b_mn_major != 0, M, N, K, alpha, A, lda, Bh, Bl, ldb, beta, C0, ldc0, bias,
                                 ld_bias, bias_cols, C, ldc, tri_rows, tri_k, split_k,
                                 static_cast<float*>(ws), enks::as_stream(stream));
}

}  // extern "C"
