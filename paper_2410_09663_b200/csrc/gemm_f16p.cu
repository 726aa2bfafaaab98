// Cross moments (K6/K7) on tcgen05 kind::f16 with fp16-pair operands.
//
// Reference: enks.py:148-153 (_pair_covariance), 234-236 (Sigma_y, Sigma_xy), applied to
// the append-only basis of engine.py: P = [A; Yc] Yc_tau^T over K = N*m.
//
// Storage: every basis row x (fp32, K long) is kept as two fp16 planes with a per-row
// power-of-two scale s = 2^e chosen so max|x| s lies in [2^13, 2^14):
//     h = fp16(x s),  l = fp16(x s - h)          (x s = h + l to ~2^-22 relative)
// so a basis element costs 4 B (like fp32) and feeds the tensor core directly: no
// in-kernel split.  The product uses three kind::f16 MMAs per K=16 step,
//     (h_a + l_a)(h_b + l_b) ~ l_a h_b + h_a l_b + h_a h_b     (dropped l_a l_b ~ 2^-22),
// products of 11-bit significands are exact in the fp32 accumulator; the result is
// unscaled in the epilogue by 1/(s_a s_b) (exact, powers of two).  Accuracy therefore
// matches 3xTF32 while moving half the bytes per K element and running at the f16 rate.
// As in gemm_tc.cu, TMEM accumulation chains are restarted every `chain` chunks and
// folded into fp32 registers with round-to-nearest adds (the tensor core truncates).
//
// Structure (one 128 x BN tile and one K range per CTA, 384 threads):
//   warp 0: TMA producer (A_h, A_l, B_h, B_l tiles, SWIZZLE_64B, 32 fp16 = 64 B rows)
//   warp 1: MMA issuer (2 K-steps x 3 MMAs per stage), warp 2: TMEM allocator,
//   warps 4-11: epilogue (two warpgroups x 128 columns of fp32 running sums).
#include <cuda.h>
#include <cuda_fp16.h>
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace enks {
namespace {

constexpr int BM = 128;
constexpr int KC = 32;               // fp16 elements per chunk row (64 B, SWIZZLE_64B)
// TMEM accumulation chain length (chunks of KC): the tensor core truncates as it accumulates, so
// a chain of c chunks carries a one-sided relative bias of about c * (KC / 16) * 3 * 2^-25 on a
// sum of positive terms (Gram / Sigma_y diagonal): 1.4e-6 at 8 chunks, 2.9e-6 at 16.  Chains are
// folded in fp32 registers with round-to-nearest adds.  tests/test_gpu_kernels.py pins the bias
// at K = 131072 (C3's contraction depth).
constexpr int kF16pChainDefault = 16;
constexpr int kThreads = 384;
constexpr int kSmemBudget = 210 * 1024;
// MN-major (shift) instance: epilogue staging, 32 rows x 32 columns (+1 pad) per epilogue warp
constexpr int kStgFloats = 32 * 33;
constexpr int kStgBytes = 8 * kStgFloats * 4;  // 33 KB
constexpr int kMnStages = 4;                   // K = p <= a few hundred: a short ring suffices

template <int BN>
struct L16 {
    static constexpr int kA = BM * KC * 2;   // 8 KB per plane
    static constexpr int kB = BN * KC * 2;   // BN x 64 B per plane
    static constexpr int kStage = 2 * kA + 2 * kB;
    static constexpr int kSlotCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
    static constexpr int kEpiWG = BN > 128 ? 2 : 1;
    static constexpr int kColsPerWG = BN > 128 ? BN / 2 : BN;
};

struct P16 {
    int64_t M, N, K;
    float alpha;
    const float* inv_sa;  // per A row
    const float* inv_sb;  // per B row
    float* out;
    int64_t ldo;
    int64_t split_stride;
    int splits;
    int stages;
    int chain;
    int products;  // 3: lh + hl + hh;  2: hl + hh (A's low plane not read)
    int b_mn;      // pair kernel: B given MN-major ([K][N], N contiguous), no per-column scale
    // fused epilogue terms (split == 1 only): + beta * C0[r, c] + bias[r, c % bias_cols]
    float beta;
    const float* c0;
    int64_t ldc0;
    const float* bias;
    int64_t ld_bias;
    int bias_cols;
};

// epilogue of one thread: row r, columns c_first .. c_first + ncol (ncol <= NC)
template <int NC>
__device__ __forceinline__ void f16p_store_row(const P16& p, int split, int64_t r, int64_t c_first,
                                               int ncol, const float (&acc)[NC]) {
    const float sa = p.alpha * p.inv_sa[r];
    float* orow = p.out + (int64_t)split * p.split_stride + r * p.ldo + c_first;
    if (!p.c0 && !p.bias) {
        if (ncol == NC && (((uintptr_t)orow) & 15) == 0) {
            // the column scales of a batch are loaded before its stores (out may alias inv_sb as
            // far as the compiler knows: loads after a store would each wait a full latency)
            constexpr int kSB = 16;
#pragma unroll
            for (int j0 = 0; j0 < NC; j0 += kSB) {
                float sv[kSB];
#pragma unroll
                for (int q = 0; q < kSB; ++q)
                    sv[q] = j0 + q < NC ? p.inv_sb[c_first + j0 + q] : 0.f;
#pragma unroll
                for (int j = j0; j < j0 + kSB && j < NC; j += 4)
                    *reinterpret_cast<float4*>(orow + j) =
                        make_float4(acc[j] * sa * sv[j - j0], acc[j + 1] * sa * sv[j - j0 + 1],
                                    acc[j + 2] * sa * sv[j - j0 + 2], acc[j + 3] * sa * sv[j - j0 + 3]);
            }
            return;
        }
#pragma unroll
        for (int j = 0; j < NC; ++j)
            if (j < ncol) orow[j] = acc[j] * sa * p.inv_sb[c_first + j];
        return;
    }
    const float* crow = p.c0 ? p.c0 + r * p.ldc0 + c_first : nullptr;
    const float* brow = p.bias ? p.bias + r * p.ld_bias : nullptr;
    const bool vec = ncol == NC && (((uintptr_t)orow | (uintptr_t)(crow ? crow : orow)) & 15) == 0 &&
                     (!brow || ((c_first % p.bias_cols) + NC <= p.bias_cols &&
                                (((uintptr_t)(brow + c_first % p.bias_cols)) & 15) == 0));
    if (vec) {  // float4 loads / stores: NC consecutive columns per thread
        const float* bb = brow ? brow + c_first % p.bias_cols : nullptr;
        // C0 / bias in batches of kVB float4 loaded before any store of the batch: out and C0
        // may alias as far as the compiler knows, so loads interleaved with stores would each
        // wait a full memory latency (the newest-slice shift, 256 columns of C0 per row)
        constexpr int kVB = 4;
#pragma unroll
        for (int j0 = 0; j0 < NC; j0 += 4 * kVB) {
            float4 cv[kVB], bv[kVB], sv[kVB];
#pragma unroll
            for (int q = 0; q < kVB; ++q) {
                const int j = j0 + 4 * q;
                sv[q] = j < NC ? make_float4(p.inv_sb[c_first + j], p.inv_sb[c_first + j + 1],
                                             p.inv_sb[c_first + j + 2], p.inv_sb[c_first + j + 3])
                               : make_float4(0.f, 0.f, 0.f, 0.f);
                cv[q] = crow && j < NC ? __ldg(reinterpret_cast<const float4*>(crow + j))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                bv[q] = bb && j < NC ? __ldg(reinterpret_cast<const float4*>(bb + j))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int q = 0; q < kVB; ++q) {
                const int j = j0 + 4 * q;
                if (j >= NC) break;
                float4 o;
                o.x = acc[j] * sa * sv[q].x;
                o.y = acc[j + 1] * sa * sv[q].y;
                o.z = acc[j + 2] * sa * sv[q].z;
                o.w = acc[j + 3] * sa * sv[q].w;
                if (crow) {
                    const float4 c = cv[q];
                    o.x += p.beta * c.x; o.y += p.beta * c.y; o.z += p.beta * c.z; o.w += p.beta * c.w;
                }
                if (bb) {
                    const float4 b = bv[q];
                    o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
                }
                *reinterpret_cast<float4*>(orow + j) = o;
            }
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        if (j < ncol) {
            float v = acc[j] * sa * p.inv_sb[c_first + j];
            if (crow) v += p.beta * crow[j];
            if (brow) v += brow[(c_first + j) % p.bias_cols];
            orow[j] = v;
        }
    }
}

__device__ __forceinline__ uint64_t desc_sw64(const void* smem) {
    const uint64_t addr = ptx::smem_u32(smem);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;  // SWIZZLE_64B
    return d;
}

// MN-major SWIZZLE_64B operand (fp16): atoms of 32 MN elements (64 B) x 8 K rows; the TMA boxes
// are 32 MN x KC K (2 KB) side by side along MN (LBO = 2048 B), 8-row K groups 512 B apart (SBO)
__device__ __forceinline__ uint64_t desc_mn_sw64(const void* smem) {
    const uint64_t addr = ptx::smem_u32(smem);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)(2048 >> 4) << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;  // SWIZZLE_64B
    return d;
}

constexpr uint32_t idesc_f16(int M, int N) {
    // D f32 (bits 4-5 = 1), A/B fp16 (format 0), both K-major, N>>3 @17, M>>4 @24
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    f16p_gemm_kernel(const __grid_constant__ CUtensorMap tAh, const __grid_constant__ CUtensorMap tAl,
                     const __grid_constant__ CUtensorMap tBh, const __grid_constant__ CUtensorMap tBl,
                     const P16 p) {
    using L = L16<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * L::kStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + S;
    uint64_t* tfull = bars + 2 * S;
    uint64_t* tempty = bars + 2 * S + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    const int64_t col0 = (int64_t)blockIdx.y * BN;
    const int split = blockIdx.z;
    const int total_chunks = (int)((p.K + KC - 1) / KC);
    const int cps = (total_chunks + p.splits - 1) / p.splits;
    const int c_lo = min(total_chunks, split * cps);
    const int n_chunks = min(total_chunks, c_lo + cps) - c_lo;
    const int chain = p.chain;
    const int n_groups = (n_chunks + chain - 1) / chain;
    constexpr uint32_t kTmemCols = 2 * L::kSlotCols;

    auto ah = [&](int s) { return smem + (size_t)s * L::kStage; };
    auto al = [&](int s) { return smem + (size_t)s * L::kStage + L::kA; };
    auto bh = [&](int s) { return smem + (size_t)s * L::kStage + 2 * L::kA; };
    auto bl = [&](int s) { return smem + (size_t)s * L::kStage + 2 * L::kA + L::kB; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int q = 0; q < 2; ++q) {
            ptx::mbar_init(&tfull[q], 1);
            ptx::mbar_init(&tempty[q], 4 * L::kEpiWG);
        }
        ptx::fence_barrier_init();
        ptx::tma_prefetch_desc(&tAh);
        ptx::tma_prefetch_desc(&tAl);
        ptx::tma_prefetch_desc(&tBh);
        ptx::tma_prefetch_desc(&tBl);
    }
    if (warp == 2) ptx::tmem_alloc(tmem_slot, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % S;
                ptx::mbar_wait(&empty[s], (uint32_t)(((i / S) & 1) ^ 1));
                ptx::mbar_arrive_expect_tx(&full[s], (p.products == 3 ? 2 : 1) * L::kA + 2 * L::kB);
                const int kc = (c_lo + i) * KC;
                ptx::tma_load_2d(&tAh, &full[s], ah(s), kc, (int32_t)row0);
                if (p.products == 3) ptx::tma_load_2d(&tAl, &full[s], al(s), kc, (int32_t)row0);
                ptx::tma_load_2d(&tBh, &full[s], bh(s), kc, (int32_t)col0);
                ptx::tma_load_2d(&tBl, &full[s], bl(s), kc, (int32_t)col0);
            }
        }
    } else if (warp == 1) {
        {  // converged: an elected lane issues (uniform-register descriptors)
            constexpr uint32_t idesc = idesc_f16(BM, BN);
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % S;
                const int g = i / chain, slot = g & 1;
                const bool first = (i % chain) == 0;
                const bool last = (i % chain) == chain - 1 || i == n_chunks - 1;
                if (first) {
                    ptx::mbar_wait(&tempty[slot], (uint32_t)(((g >> 1) & 1) ^ 1));
                    ptx::tc_fence_after();
                }
                ptx::mbar_wait(&full[s], (uint32_t)((i / S) & 1));
                ptx::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(slot * L::kSlotCols);
#pragma unroll
                for (int k = 0; k < KC / 16; ++k) {
                    const uint64_t dah = desc_sw64(ah(s) + 32 * k), dal = desc_sw64(al(s) + 32 * k);
                    const uint64_t dbh = desc_sw64(bh(s) + 32 * k), dbl = desc_sw64(bl(s) + 32 * k);
                    if (p.products == 3) {
                        ptx::mma_f16_ss_elect(d, dal, dbh, idesc, (first && k == 0) ? 0u : 1u);
                        ptx::mma_f16_ss_elect(d, dah, dbl, idesc, 1u);
                    } else {
                        ptx::mma_f16_ss_elect(d, dah, dbl, idesc, (first && k == 0) ? 0u : 1u);
                    }
                    ptx::mma_f16_ss_elect(d, dah, dbh, idesc, 1u);
                }
                ptx::mma_commit_elect(&empty[s]);
                if (last) ptx::mma_commit_elect(&tfull[slot]);
            }
        }
    } else if (warp >= 4) {
        const int wg = (warp - 4) >> 2;
        if (wg < L::kEpiWG) {
            const int erow = ((warp & 3) << 5) + lane;
            const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
            float acc[L::kColsPerWG];
#pragma unroll
            for (int j = 0; j < L::kColsPerWG; ++j) acc[j] = 0.f;
            for (int g = 0; g < n_groups; ++g) {
                const int slot = g & 1;
                ptx::mbar_wait(&tfull[slot], (uint32_t)((g >> 1) & 1));
                ptx::tc_fence_after();
                const uint32_t base =
                    tmem + lane_base + (uint32_t)(slot * L::kSlotCols + wg * L::kColsPerWG);
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
            }
            const int64_t r = row0 + erow;
            const int64_t c_first = col0 + wg * L::kColsPerWG;
            if (r < p.M && c_first < p.N)
                f16p_store_row(p, split, r, c_first, (int)min((int64_t)L::kColsPerWG, p.N - c_first),
                               acc);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc(tmem, kTmemCols);
}


// ---------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2) for N in (128, 256]: a cluster of two CTAs computes a
// 256 x 256 tile with one tcgen05.mma.cta_group::2 per product.  Each CTA stages its own
// 128 A rows and HALF of the B rows (128), so per unit of MMA work every SM moves and reads
// 2/3 of the shared-memory bytes of the single-CTA 128 x 256 kernel (whose three products
// per K step re-read the full B tile from smem and were shared-memory-bandwidth bound).
// The leader CTA (rank 0) issues the MMAs; its full[] barriers count both CTAs' TMA bytes;
// MMA completion is multicast to both CTAs' empty[] / tfull[] barriers; each CTA drains
// its own TMEM (its 128 rows x 256 columns) and arrives on the leader's tempty[].
struct LP {
    static constexpr int kA = BM * KC * 2;       // 8 KB per plane (128 rows)
    static constexpr int kB = 128 * KC * 2;      // 8 KB per plane (this CTA's 128 B rows)
    static constexpr int kStage = 2 * kA + 2 * kB;
    static constexpr int kCols = 256;            // accumulator columns per slot
};

__device__ __forceinline__ void mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// the same issued by an elected lane of a converged warp (operands in uniform registers)
__device__ __forceinline__ void mma_f16_pair_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                                   uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
#ifndef ENKS_F16P_CONV
#define ENKS_F16P_CONV 1
#endif
constexpr bool kConvPair = ENKS_F16P_CONV;

template <bool BMN>  // B MN-major (p.b_mn): a separate instance, the K-major one is unchanged
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    f16p_gemm_pair_kernel(const __grid_constant__ CUtensorMap tAh,
                          const __grid_constant__ CUtensorMap tAl,
                          const __grid_constant__ CUtensorMap tBh,
                          const __grid_constant__ CUtensorMap tBl, const P16 p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int S = p.stages;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * LP::kStage);
    uint64_t* full = bars;            // leader's are used
    uint64_t* empty = bars + S;       // both
    uint64_t* tfull = bars + 2 * S;   // both
    uint64_t* tempty = bars + 2 * S + 2;  // leader's are used
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 4);

    const uint32_t rank = ptx::cluster_ctarank();
    // warp index / TMEM base via a lane-0 shuffle: provably warp-uniform, so the converged MMA
    // warp keeps its descriptors in uniform registers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int64_t row0 = (int64_t)blockIdx.x * BM;
    // persistent over 256-column tiles (blockIdx.y, + gridDim.y, ...): the next tile's loads and
    // MMAs overlap this tile's epilogue (double-buffered TMEM slots continue across tiles)
    const int64_t n_tiles = (p.N + 255) / 256;
    const int split = blockIdx.z;
    const int total_chunks = (int)((p.K + KC - 1) / KC);
    const int cps = (total_chunks + p.splits - 1) / p.splits;
    const int c_lo = min(total_chunks, split * cps);
    const int n_chunks = min(total_chunks, c_lo + cps) - c_lo;
    const int chain = p.chain;
    const int n_groups = (n_chunks + chain - 1) / chain;
    constexpr uint32_t kTmemCols = 2 * LP::kCols;

    auto ah = [&](int s) { return smem + (size_t)s * LP::kStage; };
    auto al = [&](int s) { return smem + (size_t)s * LP::kStage + LP::kA; };
    auto bh = [&](int s) { return smem + (size_t)s * LP::kStage + 2 * LP::kA; };
    auto bl = [&](int s) { return smem + (size_t)s * LP::kStage + 2 * LP::kA + LP::kB; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int q = 0; q < 2; ++q) {
            ptx::mbar_init(&tfull[q], 1);
            ptx::mbar_init(&tempty[q], 2 * 8);  // 8 epilogue warps in each CTA of the pair
        }
        ptx::fence_barrier_init();
        ptx::tma_prefetch_desc(&tAh);
        ptx::tma_prefetch_desc(&tAl);
        ptx::tma_prefetch_desc(&tBh);
        ptx::tma_prefetch_desc(&tBl);
    }
    if (warp == 2) ptx::tmem_alloc_pair(tmem_slot, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

    if (warp == 0) {
        if (lane == 0) {
          int ig = 0;  // chunk counter across tiles (stage ring position)
          for (int64_t nt = blockIdx.y; nt < n_tiles; nt += gridDim.y) {
            const int32_t brow = (int32_t)(nt * 256 + rank * 128);
            for (int i = 0; i < n_chunks; ++i, ++ig) {
                const int s = ig % S;
                ptx::mbar_wait_bounded(&empty[s], (uint32_t)(((ig / S) & 1) ^ 1));
                if (rank == 0)
                    ptx::mbar_arrive_expect_tx(&full[s], 2 * (p.products == 3 ? LP::kStage
                                                                             : LP::kStage - LP::kA));
                const int kc = (c_lo + i) * KC;
                ptx::tma_load_2d_pair(&tAh, &full[s], ah(s), kc, (int32_t)row0);
                if (p.products == 3) ptx::tma_load_2d_pair(&tAl, &full[s], al(s), kc, (int32_t)row0);
                if constexpr (BMN) {  // this CTA's 128 columns as four 32-column MN-major boxes
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        ptx::tma_load_2d_pair(&tBh, &full[s], bh(s) + q * 2048, brow + 32 * q, kc);
                        ptx::tma_load_2d_pair(&tBl, &full[s], bl(s) + q * 2048, brow + 32 * q, kc);
                    }
                } else {
                    ptx::tma_load_2d_pair(&tBh, &full[s], bh(s), kc, brow);
                    ptx::tma_load_2d_pair(&tBl, &full[s], bl(s), kc, brow);
                }
            }
          }
        }
    } else if (warp == 1) {
        if ((kConvPair || lane == 0) && rank == 0) {
            constexpr uint32_t idesc = idesc_f16(2 * BM, 256) | (BMN ? (1u << 16) : 0u);  // B major
            auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
                if constexpr (kConvPair) mma_f16_pair_elect(d, a, b, idesc, acc);
                else mma_f16_pair(d, a, b, idesc, acc);
            };
            auto commit = [&](uint64_t* bar) {
                if constexpr (kConvPair) ptx::mma_commit_pair_elect(bar, 0x3);
                else ptx::mma_commit_pair(bar, 0x3);
            };
            int ig = 0, gbase = 0;  // chunk / chain-group counters across tiles
            for (int64_t nt = blockIdx.y; nt < n_tiles; nt += gridDim.y, gbase += n_groups) {
            for (int i = 0; i < n_chunks; ++i, ++ig) {
                const int s = ig % S;
                const int g = gbase + i / chain, slot = g & 1;
                const bool first = (i % chain) == 0;
                const bool last = (i % chain) == chain - 1 || i == n_chunks - 1;
                if (first) {
                    ptx::mbar_wait_bounded(&tempty[slot], (uint32_t)(((g >> 1) & 1) ^ 1));
                    ptx::tc_fence_after();
                }
                ptx::mbar_wait_bounded(&full[s], (uint32_t)((ig / S) & 1));
                ptx::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(slot * LP::kCols);
#pragma unroll
                for (int k = 0; k < KC / 16; ++k) {
                    const uint64_t dah = desc_sw64(ah(s) + 32 * k), dal = desc_sw64(al(s) + 32 * k);
                    // K-major: the K = 16 step is 32 B along the row; MN-major: 16 K rows (1 KB)
                    const uint64_t dbh = BMN ? desc_mn_sw64(bh(s) + 1024 * k)
                                             : desc_sw64(bh(s) + 32 * k);
                    const uint64_t dbl = BMN ? desc_mn_sw64(bl(s) + 1024 * k)
                                             : desc_sw64(bl(s) + 32 * k);
                    if (p.products == 3) {
                        mma(d, dal, dbh, (first && k == 0) ? 0u : 1u);
                        mma(d, dah, dbl, 1u);
                    } else {
                        mma(d, dah, dbl, (first && k == 0) ? 0u : 1u);
                    }
                    mma(d, dah, dbh, 1u);
                }
                commit(&empty[s]);
                if (last) commit(&tfull[slot]);
            }
            }
        }
    } else if (warp >= 4) {
        const int wg = (warp - 4) >> 2;
        constexpr int kCols = 128;  // per warpgroup
        const int erow = ((warp & 3) << 5) + lane;
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        int gbase = 0;
        for (int64_t nt = blockIdx.y; nt < n_tiles; nt += gridDim.y, gbase += n_groups) {
        const int64_t col0 = nt * 256;
        float acc[kCols];
#pragma unroll
        for (int j = 0; j < kCols; ++j) acc[j] = 0.f;
        for (int gl = 0; gl < n_groups; ++gl) {
            const int g = gbase + gl;
            const int slot = g & 1;
            ptx::mbar_wait_bounded(&tfull[slot], (uint32_t)((g >> 1) & 1));
            ptx::tc_fence_after();
            const uint32_t base = tmem + lane_base + (uint32_t)(slot * LP::kCols + wg * kCols);
#pragma unroll
            for (int c0 = 0; c0 < kCols; c0 += 32) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(base + c0, v);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[c0 + j] += __uint_as_float(v[j]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(&tempty[slot], 0);
        }
        const int64_t r = row0 + erow;
        const int64_t c_first = col0 + (int64_t)wg * kCols;
        if constexpr (BMN) {
            // wide row-major output (the newest-slice shift, N = N_members m): stage 32 x 32
            // blocks through shared memory so every store / C0 / bias access is a 512 B row run
            // of 4 rows per instruction instead of 32 rows x 16 B
            const int64_t wr0 = row0 + ((warp & 3) << 5);
            float* po = p.out + (int64_t)split * p.split_stride;
            auto al16 = [](const void* q) { return (((uintptr_t)q) & 15) == 0; };
            const bool staged =
                wr0 + 32 <= p.M && c_first + kCols <= p.N && al16(po) && p.ldo % 4 == 0 &&
                (!p.c0 || (al16(p.c0) && p.ldc0 % 4 == 0)) &&
                (!p.bias || (al16(p.bias) && p.ld_bias % 4 == 0 && p.bias_cols % 4 == 0 &&
                             (c_first % p.bias_cols) + kCols <= p.bias_cols));
            if (staged) {
                float* stg = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 512) +
                             (warp - 4) * kStgFloats;
                const float sa = p.alpha * p.inv_sa[r];
                const int cc = (lane & 7) * 4, rsub = lane >> 3;
                const int64_t bcol0 = p.bias ? c_first % p.bias_cols : 0;
#pragma unroll
                for (int c0 = 0; c0 < kCols; c0 += 32) {
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = acc[c0 + j] * sa;
                    __syncwarp();
                    const int64_t c = c_first + c0 + cc;
                    const float4 sv = *reinterpret_cast<const float4*>(p.inv_sb + c);
#pragma unroll
                    for (int i0 = 0; i0 < 8; i0 += 4) {
                        float4 cv[4], bv[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int64_t row = wr0 + (i0 + i) * 4 + rsub;
                            cv[i] = p.c0 ? __ldg(reinterpret_cast<const float4*>(p.c0 + row * p.ldc0 + c))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                            bv[i] = p.bias ? __ldg(reinterpret_cast<const float4*>(
                                                 p.bias + row * p.ld_bias + bcol0 + c0 + cc))
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int rr = (i0 + i) * 4 + rsub;
                            const float* sr = stg + rr * 33 + cc;
                            float4 o;
                            o.x = sr[0] * sv.x;
                            o.y = sr[1] * sv.y;
                            o.z = sr[2] * sv.z;
                            o.w = sr[3] * sv.w;
                            if (p.c0) {
                                o.x += p.beta * cv[i].x; o.y += p.beta * cv[i].y;
                                o.z += p.beta * cv[i].z; o.w += p.beta * cv[i].w;
                            }
                            if (p.bias) {
                                o.x += bv[i].x; o.y += bv[i].y; o.z += bv[i].z; o.w += bv[i].w;
                            }
                            *reinterpret_cast<float4*>(po + (wr0 + rr) * p.ldo + c) = o;
                        }
                    }
                }
            } else if (r < p.M && c_first < p.N) {
                f16p_store_row(p, split, r, c_first, (int)min((int64_t)kCols, p.N - c_first), acc);
            }
        } else {
            if (r < p.M && c_first < p.N)
                f16p_store_row(p, split, r, c_first, (int)min((int64_t)kCols, p.N - c_first), acc);
        }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    if (warp == 2) ptx::tmem_dealloc_pair(tmem, kTmemCols);
}

// one block per row: scale = 2^e with max|x| * scale in [2^13, 2^14); h = fp16(xs), l = fp16(xs - h)
// col_scale (optional): the row is split as src[r][k] * col_scale[k] (a per-column power of two
// folded in first, e.g. the other operand's per-row scale of a reduction over k)
__global__ void __launch_bounds__(256) f16pair_split_kernel(const float* __restrict__ src, int64_t ld,
                                                            int64_t K, __half* __restrict__ h,
                                                            __half* __restrict__ l, int64_t ldo,
                                                            float* __restrict__ inv_scale,
                                                            const float* __restrict__ col_scale) {
    const int64_t r = blockIdx.x;
    const float* row = src + r * ld;
    auto at = [&](int64_t k) { return col_scale ? row[k] * col_scale[k] : row[k]; };
    float mx = 0.f;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) mx = fmaxf(mx, fabsf(at(k)));
    __shared__ float red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
    int e = 0;
    if (mx > 0.f && isfinite(mx)) {
        int ex;
        frexpf(mx, &ex);  // mx = f * 2^ex, f in [0.5, 1)  ->  mx * 2^(14 - ex) in [2^13, 2^14)
        e = 14 - ex;
        e = max(-120, min(120, e));
    }
    const float s = ldexpf(1.f, e);
    if (threadIdx.x == 0) inv_scale[r] = ldexpf(1.f, -e);
    __half* hr = h + r * ldo;
    __half* lr = l + r * ldo;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        const float v = at(k) * s;
        const __half hv = __float2half_rn(v);
        hr[k] = hv;
        lr[k] = __float2half_rn(v - __half2float(hv));
    }
}

// Transposed re-split of fp16-pair rows: src rows r < rows (<= 256) of (h + l) * inv_src[r],
// columns c -> out row c (K-major in r) with its own power-of-two scale.  One block per 32
// source columns: coalesced row reads into shared memory, per-column max, coalesced writes.
constexpr int kTRows = 256;
__global__ void __launch_bounds__(256) f16pair_transpose_kernel(
    const __half* __restrict__ h, const __half* __restrict__ l, int64_t ldi,
    const float* __restrict__ inv_src, int rows, int64_t cols, __half* __restrict__ oh,
    __half* __restrict__ ol, int64_t ldo, float* __restrict__ inv_out) {
    __shared__ float tile[kTRows][33];
    __shared__ float red[8][33];
    __shared__ float sc[32];
    const int64_t c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t c = c0 + tx;
    float mx = 0.f;
    for (int r = ty; r < kTRows; r += 8) {
        float v = 0.f;
        if (r < rows && c < cols)
            v = (__half2float(h[r * ldi + c]) + __half2float(l[r * ldi + c])) * inv_src[r];
        tile[r][tx] = v;
        mx = fmaxf(mx, fabsf(v));
    }
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
        if (c < cols) inv_out[c] = ldexpf(1.f, -e);
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {  // output row c0 + j, lanes over r
        const int64_t oc = c0 + j;
        if (oc >= cols) continue;
        const float s = sc[j];
        for (int r = tx; r < rows; r += 32) {
            const float v = tile[r][j] * s;
            const __half hv = __float2half_rn(v);
            oh[oc * ldo + r] = hv;
            ol[oc * ldo + r] = __float2half_rn(v - __half2float(hv));
        }
    }
}

// fp32 reconstruction x = (h + l) / scale (members read-back, covariance tracking)
__global__ void f16pair_recon_kernel(const __half* __restrict__ h, const __half* __restrict__ l,
                                     int64_t ldi, const float* __restrict__ inv_scale, int64_t rows,
                                     int64_t K, float* __restrict__ out, int64_t ldo) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= K) return;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        out[r * ldo + k] =
            (__half2float(h[r * ldi + k]) + __half2float(l[r * ldi + k])) * inv_scale[r];
}

// split-K partials -> C, summed in split order (deterministic).  One thread per 4 columns of a
// row (2-D grid: no 64-bit division per element; float4 when N and ldc allow it).
__global__ void f16p_sum_splits(const float* __restrict__ ws, int split, int64_t M, int64_t N,
                                float* __restrict__ C, int64_t ldc) {
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (c >= N) return;
    const int64_t MN = M * N;
    const bool vec = c + 4 <= N && (N & 3) == 0 && (ldc & 3) == 0 && (((uintptr_t)C) & 15) == 0;
    for (int64_t r = blockIdx.y; r < M; r += gridDim.y) {
        const float* src = ws + r * N + c;
        float* dst = C + r * ldc + c;
        if (vec) {
            float4 v = __ldg(reinterpret_cast<const float4*>(src));
            for (int z = 1; z < split; ++z) {
                const float4 w = __ldg(reinterpret_cast<const float4*>(src + (int64_t)z * MN));
                v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
            }
            *reinterpret_cast<float4*>(dst) = v;
            continue;
        }
        for (int q = 0; q < 4 && c + q < N; ++q) {
            float v = src[q];
            for (int z = 1; z < split; ++z) v += src[(int64_t)z * MN + q];
            dst[q] = v;
        }
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode16() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* q = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &qr) ==
                cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(q);
    }
    return fn;
}

bool map16(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int64_t ld, int box_rows) {
    EncodeTiledFn fn = encode16();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// MN-major B ([K][N] with N contiguous): boxes of 32 N x KC K rows
bool map16_mn(CUtensorMap* m, const void* base, int64_t krows, int64_t N, int64_t ld) {
    EncodeTiledFn fn = encode16();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)krows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {32u, (cuuint32_t)KC};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
int launch16(const CUtensorMap* maps, P16 p, dim3 grid, cudaStream_t st) {
    using L = L16<BN>;
    int stages = kSmemBudget / L::kStage;
    if (stages > 8) stages = 8;
    p.stages = stages;
    const size_t smem = (size_t)stages * L::kStage + 1024 + 512;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(f16p_gemm_kernel<BN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) {
            set_error("f16p gemm: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = true;
    }
    f16p_gemm_kernel<BN><<<grid, kThreads, smem, st>>>(maps[0], maps[1], maps[2], maps[3], p);
    return check_launch("enks_gemm_f16pair");
}

int launch_pair(const CUtensorMap* maps, P16 p, dim3 grid, cudaStream_t st) {
    int stages = kSmemBudget / LP::kStage;
    if (stages > 8) stages = 8;
    if (p.b_mn) stages = kMnStages;
    p.stages = stages;
    const size_t smem = (size_t)stages * LP::kStage + 1024 + 512 + (p.b_mn ? kStgBytes : 0);
    static bool configured = false;
    if (!configured) {
        const size_t smem_k = (size_t)std::min(kSmemBudget / LP::kStage, 8) * LP::kStage + 1024 + 512;
        const size_t smem_mn = (size_t)kMnStages * LP::kStage + 1024 + 512 + kStgBytes;
        cudaError_t e = cudaFuncSetAttribute(f16p_gemm_pair_kernel<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_k);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(f16p_gemm_pair_kernel<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_mn);
        if (e != cudaSuccess) {
            set_error("f16p pair gemm: smem attribute: %s", cudaGetErrorString(e));
            return ENKS_E_CUDA;
        }
        configured = true;
    }
    if (p.b_mn)
        f16p_gemm_pair_kernel<true><<<grid, kThreads, smem, st>>>(maps[0], maps[1], maps[2], maps[3], p);
    else
        f16p_gemm_pair_kernel<false><<<grid, kThreads, smem, st>>>(maps[0], maps[1], maps[2], maps[3], p);
    return check_launch("enks_gemm_f16pair(pair)");
}

// pairs of CTAs over 74 pair slots
// SMs left free for a concurrent one-CTA kernel (the side-stream gain solve): set by the host
// around the cross-moment launches of update() (enks_set_sm_reserve), 0 otherwise
int g_sm_reserve = 0;
int usable_sms() { return kNumSMs - g_sm_reserve; }

int choose_split_pairs(int pairs, int64_t chunks) {
    int best = 1;
    double best_eff = 0.0;
    const int slots = usable_sms() / 2;
    for (int s = 1; s <= 64; ++s) {
        if (chunks / s < 8 && s > 1) break;
        const int units = pairs * s;
        const int waves = (units + slots - 1) / slots;
        const double eff = (double)units / (double)(waves * slots);
        if (eff > best_eff + 0.03) {
            best_eff = eff;
            best = s;
        }
        if (eff > 0.95) break;
    }
    return best;
}

bool use_pair(int64_t N) {
    return env_knob("ENKS_F16P_PAIR", 1) != 0 && N > 128;
}

int choose_split16(int tiles, int64_t chunks) {
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 64; ++s) {
        if (chunks / s < 8 && s > 1) break;
        const int units = tiles * s;
        const int waves = (units + usable_sms() - 1) / usable_sms();
        const double eff = (double)units / (double)(waves * usable_sms());
        if (eff > best_eff + 0.03) {
            best_eff = eff;
            best = s;
        }
        if (eff > 0.95) break;
    }
    return best;
}

}  // namespace
}  // namespace enks

extern "C" {

int enks_f16pair_split(const float* src, int64_t ld, int64_t rows, int64_t K, void* h, void* l,
                       int64_t ldo, float* inv_scale, void* stream) {
    ENKS_REQUIRE(src && h && l && inv_scale, "enks_f16pair_split: null pointer");
    if (rows <= 0 || K <= 0) return ENKS_OK;
    enks::f16pair_split_kernel<<<(unsigned)rows, 256, 0, enks::as_stream(stream)>>>(
        src, ld, K, static_cast<__half*>(h), static_cast<__half*>(l), ldo, inv_scale, nullptr);
    return enks::check_launch("enks_f16pair_split");
}

int enks_f16pair_split_cs(const float* src, int64_t ld, int64_t rows, int64_t K,
                          const float* col_scale, void* h, void* l, int64_t ldo, float* inv_scale,
                          void* stream) {
    ENKS_REQUIRE(src && col_scale && h && l && inv_scale, "enks_f16pair_split_cs: null pointer");
    if (rows <= 0 || K <= 0) return ENKS_OK;
    enks::f16pair_split_kernel<<<(unsigned)rows, 256, 0, enks::as_stream(stream)>>>(
        src, ld, K, static_cast<__half*>(h), static_cast<__half*>(l), ldo, inv_scale, col_scale);
    return enks::check_launch("enks_f16pair_split_cs");
}

int enks_f16pair_recon(const void* h, const void* l, int64_t ldi, const float* inv_scale,
                       int64_t rows, int64_t K, float* out, int64_t ldo, void* stream) {
    ENKS_REQUIRE(h && l && inv_scale && out, "enks_f16pair_recon: null pointer");
    const int64_t total = rows * K;
    if (total <= 0) return ENKS_OK;
    const dim3 grid((unsigned)((K + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535));
    enks::f16pair_recon_kernel<<<grid, 256, 0, enks::as_stream(stream)>>>(
        static_cast<const __half*>(h), static_cast<const __half*>(l), ldi, inv_scale, rows, K, out,
        ldo);
    return enks::check_launch("enks_f16pair_recon");
}

}  // extern "C"

namespace enks {
namespace {
struct Epi {
    float beta;
    const float* c0;
    int64_t ldc0;
    const float* bias;
    int64_t ld_bias;
    int bias_cols;
};

int f16p_split_for(int64_t M, int64_t N, int64_t K, bool fused) {
    if (fused) return 1;
    const int BN = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
    const int m_tiles = (int)((M + BM - 1) / BM);
    const int n_tiles = (int)((N + BN - 1) / BN);
    const int64_t chunks = (K + KC - 1) / KC;
    return use_pair(N) ? choose_split_pairs((m_tiles + 1) / 2 * n_tiles, chunks)
                       : choose_split16(m_tiles * n_tiles, chunks);
}

int gemm_f16pair_impl(int64_t M, int64_t N, int64_t K, float alpha, const void* Ah, const void* Al,
                      int64_t lda, const float* inv_sa, const void* Bh, const void* Bl, int64_t ldb,
                      const float* inv_sb, float* C, int64_t ldc, void* ws, void* stream,
                      const Epi* epi, bool b_mn = false) {
    ENKS_REQUIRE(Ah && Al && Bh && Bl && inv_sa && inv_sb && C, "enks_gemm_f16pair: null pointer");
    ENKS_REQUIRE(!b_mn || (epi && use_pair(N) && (K % KC) == 0 && (N % 8) == 0),
                 "enks_gemm_f16pair_ex_mn: needs N > 128, K %% 32 == 0, N %% 8 == 0");
    ENKS_REQUIRE(N >= 1 && K >= 1 && (lda % 8) == 0 && (ldb % 8) == 0,
                 "enks_gemm_f16pair: need 16-B aligned fp16 rows (ld %% 8 == 0)");
    ENKS_REQUIRE(N <= 256 || use_pair(N), "enks_gemm_f16pair: N > 256 needs the CTA-pair kernel");
    ENKS_REQUIRE(!epi || !epi->bias || epi->bias_cols > 0, "enks_gemm_f16pair: bias_cols <= 0");
    if (M == 0) return ENKS_OK;
    const int BN = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
    const bool pair = use_pair(N);
    CUtensorMap maps[4];
    const bool bmaps = b_mn ? (map16_mn(&maps[2], Bh, K, N, ldb) && map16_mn(&maps[3], Bl, K, N, ldb))
                            : (map16(&maps[2], Bh, N, K, ldb, pair ? 128 : BN) &&
                               map16(&maps[3], Bl, N, K, ldb, pair ? 128 : BN));
    if (!map16(&maps[0], Ah, M, K, lda, BM) || !map16(&maps[1], Al, M, K, lda, BM) || !bmaps) {
        set_error("enks_gemm_f16pair: cuTensorMapEncodeTiled failed (alignment?)");
        return ENKS_E_UNSUPPORTED;
    }
    const int m_tiles = (int)((M + BM - 1) / BM);
    const int n_tiles = (int)((N + BN - 1) / BN);
    const int split = f16p_split_for(M, N, K, epi != nullptr);
    ENKS_REQUIRE(split == 1 || ws, "enks_gemm_f16pair: split-K needs workspace");
    P16 p;
    p.M = M; p.N = N; p.K = K;
    p.alpha = alpha;
    p.inv_sa = inv_sa;
    p.inv_sb = inv_sb;
    p.splits = split;
    // chain length: kF16pChainDefault (own knob only: ENKS_TC_CHAIN tunes gemm_tc and no longer
    // leaks into this kernel)
    p.chain = env_knob("ENKS_F16P_CHAIN", kF16pChainDefault);
    p.products = debug_knob("ENKS_F16P_PRODUCTS", 3) == 2 ? 2 : 3;  // 2 breaks 1e-4
    p.b_mn = b_mn ? 1 : 0;
    if (p.chain < 1) p.chain = 1;
    const bool direct = split == 1;
    p.out = direct ? C : static_cast<float*>(ws);
    p.ldo = direct ? ldc : N;
    p.split_stride = direct ? 0 : M * N;
    p.beta = epi ? epi->beta : 0.f;
    p.c0 = epi ? epi->c0 : nullptr;
    p.ldc0 = epi ? epi->ldc0 : 0;
    p.bias = epi ? epi->bias : nullptr;
    p.ld_bias = epi ? epi->ld_bias : 0;
    p.bias_cols = epi && epi->bias_cols > 0 ? epi->bias_cols : 1;
    dim3 grid((unsigned)m_tiles, (unsigned)n_tiles, (unsigned)split);
    cudaStream_t st = as_stream(stream);
    int rc;
    if (pair) {
        grid.x = (unsigned)((m_tiles + 1) & ~1);
        // one wave of CTA pairs, each looping over 256-column tiles
        const int64_t pairs_xz = (int64_t)(grid.x / 2) * split;
        const int64_t slots = usable_sms() / 2;
        const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(n_tiles, slots / std::max<int64_t>(1, pairs_xz)));
        grid.y = (unsigned)gy;
        rc = launch_pair(maps, p, grid, st);
    } else switch (BN) {
        case 32: rc = launch16<32>(maps, p, grid, st); break;
        case 64: rc = launch16<64>(maps, p, grid, st); break;
        case 128: rc = launch16<128>(maps, p, grid, st); break;
        default: rc = launch16<256>(maps, p, grid, st); break;
    }
    if (rc || direct) return rc;
    const dim3 sgrid((unsigned)((N + 4 * 128 - 1) / (4 * 128)), (unsigned)(M < 65535 ? M : 65535));
    f16p_sum_splits<<<sgrid, 128, 0, st>>>(static_cast<float*>(ws), split, M, N, C, ldc);
    return check_launch("enks_gemm_f16pair(split reduce)");
}
}  // namespace
}  // namespace enks

extern "C" {

int enks_set_sm_reserve(int sms) {
    ENKS_REQUIRE(sms >= 0 && sms <= 16, "enks_set_sm_reserve: %d outside [0, 16]", sms);
    enks::g_sm_reserve = sms;
    return ENKS_OK;
}

int64_t enks_gemm_f16pair_ws_bytes(int64_t M, int64_t N, int64_t K) {
    const int split = enks::f16p_split_for(M, N, K, false);
    return split > 1 ? (int64_t)split * M * N * (int64_t)sizeof(float) : 0;
}

int enks_gemm_f16pair(int64_t M, int64_t N, int64_t K, float alpha, const void* Ah, const void* Al,
                      int64_t lda, const float* inv_sa, const void* Bh, const void* Bl, int64_t ldb,
                      const float* inv_sb, float* C, int64_t ldc, void* ws, void* stream) {
    return enks::gemm_f16pair_impl(M, N, K, alpha, Ah, Al, lda, inv_sa, Bh, Bl, ldb, inv_sb, C, ldc,
                                   ws, stream, nullptr);
}

int enks_gemm_f16pair_ex(int64_t M, int64_t N, int64_t K, float alpha, const void* Ah,
                         const void* Al, int64_t lda, const float* inv_sa, const void* Bh,
                         const void* Bl, int64_t ldb, const float* inv_sb, float beta,
                         const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias,
                         int bias_cols, float* C, int64_t ldc, void* stream) {
    const enks::Epi epi{beta, C0, ldc0, bias, ld_bias, bias_cols};
    return enks::gemm_f16pair_impl(M, N, K, alpha, Ah, Al, lda, inv_sa, Bh, Bl, ldb, inv_sb, C, ldc,
                                   nullptr, stream, &epi);
}

int enks_gemm_f16pair_ex_mn(int64_t M, int64_t N, int64_t K, float alpha, const void* Ah,
                            const void* Al, int64_t lda, const float* inv_sa, const void* Bh,
                            const void* Bl, int64_t ldb, const float* inv_sn, float beta,
                            const float* C0, int64_t ldc0, const float* bias, int64_t ld_bias,
                            int bias_cols, float* C, int64_t ldc, void* stream) {
    const enks::Epi epi{beta, C0, ldc0, bias, ld_bias, bias_cols};
    return enks::gemm_f16pair_impl(M, N, K, alpha, Ah, Al, lda, inv_sa, Bh, Bl, ldb, inv_sn, C,
                                   ldc, nullptr, stream, &epi, true);
}

int enks_f16pair_transpose(const void* h, const void* l, int64_t ldi, const float* inv_src,
                           int rows, int64_t cols, void* oh, void* ol, int64_t ldo, float* inv_out,
                           void* stream) {
    ENKS_REQUIRE(h && l && inv_src && oh && ol && inv_out, "enks_f16pair_transpose: null pointer");
    ENKS_REQUIRE(rows >= 1 && rows <= enks::kTRows, "enks_f16pair_transpose: rows must be 1..%d",
                 enks::kTRows);
    if (cols <= 0) return ENKS_OK;
    enks::f16pair_transpose_kernel<<<(unsigned)((cols + 31) / 32), 256, 0,
                                     enks::as_stream(stream)>>>(
        static_cast<const __half*>(h), static_cast<const __half*>(l), ldi, inv_src, rows, cols,
        static_cast<__half*>(oh), static_cast<__half*>(ol), ldo, inv_out);
    return enks::check_launch("enks_f16pair_transpose");
}

}  // extern "C"
