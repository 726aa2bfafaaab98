// Probe: kind::f16 A operand, K-major SWIZZLE_64B (32 fp16 = 64 B rows), start address shifted
// by s * 64 B (s = 0..2).  D = A[s .. s+127] * B^T vs host.
#include <cstdio>
#include <vector>
#include <cuda_fp16.h>

#include "tc_ptx.cuh"

using namespace enks;

__device__ __forceinline__ uint32_t sw64(int row, int byte) {
    // 64-B rows, 16-B chunks XOR (row >> 1) & 3  (SWIZZLE_64B: address bits [4:5] ^= bits [7:8])
    const uint32_t addr = (uint32_t)(row * 64 + byte);
    return addr ^ (((addr >> 7) & 3) << 4);
}

__device__ __forceinline__ uint64_t desc_sw64(const void* smem) {
    const uint64_t addr = ptx::smem_u32(smem);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFFull;
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(512 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__global__ void probe(float* out, int shift) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
    uint8_t* A = sm;                 // 136 rows x 64 B
    uint8_t* B = sm + 136 * 64 + 1024 - (136 * 64) % 1024;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int e = tid; e < 136 * 32; e += blockDim.x) {
        const int r = e >> 5, k = e & 31;
        *reinterpret_cast<__half*>(A + sw64(r, 2 * k)) = __float2half((float)((r * 7 + k * 3) % 5 - 2));
    }
    for (int e = tid; e < 32 * 32; e += blockDim.x) {
        const int n = e >> 5, k = e & 31;
        *reinterpret_cast<__half*>(B + sw64(n, 2 * k)) = __float2half((float)((n * 5 + k) % 7 - 3));
    }
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc(&slot, 32);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        for (int k = 0; k < 2; ++k)
            mma_f16(tmem, desc_sw64(A + shift * 64 + 32 * k), desc_sw64(B + 32 * k), idesc, k ? 1u : 0u);
        ptx::mma_commit(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    uint32_t v[32];
    ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16), v);
    ptx::tmem_ld_wait();
    for (int c = 0; c < 32; ++c) out[(warp * 32 + (tid & 31)) * 32 + c] = __uint_as_float(v[c]);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 32);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 32 * sizeof(float));
    const int smem = 32 * 1024;
    std::vector<float> h(128 * 32);
    for (int s = 0; s < 4; ++s) {
        probe<<<1, 128, smem>>>(d, s);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("launch error %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 32; ++n) {
                double ref = 0;
                for (int k = 0; k < 32; ++k)
                    ref += (double)(((m + s) * 7 + k * 3) % 5 - 2) * (double)((n * 5 + k) % 7 - 3);
                err = fmax(err, fabs(ref - h[m * 32 + n]));
            }
        printf("f16 sw64 shift=%d max_err=%g\n", s, err);
    }
    return 0;
}
