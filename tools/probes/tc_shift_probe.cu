// Probe: can a tcgen05.mma A operand (K-major, SWIZZLE_128B) start at a row that is not a
// multiple of 8 (start address + s * 128 B, descriptor base-offset field = s & 7)?
// Compares D = A[s .. s+127] * B^T against the host result for s = 0..2, with and without
// the base-offset field.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -I../../paper_2410_09663_b200/csrc
#include <cstdio>
#include <vector>

#include "tc_ptx.cuh"

using namespace enks;

__device__ __forceinline__ uint32_t sw128(int row, int byte) {
    return (uint32_t)(row * 128 + ((((byte >> 4) ^ (row & 7)) << 4) | (byte & 15)));
}

__device__ __forceinline__ uint64_t desc(const void* smem, int base_off) {
    uint64_t d = ptx::desc_kmajor_sw128(smem);
    d |= (uint64_t)(base_off & 7) << 49;
    return d;
}

__global__ void probe(float* out, int shift, int use_base) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
    uint8_t* A = sm;              // 136 rows x 128 B
    uint8_t* B = sm + 136 * 128 + 1024 - (136 * 128) % 1024;  // 1024-aligned, 32 rows
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int e = tid; e < 136 * 32; e += blockDim.x) {
        const int r = e >> 5, k = e & 31;
        *reinterpret_cast<float*>(A + sw128(r, 4 * k)) = (float)((r * 7 + k * 3) % 5 - 2);
    }
    for (int e = tid; e < 32 * 32; e += blockDim.x) {
        const int n = e >> 5, k = e & 31;
        *reinterpret_cast<float*>(B + sw128(n, 4 * k)) = (float)((n * 5 + k) % 7 - 3);
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
        constexpr uint32_t idesc = ptx::idesc_tf32(128, 32);
        for (int k = 0; k < 4; ++k) {
            const uint64_t ad = desc(A + shift * 128 + 32 * k, use_base ? shift : 0);
            const uint64_t bd = desc(B + 32 * k, 0);
            ptx::mma_tf32_ss(tmem, ad, bd, idesc, k ? 1u : 0u);
        }
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
    const int smem = 64 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<float> h(128 * 32);
    for (int use_base = 0; use_base < 2; ++use_base)
        for (int s = 0; s < 3; ++s) {
            probe<<<1, 128, smem>>>(d, s, use_base);
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
            printf("use_base=%d shift=%d max_err=%g\n", use_base, s, err);
        }
    return 0;
}
