// Library identity, error reporting and small elementwise kernels.
#include "common.cuh"

#include <stdlib.h>

#include <mutex>
#include <string>
#include <unordered_map>

#include <string.h>

namespace enks {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int env_knob(const char* name, int dflt) {
    // a handful of names, each looked up once; later calls read the cached value
    static std::mutex mu;
    static std::unordered_map<std::string, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(name);
    if (it != cache.end()) return it->second;
    const char* e = getenv(name);
    const int v = (e && *e) ? atoi(e) : dflt;
    cache.emplace(name, v);
    return v;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return ENKS_E_CUDA;
    }
    return ENKS_OK;
}

__global__ void probe_kernel(int* out) {
#ifdef __CUDA_ARCH__
    *out = __CUDA_ARCH__;
#endif
}

__global__ void sub_kernel(const float* __restrict__ a, int64_t lda, const float* __restrict__ b,
                           int64_t ldb, float* __restrict__ out, int64_t ldo, int64_t rows,
                           int64_t cols) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= cols) return;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        out[r * ldo + c] = a[r * lda + c] - b[r * ldb + c];
}

__global__ void add_kernel(const float* __restrict__ a, int64_t lda, const float* __restrict__ b,
                           int64_t ldb, float* out, int64_t ldo, int64_t rows, int64_t cols) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= cols) return;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        out[r * ldo + c] = a[r * lda + c] + b[r * ldb + c];
}

// out[0] (+)= scale * sum_ij E_ij X_ij, fp64, one CTA, fixed reduction order (deterministic)
__global__ void __launch_bounds__(1024) quad_form_kernel(const float* __restrict__ E, int64_t lde,
                                                        const float* __restrict__ X, int64_t ldx,
                                                        int64_t rows, int64_t cols, double scale,
                                                        double* out, int accumulate) {
    double acc = 0.0;
    const int64_t total = rows * cols;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
        const int64_t r = e / cols, c = e - r * cols;
        acc += (double)E[r * lde + c] * (double)X[r * ldx + c];
    }
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[0] = (accumulate ? out[0] : 0.0) + scale * t;
    }
}

}  // namespace enks

extern "C" {

int enks_quad_form(const float* E, int64_t lde, const float* X, int64_t ldx, int64_t rows,
                   int64_t cols, double scale, double* out, int accumulate, void* stream) {
    ENKS_REQUIRE(E && X && out, "enks_quad_form: null pointer");
    ENKS_REQUIRE(rows >= 0 && cols >= 0, "enks_quad_form: negative shape");
    enks::quad_form_kernel<<<1, 1024, 0, enks::as_stream(stream)>>>(E, lde, X, ldx, rows, cols,
                                                                    scale, out, accumulate);
    return enks::check_launch("enks_quad_form");
}

int enks_version(void) { return 1; }

const char* enks_last_error(void) { return enks::g_err; }

int enks_device_check(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 0;
    if (prop.major != 10 || prop.minor != 0) {
        enks::set_error("device %s is sm_%d%d; this library is built for sm_100a only", prop.name,
                        prop.major, prop.minor);
        return 0;
    }
    int* d = nullptr;
    if (cudaMalloc(&d, sizeof(int)) != cudaSuccess) return 0;
    enks::probe_kernel<<<1, 1>>>(d);
    int h = 0;
    cudaError_t e = cudaMemcpy(&h, d, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) {
        enks::set_error("probe kernel failed: %s", cudaGetErrorString(e));
        return 0;
    }
    return h == 1000 ? 1 : 0;
}

int enks_add(const float* a, int64_t lda, const float* b, int64_t ldb, float* out, int64_t ldo,
             int64_t rows, int64_t cols, void* stream) {
    ENKS_REQUIRE(a && b && out, "enks_add: null pointer");
    int64_t n = rows * cols;
    if (n == 0) return ENKS_OK;
    enks::add_kernel<<<dim3((unsigned)((cols + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535)), 256, 0,
                       enks::as_stream(stream)>>>(a, lda, b, ldb, out, ldo, rows, cols);
    return enks::check_launch("enks_add");
}

int enks_sub(const float* a, int64_t lda, const float* b, int64_t ldb, float* out, int64_t ldo,
             int64_t rows, int64_t cols, void* stream) {
    ENKS_REQUIRE(a && b && out, "enks_sub: null pointer");
    int64_t n = rows * cols;
    if (n == 0) return ENKS_OK;
    enks::sub_kernel<<<dim3((unsigned)((cols + 255) / 256), (unsigned)(rows < 65535 ? rows : 65535)), 256, 0,
                       enks::as_stream(stream)>>>(a, lda, b, ldb, out, ldo, rows, cols);
    return enks::check_launch("enks_sub");
}

}  // extern "C"
