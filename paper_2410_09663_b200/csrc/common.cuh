// Shared helpers for the enks_b200 C-ABI library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/enks_b200.h"

namespace enks {

void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Check the most recent launch; records the message and returns ENKS_E_CUDA on failure.
int check_launch(const char* what);

constexpr int kNumSMs = 148;  // B200

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace enks

#define ENKS_REQUIRE(cond, ...)               \
    do {                                      \
        if (!(cond)) {                        \
            enks::set_error(__VA_ARGS__);     \
            return ENKS_E_ARG;                \
        }                                     \
    } while (0)
