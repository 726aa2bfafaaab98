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

// Environment knobs.  Tuning knobs (launch shapes, kernel variants that give the same results to
// rounding) are read ONCE per process, at the first launch that needs them (env_knob caches).
// Debug knobs that can break the numerical contract (MMA products dropped, roles switched off,
// descriptor overrides) exist only in builds with -DENKS_DEBUG_KNOBS (tools/ A/B probes): a
// production library ignores them and uses the defaults.
int env_knob(const char* name, int dflt);  // atoi(getenv(name)) or dflt, cached per name
#ifdef ENKS_DEBUG_KNOBS
inline int debug_knob(const char* name, int dflt) { return env_knob(name, dflt); }
#else
inline int debug_knob(const char*, int dflt) { return dflt; }
#endif

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace enks

#define ENKS_REQUIRE(cond, ...)               \
    do {                                      \
        if (!(cond)) {                        \
            enks::set_error(__VA_ARGS__);     \
            return ENKS_E_ARG;                \
        }                                     \
    } while (0)
