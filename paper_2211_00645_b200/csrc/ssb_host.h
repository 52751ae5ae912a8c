// Host-side helpers shared by the libssb translation units: thread-local error
// text, status codes, launch accounting.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "ssb.h"

namespace ssb {

void set_error(const char *fmt, ...);
void count_launches(int64_t k);

// benchmark timing of the main fused kernel (ssb_profile_*)
void profile_begin(cudaStream_t st);
void profile_end(cudaStream_t st);

inline int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    set_error("%s", buf);
    return code;
}

inline int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SSB_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return SSB_OK;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// SM count of the calling thread's current device (cached per device: a process may drive
// several GPUs, e.g. one host thread per device)
inline int num_sms() {
    constexpr int kMaxDevices = 64;
    static int cache[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    int sms = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
    if (sms == 0) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
        __atomic_store_n(&cache[dev], sms, __ATOMIC_RELAXED);
    }
    return sms;
}

}  // namespace ssb
