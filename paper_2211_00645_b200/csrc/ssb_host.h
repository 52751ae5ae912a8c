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

inline int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace ssb
