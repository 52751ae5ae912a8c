// Declarations shared by the two ssb_deskew kernels (tiled fallback and TMA path).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ssb.h"

namespace ssb {

constexpr int kTmaTileRows = 60;   // canvas rows per TMA work item (15 consumer warps x 4 rows)
constexpr int kTmaTileCols = 256;  // columns per work item (32 lanes x 8)

// TMA path usable for this call (16-byte aligned buffers, W % 8 == 0, driver entry point found)?
bool tma_eligible(const ssb_deskew_desc &d, const uint16_t *raw, const void *vol, const void *xy);

// Launch the persistent TMA kernel; counters: >= 4 bytes of device scratch.
int launch_deskew_tma(const ssb_deskew_desc &d, const uint16_t *raw, uint16_t *vol, void *xy, void *xz,
                      void *yz, unsigned int *counters, int64_t UT, int64_t XT, int64_t S, int64_t chunk,
                      int xy_accumulate, cudaStream_t st);

}  // namespace ssb
