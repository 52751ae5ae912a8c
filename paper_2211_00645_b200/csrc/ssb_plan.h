// Declarations shared by the two ssb_deskew kernels (tiled fallback and TMA path).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ssb.h"

namespace ssb {

constexpr int kTmaTileRows = 60;   // canvas rows per TMA work item (15 consumer warps x 4 rows)
constexpr int kTmaTileCols = 256;  // columns per work item (32 lanes x 8)

inline int64_t row_stride_of(const ssb_deskew_desc &d) { return d.row_stride ? d.row_stride : d.width; }
inline int64_t frame_stride_of(const ssb_deskew_desc &d) {
    return d.frame_stride ? d.frame_stride : row_stride_of(d) * d.height;
}

// TMA path usable for this call (16-byte aligned buffers, W % 8 == 0, driver entry point found)?
bool tma_eligible(const ssb_deskew_desc &d, const uint16_t *raw, const void *vol, const void *xy);

// Workspace the TMA path needs (scheduler counter + u32 reduction scratch for max mode).
size_t tma_workspace_bytes(const ssb_deskew_desc &d, int64_t batch = 1);

// Access class of the persistent kernel for this call: 16 = TMA boxes (16-byte aligned rows);
// 8 / 4 / 2 = row-copy mode (1-D bulk copies per frame row, AC-byte shared loads and volume
// stores); 0 = use the generic tiled kernel.
int persistent_access_class(const ssb_deskew_desc &d, const uint16_t *raw, const void *vol, const void *xy);

// Launch the persistent kernel (+ scratch resets and the u32 -> u16 finalize).
int launch_deskew_tma(const ssb_deskew_desc &d, const uint16_t *raw, uint16_t *vol, void *xy, void *xz, void *yz,
                      void *workspace, size_t workspace_bytes, cudaStream_t st, int ac, int64_t batch = 1);

}  // namespace ssb
