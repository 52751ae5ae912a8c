/*
 * ssb.h -- C ABI of the B200 deskew + projection library (libssb.so).
 *
 * The reference (skewstream, pure Python/numpy) has no FFI layer: its boundary
 * is the Python API.  Each entry point below replaces one reference function on
 * the hot path; the Python drop-in (paper_2211_00645_b200/) binds them with
 * ctypes.  No torch types cross this boundary: device buffers are plain
 * pointers (the caller owns them; the library never keeps a pointer past the
 * call), sizes are int64, the stream is an opaque cudaStream_t (NULL = legacy
 * default stream).  Every call is asynchronous on that stream.
 *
 * Data layout (reference file:line):
 *   raw frames  (n, H, W) uint16 C-order, W contiguous            ss/pipeline.py:34-61
 *   volume      (n, U, W) uint16 C-order, zero outside each slice ss/phantom.py:390 (the "pile")
 *   XY          (U, W)  = reduce over slices (axis 0)             ss/pipeline.py:316-336
 *   XZ          (n, W)  = reduce over canvas rows (axis 1)        north_star extension
 *   YZ          (n, U)  = reduce over columns (axis 2)            north_star extension
 *   max -> uint16, sum -> uint32 (sum of the rounded uint16 voxels, exact)
 * U = H + ceil((N-1)*s - 1e-9) (ss/geometry.py:129-147); a call may cover a
 * window of canvas rows [u_begin, u_begin + u_count) (scan-axis slabs).
 */
#ifndef SSB_H
#define SSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSB_VERSION 200

/* status codes; Python maps them onto ss/errors.py classes */
#define SSB_OK 0
#define SSB_ERR_PARAM 1    /* ParameterError (a ValueError)   ss/errors.py:8  */
#define SSB_ERR_CAPACITY 2 /* CapacityError                   ss/errors.py:12 */
#define SSB_ERR_PROTOCOL 3 /* ProtocolError                   ss/errors.py:16 */
#define SSB_ERR_CUDA 4     /* SkewstreamError (device failure)                */

#define SSB_INTERP_NEAREST 0 /* ss/geometry.py:236-243 placement, frame rows copied  */
#define SSB_INTERP_LINEAR 1  /* ss/geometry.py:246-255 span, two-row lerp per frame  */

#define SSB_FORMULA_CANVAS 0   /* ss/pipeline.py:229-236  rint((1-f)*a + f*b), fp64 */
#define SSB_FORMULA_NPINTERP 1 /* ss/phantom.py:396-402   np.interp per column, fp64 */

#define SSB_REDUCE_MAX 0
#define SSB_REDUCE_SUM 1

/* flags */
#define SSB_FLAG_XY_ACCUMULATE 1 /* xy = reduce(xy, new) instead of xy = new (canvas place) */
#define SSB_FLAG_XY_U32 2        /* max mode: xy is the caller's uint32 accumulator, max-folded in place
                                    (not reset, not narrowed to uint16) -- a chunked stream keeps one
                                    across its chunks instead of a whole-canvas reset + narrowing pass
                                    per chunk; frames must take TMA boxes (16-byte aligned, W % 8 == 0) */

typedef struct ssb_deskew_desc {
    int64_t n;           /* frames in this call                                    */
    int64_t height;      /* H, rows per frame (oblique / sheet-depth axis)         */
    int64_t width;       /* W, columns per frame (invariant axis, contiguous)      */
    int64_t first_slice; /* global scan index of frame 0 (slabs keep global i*s)   */
    double shear_px;     /* s, canvas rows per slice (>= 0)                        */
    int32_t interp;      /* SSB_INTERP_*                                           */
    int32_t formula;     /* SSB_FORMULA_*                                          */
    int64_t u_begin;     /* first canvas row covered                               */
    int64_t u_count;     /* canvas rows covered (volume / XY / YZ row extent)      */
    int32_t reduce;      /* SSB_REDUCE_*                                           */
    int32_t flags;       /* SSB_FLAG_*                                             */
    int64_t row_stride;  /* elements between frame rows (0: width); lets a channel  */
    int64_t frame_stride;/* crop of a wider camera frame be deskewed in place (0: H*row_stride) */
} ssb_deskew_desc;

/* Library version (SSB_VERSION) and the last error message of this thread. */
int ssb_version(void);
const char *ssb_last_error(void);

/* Number of kernels this library has launched in the process (for the bench). */
int64_t ssb_launch_count(void);

/*
 * Kernel timing for the benchmark (per calling thread): while enabled, every
 * ssb_deskew records a CUDA event pair around its main fused kernel on the
 * launch stream.  ssb_profile_read waits for the recorded events, returns the
 * summed device milliseconds and the number of timed launches, and clears them.
 */
int ssb_profile_enable(int32_t on);
int ssb_profile_read(double *total_ms, int64_t *launches);

/* Scratch bytes ssb_deskew needs for partial projections. */
size_t ssb_deskew_workspace_bytes(const ssb_deskew_desc *d);

/*
 * Fused deskew + projections.  Replaces, for a whole stack or a slab of it:
 *   ProjectionCanvas.place x n + finalize_global   ss/pipeline.py:316-336  (formula CANVAS)
 *   phantom.reference_deskew                       ss/phantom.py:359-402   (formula NPINTERP)
 *   _interp_slice_rows per slice                   ss/pipeline.py:229-236
 * raw: device (n, H, W) uint16, row / frame strides from the descriptor (a channel
 * crop of ss/pipeline.py:105-112 is passed as a strided view, no copy).
 * vol: device (n, u_count, W) uint16 or NULL.
 * xy (u_count, W), xz (n, W), yz (n, u_count): device, uint16 (max) or
 * uint32 (sum), each may be NULL.  workspace: device, >= ssb_deskew_workspace_bytes.
 * Pointers must be 16-byte aligned for the vectorised path (any alignment works).
 */
int ssb_deskew(const ssb_deskew_desc *d, const uint16_t *raw, uint16_t *vol, void *xy, void *xz,
               void *yz, void *workspace, size_t workspace_bytes, void *stream);

/*
 * Batched fused deskew: `batch` stacks of one shape in one persistent launch.  Small stacks
 * (BASELINE config 1: 128 x 256 x 512) leave most of the 148 SMs idle one launch at a time; the
 * reference deskews them one canvas after another (ss/cli.py:332-338).  raw: device
 * (batch, n, H, W) uint16, stacks back to back (stack stride = n * frame stride of the descriptor);
 * vol (batch, n, U, W) or NULL; xy (batch, U, W), xz (batch, n, W), yz (batch, n, U), uint16 (max) or
 * uint32 (sum), each may be NULL.  Stack b's outputs equal ssb_deskew on stack b alone (falls back to
 * one launch per stack where the frames cannot take TMA boxes).  workspace:
 * >= ssb_deskew_batch_workspace_bytes(d, batch).
 */
size_t ssb_deskew_batch_workspace_bytes(const ssb_deskew_desc *d, int64_t batch);
int ssb_deskew_batch(const ssb_deskew_desc *d, int64_t batch, const uint16_t *raw, uint16_t *vol, void *xy,
                     void *xz, void *yz, void *workspace, size_t workspace_bytes, void *stream);

/*
 * Rolling-mode band recompute.  Replaces ProjectionCanvas._recompute_band
 * (ss/pipeline.py:361-377): canvas rows [lo, hi] become the strict-'>' max over
 * the live ring slices (present[k] != 0) with contributor = first maximal ring
 * index, -1 where nothing contributes.  ring: device (n_ring, H, W) uint16 where
 * ring slot k holds global slice k; canvas (U, W) uint16, contributor (U, W) int16.
 * replaced >= 0: only ring slot `replaced` changed since canvas/contributor were
 * last consistent, so voxels it did not contribute to are updated in O(1)
 * (exactly equal to the full re-max) and the ones it did are re-maxed over the ring
 * (device workspace >= ssb_rolling_workspace_bytes(hi - lo + 1, W) holds their list);
 * replaced < 0: full recompute of the band (no workspace needed).
 */
size_t ssb_rolling_workspace_bytes(int64_t band_rows, int64_t width);
int ssb_rolling_band(const uint16_t *ring, const uint8_t *present, int64_t n_ring, int64_t height,
                     int64_t width, double shear_px, int32_t interp, int64_t lo, int64_t hi,
                     uint16_t *canvas, int16_t *contributor, int64_t canvas_rows, int64_t replaced,
                     void *workspace, size_t workspace_bytes, void *stream);

/*
 * Display warp.  Replaces warp_projection (ss/pipeline.py:434-457): out row m
 * samples input row clip(m / scale, 0, rows-1) with an fp64 lerp and rint;
 * scale == 1.0 is a copy.  out_rows = round(rows * scale) (caller computes).
 */
int ssb_warp_rows(const uint16_t *proj, int64_t rows, int64_t cols, double warp_scale,
                  uint16_t *out, int64_t out_rows, void *stream);

/*
 * Projection combine for multi-GPU gathers: dst[k] = reduce(dst[k], src[k]) for
 * count elements of uint16 (elem_bits 16, max) or uint32 (elem_bits 32, max/sum).
 */
int ssb_combine(const void *src, void *dst, int64_t count, int32_t reduce, int32_t elem_bits,
                void *stream);

/*
 * Display encode, gray8 payload.  Replaces the pixel path of encode_frame_packet
 * (skewstream/server.py:83-91): offset = min, range = max - min over the image;
 * range == 0 -> all-zero bytes, else dst[k] = rint((src[k] - offset) * (255.0 / range))
 * in fp64 (numpy's op order).  src: device uint16 (count), dst: device uint8 (count);
 * stats: device, >= ssb_encode_gray8_stats_bytes(), receives {offset, range} as uint32 in
 * words 0 and 1 (the header fields g8_offset / g8_range, server.py:84-86).  One launch.
 */
size_t ssb_encode_gray8_stats_bytes(void);
int ssb_encode_gray8(const uint16_t *src, int64_t count, uint8_t *dst, uint32_t *stats, size_t stats_bytes,
                     void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SSB_H */
