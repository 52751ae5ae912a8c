// Explicit instantiations of the persistent deskew kernel's launchers: row-class TMA, 4- / 2-byte rows.
// (One translation unit per mode group so the build compiles them in parallel.)
#include "ssb_tma_kernel.cuh"

namespace ssb {
namespace tma_path {

template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 36>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 34>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 36>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 34>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);

}  // namespace tma_path
}  // namespace ssb
