// Explicit instantiations of the persistent deskew kernel's launchers: 16-byte aligned rows (TMA boxes).
// (One translation unit per mode group so the build compiles them in parallel.)
#include "ssb_tma_kernel.cuh"

namespace ssb {
namespace tma_path {

template int launch_variant<SSB_INTERP_NEAREST, SSB_FORMULA_CANVAS, 16>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_CANVAS, 16>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);
template int launch_variant<SSB_INTERP_LINEAR, SSB_FORMULA_NPINTERP, 16>(bool, bool, bool, const TmapSet &, const Params &, int,
                                                                  cudaStream_t);

}  // namespace tma_path
}  // namespace ssb
