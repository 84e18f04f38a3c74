// Instantiates the fused 2D cell-map kernels for method order m = 5.
#include "cellmap_launch.cuh"
#include "simt2d.cuh"

namespace hw {
HW_INSTANTIATE_CELLMAP(5)
HW_INSTANTIATE_SIMT2D(5)
}  // namespace hw
