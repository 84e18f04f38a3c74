// Instantiates the fused 2D cell-map kernels for method order m = 2.
#include "cellmap_launch.cuh"
#include "simt2d.cuh"

namespace hw {
HW_INSTANTIATE_CELLMAP(2)
HW_INSTANTIATE_SIMT2D(2)
}  // namespace hw
