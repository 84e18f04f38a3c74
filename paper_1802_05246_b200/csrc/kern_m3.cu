// Instantiates the fused 2D cell-map kernels for method order m = 3.
#include "cellmap_launch.cuh"
#include "simt2d.cuh"

namespace hw {
HW_INSTANTIATE_CELLMAP(3)
HW_INSTANTIATE_SIMT2D(3)
}  // namespace hw
