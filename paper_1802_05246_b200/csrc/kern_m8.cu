// Instantiates the fused 2D cell-map kernels for method order m = 8.
#include "cellmap_launch.cuh"

namespace hw {
HW_INSTANTIATE_CELLMAP(8)
}  // namespace hw
