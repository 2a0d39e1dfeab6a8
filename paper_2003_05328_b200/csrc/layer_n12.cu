// layer_n12.cu -- fused layer kernels instantiated for ring degree 2^12.
#include "layer_launch.cuh"

namespace ensei_gpu {
EG_INSTANTIATE_LAYER(12)
}  // namespace ensei_gpu
