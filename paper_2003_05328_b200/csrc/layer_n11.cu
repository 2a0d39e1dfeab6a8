// layer_n11.cu -- fused layer kernels instantiated for ring degree 2^11.
#include "layer_launch.cuh"

namespace ensei_gpu {
EG_INSTANTIATE_LAYER(11)
}  // namespace ensei_gpu
