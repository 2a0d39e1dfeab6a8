// layer_n13.cu -- fused layer kernels instantiated for ring degree 2^13.
#include "layer_launch.cuh"

namespace ensei_gpu {
EG_INSTANTIATE_LAYER(13)
}  // namespace ensei_gpu
