// Explicit instantiation of the draw kernels for float (see wd_launch.cuh).
#include "wd_launch.cuh"

namespace wd {
template int launch_draw<float>(int, int, int, int, const DrawParams<float>&, void*, size_t, cudaStream_t);
}  // namespace wd
