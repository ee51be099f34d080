// Explicit instantiation of the draw kernels for double (see wd_launch.cuh).
#include "wd_launch.cuh"

namespace wd {
template int launch_draw<double>(int, int, int, int, const DrawParams<double>&, void*, size_t, cudaStream_t);
}  // namespace wd
