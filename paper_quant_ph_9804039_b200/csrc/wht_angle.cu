// wht_angle.cu -- instantiation of the WHT tile pass for pure angle errors
// (reading G19): every Hadamard of tile bit b is
// U(phi_b) = c_b [[1, t_b], [t_b, -1]] with t_b = tan(phi_b); the butterflies
// apply [[1, t], [t, -1]] (2 packed FMAs) and the product of the pass's c_b is
// multiplied once into the loaded tile.  Compiled separately so the flavours
// build in parallel.
#include "wht_kernels.cuh"

namespace sv {

template void launch_tile_dispatch<2>(sv_dtype, const KParamsT<2> &, int, int, int, unsigned long long, cudaStream_t);

}  // namespace sv
