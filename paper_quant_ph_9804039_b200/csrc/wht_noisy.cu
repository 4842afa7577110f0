// wht_noisy.cu -- instantiation of the WHT tile pass with angle-error stages
// (reading G19): every butterfly of tile bit b is the
// reflection-rotation U(phi_b) = [[cos, sin], [sin, -cos]] instead of the
// ideal (x + y, x - y).  Same tiles, layouts, fusion and exchange as wht.cu;
// compiled separately so the two flavours build in parallel.
#include "wht_kernels.cuh"

namespace sv {

template void launch_tile_dispatch<1>(sv_dtype, const KParamsT<1> &, int, int, int, unsigned long long, cudaStream_t);

}  // namespace sv
