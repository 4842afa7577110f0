// wht_super_angle.cu -- the supertile pass with the angle-error tan form
// (NEXT-1; reading G19).  Compiled separately so the flavours build in parallel.
#include "wht_super.cuh"

namespace sv {

template void launch_super_uab<2>(int, int, const SuperParamsT<2> &, int, cudaStream_t);

}  // namespace sv
