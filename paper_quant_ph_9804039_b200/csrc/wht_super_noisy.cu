// wht_super_noisy.cu -- the supertile pass with general real 2x2 stages
// (angle errors with decoherence contractions, NEXT-1/2; readings G19/G22).
// Compiled separately so the flavours build in parallel.
#include "wht_super.cuh"

namespace sv {

template void launch_super_uab<1>(int, int, const SuperParamsT<1> &, int, cudaStream_t);

}  // namespace sv
