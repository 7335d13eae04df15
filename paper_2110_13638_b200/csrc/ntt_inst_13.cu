// ntt_inst_13.cu -- N = 2^13 instantiation of the NTT-family and key/encryption launchers.
#include "ntt_kernels.cuh"
#include "rng_kernels.cuh"

namespace edl {
EDL_INSTANTIATE_NTT(13)
EDL_INSTANTIATE_RNG(13)
}  // namespace edl
