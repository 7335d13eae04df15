// ntt_inst_11.cu -- N = 2^11 instantiation of the NTT-family and key/encryption launchers.
#include "ntt_kernels.cuh"
#include "rng_kernels.cuh"

namespace edl {
EDL_INSTANTIATE_NTT(11)
EDL_INSTANTIATE_RNG(11)
}  // namespace edl
