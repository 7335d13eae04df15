// ntt_inst_15.cu -- N = 2^15 instantiation of the NTT-family and key/encryption launchers.
#include "ntt_kernels.cuh"
#include "rng_kernels.cuh"

namespace edl {
EDL_INSTANTIATE_NTT(15)
EDL_INSTANTIATE_RNG(15)
}  // namespace edl
