// ntt_inst_16.cu -- N = 2^16 instantiation of the NTT-family and key/encryption launchers.
#include "ntt_kernels.cuh"
#include "rng_kernels.cuh"

namespace edl {
EDL_INSTANTIATE_NTT(16)
EDL_INSTANTIATE_RNG(16)
}  // namespace edl
