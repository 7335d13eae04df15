// ntt_inst_12.cu -- N = 2^12 instantiation of the NTT-family and key/encryption launchers.
#include "ntt_kernels.cuh"
#include "rng_kernels.cuh"

namespace edl {
EDL_INSTANTIATE_NTT(12)
EDL_INSTANTIATE_RNG(12)
}  // namespace edl
