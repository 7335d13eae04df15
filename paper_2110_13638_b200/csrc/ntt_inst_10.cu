// ntt_inst_10.cu -- N = 2^10 instantiation of the NTT-family and key/encryption launchers.
#include "ntt_kernels.cuh"
#include "rng_kernels.cuh"

namespace edl {
EDL_INSTANTIATE_NTT(10)
EDL_INSTANTIATE_RNG(10)
}  // namespace edl
