// ntt_inst_14.cu -- N = 2^14 instantiation of the NTT-family and key/encryption launchers.
#include "ntt_kernels.cuh"
#include "rng_kernels.cuh"

namespace edl {
EDL_INSTANTIATE_NTT(14)
EDL_INSTANTIATE_RNG(14)
}  // namespace edl
