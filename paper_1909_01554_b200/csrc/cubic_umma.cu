// cubic_umma.cu -- K2: tcgen05 tensor-core block product (placeholder until the kernel lands).
#include "common.cuh"

namespace bmmgpu {

void umma_granularity(uint64_t* gm, uint64_t* gn, uint64_t* gk_bits) {
    *gm = 128;
    *gn = 256;
    *gk_bits = 1024;
}

int launch_cubic_umma(const uint64_t*, uint64_t, const uint64_t*, uint64_t, uint64_t*, uint64_t, uint64_t, uint64_t,
                      uint64_t, bool, bool, cudaStream_t, uint64_t, uint64_t, uint64_t, uint64_t) {
    set_error("tcgen05 kernel not built in this version");
    return kEinval;
}

}  // namespace bmmgpu
