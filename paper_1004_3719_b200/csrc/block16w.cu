// Block kernels reading u16 iterates and writing u32 (the sequence's V_out),
// instantiated here rather than in seq.cu.
#define FFSPMV_BLOCK_INSTANTIATE
#include "block.cuh"

namespace ffspmv {

template FFSPMV_BLOCK_LAUNCH(uint16_t, uint32_t);

}  // namespace ffspmv
