// Block kernels over u8 iterates (the sequence for m <= 256: its unfused
// path and its V_out widening), instantiated here rather than in seq.cu.
#define FFSPMV_BLOCK_INSTANTIATE
#include "block.cuh"

namespace ffspmv {

template FFSPMV_BLOCK_LAUNCH(uint8_t, uint8_t);
template FFSPMV_BLOCK_LAUNCH(uint8_t, uint32_t);

}  // namespace ffspmv
