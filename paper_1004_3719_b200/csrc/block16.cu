// Block kernels over u16 iterates (the sequence's unfused path and its
// V_out widening), instantiated here rather than in seq.cu.
#define FFSPMV_BLOCK_INSTANTIATE
#include "block.cuh"

namespace ffspmv {

template FFSPMV_BLOCK_LAUNCH(uint16_t, uint16_t);

}  // namespace ffspmv
