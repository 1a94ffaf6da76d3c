// u32 block apply entry point (ffspmv_apply_block).
#define FFSPMV_BLOCK_INSTANTIATE
#include "block.cuh"

namespace ffspmv {

template FFSPMV_BLOCK_LAUNCH(uint32_t, uint32_t);

int launch_block(const DevOp &op, const DevMod &M, uint32_t k, uint32_t alpha,
                 const uint32_t *X, uint64_t ldx, uint32_t beta, uint32_t *Y, uint64_t ldy,
                 void *stream) {
    return launch_block_t<uint32_t, uint32_t>(op, M, k, alpha, X, ldx, beta, Y, ldy, stream);
}

}  // namespace ffspmv
