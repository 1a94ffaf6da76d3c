// L2 access-policy window helper (host side), shared by the sequence and
// the block apply.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

namespace ffspmv {

// L2 residency of a gathered operand (the sequence's V_t, the block apply's
// X): its rows are gathered at random about nnz/n times each while the
// packed matrix streams through once.  An access-policy window marks it
// persisting in L2 (hit ratio scaled to the persisting carve-out, whose
// limit is raised to the device maximum) so the matrix stream (evict-first
// loads) and the output stores do not push it out.  The stream's previous
// window is restored when the call has enqueued its launches; lines left
// persisting by an earlier window are reset to normal when a new one starts
// (the reset is immediate, not stream-ordered, so it cannot wait for the
// call's own kernels).  FFSPMV_L2_WINDOW=0 disables it (A/B measurement).
struct L2Window {
    cudaStream_t st;
    bool on = false;
    cudaStreamAttrValue saved{};
    size_t limit = 0;
    L2Window(cudaStream_t s, size_t bytes) : st(s) {
        static int enabled = -1;
        if (enabled < 0) {
            const char *e = getenv("FFSPMV_L2_WINDOW");
            enabled = (e && e[0] == '0') ? 0 : 1;
        }
        int dev = 0, maxp = 0, maxw = 0;
        if (!enabled || bytes == 0 || cudaGetDevice(&dev) ||
            cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) ||
            cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev) || maxp <= 0 || maxw <= 0)
            return;
        if (cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize)) return;
        if (limit < (size_t)maxp && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp)) return;
        if (cudaStreamGetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &saved)) return;
        cudaCtxResetPersistingL2Cache();   // lines a previous window left persisting
        on = true;
        win_bytes = std::min<size_t>(bytes, (size_t)maxw);
        ratio = std::min(1.0f, (float)maxp / (float)win_bytes);
    }
    size_t win_bytes = 0;
    float ratio = 1.0f;
    void set(const void *base) {
        if (!on) return;
        cudaStreamAttrValue v{};
        v.accessPolicyWindow.base_ptr = const_cast<void *>(base);
        v.accessPolicyWindow.num_bytes = win_bytes;
        v.accessPolicyWindow.hitRatio = ratio;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    }
    ~L2Window() {
        if (on) cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &saved);
    }
};


}  // namespace ffspmv
