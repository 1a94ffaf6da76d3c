// C ABI (include/ffspmv.h): argument checks, handle lifecycle, device
// upload, and dispatch to the kernels.  SURVEY §8 row b.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/ffspmv.h"
#include "comm.hpp"
#include "internal.hpp"

using namespace ffspmv;

namespace {

thread_local std::string g_err;

ffspmv_status fail(ffspmv_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

ffspmv_status cuda_fail(int e, const char *where) {
    g_err = std::string(where) + ": " + cudaGetErrorString((cudaError_t)e);
    return FFSPMV_ERR_CUDA;
}

struct DeviceGuard {
    int prev = -1;
    bool changed = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev && dev >= 0) {
            changed = cudaSetDevice(dev) == cudaSuccess;
        }
    }
    ~DeviceGuard() {
        if (changed) cudaSetDevice(prev);
    }
};

struct DevMem {
    void *base = nullptr;
    size_t bytes = 0;
};

bool overlaps(const void *a, size_t an, const void *b, size_t bn) {
    if (!a || !b || !an || !bn) return false;
    uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
    return a0 < b0 + bn && b0 < a0 + an;
}

}  // namespace

namespace ffspmv {
ffspmv_status set_error(ffspmv_status s, const std::string &msg) { return fail(s, msg); }
}  // namespace ffspmv

// State of a distributed handle (rank (i, j) of a P_r x P_c grid).
struct DistState {
    CommImpl *world = nullptr;             // the caller's communicator (not owned)
    CommImpl *group = nullptr;             // ranks of this column block (owned)
    uint32_t nranks = 1, pr = 1, pc = 1, i = 0, j = 0;
    uint64_t n = 0;
    std::vector<uint32_t> bstart;          // P_r + 1 band starts
    uint32_t rows_max = 1;
    void *buf = nullptr;                   // result-exchange buffers (grown on demand)
    size_t buf_bytes = 0;
};

struct ffspmv_matrix_s {
    int device = 0;
    uint32_t m = 0;
    DevMod mod{};
    DevOp op[2]{};         // 0 = A, 1 = A^T: row layout
    bool has_op[2] = {false, false};
    DevMem mem[2];
    DevPanel pan[2]{};     // 0 = A, 1 = A^T: panel layout (k = 1 products)
    bool has_pan[2] = {false, false};
    DevMem pmem[2];
    DevRuns run[2]{};      // 0 = A, 1 = A^T: runs layout (k = 1 products)
    bool has_run[2] = {false, false};
    DevMem rmem[2];
    ffspmv_info info{};
    uint32_t *flag = nullptr;          // checked-mode flag (device)
    uint32_t *stage = nullptr;         // apply_host staging (device)
    unsigned long long *tacc = nullptr; // no-transpose fallback: per-column u64 sums (device)
    size_t stage_elems = 0;
    bool checked = false;              // check_inputs option
    std::mutex mu;
    DistState *dist = nullptr;         // non-NULL: a distributed handle
};

namespace {

inline size_t a256(size_t b) { return (b + 255) & ~(size_t)255; }

// One device allocation per operator; sub-arrays 256 B aligned.
ffspmv_status upload(const HostOp &h, DevOp &d, DevMem &mem) {
    struct Part { const void *src; size_t bytes; void **dst; };
    d = DevOp{};
    d.rows = h.rows;
    d.cols = h.cols;
    d.n_slices = (uint32_t)h.slices.size();
    d.n_long = (uint32_t)h.longs.size();
    d.n_groups = (uint32_t)h.groups.size();
    d.n_split = h.n_split;
    d.n_zero_rows = (uint32_t)h.zero_rows.size();
    d.acc96 = 0;
    for (const SliceHdr &sh : h.slices) d.acc96 |= sh.regime == ACC96;
    void *p_slices, *p_perm, *p_pcol, *p_vcol, *p_vval, *p_longs, *p_groups, *p_crow, *p_cpp,
        *p_cvp, *p_zero, *p_sacc, *p_scnt;
    Part parts[] = {
        {h.slices.data(), h.slices.size() * sizeof(SliceHdr), &p_slices},
        {h.perm.data(), h.perm.size() * 4, &p_perm},
        {h.pcol.data(), h.pcol.size() * 4, &p_pcol},
        {h.vcol.data(), h.vcol.size() * 4, &p_vcol},
        {h.vval.data(), h.vval.size(), &p_vval},
        {h.longs.data(), h.longs.size() * sizeof(LongItem), &p_longs},
        {h.groups.data(), h.groups.size() * sizeof(CsrGroup), &p_groups},
        {h.csr_rows.data(), h.csr_rows.size() * 4, &p_crow},
        {h.csr_pptr.data(), h.csr_pptr.size() * 4, &p_cpp},
        {h.csr_vptr.data(), h.csr_vptr.size() * 4, &p_cvp},
        {h.zero_rows.data(), h.zero_rows.size() * 4, &p_zero},
        {nullptr, (size_t)h.n_split * 8, &p_sacc},
        {nullptr, (size_t)h.n_split * 4, &p_scnt},
    };
    size_t total = 0;
    for (auto &pt : parts) total += a256(pt.bytes);
    total = std::max<size_t>(total, 256);
    int e = cudaMalloc(&mem.base, total);
    if (e) return e == cudaErrorMemoryAllocation ? fail(FFSPMV_ERR_NOMEM, "cudaMalloc of matrix")
                                                 : cuda_fail(e, "cudaMalloc");
    mem.bytes = total;
    size_t off = 0;
    for (auto &pt : parts) {
        *pt.dst = (char *)mem.base + off;
        if (pt.bytes) {
            e = pt.src ? cudaMemcpy(*pt.dst, pt.src, pt.bytes, cudaMemcpyHostToDevice)
                       : cudaMemset(*pt.dst, 0, pt.bytes);
            if (e) { cudaFree(mem.base); mem.base = nullptr; return cuda_fail(e, "matrix upload"); }
        }
        off += a256(pt.bytes);
    }
    d.slices = (const SliceHdr *)p_slices;
    d.perm = (const uint32_t *)p_perm;
    d.pcol = (const uint32_t *)p_pcol;
    d.vcol = (const uint32_t *)p_vcol;
    d.vval = p_vval;
    d.longs = (const LongItem *)p_longs;
    d.groups = (const CsrGroup *)p_groups;
    d.csr_rows = (const uint32_t *)p_crow;
    d.csr_pptr = (const uint32_t *)p_cpp;
    d.csr_vptr = (const uint32_t *)p_cvp;
    d.zero_rows = (const uint32_t *)p_zero;
    d.split_acc = (unsigned long long *)p_sacc;
    d.split_cnt = (uint32_t *)p_scnt;
    return FFSPMV_OK;
}

ffspmv_status upload_panel(const HostPanel &h, DevPanel &d, DevMem &mem) {
    struct Part { const void *src; size_t bytes; void **dst; };
    d = DevPanel{};
    d.rows = h.rows;
    d.cols = h.cols;
    d.g = h.g;
    void *p_tiles, *p_pent, *p_vval, *p_cta, *p_part;
    Part parts[] = {
        {h.tiles.data(), h.tiles.size() * sizeof(PanelTile), &p_tiles},
        {h.pent.data(), h.pent.size() * 4, &p_pent},
        {h.vval.data(), h.vval.size(), &p_vval},
        {h.cta_t0.data(), h.cta_t0.size() * 4, &p_cta},
        {nullptr, (size_t)h.g.P * h.g.rows_pad * h.g.xbytes, &p_part},
    };
    size_t total = 0;
    for (auto &pt : parts) total += a256(pt.bytes);
    total = std::max<size_t>(total, 256);
    int e = cudaMalloc(&mem.base, total);
    if (e) return e == cudaErrorMemoryAllocation ? fail(FFSPMV_ERR_NOMEM, "cudaMalloc of panels")
                                                 : cuda_fail(e, "cudaMalloc");
    mem.bytes = total;
    size_t off = 0;
    for (auto &pt : parts) {
        *pt.dst = (char *)mem.base + off;
        if (pt.bytes && pt.src) {
            e = cudaMemcpy(*pt.dst, pt.src, pt.bytes, cudaMemcpyHostToDevice);
            if (e) { cudaFree(mem.base); mem.base = nullptr; return cuda_fail(e, "panel upload"); }
        }
        off += a256(pt.bytes);
    }
    d.tiles = (const PanelTile *)p_tiles;
    d.pent = (const uint32_t *)p_pent;
    d.vval = p_vval;
    d.cta_t0 = (const uint32_t *)p_cta;
    d.partial = p_part;
    return FFSPMV_OK;
}

ffspmv_status upload_runs(const HostRuns &h, DevRuns &d, DevMem &mem) {
    struct Part { const void *src; size_t bytes; void **dst; };
    d = DevRuns{};
    d.rows = h.rows;
    d.cols = h.cols;
    d.g = h.g;
    void *p_tiles, *p_words, *p_vval, *p_cta, *p_part, *p_xp;
    Part parts[] = {
        {h.tiles.data(), h.tiles.size() * sizeof(RunsTile), &p_tiles},
        {h.words.data(), h.words.size() * 4, &p_words},
        {h.vval.data(), h.vval.size(), &p_vval},
        {h.cta_t0.data(), h.cta_t0.size() * 4, &p_cta},
        {nullptr, (size_t)h.g.P * h.g.rows_pad * h.g.pbytes, &p_part},
        {nullptr, (size_t)h.g.P * h.g.panel_bytes, &p_xp},
    };
    size_t total = 0;
    for (auto &pt : parts) total += a256(pt.bytes);
    total = std::max<size_t>(total, 256);
    int e = cudaMalloc(&mem.base, total);
    if (e) return e == cudaErrorMemoryAllocation ? fail(FFSPMV_ERR_NOMEM, "cudaMalloc of runs")
                                                 : cuda_fail(e, "cudaMalloc");
    mem.bytes = total;
    size_t off = 0;
    for (auto &pt : parts) {
        *pt.dst = (char *)mem.base + off;
        if (pt.bytes) {
            e = pt.src ? cudaMemcpy(*pt.dst, pt.src, pt.bytes, cudaMemcpyHostToDevice)
                       : cudaMemset(*pt.dst, 0, pt.bytes);
            if (e) { cudaFree(mem.base); mem.base = nullptr; return cuda_fail(e, "runs upload"); }
        }
        off += a256(pt.bytes);
    }
    d.tiles = (const RunsTile *)p_tiles;
    d.words = (const uint32_t *)p_words;
    d.vval = p_vval;
    d.cta_t0 = (const uint32_t *)p_cta;
    d.partial = p_part;
    d.xpack = p_xp;
    return FFSPMV_OK;
}

ffspmv_status read_options(const ffspmv_options *o, BuildOptions &bo, int &device, bool &want_t,
                           bool &checked, ffspmv_comm *comm = nullptr, uint32_t *dist_rows = nullptr) {
    device = -1;
    want_t = true;
    checked = false;
    if (comm) *comm = nullptr;
    if (dist_rows) *dist_rows = 0;
    if (!o) return FFSPMV_OK;
    if (o->struct_size >= offsetof(ffspmv_options, dist_rows) + sizeof(o->dist_rows)) {
        if (comm) *comm = o->comm;
        if (dist_rows) *dist_rows = o->dist_rows;
    }
    if (o->struct_size < offsetof(ffspmv_options, strategy))
        return fail(FFSPMV_ERR_INVALID_ARG, "ffspmv_options.struct_size too small");
    device = o->device;
    want_t = o->no_transpose == 0;
    checked = o->check_inputs != 0;
    if (o->segregate_pm1 < -1 || o->segregate_pm1 > 1)
        return fail(FFSPMV_ERR_INVALID_ARG, "segregate_pm1 must be -1, 0 or 1");
    bo.segregate_pm1 = o->segregate_pm1;
    if (o->force_format < 0 || o->force_format > 3)
        return fail(FFSPMV_ERR_INVALID_ARG, "force_format out of range");
    bo.force_format = o->force_format;
    if (o->band_rows) {
        if (o->band_rows % 32) return fail(FFSPMV_ERR_INVALID_ARG, "band_rows must be a multiple of 32");
        bo.band_rows = o->band_rows;
    }
    if (o->long_row) {
        if (o->long_row > 65535) return fail(FFSPMV_ERR_INVALID_ARG, "long_row must be <= 65535");
        bo.long_row = o->long_row;
    }
    if (o->force_acc_bits && o->force_acc_bits != 32 && o->force_acc_bits != 64 &&
        o->force_acc_bits != 96)
        return fail(FFSPMV_ERR_INVALID_ARG, "force_acc_bits must be 0, 32, 64 or 96");
    bo.force_acc_bits = o->force_acc_bits;
    if (o->struct_size >= sizeof(ffspmv_options)) {
        if (o->strategy < 0 || o->strategy > 3)
            return fail(FFSPMV_ERR_INVALID_ARG, "strategy must be 0, 1, 2 or 3");
        bo.strategy = o->strategy;
        if (o->strategy != 3 && o->panel_rows && (o->panel_rows > 32768 || o->panel_rows % 32))
            return fail(FFSPMV_ERR_INVALID_ARG, "panel_rows must be a multiple of 32 <= 32768");
        if (o->panel_cols && (o->panel_cols > 262144 || o->panel_cols % 32))
            return fail(FFSPMV_ERR_INVALID_ARG, "panel_cols must be a multiple of 32 <= 262144");
        bo.panel_rows = o->panel_rows;
        bo.panel_cols = o->panel_cols;
    }
    if (o->struct_size >= offsetof(ffspmv_options, panel_xbits) + sizeof(o->panel_xbits)) {
        if (o->panel_xbits && o->panel_xbits != 2 && o->panel_xbits != 4 && o->panel_xbits != 8 &&
            o->panel_xbits != 16 && o->panel_xbits != 32)
            return fail(FFSPMV_ERR_INVALID_ARG, "panel_xbits must be 0, 2, 4, 8, 16 or 32");
        bo.xbits = o->panel_xbits;
    }
    if (bo.strategy == 3 && bo.panel_rows && (bo.panel_rows % 4 || bo.panel_rows > 16384))
        return fail(FFSPMV_ERR_INVALID_ARG, "runs: panel_rows must be a multiple of 4 <= 16384");
    return FFSPMV_OK;
}

ffspmv_status check_triples_args(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t *ri,
                                 const uint32_t *ci, const int64_t *v, uint32_t m) {
    if (m < 2) return fail(FFSPMV_ERR_MODULUS, "modulus must be >= 2");
    if (rows > 0x7FFFFFFFull || cols > 0x7FFFFFFFull)
        return fail(FFSPMV_ERR_DIM, "rows and cols must be <= 2^31-1");
    if (nnz >= (1ull << 32)) return fail(FFSPMV_ERR_DIM, "nnz must be < 2^32");
    if (nnz && (!ri || !ci || !v)) return fail(FFSPMV_ERR_INVALID_ARG, "NULL triple array");
    return FFSPMV_OK;
}

struct Built {
    HostOp rows[2];
    HostPanel pan[2];
    HostRuns run[2];
    bool has_rows[2] = {false, false};
    bool has_pan[2] = {false, false};
    bool has_run[2] = {false, false};
    double locality = 0;
};

void fill_stats(ffspmv_info &I, const Built &b, uint32_t m) {
    const HostOp &a = b.rows[0];
    I.struct_size = sizeof(ffspmv_info);
    I.modulus = m;
    I.rows = a.rows;
    I.cols = a.cols;
    I.nnz = a.nnz;
    I.nnz_pm1 = a.nnz_pm;
    I.nnz_valued = a.nnz_val;
    I.value_bytes = value_bytes_for(m);
    I.iterate_bytes = m <= 256u ? 1 : m <= 65536u ? 2 : 4;
    I.bands = a.bands;
    I.bands_sell = a.bands_sell;
    I.bands_csr = a.bands_csr;
    I.bands_coos = a.bands_coos;
    I.slices = a.slices.size();
    I.csr_groups = a.groups.size();
    I.long_rows = a.long_rows;
    I.split_rows = a.split_rows;
    I.padded_slots = a.padded_slots;
    I.acc_slices_u32 = a.acc_cnt[0];
    I.acc_slices_u64 = a.acc_cnt[1];
    I.acc_slices_u96 = a.acc_cnt[2];
    I.acc_bits_max = a.acc_bits_max;
    I.stream_bytes = a.stream_bytes;
    uint64_t vb = I.value_bytes;
    I.alg_bytes_apply = 4 * a.nnz_pm + (4 + vb) * a.nnz_val + 4ull * a.cols + 4ull * a.rows;
    bool has_t = b.has_rows[1] || b.has_pan[1] || b.has_run[1];
    if (has_t)
        I.alg_bytes_transpose = 4 * a.nnz_pm + (4 + vb) * a.nnz_val + 4ull * a.cols + 4ull * a.rows;
    I.has_transpose = has_t;
    auto strat = [&](int k) {
        return b.has_run[k] ? FFSPMV_STRATEGY_RUNS : b.has_pan[k] ? FFSPMV_STRATEGY_PANELS
                                                                  : FFSPMV_STRATEGY_ROWS;
    };
    I.strategy_apply = strat(0);
    I.strategy_transpose = !has_t ? 0 : strat(1);
    if (b.has_run[0]) {
        I.panels = b.run[0].g.P;
        I.panel_bands = b.run[0].g.B;
        I.panel_stream_bytes = b.run[0].stream_bytes;
        I.panel_xbits = b.run[0].g.xbits;
    } else if (b.has_pan[0]) {
        I.panels = b.pan[0].g.P;
        I.panel_bands = b.pan[0].g.B;
        I.panel_stream_bytes = b.pan[0].stream_bytes;
        I.panel_xbits = 8 * b.pan[0].g.xbytes;
    }
    I.gather_locality = b.locality;
}

// random columns (little 128 B line reuse) and enough work to fill the SMs:
// x is better staged in shared memory than gathered from L2
bool x_staged(const Canon &c, double loc) { return loc > 0.5 && c.idx.size() >= (1u << 20); }

// PANELS (x staged in shared memory, one shared atomic per entry): the
// default for staged x wider than a byte (m > 256)
bool choose_panels(const Canon &c, uint32_t m, const BuildOptions &bo, double loc) {
    if (bo.strategy == FFSPMV_STRATEGY_PANELS) return true;
    return bo.strategy == FFSPMV_STRATEGY_AUTO && m > 256u && x_staged(c, loc);
}

// RUNS (x staged packed in shared memory, register row runs): the default
// for m <= 256, where x packs to 2-8 bits and few panels cover the columns
bool choose_runs(const Canon &c, uint32_t m, const BuildOptions &bo, double loc) {
    if (bo.strategy == FFSPMV_STRATEGY_RUNS) return true;
    return bo.strategy == FFSPMV_STRATEGY_AUTO && m <= 256u && x_staged(c, loc);
}

// the k = 1 layout of one operator (A or A^T): RUNS, PANELS or ROWS
void pack_k1(Built &out, int k, const Canon &c, uint32_t m, const BuildOptions &bo, uint32_t nsm,
             double loc, bool need_rows) {
    if (choose_runs(c, m, bo, loc) && pack_runs(out.run[k], c, m, bo, nsm)) {
        out.has_run[k] = true;
    } else {
        out.run[k] = HostRuns();
        if (choose_panels(c, m, bo, loc) && pack_panels(out.pan[k], c, m, bo, nsm)) {
            out.has_pan[k] = true;
        } else {
            out.pan[k] = HostPanel();
            need_rows = true;
        }
    }
    if (need_rows && !out.has_rows[k]) {
        pack_operator(out.rows[k], c, m, bo);
        out.has_rows[k] = true;
    }
}

ffspmv_status build_host(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t *ri,
                         const uint32_t *ci, const int64_t *v, uint32_t m, const BuildOptions &bo,
                         bool want_t, uint32_t nsm, Built &out) {
    Canon ca;
    std::string err;
    int rc;
    try {
        rc = canonicalize(ca, rows, cols, nnz, ri, ci, v, m, err);
    } catch (const std::bad_alloc &) {
        return fail(FFSPMV_ERR_NOMEM, "host allocation during canonicalisation");
    }
    if (rc) return fail((ffspmv_status)rc, err);
    try {
        out.locality = gather_locality(ca);
        // block apply + sequence always use the rows layout of A
        pack_k1(out, 0, ca, m, bo, nsm, out.locality, true);
        if (want_t) {
            Canon ct;
            transpose_canon(ct, ca);
            ca = Canon();
            pack_k1(out, 1, ct, m, bo, nsm, gather_locality(ct), false);
        }
    } catch (const std::bad_alloc &) {
        return fail(FFSPMV_ERR_NOMEM, "host allocation during packing");
    }
    for (int k = 0; k < 2; ++k)
        if (out.rows[k].pcol.size() >= (1ull << 32) || out.rows[k].vcol.size() >= (1ull << 32) ||
            out.pan[k].pent.size() >= (1ull << 32) || out.run[k].words.size() >= (1ull << 32))
            return fail(FFSPMV_ERR_DIM, "packed streams exceed 2^32 slots");
    return FFSPMV_OK;
}

// nnz-balanced contiguous row bands: b[0] = 0 <= ... <= b[P] = rows, b[r] =
// the first row with at least r / P of the entries before it (the same
// partition on every rank: it depends on the matrix only)
std::vector<uint32_t> row_bands(const Canon &c, uint32_t P) {
    std::vector<uint32_t> b(P + 1, 0);
    const uint64_t total = c.ptr.back();
    for (uint32_t r = 1; r < P; ++r) {
        const double target = (double)total * r / P;
        b[r] = (uint32_t)(std::lower_bound(c.ptr.begin(), c.ptr.end(), (uint64_t)std::ceil(target)) - c.ptr.begin());
        b[r] = std::max(b[r - 1], std::min<uint32_t>(b[r], (uint32_t)c.nrows));
    }
    b[P] = (uint32_t)c.nrows;
    return b;
}

uint32_t device_sms(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0)
        n = 148;
    return (uint32_t)n;
}

}  // namespace

ffspmv_status create_dist(ffspmv_matrix *out, uint64_t rows, uint64_t cols, uint64_t nnz,
                          const uint32_t *row_idx, const uint32_t *col_idx, const int64_t *vals,
                          uint32_t modulus, BuildOptions bo, int device, bool checked, ffspmv_comm comm,
                          uint32_t dist_rows, std::chrono::steady_clock::time_point t0) {
    CommImpl *world = comm_impl(comm);
    if (!world) return fail(FFSPMV_ERR_INVALID_ARG, "invalid communicator");
    if (rows != cols) return fail(FFSPMV_ERR_NONSQUARE, "a distributed handle needs a square matrix");
    const uint32_t nranks = (uint32_t)comm_size(world), rank = (uint32_t)comm_rank(world);
    const uint32_t pr = dist_rows ? dist_rows : nranks;
    if (pr < 1 || nranks % pr) return fail(FFSPMV_ERR_INVALID_ARG, "dist_rows must divide the rank count");
    const uint32_t pc = nranks / pr, bi = rank / pc, bj = rank % pc;
    int e;
    if (device < 0 && (e = cudaGetDevice(&device))) return cuda_fail(e, "cudaGetDevice");
    DeviceGuard guard(device);
    Canon ca;
    std::string err;
    try {
        if (int rc = canonicalize(ca, rows, cols, nnz, row_idx, col_idx, vals, modulus, err))
            return fail((ffspmv_status)rc, err);
    } catch (const std::bad_alloc &) {
        return fail(FFSPMV_ERR_NOMEM, "host allocation during canonicalisation");
    }
    auto *ds = new DistState();
    ds->world = world;
    ds->nranks = nranks;
    ds->pr = pr;
    ds->pc = pc;
    ds->i = bi;
    ds->j = bj;
    ds->n = rows;
    ds->bstart = row_bands(ca, pr);
    uint32_t rmax = 1;
    for (uint32_t r = 0; r < pr; ++r) rmax = std::max(rmax, ds->bstart[r + 1] - ds->bstart[r]);
    ds->rows_max = rmax;
    if ((uint64_t)pr * rmax >= 0x7FFFFFFFull) { delete ds; return fail(FFSPMV_ERR_DIM, "padded iterate too tall"); }
    // band i, columns renumbered into the padded iterate layout
    Canon cb;
    const uint32_t b0 = ds->bstart[bi], b1 = ds->bstart[bi + 1];
    cb.nrows = b1 - b0;
    cb.ncols = (uint64_t)pr * rmax;
    cb.ptr.assign(cb.nrows + 1, 0);
    try {
        const uint64_t e0 = ca.ptr[b0], e1 = ca.ptr[b1];
        cb.idx.resize(e1 - e0);
        cb.val.assign(ca.val.begin() + e0, ca.val.begin() + e1);
        for (uint32_t r = 0; r < cb.nrows; ++r) cb.ptr[r + 1] = ca.ptr[b0 + r + 1] - e0;
        for (uint64_t t = e0; t < e1; ++t) {
            const uint32_t c = ca.idx[t];
            const uint32_t q = (uint32_t)(std::upper_bound(ds->bstart.begin(), ds->bstart.end(), c) -
                                          ds->bstart.begin()) - 1;
            cb.idx[t - e0] = q * rmax + (c - ds->bstart[q]);
        }
        ca = Canon();
        Built B;
        pack_operator(B.rows[0], cb, modulus, bo);
        B.has_rows[0] = true;
        ffspmv_matrix h = new (std::nothrow) ffspmv_matrix_s();
        if (!h) { delete ds; return fail(FFSPMV_ERR_NOMEM, "handle allocation"); }
        h->device = device;
        h->m = modulus;
        h->mod = make_mod(modulus);
        h->dist = ds;
        ffspmv_status s;
        if ((s = upload(B.rows[0], h->op[0], h->mem[0]))) { delete ds; delete h; return s; }
        h->has_op[0] = true;
        if ((e = cudaMalloc((void **)&h->flag, 256))) {
            cudaFree(h->mem[0].base);
            delete ds;
            delete h;
            return cuda_fail(e, "cudaMalloc flag");
        }
        fill_stats(h->info, B, modulus);
        h->info.rows = rows;
        h->info.cols = cols;
        h->info.nnz_input = nnz;
        h->info.dist_ranks = nranks;
        h->info.dist_grid_rows = pr;
        h->info.dist_band_row0 = b0;
        h->info.dist_band_rows = b1 - b0;
        h->info.has_transpose = 0;
        h->info.device_bytes = h->mem[0].bytes + 256;
        h->checked = checked;
        // the column-block communicator: ranks (., j), ordered by band
        ds->group = comm_split(world, (int)bj, (int)bi, (int)pr, (int)bi, err);
        if (!ds->group) {
            ffspmv_destroy(h);
            return fail(FFSPMV_ERR_NCCL, err);
        }
        h->info.create_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = h;
        return FFSPMV_OK;
    } catch (const std::bad_alloc &) {
        delete ds;
        return fail(FFSPMV_ERR_NOMEM, "host allocation while packing the band");
    }
}

extern "C" {

ffspmv_status ffspmv_create(ffspmv_matrix *out, uint64_t rows, uint64_t cols, uint64_t nnz,
                            const uint32_t *row_idx, const uint32_t *col_idx, const int64_t *vals,
                            uint32_t modulus, const ffspmv_options *opts) {
    auto t0 = std::chrono::steady_clock::now();
    if (!out) return fail(FFSPMV_ERR_INVALID_ARG, "out is NULL");
    ffspmv_status s = check_triples_args(rows, cols, nnz, row_idx, col_idx, vals, modulus);
    if (s) return s;
    BuildOptions bo;
    int device;
    bool want_t, checked;
    ffspmv_comm comm = nullptr;
    uint32_t dist_rows = 0;
    if ((s = read_options(opts, bo, device, want_t, checked, &comm, &dist_rows))) return s;
    if (comm) return create_dist(out, rows, cols, nnz, row_idx, col_idx, vals, modulus, bo, device, checked,
                                 comm, dist_rows, t0);
    if (device < 0) {
        int e = cudaGetDevice(&device);
        if (e) return cuda_fail(e, "cudaGetDevice");
    }
    int ndev = 0;
    int e = cudaGetDeviceCount(&ndev);
    if (e) return cuda_fail(e, "cudaGetDeviceCount");
    if (device >= ndev) return fail(FFSPMV_ERR_INVALID_ARG, "device ordinal out of range");
    DeviceGuard guard(device);

    Built B;
    if ((s = build_host(rows, cols, nnz, row_idx, col_idx, vals, modulus, bo, want_t,
                        device_sms(device), B)))
        return s;
    ffspmv_matrix h = new (std::nothrow) ffspmv_matrix_s();
    if (!h) return fail(FFSPMV_ERR_NOMEM, "handle allocation");
    h->device = device;
    h->m = modulus;
    h->mod = make_mod(modulus);
    auto cleanup = [&]() {
        for (int k = 0; k < 2; ++k) {
            if (h->mem[k].base) cudaFree(h->mem[k].base);
            if (h->pmem[k].base) cudaFree(h->pmem[k].base);
            if (h->rmem[k].base) cudaFree(h->rmem[k].base);
        }
        if (h->flag) cudaFree(h->flag);
        delete h;
    };
    for (int k = 0; k < 2; ++k) {
        if (B.has_rows[k]) {
            if ((s = upload(B.rows[k], h->op[k], h->mem[k]))) { cleanup(); return s; }
            h->has_op[k] = true;
        }
        if (B.has_pan[k]) {
            if ((s = upload_panel(B.pan[k], h->pan[k], h->pmem[k]))) { cleanup(); return s; }
            h->has_pan[k] = true;
        }
        if (B.has_run[k]) {
            if ((s = upload_runs(B.run[k], h->run[k], h->rmem[k]))) { cleanup(); return s; }
            h->has_run[k] = true;
        }
    }
    if ((e = cudaMalloc((void **)&h->flag, 256))) {
        cleanup();
        return cuda_fail(e, "cudaMalloc flag");
    }
    if (!want_t) {
        // the transpose fallback's column sums
        if ((e = cudaMalloc((void **)&h->tacc, std::max<uint64_t>(cols, 1) * 8)) ||
            (e = cudaMemset(h->tacc, 0, std::max<uint64_t>(cols, 1) * 8))) {
            if (h->tacc) cudaFree(h->tacc);
            cleanup();
            return cuda_fail(e, "cudaMalloc transpose scratch");
        }
    }
    fill_stats(h->info, B, modulus);
    h->info.nnz_input = nnz;
    h->info.device_bytes = h->mem[0].bytes + h->mem[1].bytes + h->pmem[0].bytes + h->pmem[1].bytes +
                           h->rmem[0].bytes + h->rmem[1].bytes + 256 + (h->tacc ? std::max<uint64_t>(cols, 1) * 8 : 0);
    h->info.has_transpose = 1;   // built, or the scatter fallback
    h->info.create_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    h->checked = checked;
    *out = h;
    return FFSPMV_OK;
}

ffspmv_status ffspmv_destroy(ffspmv_matrix A) {
    if (!A) return fail(FFSPMV_ERR_INVALID_ARG, "NULL handle");
    DeviceGuard guard(A->device);
    for (auto &mem : A->mem)
        if (mem.base) cudaFree(mem.base);
    for (auto &mem : A->pmem)
        if (mem.base) cudaFree(mem.base);
    for (auto &mem : A->rmem)
        if (mem.base) cudaFree(mem.base);
    if (A->flag) cudaFree(A->flag);
    if (A->stage) cudaFree(A->stage);
    if (A->tacc) cudaFree(A->tacc);
    if (A->dist) {
        if (A->dist->buf) cudaFree(A->dist->buf);
        comm_free(A->dist->group);
        delete A->dist;
    }
    delete A;
    return FFSPMV_OK;
}

ffspmv_status ffspmv_get_info(ffspmv_matrix A, ffspmv_info *out) {
    if (!A || !out) return fail(FFSPMV_ERR_INVALID_ARG, "NULL argument");
    *out = A->info;
    return FFSPMV_OK;
}

ffspmv_status ffspmv_analyze(uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t *row_idx,
                             const uint32_t *col_idx, const int64_t *vals, uint32_t modulus,
                             const ffspmv_options *opts, ffspmv_info *info, int transpose,
                             uint32_t *rec_row, uint32_t *rec_col, uint32_t *rec_val,
                             uint64_t rec_cap, uint64_t *rec_n) {
    auto t0 = std::chrono::steady_clock::now();
    ffspmv_status s = check_triples_args(rows, cols, nnz, row_idx, col_idx, vals, modulus);
    if (s) return s;
    BuildOptions bo;
    int device;
    bool want_t, checked;
    if ((s = read_options(opts, bo, device, want_t, checked))) return s;
    if (transpose) want_t = true;
    Built B;
    if ((s = build_host(rows, cols, nnz, row_idx, col_idx, vals, modulus, bo, want_t, 148, B)))
        return s;
    if (info) {
        ffspmv_info I{};
        fill_stats(I, B, modulus);
        I.nnz_input = nnz;
        I.create_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *info = I;
    }
    if (rec_row || rec_col || rec_val) {
        if (!rec_row || !rec_col || !rec_val || !rec_n)
            return fail(FFSPMV_ERR_INVALID_ARG, "reconstruction needs all of rec_row/col/val/n");
        const int k = transpose ? 1 : 0;
        const uint32_t vb = value_bytes_for(modulus);
        uint64_t n = B.has_run[k]   ? reconstruct_runs(B.run[k], modulus, vb, rec_row, rec_col, rec_val, rec_cap)
                     : B.has_pan[k] ? reconstruct_panels(B.pan[k], modulus, vb, rec_row, rec_col, rec_val, rec_cap)
                                    : reconstruct(B.rows[k], modulus, vb, rec_row, rec_col, rec_val, rec_cap);
        *rec_n = n;
        if (n > rec_cap) return fail(FFSPMV_ERR_NOMEM, "reconstruction capacity too small");
    }
    return FFSPMV_OK;
}

}  // extern "C"

namespace {

void op_dims(ffspmv_matrix A, int which, uint64_t &rows, uint64_t &cols) {
    if (A->has_run[which]) { rows = A->run[which].rows; cols = A->run[which].cols; }
    else if (A->has_pan[which]) { rows = A->pan[which].rows; cols = A->pan[which].cols; }
    else { rows = A->op[which].rows; cols = A->op[which].cols; }
}

ffspmv_status check_vec(ffspmv_matrix A, const uint32_t *v, uint64_t n, uint64_t ld, uint64_t w,
                        void *stream, const char *name) {
    if (!A->checked || !n || !w) return FFSPMV_OK;
    int e = cudaMemsetAsync(A->flag, 0, 4, (cudaStream_t)stream);
    if (!e) e = launch_check_canonical(v, n, ld, w, A->m, A->flag, stream);
    uint32_t h = 0;
    if (!e) e = cudaMemcpyAsync(&h, A->flag, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (!e) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e) return cuda_fail(e, "check_inputs");
    if (h) return fail(FFSPMV_ERR_INVALID_ARG, std::string(name) + " has an entry >= m");
    return FFSPMV_OK;
}

ffspmv_status no_dist(ffspmv_matrix A) {
    return fail(FFSPMV_ERR_UNSUPPORTED,
                "a distributed handle supports ffspmv_sequence, ffspmv_apply and ffspmv_apply_block only");
}

// Grow the handle's result-exchange buffer (calls on a distributed handle do
// not overlap).
ffspmv_status dist_buf(DistState &d, size_t want) {
    if (want <= d.buf_bytes) return FFSPMV_OK;
    if (d.buf) cudaFree(d.buf);
    d.buf = nullptr;
    d.buf_bytes = 0;
    if (int e = cudaMalloc(&d.buf, want)) return cuda_fail(e, "cudaMalloc exchange buffers");
    d.buf_bytes = want;
    return FFSPMV_OK;
}

// Row-sharded single product on a distributed handle (SURVEY §8e "single
// apply / block apply shard naturally"): rank (i, j) computes
// Y[band i, block j] = alpha A[band i, :] X[:, block j] + beta Y[...] in place
// in the caller's Y (X scattered once into the band operator's padded column
// layout), then every rank's block is all-gathered and written into Y, so Y
// (replicated, n x k contiguous) is identical on every rank and equal to the
// one-GPU result.  k = 1 is ffspmv_apply.
ffspmv_status block_dist(ffspmv_matrix A, uint32_t k, uint32_t alpha, const uint32_t *X, uint32_t beta,
                         uint32_t *Y, void *stream) {
    DistState &d = *A->dist;
    const DevOp &op = A->op[0];
    const uint32_t c0 = (uint32_t)((uint64_t)k * d.j / d.pc);
    const uint32_t kc = (uint32_t)((uint64_t)k * (d.j + 1) / d.pc) - c0;
    const uint32_t kcmax = (k + d.pc - 1) / d.pc;
    const uint64_t npad = op.cols, h = op.rows, row0 = d.bstart[d.i];
    alpha %= A->m;
    beta %= A->m;
    ffspmv_status s;
    if ((s = check_vec(A, X, d.n, k, k, stream, "X"))) return s;
    if (beta && (s = check_vec(A, Y, d.n, k, k, stream, "Y"))) return s;
    const size_t xb = a256(npad * kcmax * 4ull), vslot = (size_t)d.rows_max * kcmax * 4;
    if ((s = dist_buf(d, xb + a256(vslot) + a256(vslot * d.nranks) + a256(4 * (d.pr + 1))))) return s;
    uint32_t *Xp = (uint32_t *)d.buf;
    uint32_t *Vb = (uint32_t *)((char *)d.buf + xb);
    uint32_t *Gv = (uint32_t *)((char *)Vb + a256(vslot));
    uint32_t *bdev = (uint32_t *)((char *)Gv + a256(vslot * d.nranks));
    cudaStream_t st = (cudaStream_t)stream;
    int e;
    if ((e = cudaMemcpyAsync(bdev, d.bstart.data(), 4ull * (d.pr + 1), cudaMemcpyHostToDevice, st)))
        return cuda_fail(e, "band starts");
    if (kc) {
        if ((e = launch_dist_prep_x(X, k, c0, kc, npad, d.rows_max, bdev, Xp, stream)))
            return cuda_fail(e, "scatter X");
        if (h && (e = launch_block(op, A->mod, kc, alpha, Xp, kc, beta, Y + row0 * k + c0, k, stream)))
            return cuda_fail(e, "band block apply");
        // packed with the block's own width (k_dist_put_V's slot layout)
        if (h && (e = cudaMemcpy2DAsync(Vb, kc * 4ull, Y + row0 * k + c0, k * 4ull, kc * 4ull, h,
                                        cudaMemcpyDeviceToDevice, st)))
            return cuda_fail(e, "pack band block");
    }
    std::string err;
    if ((e = comm_allgather(d.world, Vb, Gv, vslot, stream, err)))
        return fail(e < 0 ? FFSPMV_ERR_NCCL : FFSPMV_ERR_CUDA, err);
    if ((e = launch_dist_put_V(Gv, d.n, k, kcmax, d.rows_max, d.pr, d.pc, bdev, Y, stream)))
        return cuda_fail(e, "assemble Y");
    return FFSPMV_OK;
}

ffspmv_status apply_op(ffspmv_matrix A, int which, uint32_t alpha, const uint32_t *x, uint64_t nx,
                       uint32_t beta, uint32_t *y, uint64_t ny, void *stream) {
    if (!A) return fail(FFSPMV_ERR_INVALID_ARG, "NULL handle");
    if (A->dist) {
        if (which != 0) return no_dist(A);
        if (nx != A->dist->n || ny != A->dist->n)
            return fail(FFSPMV_ERR_DIM, "x and y must have " + std::to_string(A->dist->n) + " entries");
        if (A->dist->n && (!x || !y)) return fail(FFSPMV_ERR_INVALID_ARG, "NULL vector");
        if (overlaps(x, nx * 4, y, ny * 4)) return fail(FFSPMV_ERR_INVALID_ARG, "x overlaps y");
        DeviceGuard guard(A->device);
        return block_dist(A, 1, alpha, x, beta, y, stream);
    }
    const bool scatter = which == 1 && !A->has_op[1] && !A->has_pan[1] && !A->has_run[1];
    if (scatter && !A->tacc) return fail(FFSPMV_ERR_UNSUPPORTED, "transpose not available");
    uint64_t orows, ocols;
    if (scatter) { orows = A->op[0].cols; ocols = A->op[0].rows; }
    else op_dims(A, which, orows, ocols);
    if (nx != ocols || ny != orows)
        return fail(FFSPMV_ERR_DIM, "x must have " + std::to_string(ocols) + " and y " +
                                        std::to_string(orows) + " entries");
    if ((nx && !x) || (ny && !y)) return fail(FFSPMV_ERR_INVALID_ARG, "NULL vector");
    if (overlaps(x, nx * 4, y, ny * 4)) return fail(FFSPMV_ERR_INVALID_ARG, "x overlaps y");
    alpha %= A->m;
    beta %= A->m;
    DeviceGuard guard(A->device);
    ffspmv_status s;
    if ((s = check_vec(A, x, nx, 1, 1, stream, "x"))) return s;
    if (beta && (s = check_vec(A, y, ny, 1, 1, stream, "y"))) return s;
    int e = scatter             ? launch_apply_scatter_t(A->op[0], A->mod, alpha, x, beta, y, A->tacc, stream)
            : A->has_run[which] ? launch_runs_apply(A->run[which], A->mod, alpha, x, beta, y, stream)
            : A->has_pan[which] ? launch_panel_apply(A->pan[which], A->mod, alpha, x, beta, y, stream)
                                : launch_apply(A->op[which], A->mod, alpha, x, beta, y, stream);
    if (e) return cuda_fail(e, "apply launch");
    return FFSPMV_OK;
}

// in-place all-gather of the band iterates among the ranks of a column block
int dist_exchange(void *ctx, void *buf, size_t bytes, void *stream) {
    DistState *d = (DistState *)ctx;
    std::string err;
    const int e = comm_allgather(d->group, (char *)buf + (size_t)d->i * bytes, buf, bytes, stream, err);
    if (e) fail(e < 0 ? FFSPMV_ERR_NCCL : FFSPMV_ERR_CUDA, err);
    return e;
}

ffspmv_status dist_status(int e, const char *where) {
    if (e < 0) return FFSPMV_ERR_NCCL;          // message already recorded
    return cuda_fail(e, where);
}

ffspmv_status sequence_dist(ffspmv_matrix A, uint32_t k, const uint32_t *X, uint32_t ku, const uint32_t *U,
                            uint64_t L, uint32_t *S, uint32_t *V_out, void *workspace, size_t workspace_bytes,
                            void *stream) {
    DistState &d = *A->dist;
    const DevOp &op = A->op[0];
    const uint32_t c0 = (uint32_t)((uint64_t)k * d.j / d.pc);
    const uint32_t kc = (uint32_t)((uint64_t)k * (d.j + 1) / d.pc) - c0;
    const uint32_t kcmax = (k + d.pc - 1) / d.pc;
    const size_t need = sequence_dist_workspace(op, A->mod, std::max<uint32_t>(kc, 1), ku, d.pr);
    if (!workspace || workspace_bytes < need)
        return fail(FFSPMV_ERR_NOMEM, "workspace smaller than ffspmv_workspace_size (" + std::to_string(need) +
                                          " bytes)");
    ffspmv_status s;
    if ((s = check_vec(A, X, d.n, k, k, stream, "X"))) return s;
    if (U && (s = check_vec(A, U, d.n, ku, ku, stream, "U"))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    int e;
    if (L == 0) {
        if (V_out && d.n && (e = cudaMemcpyAsync(V_out, X, d.n * k * 4ull, cudaMemcpyDeviceToDevice, st)))
            return cuda_fail(e, "copy V_out");
        return FFSPMV_OK;
    }
    // exchange buffers: band residues T (one slot), all slots G, band V_L
    // block Vb and all blocks Gv, the band starts on the device
    const size_t tslot = (size_t)L * ku * kcmax * 4, vslot = (size_t)d.rows_max * kcmax * 4;
    const size_t want = tslot * (1 + d.nranks) + (V_out ? vslot * (1 + d.nranks) : 0) + 4 * (d.pr + 1) + 4096;
    if (want > d.buf_bytes) {
        if (d.buf) cudaFree(d.buf);
        d.buf = nullptr;
        d.buf_bytes = 0;
        if ((e = cudaMalloc(&d.buf, want))) return cuda_fail(e, "cudaMalloc exchange buffers");
        d.buf_bytes = want;
    }
    char *p = (char *)d.buf;
    uint32_t *T = (uint32_t *)p;
    uint32_t *G = (uint32_t *)(p + a256(tslot));
    uint32_t *bdev = (uint32_t *)(p + a256(tslot) + a256(tslot * d.nranks));
    uint32_t *Vb = (uint32_t *)((char *)bdev + a256(4 * (d.pr + 1)));
    uint32_t *Gv = (uint32_t *)((char *)Vb + a256(vslot));
    if (kc) {
        DistSeq ds;
        ds.pr = d.pr;
        ds.rows_max = d.rows_max;
        ds.bstart = d.bstart.data();
        ds.row0 = d.bstart[d.i];
        ds.own = (uint64_t)d.i * d.rows_max;
        ds.c0 = c0;
        ds.kc = kc;
        ds.exchange = dist_exchange;
        ds.ctx = &d;
        e = launch_sequence_dist(op, A->mod, X, k, ku, U, L, T, V_out ? Vb : nullptr, workspace, ds, stream);
        if (e) return dist_status(e, "distributed sequence");
    }
    std::string err;
    if ((e = comm_allgather(d.world, T, G, tslot, stream, err))) return fail(e < 0 ? FFSPMV_ERR_NCCL : FFSPMV_ERR_CUDA, err);
    if ((e = launch_dist_sum_S(G, L, ku, k, kcmax, d.pr, d.pc, A->mod, S, stream))) return cuda_fail(e, "sum S");
    if (V_out) {
        if ((e = cudaMemcpyAsync(bdev, d.bstart.data(), 4ull * (d.pr + 1), cudaMemcpyHostToDevice, st)))
            return cuda_fail(e, "band starts");
        if ((e = comm_allgather(d.world, Vb, Gv, vslot, stream, err)))
            return fail(e < 0 ? FFSPMV_ERR_NCCL : FFSPMV_ERR_CUDA, err);
        if ((e = launch_dist_put_V(Gv, d.n, k, kcmax, d.rows_max, d.pr, d.pc, bdev, V_out, stream)))
            return cuda_fail(e, "assemble V_out");
    }
    return FFSPMV_OK;
}

}  // namespace

extern "C" {

ffspmv_status ffspmv_apply(ffspmv_matrix A, uint32_t alpha, const uint32_t *x, uint64_t nx,
                           uint32_t beta, uint32_t *y, uint64_t ny, void *stream) {
    return apply_op(A, 0, alpha, x, nx, beta, y, ny, stream);
}

ffspmv_status ffspmv_apply_transpose(ffspmv_matrix A, uint32_t alpha, const uint32_t *x,
                                     uint64_t nx, uint32_t beta, uint32_t *y, uint64_t ny,
                                     void *stream) {
    return apply_op(A, 1, alpha, x, nx, beta, y, ny, stream);
}

ffspmv_status ffspmv_apply_block(ffspmv_matrix A, uint32_t k, uint32_t alpha, const uint32_t *X,
                                 uint64_t ldx, uint32_t beta, uint32_t *Y, uint64_t ldy,
                                 void *stream) {
    if (!A) return fail(FFSPMV_ERR_INVALID_ARG, "NULL handle");
    if (k == 0) return fail(FFSPMV_ERR_INVALID_ARG, "k must be >= 1");
    if (ldx < k || ldy < k) return fail(FFSPMV_ERR_INVALID_ARG, "leading dimension < k");
    if (A->dist) {
        const uint64_t n = A->dist->n;
        if (ldx != k || ldy != k)
            return fail(FFSPMV_ERR_UNSUPPORTED, "a distributed block apply needs ldx = ldy = k");
        if (n && (!X || !Y)) return fail(FFSPMV_ERR_INVALID_ARG, "NULL block");
        if (overlaps(X, n * k * 4, Y, n * k * 4)) return fail(FFSPMV_ERR_INVALID_ARG, "X overlaps Y");
        if (n * k >= (1ull << 32)) return fail(FFSPMV_ERR_DIM, "n * k must be < 2^32 elements");
        DeviceGuard guard(A->device);
        return block_dist(A, k, alpha, X, beta, Y, stream);
    }
    const DevOp &op = A->op[0];
    if ((op.cols && !X) || (op.rows && !Y)) return fail(FFSPMV_ERR_INVALID_ARG, "NULL block");
    if (overlaps(X, op.cols * ldx * 4, Y, op.rows * ldy * 4))
        return fail(FFSPMV_ERR_INVALID_ARG, "X overlaps Y");
    if ((uint64_t)op.cols * ldx >= (1ull << 32))
        return fail(FFSPMV_ERR_DIM, "cols * ldx must be < 2^32 elements");
    alpha %= A->m;
    beta %= A->m;
    DeviceGuard guard(A->device);
    ffspmv_status s;
    if ((s = check_vec(A, X, op.cols, ldx, k, stream, "X"))) return s;
    if (beta && (s = check_vec(A, Y, op.rows, ldy, k, stream, "Y"))) return s;
    // (an L2 persisting window over X was measured slower here: c4 k = 8
    // 0.115 -> 0.150 ms with L2 flushed between calls)
    int e = launch_block(op, A->mod, k, alpha, X, ldx, beta, Y, ldy, stream);
    if (e) return cuda_fail(e, "block launch");
    return FFSPMV_OK;
}

ffspmv_status ffspmv_apply_host(ffspmv_matrix A, int which, uint32_t alpha, const uint32_t *x_host,
                                uint32_t beta, uint32_t *y_host, void *stream) {
    if (!A) return fail(FFSPMV_ERR_INVALID_ARG, "NULL handle");
    if (A->dist) return no_dist(A);
    if (which != FFSPMV_OP_APPLY && which != FFSPMV_OP_TRANSPOSE)
        return fail(FFSPMV_ERR_INVALID_ARG, "op must be FFSPMV_OP_APPLY or FFSPMV_OP_TRANSPOSE");
    const bool scatter = which == 1 && !A->has_op[1] && !A->has_pan[1] && !A->has_run[1];
    struct { uint64_t rows, cols; } op{};
    if (scatter) { op.rows = A->op[0].cols; op.cols = A->op[0].rows; }
    else op_dims(A, which, op.rows, op.cols);
    if ((op.cols && !x_host) || (op.rows && !y_host))
        return fail(FFSPMV_ERR_INVALID_ARG, "NULL host vector");
    std::lock_guard<std::mutex> lk(A->mu);
    DeviceGuard guard(A->device);
    size_t need = (size_t)op.cols + op.rows;
    int e;
    if (need > A->stage_elems) {
        if (A->stage) cudaFree(A->stage);
        A->stage = nullptr;
        A->stage_elems = 0;
        if ((e = cudaMalloc((void **)&A->stage, std::max<size_t>(need, 1) * 4)))
            return cuda_fail(e, "cudaMalloc staging");
        A->stage_elems = need;
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t *dx = A->stage, *dy = A->stage + op.cols;
    uint32_t b = beta % A->m;
    if (op.cols && (e = cudaMemcpyAsync(dx, x_host, op.cols * 4ull, cudaMemcpyHostToDevice, st)))
        return cuda_fail(e, "copy x");
    if (b && op.rows && (e = cudaMemcpyAsync(dy, y_host, op.rows * 4ull, cudaMemcpyHostToDevice, st)))
        return cuda_fail(e, "copy y");
    ffspmv_status s = apply_op(A, which, alpha, dx, op.cols, beta, dy, op.rows, stream);
    if (s) return s;
    if (op.rows && (e = cudaMemcpyAsync(y_host, dy, op.rows * 4ull, cudaMemcpyDeviceToHost, st)))
        return cuda_fail(e, "copy y back");
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "synchronize");
    return FFSPMV_OK;
}

ffspmv_status ffspmv_workspace_size(ffspmv_matrix A, int which, uint32_t k, uint32_t ku,
                                    size_t *bytes) {
    if (!A || !bytes) return fail(FFSPMV_ERR_INVALID_ARG, "NULL argument");
    if (which == FFSPMV_OP_PROJECT) {
        if (k == 0 || ku == 0) return fail(FFSPMV_ERR_INVALID_ARG, "k and ku must be >= 1");
        DeviceGuard guard(A->device);
        *bytes = project_workspace(A->op[0].rows, k, ku);
        return FFSPMV_OK;
    }
    if (which != FFSPMV_OP_SEQUENCE) { *bytes = 0; return FFSPMV_OK; }
    if (k == 0) return fail(FFSPMV_ERR_INVALID_ARG, "k must be >= 1");
    if (ku == 0) ku = k;
    DeviceGuard guard(A->device);
    if (A->dist) {
        const DistState &d = *A->dist;
        const uint32_t kc = (uint32_t)((uint64_t)k * (d.j + 1) / d.pc - (uint64_t)k * d.j / d.pc);
        *bytes = sequence_dist_workspace(A->op[0], A->mod, std::max<uint32_t>(kc, 1), ku, d.pr);
        return FFSPMV_OK;
    }
    *bytes = sequence_workspace(A->op[0], A->mod, k, ku);
    return FFSPMV_OK;
}

ffspmv_status ffspmv_sequence(ffspmv_matrix A, uint32_t k, const uint32_t *X, uint32_t ku,
                              const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out,
                              void *workspace, size_t workspace_bytes, void *stream) {
    if (!A) return fail(FFSPMV_ERR_INVALID_ARG, "NULL handle");
    const DevOp &op = A->op[0];
    if (!A->dist && op.rows != op.cols) return fail(FFSPMV_ERR_NONSQUARE, "sequence needs a square matrix");
    if (k == 0) return fail(FFSPMV_ERR_INVALID_ARG, "k must be >= 1");
    if (!U) {
        if (ku != 0 && ku != k) return fail(FFSPMV_ERR_INVALID_ARG, "U == NULL requires ku == k");
        ku = k;
    } else if (ku == 0) {
        return fail(FFSPMV_ERR_INVALID_ARG, "ku must be >= 1");
    }
    const uint64_t n = A->dist ? A->dist->n : op.rows;
    // the step kernels index the iterate with 32-bit element offsets
    if (n * k >= (1ull << 32) || n * ku >= (1ull << 32))
        return fail(FFSPMV_ERR_DIM, "n * k and n * ku must be < 2^32 elements");
    if (n && !X) return fail(FFSPMV_ERR_INVALID_ARG, "NULL X");
    if (L && !S) return fail(FFSPMV_ERR_INVALID_ARG, "NULL S");
    if (overlaps(S, L * ku * k * 4ull, X, n * k * 4ull) ||
        overlaps(V_out, n * k * 4ull, X, n * k * 4ull) ||
        overlaps(V_out, n * k * 4ull, S, L * ku * k * 4ull) ||
        overlaps(S, L * ku * k * 4ull, U, n * ku * 4ull))
        return fail(FFSPMV_ERR_INVALID_ARG, "S / V_out overlap an input");
    DeviceGuard guard(A->device);
    if (A->dist) return sequence_dist(A, k, X, ku, U, L, S, V_out, workspace, workspace_bytes, stream);
    size_t need = sequence_workspace(op, A->mod, k, ku);
    if (n && (!workspace || workspace_bytes < need))
        return fail(FFSPMV_ERR_NOMEM, "workspace smaller than ffspmv_workspace_size (" +
                                          std::to_string(need) + " bytes)");
    ffspmv_status s;
    if ((s = check_vec(A, X, n, k, k, stream, "X"))) return s;
    if (U && (s = check_vec(A, U, n, ku, ku, stream, "U"))) return s;
    if (n == 0) {
        if (L && (S)) {
            int e = cudaMemsetAsync(S, 0, L * ku * k * 4ull, (cudaStream_t)stream);
            if (e) return cuda_fail(e, "memset S");
        }
        return FFSPMV_OK;
    }
    int e = launch_sequence(op, A->mod, k, X, ku, U, L, S, V_out, workspace, workspace_bytes, stream);
    if (e) return cuda_fail(e, "sequence launch");
    return FFSPMV_OK;
}

ffspmv_status ffspmv_project(ffspmv_matrix A, uint32_t k, const uint32_t *V, uint32_t ku,
                             const uint32_t *U, uint32_t *S, void *workspace,
                             size_t workspace_bytes, void *stream) {
    if (!A) return fail(FFSPMV_ERR_INVALID_ARG, "NULL handle");
    if (A->dist) return no_dist(A);
    if (k == 0 || ku == 0) return fail(FFSPMV_ERR_INVALID_ARG, "k and ku must be >= 1");
    const uint64_t n = A->op[0].rows;
    if ((n && (!V || !U)) || !S) return fail(FFSPMV_ERR_INVALID_ARG, "NULL V, U or S");
    if (overlaps(S, (size_t)ku * k * 4, V, n * k * 4) || overlaps(S, (size_t)ku * k * 4, U, n * ku * 4))
        return fail(FFSPMV_ERR_INVALID_ARG, "S overlaps an input");
    DeviceGuard guard(A->device);
    const size_t need = project_workspace(n, k, ku);
    if (n && (!workspace || workspace_bytes < need))
        return fail(FFSPMV_ERR_NOMEM, "workspace smaller than ffspmv_workspace_size (" +
                                          std::to_string(need) + " bytes)");
    ffspmv_status s;
    if ((s = check_vec(A, V, n, k, k, stream, "V"))) return s;
    if ((s = check_vec(A, U, n, ku, ku, stream, "U"))) return s;
    int e = launch_project(A->mod, n, k, V, ku, U, S, workspace, stream);
    if (e) return cuda_fail(e, "project launch");
    return FFSPMV_OK;
}

ffspmv_status ffspmv_sum_mod(ffspmv_matrix A, uint64_t count, uint32_t nparts,
                             const uint32_t *parts, uint32_t *out, void *stream) {
    if (!A) return fail(FFSPMV_ERR_INVALID_ARG, "NULL handle");
    if (count && (!parts || !out || nparts == 0))
        return fail(FFSPMV_ERR_INVALID_ARG, "NULL parts/out or nparts == 0");
    DeviceGuard guard(A->device);
    int e = launch_sum_mod(A->mod, count, nparts, parts, out, stream);
    if (e) return cuda_fail(e, "sum_mod launch");
    return FFSPMV_OK;
}

const char *ffspmv_status_string(ffspmv_status s) {
    switch (s) {
        case FFSPMV_OK: return "FFSPMV_OK";
        case FFSPMV_ERR_INVALID_ARG: return "FFSPMV_ERR_INVALID_ARG";
        case FFSPMV_ERR_MODULUS: return "FFSPMV_ERR_MODULUS";
        case FFSPMV_ERR_INDEX: return "FFSPMV_ERR_INDEX";
        case FFSPMV_ERR_DIM: return "FFSPMV_ERR_DIM";
        case FFSPMV_ERR_NONSQUARE: return "FFSPMV_ERR_NONSQUARE";
        case FFSPMV_ERR_UNSUPPORTED: return "FFSPMV_ERR_UNSUPPORTED";
        case FFSPMV_ERR_NOMEM: return "FFSPMV_ERR_NOMEM";
        case FFSPMV_ERR_CUDA: return "FFSPMV_ERR_CUDA";
        case FFSPMV_ERR_NCCL: return "FFSPMV_ERR_NCCL";
    }
    return "FFSPMV_ERR_UNKNOWN";
}

const char *ffspmv_last_error(void) { return g_err.c_str(); }

int ffspmv_version(void) { return 100; }

uint64_t ffspmv_kernel_launches(void) { return kernel_launch_count(); }

}  // extern "C"
