// Internal layout shared by the host builder (builder.cpp), the C ABI
// (abi.cpp) and the CUDA kernels (kernels.cu).  Nothing here is part of the
// public ABI (include/ffspmv.h).  See DESIGN.md §"Data layout in HBM".
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace ffspmv {

// A slot whose column is PAD_COL contributes nothing (ELL padding).
// Valid columns are < 2^31 - 1, so the sentinel never collides.
constexpr uint32_t PAD_COL = 0x7FFFFFFFu;
// dynamic shared memory a k_panel CTA may use (227 KB opt-in maximum)
constexpr uint64_t PANEL_SMEM_MAX = 232448;
// Bit 31 of an index-only (+-1) slot is the sign: set = "-1".
constexpr uint32_t SIGN_BIT = 0x80000000u;
constexpr uint32_t COL_MASK = 0x7FFFFFFFu;
constexpr uint32_t PAD_ROW = 0xFFFFFFFFu;
constexpr uint32_t NO_SPLIT = 0xFFFFFFFFu;

// Accumulator width (P:129-147 delayed reduction with integer carriers).
enum Regime : uint8_t { ACC32 = 0, ACC64 = 1, ACC96 = 2 };

// One 32-row slice of a SELL band.  Slot j of lane l lives at
// off + j*32 + l in its stream (column-major inside the slice).
struct SliceHdr {
    uint32_t off_p;   // element offset of the +-1 stream slots
    uint32_t off_v;   // element offset of the valued stream slots (cols + vals)
    uint16_t wp;      // +-1 slots per lane
    uint16_t wv;      // valued slots per lane
    uint8_t regime;   // Regime
    uint8_t nrows;    // live lanes (rows) in the slice
    uint16_t band;    // band index (diagnostics)
};
static_assert(sizeof(SliceHdr) == 16, "SliceHdr is 16 bytes");

// A long row (or one chunk of a split long row) of the COO/CSR tail.
// Chunks of one row are consecutive in the long-item array.
struct LongItem {
    uint32_t row;
    uint32_t off_p, len_p;   // +-1 entries of this chunk
    uint32_t off_v, len_v;   // valued entries of this chunk
    uint32_t split;          // NO_SPLIT, or index of the split-row scratch cell
    uint32_t chunk;          // chunk index inside the row
    uint32_t nch_reg;        // nchunks | regime << 28 (regime of one lane's share)
};
static_assert(sizeof(LongItem) == 32, "LongItem is 32 bytes");

// A warp's worth of rows of a CSR-vector or COO_S band: V = 1 << vlog lanes
// per row, 32 >> vlog rows per warp pass.  Rows are listed in csr_rows
// (natural order for CSR, non-empty rows only for COO_S); listed row i owns
// +-1 entries [csr_pptr[i], csr_pptr[i+1]) and valued entries
// [csr_vptr[i], csr_vptr[i+1]).
struct CsrGroup {
    uint32_t first;   // index of the first listed row
    uint16_t nrows;   // listed rows in this group (<= 32)
    uint8_t vlog;     // log2 lanes per row
    uint8_t regime;
    uint32_t band;
    uint32_t pad_;
};
static_assert(sizeof(CsrGroup) == 16, "CsrGroup is 16 bytes");

// Modulus constants for Barrett reduction of u64 / u96 sums.
struct DevMod {
    uint32_t m;
    uint32_t vbytes;     // bytes per stored value (1, 2, 4)
    uint64_t mu;         // floor(2^64 / m)
    uint64_t r64;        // 2^64 mod m
    uint32_t mu32;       // floor(2^32 / m) (used when m <= 2^16)
    uint32_t r32;        // 2^32 mod m
};

// Device view of one packed operator (A or A^T).
struct DevOp {
    uint32_t rows, cols;
    uint32_t n_slices, n_long, n_groups, n_split;
    uint32_t n_zero_rows;          // rows of COO_S bands with no entries
    uint32_t acc96;                // 1: some SELL slice needs the u96 regime
    const SliceHdr *slices;
    const uint32_t *perm;          // slice lane -> row (PAD_ROW for dead lanes)
    const uint32_t *pcol;          // +-1 stream: col | sign, PAD_COL pads
    const uint32_t *vcol;          // valued stream: col, PAD_COL pads
    const void *vval;              // values (vbytes each), 0 for pads
    const LongItem *longs;
    const CsrGroup *groups;
    const uint32_t *csr_rows, *csr_pptr, *csr_vptr;
    const uint32_t *zero_rows;     // rows written as beta*y only
    unsigned long long *split_acc; // per split row: sum of chunk residues
    uint32_t *split_cnt;           // per split row: chunks arrived
};

// Host-side packed operator.
struct HostOp {
    uint32_t rows = 0, cols = 0;
    std::vector<SliceHdr> slices;
    std::vector<uint32_t> perm;
    std::vector<uint32_t> pcol, vcol;
    std::vector<uint8_t> vval;       // vbytes per element
    std::vector<LongItem> longs;
    uint32_t n_split = 0;
    std::vector<CsrGroup> groups;
    std::vector<uint32_t> csr_rows, csr_pptr, csr_vptr;
    std::vector<uint32_t> zero_rows;
    // statistics
    uint64_t nnz = 0, nnz_pm = 0, nnz_val = 0;
    uint32_t bands = 0, bands_sell = 0, bands_csr = 0, bands_coos = 0;
    uint64_t long_rows = 0, split_rows = 0, padded_slots = 0;
    uint32_t acc_cnt[3] = {0, 0, 0};
    uint32_t acc_bits_max = 32;
    uint64_t stream_bytes = 0;
};

struct BuildOptions {
    int segregate_pm1 = 0;     // 0 auto, 1 on, -1 off
    int force_format = 0;
    uint32_t band_rows = 4096;
    uint32_t long_row = 512;
    uint32_t split_chunk = 1u << 14;
    int force_acc_bits = 0;
    int strategy = 0;          // 0 auto, 1 rows (x gathered from L2), 2 panels (x in smem),
                               // 3 runs (packed x in smem, register row runs)
    uint32_t panel_rows = 0;   // 0 = default R (testing: smaller tiles)
    uint32_t panel_cols = 0;   // 0 = default W (testing: smaller panels)
    uint32_t xbits = 0;        // runs: 0 = narrowest for m; else forced (2/4/8/16/32, >= need)
};

// ------------------------------------------------------------------ panels --
// 2-D tiled operator for k = 1 (apply / transpose): the columns are cut into
// panels of W columns whose slice of x is staged in shared memory (the paper's
// column-wise split of A, with x staged on chip); the rows into
// bands of R rows whose accumulators live in shared memory.  Tile t = p*B + b
// holds the entries of panel p x band b in three sections -- +1 entries, -1
// entries, valued entries -- each padded to a multiple of 4 ("quads") with a
// dummy word that adds into the spare accumulator R.  An entry is one u32:
// the byte offset of its column in the staged x panel, (col - p*W) * xbytes,
// in bits [rs, 32), and its band row, row - b*R, in bits [0, rs); rs = 14 /
// 15 / 14 for x staged as u8 / u16 / u32 (W = 196608 / 65536 / 49152 columns
// = 192 / 128 / 192 KB of shared memory, R = 4088 / 8160 / 2200 band rows of
// u32 accumulators, one band per thread group of the kernel, two groups).  A
// tile writes one residue per band row into partial[p][row] (row stride rows_pad, a multiple of 16); a reduction pass
// sums the P partials of each row (Fig. 2 "foreach submatrix Ai in A do
// spmv(y, Ai, x); reduce(y, m)").
struct Canon;

struct PanelGeom {
    uint32_t W = 0, R = 0, P = 0, B = 0;
    uint32_t xbytes = 4;       // bytes per staged x element (1, 2, 4)
    uint32_t split = 0;        // 1: accumulate residues as two u32 halves (m > 65536)
    uint32_t nctas = 0;        // persistent CTAs (one per SM)
    uint32_t rs = 14;          // row bits of the packed word
    uint32_t lazy = 0;         // 1: valued products enter the sum as Barrett remainders < 2m
    uint32_t rows_pad = 0;     // partial row stride (rows rounded up to 16)
};

// One tile: quads [q0, q0 + nqp) are +1 entries, the next nqm quads -1
// entries, the next nqv quads valued entries whose values are value quads
// [vq0, vq0 + nqv).  p, b: panel and band; rn: live band rows.
struct PanelTile {
    uint32_t q0, nqp, nqm, nqv, vq0, p, b, rn;
};
static_assert(sizeof(PanelTile) == 32, "PanelTile is 32 bytes");

struct HostPanel {
    uint32_t rows = 0, cols = 0;
    PanelGeom g;
    std::vector<PanelTile> tiles;      // P*B tiles, panel-major
    std::vector<uint32_t> pent;        // packed entries, 4 per quad
    std::vector<uint8_t> vval;         // values of the valued quads (4 * vbytes per quad)
    std::vector<uint32_t> cta_t0;      // nctas + 1 tile boundaries
    uint64_t nnz_pm = 0, nnz_val = 0, stream_bytes = 0;
};

struct DevPanel {
    uint32_t rows, cols;
    PanelGeom g;
    const PanelTile *tiles;
    const uint32_t *pent, *cta_t0;
    const void *vval;
    void *partial;                     // P * rows_pad * xbytes scratch
};

// Chooses W, R, element widths for modulus m.
PanelGeom panel_geometry(uint64_t rows, uint64_t cols, uint32_t m, const BuildOptions &bo,
                         uint32_t nsm);
// false when a tile row's sum could overflow its u32 accumulator (the caller
// then keeps the rows layout).
bool pack_panels(HostPanel &hp, const Canon &a, uint32_t m, const BuildOptions &bo, uint32_t nsm);
uint64_t reconstruct_panels(const HostPanel &hp, uint32_t m, uint32_t vbytes, uint32_t *rr,
                            uint32_t *rc, uint32_t *rv, uint64_t cap);
// Column-locality of the rows layout: distinct 128 B x lines touched per
// 256-row band divided by nonzeros (1 = no reuse, random columns).
double gather_locality(const Canon &a);
int launch_panel_apply(const DevPanel &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                       uint32_t beta, uint32_t *y, void *stream);

// -------------------------------------------------------------------- runs --
// Second 2-D tiled operator for k = 1 (FFSPMV_STRATEGY_RUNS).  Same tiling
// idea as PANELS (the column-wise split of P:290-295: column panel p x row
// band, x panel staged in shared memory, one residue per band row per panel
// summed by a reduction pass, Fig. 2), but:
//   * the x panel is staged PACKED (xbits = 2 / 4 / 8 / 16 / 32 bits per
//     residue): a pre-pass packs x once per call and each CTA copies its
//     panel with bulk-async copies;
//   * a unit (panel p x an R-row band, unit u = p * B + b) holds three
//     sections, +1, -1 and valued entries, each sorted by row and
//     cut into chunks of 32 lanes x RUN_E consecutive entries, so a lane sums
//     a run of one row in a register and touches shared memory only when its
//     row changes;
//   * every warp owns private band accumulators and takes whole units, so no
//     CTA barrier separates units.
//
// Entry word: byte offset of the 32-bit word of the staged panel holding the
// column's residue in bits [5 + rs, 32), the band row in bits [5, 5 + rs), the
// residue's bit offset inside that word in bits [0, 5).  Chunk c of a section
// holds entries [256 c, 256 c + 256) (RUN_E = 8): entry 8 l + j goes to lane
// l, slot j, at word 256 c + 128 (j / 4) + 4 l + (j % 4) (two coalesced
// 16-byte loads per lane) and, for values, at 256 c + 8 l + j.  Padding
// entries point at the zero word past the panel (byte offset panel_bytes).
// RUN_E and RUN_WARPS: measured on c3 (tools/time_apply.py, A/B builds of
// tools/build_variant_flags.sh): 24 warps x 8 entries per lane (72 regs) at
// 72.7 us beat 32 x 8 (74.8), 16 x 8 (78.9) and 24 x 16 (76.8, spills).
#ifndef FFSPMV_RUN_E
#define FFSPMV_RUN_E 8
#endif
#ifndef FFSPMV_RUN_WARPS
#define FFSPMV_RUN_WARPS 24
#endif
constexpr uint32_t RUN_E = FFSPMV_RUN_E;
constexpr uint32_t RUN_CHUNK = 32 * RUN_E;
constexpr uint32_t RUN_WARPS = FFSPMV_RUN_WARPS;   // warps per k_runs CTA, each with private band accumulators

struct RunsGeom {
    uint32_t W = 0, R = 0, P = 0, B = 0;
    uint32_t xbits = 32;       // bits per staged x residue (2, 4, 8, 16, 32)
    uint32_t wide = 0;         // 1: m > 2^16 (u64 run sums, split u32 band accumulators)
    uint32_t pbytes = 4;       // bytes per partial residue (1, 2, 4)
    uint32_t rs = 9;           // row bits of the entry word (R <= 2^rs)
    uint32_t nctas = 0;        // persistent CTAs (one per SM)
    uint32_t panel_bytes = 0;  // bytes of one packed x panel (multiple of 16)
    uint32_t rows_pad = 0;     // partial row stride (rows rounded up to 16)
};

// One unit: chunks [c0, c0 + npc) of +1 entries, the next nmc chunks of -1
// entries, the next nvc chunks of valued entries whose values are value
// chunks [vc0, vc0 + nvc); rn: live band rows.  Units are panel-major: unit
// u covers panel u / B and band u % B.
struct RunsTile {
    uint32_t c0, npc, nmc, nvc, vc0, rn, pad0, pad1;
};
static_assert(sizeof(RunsTile) == 32, "RunsTile is 32 bytes");

struct HostRuns {
    uint32_t rows = 0, cols = 0;
    RunsGeom g;
    std::vector<RunsTile> tiles;       // P*B tiles, panel-major
    std::vector<uint32_t> words;       // RUN_CHUNK words per chunk
    std::vector<uint8_t> vval;         // RUN_CHUNK values (vbytes each) per value chunk
    std::vector<uint32_t> cta_t0;      // nctas + 1 tile boundaries
    uint64_t nnz_pm = 0, nnz_val = 0, stream_bytes = 0;
};

struct DevRuns {
    uint32_t rows, cols;
    RunsGeom g;
    const RunsTile *tiles;
    const uint32_t *words, *cta_t0;
    const void *vval;
    void *partial;                     // P * rows_pad * pbytes scratch
    void *xpack;                       // P * panel_bytes scratch (packed x)
};

RunsGeom runs_geometry(uint64_t rows, uint64_t cols, uint64_t nnz, uint32_t m,
                       const BuildOptions &bo, uint32_t nsm);
// false when a band row's u32 accumulator could overflow (m <= 2^16; the
// caller then keeps another layout)
bool pack_runs(HostRuns &hr, const Canon &a, uint32_t m, const BuildOptions &bo, uint32_t nsm);
uint64_t reconstruct_runs(const HostRuns &hr, uint32_t m, uint32_t vbytes, uint32_t *rr,
                          uint32_t *rc, uint32_t *rv, uint64_t cap);
int launch_runs_apply(const DevRuns &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                      uint32_t beta, uint32_t *y, void *stream);

// Canonical CSR: rows sorted by column, duplicates summed mod m, zeros dropped.
struct Canon {
    uint64_t nrows = 0, ncols = 0;
    std::vector<uint64_t> ptr;
    std::vector<uint32_t> idx;
    std::vector<uint32_t> val;   // residues in [1, m-1]
};

// builder.cpp
int canonicalize(Canon &out, uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t *ri,
                 const uint32_t *ci, const int64_t *v, uint32_t m, std::string &err);
void transpose_canon(Canon &out, const Canon &a);
void pack_operator(HostOp &op, const Canon &a, uint32_t m, const BuildOptions &bo);
uint64_t reconstruct(const HostOp &op, uint32_t m, uint32_t vbytes, uint32_t *rr, uint32_t *rc,
                     uint32_t *rv, uint64_t cap);
uint32_t value_bytes_for(uint32_t m);
DevMod make_mod(uint32_t m);

// kernels.cu launchers (return cudaError_t as int)
int launch_apply(const DevOp &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                 uint32_t beta, uint32_t *y, void *stream);
int launch_block(const DevOp &op, const DevMod &M, uint32_t k, uint32_t alpha,
                 const uint32_t *X, uint64_t ldx, uint32_t beta, uint32_t *Y, uint64_t ldy,
                 void *stream);
size_t sequence_workspace(const DevOp &op, const DevMod &M, uint32_t k, uint32_t ku);
size_t project_workspace(uint64_t n, uint32_t k, uint32_t ku);
int launch_project(const DevMod &M, uint64_t n, uint32_t k, const uint32_t *V, uint32_t ku,
                   const uint32_t *U, uint32_t *S, void *ws, void *stream);
int launch_sum_mod(const DevMod &M, uint64_t count, uint32_t nparts, const uint32_t *parts,
                   uint32_t *out, void *stream);
int launch_sequence(const DevOp &op, const DevMod &M, uint32_t k, const uint32_t *X,
                    uint32_t ku, const uint32_t *U, uint64_t L, uint32_t *S, uint32_t *V_out,
                    void *ws, size_t ws_bytes, void *stream);
int launch_check_canonical(const uint32_t *v, uint64_t n, uint64_t ld, uint64_t w, uint32_t m,
                           uint32_t *flag_dev, void *stream);
// y <- alpha A^T x + beta y by scattering the rows layout of A into acc (cols
// u64, zero on entry, cleared again on exit) -- the no-transpose fallback
int launch_apply_scatter_t(const DevOp &op, const DevMod &M, uint32_t alpha, const uint32_t *x,
                           uint32_t beta, uint32_t *y, unsigned long long *acc, void *stream);

// distributed sequence (seq.cu): rank (i, j) of a P_r x P_c grid
struct DistSeq {
    uint32_t pr, rows_max;         // row bands, rows of a padded band slot
    const uint32_t *bstart;        // HOST: P_r + 1 band starts
    uint64_t row0;                 // first row of this rank's band
    uint64_t own;                  // this rank's slot: i * rows_max
    uint32_t c0, kc;               // this rank's column block of X
    // in-place all-gather of buf (P_r slots of bytes_per_rank) among the P_r
    // ranks of this column block, on stream (0 or a cudaError_t / -1 for NCCL)
    int (*exchange)(void *ctx, void *buf, size_t bytes_per_rank, void *stream);
    void *ctx;
};
size_t sequence_dist_workspace(const DevOp &op, const DevMod &M, uint32_t kc, uint32_t ku, uint32_t pr);
int launch_sequence_dist(const DevOp &op, const DevMod &M, const uint32_t *X, uint32_t k, uint32_t ku,
                         const uint32_t *U, uint64_t L, uint32_t *S_band, uint32_t *V_band, void *ws,
                         const DistSeq &d, void *stream);
int launch_dist_sum_S(const uint32_t *G, uint64_t L, uint32_t ku, uint32_t k, uint32_t kcmax, uint32_t pr,
                      uint32_t pc, const DevMod &M, uint32_t *S, void *stream);
// X (n x k, caller layout) -> columns [c0, c0 + kc) in the padded band layout
int launch_dist_prep_x(const uint32_t *X, uint32_t k, uint32_t c0, uint32_t kc, uint64_t npad,
                       uint32_t rows_max, const uint32_t *bstart_dev, uint32_t *Xp, void *stream);
int launch_dist_put_V(const uint32_t *Gv, uint64_t n, uint32_t k, uint32_t kcmax, uint32_t rows_max,
                      uint32_t pr, uint32_t pc, const uint32_t *bstart_dev, uint32_t *V_out, void *stream);
uint64_t kernel_launch_count();

}  // namespace ffspmv
