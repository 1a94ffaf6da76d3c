/*
 * ffspmv.h — C ABI of the B200-native exact sparse hot path of
 * Boyer, Dumas & Giorgi, "Exact Sparse Matrix-Vector Multiplication on GPU's
 * and Multicore Architectures" (arXiv:1004.3719).  "P:n" cites line n of the
 * paper text; DESIGN.md lists every reading taken
 * where the paper is silent.
 *
 * The ring is Z/mZ with 2 <= m <= 2^32-1 and canonical representatives
 * [0, m-1] ("m smaller than a machine word"; "we represent the
 * ring on [0, m-1]").  Every vector/block element crossing this boundary is a
 * uint32_t in [0, m-1].  Arithmetic is exact: every result is the unique
 * residue, bit-identical whatever format, band size, accumulator width,
 * stream or GPU count is used.
 *
 * Memory / ownership conventions (all entry points):
 *   - Pointers named *_host are host memory; every other vector/block/S
 *     pointer is DEVICE memory owned by the caller (e.g. a torch tensor's
 *     data_ptr()), on the device the matrix was created on.
 *   - ffspmv_create copies what it needs; the caller may free the triples
 *     on return.  The handle owns its device memory; ffspmv_destroy frees it.
 *   - Compute calls are asynchronous on the caller's stream (a cudaStream_t
 *     passed as void*; NULL = the legacy default stream).  Argument errors
 *     return immediately; device faults surface at the caller's next sync.
 *   - A handle is immutable after create: calls on distinct outputs may run
 *     concurrently, except that apply / apply_transpose use an internal
 *     scratch when the operator uses PANELS (info.strategy_* == PANELS) or has
 *     split rows (info.split_rows > 0): those calls on one handle must then be
 *     ordered on one stream.
 *   - On error a status is returned (never an abort), out-parameters are
 *     untouched, and ffspmv_last_error() holds a thread-local message.
 */
#ifndef FFSPMV_H
#define FFSPMV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FFSPMV_API __attribute__((visibility("default")))
#else
#define FFSPMV_API
#endif

typedef enum {
    FFSPMV_OK = 0,
    FFSPMV_ERR_INVALID_ARG = 1, /* NULL pointer, k == 0, bad option, x aliases y,
                                   non-canonical input in checked mode            */
    FFSPMV_ERR_MODULUS = 2,     /* m < 2                                          */
    FFSPMV_ERR_INDEX = 3,       /* a triple has row >= rows or col >= cols        */
    FFSPMV_ERR_DIM = 4,         /* vector length disagrees with A; rows or cols
                                   > 2^31-1; nnz >= 2^32                          */
    FFSPMV_ERR_NONSQUARE = 5,   /* ffspmv_sequence on a rows != cols matrix       */
    FFSPMV_ERR_UNSUPPORTED = 6, /* operation not available for this handle (a
                                   distributed handle runs ffspmv_sequence only)  */
    FFSPMV_ERR_NOMEM = 7,       /* host or device allocation failed / workspace
                                   smaller than ffspmv_workspace_size            */
    FFSPMV_ERR_CUDA = 8,        /* a CUDA runtime call failed (no device, ...)    */
    FFSPMV_ERR_NCCL = 9         /* a collective failed                            */
} ffspmv_status;

/* Opaque matrix handle: A (and by default A^T) packed on one device. */
typedef struct ffspmv_matrix_s *ffspmv_matrix;

/* Opaque communicator of the distributed sequence (one rank per GPU over
 * NCCL, or an in-process group for testing): see ffspmv_comm_create. */
typedef struct ffspmv_comm_s *ffspmv_comm;

/* Band formats (§2.4.4-2.4.5).  AUTO lets the per-band chooser
 * pick the format that moves the fewest HBM bytes. */
enum {
    FFSPMV_FMT_AUTO = 0,
    FFSPMV_FMT_SELL = 1, /* sliced ELL_R: 32-row slices, column-major slots, rows
                            sorted by length inside the band */
    FFSPMV_FMT_CSR = 2,  /* CSR-vector: V lanes per row, natural order
                            (Bell's vector approach)           */
    FFSPMV_FMT_COOS = 3  /* COO_S: CSR-vector over the non-empty rows only
                                                                      */
};

/* Layout of the k = 1 products (apply, apply_transpose).  ROWS: the band
 * formats above, x gathered from L2 per nonzero.  PANELS and RUNS: A cut
 * into column panels x row bands (the column-wise split of P:290-295); each
 * tile stages its slice of x in shared memory and accumulates its band rows
 * there, and the panels' partial residues are summed per row (Fig. 2,
 * P:210-222).  PANELS adds every entry into a shared accumulator; RUNS stages
 * x packed (2/4/8/16/32 bits per residue), sorts each tile by row so a lane
 * sums runs of one row in registers, and lets the last panel of a band write
 * y.  AUTO picks RUNS when the columns show little locality (random gathers
 * would be L2-bound), else ROWS.  Block apply and the sequence use ROWS. */
enum { FFSPMV_STRATEGY_AUTO = 0, FFSPMV_STRATEGY_ROWS = 1, FFSPMV_STRATEGY_PANELS = 2,
       FFSPMV_STRATEGY_RUNS = 3 };

/* Operation selectors for ffspmv_apply_host / ffspmv_workspace_size. */
enum { FFSPMV_OP_APPLY = 0, FFSPMV_OP_TRANSPOSE = 1, FFSPMV_OP_BLOCK = 2, FFSPMV_OP_SEQUENCE = 3,
       FFSPMV_OP_PROJECT = 4 };

/* Creation options.  A zero-initialised struct (with struct_size set) means
 * "all defaults". */
typedef struct {
    uint32_t struct_size;    /* sizeof(ffspmv_options)                            */
    int32_t device;          /* CUDA device ordinal; -1 or 0.. ; default: current */
    int32_t no_transpose;    /* 1: do not store A^T: apply_transpose then scatters
                                the rows of A into per-column u64 sums with
                                global atomics ("A and A^T cannot be
                                simultaneously stored")                          */
    int32_t segregate_pm1;   /* 0 auto (default), 1 always, -1 never: the +-1
                                index-only stream of P:272-288 ("the user can
                                indicate if she wants to try and make use of
                                +-1")                                      */
    int32_t force_format;    /* FFSPMV_FMT_*: the format to fill "in priority"
                                (P:333); AUTO = chooser                          */
    uint32_t band_rows;      /* rows per band (unit of format choice), multiple
                                of 32; 0 = default 4096                           */
    uint32_t long_row;       /* rows with more nonzeros go to the long-row tail;
                                0 = default 512                                   */
    int32_t force_acc_bits;  /* 0 auto; 32/64/96 = lower bound on the accumulator
                                width (testing: results must not change)         */
    int32_t check_inputs;    /* 1: apply/sequence verify that x / X / U / y are
                                canonical (one extra pass + sync per call)       */
    int32_t strategy;        /* apply / apply_transpose layout: FFSPMV_STRATEGY_* */
    uint32_t panel_rows;     /* PANELS / RUNS: rows per band, 0 = default (testing) */
    uint32_t panel_cols;     /* PANELS / RUNS: columns per panel, 0 = default      */
    uint32_t panel_xbits;    /* RUNS: bits per staged x residue, 0 = narrowest for
                                m; 2, 4, 8, 16, 32 (results must not change)     */
    ffspmv_comm comm;        /* non-NULL: a DISTRIBUTED handle (see below)        */
    uint32_t dist_rows;      /* distributed: P_r, the row bands of the P_r x P_c
                                grid (P_c = ranks / P_r); 0 = all ranks (ROWS)   */
} ffspmv_options;

/* Summary of a built (or analysed) matrix. */
typedef struct {
    uint32_t struct_size;
    uint32_t modulus;
    uint64_t rows, cols;
    uint64_t nnz_input;       /* triples given                                    */
    uint64_t nnz;             /* canonical nonzeros (duplicates summed, zeros
                                 dropped)                                         */
    uint64_t nnz_pm1;         /* entries +-1 carried in the index-only stream     */
    uint64_t nnz_valued;      /* entries carried with a value                     */
    uint32_t value_bytes;     /* 1, 2 or 4 bytes per stored value                 */
    uint32_t iterate_bytes;   /* bytes per element of the sequence iterate        */
    uint32_t bands, bands_sell, bands_csr, bands_coos;
    uint64_t slices;          /* 32-row SELL slices                               */
    uint64_t csr_groups;      /* CSR / COO_S warp groups                          */
    uint64_t long_rows;       /* rows in the long-row tail                        */
    uint64_t split_rows;      /* long rows split over several warps               */
    uint64_t padded_slots;    /* stored slots incl. padding (both streams)        */
    uint32_t acc_slices_u32, acc_slices_u64, acc_slices_u96;
    uint32_t acc_bits_max;
    uint64_t device_bytes;    /* device memory owned by the handle                */
    uint64_t stream_bytes;    /* bytes of the packed A read by one apply          */
    uint64_t alg_bytes_apply; /* algorithmic bytes of y <- Ax:
                                 4 nnz_pm1 + (4 + value_bytes) nnz_valued
                                 + 4 cols + 4 rows                                */
    uint64_t alg_bytes_transpose;
    uint32_t has_transpose;
    double create_seconds;
    uint32_t strategy_apply;      /* FFSPMV_STRATEGY_ROWS or _PANELS actually used */
    uint32_t strategy_transpose;
    uint32_t panels, panel_bands; /* P and B of the apply operator (PANELS / RUNS) */
    uint64_t panel_stream_bytes;  /* packed bytes read by one PANELS / RUNS apply  */
    double gather_locality;       /* distinct 128 B x lines / nonzeros (sampled)   */
    uint32_t panel_xbits;         /* bits per staged x residue (PANELS / RUNS)     */
    uint32_t dist_ranks;          /* distributed handle: ranks (else 0)            */
    uint32_t dist_grid_rows;      /* P_r of the P_r x P_c grid                     */
    uint64_t dist_band_row0;      /* first row of this rank's band                 */
    uint64_t dist_band_rows;      /* rows of this rank's band                      */
} ffspmv_info;

/* --- lifecycle ------------------------------------------------------------ */

/* Build A from COO triples, on the device, for modulus m.
 * row_idx/col_idx/vals are HOST arrays of length nnz, 0-based; values are
 * signed and reduced to their Euclidean residue.  Duplicates are
 * summed mod m and zero residues dropped (R3, R4).  Steps (SURVEY
 * §8 a-1..a-4): canonicalise, split +-1 into an index-only stream,
 * per-band format choice, accumulator width per slice from m and
 * the row weights.
 * Errors: INVALID_ARG (out NULL, nnz > 0 with NULL arrays, bad options),
 * MODULUS (m < 2), INDEX, DIM (rows/cols > 2^31-1, nnz >= 2^32), NOMEM, CUDA. */
FFSPMV_API ffspmv_status ffspmv_create(ffspmv_matrix *out, uint64_t rows, uint64_t cols,
                                       uint64_t nnz, const uint32_t *row_idx,
                                       const uint32_t *col_idx, const int64_t *vals,
                                       uint32_t modulus, const ffspmv_options *opts);

FFSPMV_API ffspmv_status ffspmv_destroy(ffspmv_matrix A);

FFSPMV_API ffspmv_status ffspmv_get_info(ffspmv_matrix A, ffspmv_info *out);

/* Host-only planner: run the create pipeline without touching a device and
 * report the plan.  If rec_* are non-NULL (each of capacity rec_cap), also
 * write the triples of A (transpose = 0) or A^T (transpose = 1) as
 * reconstructed FROM THE PACKED LAYOUT (every piece, slot and stream summed
 * back), returning their count in *rec_n.  This is how CPU tests check that
 * the sum of the pieces equals A.  Errors as ffspmv_create. */
FFSPMV_API ffspmv_status ffspmv_analyze(uint64_t rows, uint64_t cols, uint64_t nnz,
                                        const uint32_t *row_idx, const uint32_t *col_idx,
                                        const int64_t *vals, uint32_t modulus,
                                        const ffspmv_options *opts, ffspmv_info *info,
                                        int transpose, uint32_t *rec_row, uint32_t *rec_col,
                                        uint32_t *rec_val, uint64_t rec_cap, uint64_t *rec_n);

/* --- products (device pointers, asynchronous on stream) -------------------- */

/* y <- (alpha*A*x + beta*y) mod m.  x: cols entries (nx), y: rows
 * entries (ny).  alpha, beta are reduced mod m; beta == 0 (mod m) means y is
 * not read ("apply ... first setting y elements to zero").
 * Errors: INVALID_ARG (NULL, x overlaps y, non-canonical input in checked
 * mode), DIM (nx != cols or ny != rows), CUDA. */
FFSPMV_API ffspmv_status ffspmv_apply(ffspmv_matrix A, uint32_t alpha, const uint32_t *x,
                                      uint64_t nx, uint32_t beta, uint32_t *y, uint64_t ny,
                                      void *stream);

/* y <- (alpha*A^T*x + beta*y) mod m   ("the transpose product").
 * x: rows entries, y: cols entries.  On a handle built with no_transpose the
 * product scatters A's entries (terms reduced below m + 1, u64 column sums:
 * exact whatever the order of the atomics) and uses a per-handle scratch:
 * such calls on one handle must be ordered on one stream. */
FFSPMV_API ffspmv_status ffspmv_apply_transpose(ffspmv_matrix A, uint32_t alpha,
                                                const uint32_t *x, uint64_t nx, uint32_t beta,
                                                uint32_t *y, uint64_t ny, void *stream);

/* Y <- (alpha*A*X + beta*Y) mod m   (multi-vectors P:351-378).  X is
 * cols x k, Y is rows x k, both row-major with k contiguous entries per matrix
 * row (the paper's "column-major" multi-vector) and leading
 * dimensions ldx, ldy >= k.  Any k >= 1.  Each nonzero is read once per 32
 * vector columns.  Errors: INVALID_ARG (k == 0, ld < k, X overlaps Y), CUDA. */
FFSPMV_API ffspmv_status ffspmv_apply_block(ffspmv_matrix A, uint32_t k, uint32_t alpha,
                                            const uint32_t *X, uint64_t ldx, uint32_t beta,
                                            uint32_t *Y, uint64_t ldy, void *stream);

/* End-to-end variant on HOST buffers (the black-box call of P:380-381): copies
 * x_host to the device, runs op (FFSPMV_OP_APPLY or FFSPMV_OP_TRANSPOSE), and
 * copies the result into y_host (read first if beta != 0).  Uses a staging
 * area owned by the handle (allocated on first use), so calls on one handle
 * must not overlap.  Synchronous: returns after y_host is written. */
FFSPMV_API ffspmv_status ffspmv_apply_host(ffspmv_matrix A, int op, uint32_t alpha,
                                           const uint32_t *x_host, uint32_t beta,
                                           uint32_t *y_host, void *stream);

/* --- block Wiedemann sequence ---------------------------------------------- */

/* Workspace bytes for ffspmv_sequence with block width k and ku projections. */
FFSPMV_API ffspmv_status ffspmv_workspace_size(ffspmv_matrix A, int op, uint32_t k,
                                               uint32_t ku, size_t *bytes);

/* Projected block Krylov sequence (§3 step 1; §2.5.2 for the
 * device-resident iteration):
 *   V_0 = X,  V_{t+1} = A V_t mod m,
 *   S[t][a][b] = sum_r U[r][a] * V_t[r][b] mod m   for 0 <= t < L.
 * A must be square (n x n).  X: n x k, U: n x ku (row-major, device);
 * U == NULL means U = X (ku must equal k): the paper's Y^T A^i Y.  S: L x ku x k
 * row-major (device).  V_out (nullable, device n x k) receives A^L X, so a
 * second call with X = V_out continues the sequence exactly (chaining).
 * workspace: device scratch of at least ffspmv_workspace_size(A, SEQUENCE, k,
 * ku) bytes.  Errors: NONSQUARE, INVALID_ARG, NOMEM (workspace too small),
 * CUDA. */
FFSPMV_API ffspmv_status ffspmv_sequence(ffspmv_matrix A, uint32_t k, const uint32_t *X,
                                         uint32_t ku, const uint32_t *U, uint64_t L,
                                         uint32_t *S, uint32_t *V_out, void *workspace,
                                         size_t workspace_bytes, void *stream);

/* Projection of one block (the "dense dot products by U^T" of P:459-460):
 *   S[a][b] = sum_r U[r][a] * V[r][b] mod m,  r < rows(A),
 * V: rows(A) x k, U: rows(A) x ku (device, row-major), S: ku x k (device).
 * Used by the row-banded multi-GPU sequence, where A is a rank's band and V,
 * U its rows.  workspace >= ffspmv_workspace_size(A, FFSPMV_OP_PROJECT, k, ku).
 * Errors: INVALID_ARG, NOMEM (workspace), CUDA. */
FFSPMV_API ffspmv_status ffspmv_project(ffspmv_matrix A, uint32_t k, const uint32_t *V,
                                        uint32_t ku, const uint32_t *U, uint32_t *S,
                                        void *workspace, size_t workspace_bytes, void *stream);

/* out[i] = sum_p parts[p * count + i] mod m, for combining per-rank residues
 * (e.g. the band projections after an all-gather).  Device pointers. */
FFSPMV_API ffspmv_status ffspmv_sum_mod(ffspmv_matrix A, uint64_t count, uint32_t nparts,
                                        const uint32_t *parts, uint32_t *out, void *stream);

/* --- distributed sequence ("parallel sequence generation") -------- *
 *
 * One rank per GPU.  A communicator comes from NCCL (loaded at run time from
 * libnccl.so.2, so the library itself has no NCCL link dependency):
 *   rank 0: ffspmv_comm_unique_id(id); broadcast the 128 bytes (e.g. over a
 *   torch.distributed process group); every rank: ffspmv_comm_create(&c, id,
 *   nranks, rank) -- collective, like ncclCommInitRank.
 * ffspmv_comm_create_local(out[nranks], nranks) makes an in-process group
 * instead (ranks = host threads on one device, collectives = device copies,
 * synchronous): the same distributed code path, testable on one GPU.
 *
 * A DISTRIBUTED handle: every rank calls ffspmv_create with the FULL triple
 * list of a square n x n matrix and options.comm (collective).  The ranks
 * form a P_r x P_c grid (rank = i * P_c + j, P_r = options.dist_rows or all
 * ranks); rank (i, j) keeps row band i of A (nnz-balanced contiguous bands,
 * the same on every rank) and, in ffspmv_sequence, column block j of X
 * (columns [k j / P_c, k (j + 1) / P_c)).  Per step it computes its band of
 * V_{t+1}[:, block j] (band SpMM + fused band projection) and all-gathers
 * the band iterates among the P_r ranks of block j on the caller's stream
 * (NCCL: ncclAllGather over the column-group communicator, an
 * ncclCommSplit of comm).  P_c = 1 is the row-band mode of P:462-463 ("let
 * the SpMV library take care of the iteration"), P_r = 1 the column mode of
 * P:457-460 ("ship independent set of vector blocks ... then gather").
 * ffspmv_sequence takes the same arguments as on one GPU -- X, U (full
 * n x k / n x ku, replicated), S (full L x ku x k) and V_out (full) on every
 * rank -- and returns results identical to the one-GPU call.
 * ffspmv_apply_block (and ffspmv_apply, its k = 1 case) on a distributed
 * handle is the row-sharded single product: rank (i, j)
 * computes Y[band i, block j] = alpha A X + beta Y in place, then the blocks
 * of all ranks are all-gathered into Y, so Y (replicated on entry, n x k
 * contiguous: ldx = ldy = k, else FFSPMV_ERR_UNSUPPORTED) is the full
 * one-GPU result on every rank on return.  ffspmv_sequence,
 * ffspmv_apply(_block), ffspmv_workspace_size and ffspmv_get_info accept a
 * distributed handle (the others -- the transpose, apply_host, project,
 * sum_mod -- return FFSPMV_ERR_UNSUPPORTED).  Calls on a
 * distributed handle must not overlap (it owns the result-exchange buffers,
 * allocated on first use and grown with L). */
FFSPMV_API ffspmv_status ffspmv_comm_unique_id(void *id_128);
FFSPMV_API ffspmv_status ffspmv_comm_create(ffspmv_comm *out, const void *id_128, int nranks,
                                            int rank);
FFSPMV_API ffspmv_status ffspmv_comm_create_local(ffspmv_comm *out, int nranks);
/* Destroy after every handle created with it. */
FFSPMV_API ffspmv_status ffspmv_comm_destroy(ffspmv_comm c);

/* --- diagnostics ------------------------------------------------------------ */

FFSPMV_API const char *ffspmv_status_string(ffspmv_status s);

/* Thread-local detail message for the last non-OK status on this thread. */
FFSPMV_API const char *ffspmv_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
FFSPMV_API int ffspmv_version(void);

/* Number of CUDA kernels this library has launched in this process (all
 * threads), for launch accounting in benchmarks. */
FFSPMV_API uint64_t ffspmv_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* FFSPMV_H */
