/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the
 * exact sparse hot path of Boyer, Dumas & Giorgi (arXiv:1004.3719,
 * /root/reference/PAPER.md, cited "P:line") computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_1004_3719_b200/)
 * never links, imports or executes it, and this file shares no code,
 * header, constant or helper with the CUDA path.
 *
 * Every function is the plain definition of the result written out:
 *   - the ring is Z/mZ with canonical representatives [0, m-1]
 *     ("we represent the ring on [0, m-1]");
 *   - a matrix is a list of COO triples ("three vectors of size
 *     nbnz, named data, colid and rowid"); duplicate triples are summed
 *     (reading R3) because the sum of the triples IS the entry;
 *   - every inner product is accumulated exactly in an unsigned 128-bit
 *     integer and reduced ONCE at the end — the paper's delayed reduction
 *     (§2.2) taken to its limit: each term is < 2^64 and fewer
 *     than 2^64 terms are ever summed, so nothing can overflow;
 *   - alpha and beta follow P:99-101 (§2): y <- alpha*A*x + beta*y,
 *     computed as alpha*(Ax) + beta*y, which is the same residue as
 *     "pre-multiplying x and y by alpha and beta".
 *
 * No sort, no duplicate merge, no zero drop, no blocking, no formats: the
 * oracle touches the raw triples exactly as given.
 *
 * Return value of every entry point: 0 on success, -1 on a violated
 * precondition (index out of range, m < 2, non-canonical vector entry).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* Euclidean residue of a signed 64-bit input value in [0, m-1].
 * P:145 "a[i], b[i] are reduced modulo m at first"; negative inputs
 * (e.g. -1 for the paper's "-1" entries) map to m-1. */
static uint64_t residue(int64_t v, uint32_t m)
{
    int64_t r = v % (int64_t)m;           /* C99: sign of r follows v */
    if (r < 0) r += (int64_t)m;
    return (uint64_t)r;
}

/* (alpha * a + beta * b) mod m with a = exact sum (u128), b canonical. */
static uint32_t combine(u128 acc, uint32_t alpha, uint32_t b, uint32_t beta, uint32_t m)
{
    u128 am = (u128)(alpha % m);
    u128 bm = (u128)(beta % m);
    u128 r = am * (acc % m) + bm * (u128)b;   /* < 2 * 2^64: fits */
    return (uint32_t)(r % m);
}

static int check_triples(uint64_t rows, uint64_t cols, uint64_t nnz,
                         const uint32_t *ri, const uint32_t *ci)
{
    for (uint64_t t = 0; t < nnz; ++t)
        if (ri[t] >= rows || ci[t] >= cols) return -1;
    return 0;
}

static int check_canonical(const uint32_t *v, uint64_t n, uint32_t m)
{
    for (uint64_t i = 0; i < n; ++i)
        if (v[i] >= m) return -1;
    return 0;
}

/* y <- alpha*A*x + beta*y   (§2; the JIT listing P:254-261 fixes
 * y <- y + Ax with one reduction per row).  x has cols entries, y rows. */
int oracle_apply(uint64_t rows, uint64_t cols, uint64_t nnz,
                 const uint32_t *ri, const uint32_t *ci, const int64_t *val,
                 uint32_t m, uint32_t alpha, const uint32_t *x,
                 uint32_t beta, uint32_t *y)
{
    if (m < 2 || check_triples(rows, cols, nnz, ri, ci)) return -1;
    if (check_canonical(x, cols, m)) return -1;
    if (beta % m && check_canonical(y, rows, m)) return -1;
    u128 *acc = (u128 *)calloc(rows ? rows : 1, sizeof(u128));
    if (!acc) return -1;
    for (uint64_t t = 0; t < nnz; ++t)
        acc[ri[t]] += (u128)residue(val[t], m) * (u128)x[ci[t]];
    for (uint64_t i = 0; i < rows; ++i)
        y[i] = combine(acc[i], alpha, (beta % m) ? y[i] : 0u, beta, m);
    free(acc);
    return 0;
}

/* y <- alpha*A^T*x + beta*y   (§1 "together with the transpose
 * product").  x has rows entries, y cols. */
int oracle_apply_transpose(uint64_t rows, uint64_t cols, uint64_t nnz,
                           const uint32_t *ri, const uint32_t *ci, const int64_t *val,
                           uint32_t m, uint32_t alpha, const uint32_t *x,
                           uint32_t beta, uint32_t *y)
{
    if (m < 2 || check_triples(rows, cols, nnz, ri, ci)) return -1;
    if (check_canonical(x, rows, m)) return -1;
    if (beta % m && check_canonical(y, cols, m)) return -1;
    u128 *acc = (u128 *)calloc(cols ? cols : 1, sizeof(u128));
    if (!acc) return -1;
    for (uint64_t t = 0; t < nnz; ++t)
        acc[ci[t]] += (u128)residue(val[t], m) * (u128)x[ri[t]];
    for (uint64_t j = 0; j < cols; ++j)
        y[j] = combine(acc[j], alpha, (beta % m) ? y[j] : 0u, beta, m);
    free(acc);
    return 0;
}

/* Y <- alpha*A*X + beta*Y   (§2 "X and Y are sets of vectors").
 * X is cols x k with leading dimension ldx (k contiguous entries per matrix
 * row: the paper's "column-major" multi-vector); Y is rows x k
 * with leading dimension ldy. */
int oracle_apply_block(uint64_t rows, uint64_t cols, uint64_t nnz,
                       const uint32_t *ri, const uint32_t *ci, const int64_t *val,
                       uint32_t m, uint32_t k, uint32_t alpha,
                       const uint32_t *X, uint64_t ldx,
                       uint32_t beta, uint32_t *Y, uint64_t ldy)
{
    if (m < 2 || k == 0 || ldx < k || ldy < k) return -1;
    if (check_triples(rows, cols, nnz, ri, ci)) return -1;
    for (uint64_t j = 0; j < cols; ++j)
        if (check_canonical(X + j * ldx, k, m)) return -1;
    if (beta % m)
        for (uint64_t i = 0; i < rows; ++i)
            if (check_canonical(Y + i * ldy, k, m)) return -1;
    u128 *acc = (u128 *)calloc(rows * (uint64_t)k + 1, sizeof(u128));
    if (!acc) return -1;
    for (uint64_t t = 0; t < nnz; ++t) {
        uint64_t a = residue(val[t], m);
        for (uint32_t c = 0; c < k; ++c)
            acc[(uint64_t)ri[t] * k + c] += (u128)a * (u128)X[(uint64_t)ci[t] * ldx + c];
    }
    for (uint64_t i = 0; i < rows; ++i)
        for (uint32_t c = 0; c < k; ++c) {
            uint32_t yold = (beta % m) ? Y[i * ldy + c] : 0u;
            Y[i * ldy + c] = combine(acc[i * k + c], alpha, yold, beta, m);
        }
    free(acc);
    return 0;
}

/* Projected block Krylov sequence (§3 step 1, "S_i = Y^T A^i Y for
 * i = 0..2n/s+O(1)", with the left projection generalised to U as in the
 * north star):
 *   V_0 = X;  S_t[a][b] = sum_r U[r][a] * V_t[r][b]  mod m,  0 <= t < L;
 *   V_{t+1} = A V_t mod m   (the device-resident iteration of P:389-399).
 * A must be square (n x n).  X is n x k (row-major, k contiguous), U is
 * n x ku; U == NULL means U = X (ku must equal k).  S is L x ku x k
 * row-major.  V_out (nullable) receives V_L = A^L X. */
int oracle_sequence(uint64_t n, uint64_t nnz,
                    const uint32_t *ri, const uint32_t *ci, const int64_t *val,
                    uint32_t m, uint32_t k, const uint32_t *X,
                    uint32_t ku, const uint32_t *U,
                    uint64_t L, uint32_t *S, uint32_t *V_out)
{
    if (m < 2 || k == 0) return -1;
    if (U == NULL) { U = X; if (ku != k) return -1; }
    if (ku == 0) return -1;
    if (check_triples(n, n, nnz, ri, ci)) return -1;
    if (check_canonical(X, n * (uint64_t)k, m)) return -1;
    if (check_canonical(U, n * (uint64_t)ku, m)) return -1;
    uint32_t *V = (uint32_t *)malloc((n * (uint64_t)k + 1) * sizeof(uint32_t));
    uint32_t *W = (uint32_t *)malloc((n * (uint64_t)k + 1) * sizeof(uint32_t));
    if (!V || !W) { free(V); free(W); return -1; }
    memcpy(V, X, n * (uint64_t)k * sizeof(uint32_t));
    for (uint64_t t = 0; t < L; ++t) {
        /* S_t = U^T V_t : plain dot products over all n rows. */
        for (uint32_t a = 0; a < ku; ++a)
            for (uint32_t b = 0; b < k; ++b) {
                u128 s = 0;
                for (uint64_t r = 0; r < n; ++r)
                    s += (u128)U[r * ku + a] * (u128)V[r * k + b];
                S[(t * ku + a) * (uint64_t)k + b] = (uint32_t)(s % m);
            }
        /* V_{t+1} = A V_t  (alpha = 1, beta = 0). */
        if (oracle_apply_block(n, n, nnz, ri, ci, val, m, k, 1u, V, k, 0u, W, k)) {
            free(V); free(W); return -1;
        }
        uint32_t *tmp = V; V = W; W = tmp;
    }
    if (V_out) memcpy(V_out, V, n * (uint64_t)k * sizeof(uint32_t));
    free(V); free(W);
    return 0;
}

/* ------------------------------------------------------------------------
 * Threaded timing mode (used ONLY to time the oracle
 * on the host's cores for bench.py's cpu_baseline / --impl reference, and
 * pinned against the serial functions above by tests/test_oracle_pins.py).
 *
 * Same definition, same u128 accumulate-then-reduce: the caller passes the
 * triples sorted by their OUTPUT index `key` (the row for A x, the column for
 * A^T x) -- sorting is done outside the timed region -- and the triple list
 * is cut into nthreads contiguous ranges whose boundaries are moved to key
 * changes, so every output accumulator is owned by exactly one thread: no
 * races, no change to any sum.  `src` is the other index (the one x is read
 * at).
 * ------------------------------------------------------------------------ */

/* thread t's triple range [*lo, *hi): the t-th nnz/T slice, both ends moved
 * forward to the first triple of a new key */
static void mt_range(const uint32_t *key, uint64_t nnz, int t, int T, uint64_t *lo, uint64_t *hi)
{
    uint64_t a = nnz * (uint64_t)t / (uint64_t)T, b = nnz * (uint64_t)(t + 1) / (uint64_t)T;
    while (a > 0 && a < nnz && key[a] == key[a - 1]) ++a;
    while (b > 0 && b < nnz && key[b] == key[b - 1]) ++b;
    *lo = a;
    *hi = b < a ? a : b;
}

static int check_sorted(const uint32_t *key, uint64_t nnz)
{
    for (uint64_t t = 1; t < nnz; ++t)
        if (key[t] < key[t - 1]) return -1;
    return 0;
}

/* y[key] <- alpha * sum A x + beta * y over nout outputs, k vectors:
 * X is nin x k (ldx = k), Y is nout x k (ldy = k). */
int oracle_apply_sorted_mt(uint64_t nout, uint64_t nin, uint64_t nnz,
                           const uint32_t *key, const uint32_t *src, const int64_t *val,
                           uint32_t m, uint32_t k, uint32_t alpha, const uint32_t *X,
                           uint32_t beta, uint32_t *Y, int nthreads)
{
    if (m < 2 || k == 0 || nthreads < 1) return -1;
    if (check_triples(nout, nin, nnz, key, src) || check_sorted(key, nnz)) return -1;
    if (check_canonical(X, nin * (uint64_t)k, m)) return -1;
    if (beta % m && check_canonical(Y, nout * (uint64_t)k, m)) return -1;
    u128 *acc = (u128 *)calloc(nout * (uint64_t)k + 1, sizeof(u128));
    if (!acc) return -1;
    #pragma omp parallel num_threads(nthreads)
    {
        int t = 0, T = 1;
#ifdef _OPENMP
        t = omp_get_thread_num();
        T = omp_get_num_threads();
#endif
        uint64_t lo, hi;
        mt_range(key, nnz, t, T, &lo, &hi);
        for (uint64_t e = lo; e < hi; ++e) {
            uint64_t a = residue(val[e], m);
            for (uint32_t c = 0; c < k; ++c)
                acc[(uint64_t)key[e] * k + c] += (u128)a * (u128)X[(uint64_t)src[e] * k + c];
        }
        #pragma omp barrier
        for (uint64_t i = nout * (uint64_t)t / (uint64_t)T; i < nout * (uint64_t)(t + 1) / (uint64_t)T; ++i)
            for (uint32_t c = 0; c < k; ++c) {
                uint32_t yold = (beta % m) ? Y[i * k + c] : 0u;
                Y[i * k + c] = combine(acc[i * k + c], alpha, yold, beta, m);
            }
    }
    free(acc);
    return 0;
}

/* The sequence of oracle_sequence with the block apply above (triples
 * sorted by row) and the projection S_t = U^T V_t summed over nthreads row
 * ranges (per-thread u128 partial sums, added in thread order, reduced once). */
int oracle_sequence_mt(uint64_t n, uint64_t nnz,
                       const uint32_t *ri, const uint32_t *ci, const int64_t *val,
                       uint32_t m, uint32_t k, const uint32_t *X,
                       uint32_t ku, const uint32_t *U,
                       uint64_t L, uint32_t *S, uint32_t *V_out, int nthreads)
{
    if (m < 2 || k == 0 || nthreads < 1) return -1;
    if (U == NULL) { U = X; if (ku != k) return -1; }
    if (ku == 0) return -1;
    if (check_triples(n, n, nnz, ri, ci) || check_sorted(ri, nnz)) return -1;
    if (check_canonical(X, n * (uint64_t)k, m)) return -1;
    if (check_canonical(U, n * (uint64_t)ku, m)) return -1;
    uint32_t *V = (uint32_t *)malloc((n * (uint64_t)k + 1) * sizeof(uint32_t));
    uint32_t *W = (uint32_t *)malloc((n * (uint64_t)k + 1) * sizeof(uint32_t));
    u128 *part = (u128 *)calloc((uint64_t)nthreads * ku * k + 1, sizeof(u128));
    if (!V || !W || !part) { free(V); free(W); free(part); return -1; }
    memcpy(V, X, n * (uint64_t)k * sizeof(uint32_t));
    for (uint64_t t = 0; t < L; ++t) {
        memset(part, 0, (uint64_t)nthreads * ku * k * sizeof(u128));
        #pragma omp parallel num_threads(nthreads)
        {
            int th = 0, T = 1;
#ifdef _OPENMP
            th = omp_get_thread_num();
            T = omp_get_num_threads();
#endif
            u128 *p = part + (uint64_t)th * ku * k;
            for (uint64_t r = n * (uint64_t)th / (uint64_t)T; r < n * (uint64_t)(th + 1) / (uint64_t)T; ++r)
                for (uint32_t a = 0; a < ku; ++a)
                    for (uint32_t b = 0; b < k; ++b)
                        p[(uint64_t)a * k + b] += (u128)U[r * ku + a] * (u128)V[r * k + b];
        }
        for (uint32_t a = 0; a < ku; ++a)
            for (uint32_t b = 0; b < k; ++b) {
                u128 s = 0;
                for (int th = 0; th < nthreads; ++th) s += part[((uint64_t)th * ku + a) * k + b];
                S[(t * ku + a) * (uint64_t)k + b] = (uint32_t)(s % m);
            }
        if (oracle_apply_sorted_mt(n, n, nnz, ri, ci, val, m, k, 1u, V, 0u, W, nthreads)) {
            free(V); free(W); free(part); return -1;
        }
        uint32_t *tmp = V; V = W; W = tmp;
    }
    if (V_out) memcpy(V_out, V, n * (uint64_t)k * sizeof(uint32_t));
    free(V); free(W); free(part);
    return 0;
}

/* Version tag so a stale build is detectable. */
int oracle_version(void) { return 2; }
