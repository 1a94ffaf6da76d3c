// Host packing of the RUNS operator (see internal.hpp "runs"): the column-
// wise split of A into panels x row bands, each unit's entries
// split into +1 / -1 / valued sections, sorted by row and laid
// out as register runs.
#include <algorithm>
#include <cstring>

#include "internal.hpp"

namespace ffspmv {

namespace {

uint32_t xbits_for(uint32_t m) {
    // narrowest staged width holding every residue 0 .. m-1
    if (m <= 4u) return 2;
    if (m <= 16u) return 4;
    if (m <= 256u) return 8;
    if (m <= 65536u) return 16;
    return 32;
}

uint32_t log2ceil(uint32_t v) {
    uint32_t r = 0;
    while ((1u << r) < v) ++r;
    return r;
}

}  // namespace

RunsGeom runs_geometry(uint64_t rows, uint64_t cols, uint64_t nnz, uint32_t m,
                       const BuildOptions &bo, uint32_t nsm) {
    RunsGeom g;
    g.xbits = std::max(xbits_for(m), bo.xbits ? bo.xbits : 0u);
    g.wide = m > 65536u ? 1 : 0;
    g.pbytes = m <= 256u ? 1 : m <= 65536u ? 2 : 4;
    const uint64_t aw = g.wide ? 2 : 1;
    // shared memory: packed x panel + 16 zero bytes (the padding entries'
    // word) | alignment slack | RUN_WARPS warp-private accumulator blocks of
    // 2^rs rows (twice when wide) | mbarrier and counter
    auto panels_for = [&](uint32_t R, uint32_t &W, uint32_t &rs) {
        rs = std::max<uint32_t>(2, log2ceil(R));
        const uint64_t block = aw * (4ull << rs);
        const uint64_t fixed = 16 + block + (uint64_t)RUN_WARPS * block + 64;
        uint64_t pbytes = fixed < PANEL_SMEM_MAX ? PANEL_SMEM_MAX - fixed : 0;
        // the word offset (<= panel_bytes, the padding word) takes the
        // 27 - rs bits above the row and shift fields
        pbytes = std::min<uint64_t>(pbytes, (1ull << (27 - rs)) - 16);
        uint64_t wmax = pbytes * 8 / g.xbits;
        if (bo.panel_cols) wmax = std::min<uint64_t>(wmax, bo.panel_cols);
        wmax = std::max<uint64_t>(64, wmax / 64 * 64);
        const uint64_t P = std::max<uint64_t>(1, (cols + wmax - 1) / wmax);
        // balanced panels, a multiple of 64 columns (16-byte packed panels)
        uint64_t w = (cols + P - 1) / P;
        W = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(64, (w + 63) / 64 * 64), wmax);
        return (uint32_t)std::max<uint64_t>(1, (cols + W - 1) / W);
    };
    // rows per unit R: about 1024 entries per unit (the write-out of R band
    // rows and the padding of the unit's last chunks are amortised over
    // them; measured on c3: 256-row units 72.7 us, 512 80.9, 1024 91.1),
    // 64 <= R <= 512
    uint32_t W = 0, rs = 0;
    uint32_t R = 256;
    if (bo.panel_rows) {
        R = bo.panel_rows;
    } else if (rows && nnz) {
        const uint32_t P0 = panels_for(R, W, rs);
        const double per_row = (double)nnz / (double)rows / P0;   // entries per row and panel
        R = 64;
        while (R < 512 && R * per_row < 1024.0) R *= 2;
    }
    g.R = R;
    g.P = panels_for(R, W, rs);
    g.W = W;
    g.rs = rs;
    g.B = (uint32_t)std::max<uint64_t>(1, (rows + g.R - 1) / g.R);
    g.nctas = std::max<uint32_t>(1, nsm);
    g.panel_bytes = (uint32_t)((uint64_t)g.W * g.xbits / 8);
    g.rows_pad = (uint32_t)((rows + 15) / 16 * 16);
    return g;
}

// entry word of element idx of the panel in band row rl (internal.hpp)
static inline uint32_t run_word(const RunsGeom &g, uint32_t idx, uint32_t rl) {
    const uint32_t per = 32 / g.xbits;               // residues per 32-bit word
    const uint32_t off = 4 * (idx / per);            // byte offset of the word
    const uint32_t sh = g.xbits * (idx % per);       // bit offset inside it (< 32)
    return off << (5 + g.rs) | rl << 5 | sh;
}

bool pack_runs(HostRuns &hr, const Canon &a, uint32_t m, const BuildOptions &bo, uint32_t nsm) {
    hr = HostRuns();
    hr.rows = (uint32_t)a.nrows;
    hr.cols = (uint32_t)a.ncols;
    RunsGeom &g = hr.g;
    g = runs_geometry(a.nrows, a.ncols, a.idx.size(), m, bo, nsm);
    if (a.nrows == 0) return false;
    const uint32_t vb = value_bytes_for(m);
    const uint64_t T = (uint64_t)g.P * g.B;
    bool seg = bo.segregate_pm1 >= 0;
    uint64_t npm_all = 0;
    for (uint32_t v : a.val) npm_all += (v == 1u || (m > 2 && v == m - 1));
    if (bo.segregate_pm1 == 0 && npm_all * 20 < a.val.size()) seg = false;
    // section of an entry: 0 = +1, 1 = -1, 2 = valued (m = 2: 1 == m - 1 is +1)
    auto section = [&](uint32_t v) -> int {
        if (seg && v == 1u) return 0;
        if (seg && m > 2 && v == m - 1) return 1;
        return 2;
    };

    // entries per (unit, section) and, for m <= 2^16, the worst band-row sum
    // of one unit: +1 adds x <= m-1, -1 adds m - x <= m, valued adds a lazy
    // Barrett remainder < 2m
    std::vector<uint64_t> cnt(3 * T, 0);
    uint64_t worst = 0;
    for (uint64_t r = 0; r < a.nrows; ++r) {
        const uint64_t b = r / g.R;
        uint64_t p_cur = ~0ull, k[3] = {0, 0, 0};
        auto close = [&]() {
            worst = std::max<uint64_t>(worst, k[0] * (m - 1) + k[1] * m + k[2] * (2ull * m - 1));
            k[0] = k[1] = k[2] = 0;
        };
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            const uint64_t p = a.idx[t] / g.W;
            if (p != p_cur) { close(); p_cur = p; }
            const int s = section(a.val[t]);
            k[s]++;
            cnt[3 * (p * g.B + b) + s]++;
        }
        close();
    }
    if (!g.wide && worst >= (1ull << 32)) return false;

    // units: chunk counts per section; every unit gets at least one chunk so
    // the kernel's per-warp pipeline never meets an empty unit
    hr.tiles.resize(T);
    uint64_t c = 0, vc = 0;
    for (uint64_t t = 0; t < T; ++t) {
        RunsTile &tl = hr.tiles[t];
        tl.c0 = (uint32_t)c;
        tl.npc = (uint32_t)((cnt[3 * t] + RUN_CHUNK - 1) / RUN_CHUNK);
        tl.nmc = (uint32_t)((cnt[3 * t + 1] + RUN_CHUNK - 1) / RUN_CHUNK);
        tl.nvc = (uint32_t)((cnt[3 * t + 2] + RUN_CHUNK - 1) / RUN_CHUNK);
        if (tl.npc + tl.nmc + tl.nvc == 0) tl.npc = 1;
        tl.vc0 = (uint32_t)vc;
        const uint64_t b = t % g.B;
        tl.rn = (uint32_t)std::min<uint64_t>(g.R, a.nrows - b * g.R);
        tl.pad0 = tl.pad1 = 0;
        c += tl.npc + tl.nmc + tl.nvc;
        vc += tl.nvc;
        hr.nnz_pm += cnt[3 * t] + cnt[3 * t + 1];
        hr.nnz_val += cnt[3 * t + 2];
    }
    if (c * RUN_CHUNK >= (1ull << 32)) throw std::bad_alloc();
    hr.words.assign(c * RUN_CHUNK, 0);
    hr.vval.assign(vc * RUN_CHUNK * vb, 0);
    // fill in row order: each section comes out sorted by (row, col); entry
    // i of a section goes to chunk i / 512, lane (i % 512) / 16, slot i % 16
    std::vector<uint64_t> cur(3 * T, 0);
    auto wpos = [](uint64_t base_chunk, uint64_t i) {
        const uint64_t ch = i / RUN_CHUNK, e = i % RUN_CHUNK, lane = e / RUN_E, j = e % RUN_E;
        return (base_chunk + ch) * RUN_CHUNK + 128 * (j / 4) + 4 * lane + (j % 4);
    };
    auto sec_base = [&](const RunsTile &tl, int s) -> uint64_t {
        return (uint64_t)tl.c0 + (s > 0 ? tl.npc : 0) + (s > 1 ? tl.nmc : 0);
    };
    for (uint64_t r = 0; r < a.nrows; ++r) {
        const uint64_t b = r / g.R;
        const uint32_t rl = (uint32_t)(r - b * g.R);
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            const uint32_t col = a.idx[t], v = a.val[t];
            const uint64_t p = col / g.W;
            const uint64_t unit = p * g.B + b;
            const RunsTile &tl = hr.tiles[unit];
            const int s = section(v);
            const uint64_t i = cur[3 * unit + s]++;
            hr.words[wpos(sec_base(tl, s), i)] = run_word(g, (uint32_t)(col - p * g.W), rl);
            if (s == 2) {
                const uint64_t vi = ((uint64_t)tl.vc0 + i / RUN_CHUNK) * RUN_CHUNK + i % RUN_CHUNK;
                std::memcpy(&hr.vval[vi * vb], &v, vb);
            }
        }
    }
    // padding entries (the tail of a section's last chunk): the section's
    // last row (row 0 for a unit's forced empty chunk) and the zero word past
    // the panel (byte offset panel_bytes), value 0: they extend the last run
    // and add nothing
    for (uint64_t t = 0; t < T; ++t) {
        const RunsTile &tl = hr.tiles[t];
        const uint32_t nch[3] = {tl.npc, tl.nmc, tl.nvc};
        for (int s = 0; s < 3; ++s) {
            const uint64_t n = cnt[3 * t + s], base = sec_base(tl, s), end = (uint64_t)nch[s] * RUN_CHUNK;
            if (n == end) continue;
            const uint32_t last_row = n ? (hr.words[wpos(base, n - 1)] >> 5) & ((1u << g.rs) - 1) : 0u;
            const uint32_t padw = g.panel_bytes << (5 + g.rs) | last_row << 5;
            for (uint64_t i = n; i < end; ++i) hr.words[wpos(base, i)] = padw;
        }
    }
    // CTA schedule: contiguous unit ranges (panel-major, so a CTA restages its
    // x panel only when its range crosses a panel boundary), balanced by
    // chunks + the per-unit band write-out
    std::vector<double> cost(T);
    double total = 0;
    for (uint64_t t = 0; t < T; ++t) {
        const RunsTile &tl = hr.tiles[t];
        cost[t] = (double)RUN_CHUNK * (tl.npc + tl.nmc + tl.nvc) + 0.5 * (double)tl.rn;
        total += cost[t];
    }
    hr.cta_t0.assign(g.nctas + 1, (uint32_t)T);
    hr.cta_t0[0] = 0;
    double acc = 0;
    uint32_t k = 1;
    for (uint64_t t = 0; t < T && k < g.nctas; ++t) {
        acc += cost[t];
        while (k < g.nctas && acc >= total * k / g.nctas) hr.cta_t0[k++] = (uint32_t)(t + 1);
    }
    for (; k < g.nctas; ++k) hr.cta_t0[k] = (uint32_t)T;
    hr.stream_bytes = 4 * hr.words.size() + hr.vval.size() + T * sizeof(RunsTile);
    return true;
}

uint64_t reconstruct_runs(const HostRuns &hr, uint32_t m, uint32_t vb, uint32_t *rr, uint32_t *rc,
                          uint32_t *rv, uint64_t cap) {
    uint64_t n = 0;
    const RunsGeom &g = hr.g;
    const uint32_t rmask = (1u << g.rs) - 1, per = 32 / g.xbits;
    for (uint64_t t = 0; t < hr.tiles.size(); ++t) {
        const RunsTile &tl = hr.tiles[t];
        const uint64_t p = t / g.B, b = t % g.B;
        for (uint32_t ch = 0; ch < tl.npc + tl.nmc + tl.nvc; ++ch) {
            const int s = ch < tl.npc ? 0 : ch < tl.npc + tl.nmc ? 1 : 2;
            for (uint32_t lane = 0; lane < 32; ++lane)
                for (uint32_t j = 0; j < RUN_E; ++j) {
                    const uint64_t wi = (uint64_t)(tl.c0 + ch) * RUN_CHUNK + 128 * (j / 4) + 4 * lane + (j % 4);
                    const uint32_t w = hr.words[wi];
                    const uint32_t row = (w >> 5) & rmask, sh = w & 31, off = w >> (5 + g.rs);
                    uint32_t v = 0;
                    if (s == 2) {
                        const uint64_t vi = (uint64_t)(tl.vc0 + ch - tl.npc - tl.nmc) * RUN_CHUNK + RUN_E * lane + j;
                        std::memcpy(&v, &hr.vval[vi * vb], vb);
                    } else {
                        v = s == 0 ? 1u : m - 1;
                    }
                    if (off == g.panel_bytes) {           // padding: the zero word, value 0
                        if (sh != 0 || (s == 2 && v != 0)) return ~0ull;
                        continue;
                    }
                    if (off % 4 || off >= g.panel_bytes || sh % g.xbits || row >= tl.rn) return ~0ull;
                    const uint64_t idx = (uint64_t)(off / 4) * per + sh / g.xbits;
                    if (idx >= g.W) return ~0ull;
                    if (n < cap) {
                        rr[n] = (uint32_t)(b * g.R + row);
                        rc[n] = (uint32_t)(p * g.W + idx);
                        rv[n] = v;
                    }
                    ++n;
                }
        }
    }
    return n;
}

}  // namespace ffspmv
