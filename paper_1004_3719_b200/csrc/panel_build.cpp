// Host packing of the 2-D panel operator (see internal.hpp "panels").
#include <algorithm>
#include <cstring>
#include <unordered_set>

#include "internal.hpp"

namespace ffspmv {

PanelGeom panel_geometry(uint64_t rows, uint64_t cols, uint32_t m, const BuildOptions &bo,
                         uint32_t nsm) {
    PanelGeom g;
    // staged x element = narrowest type holding a residue
    g.xbytes = m <= 256u ? 1 : m <= 65536u ? 2 : 4;
    g.split = m > 65536u ? 1 : 0;
    // smem: W * xbytes (x panel) + R * 4 * (1 + split) (accumulators) <= 227 KB.
    // Row sums must stay < 2^32 in a u32 accumulator: W * (m-1) < 2^32 for
    // u8 (W = 196608) and u16 (W = 65536); SPLIT halves are < 2^16 each.
    if (g.xbytes == 1) { g.W = 196608u; g.cb = 18; g.R = 8176u; }
    else if (g.xbytes == 2) { g.W = 65536u; g.cb = 16; g.R = 16320u; }
    else { g.W = 49152u; g.cb = 16; g.R = 4464u; }
    if (bo.panel_cols) g.W = std::min<uint32_t>(bo.panel_cols, g.W);
    if (bo.panel_rows) g.R = std::min<uint32_t>(bo.panel_rows, g.R);
    g.P = (uint32_t)((cols + g.W - 1) / g.W);
    g.B = (uint32_t)((rows + g.R - 1) / g.R);
    g.nctas = std::max<uint32_t>(1, nsm);
    return g;
}

void pack_panels(HostPanel &hp, const Canon &a, uint32_t m, const BuildOptions &bo, uint32_t nsm) {
    hp = HostPanel();
    hp.rows = (uint32_t)a.nrows;
    hp.cols = (uint32_t)a.ncols;
    PanelGeom &g = hp.g;
    g = panel_geometry(a.nrows, a.ncols, m, bo, nsm);
    const uint32_t vb = value_bytes_for(m);
    const uint64_t T = (uint64_t)g.P * g.B;
    bool seg = bo.segregate_pm1 >= 0;
    uint64_t npm_all = 0;
    for (uint32_t v : a.val) npm_all += (v == 1u || (m > 2 && v == m - 1));
    if (bo.segregate_pm1 == 0 && npm_all * 20 < a.val.size()) seg = false;
    auto is_pm = [&](uint32_t v) { return seg && (v == 1u || (m > 2 && v == m - 1)); };

    // counting sort of the entries by tile (rows visited in order -> each
    // tile's entries come out sorted by (row, col)).  Tile t occupies
    // ent[tp[t], tp[t+1]): its +-1 entries first, then its valued entries,
    // whose values are vval[tv[t] ...] in the same order.
    hp.tp.assign(T + 1, 0);
    hp.tv.assign(T + 1, 0);
    std::vector<uint32_t> npm(T, 0);
    for (uint64_t r = 0; r < a.nrows; ++r) {
        uint64_t b = r / g.R;
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            uint64_t tile = (uint64_t)(a.idx[t] / g.W) * g.B + b;
            hp.tp[tile + 1]++;
            if (is_pm(a.val[t])) npm[tile]++;
            else hp.tv[tile + 1]++;
        }
    }
    for (uint64_t t = 0; t < T; ++t) { hp.tp[t + 1] += hp.tp[t]; hp.tv[t + 1] += hp.tv[t]; }
    hp.nnz_val = hp.tv[T];
    hp.nnz_pm = hp.tp[T] - hp.nnz_val;
    hp.pent.resize(hp.tp[T]);
    hp.vval.resize(hp.nnz_val * vb);
    std::vector<uint32_t> pp(T), pv(T), pvv(T);
    for (uint64_t t = 0; t < T; ++t) { pp[t] = hp.tp[t]; pv[t] = hp.tp[t] + npm[t]; pvv[t] = hp.tv[t]; }
    for (uint64_t r = 0; r < a.nrows; ++r) {
        uint64_t b = r / g.R;
        uint32_t rl = (uint32_t)(r - b * g.R) << (g.cb + 1);
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            uint32_t c = a.idx[t], v = a.val[t];
            uint64_t p = c / g.W;
            uint64_t tile = p * g.B + b;
            uint32_t word = rl | (uint32_t)(c - p * g.W);
            if (is_pm(v)) {
                hp.pent[pp[tile]++] = word | (v == 1u ? 0u : (1u << g.cb));
            } else {
                hp.pent[pv[tile]++] = word;
                std::memcpy(&hp.vval[(uint64_t)(pvv[tile]++) * vb], &v, vb);
            }
        }
    }
    // CTA schedule: contiguous tile ranges (panel-major, so a CTA reloads its
    // x panel only when its range crosses a panel boundary), balanced by
    // entries + the per-tile band write-out + panel loads.
    std::vector<double> cost(T);
    double total = 0;
    for (uint64_t t = 0; t < T; ++t) {
        uint64_t e = hp.tp[t + 1] - hp.tp[t];
        uint64_t b = t % g.B;
        uint64_t rn = std::min<uint64_t>(g.R, a.nrows - b * g.R);
        cost[t] = (double)e + 0.5 * (double)rn;
        total += cost[t];
    }
    hp.cta_t0.assign(g.nctas + 1, (uint32_t)T);
    hp.cta_t0[0] = 0;
    double acc = 0;
    uint32_t c = 1;
    for (uint64_t t = 0; t < T && c < g.nctas; ++t) {
        acc += cost[t];
        while (c < g.nctas && acc >= total * c / g.nctas) hp.cta_t0[c++] = (uint32_t)(t + 1);
    }
    for (; c < g.nctas; ++c) hp.cta_t0[c] = (uint32_t)T;
    hp.stream_bytes = hp.nnz_pm * 4 + hp.nnz_val * (4ull + vb) + (T + 1) * 8;
    hp.vent.clear();
}

uint64_t reconstruct_panels(const HostPanel &hp, uint32_t m, uint32_t vb, uint32_t *rr,
                            uint32_t *rc, uint32_t *rv, uint64_t cap) {
    uint64_t n = 0;
    auto emit = [&](uint32_t r, uint32_t c, uint32_t v) {
        if (n < cap) { rr[n] = r; rc[n] = c; rv[n] = v; }
        ++n;
    };
    const PanelGeom &g = hp.g;
    for (uint64_t t = 0; t < (uint64_t)g.P * g.B; ++t) {
        uint64_t p = t / g.B, b = t % g.B;
        const uint32_t nv = hp.tv[t + 1] - hp.tv[t], np = hp.tp[t + 1] - hp.tp[t] - nv;
        for (uint32_t e = hp.tp[t]; e < hp.tp[t + 1]; ++e) {
            const uint32_t w = hp.pent[e], j = e - hp.tp[t];
            uint32_t v;
            if (j < np) {
                v = (w & (1u << g.cb)) ? m - 1 : 1u;
            } else {
                v = 0;
                std::memcpy(&v, &hp.vval[(uint64_t)(hp.tv[t] + j - np) * vb], vb);
            }
            emit((uint32_t)(b * g.R + (w >> (g.cb + 1))), (uint32_t)(p * g.W + (w & ((1u << g.cb) - 1))), v);
        }
    }
    return n;
}

double gather_locality(const Canon &a) {
    uint64_t lines = 0, nnz = 0;
    std::unordered_set<uint32_t> seen;
    const uint64_t band = 256, step = std::max<uint64_t>(1, a.nrows / band / 64);  // sample <= 64 bands
    for (uint64_t b0 = 0; b0 < a.nrows; b0 += band * step) {
        seen.clear();
        uint64_t b1 = std::min<uint64_t>(a.nrows, b0 + band);
        for (uint64_t t = a.ptr[b0]; t < a.ptr[b1]; ++t) seen.insert(a.idx[t] >> 5);
        lines += seen.size();
        nnz += a.ptr[b1] - a.ptr[b0];
    }
    return nnz ? (double)lines / (double)nnz : 0.0;
}

}  // namespace ffspmv
