// Host packing of the 2-D panel operator (see internal.hpp "panels").
#include <algorithm>
#include <functional>
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
    // smem: W * xbytes (x panel) + 2 * (R + 1) * 4 * (1 + split) (the
    // accumulators + dummy row of the kernel's two thread groups) + the
    // tile-header cache (PANEL_HC) <= 227 KB.  Packed word: byte offset (< W * xbytes) above rs
    // row bits, R < 2^rs.
    if (g.xbytes == 1) { g.W = 196608u; g.R = 4088u; }
    else if (g.xbytes == 2) { g.W = 65536u; g.R = 8160u; }
    else { g.W = 49152u; g.R = 2200u; }
    // explicit geometry (tuning / tests): R first, then W shrunk to the
    // shared-memory budget and to the bits the row field leaves
    if (bo.panel_rows) g.R = bo.panel_rows;
    if (bo.panel_cols) {
        const uint64_t acc = 2ull * (((1 + g.split) * (g.R + 1ull) + 3) / 4 * 4) * 4;
        const uint64_t hc = (g.split ? 16u : 64u) * 32u + 16u;
        const uint64_t fit = acc + hc < PANEL_SMEM_MAX ? (PANEL_SMEM_MAX - acc - hc) / g.xbytes / 32 * 32 : 32;
        g.W = (uint32_t)std::min<uint64_t>(bo.panel_cols, fit);
    }
    // row field: the smallest rs with R (the dummy row) < 2^rs; the byte
    // offset of x takes the remaining 32 - rs bits
    g.rs = 1;
    while ((1u << g.rs) <= g.R) ++g.rs;
    while ((uint64_t)g.W * g.xbytes > (1ull << (32 - g.rs))) g.W -= 32;
    g.P = (uint32_t)((cols + g.W - 1) / g.W);
    g.B = (uint32_t)((rows + g.R - 1) / g.R);
    g.nctas = std::max<uint32_t>(1, nsm);
    g.rows_pad = (uint32_t)((rows + 15) / 16 * 16);
    return g;
}

namespace {

// Reassign the entries of one section (tile quads [sa, sb)) to its slots
// 4 q + u.  The slots executed by one warp instruction are {4 q + u : q in one
// 32-aligned quad group}; each such set takes entries with distinct acc banks
// (row mod 32) and distinct x banks (4-byte word of the column mod 32) while
// the pool allows, drawing from the whole section.
void arrange_section(HostPanel &hp, const PanelTile &tl, const PanelGeom &g, uint32_t vb, uint32_t sa,
                     uint32_t sb, bool valued) {
    if (sb - sa < 2) return;
    const uint32_t n = 4 * (sb - sa);
    const uint64_t e0 = 4ull * (tl.q0 + sa);
    const uint64_t v0 = valued ? 4ull * tl.vq0 + (4ull * sa - 4ull * (tl.nqp + tl.nqm)) : 0;
    const uint32_t rmask = (1u << g.rs) - 1;
    std::vector<uint32_t> w(n), v(n, 0);
    std::vector<uint32_t> bucket[32][32];
    uint32_t rb_count[32] = {0}, cb_count[32] = {0};
    for (uint32_t i = 0; i < n; ++i) {
        w[i] = hp.pent[e0 + i];
        if (valued) std::memcpy(&v[i], &hp.vval[(v0 + i) * vb], vb);
        const uint32_t rb = (w[i] & rmask) & 31, cbk = ((w[i] >> g.rs) >> 2) & 31;
        bucket[rb][cbk].push_back(i);
        rb_count[rb]++;
        cb_count[cbk]++;
    }
    std::vector<uint32_t> ow(n), ov(n);
    uint32_t avail[32];   // avail[rb]: column banks with entries left
    for (uint32_t r = 0; r < 32; ++r) {
        avail[r] = 0;
        for (uint32_t c = 0; c < 32; ++c)
            if (!bucket[r][c].empty()) avail[r] |= 1u << c;
    }
    // Phase 1: every instruction set takes a maximum bank-distinct matching
    // (at most k entries); phase 2 fills the slots left open where the pool
    // ran short of distinct pairs, distinct row banks first.
    struct Set { uint32_t ga, u, k, got, used_rb, used_cb; };
    std::vector<Set> sets;
    auto take = [&](Set &st, uint32_t rb, uint32_t cbk) {
        const uint32_t i = bucket[rb][cbk].back();
        bucket[rb][cbk].pop_back();
        if (bucket[rb][cbk].empty()) avail[rb] &= ~(1u << cbk);
        rb_count[rb]--;
        cb_count[cbk]--;
        const uint32_t slot = 4 * (st.ga + st.got - sa) + st.u;
        ow[slot] = w[i];
        ov[slot] = v[i];
        st.used_rb |= 1u << rb;
        st.used_cb |= 1u << cbk;
        ++st.got;
    };
    uint32_t rot = 0;
    for (uint32_t ga = sa; ga < sb;) {
        const uint32_t gb = std::min<uint32_t>(sb, (ga / 32 + 1) * 32);
        const uint32_t k = gb - ga;
        for (uint32_t u = 0; u < 4; ++u) {
            Set st{ga, u, k, 0, 0, 0};
            const uint32_t want = k;
            // maximum matching row bank -> column bank over non-empty buckets
            // (greedy, then augmenting paths); the fullest banks go first so
            // the pool drains evenly
            int mr[32], mc[32];
            for (int i = 0; i < 32; ++i) mr[i] = mc[i] = -1;
            uint32_t order[32];
            for (uint32_t i = 0; i < 32; ++i) order[i] = (i + rot) & 31;
            std::stable_sort(order, order + 32, [&](uint32_t x, uint32_t y) { return rb_count[x] > rb_count[y]; });
            uint32_t pairs = 0;
            for (uint32_t j = 0; j < 32 && pairs < want; ++j) {
                const uint32_t r = order[j];
                int best = -1;
                for (uint32_t c = 0; c < 32; ++c)
                    if ((avail[r] >> c & 1) && mc[c] < 0 && (best < 0 || cb_count[c] > cb_count[best])) best = (int)c;
                if (best >= 0) {
                    mr[r] = best;
                    mc[best] = (int)r;
                    ++pairs;
                }
            }
            for (uint32_t j = 0; j < 32 && pairs < want; ++j) {
                const uint32_t r = order[j];
                if (mr[r] >= 0 || !avail[r]) continue;
                uint32_t seen = 0;
                std::function<bool(uint32_t)> aug = [&](uint32_t x) -> bool {
                    uint32_t cand = avail[x] & ~seen;
                    while (cand) {
                        const int c = __builtin_ctz(cand);
                        cand &= cand - 1;
                        seen |= 1u << c;
                        if (mc[c] < 0 || aug((uint32_t)mc[c])) {
                            mr[x] = c;
                            mc[c] = (int)x;
                            return true;
                        }
                    }
                    return false;
                };
                if (aug(r)) ++pairs;
            }
            for (uint32_t r = 0; r < 32; ++r)
                if (mr[r] >= 0) take(st, r, (uint32_t)mr[r]);
            sets.push_back(st);
            rot += 7;
        }
        ga = gb;
    }
    for (Set &st : sets) {
        for (int pass = 0; pass < 3 && st.got < st.k; ++pass)
            for (uint32_t r = 0; r < 32 && st.got < st.k; ++r) {
                if (!avail[r] || (pass < 2 && (st.used_rb >> r & 1))) continue;
                const uint32_t free_c = pass == 0 ? avail[r] & ~st.used_cb : avail[r];
                if (!free_c) continue;
                take(st, r, (uint32_t)__builtin_ctz(free_c));
                if (pass == 2)
                    while (st.got < st.k && avail[r]) take(st, r, (uint32_t)__builtin_ctz(avail[r]));
            }
    }
    for (uint32_t i = 0; i < n; ++i) {
        hp.pent[e0 + i] = ow[i];
        if (valued) std::memcpy(&hp.vval[(v0 + i) * vb], &ov[i], vb);
    }
}

}  // namespace

bool pack_panels(HostPanel &hp, const Canon &a, uint32_t m, const BuildOptions &bo, uint32_t nsm) {
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
    // section of an entry: 0 = +1, 1 = -1, 2 = valued (m = 2: 1 == m - 1 is +1)
    auto kind = [&](uint32_t v) -> int {
        if (seg && v == 1u) return 0;
        if (seg && m > 2 && v == m - 1) return 1;
        return 2;
    };

    // counts per tile and section; per (row, panel) bounds of the u32 sums:
    // +1 adds x <= m-1, -1 adds m - x <= m, valued adds (a x mod m) <= m-1, or
    // its Barrett remainder <= 2m-1 when lazy.
    std::vector<uint32_t> cnt(3 * T, 0);
    const uint64_t m1 = m - 1;
    uint64_t worst_exact = 0, worst_lazy = 0;
    for (uint64_t r = 0; r < a.nrows; ++r) {
        const uint64_t b = r / g.R;
        uint64_t p_cur = ~0ull, k[3] = {0, 0, 0};
        auto close = [&]() {
            worst_exact = std::max(worst_exact, k[0] * m1 + k[1] * m + k[2] * m1);
            worst_lazy = std::max(worst_lazy, k[0] * m1 + k[1] * m + k[2] * (2 * (uint64_t)m - 1));
            k[0] = k[1] = k[2] = 0;
        };
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            const uint64_t p = a.idx[t] / g.W;
            if (p != p_cur) { close(); p_cur = p; }
            const int s = kind(a.val[t]);
            k[s]++;
            cnt[3 * (p * g.B + b) + s]++;
        }
        close();
    }
    if (!g.split) {
        if (worst_exact >= (1ull << 32)) return false;
        g.lazy = worst_lazy < (1ull << 32) ? 1 : 0;
    }
    // tiles: quad offsets (panel-major), value quad offsets
    hp.tiles.resize(T);
    uint64_t q = 0, vq = 0;
    for (uint64_t t = 0; t < T; ++t) {
        PanelTile &tl = hp.tiles[t];
        tl.q0 = (uint32_t)q;
        tl.nqp = (cnt[3 * t] + 3) / 4;
        tl.nqm = (cnt[3 * t + 1] + 3) / 4;
        tl.nqv = (cnt[3 * t + 2] + 3) / 4;
        tl.vq0 = (uint32_t)vq;
        tl.p = (uint32_t)(t / g.B);
        tl.b = (uint32_t)(t % g.B);
        tl.rn = (uint32_t)std::min<uint64_t>(g.R, a.nrows - (uint64_t)tl.b * g.R);
        q += tl.nqp + tl.nqm + tl.nqv;
        vq += tl.nqv;
        hp.nnz_pm += cnt[3 * t] + cnt[3 * t + 1];
        hp.nnz_val += cnt[3 * t + 2];
    }
    if (q >= (1ull << 30)) throw std::bad_alloc();   // quad offsets are u32 word/4 indices
    const uint32_t dummy = g.R;                     // byte offset 0, spare row R
    hp.pent.assign(4 * q, dummy);
    hp.vval.assign(4 * vq * vb, 0);
    // fill: rows in order -> each section comes out sorted by (row, col)
    std::vector<uint64_t> cur(3 * T);
    for (uint64_t t = 0; t < T; ++t) {
        const PanelTile &tl = hp.tiles[t];
        cur[3 * t] = 4ull * tl.q0;
        cur[3 * t + 1] = 4ull * (tl.q0 + tl.nqp);
        cur[3 * t + 2] = 4ull * (tl.q0 + tl.nqp + tl.nqm);
    }
    for (uint64_t r = 0; r < a.nrows; ++r) {
        const uint64_t b = r / g.R;
        const uint32_t rl = (uint32_t)(r - b * g.R);
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            const uint32_t c = a.idx[t], v = a.val[t];
            const uint64_t p = c / g.W;
            const uint64_t tile = p * g.B + b;
            const int s = kind(v);
            const uint64_t at = cur[3 * tile + s]++;
            hp.pent[at] = ((uint32_t)(c - p * g.W) * g.xbytes) << g.rs | rl;
            if (s == 2) {
                const PanelTile &tl = hp.tiles[tile];
                const uint64_t vi = 4ull * tl.vq0 + (at - 4ull * (tl.q0 + tl.nqp + tl.nqm));
                std::memcpy(&hp.vval[vi * vb], &v, vb);
            }
        }
    }
    // Shared-memory bank order: warp w processes tile quads [32 j, 32 j + 32)
    // in one pass, entry u of every quad in the same instruction (a gather of
    // x and an atomic add into acc).  Inside each such group and section the
    // entries are reassigned to (quad, u) slots so that the 32 entries of one
    // instruction hit distinct banks of acc (row mod 32) and of the x panel
    // (4-byte word of the column mod 32) where possible.
    for (uint64_t t = 0; t < T; ++t) {
        const PanelTile &tl = hp.tiles[t];
        const uint32_t sec[4] = {0, tl.nqp, tl.nqp + tl.nqm, tl.nqp + tl.nqm + tl.nqv};
        for (int k = 0; k < 3; ++k) arrange_section(hp, tl, g, vb, sec[k], sec[k + 1], k == 2);
    }
    // CTA schedule: contiguous tile ranges (panel-major, so a CTA reloads its
    // x panel only when its range crosses a panel boundary), balanced by
    // entries + the per-tile band write-out.
    std::vector<double> cost(T);
    double total = 0;
    for (uint64_t t = 0; t < T; ++t) {
        const PanelTile &tl = hp.tiles[t];
        cost[t] = 4.0 * (tl.nqp + tl.nqm + tl.nqv) + 0.5 * (double)tl.rn;
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
    hp.stream_bytes = 16 * q + 4 * vq * vb + T * sizeof(PanelTile);
    return true;
}

uint64_t reconstruct_panels(const HostPanel &hp, uint32_t m, uint32_t vb, uint32_t *rr,
                            uint32_t *rc, uint32_t *rv, uint64_t cap) {
    uint64_t n = 0;
    const PanelGeom &g = hp.g;
    const uint32_t rmask = (1u << g.rs) - 1;
    for (const PanelTile &tl : hp.tiles) {
        const uint64_t e0 = 4ull * tl.q0, e1 = e0 + 4ull * tl.nqp, e2 = e1 + 4ull * tl.nqm,
                       e3 = e2 + 4ull * tl.nqv;
        for (uint64_t e = e0; e < e3; ++e) {
            const uint32_t w = hp.pent[e];
            if ((w & rmask) == g.R) {           // padding
                if ((w >> g.rs) != 0) return ~0ull;
                continue;
            }
            uint32_t v;
            if (e < e1) {
                v = 1u;
            } else if (e < e2) {
                v = m - 1;
            } else {
                v = 0;
                std::memcpy(&v, &hp.vval[(4ull * tl.vq0 + (e - e2)) * vb], vb);
            }
            const uint32_t off = w >> g.rs;
            if (off % g.xbytes) return ~0ull;
            if (n < cap) {
                rr[n] = tl.b * g.R + (w & rmask);
                rc[n] = tl.p * g.W + off / g.xbytes;
                rv[n] = v;
            }
            ++n;
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
