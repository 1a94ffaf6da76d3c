// Host format builder: SURVEY §8 rows a-1 .. a-4.
//
//   a-1 canonicalise   residues, duplicate sum, zero drop, (row, col) order
//                      (P:109-110 COO; readings R3-R5)
//   a-2 +-1 split      index-only stream with the sign in bit 31
//   a-3 bands/chooser  per row band: SELL (sliced ELL_R, rows sorted by
//                      length inside the band), CSR-vector, COO_S, plus the
//                      long-row tail
//   a-4 accumulator    u32 / u64 / u96 per slice from m and the row weights
//                      ("at most M/m^2 such accumulations")
#include <algorithm>
#include <cstring>
#include <numeric>

#include "internal.hpp"

namespace ffspmv {

typedef unsigned __int128 u128;

uint32_t value_bytes_for(uint32_t m) {
    // Stored values are residues in [2, m-2] (1 and m-1 go to the +-1 stream
    // unless segregation is off, then [1, m-1]): the narrowest unsigned type.
    if (m <= 256u) return 1;
    if (m <= 65536u) return 2;
    return 4;
}

DevMod make_mod(uint32_t m) {
    DevMod d;
    d.m = m;
    d.vbytes = value_bytes_for(m);
    u128 two64 = (u128)1 << 64;
    d.mu = (uint64_t)(two64 / m);
    d.r64 = (uint64_t)(two64 % m);
    d.mu32 = (uint32_t)std::min<uint64_t>((1ull << 32) / m, 0xFFFFFFFFull);
    d.r32 = (uint32_t)((1ull << 32) % m);
    return d;
}

static inline uint32_t residue(int64_t v, uint32_t m) {
    int64_t r = v % (int64_t)m;
    if (r < 0) r += (int64_t)m;
    return (uint32_t)r;
}

// Counting sort by major index, then sort each major segment by minor index,
// sum duplicates mod m and drop zero residues.
int canonicalize(Canon &out, uint64_t rows, uint64_t cols, uint64_t nnz, const uint32_t *ri,
                 const uint32_t *ci, const int64_t *v, uint32_t m, std::string &err) {
    out.nrows = rows;
    out.ncols = cols;
    std::vector<uint64_t> cnt(rows + 1, 0);
    for (uint64_t t = 0; t < nnz; ++t) {
        if (ri[t] >= rows || ci[t] >= cols) {
            err = "triple " + std::to_string(t) + " (" + std::to_string(ri[t]) + ", " +
                  std::to_string(ci[t]) + ") outside " + std::to_string(rows) + " x " +
                  std::to_string(cols);
            return 3;  // FFSPMV_ERR_INDEX
        }
        cnt[ri[t] + 1]++;
    }
    for (uint64_t r = 0; r < rows; ++r) cnt[r + 1] += cnt[r];
    std::vector<uint64_t> packed(nnz);
    {
        std::vector<uint64_t> pos(cnt.begin(), cnt.end() - 1);
        for (uint64_t t = 0; t < nnz; ++t)
            packed[pos[ri[t]]++] = ((uint64_t)ci[t] << 32) | residue(v[t], m);
    }
    out.ptr.assign(rows + 1, 0);
    out.idx.resize(nnz);
    out.val.resize(nnz);
    uint64_t w = 0;
    for (uint64_t r = 0; r < rows; ++r) {
        uint64_t b = cnt[r], e = cnt[r + 1];
        uint64_t *p = packed.data();
        if (e - b <= 32) {  // insertion sort: rows are short and often sorted
            for (uint64_t i = b + 1; i < e; ++i) {
                uint64_t key = p[i];
                uint64_t j = i;
                while (j > b && (p[j - 1] >> 32) > (key >> 32)) { p[j] = p[j - 1]; --j; }
                p[j] = key;
            }
        } else {
            std::stable_sort(p + b, p + e, [](uint64_t a, uint64_t c) { return (a >> 32) < (c >> 32); });
        }
        uint64_t i = b;
        while (i < e) {
            uint32_t col = (uint32_t)(p[i] >> 32);
            uint64_t s = 0;
            while (i < e && (uint32_t)(p[i] >> 32) == col) {
                s += (uint32_t)p[i];
                if (s >= m) s -= m;  // both terms < m: one subtraction
                ++i;
            }
            if (s) { out.idx[w] = col; out.val[w] = (uint32_t)s; ++w; }
        }
        out.ptr[r + 1] = w;
    }
    out.idx.resize(w);
    out.val.resize(w);
    return 0;
}

void transpose_canon(Canon &out, const Canon &a) {
    out.nrows = a.ncols;
    out.ncols = a.nrows;
    uint64_t nnz = a.idx.size();
    out.ptr.assign(out.nrows + 1, 0);
    for (uint64_t t = 0; t < nnz; ++t) out.ptr[a.idx[t] + 1]++;
    for (uint64_t r = 0; r < out.nrows; ++r) out.ptr[r + 1] += out.ptr[r];
    out.idx.resize(nnz);
    out.val.resize(nnz);
    std::vector<uint64_t> pos(out.ptr.begin(), out.ptr.end() - 1);
    for (uint64_t r = 0; r < a.nrows; ++r)   // rows visited in order -> sorted
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            uint64_t p = pos[a.idx[t]]++;
            out.idx[p] = (uint32_t)r;
            out.val[p] = a.val[t];
        }
}

namespace {

struct RowInfo {
    uint32_t lp, lv;     // +-1 and valued entry counts
};

// Worst-case accumulator content of a row: each +-1 addend is x or m - x
// (<= m), each valued addend a*x <= (m-1)^2.
static inline u128 row_bound(uint64_t lp, uint64_t lv, uint32_t m) {
    return (u128)lp * m + (u128)lv * (u128)(m - 1) * (u128)(m - 1);
}

static inline uint8_t regime_for(u128 bound, int force_bits) {
    uint8_t r;
    if (bound <= (u128)0xFFFFFFFFu) r = ACC32;
    else if (bound <= (u128)~(uint64_t)0) r = ACC64;
    else r = ACC96;
    if (force_bits >= 96) r = ACC96;
    else if (force_bits >= 64 && r < ACC64) r = ACC64;
    return r;
}

struct Packer {
    HostOp &op;
    const Canon &a;
    uint32_t m, vb;
    bool seg;
    const BuildOptions &bo;
    std::vector<RowInfo> info;
    // per-row entry lists are formed on the fly from the canonical CSR

    Packer(HostOp &o, const Canon &c, uint32_t mod, const BuildOptions &b)
        : op(o), a(c), m(mod), vb(value_bytes_for(mod)), bo(b) {}

    bool is_pm(uint32_t v) const {
        if (!seg) return false;
        return v == 1u || (m > 2 && v == m - 1);  // m = 2: 1 == -1 goes to "+1" (R9)
    }

    void put_val(uint32_t v) {
        size_t o = op.vval.size();
        op.vval.resize(o + vb);
        std::memcpy(&op.vval[o], &v, vb);  // little endian: low bytes
    }

    // Emit the +-1 entries of row r (in column order) into pcol, and the
    // valued entries into vcol/vval.
    void emit_row_entries(uint64_t r) {
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            uint32_t v = a.val[t];
            if (is_pm(v)) op.pcol.push_back(a.idx[t] | (v == 1u ? 0u : SIGN_BIT));
        }
        for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
            uint32_t v = a.val[t];
            if (!is_pm(v)) { op.vcol.push_back(a.idx[t]); put_val(v); }
        }
    }

    void update_acc_stats(uint8_t reg) {
        op.acc_cnt[reg]++;
        uint32_t bits = reg == ACC32 ? 32 : reg == ACC64 ? 64 : 96;
        op.acc_bits_max = std::max(op.acc_bits_max, bits);
    }

    // ---------------- SELL: rows sorted by (lv desc, lp desc, row) ----------
    void sell_order(std::vector<uint32_t> &rows) const {
        std::stable_sort(rows.begin(), rows.end(), [&](uint32_t x, uint32_t y) {
            if (info[x].lv != info[y].lv) return info[x].lv > info[y].lv;
            return info[x].lp > info[y].lp;
        });
    }

    uint64_t sell_cost(std::vector<uint32_t> rows) const {
        sell_order(rows);
        uint64_t bytes = 0;
        for (size_t s = 0; s < rows.size(); s += 32) {
            uint32_t wp = 0, wv = 0;
            for (size_t l = s; l < std::min(rows.size(), s + 32); ++l) {
                wp = std::max(wp, info[rows[l]].lp);
                wv = std::max(wv, info[rows[l]].lv);
            }
            bytes += 32ull * (wp * 4ull + wv * (4ull + vb)) + 32 * 4 + sizeof(SliceHdr);
        }
        return bytes;
    }

    void pack_sell(std::vector<uint32_t> rows, uint32_t band) {
        sell_order(rows);
        for (size_t s = 0; s < rows.size(); s += 32) {
            size_t n = std::min(rows.size() - s, (size_t)32);
            SliceHdr h{};
            uint32_t wp = 0, wv = 0;
            u128 bound = 0;
            for (size_t l = 0; l < n; ++l) {
                const RowInfo &ri = info[rows[s + l]];
                wp = std::max(wp, ri.lp);
                wv = std::max(wv, ri.lv);
                bound = std::max(bound, row_bound(ri.lp, ri.lv, m));
            }
            h.off_p = (uint32_t)op.pcol.size();
            h.off_v = (uint32_t)op.vcol.size();
            h.wp = (uint16_t)wp;
            h.wv = (uint16_t)wv;
            h.regime = regime_for(bound, bo.force_acc_bits);
            h.nrows = (uint8_t)n;
            h.band = (uint16_t)std::min<uint32_t>(band, 0xFFFF);
            update_acc_stats(h.regime);
            // per-lane entry lists
            std::vector<std::vector<uint32_t>> pl(32), vl(32), vv(32);
            for (size_t l = 0; l < n; ++l) {
                uint32_t r = rows[s + l];
                for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
                    uint32_t v = a.val[t];
                    if (is_pm(v)) pl[l].push_back(a.idx[t] | (v == 1u ? 0u : SIGN_BIT));
                    else { vl[l].push_back(a.idx[t]); vv[l].push_back(v); }
                }
            }
            for (uint32_t j = 0; j < wp; ++j)
                for (size_t l = 0; l < 32; ++l)
                    op.pcol.push_back(j < pl[l].size() ? pl[l][j] : PAD_COL);
            for (uint32_t j = 0; j < wv; ++j)
                for (size_t l = 0; l < 32; ++l) {
                    bool live = j < vl[l].size();
                    op.vcol.push_back(live ? vl[l][j] : PAD_COL);
                    put_val(live ? vv[l][j] : 0u);
                }
            for (size_t l = 0; l < 32; ++l) op.perm.push_back(l < n ? rows[s + l] : PAD_ROW);
            op.padded_slots += 32ull * (wp + wv);
            op.stream_bytes += 32ull * (wp * 4ull + wv * (4ull + vb)) + 32 * 4 + sizeof(SliceHdr);
            op.slices.push_back(h);
        }
    }

    // ---------------- CSR-vector / COO_S --------------------------------------
    static uint32_t lanes_for(double mean_len) {
        uint32_t v = 1;
        while (v < 32 && v < mean_len) v <<= 1;
        return v;
    }

    uint64_t csr_cost(const std::vector<uint32_t> &rows, bool coos) const {
        uint64_t bytes = 0, listed = 0;
        for (uint32_t r : rows) {
            const RowInfo &ri = info[r];
            if (coos && ri.lp + ri.lv == 0) { bytes += 4; continue; }  // zero-row list
            bytes += ri.lp * 4ull + ri.lv * (4ull + vb) + 8 + (coos ? 4 : 0);
            ++listed;
        }
        bytes += ((listed + 31) / 32) * sizeof(CsrGroup);
        return bytes + bytes / 10;  // lane-utilisation penalty (tunable)
    }

    void pack_csr(const std::vector<uint32_t> &rows, bool coos, uint32_t band) {
        std::vector<uint32_t> listed;
        uint64_t total = 0;
        for (uint32_t r : rows) {
            const RowInfo &ri = info[r];
            if (coos && ri.lp + ri.lv == 0) { op.zero_rows.push_back(r); op.stream_bytes += 4; continue; }
            listed.push_back(r);
            total += ri.lp + ri.lv;
        }
        if (listed.empty()) return;
        uint32_t V = lanes_for(listed.empty() ? 1.0 : (double)total / listed.size());
        uint32_t vlog = 0;
        while ((1u << vlog) < V) ++vlog;
        for (size_t g = 0; g < listed.size(); g += 32) {
            size_t n = std::min(listed.size() - g, (size_t)32);
            CsrGroup cg{};
            cg.first = (uint32_t)op.csr_rows.size();
            cg.nrows = (uint16_t)n;
            cg.vlog = (uint8_t)vlog;
            cg.band = band;
            u128 bound = 0;
            for (size_t i = 0; i < n; ++i) {
                uint32_t r = listed[g + i];
                bound = std::max(bound, row_bound(info[r].lp, info[r].lv, m));
                op.csr_rows.push_back(r);   // entries emitted by flush_csr()
                op.stream_bytes += info[r].lp * 4ull + info[r].lv * (4ull + vb) + 8 + (coos ? 4 : 0);
            }
            cg.regime = regime_for(bound, bo.force_acc_bits);
            update_acc_stats(cg.regime);
            op.groups.push_back(cg);
            op.stream_bytes += sizeof(CsrGroup);
        }
    }

    // All CSR / COO_S rows are emitted after every SELL band, contiguously,
    // so listed row i ends exactly where listed row i+1 starts.
    void flush_csr() {
        for (uint32_t r : op.csr_rows) {
            op.csr_pptr.push_back((uint32_t)op.pcol.size());
            op.csr_vptr.push_back((uint32_t)op.vcol.size());
            emit_row_entries(r);
        }
        op.csr_pptr.push_back((uint32_t)op.pcol.size());
        op.csr_vptr.push_back((uint32_t)op.vcol.size());
    }

    // ---------------- long-row tail ------------------------------------------
    void pack_long(const std::vector<uint32_t> &rows) {
        for (uint32_t r : rows) {
            const RowInfo &ri = info[r];
            uint32_t off_p = (uint32_t)op.pcol.size(), off_v = (uint32_t)op.vcol.size();
            emit_row_entries(r);
            uint64_t total = (uint64_t)ri.lp + ri.lv;
            uint32_t nch = (uint32_t)((total + bo.split_chunk - 1) / bo.split_chunk);
            if (nch < 1) nch = 1;
            uint32_t split = NO_SPLIT;
            if (nch > 1) { split = op.n_split++; op.split_rows++; }
            for (uint32_t c = 0; c < nch; ++c) {
                LongItem it{};
                it.row = r;
                uint32_t p0 = (uint32_t)((uint64_t)ri.lp * c / nch), p1 = (uint32_t)((uint64_t)ri.lp * (c + 1) / nch);
                uint32_t v0 = (uint32_t)((uint64_t)ri.lv * c / nch), v1 = (uint32_t)((uint64_t)ri.lv * (c + 1) / nch);
                it.off_p = off_p + p0; it.len_p = p1 - p0;
                it.off_v = off_v + v0; it.len_v = v1 - v0;
                it.split = split;
                it.chunk = c;
                uint8_t reg = regime_for(row_bound((it.len_p + 31) / 32, (it.len_v + 31) / 32, m),
                                         bo.force_acc_bits);
                it.nch_reg = nch | ((uint32_t)reg << 28);
                update_acc_stats(reg);
                op.longs.push_back(it);
            }
            op.long_rows++;
            op.stream_bytes += ri.lp * 4ull + ri.lv * (4ull + vb) + sizeof(LongItem) * nch;
        }
    }

    void run() {
        uint64_t rows = a.nrows;
        seg = bo.segregate_pm1 >= 0;
        info.resize(rows);
        uint64_t npm_all = 0;
        for (uint64_t r = 0; r < rows; ++r) {
            uint32_t lp = 0, lv = 0;
            for (uint64_t t = a.ptr[r]; t < a.ptr[r + 1]; ++t) {
                uint32_t v = a.val[t];
                if (v == 1u || (m > 2 && v == m - 1)) ++lp; else ++lv;
            }
            info[r] = {lp, lv};
            npm_all += lp;
        }
        // Auto: segregate when the +-1 entries are a noticeable share; with no
        // +-1 at all a second stream only adds slice headers.
        if (bo.segregate_pm1 == 0 && npm_all * 20 < a.idx.size()) seg = false;
        if (!seg)
            for (uint64_t r = 0; r < rows; ++r) { info[r].lv += info[r].lp; info[r].lp = 0; }
        for (uint64_t r = 0; r < rows; ++r) { op.nnz_pm += info[r].lp; op.nnz_val += info[r].lv; }
        op.nnz = a.idx.size();

        uint32_t br = std::max<uint32_t>(32, bo.band_rows / 32 * 32);
        std::vector<uint32_t> longs;
        for (uint64_t b0 = 0; b0 < rows; b0 += br) {
            uint32_t band = op.bands++;
            uint64_t b1 = std::min<uint64_t>(rows, b0 + br);
            std::vector<uint32_t> body;
            body.reserve(b1 - b0);
            for (uint64_t r = b0; r < b1; ++r) {
                if ((uint64_t)info[r].lp + info[r].lv > bo.long_row) longs.push_back((uint32_t)r);
                else body.push_back((uint32_t)r);
            }
            int fmt = bo.force_format;
            if (fmt == 0) {
                uint64_t cs = sell_cost(body);
                uint64_t cc = csr_cost(body, false);
                uint64_t co = csr_cost(body, true);
                fmt = 1;
                if (cc < cs) fmt = 2;
                if (co < std::min(cs, cc)) fmt = 3;
            }
            if (fmt == 1) { pack_sell(body, band); op.bands_sell++; }
            else if (fmt == 2) { pack_csr(body, false, band); op.bands_csr++; }
            else { pack_csr(body, true, band); op.bands_coos++; }
        }
        // longest rows first so they start in the first wave (tail balance)
        std::stable_sort(longs.begin(), longs.end(), [&](uint32_t x, uint32_t y) {
            return info[x].lp + info[x].lv > info[y].lp + info[y].lv;
        });
        flush_csr();
        pack_long(longs);
    }
};

}  // namespace

void pack_operator(HostOp &op, const Canon &a, uint32_t m, const BuildOptions &bo) {
    op = HostOp();
    op.rows = (uint32_t)a.nrows;
    op.cols = (uint32_t)a.ncols;
    Packer p(op, a, m, bo);
    p.run();
}

uint64_t reconstruct(const HostOp &op, uint32_t m, uint32_t vb, uint32_t *rr, uint32_t *rc,
                     uint32_t *rv, uint64_t cap) {
    uint64_t n = 0;
    auto emit = [&](uint32_t r, uint32_t c, uint32_t v) {
        if (n < cap) { rr[n] = r; rc[n] = c; rv[n] = v; }
        ++n;
    };
    auto val_at = [&](uint64_t i) {
        uint32_t v = 0;
        std::memcpy(&v, &op.vval[i * vb], vb);
        return v;
    };
    auto pm = [&](uint32_t r, uint32_t c) {
        if (c == PAD_COL) return;
        emit(r, c & COL_MASK, (c & SIGN_BIT) ? m - 1 : 1u);
    };
    for (size_t s = 0; s < op.slices.size(); ++s) {
        const SliceHdr &h = op.slices[s];
        for (uint32_t l = 0; l < 32; ++l) {
            uint32_t r = op.perm[s * 32 + l];
            for (uint32_t j = 0; j < h.wp; ++j) {
                uint32_t c = op.pcol[h.off_p + j * 32 + l];
                if (r == PAD_ROW) continue;
                pm(r, c);
            }
            for (uint32_t j = 0; j < h.wv; ++j) {
                uint64_t i = h.off_v + j * 32 + l;
                if (r == PAD_ROW || op.vcol[i] == PAD_COL) continue;
                emit(r, op.vcol[i], val_at(i));
            }
        }
    }
    for (const LongItem &it : op.longs) {
        for (uint32_t j = 0; j < it.len_p; ++j) pm(it.row, op.pcol[it.off_p + j]);
        for (uint32_t j = 0; j < it.len_v; ++j) emit(it.row, op.vcol[it.off_v + j], val_at(it.off_v + j));
    }
    for (const CsrGroup &g : op.groups)
        for (uint32_t i = g.first; i < g.first + g.nrows; ++i) {
            uint32_t r = op.csr_rows[i];
            for (uint32_t t = op.csr_pptr[i]; t < op.csr_pptr[i + 1]; ++t) pm(r, op.pcol[t]);
            for (uint32_t t = op.csr_vptr[i]; t < op.csr_vptr[i + 1]; ++t) emit(r, op.vcol[t], val_at(t));
        }
    return n;
}

}  // namespace ffspmv
