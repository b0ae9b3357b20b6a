// Tile plan for indirect-increment loops (the B200 counterpart of OP2's block
// partitioning for locality; reference plan.py:55-131 builds contiguous
// blocks + colours, which this does not replace — it is a second, internal
// plan the kernels consume).
//
// The target set (e.g. nodes) is cut into *tiles*: compact clusters of targets
// grown greedily over the mesh graph.  A tile OWNS its targets: it evaluates
// every element that increments one of them, so the increments of an owned
// target are all produced inside one CTA and applied there — no colours
// between CTAs, no atomics, no partial sums.  Elements whose targets belong
// to two tiles (the cut) are evaluated by both; each keeps only the
// increments of its own targets.  A tile's working set — owned targets plus
// the targets its elements read (its halo) — is staged in shared memory once,
// so each element's gathers are shared-memory reads: cluster compactness is
// what turns L2->SM traffic from "every incidence" into "every staged node".
//
// Growth: seeds in ascending target id; a tile adds the frontier target that
// stages the fewest new targets (ties: lowest id) while the shared-memory
// budget (stage_bytes per staged target + own_bytes per owned target) and
// the owned-count cap hold.
//
// Per tile, exported:
//   list      staged targets: owned first (ascending), then halo (ascending)
//   nown      owned count;  list_off  offsets of the staged lists
//   elem      elements evaluated (ascending);  elem_off  offsets
//   loc       per element, per map column: local index in the staged list
//   ecol      per element: colour (bits 0-6) among elements sharing an owned
//             INC target in this tile (applied in colour phases), bit 7 set
//             when this tile is the element's reduction owner (the tile that
//             owns its `red_col` target), so globals count each element once
//   ncol      colours of the tile
#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <vector>

#include "ml_common.h"

struct ml_tile {
    std::vector<int32_t> list_off, nown, list, elem_off, elem, ncol;
    // per owned target: its incidences (element index in the tile, map column)
    // in element-then-column order — the tile-gather variant's lists
    std::vector<int32_t> inc_base, inc_off;
    std::vector<uint16_t> inc_k;
    std::vector<uint8_t> inc_c;
    std::vector<uint16_t> loc;
    std::vector<uint8_t> ecol;
    int64_t umax = 0, cmax = 0, emax = 0;
    int32_t maxcol = 0;
};

namespace {

constexpr int MAX_TILE_COLOURS = 127;

struct Csr {
    std::vector<int64_t> off;
    std::vector<int32_t> val;
};

}  // namespace

extern "C" int ml_tile_build(int64_t n, int32_t arity, const int64_t *table, int64_t ntargets,
                             uint32_t inc_mask, int32_t red_col, int64_t stage_bytes,
                             int64_t own_bytes, int64_t budget, int32_t cmax, const double *coords,
                             int32_t cdim, ml_tile_t **out) {
    if (!out || n < 0 || arity < 1 || arity > 32 || ntargets < 0 || (n && !table) || stage_bytes < 0 ||
        own_bytes < 0 || budget < 1 || cmax < 1 || red_col < 0 || red_col >= arity ||
        (inc_mask & ((arity < 32 ? (1u << arity) : 0u) - 1u)) == 0)
        ML_FAIL(ML_EINVAL, "ml_tile_build: bad arguments");
    if (n >= (int64_t(1) << 31) || ntargets >= (int64_t(1) << 31))
        ML_FAIL(ML_EINVAL, "ml_tile_build: sets beyond int32 ids");
    ML_GUARD_BEGIN
    auto t = std::make_unique<ml_tile>();
    for (int64_t i = 0; i < n * arity; ++i)
        if (table[i] < 0 || table[i] >= ntargets) throw std::out_of_range("map entry outside the target set");

    // inc(v): elements incrementing v (ascending, deduplicated)
    Csr inc;
    inc.off.assign(size_t(ntargets) + 1, 0);
    for (int64_t e = 0; e < n; ++e)
        for (int c = 0; c < arity; ++c) {
            if (!(inc_mask >> c & 1)) continue;
            bool dup = false;
            for (int d = 0; d < c; ++d) dup |= (inc_mask >> d & 1) && table[e * arity + d] == table[e * arity + c];
            if (!dup) inc.off[table[e * arity + c] + 1]++;
        }
    for (int64_t v = 0; v < ntargets; ++v) inc.off[v + 1] += inc.off[v];
    inc.val.resize(size_t(inc.off[ntargets]));
    {
        std::vector<int64_t> fill(inc.off.begin(), inc.off.end() - 1);
        for (int64_t e = 0; e < n; ++e)
            for (int c = 0; c < arity; ++c) {
                if (!(inc_mask >> c & 1)) continue;
                bool dup = false;
                for (int d = 0; d < c; ++d)
                    dup |= (inc_mask >> d & 1) && table[e * arity + d] == table[e * arity + c];
                if (!dup) inc.val[fill[table[e * arity + c]]++] = int32_t(e);
            }
    }
    // nbr(v): targets a tile owning v must stage (every column of inc(v)), incl. v
    Csr nbr;
    nbr.off.assign(size_t(ntargets) + 1, 0);
    {
        std::vector<int32_t> stamp(size_t(ntargets), -1), tmp;
        for (int pass = 0; pass < 2; ++pass) {
            std::fill(stamp.begin(), stamp.end(), -1);
            if (pass == 1) {
                for (int64_t v = 0; v < ntargets; ++v) nbr.off[v + 1] += nbr.off[v];
                nbr.val.resize(size_t(nbr.off[ntargets]));
            }
            for (int64_t v = 0; v < ntargets; ++v) {
                tmp.clear();
                for (int64_t k = inc.off[v]; k < inc.off[v + 1]; ++k) {
                    const int64_t e = inc.val[k];
                    for (int c = 0; c < arity; ++c) {
                        const int64_t u = table[e * arity + c];
                        if (stamp[u] != int32_t(v)) {
                            stamp[u] = int32_t(v);
                            tmp.push_back(int32_t(u));
                        }
                    }
                }
                if (pass == 0) {
                    nbr.off[v + 1] = int64_t(tmp.size());
                } else {
                    std::sort(tmp.begin(), tmp.end());
                    std::copy(tmp.begin(), tmp.end(), nbr.val.begin() + nbr.off[v]);
                }
            }
        }
    }

    // ---- partition the incremented targets into tiles: recursive bisection ----
    std::vector<int32_t> pts;
    for (int64_t v = 0; v < ntargets; ++v)
        if (inc.off[v + 1] > inc.off[v]) pts.push_back(int32_t(v));
    std::vector<double> xyz;                                // [ntargets][3]
    int cd = 0;
    if (coords && cdim > 0) {
        cd = std::min(cdim, 3);
        xyz.assign(size_t(ntargets) * 3, 0.0);
        for (int64_t v = 0; v < ntargets; ++v)
            for (int k = 0; k < cd; ++k) xyz[v * 3 + k] = coords[v * cdim + k];
    } else {
        // pseudo-coordinates: hop distances from three far-apart landmarks
        cd = 3;
        xyz.assign(size_t(ntargets) * 3, 0.0);
        std::vector<int32_t> dist(static_cast<size_t>(ntargets)), mind(static_cast<size_t>(ntargets), INT32_MAX), bfs;
        int64_t land = pts.empty() ? 0 : pts[0];
        for (int k = 0; k < 4 && !pts.empty(); ++k) {
            std::fill(dist.begin(), dist.end(), -1);
            bfs.assign(1, int32_t(land));
            dist[land] = 0;
            for (size_t h = 0; h < bfs.size(); ++h) {
                const int32_t v = bfs[h];
                for (int64_t q = nbr.off[v]; q < nbr.off[v + 1]; ++q)
                    if (dist[nbr.val[q]] < 0) dist[nbr.val[q]] = dist[v] + 1, bfs.push_back(nbr.val[q]);
            }
            int32_t far = 0;
            for (int64_t v = 0; v < ntargets; ++v) far = std::max(far, dist[v]);
            if (k > 0)                                       // landmark 0 only seeds the first sweep
                for (int64_t v = 0; v < ntargets; ++v) xyz[v * 3 + (k - 1)] = dist[v] < 0 ? far + 1 : dist[v];
            int64_t best = land, bestd = -1;
            for (int32_t v : pts) {
                const int32_t d = dist[v] < 0 ? far + 1 : dist[v];
                if (k > 0) mind[v] = std::min(mind[v], d);
                const int64_t score = k == 0 ? d : mind[v];
                if (score > bestd) bestd = score, best = v;
            }
            land = best;
        }
    }
    std::vector<int32_t> staged(size_t(ntargets), -1);     // stamp: staged by the current set
    int32_t stamp = 0;
    auto staged_count = [&](const int32_t *a, const int32_t *b) {
        ++stamp;
        int64_t cnt = 0;
        for (const int32_t *p = a; p < b; ++p)
            for (int64_t q = nbr.off[*p]; q < nbr.off[*p + 1]; ++q)
                if (staged[nbr.val[q]] != stamp) staged[nbr.val[q]] = stamp, ++cnt;
        return cnt;
    };
    std::vector<int64_t> cut{0};                            // tile boundaries in pts
    std::vector<std::pair<int64_t, int64_t>> stack{{0, int64_t(pts.size())}};
    while (!stack.empty()) {
        auto [a, b] = stack.back();
        stack.pop_back();
        if (b <= a) continue;
        const int64_t m = b - a;
        if (m <= cmax && staged_count(pts.data() + a, pts.data() + b) * stage_bytes + m * own_bytes <= budget) {
            cut.push_back(b);
            continue;
        }
        if (m == 1)
            throw std::length_error("tile budget too small for target " + std::to_string(pts[a]) +
                                    " (stages " + std::to_string(nbr.off[pts[a] + 1] - nbr.off[pts[a]]) +
                                    " targets)");
        int ax = 0;
        double ext = -1;
        for (int k = 0; k < cd; ++k) {
            double lo = 1e300, hi = -1e300;
            for (int64_t i = a; i < b; ++i) lo = std::min(lo, xyz[pts[i] * 3 + k]), hi = std::max(hi, xyz[pts[i] * 3 + k]);
            if (hi - lo > ext) ext = hi - lo, ax = k;
        }
        const int64_t mid = a + (m + 1) / 2;
        std::nth_element(pts.begin() + a, pts.begin() + mid, pts.begin() + b, [&](int32_t x, int32_t y) {
            const double cx = xyz[int64_t(x) * 3 + ax], cy = xyz[int64_t(y) * 3 + ax];
            return cx < cy || (cx == cy && x < y);
        });
        stack.emplace_back(mid, b);                         // left half is processed first
        stack.emplace_back(a, mid);
    }

    std::vector<int32_t> owner(size_t(ntargets), -1);      // tile owning a target
    for (size_t k = 0; k + 1 < cut.size(); ++k)
        for (int64_t i = cut[k]; i < cut[k + 1]; ++i) owner[pts[i]] = int32_t(k);
    std::vector<int32_t> local(size_t(ntargets), 0);
    std::vector<int32_t> estamp(size_t(n), -1);
    std::vector<int32_t> owned, halo, elems;
    std::vector<uint64_t> used;                            // per owned target: colour mask (2 words)
    t->list_off.push_back(0);
    t->elem_off.push_back(0);
    for (size_t k = 0; k + 1 < cut.size(); ++k) {
        const int32_t tid = int32_t(k);
        owned.assign(pts.begin() + cut[k], pts.begin() + cut[k + 1]);
        ++stamp;
        halo.clear();
        for (int32_t v : owned)
            for (int64_t q = nbr.off[v]; q < nbr.off[v + 1]; ++q) {
                const int32_t u = nbr.val[q];
                if (staged[u] != stamp) {
                    staged[u] = stamp;
                    if (owner[u] != tid) halo.push_back(u);
                }
            }
        // staged list: owned ascending, then halo ascending
        std::sort(owned.begin(), owned.end());
        std::sort(halo.begin(), halo.end());
        int32_t li = 0;
        for (int32_t u : owned) local[u] = li++, t->list.push_back(u);
        for (int32_t u : halo) local[u] = li++, t->list.push_back(u);
        if (li > 65535) throw std::length_error("tile stages more than 65535 targets");
        t->list_off.push_back(int32_t(t->list.size()));
        t->nown.push_back(int32_t(owned.size()));
        // elements: every element incrementing an owned target, ascending
        elems.clear();
        for (int32_t v : owned)
            for (int64_t k = inc.off[v]; k < inc.off[v + 1]; ++k) {
                const int32_t e = inc.val[k];
                if (estamp[e] != tid) {
                    estamp[e] = tid;
                    elems.push_back(e);
                }
            }
        std::sort(elems.begin(), elems.end());
        // colours: greedy first fit over the element's owned INC targets
        used.assign(owned.size() * 2, 0);
        int32_t ncol = 0;
        for (int32_t e : elems) {
            uint64_t m0 = 0, m1 = 0;
            for (int c = 0; c < arity; ++c) {
                if (!(inc_mask >> c & 1)) continue;
                const int32_t l = local[table[int64_t(e) * arity + c]];
                if (l < int32_t(owned.size())) m0 |= used[2 * l], m1 |= used[2 * l + 1];
            }
            int col = 0;
            while (col < 128 && ((col < 64 ? m0 >> col : m1 >> (col - 64)) & 1)) ++col;
            if (col >= MAX_TILE_COLOURS)
                throw std::length_error("tile needs more than 127 colours (hub target)");
            for (int c = 0; c < arity; ++c) {
                if (!(inc_mask >> c & 1)) continue;
                const int32_t l = local[table[int64_t(e) * arity + c]];
                if (l < int32_t(owned.size())) used[2 * l + (col >> 6)] |= uint64_t(1) << (col & 63);
            }
            ncol = std::max(ncol, col + 1);
            const bool red_owner = owner[table[int64_t(e) * arity + red_col]] == tid;
            t->elem.push_back(e);
            t->ecol.push_back(uint8_t(col | (red_owner ? 0x80 : 0)));
            for (int c = 0; c < arity; ++c) t->loc.push_back(uint16_t(local[table[int64_t(e) * arity + c]]));
        }
        // owned-target incidence lists (element order, then column)
        {
            const int32_t C = int32_t(owned.size());
            const size_t e0 = t->elem.size() - elems.size();
            if (elems.size() > 65535) throw std::length_error("tile has more than 65535 elements");
            std::vector<int32_t> cnt(size_t(C) + 1, 0);
            for (size_t k = 0; k < elems.size(); ++k)
                for (int c = 0; c < arity; ++c)
                    if ((inc_mask >> c & 1) && t->loc[(e0 + k) * arity + c] < C)
                        cnt[t->loc[(e0 + k) * arity + c] + 1]++;
            for (int32_t j = 0; j < C; ++j) cnt[j + 1] += cnt[j];
            t->inc_base.push_back(int32_t(t->inc_off.size()));
            const int32_t kb = int32_t(t->inc_k.size());
            for (int32_t j = 0; j <= C; ++j) t->inc_off.push_back(kb + cnt[j]);
            t->inc_k.resize(size_t(kb) + cnt[C]);
            t->inc_c.resize(size_t(kb) + cnt[C]);
            std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
            for (size_t k = 0; k < elems.size(); ++k)
                for (int c = 0; c < arity; ++c) {
                    const int32_t l = t->loc[(e0 + k) * arity + c];
                    if ((inc_mask >> c & 1) && l < C) {
                        const int32_t q = kb + fill[l]++;
                        t->inc_k[q] = uint16_t(k);
                        t->inc_c[q] = uint8_t(c);
                    }
                }
        }
        t->elem_off.push_back(int32_t(t->elem.size()));
        t->ncol.push_back(ncol);
        t->umax = std::max<int64_t>(t->umax, li);
        t->cmax = std::max<int64_t>(t->cmax, int64_t(owned.size()));
        t->emax = std::max<int64_t>(t->emax, int64_t(elems.size()));
        t->maxcol = std::max(t->maxcol, ncol);
        if (t->elem.size() >= (size_t(1) << 31)) throw std::length_error("tile element lists beyond int32");
    }
    *out = t.release();
    return ML_OK;
    ML_GUARD_END
}

extern "C" int ml_tile_sizes(const ml_tile_t *t, int64_t *ntiles, int64_t *nlist, int64_t *nelem,
                             int64_t *umax, int64_t *cmax, int64_t *emax, int32_t *maxcol) {
    if (!t) ML_FAIL(ML_EINVAL, "ml_tile_sizes: null");
    if (ntiles) *ntiles = int64_t(t->nown.size());
    if (nlist) *nlist = int64_t(t->list.size());
    if (nelem) *nelem = int64_t(t->elem.size());
    if (umax) *umax = t->umax;
    if (cmax) *cmax = t->cmax;
    if (emax) *emax = t->emax;
    if (maxcol) *maxcol = t->maxcol;
    return ML_OK;
}

extern "C" int ml_tile_export(const ml_tile_t *t, int32_t *list_off, int32_t *nown, int32_t *list,
                              int32_t *elem_off, int32_t *elem, uint16_t *loc, uint8_t *ecol,
                              int32_t *ncol) {
    if (!t) ML_FAIL(ML_EINVAL, "ml_tile_export: null");
    if (list_off) std::copy(t->list_off.begin(), t->list_off.end(), list_off);
    if (nown) std::copy(t->nown.begin(), t->nown.end(), nown);
    if (list) std::copy(t->list.begin(), t->list.end(), list);
    if (elem_off) std::copy(t->elem_off.begin(), t->elem_off.end(), elem_off);
    if (elem) std::copy(t->elem.begin(), t->elem.end(), elem);
    if (loc) std::copy(t->loc.begin(), t->loc.end(), loc);
    if (ecol) std::copy(t->ecol.begin(), t->ecol.end(), ecol);
    if (ncol) std::copy(t->ncol.begin(), t->ncol.end(), ncol);
    return ML_OK;
}

extern "C" int ml_tile_export_incidences(const ml_tile_t *t, int64_t *ninc, int32_t *inc_base,
                                         int32_t *inc_off, uint16_t *inc_k, uint8_t *inc_c) {
    if (!t) ML_FAIL(ML_EINVAL, "ml_tile_export_incidences: null");
    if (ninc) *ninc = int64_t(t->inc_k.size());
    if (inc_base) std::copy(t->inc_base.begin(), t->inc_base.end(), inc_base);
    if (inc_off) std::copy(t->inc_off.begin(), t->inc_off.end(), inc_off);
    if (inc_k) std::copy(t->inc_k.begin(), t->inc_k.end(), inc_k);
    if (inc_c) std::copy(t->inc_c.begin(), t->inc_c.end(), inc_c);
    return ML_OK;
}

extern "C" int ml_tile_free(ml_tile_t *t) {
    delete t;
    return ML_OK;
}
