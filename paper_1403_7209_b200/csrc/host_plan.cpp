// Execution plan builder — bit-exact replacement of reference plan.py:55-131.
//
// Blocks are contiguous ranges of `block_size` iteration elements (the last
// ragged).  Write targets are (dat key, map column) ids made disjoint across
// dats with per-key offsets whose width is max(first column of the key)+1
// (the reference quirk at plan.py:77-81 is reproduced: later columns of the
// same dat may alias into the next key's range -> extra, safe conflicts).
//
// Block colouring (plan.py:82-103): greedy first fit in block order, a block
// avoiding the colours of lower-index blocks that share any write target.
// Processing blocks in order and recording, per target, the colour set of
// the blocks already coloured that touch it yields exactly that forbidden
// set, in O(refs * words) instead of building the block adjacency graph.
//
// Element colouring (plan.py:105-123): per block, in element order, the
// smallest colour unused by earlier elements of the block sharing a target.
// Blocks are independent, so this pass runs in parallel over blocks.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <unordered_map>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "ml_common.h"

struct ml_plan {
    int64_t n = 0, bs = 1, nb = 0, nc = 0, max_ecol = 1;
    std::vector<int32_t> block_color, elem_ncolors, elem_color;
    std::vector<int64_t> color_off;
    std::vector<int32_t> blocks_by_color;
};

namespace {

// Colour set per target: word 0 inline, higher words spilled to a map.
class ColourSets {
  public:
    explicit ColourSets(size_t ntargets) : w0_(ntargets, 0) {}

    void accumulate(int64_t t, std::vector<uint64_t> &acc) const {
        acc[0] |= w0_[t];
        if (!spill_.empty()) {
            auto it = spill_.find(t);
            if (it != spill_.end()) {
                const auto &w = it->second;
                if (acc.size() < w.size() + 1) acc.resize(w.size() + 1, 0);
                for (size_t i = 0; i < w.size(); ++i) acc[i + 1] |= w[i];
            }
        }
    }
    void add(int64_t t, int64_t c) {
        if (c < 64) {
            w0_[t] |= uint64_t(1) << c;
            return;
        }
        auto &w = spill_[t];
        size_t word = size_t(c / 64) - 1;
        if (w.size() <= word) w.resize(word + 1, 0);
        w[word] |= uint64_t(1) << (c % 64);
    }
    void clear(int64_t t) {
        w0_[t] = 0;
        if (!spill_.empty()) spill_.erase(t);
    }

  private:
    std::vector<uint64_t> w0_;
    std::unordered_map<int64_t, std::vector<uint64_t>> spill_;
};

inline int64_t lowest_free(const std::vector<uint64_t> &acc) {
    for (size_t i = 0; i < acc.size(); ++i)
        if (~acc[i]) return int64_t(i) * 64 + __builtin_ctzll(~acc[i]);
    return int64_t(acc.size()) * 64;
}

// Element colouring of one block, with a block-local target -> colour-set map.
struct BlockColourer {
    std::unordered_map<int64_t, std::vector<uint64_t>> sets;
    std::vector<uint64_t> acc;

    int64_t colour_block(int64_t lo, int64_t hi, int32_t ncols, const int64_t *const *cols,
                         const int64_t *base, int32_t *ecol) {
        sets.clear();
        int64_t top = 0;
        for (int64_t e = lo; e < hi; ++e) {
            acc.assign(1, 0);
            for (int32_t j = 0; j < ncols; ++j) {
                auto it = sets.find(cols[j][e] + base[j]);
                if (it == sets.end()) continue;
                if (acc.size() < it->second.size()) acc.resize(it->second.size(), 0);
                for (size_t w = 0; w < it->second.size(); ++w) acc[w] |= it->second[w];
            }
            int64_t c = lowest_free(acc);
            ecol[e] = int32_t(c);
            top = std::max(top, c);
            size_t word = size_t(c / 64);
            for (int32_t j = 0; j < ncols; ++j) {
                auto &s = sets[cols[j][e] + base[j]];
                if (s.size() <= word) s.resize(word + 1, 0);
                s[word] |= uint64_t(1) << (c % 64);
            }
        }
        return top + 1;
    }
};

}  // namespace

extern "C" int ml_plan_build(int64_t n, int32_t ncols, const int64_t *const *cols,
                             const int32_t *col_key, int64_t block_size, ml_plan_t **out) {
    if (!out) ML_FAIL(ML_EINVAL, "ml_plan_build: null output");
    if (block_size < 1) ML_FAIL(ML_EINVAL, "block size must be >= 1, got %lld", (long long)block_size);
    if (n < 0 || ncols < 0) ML_FAIL(ML_EINVAL, "ml_plan_build: negative size");
    ML_GUARD_BEGIN
    auto p = std::make_unique<ml_plan>();
    p->n = n;
    p->bs = block_size;
    const int64_t nb = n ? (n + block_size - 1) / block_size : 0;
    p->nb = nb;
    p->block_color.assign(nb, 0);
    p->elem_ncolors.assign(nb, 1);
    p->elem_color.assign(n, 0);

    if (ncols > 0 && n > 0) {
        // per-key offsets; width from the FIRST column seen for each key
        std::vector<int64_t> base(ncols);
        std::vector<std::pair<int32_t, int64_t>> key_base;
        int64_t offset = 0;
        for (int32_t j = 0; j < ncols; ++j) {
            int64_t b = -1;
            for (auto &kb : key_base)
                if (kb.first == col_key[j]) b = kb.second;
            if (b < 0) {
                int64_t mx = -1;
                for (int64_t e = 0; e < n; ++e) mx = std::max(mx, cols[j][e]);
                key_base.emplace_back(col_key[j], offset);
                b = offset;
                offset += mx + 1;
            }
            base[j] = b;
        }
        int64_t ntargets = 0;
        for (int32_t j = 0; j < ncols; ++j) {
            int64_t mx = -1;
            for (int64_t e = 0; e < n; ++e) {
                if (cols[j][e] < 0) throw std::invalid_argument("negative map entry in plan column");
                mx = std::max(mx, cols[j][e]);
            }
            ntargets = std::max(ntargets, base[j] + mx + 1);
        }

        // block colouring: sequential greedy first fit in block order
        ColourSets used{static_cast<size_t>(ntargets)};
        std::vector<uint64_t> acc;
        int64_t nc = 0;
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t lo = b * block_size, hi = std::min(n, lo + block_size);
            acc.assign(1, 0);
            for (int32_t j = 0; j < ncols; ++j) {
                const int64_t *c = cols[j];
                const int64_t o = base[j];
                for (int64_t e = lo; e < hi; ++e) used.accumulate(c[e] + o, acc);
            }
            const int64_t col = lowest_free(acc);
            p->block_color[b] = int32_t(col);
            nc = std::max(nc, col + 1);
            for (int32_t j = 0; j < ncols; ++j) {
                const int64_t *c = cols[j];
                const int64_t o = base[j];
                for (int64_t e = lo; e < hi; ++e) used.add(c[e] + o, col);
            }
        }
        p->nc = nc;

        // element colouring: independent per block
        int64_t max_ecol = 1;
#pragma omp parallel reduction(max : max_ecol)
        {
            BlockColourer bc;
#pragma omp for schedule(dynamic, 64)
            for (int64_t b = 0; b < nb; ++b) {
                const int64_t lo = b * block_size, hi = std::min(n, lo + block_size);
                const int64_t k = bc.colour_block(lo, hi, ncols, cols, base.data(), p->elem_color.data());
                p->elem_ncolors[b] = int32_t(k);
                max_ecol = std::max(max_ecol, k);
            }
        }
        p->max_ecol = max_ecol;

    } else {
        p->nc = nb ? 1 : 0;
    }

    // blocks grouped by colour (stable), colour offsets
    p->color_off.assign(p->nc + 1, 0);
    for (int64_t b = 0; b < nb; ++b) p->color_off[p->block_color[b] + 1]++;
    for (int64_t c = 0; c < p->nc; ++c) p->color_off[c + 1] += p->color_off[c];
    p->blocks_by_color.assign(nb, 0);
    {
        std::vector<int64_t> fill(p->color_off.begin(), p->color_off.end() - (p->nc ? 1 : 0));
        if (p->nc == 0) fill.clear();
        for (int64_t b = 0; b < nb; ++b) p->blocks_by_color[fill[p->block_color[b]]++] = int32_t(b);
    }
    *out = p.release();
    return ML_OK;
    ML_GUARD_END
}

extern "C" int ml_plan_sizes(const ml_plan_t *p, int64_t *nblocks, int64_t *ncolors,
                             int64_t *max_elem_colors) {
    if (!p) ML_FAIL(ML_EINVAL, "ml_plan_sizes: null plan");
    if (nblocks) *nblocks = p->nb;
    if (ncolors) *ncolors = p->nc;
    if (max_elem_colors) *max_elem_colors = p->max_ecol;
    return ML_OK;
}

extern "C" int ml_plan_export(const ml_plan_t *p, int64_t *block_color, int64_t *elem_ncolors,
                              int64_t *color_offsets, int64_t *blocks_by_color,
                              int64_t *elem_color, int64_t *block_elem_order) {
    if (!p) ML_FAIL(ML_EINVAL, "ml_plan_export: null plan");
    ML_GUARD_BEGIN
    for (int64_t b = 0; b < p->nb; ++b) {
        if (block_color) block_color[b] = p->block_color[b];
        if (elem_ncolors) elem_ncolors[b] = p->elem_ncolors[b];
        if (blocks_by_color) blocks_by_color[b] = p->blocks_by_color[b];
    }
    if (color_offsets)
        for (int64_t c = 0; c <= p->nc; ++c) color_offsets[c] = p->color_off[c];
    if (elem_color)
        for (int64_t e = 0; e < p->n; ++e) elem_color[e] = p->elem_color[e];
    if (block_elem_order) {
        // per block: element ids stably sorted by element colour (counting sort)
        std::vector<int64_t> count;
        for (int64_t b = 0; b < p->nb; ++b) {
            const int64_t lo = b * p->bs, hi = std::min(p->n, lo + p->bs);
            count.assign(size_t(p->elem_ncolors[b]) + 1, 0);
            for (int64_t e = lo; e < hi; ++e) count[p->elem_color[e] + 1]++;
            for (size_t c = 1; c < count.size(); ++c) count[c] += count[c - 1];
            for (int64_t e = lo; e < hi; ++e) block_elem_order[lo + count[p->elem_color[e]]++] = e;
        }
    }
    return ML_OK;
    ML_GUARD_END
}

extern "C" int ml_plan_free(ml_plan_t *p) {
    delete p;
    return ML_OK;
}

// ---- staging lists for shared-memory increment accumulation -------------------------
// Per block and per group (one INC dat), the ascending unique targets of the
// group's columns over the block's elements, and for every (element, column)
// the target's position in that list (uint16: a block has <= 65535 targets).
struct ml_staging {
    int64_t n = 0, bs = 1, nb = 0;
    int32_t ngroups = 0;
    std::vector<std::vector<int32_t>> off, list;   // per group
    std::vector<int64_t> umax;                     // per group
    std::vector<std::vector<uint16_t>> loc;        // per column
    // segmented mode: per unique target (global index into list), its
    // contributing (arg position, element in block) slots in element order
    std::vector<std::vector<int32_t>> toff;        // per group [total+1]
    std::vector<std::vector<uint16_t>> src;        // per group
    // arrival mode: per list entry, the partial slot of a target shared by
    // several blocks (-1: the block owns the target alone); per target id,
    // the first slot and the number of blocks touching it
    std::vector<std::vector<int32_t>> pslot, poff, nblk;
    std::vector<int64_t> nslots;
};

extern "C" int ml_staging_build(int64_t n, int64_t block_size, int32_t ncols,
                                const int64_t *const *cols, const int32_t *col_group,
                                ml_staging_t **out) {
    if (!out || block_size < 1 || n < 0 || ncols < 0) ML_FAIL(ML_EINVAL, "ml_staging_build: bad arguments");
    ML_GUARD_BEGIN
    auto s = std::make_unique<ml_staging>();
    s->n = n;
    s->bs = block_size;
    s->nb = n ? (n + block_size - 1) / block_size : 0;
    int32_t ng = 0;
    for (int32_t j = 0; j < ncols; ++j) ng = std::max(ng, col_group[j] + 1);
    s->ngroups = ng;
    s->off.assign(ng, std::vector<int32_t>(size_t(s->nb) + 1, 0));
    s->list.assign(ng, {});
    s->umax.assign(ng, 0);
    s->loc.assign(ncols, std::vector<uint16_t>(size_t(n), 0));
    std::vector<int64_t> buf;
    s->toff.assign(ng, {});
    s->src.assign(ng, {});
    struct Ref { int64_t tgt; int32_t elem, pos; };
    std::vector<Ref> refs;
    for (int32_t g = 0; g < ng; ++g) {
        auto &list = s->list[g];
        auto &toff = s->toff[g];
        auto &src = s->src[g];
        toff.push_back(0);
        for (int64_t b = 0; b < s->nb; ++b) {
            const int64_t lo = b * block_size, hi = std::min(n, lo + block_size);
            buf.clear();
            refs.clear();
            int32_t pos = 0;
            for (int32_t j = 0; j < ncols; ++j)
                if (col_group[j] == g) {
                    for (int64_t e = lo; e < hi; ++e) {
                        buf.push_back(cols[j][e]);
                        refs.push_back({cols[j][e], int32_t(e - lo), pos});
                    }
                    ++pos;
                }
            std::sort(buf.begin(), buf.end());
            buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
            if (buf.size() > 65535) throw std::length_error("more than 65535 staged targets in one block");
            if (buf.size() && buf.back() >= (int64_t(1) << 31)) throw std::length_error("target id exceeds int32");
            s->umax[g] = std::max<int64_t>(s->umax[g], int64_t(buf.size()));
            for (int32_t j = 0; j < ncols; ++j)
                if (col_group[j] == g)
                    for (int64_t e = lo; e < hi; ++e)
                        s->loc[j][e] = uint16_t(std::lower_bound(buf.begin(), buf.end(), cols[j][e]) - buf.begin());
            for (int64_t t : buf) list.push_back(int32_t(t));
            s->off[g][b + 1] = int32_t(list.size());
            // contributions per target in element order, then argument order
            std::sort(refs.begin(), refs.end(), [](const Ref &x, const Ref &y) {
                if (x.tgt != y.tgt) return x.tgt < y.tgt;
                if (x.elem != y.elem) return x.elem < y.elem;
                return x.pos < y.pos;
            });
            size_t r = 0;
            for (int64_t t : buf) {
                while (r < refs.size() && refs[r].tgt == t) {
                    if (refs[r].elem > 255 || refs[r].pos > 255)
                        throw std::length_error("segmented staging needs block_size <= 256");
                    src.push_back(uint16_t(refs[r].pos * 256 + refs[r].elem));
                    ++r;
                }
                toff.push_back(int32_t(src.size()));
            }
        }
    }
    // arrival lists: blocks touching each target, in block order
    s->pslot.assign(ng, {});
    s->poff.assign(ng, {});
    s->nblk.assign(ng, {});
    s->nslots.assign(ng, 0);
    for (int32_t g = 0; g < ng; ++g) {
        const auto &list = s->list[g];
        int64_t ntgt = 0;
        for (int32_t t : list) ntgt = std::max<int64_t>(ntgt, int64_t(t) + 1);
        auto &nblk = s->nblk[g];
        auto &poff = s->poff[g];
        nblk.assign(size_t(ntgt), 0);
        for (int32_t t : list) nblk[t]++;
        poff.assign(size_t(ntgt), -1);
        int64_t slots = 0;
        for (int64_t t = 0; t < ntgt; ++t)
            if (nblk[t] > 1) {
                poff[t] = int32_t(slots);
                slots += nblk[t];
            }
        if (slots >= (int64_t(1) << 31)) throw std::length_error("too many partial slots");
        s->nslots[g] = slots;
        std::vector<int32_t> seen(size_t(ntgt), 0);
        auto &pslot = s->pslot[g];
        pslot.resize(list.size());
        for (size_t k = 0; k < list.size(); ++k) {     // list is block-major: block order
            const int32_t t = list[k];
            pslot[k] = nblk[t] > 1 ? poff[t] + seen[t]++ : -1;
        }
    }
    *out = s.release();
    return ML_OK;
    ML_GUARD_END
}

extern "C" int ml_staging_sizes(const ml_staging_t *s, int32_t g, int64_t *total, int64_t *umax) {
    if (!s || g < 0 || g >= s->ngroups) ML_FAIL(ML_EINVAL, "ml_staging_sizes: bad group");
    if (total) *total = int64_t(s->list[g].size());
    if (umax) *umax = s->umax[g];
    return ML_OK;
}

extern "C" int ml_staging_export(const ml_staging_t *s, int32_t g, int32_t *off, int32_t *list) {
    if (!s || g < 0 || g >= s->ngroups) ML_FAIL(ML_EINVAL, "ml_staging_export: bad group");
    if (off) std::copy(s->off[g].begin(), s->off[g].end(), off);
    if (list) std::copy(s->list[g].begin(), s->list[g].end(), list);
    return ML_OK;
}

extern "C" int ml_staging_export_loc(const ml_staging_t *s, int32_t col, uint16_t *loc) {
    if (!s || col < 0 || col >= int32_t(s->loc.size())) ML_FAIL(ML_EINVAL, "ml_staging_export_loc: bad column");
    std::copy(s->loc[col].begin(), s->loc[col].end(), loc);
    return ML_OK;
}

extern "C" int ml_staging_export_seg(const ml_staging_t *s, int32_t g, int64_t *nrefs, int32_t *toff,
                                     uint16_t *src) {
    if (!s || g < 0 || g >= s->ngroups) ML_FAIL(ML_EINVAL, "ml_staging_export_seg: bad group");
    if (nrefs) *nrefs = int64_t(s->src[g].size());
    if (toff) std::copy(s->toff[g].begin(), s->toff[g].end(), toff);
    if (src) std::copy(s->src[g].begin(), s->src[g].end(), src);
    return ML_OK;
}

extern "C" int ml_staging_export_arrival(const ml_staging_t *s, int32_t g, int64_t *ntargets,
                                         int64_t *nslots, int32_t *pslot, int32_t *poff, int32_t *nblk) {
    if (!s || g < 0 || g >= s->ngroups) ML_FAIL(ML_EINVAL, "ml_staging_export_arrival: bad group");
    if (ntargets) *ntargets = int64_t(s->nblk[g].size());
    if (nslots) *nslots = s->nslots[g];
    if (pslot) std::copy(s->pslot[g].begin(), s->pslot[g].end(), pslot);
    if (poff) std::copy(s->poff[g].begin(), s->poff[g].end(), poff);
    if (nblk) std::copy(s->nblk[g].begin(), s->nblk[g].end(), nblk);
    return ML_OK;
}

extern "C" int ml_staging_free(ml_staging_t *s) {
    delete s;
    return ML_OK;
}
