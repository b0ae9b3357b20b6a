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
