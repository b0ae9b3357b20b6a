// Dataflow schedule for indirect-increment loops (derived from a plan; the plan
// itself — reference plan.py:55-131 — is unchanged).
//
// The queue visits blocks in (window, colour, index) order: the iteration set
// is cut into `nwindows` ranges of consecutive blocks, and inside a window the
// plan's block colours are visited in order.  A window's working set is sized
// to fit the 126 MB L2, so node data shared by neighbouring blocks of different
// colours is re-read from L2, not HBM.  Two blocks that share a write target
// never run their write-backs concurrently: the later one in the queue waits for
// the earlier one (its dependency).  Dependencies always point backwards in the
// queue, so a persistent grid that dequeues in order cannot deadlock; the
// queue order is fixed, so every target receives its increments in a fixed
// order — results are deterministic run to run.
#include <algorithm>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <vector>

#include "ml_common.h"

struct ml_schedule {
    bool ok = true;                    // false: a hub target makes deps quadratic
    std::vector<int32_t> queue, dep_off, dep_list;
};

extern "C" int ml_schedule_build(int64_t n, int32_t ncols, const int64_t *const *cols,
                                 const int32_t *col_key, int64_t block_size,
                                 const int64_t *block_color, int32_t nwindows, ml_schedule_t **out) {
    if (!out || n < 0 || ncols < 0 || block_size < 1 || nwindows < 1)
        ML_FAIL(ML_EINVAL, "ml_schedule_build: bad arguments");
    ML_GUARD_BEGIN
    auto s = std::make_unique<ml_schedule>();
    const int64_t nb = n ? (n + block_size - 1) / block_size : 0;
    // queue: (window, colour, block)
    s->queue.resize(nb);
    for (int64_t b = 0; b < nb; ++b) s->queue[b] = int32_t(b);
    auto window = [&](int64_t b) { return b * nwindows / std::max<int64_t>(nb, 1); };
    std::stable_sort(s->queue.begin(), s->queue.end(), [&](int32_t x, int32_t y) {
        const int64_t wx = window(x), wy = window(y);
        if (wx != wy) return wx < wy;
        return block_color[x] < block_color[y];
    });
    std::vector<int32_t> pos(nb);
    for (int64_t q = 0; q < nb; ++q) pos[s->queue[q]] = int32_t(q);

    // exact write targets: one id range per dat key
    std::vector<int64_t> base(ncols, 0);
    {
        std::vector<std::pair<int32_t, int64_t>> key_hi;   // key -> max id over all its columns
        for (int32_t j = 0; j < ncols; ++j) {
            int64_t mx = -1;
            for (int64_t e = 0; e < n; ++e) mx = std::max(mx, cols[j][e]);
            bool found = false;
            for (auto &kh : key_hi)
                if (kh.first == col_key[j]) {
                    kh.second = std::max(kh.second, mx);
                    found = true;
                }
            if (!found) key_hi.emplace_back(col_key[j], mx);
        }
        int64_t off = 0;
        std::vector<std::pair<int32_t, int64_t>> key_base;
        for (auto &kh : key_hi) {
            key_base.emplace_back(kh.first, off);
            off += kh.second + 1;
        }
        for (int32_t j = 0; j < ncols; ++j)
            for (auto &kb : key_base)
                if (kb.first == col_key[j]) base[j] = kb.second;
    }
    std::vector<std::pair<int64_t, int32_t>> tb;   // (target, block), unique
    tb.reserve(size_t(n) * ncols);
    for (int32_t j = 0; j < ncols; ++j)
        for (int64_t e = 0; e < n; ++e) tb.emplace_back(cols[j][e] + base[j], int32_t(e / block_size));
    std::sort(tb.begin(), tb.end());
    tb.erase(std::unique(tb.begin(), tb.end()), tb.end());
    std::vector<std::pair<int32_t, int32_t>> edges;   // (later block, earlier block)
    for (size_t i = 0; i < tb.size() && s->ok;) {
        size_t k = i;
        while (k < tb.size() && tb[k].first == tb[i].first) ++k;
        if (k - i > 512) {
            s->ok = false;
            break;
        }
        for (size_t a = i; a < k; ++a)
            for (size_t c = a + 1; c < k; ++c) {
                int32_t x = tb[a].second, y = tb[c].second;
                if (pos[x] < pos[y]) std::swap(x, y);
                edges.emplace_back(x, y);
            }
        i = k;
    }
    if (s->ok) {
        std::sort(edges.begin(), edges.end());
        edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
        s->dep_off.assign(size_t(nb) + 1, 0);
        for (auto &ed : edges) s->dep_off[ed.first + 1]++;
        for (int64_t b = 0; b < nb; ++b) s->dep_off[b + 1] += s->dep_off[b];
        s->dep_list.resize(edges.size());
        for (size_t i = 0; i < edges.size(); ++i) s->dep_list[i] = edges[i].second;
    }
    *out = s.release();
    return ML_OK;
    ML_GUARD_END
}

extern "C" int ml_schedule_export(const ml_schedule_t *s, int64_t *ndeps, int32_t *queue,
                                  int32_t *dep_off, int32_t *dep_list) {
    if (!s) ML_FAIL(ML_EINVAL, "ml_schedule_export: null schedule");
    if (ndeps) *ndeps = s->ok ? int64_t(s->dep_list.size()) : -1;
    if (queue) std::copy(s->queue.begin(), s->queue.end(), queue);
    if (s->ok && dep_off) std::copy(s->dep_off.begin(), s->dep_off.end(), dep_off);
    if (s->ok && dep_list) std::copy(s->dep_list.begin(), s->dep_list.end(), dep_list);
    return ML_OK;
}

extern "C" int ml_schedule_free(ml_schedule_t *s) {
    delete s;
    return ML_OK;
}

// ---- target-centric ("gather") schedule ------------------------------------------------------
// For an INC loop whose indirect writes all increment one dat, every target
// element is owned by one thread, which re-evaluates the kernel for each
// (element, INC argument) that hits it and keeps only that argument's
// increment.  The incidence lists are ordered by (element, argument) — the
// order in which the reference serial executor (executor.py:206-217) applies
// the increments — so each target accumulates exactly the serial sequence,
// with no colouring, no atomics and no cross-thread conflicts.
struct ml_gather {
    std::vector<int32_t> off, elem;
    std::vector<uint8_t> pos;
};

extern "C" int ml_gather_build(int64_t n, int32_t ncols, const int64_t *const *cols, int64_t ntargets,
                               ml_gather_t **out) {
    if (!out || n < 0 || ncols < 1 || ncols > 255 || ntargets < 0)
        ML_FAIL(ML_EINVAL, "ml_gather_build: bad arguments");
    if (n * ncols >= (int64_t(1) << 31)) ML_FAIL(ML_EINVAL, "ml_gather_build: too many incidences");
    ML_GUARD_BEGIN
    auto g = std::make_unique<ml_gather>();
    g->off.assign(size_t(ntargets) + 1, 0);
    for (int32_t j = 0; j < ncols; ++j)
        for (int64_t e = 0; e < n; ++e) {
            const int64_t t = cols[j][e];
            if (t < 0 || t >= ntargets) throw std::out_of_range("target outside the target set");
            g->off[t + 1]++;
        }
    for (int64_t t = 0; t < ntargets; ++t) g->off[t + 1] += g->off[t];
    g->elem.resize(size_t(n) * ncols);
    g->pos.resize(size_t(n) * ncols);
    std::vector<int32_t> fill(g->off.begin(), g->off.end() - 1);
    for (int64_t e = 0; e < n; ++e)          // element-major, then argument: serial order
        for (int32_t j = 0; j < ncols; ++j) {
            const int64_t t = cols[j][e];
            const int32_t k = fill[t]++;
            g->elem[k] = int32_t(e);
            g->pos[k] = uint8_t(j);
        }
    *out = g.release();
    return ML_OK;
    ML_GUARD_END
}

extern "C" int ml_gather_export(const ml_gather_t *g, int32_t *off, int32_t *elem, uint8_t *pos) {
    if (!g) ML_FAIL(ML_EINVAL, "ml_gather_export: null");
    if (off) std::copy(g->off.begin(), g->off.end(), off);
    if (elem) std::copy(g->elem.begin(), g->elem.end(), elem);
    if (pos) std::copy(g->pos.begin(), g->pos.end(), pos);
    return ML_OK;
}

extern "C" int ml_gather_free(ml_gather_t *g) {
    delete g;
    return ML_OK;
}
