// Target-centric ("gather") incidence lists of an indirect-write loop: per
// target, its (element, written-argument) incidences in serial order (C++
// host code; consumed by the gather and primary-fold schedules).
#include <algorithm>
#include <cstdint>
#include <memory>
#include <new>
#include <stdexcept>
#include <vector>

#include "ml_common.h"

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
