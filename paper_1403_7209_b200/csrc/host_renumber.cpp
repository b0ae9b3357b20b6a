// Locality renumbering — replacement of reference renumber.py:53-128.
//
// ml_co_occurrence: adjacency of a set from the maps that target it; every
// column pair (i < j) of a row is an edge, self pairs dropped, symmetrised,
// de-duplicated, neighbours ascending (renumber.py:53-81).
//
// ml_cm_order: Cuthill–McKee (NOT reversed — the reference calls it RCM but
// never reverses, and its tests pin an ordered path to the identity):
// components in order of their lowest vertex; each traversal starts at the
// component's minimum (degree, index) vertex; unseen neighbours are appended
// in (degree, index) order (renumber.py:84-119).  Pre-sorting every
// adjacency list once by (degree, index) gives the same sequence as sorting
// the unseen subset at each visit.
#include <algorithm>
#include <cstdint>
#include <new>
#include <stdexcept>
#include <vector>

#include "ml_common.h"

extern "C" int ml_co_occurrence(int64_t n, int32_t nmaps, const int64_t *const *tables,
                                const int64_t *rows, const int32_t *arity, int64_t *indptr,
                                int64_t *indices, int64_t *nnz) {
    if (n < 0 || nmaps < 0 || !nnz) ML_FAIL(ML_EINVAL, "ml_co_occurrence: bad arguments");
    ML_GUARD_BEGIN
    std::vector<int64_t> deg(size_t(n) + 1, 0);
    for (int32_t m = 0; m < nmaps; ++m) {
        const int64_t *t = tables[m];
        const int32_t a = arity[m];
        for (int64_t r = 0; r < rows[m]; ++r)
            for (int32_t i = 0; i < a; ++i)
                for (int32_t j = i + 1; j < a; ++j) {
                    int64_t x = t[r * a + i], y = t[r * a + j];
                    if (x == y) continue;
                    if (x < 0 || x >= n || y < 0 || y >= n) throw std::out_of_range("map entry outside set");
                    deg[x + 1]++;
                    deg[y + 1]++;
                }
    }
    for (int64_t v = 0; v < n; ++v) deg[v + 1] += deg[v];
    std::vector<int64_t> adj(size_t(deg[n]));
    std::vector<int64_t> fill(deg.begin(), deg.end() - 1);
    for (int32_t m = 0; m < nmaps; ++m) {
        const int64_t *t = tables[m];
        const int32_t a = arity[m];
        for (int64_t r = 0; r < rows[m]; ++r)
            for (int32_t i = 0; i < a; ++i)
                for (int32_t j = i + 1; j < a; ++j) {
                    int64_t x = t[r * a + i], y = t[r * a + j];
                    if (x == y) continue;
                    adj[fill[x]++] = y;
                    adj[fill[y]++] = x;
                }
    }
    // sort + unique each row, compact
    int64_t total = 0;
    std::vector<int64_t> ptr(size_t(n) + 1, 0);
    for (int64_t v = 0; v < n; ++v) {
        auto b = adj.begin() + deg[v], e = adj.begin() + deg[v + 1];
        std::sort(b, e);
        auto u = std::unique(b, e);
        int64_t k = u - b;
        std::copy(b, u, adj.begin() + total);
        total += k;
        ptr[v + 1] = total;
    }
    *nnz = total;
    if (indices) {
        if (!indptr) ML_FAIL(ML_EINVAL, "ml_co_occurrence: indptr required with indices");
        std::copy(ptr.begin(), ptr.end(), indptr);
        std::copy(adj.begin(), adj.begin() + total, indices);
    }
    return ML_OK;
    ML_GUARD_END
}

extern "C" int ml_cm_order(int64_t n, const int64_t *indptr, const int64_t *indices,
                           int64_t *order) {
    if (n < 0 || (n && (!indptr || !order))) ML_FAIL(ML_EINVAL, "ml_cm_order: bad arguments");
    ML_GUARD_BEGIN
    std::vector<int64_t> degree(n);
    for (int64_t v = 0; v < n; ++v) degree[v] = indptr[v + 1] - indptr[v];
    // adjacency re-sorted by (degree, index)
    std::vector<int64_t> nb(indices, indices + (n ? indptr[n] : 0));
    for (int64_t v = 0; v < n; ++v)
        std::sort(nb.begin() + indptr[v], nb.begin() + indptr[v + 1], [&](int64_t a, int64_t b) {
            return degree[a] != degree[b] ? degree[a] < degree[b] : a < b;
        });
    std::vector<char> found(n, 0), seen(n, 0);
    std::vector<int64_t> comp;
    int64_t pos = 0;
    for (int64_t lead = 0; lead < n; ++lead) {
        if (found[lead]) continue;
        comp.clear();
        comp.push_back(lead);
        found[lead] = 1;
        for (size_t h = 0; h < comp.size(); ++h) {
            const int64_t v = comp[h];
            for (int64_t k = indptr[v]; k < indptr[v + 1]; ++k)
                if (!found[indices[k]]) {
                    found[indices[k]] = 1;
                    comp.push_back(indices[k]);
                }
        }
        int64_t start = comp[0];
        for (int64_t v : comp)
            if (degree[v] < degree[start] || (degree[v] == degree[start] && v < start)) start = v;
        int64_t head = pos;
        order[pos++] = start;
        seen[start] = 1;
        while (head < pos) {
            const int64_t v = order[head++];
            for (int64_t k = indptr[v]; k < indptr[v + 1]; ++k) {
                const int64_t w = nb[k];
                if (!seen[w]) {
                    seen[w] = 1;
                    order[pos++] = w;
                }
            }
        }
    }
    return ML_OK;
    ML_GUARD_END
}
