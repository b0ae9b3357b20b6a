// Experiment (not product code): the fused iflux+vflux loop's primary-fold
// pass 1 written by hand for three device layouts of the wide node dats, to
// measure how much of the loop's time is address arithmetic and latency
// rather than bytes.  Same arithmetic as csrc/functors_proxy.cu ProxyFluxes.
//
//   SOA    component c of node e at c*pitch + e        (runtime pitch: the engine today)
//   AOSOA  blocks of 32 nodes: (e/32)*32*D + c*32 + e%32  (compile-time component offsets)
//   x, w   AoS (dim 3) in every variant, as the auto-SOA policy stores them
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -shared
//        -Xcompiler -fPIC -o scripts/_exp_flux.so scripts/exp_flux_layout.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <cuda/std/type_traits>

namespace {

constexpr int NQ = 6, NG = 18, NLIM = 8, NAUX = 19;

struct Data {
    const double *w, *q, *x, *lim, *grad, *aux;
    double *res, *slots;
    const int32_t *off1, *elem1, *tl1, *rec, *slotpos;
    int64_t n1, pitch;
};

template <int LAY>
struct View {
    const double *p;
    int64_t pitch;
    __device__ __forceinline__ double operator[](int c) const {
        if constexpr (LAY == 0) return p[c * pitch];
        else if constexpr (LAY == 2) {       // padded AoS rows: 16-byte pair loads, pairs reused
            const double2 v = __ldg(reinterpret_cast<const double2 *>(p) + (c >> 1));
            return (c & 1) ? v.y : v.x;
        } else return p[c * 32];
    }
};
template <int D>
__host__ __device__ constexpr int padded() { return (D + 1) / 2 * 2; }

__device__ __forceinline__ double ld_keep(const double *p) {
    double v;
    asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream(const double *p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
// HINT 0: plain; 1: evict_last (own rows); 2: no_allocate (neighbour rows)
template <int LAY, int HINT>
struct HView {
    const double *p;
    int64_t pitch;
    __device__ __forceinline__ double operator[](int c) const {
        const double *q = LAY == 0 ? p + c * pitch : p + c * 32;
        if constexpr (HINT == 1) return ld_keep(q);
        else if constexpr (HINT == 2) return ld_stream(q);
        else return *q;
    }
};
template <int LAY, int D, int HINT>
__device__ __forceinline__ HView<LAY, HINT> hview(const double *base, int64_t e, int64_t pitch) {
    if constexpr (LAY == 0) return HView<LAY, HINT>{base + e, pitch};
    else return HView<LAY, HINT>{base + (e >> 5) * (32 * D) + (e & 31), pitch};
}

template <int LAY, int D>
__device__ __forceinline__ View<LAY> view(const double *base, int64_t e, int64_t pitch) {
    if constexpr (LAY == 0) return View<LAY>{base + e, pitch};
    else if constexpr (LAY == 2) return View<LAY>{base + e * padded<D>(), pitch};
    else return View<LAY>{base + (e >> 5) * (32 * D) + (e & 31), pitch};
}

template <int LAY, int D>
__device__ __forceinline__ int64_t idx(int64_t e, int c, int64_t pitch) {
    if constexpr (LAY == 0) return c * pitch + e;
    else if constexpr (LAY == 2) return e * padded<D>() + c;
    else return (e >> 5) * (32 * D) + c * 32 + (e & 31);
}

template <int LAY>
__device__ __forceinline__ void eval_edge(const Data &d, int64_t e, int64_t a, int64_t b, double *r1,
                                          double *r2) {
    const int64_t P = d.pitch;
    const double *w = d.w + e * 3, *x1 = d.x + a * 3, *x2 = d.x + b * 3;
    const auto q1 = view<LAY, NQ>(d.q, a, P), q2 = view<LAY, NQ>(d.q, b, P);
    const auto l1 = view<LAY, NLIM>(d.lim, a, P), l2 = view<LAY, NLIM>(d.lim, b, P);
    const auto g1 = view<LAY, NG>(d.grad, a, P), g2 = view<LAY, NG>(d.grad, b, P);
    const auto a1 = view<LAY, NAUX>(d.aux, a, P), a2 = view<LAY, NAUX>(d.aux, b, P);
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double an = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NLIM; ++j) {
            const double tt = l1[j] + l2[j];
            s = s + tt * tt;
        }
        const double lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s));
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double f = lam * (q2[v] - q1[v]);
            r1[v] = 0.0 + f;
            r2[v] = 0.0 - f;
        }
    }
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds2 = d0 * d0 + d1 * d1 + d2 * d2 + 1e-12;
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double wd = w0 * d0 + w1 * d1 + w2 * d2;
        double mu = 0.0;
#pragma unroll
        for (int j = 0; j < NAUX; ++j) mu = mu + (a1[j] + a2[j]);
        mu = 0.01 * mu / (2.0 * NAUX);
        const double awd = fabs(wd);
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const int bb = 3 * v;
            const double gx = 0.5 * (g1[bb] + g2[bb]);
            const double gy = 0.5 * (g1[bb + 1] + g2[bb + 1]);
            const double gz = 0.5 * (g1[bb + 2] + g2[bb + 2]);
            const double dq = q2[v] - q1[v];
            const double corr = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2;
            const double f = mu * (0.001 * (gx * w0 + gy * w1 + gz * w2) + corr * awd);
            r1[v] += f;
            r2[v] -= f;
        }
    }
}

__device__ __forceinline__ void store_slot(const Data &d, int64_t e, const double *r2) {
    double *dst = d.slots + int64_t(__ldg(d.slotpos + e)) * NQ;
#pragma unroll
    for (int c = 0; c < NQ; c += 2)
        __stcg(reinterpret_cast<double2 *>(dst + c), make_double2(r2[c], r2[c + 1]));
}

// thread per target, its primary edges in sequence (the engine's pfold pass 1)
template <int LAY, int MINB>
__global__ void __launch_bounds__(256 / (MINB > 2 ? 2 : 1), MINB) k_flux(const __grid_constant__ Data d) {
    const int64_t P = d.pitch;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < d.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = __ldg(d.tl1 + t);
        double run[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(tg, c, P)];
        for (int k = __ldg(d.off1 + t), ke = __ldg(d.off1 + t + 1); k < ke; ++k) {
            const int64_t e = __ldg(d.elem1 + k);
            const int64_t a = __ldg(d.rec + 2 * int64_t(k)), b = __ldg(d.rec + 2 * int64_t(k) + 1);
            double r1[NQ], r2[NQ];
            eval_edge<LAY>(d, e, a, b, r1, r2);
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] += r1[c];
            store_slot(d, e, r2);
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = run[c];
    }
}

// lane per edge: a warp takes whole rows (targets) whose primary edges fit in
// 32 lanes (wrow: first row of each warp task); the row's first lane adds the
// row's increments in edge order via shuffles
template <int LAY>
__global__ void __launch_bounds__(256) k_flux_lanes(const __grid_constant__ Data d, const int32_t *wrow,
                                                    int64_t ntask) {
    const int64_t P = d.pitch;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t w = wid; w < ntask; w += nw) {
        const int r0 = __ldg(wrow + w), rN = __ldg(wrow + w + 1);
        const int base = __ldg(d.off1 + r0), end = __ldg(d.off1 + rN);
        const int k = base + lane;
        const bool act = k < end;
        // segment starts: lane j <= r1-r0 marks the lane where row r0+j starts
        unsigned bit = 0;
        if (lane <= rN - r0) {
            const int st = __ldg(d.off1 + r0 + lane) - base;
            bit = st < 32 ? (1u << st) : 0u;
        }
        const unsigned starts = __reduce_or_sync(0xffffffffu, bit);
        const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
        const int lead = 31 - __clz(starts & upto);
        const bool is_lead = act && lead == lane;
        double r1[NQ], r2[NQ];
        if (act) {
            const int64_t e = __ldg(d.elem1 + k);
            const int64_t a = __ldg(d.rec + 2 * int64_t(k)), b = __ldg(d.rec + 2 * int64_t(k) + 1);
            eval_edge<LAY>(d, e, a, b, r1, r2);
            store_slot(d, e, r2);
        } else {
#pragma unroll
            for (int c = 0; c < NQ; ++c) r1[c] = 0.0;
        }
        // row length of this lane's row (leaders only matter)
        const unsigned after = starts & ~upto;
        const int nxt = after ? __ffs(after) - 1 : (end - base);
        const int len = act ? nxt - lane : 0;
        const int maxlen = __reduce_max_sync(0xffffffffu, is_lead ? len : 0);
        double run[NQ];
        int64_t tg = 0;
        if (is_lead) {
            tg = __ldg(d.tl1 + r0 + __popc(starts & upto) - 1);
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(tg, c, P)];
        }
        for (int j = 0; j < maxlen; ++j) {
            const int src = lane + j < 32 ? lane + j : 31;
#pragma unroll
            for (int c = 0; c < NQ; ++c) {
                const double v = __shfl_sync(0xffffffffu, r1[c], src);
                if (is_lead && j < len) run[c] += v;
            }
        }
        if (is_lead) {
#pragma unroll
            for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = run[c];
        }
    }
}

// lane per edge with per-lane records: lane record {a, b, e, slot row} (a < 0:
// idle lane) and per warp task the mask of lanes that start a row; the row's
// first lane (whose a is the row's target) loads the target's res early and
// adds the row's increments in edge order via shuffles
template <int LAY>
__global__ void __launch_bounds__(256) k_flux_lrec(const __grid_constant__ Data d, const int4 *lrec,
                                                   const uint32_t *tmask, int64_t ntask) {
    const int64_t P = d.pitch;
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t w = wid; w < ntask; w += nw) {
        const int4 r = __ldg(lrec + w * 32 + lane);
        const unsigned starts = __ldg(tmask + w);
        const bool act = r.x >= 0;
        const unsigned upto = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
        const bool is_lead = act && ((starts >> lane) & 1u);
        const unsigned after = starts & ~upto;
        const unsigned actm = __ballot_sync(0xffffffffu, act);
        const int nact = __popc(actm);
        const int nxt = after ? __ffs(after) - 1 : nact;
        const int len = is_lead ? nxt - lane : 0;
        double run[NQ];
        if (is_lead) {
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(r.x, c, P)];
        }
        double r1[NQ], r2[NQ];
        if (act) {
            eval_edge<LAY>(d, r.z, r.x, r.y, r1, r2);
            double *dst = d.slots + int64_t(r.w) * NQ;
#pragma unroll
            for (int c = 0; c < NQ; c += 2)
                __stcg(reinterpret_cast<double2 *>(dst + c), make_double2(r2[c], r2[c + 1]));
        } else {
#pragma unroll
            for (int c = 0; c < NQ; ++c) r1[c] = 0.0;
        }
        const int maxlen = __reduce_max_sync(0xffffffffu, len);
        for (int j = 0; j < maxlen; ++j) {
            const int src = lane + j < 32 ? lane + j : 31;
#pragma unroll
            for (int c = 0; c < NQ; ++c) {
                const double v = __shfl_sync(0xffffffffu, r1[c], src);
                if (j < len) run[c] += v;
            }
        }
        if (is_lead) {
#pragma unroll
            for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(r.x, c, P)] = run[c];
        }
    }
}

// thread per target, its primary edges evaluated K at a time in lockstep: the
// target's own components are loaded once per group and used by all K edges;
// per component the K increments are added to the target's running value in
// edge order (the same per-target order as k_flux)
template <int LAY, int K>
__global__ void __launch_bounds__(256, 2) k_flux_lock(const __grid_constant__ Data d) {
    const int64_t P = d.pitch;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < d.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = __ldg(d.tl1 + t);
        double run[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(a, c, P)];
        const auto q1 = view<LAY, NQ>(d.q, a, P);
        const auto l1 = view<LAY, NLIM>(d.lim, a, P);
        const auto g1 = view<LAY, NG>(d.grad, a, P);
        const auto a1 = view<LAY, NAUX>(d.aux, a, P);
        const double *x1 = d.x + a * 3;
        for (int k0 = __ldg(d.off1 + t), ke = __ldg(d.off1 + t + 1); k0 < ke; k0 += K) {
            const int nk = ke - k0 < K ? ke - k0 : K;
            int64_t e[K], b[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const int k = j < nk ? k0 + j : k0;           // idle slots repeat the first edge
                e[j] = __ldg(d.elem1 + k);
                b[j] = __ldg(d.rec + 2 * int64_t(k) + 1);
            }
            double d0[K], d1[K], d2[K], w0[K], w1[K], w2[K], lam[K], mu[K], ds2[K], awd[K];
            const double xa0 = x1[0], xa1 = x1[1], xa2 = x1[2];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const double *x2 = d.x + b[j] * 3, *w = d.w + e[j] * 3;
                d0[j] = x2[0] - xa0; d1[j] = x2[1] - xa1; d2[j] = x2[2] - xa2;
                w0[j] = w[0]; w1[j] = w[1]; w2[j] = w[2];
            }
            // iflux scalars
            double s[K];
#pragma unroll
            for (int j = 0; j < K; ++j) s[j] = 0.0;
#pragma unroll
            for (int c = 0; c < NLIM; ++c) {
                const double own = l1[c];
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const double tt = own + view<LAY, NLIM>(d.lim, b[j], P)[c];
                    s[j] = s[j] + tt * tt;
                }
            }
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const double ds = sqrt(d0[j] * d0[j] + d1[j] * d1[j] + d2[j] * d2[j]);
                const double an = sqrt(w0[j] * w0[j] + w1[j] * w1[j] + w2[j] * w2[j]);
                lam[j] = an / ((1.0 + ds) * (1.0 + 0.0625 * s[j]));
                ds2[j] = d0[j] * d0[j] + d1[j] * d1[j] + d2[j] * d2[j] + 1e-12;
                awd[j] = fabs(w0[j] * d0[j] + w1[j] * d1[j] + w2[j] * d2[j]);
                mu[j] = 0.0;
            }
#pragma unroll
            for (int c = 0; c < NAUX; ++c) {
                const double own = a1[c];
#pragma unroll
                for (int j = 0; j < K; ++j) mu[j] = mu[j] + (own + view<LAY, NAUX>(d.aux, b[j], P)[c]);
            }
#pragma unroll
            for (int j = 0; j < K; ++j) mu[j] = 0.01 * mu[j] / (2.0 * NAUX);
            double *slot[K];
#pragma unroll
            for (int j = 0; j < K; ++j) slot[j] = d.slots + int64_t(__ldg(d.slotpos + e[j])) * NQ;
#pragma unroll
            for (int v = 0; v < NQ; ++v) {
                const int bb = 3 * v;
                const double qa = q1[v], ga0 = g1[bb], ga1 = g1[bb + 1], ga2 = g1[bb + 2];
                double r2v[K];
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    const auto q2 = view<LAY, NQ>(d.q, b[j], P);
                    const auto g2 = view<LAY, NG>(d.grad, b[j], P);
                    const double dqi = q2[v] - qa;
                    const double fi = lam[j] * dqi;
                    const double gx = 0.5 * (ga0 + g2[bb]);
                    const double gy = 0.5 * (ga1 + g2[bb + 1]);
                    const double gz = 0.5 * (ga2 + g2[bb + 2]);
                    const double corr = (dqi - (gx * d0[j] + gy * d1[j] + gz * d2[j])) / ds2[j];
                    const double fv = mu[j] * (0.001 * (gx * w0[j] + gy * w1[j] + gz * w2[j]) + corr * awd[j]);
                    if (j < nk) run[v] += (0.0 + fi) + fv;
                    r2v[j] = (0.0 - fi) - fv;
                }
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (j < nk) __stcg(slot[j] + v, r2v[j]);
            }
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(a, c, P)] = run[c];
    }
}

// thread per target; the neighbour's (second endpoint's) rows are loaded into
// registers in one wave before the arithmetic, the next edge's record is
// prefetched while the current edge computes.  MINB CTAs of 256 per SM.
template <int LAY>
struct RegRow {
    double q[NQ], x[3], l[NLIM], g[NG], a[NAUX];
    __device__ __forceinline__ void load(const Data &d, int64_t b) {
        const int64_t P = d.pitch;
        const auto vq = view<LAY, NQ>(d.q, b, P);
        const auto vl = view<LAY, NLIM>(d.lim, b, P);
        const auto vg = view<LAY, NG>(d.grad, b, P);
        const auto va = view<LAY, NAUX>(d.aux, b, P);
#pragma unroll
        for (int c = 0; c < NQ; ++c) q[c] = vq[c];
#pragma unroll
        for (int c = 0; c < 3; ++c) x[c] = d.x[b * 3 + c];
#pragma unroll
        for (int c = 0; c < NLIM; ++c) l[c] = vl[c];
#pragma unroll
        for (int c = 0; c < NG; ++c) g[c] = vg[c];
#pragma unroll
        for (int c = 0; c < NAUX; ++c) a[c] = va[c];
    }
};

template <int LAY>
__device__ __forceinline__ void eval_edge_reg(const Data &d, int64_t e, int64_t a, const RegRow<LAY> &nb,
                                              double *r1, double *r2) {
    const int64_t P = d.pitch;
    const double *w = d.w + e * 3, *x1 = d.x + a * 3;
    const double *x2 = nb.x;
    const auto q1 = view<LAY, NQ>(d.q, a, P);
    const auto l1 = view<LAY, NLIM>(d.lim, a, P);
    const auto g1 = view<LAY, NG>(d.grad, a, P);
    const auto a1 = view<LAY, NAUX>(d.aux, a, P);
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double an = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NLIM; ++j) {
            const double tt = l1[j] + nb.l[j];
            s = s + tt * tt;
        }
        const double lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s));
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double f = lam * (nb.q[v] - q1[v]);
            r1[v] = 0.0 + f;
            r2[v] = 0.0 - f;
        }
    }
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds2 = d0 * d0 + d1 * d1 + d2 * d2 + 1e-12;
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double wd = w0 * d0 + w1 * d1 + w2 * d2;
        double mu = 0.0;
#pragma unroll
        for (int j = 0; j < NAUX; ++j) mu = mu + (a1[j] + nb.a[j]);
        mu = 0.01 * mu / (2.0 * NAUX);
        const double awd = fabs(wd);
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const int bb = 3 * v;
            const double gx = 0.5 * (g1[bb] + nb.g[bb]);
            const double gy = 0.5 * (g1[bb + 1] + nb.g[bb + 1]);
            const double gz = 0.5 * (g1[bb + 2] + nb.g[bb + 2]);
            const double dq = nb.q[v] - q1[v];
            const double corr = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2;
            const double f = mu * (0.001 * (gx * w0 + gy * w1 + gz * w2) + corr * awd);
            r1[v] += f;
            r2[v] -= f;
        }
    }
}

template <int LAY, int MINB>
__global__ void __launch_bounds__(256, MINB) k_flux_reg(const __grid_constant__ Data d) {
    const int64_t P = d.pitch;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < d.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = __ldg(d.tl1 + t);
        double run[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(tg, c, P)];
        int k = __ldg(d.off1 + t);
        const int ke = __ldg(d.off1 + t + 1);
        int64_t e = k < ke ? __ldg(d.elem1 + k) : 0;
        int64_t b = k < ke ? __ldg(d.rec + 2 * int64_t(k) + 1) : 0;
        for (; k < ke; ++k) {
            RegRow<LAY> nb;
            nb.load(d, b);
            const int64_t ecur = e;
            if (k + 1 < ke) {                      // next record while this edge computes
                e = __ldg(d.elem1 + k + 1);
                b = __ldg(d.rec + 2 * int64_t(k + 1) + 1);
            }
            double r1[NQ], r2[NQ];
            eval_edge_reg<LAY>(d, ecur, tg, nb, r1, r2);
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] += r1[c];
            store_slot(d, ecur, r2);
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = run[c];
    }
}

template <int LAY, int H1, int H2>
__device__ __forceinline__ void eval_edge_h(const Data &d, int64_t e, int64_t a, int64_t b, double *r1,
                                            double *r2) {
    const int64_t P = d.pitch;
    const double *w = d.w + e * 3, *x1 = d.x + a * 3, *x2 = d.x + b * 3;
    const auto q1 = hview<LAY, NQ, H1>(d.q, a, P);
    const auto q2 = hview<LAY, NQ, H2>(d.q, b, P);
    const auto l1 = hview<LAY, NLIM, H1>(d.lim, a, P);
    const auto l2 = hview<LAY, NLIM, H2>(d.lim, b, P);
    const auto g1 = hview<LAY, NG, H1>(d.grad, a, P);
    const auto g2 = hview<LAY, NG, H2>(d.grad, b, P);
    const auto a1 = hview<LAY, NAUX, H1>(d.aux, a, P);
    const auto a2 = hview<LAY, NAUX, H2>(d.aux, b, P);
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double an = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NLIM; ++j) {
            const double tt = l1[j] + l2[j];
            s = s + tt * tt;
        }
        const double lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s));
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double f = lam * (q2[v] - q1[v]);
            r1[v] = 0.0 + f;
            r2[v] = 0.0 - f;
        }
    }
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds2 = d0 * d0 + d1 * d1 + d2 * d2 + 1e-12;
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double wd = w0 * d0 + w1 * d1 + w2 * d2;
        double mu = 0.0;
#pragma unroll
        for (int j = 0; j < NAUX; ++j) mu = mu + (a1[j] + a2[j]);
        mu = 0.01 * mu / (2.0 * NAUX);
        const double awd = fabs(wd);
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const int bb = 3 * v;
            const double gx = 0.5 * (g1[bb] + g2[bb]);
            const double gy = 0.5 * (g1[bb + 1] + g2[bb + 1]);
            const double gz = 0.5 * (g1[bb + 2] + g2[bb + 2]);
            const double dq = q2[v] - q1[v];
            const double corr = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2;
            const double f = mu * (0.001 * (gx * w0 + gy * w1 + gz * w2) + corr * awd);
            r1[v] += f;
            r2[v] -= f;
        }
    }
}

// thread per target with cache hints (H1 own rows, H2 neighbour rows) and, with
// PF, the next edge's record prefetched while the current edge computes
template <int LAY, int H1, int H2, int PF>
__global__ void __launch_bounds__(256, 2) k_flux_h(const __grid_constant__ Data d) {
    const int64_t P = d.pitch;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < d.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = __ldg(d.tl1 + t);
        double run[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(tg, c, P)];
        int k = __ldg(d.off1 + t);
        const int ke = __ldg(d.off1 + t + 1);
        int64_t e = 0, b = 0;
        if (PF && k < ke) {
            e = __ldg(d.elem1 + k);
            b = __ldg(d.rec + 2 * int64_t(k) + 1);
        }
        for (; k < ke; ++k) {
            int64_t ecur, bcur;
            if (PF) {
                ecur = e;
                bcur = b;
                if (k + 1 < ke) {
                    e = __ldg(d.elem1 + k + 1);
                    b = __ldg(d.rec + 2 * int64_t(k + 1) + 1);
                }
            } else {
                ecur = __ldg(d.elem1 + k);
                bcur = __ldg(d.rec + 2 * int64_t(k) + 1);
            }
            double r1[NQ], r2[NQ];
            eval_edge_h<LAY, H1, H2>(d, ecur, tg, bcur, r1, r2);
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] += r1[c];
            store_slot(d, ecur, r2);
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = run[c];
    }
}

// warp-pair split: CTA = 4 warp pairs; pair p owns 32 targets (one per lane).
// Warp 2p (role A) loads q, grad, x, w and forms the per-component terms;
// warp 2p+1 (role B) loads lim, aux, x, w and forms the scalars lam and mu,
// handed to A through shared memory between two named barriers per edge.
// Same arithmetic (expression trees) as eval_edge.
__device__ __forceinline__ void bar_pair(int id) {
    asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

template <int LAY, int MINB>
__global__ void __launch_bounds__(256, MINB) k_flux_split(const __grid_constant__ Data d) {
    __shared__ double sh[4][2][32];
    const int64_t P = d.pitch;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, pair = warp >> 1;
    const bool roleA = (warp & 1) == 0;
    const int bid = 1 + pair;                     // named barrier per pair (0 is __syncthreads)
    for (int64_t t0 = (int64_t(blockIdx.x) * 4 + pair) * 32; t0 < d.n1; t0 += int64_t(gridDim.x) * 128) {
        const int64_t t = t0 + lane;
        const bool act = t < d.n1;
        const int64_t tg = act ? __ldg(d.tl1 + t) : 0;
        const int k0 = act ? __ldg(d.off1 + t) : 0, k1 = act ? __ldg(d.off1 + t + 1) : 0;
        int len = k1 - k0;
        // both warps of the pair walk max(len) steps in lockstep
        for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
        double run[NQ];
        if (roleA && act) {
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(tg, c, P)];
        }
        for (int j = 0; j < len; ++j) {
            const bool live = act && k0 + j < k1;
            const int k = k0 + j;
            int64_t e = 0, b = 0;
            if (live) {
                e = __ldg(d.elem1 + k);
                b = __ldg(d.rec + 2 * int64_t(k) + 1);
            }
            const double *x1 = d.x + tg * 3, *x2 = d.x + b * 3, *w = d.w + e * 3;
            if (!roleA) {
                double lam = 0.0, mu = 0.0;
                if (live) {
                    const auto l1 = view<LAY, NLIM>(d.lim, tg, P), l2 = view<LAY, NLIM>(d.lim, b, P);
                    const auto a1 = view<LAY, NAUX>(d.aux, tg, P), a2 = view<LAY, NAUX>(d.aux, b, P);
                    const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
                    const double ds = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
                    const double w0 = w[0], w1 = w[1], w2 = w[2];
                    const double an = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
                    double s = 0.0;
#pragma unroll
                    for (int jj = 0; jj < NLIM; ++jj) {
                        const double tt = l1[jj] + l2[jj];
                        s = s + tt * tt;
                    }
                    lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s));
#pragma unroll
                    for (int jj = 0; jj < NAUX; ++jj) mu = mu + (a1[jj] + a2[jj]);
                    mu = 0.01 * mu / (2.0 * NAUX);
                }
                sh[pair][0][lane] = lam;
                sh[pair][1][lane] = mu;
                bar_pair(bid);                        // values ready
                bar_pair(bid);                        // A has read them
            } else {
                double fq[NQ], dqs[NQ], corr[NQ];
                double awd = 0.0;
                if (live) {
                    const auto q1 = view<LAY, NQ>(d.q, tg, P), q2 = view<LAY, NQ>(d.q, b, P);
                    const auto g1 = view<LAY, NG>(d.grad, tg, P), g2 = view<LAY, NG>(d.grad, b, P);
                    const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
                    const double ds2 = d0 * d0 + d1 * d1 + d2 * d2 + 1e-12;
                    const double w0 = w[0], w1 = w[1], w2 = w[2];
                    const double wd = w0 * d0 + w1 * d1 + w2 * d2;
                    awd = fabs(wd);
#pragma unroll
                    for (int v = 0; v < NQ; ++v) {
                        const int bb = 3 * v;
                        const double gx = 0.5 * (g1[bb] + g2[bb]);
                        const double gy = 0.5 * (g1[bb + 1] + g2[bb + 1]);
                        const double gz = 0.5 * (g1[bb + 2] + g2[bb + 2]);
                        const double dq = q2[v] - q1[v];
                        dqs[v] = dq;
                        corr[v] = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2;
                        fq[v] = 0.001 * (gx * w0 + gy * w1 + gz * w2);
                    }
                }
                bar_pair(bid);
                const double lam = sh[pair][0][lane], mu = sh[pair][1][lane];
                bar_pair(bid);
                if (live) {
                    double r2[NQ];
#pragma unroll
                    for (int v = 0; v < NQ; ++v) {
                        const double fi = lam * dqs[v];
                        const double f = mu * (fq[v] + corr[v] * awd);
                        run[v] += (0.0 + fi) + f;
                        r2[v] = (0.0 - fi) - f;
                    }
                    store_slot(d, e, r2);
                }
            }
        }
        if (roleA && act) {
#pragma unroll
            for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = run[c];
        }
    }
}

// Own-row cache: the target's own rows of the dats in MASK (bit 0 q, 1 lim,
// 2 grad, 3 aux) are copied once per target into shared memory
// (component-major, stride blockDim) and the edge evaluations read them
// there; neighbour rows as in k_flux<0> (SOA).
template <class Q1, class L1, class G1, class A1>
__device__ __forceinline__ void eval_edge_v(const Data &d, int64_t e, int64_t a, int64_t b, Q1 q1, L1 l1,
                                            G1 g1, A1 a1, double *r1, double *r2) {
    const int64_t P = d.pitch;
    const double *w = d.w + e * 3, *x1 = d.x + a * 3, *x2 = d.x + b * 3;
    const auto q2 = view<0, NQ>(d.q, b, P);
    const auto l2 = view<0, NLIM>(d.lim, b, P);
    const auto g2 = view<0, NG>(d.grad, b, P);
    const auto a2 = view<0, NAUX>(d.aux, b, P);
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double an = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NLIM; ++j) {
            const double tt = l1[j] + l2[j];
            s = s + tt * tt;
        }
        const double lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s));
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double f = lam * (q2[v] - q1[v]);
            r1[v] = 0.0 + f;
            r2[v] = 0.0 - f;
        }
    }
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds2 = d0 * d0 + d1 * d1 + d2 * d2 + 1e-12;
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double wd = w0 * d0 + w1 * d1 + w2 * d2;
        double mu = 0.0;
#pragma unroll
        for (int j = 0; j < NAUX; ++j) mu = mu + (a1[j] + a2[j]);
        mu = 0.01 * mu / (2.0 * NAUX);
        const double awd = fabs(wd);
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const int bb = 3 * v;
            const double gx = 0.5 * (g1[bb] + g2[bb]);
            const double gy = 0.5 * (g1[bb + 1] + g2[bb + 1]);
            const double gz = 0.5 * (g1[bb + 2] + g2[bb + 2]);
            const double dq = q2[v] - q1[v];
            const double corr = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2;
            const double f = mu * (0.001 * (gx * w0 + gy * w1 + gz * w2) + corr * awd);
            r1[v] += f;
            r2[v] -= f;
        }
    }
}

struct SView {           // shared-memory own row, component stride = blockDim
    const double *p;
    __device__ __forceinline__ double operator[](int c) const { return p[c * 256]; }
};

template <int D>
__device__ __forceinline__ void cache_row(double *dst, const double *src, int64_t a, int64_t P) {
#pragma unroll
    for (int c = 0; c < D; ++c) dst[c * 256] = __ldg(src + c * P + a);
}

template <int MASK>
__global__ void __launch_bounds__(256, 2) k_flux_own(const __grid_constant__ Data d) {
    extern __shared__ double sm[];
    constexpr int OQ = 0, OL = OQ + ((MASK & 1) ? NQ : 0), OG = OL + ((MASK & 2) ? NLIM : 0),
                  OA = OG + ((MASK & 4) ? NG : 0);
    double *my = sm + threadIdx.x;
    const int64_t P = d.pitch;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < d.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = __ldg(d.tl1 + t);
        if constexpr (MASK & 1) cache_row<NQ>(my + OQ * 256, d.q, tg, P);
        if constexpr (MASK & 2) cache_row<NLIM>(my + OL * 256, d.lim, tg, P);
        if constexpr (MASK & 4) cache_row<NG>(my + OG * 256, d.grad, tg, P);
        if constexpr (MASK & 8) cache_row<NAUX>(my + OA * 256, d.aux, tg, P);
        double run[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] = d.res[c * P + tg];
        for (int k = __ldg(d.off1 + t), ke = __ldg(d.off1 + t + 1); k < ke; ++k) {
            const int64_t e = __ldg(d.elem1 + k);
            const int64_t a = __ldg(d.rec + 2 * int64_t(k)), b = __ldg(d.rec + 2 * int64_t(k) + 1);
            double r1[NQ], r2[NQ];
            auto pick = [&](auto cached, const double *base, int off) {
                if constexpr (decltype(cached)::value) return SView{my + off * 256};
                else return view<0, 1>(base, a, P);
            };
            eval_edge_v(d, e, a, b, pick(cuda::std::bool_constant<(MASK & 1) != 0>{}, d.q, OQ),
                        pick(cuda::std::bool_constant<(MASK & 2) != 0>{}, d.lim, OL),
                        pick(cuda::std::bool_constant<(MASK & 4) != 0>{}, d.grad, OG),
                        pick(cuda::std::bool_constant<(MASK & 8) != 0>{}, d.aux, OA), r1, r2);
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] += r1[c];
            store_slot(d, e, r2);
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[c * P + tg] = run[c];
    }
}

// Neighbour rows staged in shared memory with cp.async (8-byte LDGSTS, one
// per component), double-buffered across each thread's sequence of edges:
// the copies of edge i+1 are in flight while edge i computes, so a thread's
// memory-level parallelism is not bounded by its registers.  STAGE picks the
// staged neighbour dats (bit 0 q, 1 lim, 2 grad, 3 aux); the rest, and all
// own rows, are read as in k_flux<0>.
template <class Q1, class L1, class G1, class A1, class Q2, class L2, class G2, class A2>
__device__ __forceinline__ void eval_edge_vv(const Data &d, int64_t e, int64_t a, int64_t b, Q1 q1, L1 l1,
                                             G1 g1, A1 a1, Q2 q2, L2 l2, G2 g2, A2 a2, double *r1,
                                             double *r2) {
    const double *w = d.w + e * 3, *x1 = d.x + a * 3, *x2 = d.x + b * 3;
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double an = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NLIM; ++j) {
            const double tt = l1[j] + l2[j];
            s = s + tt * tt;
        }
        const double lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s));
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double f = lam * (q2[v] - q1[v]);
            r1[v] = 0.0 + f;
            r2[v] = 0.0 - f;
        }
    }
    {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds2 = d0 * d0 + d1 * d1 + d2 * d2 + 1e-12;
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double wd = w0 * d0 + w1 * d1 + w2 * d2;
        double mu = 0.0;
#pragma unroll
        for (int j = 0; j < NAUX; ++j) mu = mu + (a1[j] + a2[j]);
        mu = 0.01 * mu / (2.0 * NAUX);
        const double awd = fabs(wd);
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const int bb = 3 * v;
            const double gx = 0.5 * (g1[bb] + g2[bb]);
            const double gy = 0.5 * (g1[bb + 1] + g2[bb + 1]);
            const double gz = 0.5 * (g1[bb + 2] + g2[bb + 2]);
            const double dq = q2[v] - q1[v];
            const double corr = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2;
            const double f = mu * (0.001 * (gx * w0 + gy * w1 + gz * w2) + corr * awd);
            r1[v] += f;
            r2[v] -= f;
        }
    }
}

template <int TPB>
struct CView {           // staged neighbour row: component stride = threads per CTA
    const double *p;
    __device__ __forceinline__ double operator[](int c) const { return p[c * TPB]; }
};

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int STAGE, int TPB>
struct Staged {
    static constexpr int DQ = (STAGE & 1) ? NQ : 0, DL = (STAGE & 2) ? NLIM : 0, DG = (STAGE & 4) ? NG : 0,
                         DA = (STAGE & 8) ? NAUX : 0;
    static constexpr int OQ = 0, OL = DQ, OG = OL + DL, OA = OG + DG, D = OA + DA;
    template <int DIM>
    __device__ static void issue(double *buf, const double *base, int64_t b, int64_t P) {
#pragma unroll
        for (int c = 0; c < DIM; ++c) cp_async8(buf + c * TPB, base + c * P + b);
    }
    __device__ static void fetch(double *buf, const Data &d, int64_t b) {
        const int64_t P = d.pitch;
        if constexpr (DQ) issue<NQ>(buf + OQ * TPB, d.q, b, P);
        if constexpr (DL) issue<NLIM>(buf + OL * TPB, d.lim, b, P);
        if constexpr (DG) issue<NG>(buf + OG * TPB, d.grad, b, P);
        if constexpr (DA) issue<NAUX>(buf + OA * TPB, d.aux, b, P);
    }
};

template <int STAGE, int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) k_flux_cpa(const __grid_constant__ Data d) {
    using SG = Staged<STAGE, TPB>;
    extern __shared__ double smc[];
    double *const mine = smc + threadIdx.x;
    auto buf = [&](int i) { return mine + i * (SG::D * TPB); };
    const int64_t P = d.pitch, stride = int64_t(gridDim.x) * TPB;
    int64_t t = int64_t(blockIdx.x) * TPB + threadIdx.x;
    if (t >= d.n1) return;
    // cursor over this thread's edges: (target row t, incidence k, end ke)
    int k = __ldg(d.off1 + t), ke = __ldg(d.off1 + t + 1);
    // prefetch the first edge
    int64_t t_n = t;
    int k_n = k, ke_n = ke;
    auto advance = [&](int64_t &tt, int &kk, int &kke) {
        if (++kk >= kke) {
            tt += stride;
            if (tt < d.n1) {
                kk = __ldg(d.off1 + tt);
                kke = __ldg(d.off1 + tt + 1);
            }
        }
    };
    while (t_n < d.n1 && k_n >= ke_n) {            // rows without edges
        t_n += stride;
        if (t_n < d.n1) { k_n = __ldg(d.off1 + t_n); ke_n = __ldg(d.off1 + t_n + 1); }
    }
    t = t_n; k = k_n; ke = ke_n;
    if (t >= d.n1) return;
    SG::fetch(buf(0), d, __ldg(d.rec + 2 * int64_t(k) + 1));
    cp_commit();
    int cur = 0;
    double run[NQ];
    int64_t tg = __ldg(d.tl1 + t);
#pragma unroll
    for (int c = 0; c < NQ; ++c) run[c] = d.res[c * P + tg];
    while (t < d.n1) {
        // next edge: issue its copies into the other buffer
        t_n = t; k_n = k; ke_n = ke;
        advance(t_n, k_n, ke_n);
        while (t_n < d.n1 && k_n >= ke_n) {
            t_n += stride;
            if (t_n < d.n1) { k_n = __ldg(d.off1 + t_n); ke_n = __ldg(d.off1 + t_n + 1); }
        }
        if (t_n < d.n1) SG::fetch(buf(cur ^ 1), d, __ldg(d.rec + 2 * int64_t(k_n) + 1));
        cp_commit();
        cp_wait<1>();                                  // this edge's copies have landed
        const int64_t e = __ldg(d.elem1 + k);
        const int64_t a = __ldg(d.rec + 2 * int64_t(k)), b = __ldg(d.rec + 2 * int64_t(k) + 1);
        double r1[NQ], r2[NQ];
        const double *sb = buf(cur);
        auto nb = [&](auto staged, const double *base, int off) {
            if constexpr (decltype(staged)::value) return CView<TPB>{sb + off * TPB};
            else return view<0, 1>(base, b, P);
        };
        eval_edge_vv(d, e, a, b, view<0, NQ>(d.q, a, P), view<0, NLIM>(d.lim, a, P), view<0, NG>(d.grad, a, P),
                     view<0, NAUX>(d.aux, a, P),
                     nb(cuda::std::bool_constant<(STAGE & 1) != 0>{}, d.q, SG::OQ),
                     nb(cuda::std::bool_constant<(STAGE & 2) != 0>{}, d.lim, SG::OL),
                     nb(cuda::std::bool_constant<(STAGE & 4) != 0>{}, d.grad, SG::OG),
                     nb(cuda::std::bool_constant<(STAGE & 8) != 0>{}, d.aux, SG::OA), r1, r2);
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] += r1[c];
        store_slot(d, e, r2);
        if (t_n != t) {                                // target finished
#pragma unroll
            for (int c = 0; c < NQ; ++c) d.res[c * P + tg] = run[c];
            if (t_n < d.n1) {
                tg = __ldg(d.tl1 + t_n);
#pragma unroll
                for (int c = 0; c < NQ; ++c) run[c] = d.res[c * P + tg];
            }
        }
        t = t_n; k = k_n; ke = ke_n;
        cur ^= 1;
    }
    cp_wait<0>();
}

// Neighbour rows moved by the TMA engine: padded-AoS rows (16-byte multiples)
// of the staged dats go global -> shared with one cp.async.bulk per row,
// completing on a per-thread mbarrier, double-buffered across the thread's
// edges.  Own rows: padded-AoS 16-byte pair loads (View<2>).
__device__ __forceinline__ uint32_t s32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t *b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(dst)),
                 "l"(src), "r"(bytes), "r"(s32(b))
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(s32(b)), "r"(parity)
                     : "memory");
    } while (!done);
}

struct RowS {            // a staged AoS row in shared memory
    const double *p;
    __device__ __forceinline__ double operator[](int c) const { return p[c]; }
};

template <int STAGE>
struct BulkRows {
    static constexpr int DQ = (STAGE & 1) ? padded<NQ>() : 0, DL = (STAGE & 2) ? padded<NLIM>() : 0,
                         DG = (STAGE & 4) ? padded<NG>() : 0, DA = (STAGE & 8) ? padded<NAUX>() : 0;
    static constexpr int OQ = 0, OL = DQ, OG = OL + DL, OA = OG + DG, D = OA + DA;   // doubles per stage
    __device__ static void fetch(double *buf, uint64_t *bar, const Data &d, int64_t b) {
        bar_expect(bar, uint32_t(D * 8));
        if constexpr (DQ) bulk(buf + OQ, d.q + b * DQ, DQ * 8, bar);
        if constexpr (DL) bulk(buf + OL, d.lim + b * DL, DL * 8, bar);
        if constexpr (DG) bulk(buf + OG, d.grad + b * DG, DG * 8, bar);
        if constexpr (DA) bulk(buf + OA, d.aux + b * DA, DA * 8, bar);
    }
};

template <int STAGE, int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) k_flux_bulk(const __grid_constant__ Data d) {
    using BR = BulkRows<STAGE>;
    extern __shared__ __align__(16) double smb[];
    __shared__ __align__(8) uint64_t bars[2][TPB];
    double *const mine = smb + threadIdx.x * (2 * BR::D);
    auto bar = [&](int i) { return &bars[i][threadIdx.x]; };
    bar_init(bar(0));
    bar_init(bar(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t stride = int64_t(gridDim.x) * TPB;
    int64_t t = int64_t(blockIdx.x) * TPB + threadIdx.x;
    auto skip_empty = [&](int64_t &tt, int &kk, int &kke) {
        while (tt < d.n1 && kk >= kke) {
            tt += stride;
            if (tt < d.n1) { kk = __ldg(d.off1 + tt); kke = __ldg(d.off1 + tt + 1); }
        }
    };
    int k = 0, ke = 0;
    if (t < d.n1) { k = __ldg(d.off1 + t); ke = __ldg(d.off1 + t + 1); }
    skip_empty(t, k, ke);
    if (t >= d.n1) return;
    BR::fetch(mine, bar(0), d, __ldg(d.rec + 2 * int64_t(k) + 1));
    uint32_t phase = 0;
    int cur = 0;
    double run[NQ];
    int64_t tg = __ldg(d.tl1 + t);
#pragma unroll
    for (int c = 0; c < NQ; ++c) run[c] = d.res[tg * NQ + c];
    while (t < d.n1) {
        int64_t t_n = t;
        int k_n = k + 1, ke_n = ke;
        if (k_n >= ke_n) {
            t_n += stride;
            if (t_n < d.n1) { k_n = __ldg(d.off1 + t_n); ke_n = __ldg(d.off1 + t_n + 1); }
        }
        skip_empty(t_n, k_n, ke_n);
        if (t_n < d.n1) BR::fetch(mine + (cur ^ 1) * BR::D, bar(cur ^ 1), d, __ldg(d.rec + 2 * int64_t(k_n) + 1));
        bar_wait(bar(cur), (phase >> cur) & 1u);
        phase ^= 1u << cur;
        const int64_t e = __ldg(d.elem1 + k);
        const int64_t a = __ldg(d.rec + 2 * int64_t(k)), b = __ldg(d.rec + 2 * int64_t(k) + 1);
        const double *sb = mine + cur * BR::D;
        auto nb = [&](auto staged, const double *base, int off, auto dimc) {
            if constexpr (decltype(staged)::value) return RowS{sb + off};
            else return view<2, decltype(dimc)::value>(base, b, 0);
        };
        double r1[NQ], r2[NQ];
        eval_edge_vv(d, e, a, b, view<2, NQ>(d.q, a, 0), view<2, NLIM>(d.lim, a, 0), view<2, NG>(d.grad, a, 0),
                     view<2, NAUX>(d.aux, a, 0),
                     nb(cuda::std::bool_constant<(STAGE & 1) != 0>{}, d.q, BR::OQ, cuda::std::integral_constant<int, NQ>{}),
                     nb(cuda::std::bool_constant<(STAGE & 2) != 0>{}, d.lim, BR::OL, cuda::std::integral_constant<int, NLIM>{}),
                     nb(cuda::std::bool_constant<(STAGE & 4) != 0>{}, d.grad, BR::OG, cuda::std::integral_constant<int, NG>{}),
                     nb(cuda::std::bool_constant<(STAGE & 8) != 0>{}, d.aux, BR::OA, cuda::std::integral_constant<int, NAUX>{}),
                     r1, r2);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before this buffer's next bulk write
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] += r1[c];
        store_slot(d, e, r2);
        if (t_n != t) {
#pragma unroll
            for (int c = 0; c < NQ; ++c) d.res[tg * NQ + c] = run[c];
            if (t_n < d.n1) {
                tg = __ldg(d.tl1 + t_n);
#pragma unroll
                for (int c = 0; c < NQ; ++c) run[c] = d.res[tg * NQ + c];
            }
        }
        t = t_n; k = k_n; ke = ke_n;
        cur ^= 1;
    }
}

// L2 prefetch of the next edge's neighbour rows (no registers held): at edge
// k the thread issues prefetch.global.L2 for the lines of edge k+1's
// neighbour row of the dats in PF (bit 0 q, 1 lim, 2 grad, 3 aux).
__device__ __forceinline__ void pf_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
template <int LAY, int D>
__device__ __forceinline__ void prefetch_row(const double *base, int64_t b, int64_t P) {
    if constexpr (LAY == 0) {
#pragma unroll
        for (int c = 0; c < D; ++c) pf_l2(base + c * P + b);
    } else {      // AoSoA-32: component c at block + c*32: 256-byte segments
#pragma unroll
        for (int c = 0; c < D; ++c) pf_l2(base + (b >> 5) * (32 * D) + c * 32 + (b & 31));
    }
}
template <int LAY, int PF>
__global__ void __launch_bounds__(256, 2) k_flux_pf(const __grid_constant__ Data d) {
    const int64_t P = d.pitch;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < d.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = __ldg(d.tl1 + t);
        double run[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(tg, c, P)];
        const int kb = __ldg(d.off1 + t), ke = __ldg(d.off1 + t + 1);
        for (int k = kb; k < ke; ++k) {
            if (k + 1 < ke) {
                const int64_t bn = __ldg(d.rec + 2 * int64_t(k + 1) + 1);
                if constexpr (PF & 1) prefetch_row<LAY, NQ>(d.q, bn, P);
                if constexpr (PF & 2) prefetch_row<LAY, NLIM>(d.lim, bn, P);
                if constexpr (PF & 4) prefetch_row<LAY, NG>(d.grad, bn, P);
                if constexpr (PF & 8) prefetch_row<LAY, NAUX>(d.aux, bn, P);
            }
            const int64_t e = __ldg(d.elem1 + k);
            const int64_t a = __ldg(d.rec + 2 * int64_t(k)), b = __ldg(d.rec + 2 * int64_t(k) + 1);
            double r1[NQ], r2[NQ];
            eval_edge<LAY>(d, e, a, b, r1, r2);
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] += r1[c];
            store_slot(d, e, r2);
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = run[c];
    }
}

// The primary increment accumulated in shared memory instead of registers
// (frees 12 registers for loads in flight).
template <int LAY>
__global__ void __launch_bounds__(256) k_flux_smrun(const __grid_constant__ Data d) {
    __shared__ double acc[NQ][256];
    const int64_t P = d.pitch;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < d.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = __ldg(d.tl1 + t);
#pragma unroll
        for (int c = 0; c < NQ; ++c) acc[c][threadIdx.x] = d.res[idx<LAY, NQ>(tg, c, P)];
        for (int k = __ldg(d.off1 + t), ke = __ldg(d.off1 + t + 1); k < ke; ++k) {
            const int64_t e = __ldg(d.elem1 + k);
            const int64_t a = __ldg(d.rec + 2 * int64_t(k)), b = __ldg(d.rec + 2 * int64_t(k) + 1);
            double r1[NQ], r2[NQ];
            eval_edge<LAY>(d, e, a, b, r1, r2);
#pragma unroll
            for (int c = 0; c < NQ; ++c) acc[c][threadIdx.x] += r1[c];
            store_slot(d, e, r2);
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = acc[c][threadIdx.x];
    }
}

// Slot-major incidence lists: incidence j of pass-1 row t at j * n1 + t
// (rows have <= 3 primary incidences on this mesh), so a warp's index loads
// (element id, both map entries) are contiguous.
template <int LAY>
__global__ void __launch_bounds__(256) k_flux_sm(const __grid_constant__ Data d, const int32_t *cnt,
                                                 const int32_t *elem_sm, const int32_t *rec_sm) {
    const int64_t P = d.pitch, n1 = d.n1;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n1; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = __ldg(d.tl1 + t);
        double run[NQ];
#pragma unroll
        for (int c = 0; c < NQ; ++c) run[c] = d.res[idx<LAY, NQ>(tg, c, P)];
        const int nk = __ldg(cnt + t);
        for (int j = 0; j < nk; ++j) {
            const int64_t e = __ldg(elem_sm + j * n1 + t);
            const int64_t a = __ldg(rec_sm + (2 * j) * n1 + t), b = __ldg(rec_sm + (2 * j + 1) * n1 + t);
            double r1[NQ], r2[NQ];
            eval_edge<LAY>(d, e, a, b, r1, r2);
#pragma unroll
            for (int c = 0; c < NQ; ++c) run[c] += r1[c];
            store_slot(d, e, r2);
        }
#pragma unroll
        for (int c = 0; c < NQ; ++c) d.res[idx<LAY, NQ>(tg, c, P)] = run[c];
    }
}

}  // namespace

extern "C" int exp_flux_run(int layout, const void *w, const void *q, const void *x, const void *lim,
                            const void *grad, const void *aux, void *res, void *slots, const void *off1,
                            const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                            int64_t n1, int64_t pitch, int grid, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int lay = layout & 1, occ = layout >> 1;   // occ 0: 256x2, 1: 128x5, 2: 128x6
    if (occ == 0) {
        if (lay == 0) k_flux<0, 2><<<grid, 256, 0, s>>>(d);
        else k_flux<1, 2><<<grid, 256, 0, s>>>(d);
    } else if (occ == 1) {
        if (lay == 0) k_flux<0, 5><<<grid * 5, 128, 0, s>>>(d);
        else k_flux<1, 5><<<grid * 5, 128, 0, s>>>(d);
    } else {
        if (lay == 0) k_flux<0, 6><<<grid * 6, 128, 0, s>>>(d);
        else k_flux<1, 6><<<grid * 6, 128, 0, s>>>(d);
    }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_lanes(int layout, const void *w, const void *q, const void *x, const void *lim,
                              const void *grad, const void *aux, void *res, void *slots, const void *off1,
                              const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                              int64_t n1, int64_t pitch, const void *wrow, int64_t ntask, int grid,
                              void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t *wr = static_cast<const int32_t *>(wrow);
    if (layout == 0) k_flux_lanes<0><<<grid, 256, 0, s>>>(d, wr, ntask);
    else k_flux_lanes<1><<<grid, 256, 0, s>>>(d, wr, ntask);
    return int(cudaGetLastError());
}

extern "C" int exp_flux_lrec(int layout, const void *w, const void *q, const void *x, const void *lim,
                             const void *grad, const void *aux, void *res, void *slots, int64_t pitch,
                             const void *lrec, const void *tmask, int64_t ntask, int grid, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           nullptr, nullptr, nullptr, nullptr, nullptr, 0, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int4 *lr = static_cast<const int4 *>(lrec);
    const uint32_t *tm = static_cast<const uint32_t *>(tmask);
    if (layout == 0) k_flux_lrec<0><<<grid, 256, 0, s>>>(d, lr, tm, ntask);
    else k_flux_lrec<1><<<grid, 256, 0, s>>>(d, lr, tm, ntask);
    return int(cudaGetLastError());
}

extern "C" int exp_flux_lock(int layout, const void *w, const void *q, const void *x, const void *lim,
                             const void *grad, const void *aux, void *res, void *slots, const void *off1,
                             const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                             int64_t n1, int64_t pitch, int grid, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int lay = layout & 1, k = layout >> 1;
    if (k == 3) { if (lay == 0) k_flux_lock<0, 3><<<grid, 256, 0, s>>>(d); else k_flux_lock<1, 3><<<grid, 256, 0, s>>>(d); }
    else if (k == 2) { if (lay == 0) k_flux_lock<0, 2><<<grid, 256, 0, s>>>(d); else k_flux_lock<1, 2><<<grid, 256, 0, s>>>(d); }
    else { if (lay == 0) k_flux_lock<0, 4><<<grid, 256, 0, s>>>(d); else k_flux_lock<1, 4><<<grid, 256, 0, s>>>(d); }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_reg(int layout, const void *w, const void *q, const void *x, const void *lim,
                            const void *grad, const void *aux, void *res, void *slots, const void *off1,
                            const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                            int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int lay = layout & 1, minb = layout >> 1;
    if (minb == 1) { if (lay == 0) k_flux_reg<0, 1><<<sms, 256, 0, s>>>(d); else k_flux_reg<1, 1><<<sms, 256, 0, s>>>(d); }
    else { if (lay == 0) k_flux_reg<0, 2><<<2 * sms, 256, 0, s>>>(d); else k_flux_reg<1, 2><<<2 * sms, 256, 0, s>>>(d); }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_h(int variant, const void *w, const void *q, const void *x, const void *lim,
                          const void *grad, const void *aux, void *res, void *slots, const void *off1,
                          const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                          int64_t n1, int64_t pitch, int grid, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (variant) {          // layout bit 0; then (hints, prefetch) combos
    case 0: k_flux_h<0, 0, 0, 1><<<grid, 256, 0, s>>>(d); break;
    case 1: k_flux_h<1, 0, 0, 1><<<grid, 256, 0, s>>>(d); break;
    case 2: k_flux_h<0, 1, 2, 0><<<grid, 256, 0, s>>>(d); break;
    case 3: k_flux_h<1, 1, 2, 0><<<grid, 256, 0, s>>>(d); break;
    case 4: k_flux_h<0, 1, 2, 1><<<grid, 256, 0, s>>>(d); break;
    case 5: k_flux_h<1, 1, 2, 1><<<grid, 256, 0, s>>>(d); break;
    case 6: k_flux_h<0, 0, 2, 0><<<grid, 256, 0, s>>>(d); break;
    default: k_flux_h<1, 0, 2, 0><<<grid, 256, 0, s>>>(d); break;
    }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_split(int variant, const void *w, const void *q, const void *x, const void *lim,
                              const void *grad, const void *aux, void *res, void *slots, const void *off1,
                              const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                              int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (variant) {
    case 0: k_flux_split<0, 2><<<2 * sms, 256, 0, s>>>(d); break;
    case 1: k_flux_split<1, 2><<<2 * sms, 256, 0, s>>>(d); break;
    case 2: k_flux_split<0, 3><<<3 * sms, 256, 0, s>>>(d); break;
    case 3: k_flux_split<1, 3><<<3 * sms, 256, 0, s>>>(d); break;
    case 4: k_flux_split<0, 4><<<4 * sms, 256, 0, s>>>(d); break;
    default: k_flux_split<1, 4><<<4 * sms, 256, 0, s>>>(d); break;
    }
    return int(cudaGetLastError());
}

// padded AoS for the wide node dats (rows of whole 16-byte pairs)
extern "C" int exp_flux_aos(int minb, const void *w, const void *q, const void *x, const void *lim,
                            const void *grad, const void *aux, void *res, void *slots, const void *off1,
                            const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                            int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (minb == 5) k_flux<2, 5><<<sms * 5, 128, 0, s>>>(d);
    else k_flux<2, 2><<<sms * 2, 256, 0, s>>>(d);
    return int(cudaGetLastError());
}

extern "C" int exp_flux_own(int mask, const void *w, const void *q, const void *x, const void *lim,
                            const void *grad, const void *aux, void *res, void *slots, const void *off1,
                            const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                            int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto go = [&](auto kern, int dims) {
        const size_t bytes = size_t(dims) * 256 * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
        kern<<<2 * sms, 256, bytes, s>>>(d);
    };
    switch (mask) {
    case 8: go(k_flux_own<8>, NAUX); break;
    case 12: go(k_flux_own<12>, NAUX + NG); break;
    case 4: go(k_flux_own<4>, NG); break;
    case 15: go(k_flux_own<15>, NAUX + NG + NLIM + NQ); break;
    default: go(k_flux_own<0>, 1); break;
    }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_cpa(int variant, const void *w, const void *q, const void *x, const void *lim,
                            const void *grad, const void *aux, void *res, void *slots, const void *off1,
                            const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                            int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto go = [&](auto kern, int tpb, int dims, int ctas_per_sm) {
        const size_t bytes = size_t(2) * dims * tpb * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
        kern<<<ctas_per_sm * sms, tpb, bytes, s>>>(d);
    };
    switch (variant) {
    case 0: go(k_flux_cpa<12, 128, 3>, 128, NG + NAUX, 3); break;          // grad+aux, 128x3 (76 KB)
    case 1: go(k_flux_cpa<8, 128, 4>, 128, NAUX, 4); break;                // aux only, 128x4
    case 2: go(k_flux_cpa<15, 128, 2>, 128, NQ + NLIM + NG + NAUX, 2); break;   // all, 128x2
    case 3: go(k_flux_cpa<12, 64, 6>, 64, NG + NAUX, 6); break;            // grad+aux, 64x6
    default: go(k_flux_cpa<4, 128, 4>, 128, NG, 4); break;                 // grad only, 128x4
    }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_bulk(int variant, const void *w, const void *q, const void *x, const void *lim,
                             const void *grad, const void *aux, void *res, void *slots, const void *off1,
                             const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                             int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto go = [&](auto kern, int tpb, int dbl, int ctas_per_sm) {
        const size_t bytes = size_t(2) * dbl * tpb * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
        kern<<<ctas_per_sm * sms, tpb, bytes, s>>>(d);
    };
    switch (variant) {
    case 0: go(k_flux_bulk<12, 128, 2>, 128, BulkRows<12>::D, 2); break;     // grad+aux
    case 1: go(k_flux_bulk<15, 64, 3>, 64, BulkRows<15>::D, 3); break;       // all four
    case 2: go(k_flux_bulk<8, 128, 3>, 128, BulkRows<8>::D, 3); break;       // aux
    default: go(k_flux_bulk<12, 64, 4>, 64, BulkRows<12>::D, 4); break;      // grad+aux, 64x4
    }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_pf(int variant, const void *w, const void *q, const void *x, const void *lim,
                           const void *grad, const void *aux, void *res, void *slots, const void *off1,
                           const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                           int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (variant) {
    case 0: k_flux_pf<0, 12><<<2 * sms, 256, 0, s>>>(d); break;   // SOA, grad+aux
    case 1: k_flux_pf<1, 12><<<2 * sms, 256, 0, s>>>(d); break;   // AoSoA, grad+aux
    case 2: k_flux_pf<1, 15><<<2 * sms, 256, 0, s>>>(d); break;   // AoSoA, all
    case 3: k_flux_pf<0, 15><<<2 * sms, 256, 0, s>>>(d); break;   // SOA, all
    default: k_flux_pf<1, 0><<<2 * sms, 256, 0, s>>>(d); break;   // AoSoA, none (reference)
    }
    return int(cudaGetLastError());
}

extern "C" int exp_flux_smrun(int variant, const void *w, const void *q, const void *x, const void *lim,
                              const void *grad, const void *aux, void *res, void *slots, const void *off1,
                              const void *elem1, const void *tl1, const void *rec, const void *slotpos,
                              int64_t n1, int64_t pitch, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           static_cast<const int32_t *>(off1), static_cast<const int32_t *>(elem1),
           static_cast<const int32_t *>(tl1), static_cast<const int32_t *>(rec),
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (variant == 0) k_flux_smrun<0><<<2 * sms, 256, 0, s>>>(d);
    else k_flux_smrun<1><<<2 * sms, 256, 0, s>>>(d);
    return int(cudaGetLastError());
}

extern "C" int exp_flux_sm(int layout, const void *w, const void *q, const void *x, const void *lim,
                           const void *grad, const void *aux, void *res, void *slots, const void *tl1,
                           const void *slotpos, int64_t n1, int64_t pitch, const void *cnt, const void *elem_sm,
                           const void *rec_sm, int sms, void *stream) {
    Data d{static_cast<const double *>(w), static_cast<const double *>(q), static_cast<const double *>(x),
           static_cast<const double *>(lim), static_cast<const double *>(grad),
           static_cast<const double *>(aux), static_cast<double *>(res), static_cast<double *>(slots),
           nullptr, nullptr, static_cast<const int32_t *>(tl1), nullptr,
           static_cast<const int32_t *>(slotpos), n1, pitch};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t *c = static_cast<const int32_t *>(cnt), *es = static_cast<const int32_t *>(elem_sm),
                  *rs = static_cast<const int32_t *>(rec_sm);
    if (layout == 0) k_flux_sm<0><<<2 * sms, 256, 0, s>>>(d, c, es, rs);
    else k_flux_sm<1><<<2 * sms, 256, 0, s>>>(d, c, es, rs);
    return int(cudaGetLastError());
}
