// Device functors of the Hydra-shaped proxy iteration (paper_1403_7209_b200/
// apps.py: build_hydra_proxy).  Loop shapes follow the paper's per-loop data
// table: iflux = ifluxedge (direct 3/0, indirect 34/12
// doubles), vflux = vfluxedge (direct 3/0, indirect 92/12 doubles).  Each
// body repeats its Python twin's expression tree exactly (no FMA
// contraction: the library builds with -fmad=false).
#include "engine.cuh"

namespace ml {
namespace {

constexpr int NQ = 6, NG = 18, NLIM = 8, NAUX = 19;

struct ProxySave {
    static constexpr bool dense_writes = true;   // every direct WRITE component is written
    template <class T> using sig = Sig<Arg<KD, MR, NQ, T>, Arg<KD, MW, NQ, T>>;
    template <class Q, class QO>
    __device__ static void apply(const Consts &, Q q, QO q_old) {
#pragma unroll
        for (int v = 0; v < NQ; ++v) q_old[v] = q[v];
    }
};

struct ProxyDt {
    static constexpr bool dense_writes = true;   // every direct WRITE component is written
    template <class T>
    using sig = Sig<Arg<KD, MR, NQ, T>, Arg<KD, MR, 1, T>, Arg<KD, MW, 1, T>, Arg<KG, MMIN, 1, T>>;
    template <class Q, class V, class D, class M>
    __device__ static void apply(const Consts &k, Q q, V vol, D dt_loc, M dt_min) {
        double s = 1.0;
#pragma unroll
        for (int v = 0; v < NQ; ++v) s = s + fabs(q[v]);
        const double d = k.f[0] * vol[0] / s;
        dt_loc[0] = d;
        if (d < dt_min[0]) dt_min[0] = d;
    }
};

// Loop chain save -> dt_calc (both direct over the nodes, both read q): one
// pass copies q to q_old and computes the local time step from the same
// loaded q row.
struct ProxySaveDt {
    static constexpr bool dense_writes = true;   // every direct WRITE component is written
    static constexpr int first_args[2] = {0, 1};           // save: q q_old
    static constexpr int second_args[4] = {0, 2, 3, 4};    // dt_calc: q vol dt_loc dt_min
    template <class T>
    using sig = Sig<Arg<KD, MR, NQ, T>, Arg<KD, MW, NQ, T>, Arg<KD, MR, 1, T>, Arg<KD, MW, 1, T>,
                    Arg<KG, MMIN, 1, T>>;
    template <class Q, class QO, class V, class D, class M>
    __device__ static void apply(const Consts &k, Q q, QO q_old, V vol, D dt_loc, M dt_min) {
        ProxySave::apply(k, q, q_old);
        ProxyDt::apply(k, q, vol, dt_loc, dt_min);
    }
};

struct ProxyGrad {
    static constexpr int rec_cols[7] = {-1, 0, 1, 0, 1, 0, 1};   // w, then (node 1, node 2) pairs
    template <class T>
    using sig = Sig<Arg<KD, MR, 3, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, 3, T>,
                    Arg<KI, MR, 3, T>, Arg<KI, MINC, NG, T>, Arg<KI, MINC, NG, T>>;
    template <class W, class Q1, class Q2, class X1, class X2, class G1, class G2>
    __device__ static void apply(const Consts &, W w, Q1 q1, Q2 q2, X1 x1, X2 x2, G1 g1, G2 g2) {
        const double dx[3] = {x2[0] - x1[0], x2[1] - x1[1], x2[2] - x1[2]};
        const double ww[3] = {w[0], w[1], w[2]};
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double a = q1[v], b = q2[v];
            const double qa = 0.5 * (a + b);
            const double dq = b - a;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double f = qa * ww[k] + 0.125 * dq * dx[k];
                g1[3 * v + k] += f;
                g2[3 * v + k] -= f;
            }
        }
    }
};

struct ProxyIflux {
    static constexpr int rec_cols[9] = {-1, 0, 1, 0, 1, 0, 1, 0, 1};   // w, then (node 1, node 2) pairs
    template <class T>
    using sig = Sig<Arg<KD, MR, 3, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, 3, T>,
                    Arg<KI, MR, 3, T>, Arg<KI, MR, NLIM, T>, Arg<KI, MR, NLIM, T>,
                    Arg<KI, MINC, NQ, T>, Arg<KI, MINC, NQ, T>>;
    template <class W, class Q1, class Q2, class X1, class X2, class L1, class L2, class R1, class R2>
    __device__ static void apply(const Consts &, W w, Q1 q1, Q2 q2, X1 x1, X2 x2, L1 l1, L2 l2,
                                 R1 r1, R2 r2) {
        const double d0 = x2[0] - x1[0], d1 = x2[1] - x1[1], d2 = x2[2] - x1[2];
        const double ds = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        const double an = sqrt(w0 * w0 + w1 * w1 + w2 * w2);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NLIM; ++j) {
            const double t = l1[j] + l2[j];
            s = s + t * t;
        }
        const double lam = an / ((1.0 + ds) * (1.0 + 0.0625 * s));
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double f = lam * (q2[v] - q1[v]);
            r1[v] += f;
            r2[v] -= f;
        }
    }
};

struct ProxyVflux {
    static constexpr int rec_cols[11] = {-1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1};   // w, then (node 1, node 2) pairs
    template <class T>
    using sig = Sig<Arg<KD, MR, 3, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, NG, T>,
                    Arg<KI, MR, NG, T>, Arg<KI, MR, 3, T>, Arg<KI, MR, 3, T>, Arg<KI, MR, NAUX, T>,
                    Arg<KI, MR, NAUX, T>, Arg<KI, MINC, NQ, T>, Arg<KI, MINC, NQ, T>>;
    template <class W, class Q1, class Q2, class G1, class G2, class X1, class X2, class A1, class A2,
              class R1, class R2>
    __device__ static void apply(const Consts &, W w, Q1 q1, Q2 q2, G1 g1, G2 g2, X1 x1, X2 x2,
                                 A1 a1, A2 a2, R1 r1, R2 r2) {
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
            const int b = 3 * v;
            const double gx = 0.5 * (g1[b] + g2[b]);
            const double gy = 0.5 * (g1[b + 1] + g2[b + 1]);
            const double gz = 0.5 * (g1[b + 2] + g2[b + 2]);
            const double dq = q2[v] - q1[v];
            const double corr = (dq - (gx * d0 + gy * d1 + gz * d2)) / ds2;
            const double f = mu * (0.001 * (gx * w0 + gy * w1 + gz * w2) + corr * awd);
            r1[v] += f;
            r2[v] -= f;
        }
    }
};

// Loop chain iflux -> vflux (both gather the same edge's node rows and
// increment res): one pass evaluates iflux then vflux on each edge with the
// same expression trees, vflux's increments added after iflux's, so each
// edge's node rows are fetched once for both loops.
struct ProxyFluxes {
    static constexpr int rec_cols[13] = {-1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1};   // w, then (node 1, node 2) pairs
    // fused argument of each iflux argument (w q1 q2 x1 x2 l1 l2 r1 r2) and
    // each vflux argument (w q1 q2 g1 g2 x1 x2 a1 a2 r1 r2): w, q, x and res
    // are shared, grad and aux come from vflux alone
    static constexpr int first_args[9] = {0, 1, 2, 3, 4, 5, 6, 11, 12};
    static constexpr int second_args[11] = {0, 1, 2, 7, 8, 3, 4, 9, 10, 11, 12};
    template <class T>
    using sig = Sig<Arg<KD, MR, 3, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, 3, T>,
                    Arg<KI, MR, 3, T>, Arg<KI, MR, NLIM, T>, Arg<KI, MR, NLIM, T>, Arg<KI, MR, NG, T>,
                    Arg<KI, MR, NG, T>, Arg<KI, MR, NAUX, T>, Arg<KI, MR, NAUX, T>,
                    Arg<KI, MINC, NQ, T>, Arg<KI, MINC, NQ, T>>;
    template <class W, class Q1, class Q2, class X1, class X2, class L1, class L2, class G1, class G2,
              class A1, class A2, class R1, class R2>
    __device__ static void apply(const Consts &k, W w, Q1 q1, Q2 q2, X1 x1, X2 x2, L1 l1, L2 l2, G1 g1, G2 g2,
                                 A1 a1, A2 a2, R1 r1, R2 r2) {
        ProxyIflux::apply(k, w, q1, q2, x1, x2, l1, l2, r1, r2);
        ProxyVflux::apply(k, w, q1, q2, g1, g2, x1, x2, a1, a2, r1, r2);
    }
};

struct ProxyUpdate {
    static constexpr bool dense_writes = true;   // every direct WRITE component is written
    template <class T>
    using sig = Sig<Arg<KD, MW, NQ, T>, Arg<KD, MR, NQ, T>, Arg<KD, MRW, NQ, T>, Arg<KD, MR, 1, T>,
                    Arg<KD, MW, NG, T>, Arg<KG, MR, 1, T>, Arg<KG, MINC, 1, T>>;
    template <class Q, class QO, class R, class V, class G, class DT, class RMS>
    __device__ static void apply(const Consts &, Q q, QO q_old, R res, V vol, G grad, DT dt_min,
                                 RMS rms) {
        const double s = dt_min[0] / vol[0];
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            const double r = res[v];
            q[v] = q_old[v] + s * r;
            rms[0] += r * r;
            res[v] = 0.0;
        }
#pragma unroll
        for (int k = 0; k < NG; ++k) grad[k] = 0.0;
    }
};

struct ProxyBc {
    static constexpr int rec_cols[4] = {0, 1, 0, 1};   // (node 1, node 2) pairs
    static constexpr bool write_only = true;   // indirect WRITE components all written, none read
    template <class T>
    using sig = Sig<Arg<KI, MW, NQ, T>, Arg<KI, MW, NQ, T>, Arg<KI, MR, NQ, T>, Arg<KI, MR, NQ, T>>;
    template <class Q1, class Q2, class B1, class B2>
    __device__ static void apply(const Consts &, Q1 q1, Q2 q2, B1 b1, B2 b2) {
#pragma unroll
        for (int v = 0; v < NQ; ++v) {
            q1[v] = b1[v];
            q2[v] = b2[v];
        }
    }
};

}  // namespace

ML_REGISTER("proxy_save", ProxySave, double);
ML_REGISTER("proxy_dt", ProxyDt, double);
ML_REGISTER("proxy_save_dt", ProxySaveDt, double);
ML_REGISTER_CHAIN("proxy_save", "proxy_dt", "proxy_save_dt", ProxySaveDt);
ML_REGISTER("proxy_grad", ProxyGrad, double);
ML_REGISTER("proxy_iflux", ProxyIflux, double);
ML_REGISTER("proxy_vflux", ProxyVflux, double);
ML_REGISTER("proxy_update", ProxyUpdate, double);
ML_REGISTER("proxy_fluxes", ProxyFluxes, double);
ML_REGISTER_CHAIN("proxy_iflux", "proxy_vflux", "proxy_fluxes", ProxyFluxes);
ML_REGISTER("proxy_bc", ProxyBc, double);

}  // namespace ml
