// libmeshloop_b200 runtime: device/stream management, memory, functor registry,
// loop launch (colour schedule + deterministic reduction combine), native
// programs with CUDA-graph replay, timers and the L2 flush used by the bench.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "engine.cuh"
#include "ml_common.h"

namespace ml {

static thread_local std::string g_error;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
}
const char *get_error() { return g_error.c_str(); }

// ---- functor registry -------------------------------------------------------------
static std::vector<FunctorEntry> &registry() {
    static std::vector<FunctorEntry> r;
    return r;
}
void register_functor(const FunctorEntry &e) { registry().push_back(e); }
static std::vector<ChainEntry> &chains() {
    static std::vector<ChainEntry> c;
    return c;
}
void register_chain(const ChainEntry &c) { chains().push_back(c); }

// ---- per-device state ------------------------------------------------------------
struct DeviceState {
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaStream_t copy[2] = {nullptr, nullptr};     // H2D, D2H copy streams
    // segmented uploads on the H2D stream: PCIe copy into one of two staging
    // buffers, repack kernel on `repack` (ml_order from H2D covers it)
    cudaStream_t repack = nullptr;
    cudaEvent_t stage_copied[2] = {}, stage_done[2] = {}, repack_ev = nullptr;
    void *stage[2] = {nullptr, nullptr};
    uint64_t stage_cap[2] = {0, 0};
    int stage_next = 0;
    cudaEvent_t order_ev[64] = {};
    int order_next = 0;
    int sm_count = 0;
    int64_t l2_bytes = 0;
    void *flush_buf = nullptr;
    size_t flush_bytes = 0;
};
static DeviceState g_dev;
static std::mutex g_init_mu;

static int ensure_init() {
    if (g_dev.stream) return ML_OK;
    ML_FAIL(ML_EINVAL, "libmeshloop_b200: ml_init() has not been called");
}

// ---- reduction combine ------------------------------------------------------------
bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("ML_PDL");          // ML_PDL=0 turns it off
        return e ? std::atoi(e) != 0 : true;
    }();
    return on;
}

template <class T, int M>
__global__ void __launch_bounds__(256) k_combine(T *g, const T *part, int64_t nparts, int dim) {
    pdl_wait();
    __shared__ double smem[32];
    for (int c = 0; c < dim; ++c) {
        T v = reduce_identity<T, M>();
        for (int64_t i = threadIdx.x; i < nparts; i += blockDim.x) v = combine<M>(v, part[i * dim + c]);
        v = block_reduce<T, M>(v, reinterpret_cast<T *>(smem));
        if (threadIdx.x == 0) g[c] = combine<M>(g[c], v);
        __syncthreads();
    }
}

template <class T>
static void launch_combine(int mode, T *g, const T *part, int64_t nparts, int dim, cudaStream_t s) {
    if (mode == MINC) launch_k(k_combine<T, MINC>, dim3(1), dim3(256), 0, s, g, part, nparts, dim);
    else if (mode == MMIN) launch_k(k_combine<T, MMIN>, dim3(1), dim3(256), 0, s, g, part, nparts, dim);
    else launch_k(k_combine<T, MMAX>, dim3(1), dim3(256), 0, s, g, part, nparts, dim);
}

static int round_up32(int64_t x) { return int((x + 31) / 32 * 32); }

static int validate(const ml_loop_t *L, const FunctorEntry &f) {
    const char *nm = L->name ? L->name : "?";
    if (L->nargs != f.nargs)
        ML_FAIL(ML_EINVAL, "loop '%s': functor '%s' takes %d args, loop has %d", nm, f.name, f.nargs,
                L->nargs);
    for (int i = 0; i < f.nargs; ++i) {
        const ml_arg_t &a = L->args[i];
        if (a.kind != f.kind[i] || a.mode != f.mode[i] || a.dim != f.dim[i] || a.dtype != f.atype[i])
            ML_FAIL(ML_EINVAL,
                    "loop '%s' arg %d: functor '%s' expects (kind %d, mode %d, dim %d, dtype %d), "
                    "got (kind %d, mode %d, dim %d, dtype %d)",
                    nm, i, f.name, f.kind[i], f.mode[i], f.dim[i], f.atype[i], a.kind, a.mode, a.dim,
                    a.dtype);
        if (!a.data && !(a.kind != ML_GLOBAL && a.set_size == 0))
            ML_FAIL(ML_EINVAL, "loop '%s' arg %d: null device pointer", nm, i);
        if (a.kind == ML_INDIRECT && !a.map && L->n > 0)
            ML_FAIL(ML_EINVAL, "loop '%s' arg %d: indirect arg without device map", nm, i);
        if (a.kind != ML_GLOBAL && a.layout == ML_SOA && a.seg_shift == 0 && a.pitch != 0 && a.pitch < a.set_size)
            ML_FAIL(ML_EINVAL, "loop '%s' arg %d: SOA pitch %lld below the set size %lld", nm, i,
                    (long long)a.pitch, (long long)a.set_size);
        if (a.kind != ML_GLOBAL && (a.seg_shift < 0 || a.seg_shift > 30))
            ML_FAIL(ML_EINVAL, "loop '%s' arg %d: bad segment shift %d", nm, i, a.seg_shift);
    }
    return ML_OK;
}

// Layout policy of a launch (engine.cuh): 1 when every dat argument follows the
// reference's auto-SOA policy (dim <= 4 AOS — or any layout at dim 1 — wider
// dats SOA) with 16-byte aligned payloads and an even SOA pitch, so the
// compile-time strides of the LP = 1 kernels apply; 0 otherwise.
static int layout_policy(const ml_loop_t *L) {
    for (int i = 0; i < L->nargs; ++i) {
        const ml_arg_t &a = L->args[i];
        if (a.kind == ML_GLOBAL) continue;
        if (a.dim > AUTO_SOA_DIM) {
            const int want = a.dim >= ML_SEG_MIN_DIM && a.dim <= ML_SEG_MAX_DIM ? SEG_SHIFT : 0;
            if (a.layout != ML_SOA || a.seg_shift != want) return 0;
            if (!want && ((a.pitch ? a.pitch : a.set_size) & 1)) return 0;   // 16-byte pairs
        } else if (a.dim > 1 && a.layout != ML_AOS) {
            return 0;
        }
        if (reinterpret_cast<uintptr_t>(a.data) & 15) return 0;
    }
    return 1;
}

static uint64_t scratch_bytes(const ml_loop_t *L, const FunctorEntry &f) {
    uint64_t bytes = 0;
    const int64_t nb = std::max<int64_t>({L->plan.nblocks, (L->gather_ntargets + 255) / 256,
                                          (L->n + 255) / 256, int64_t(1)});
    for (int i = 0; i < f.nargs; ++i)
        if (f.kind[i] == KG && f.mode[i] != MR) bytes += uint64_t(nb) * f.dim[i] * 8 + 256;
    return bytes ? bytes + 256 : 0;   // + the last-CTA ticket (zero-filled at allocation)
}

// resident-CTA counts per (functor, kernel, threads) — occupancy queries are not free
static int cached_occupancy(int functor, int kernel, int threads, int (*query)(int)) {
    static std::vector<std::pair<std::tuple<int, int, int>, int>> cache;
    const auto key = std::make_tuple(functor, kernel, threads);
    for (auto &kv : cache)
        if (kv.first == key) return kv.second;
    const int occ = query ? query(threads) : 0;
    cache.push_back({key, occ});
    return occ;
}

static int enqueue_loop_impl(const ml_loop_t *L, cudaStream_t stream);

// NVTX range per loop enqueue (named after the loop), so nsys/ncu timelines
// attribute every launch and combine to its op_par_loop
static int enqueue_loop(const ml_loop_t *L, cudaStream_t stream) {
    nvtxRangePushA(L && L->name ? L->name : "loop");
    const int rc = enqueue_loop_impl(L, stream);
    nvtxRangePop();
    return rc;
}

static int enqueue_loop_impl(const ml_loop_t *L, cudaStream_t stream) {
    auto &reg = registry();
    if (L->functor < 0 || L->functor >= int(reg.size()))
        ML_FAIL(ML_ENOFUNCTOR, "loop '%s': bad functor id %d", L->name ? L->name : "?", L->functor);
    const FunctorEntry &f = reg[L->functor];
    int rc = validate(L, f);
    if (rc) return rc;
    if (L->n == 0) return ML_OK;   // empty iteration set: no launch, globals untouched
    const int64_t bs = L->plan.block_size;
    const int64_t nb = L->plan.nblocks;
    if (bs < 1 || nb != (L->n + bs - 1) / bs)
        ML_FAIL(ML_EINVAL, "loop '%s': plan does not cover the iteration set", L->name);

    LaunchParams p{};
    p.n = L->n;
    p.rlim = L->rlim < 0 ? L->n : L->rlim;
    p.bs = int32_t(bs);
    for (int i = 0; i < 4; ++i) {
        p.k.f[i] = L->fconst[i];
        p.k.i[i] = L->iconst[i];
    }
    char *scratch = static_cast<char *>(L->scratch);
    bool has_reduce = false;
    const int64_t pstride = std::max<int64_t>({nb, (L->gather_ntargets + 255) / 256,
                                               (L->n + 255) / 256, int64_t(1)});
    for (int i = 0; i < f.nargs; ++i) {
        const ml_arg_t &a = L->args[i];
        ArgRt &r = p.a[i];
        r.data = a.data;
        if (a.kind == ML_INDIRECT) r.map = a.map + int64_t(a.slot) * a.map_from;
        if (a.kind == ML_GLOBAL) {
            r.se = 0;
            r.sc = 1;
            if (a.mode != ML_READ) {
                if (!scratch) ML_FAIL(ML_EINVAL, "loop '%s': reduction needs scratch", L->name);
                p.part[i] = scratch;
                scratch += uint64_t(pstride) * a.dim * 8 + 256;
                has_reduce = true;
            }
        } else if (a.layout == ML_AOS || a.dim == 1) {
            r.se = a.dim;
            r.sc = 1;
        } else if (a.seg_shift > 0) {             // segmented SOA
            r.se = 0;
            r.sh = a.seg_shift;
            r.sc = (int64_t(1) << a.seg_shift) + ML_SEG_PAD;
            r.sb = r.sc * a.dim;
        } else {
            r.se = 1;
            r.sc = a.pitch ? a.pitch : a.set_size;
        }
    }
    const int lp = layout_policy(L);
    // LP 2: the LP 1 layouts and the functor's compile-time record columns,
    // when the host validated the loop's records against them (rec_fixed)
    int glp = lp;
    if (lp == 1 && L->rec_fixed && f.nrec_cols == f.nargs && L->pf_rec && L->pf_ncol >= 1) {
        bool same = true;
        for (int i = 0; i < f.nargs; ++i)
            if (L->args[i].kind == ML_INDIRECT && L->pf_rcol[i] != f.rec_cols[i]) same = false;
        int width = 0;
        for (int i = 0; i < f.nargs; ++i) width = std::max(width, int(f.rec_cols[i]) + 1);
        if (!same || width != L->pf_ncol)
            ML_FAIL(ML_EINVAL, "loop '%s': rec_fixed set but its records differ from the functor's columns",
                    L->name);
        glp = 2;
    }

    int64_t nparts = nb;   // reduction partials written by the launch(es)
    bool last_colour = true;   // false: a partial colour range that does not end the loop
    // single-launch schedules fold their partials in the kernel (last CTA);
    // the colour schedules launch k_combine after their colour launches
    unsigned *const ticket = has_reduce ? reinterpret_cast<unsigned *>(scratch) : nullptr;
    bool single_launch = false;
    if (L->pf_n1 > 0) {
        // primary fold: pass 1 over targets' primary incidences (persistent grid),
        // pass 2 folds the secondary slots
        if (!f.pfold1[0] || !L->pf_off1 || !L->pf_elem1 || (f.pfold_nslot > 0 && (!L->pf_slots ||
            (L->pf_n2 > 0 && (!L->pf_off2 || !L->pf_elem2 || !L->pf_pos2)))))
            ML_FAIL(ML_EINVAL, "loop '%s': primary-fold lists missing", L->name);
        PFoldParams &pf = p.pf;
        pf.n1 = L->pf_n1;
        pf.off1 = L->pf_off1;
        pf.elem1 = L->pf_elem1;
        pf.tl1 = L->pf_tl1;
        pf.n2 = f.pfold_nslot > 0 ? L->pf_n2 : 0;
        pf.off2 = L->pf_off2;
        pf.elem2 = L->pf_elem2;
        pf.tl2 = L->pf_tl2;
        pf.pos2 = L->pf_pos2;
        pf.slots = L->pf_slots;
        pf.slotpos = L->pf_slotpos;
        if (f.pfold_nslot > 0 && !pf.slotpos) ML_FAIL(ML_EINVAL, "loop '%s': pfold slot positions missing", L->name);
        pf.nslot = f.pfold_nslot;
        pf.dgp = f.pfold_dgp;
        pf.seg1 = L->pf_seg1;
        pf.seg2 = L->pf_seg2;
        pf.part1 = L->pf_part1;
        pf.part2 = L->pf_part2;
        if ((L->pf_nhub1 > 0 && (!pf.seg1 || !pf.part1 || !L->pf_hub1_tl || !L->pf_hub1_off)) ||
            (L->pf_nhub2 > 0 && (!pf.seg2 || !pf.part2 || !L->pf_hub2_tl || !L->pf_hub2_off)))
            ML_FAIL(ML_EINVAL, "loop '%s': primary-fold hub lists missing", L->name);
        if (!L->pf_rec || L->pf_ncol < 1)
            ML_FAIL(ML_EINVAL, "loop '%s': primary fold needs per-incidence map records", L->name);
        pf.rec = L->pf_rec;
        pf.ncol = L->pf_ncol;
        for (int i = 0; i < MAX_ARGS; ++i) pf.rcol[i] = L->pf_rcol[i];
        p.ticket = ticket;
        single_launch = true;
        if (pf.rec)
            for (int i = 0; i < f.nargs; ++i)
                if (L->args[i].kind == ML_INDIRECT && (pf.rcol[i] < 0 || pf.rcol[i] >= pf.ncol))
                    ML_FAIL(ML_EINVAL, "loop '%s': pfold record column of argument %d out of range", L->name, i);
        {
            const int plp = f.pfold1[glp] ? glp : lp;
            const int occ = f.pfold_occupancy[plp] ? f.pfold_occupancy[plp]() : 0;
            nparts = std::max<int64_t>(1, std::min<int64_t>((pf.n1 + 255) / 256,
                                                            occ > 0 ? int64_t(occ) * g_dev.sm_count : INT64_MAX));
            if (nparts > pstride) ML_FAIL(ML_EINVAL, "loop '%s': primary fold needs more scratch", L->name);
            f.pfold1[plp](p, dim3(unsigned(nparts)), dim3(256), 0, stream);
            if (L->pf_nhub1 > 0) f.pfold_hubs(p, L->pf_nhub1, L->pf_hub1_tl, L->pf_hub1_off, pf.part1, stream);
            if (pf.n2 > 0) {
                const int64_t g2 = std::min<int64_t>((pf.n2 + 255) / 256, int64_t(8) * g_dev.sm_count);
                f.pfold2(p, dim3(unsigned(g2)), dim3(256), 0, stream);
                if (L->pf_nhub2 > 0) f.pfold_hubs(p, L->pf_nhub2, L->pf_hub2_tl, L->pf_hub2_off, pf.part2, stream);
            }
        }
    } else if (f.ind_write && f.gather[0] && L->gather_ntargets > 0 && L->gather_off && L->gather_elem &&
               L->gather_pos) {
        // target-centric: one thread per target, serial-order accumulation,
        // persistent grid (resident CTAs x SMs striding over the targets)
        p.g_ntargets = L->gather_ntargets;
        p.g_off = L->gather_off;
        p.g_elem = L->gather_elem;
        p.g_pos = L->gather_pos;
        p.g_tlist = L->gather_targets;
        // per-incidence map records (pf_rec/pf_ncol/pf_rcol, as the primary
        // fold's pass 1): the kernel reads an incidence's map entries beside
        // its element id, one dependent load fewer
        if (!L->pf_rec || L->pf_ncol < 1)
            ML_FAIL(ML_EINVAL, "loop '%s': gather schedule needs per-incidence map records", L->name);
        p.pf.rec = L->pf_rec;
        p.pf.ncol = L->pf_ncol;
        for (int i = 0; i < MAX_ARGS; ++i) p.pf.rcol[i] = L->pf_rcol[i];
        for (int i = 0; i < f.nargs; ++i)
            if (L->args[i].kind == ML_INDIRECT && (L->pf_rcol[i] < 0 || L->pf_rcol[i] >= L->pf_ncol))
                ML_FAIL(ML_EINVAL, "loop '%s': record column of argument %d out of range", L->name, i);
        p.ticket = ticket;
        single_launch = true;
        nparts = (L->gather_ntargets + 255) / 256;
        const int gl = f.gather[glp] ? glp : lp;
        if (const int per_sm = f.gather_occupancy[gl] ? f.gather_occupancy[gl]() : 0; per_sm > 0)
            nparts = std::min<int64_t>(nparts, int64_t(per_sm) * g_dev.sm_count);
        if (nparts > pstride)
            ML_FAIL(ML_EINVAL, "loop '%s': gather schedule needs more reduction scratch", L->name);
        if (L->gather_seg) {
            if (!f.gather_hubs || !L->gather_part || !L->gather_hub_tl || !L->gather_hub_off)
                ML_FAIL(ML_EINVAL, "loop '%s': hub lists incomplete (INC gather only)", L->name);
            p.g_seg = L->gather_seg;
            p.g_part = L->gather_part;
            p.g_nhub = L->gather_nhub;
            p.g_hub_tl = L->gather_hub_tl;
            p.g_hub_off = L->gather_hub_off;
        }
        f.gather[gl](p, dim3(unsigned(nparts)), dim3(256), 0, stream);
        if (L->gather_seg && L->gather_nhub > 0)
            f.gather_hubs(p, dim3(unsigned((L->gather_nhub + 255) / 256)), dim3(256), 0, stream);
    } else if (!f.ind_write) {
        // direct: persistent grid (resident CTAs x SMs); LP = 1 threads own two
        // elements each (16-byte direct accesses)
        const int threads = 256;
        const int occ = cached_occupancy(L->functor, lp, threads, f.direct_occupancy[lp]);
        const int64_t per = lp ? 2 * threads : threads;
        nparts = std::max<int64_t>(1, (L->n + per - 1) / per);
        if (occ > 0) nparts = std::min<int64_t>(nparts, int64_t(occ) * g_dev.sm_count);
        if (nparts > pstride) ML_FAIL(ML_EINVAL, "loop '%s': direct loop needs more scratch", L->name);
        p.ticket = ticket;
        single_launch = true;
        f.direct[lp](p, dim3(unsigned(nparts)), dim3(unsigned(threads)), 0, stream);
    } else {
        // the reference plan's colours: one launch per block colour
        if (!L->plan.color_offsets || !L->plan.blocks || !L->plan.elem_color || !L->plan.elem_ncolors)
            ML_FAIL(ML_EINVAL, "loop '%s': indirect writes need a coloured plan", L->name);
        p.ecol = L->plan.elem_color;
        p.encol = L->plan.elem_ncolors;
        const bool staged = f.staged && bs <= 256;
        const LaunchFn fn = staged ? f.staged : f.phased;
        const int threads = staged ? round_up32(bs) : std::clamp(round_up32(bs), 32, 256);
        const int64_t c0 = std::max<int64_t>(0, L->colour_begin);
        const int64_t c1 = L->colour_end > 0 ? std::min<int64_t>(L->colour_end, L->plan.ncolors) : L->plan.ncolors;
        if (c1 < L->plan.ncolors) last_colour = false;
        for (int64_t c = c0; c < c1; ++c) {
            const int64_t off = L->plan.color_offsets[c], cnt = L->plan.color_offsets[c + 1] - off;
            if (cnt <= 0) continue;
            p.blocks = L->plan.blocks + off;
            fn(p, dim3(unsigned(cnt)), dim3(unsigned(threads)), 0, stream);
        }
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) ML_FAIL(ML_ECUDA, "loop '%s': launch failed: %s", L->name, cudaGetErrorString(err));

    for (int i = 0; i < f.nargs && last_colour && !single_launch; ++i) {
        const ml_arg_t &a = L->args[i];
        if (a.kind != ML_GLOBAL || a.mode == ML_READ) continue;
        if (a.dtype == ML_F64)
            launch_combine<double>(a.mode, static_cast<double *>(a.data), static_cast<const double *>(p.part[i]),
                                   nparts, a.dim, stream);
        else
            launch_combine<int64_t>(a.mode, static_cast<int64_t *>(a.data),
                                    static_cast<const int64_t *>(p.part[i]), nparts, a.dim, stream);
    }
    err = cudaGetLastError();
    if (err != cudaSuccess) ML_FAIL(ML_ECUDA, "loop '%s': combine failed: %s", L->name, cudaGetErrorString(err));
    return ML_OK;
}

__global__ void k_map_to_i32(int32_t *dst, const int64_t *src, int64_t rows, int32_t arity) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows * arity;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / arity, c = i % arity;
        dst[c * rows + r] = int32_t(src[i]);
    }
}

}  // namespace ml

using namespace ml;

// ---- ABI: runtime --------------------------------------------------------------------
extern "C" const char *ml_last_error(void) { return get_error(); }
extern "C" int ml_version(void) { return 1; }

extern "C" int ml_init(int device) {
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (g_dev.stream && g_dev.device == device) return ML_OK;
    int n = 0;
    ML_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) ML_FAIL(ML_EINVAL, "ml_init: device %d of %d", device, n);
    ML_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    ML_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        ML_FAIL(ML_ECUDA, "ml_init: device %d is sm_%d%d; this library is built for sm_100a only", device,
                prop.major, prop.minor);
    if (g_dev.stream) cudaStreamDestroy(g_dev.stream);
    for (auto &c : g_dev.copy)
        if (c) cudaStreamDestroy(c), c = nullptr;
    ML_CUDA(cudaStreamCreateWithFlags(&g_dev.stream, cudaStreamNonBlocking));
    for (auto &c : g_dev.copy) ML_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
    if (g_dev.repack) cudaStreamDestroy(g_dev.repack);
    ML_CUDA(cudaStreamCreateWithFlags(&g_dev.repack, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        if (!g_dev.stage_copied[k]) ML_CUDA(cudaEventCreateWithFlags(&g_dev.stage_copied[k], cudaEventDisableTiming));
        if (!g_dev.stage_done[k]) ML_CUDA(cudaEventCreateWithFlags(&g_dev.stage_done[k], cudaEventDisableTiming));
    }
    if (!g_dev.repack_ev) ML_CUDA(cudaEventCreateWithFlags(&g_dev.repack_ev, cudaEventDisableTiming));
    for (auto &e : g_dev.order_ev)
        if (!e) ML_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g_dev.device = device;
    g_dev.sm_count = prop.multiProcessorCount;
    g_dev.l2_bytes = prop.l2CacheSize;
    return ML_OK;
}

extern "C" int ml_device_info(ml_device_info_t *out) {
    int rc = ensure_init();
    if (rc) return rc;
    cudaDeviceProp prop;
    ML_CUDA(cudaGetDeviceProperties(&prop, g_dev.device));
    std::memset(out, 0, sizeof *out);
    std::strncpy(out->name, prop.name, sizeof(out->name) - 1);
    out->sm_count = prop.multiProcessorCount;
    out->cc_major = prop.major;
    out->cc_minor = prop.minor;
    out->l2_bytes = prop.l2CacheSize;
    out->hbm_bytes = int64_t(prop.totalGlobalMem);
    return ML_OK;
}

extern "C" int ml_synchronize(void) {
    int rc = ensure_init();
    if (rc) return rc;
    ML_CUDA(cudaStreamSynchronize(g_dev.stream));
    return ML_OK;
}

// ---- ABI: memory -----------------------------------------------------------------------
extern "C" int ml_alloc(uint64_t bytes, void **dptr) {
    int rc = ensure_init();
    if (rc) return rc;
    *dptr = nullptr;
    if (bytes == 0) return ML_OK;
    cudaError_t e = cudaMalloc(dptr, bytes);
    if (e != cudaSuccess) ML_FAIL(ML_ENOMEM, "cudaMalloc(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
    return ML_OK;
}
extern "C" int ml_free(void *dptr) {
    if (dptr) ML_CUDA(cudaFree(dptr));
    return ML_OK;
}
extern "C" int ml_host_alloc(uint64_t bytes, void **hptr) {
    int rc = ensure_init();
    if (rc) return rc;
    cudaError_t e = cudaHostAlloc(hptr, std::max<uint64_t>(bytes, 8), cudaHostAllocPortable);
    if (e != cudaSuccess) ML_FAIL(ML_ENOMEM, "cudaHostAlloc(%llu) failed: %s", (unsigned long long)bytes, cudaGetErrorString(e));
    return ML_OK;
}
extern "C" int ml_host_free(void *hptr) {
    if (hptr) ML_CUDA(cudaFreeHost(hptr));
    return ML_OK;
}
extern "C" int ml_upload(void *dst, const void *src, uint64_t bytes) {
    int rc = ensure_init();
    if (rc) return rc;
    if (bytes) ML_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g_dev.stream));
    return ML_OK;
}
extern "C" int ml_download(void *dst, const void *src, uint64_t bytes) {
    int rc = ensure_init();
    if (rc) return rc;
    if (bytes) ML_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g_dev.stream));
    ML_CUDA(cudaStreamSynchronize(g_dev.stream));
    return ML_OK;
}
extern "C" int ml_memset(void *dst, int value, uint64_t bytes) {
    int rc = ensure_init();
    if (rc) return rc;
    if (bytes) ML_CUDA(cudaMemsetAsync(dst, value, bytes, g_dev.stream));
    return ML_OK;
}
extern "C" int ml_upload2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                           uint64_t height) {
    int rc = ensure_init();
    if (rc) return rc;
    if (width && height)
        ML_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, g_dev.stream));
    return ML_OK;
}
extern "C" int ml_download2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                             uint64_t height) {
    int rc = ensure_init();
    if (rc) return rc;
    if (width && height)
        ML_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, g_dev.stream));
    ML_CUDA(cudaStreamSynchronize(g_dev.stream));
    return ML_OK;
}
extern "C" int ml_copy_h2d_2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                              uint64_t height) {
    int rc = ensure_init();
    if (rc) return rc;
    if (width && height)
        ML_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, g_dev.copy[0]));
    return ML_OK;
}
extern "C" int ml_copy_d2h_2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                              uint64_t height) {
    int rc = ensure_init();
    if (rc) return rc;
    if (width && height)
        ML_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, g_dev.copy[1]));
    return ML_OK;
}
extern "C" int ml_seg_params(int32_t *seg_shift, int32_t *seg_pad, int32_t *seg_max_dim,
                             int32_t *seg_min_dim) {
    if (seg_shift) *seg_shift = ML_SEG_SHIFT;
    if (seg_pad) *seg_pad = ML_SEG_PAD;
    if (seg_max_dim) *seg_max_dim = ML_SEG_MAX_DIM;
    if (seg_min_dim) *seg_min_dim = ML_SEG_MIN_DIM;
    return ML_OK;
}
static cudaStream_t stream_of(int32_t which);
// Segmented <-> plain SOA on the device: component c of element e sits at
// c * n + e in the plain (host-order) copy and at
// (e >> s) * P * dim + c * P + (e & (2^s - 1)) in the segmented one.  Both
// sides are contiguous runs along e, so the kernel is a coalesced copy.
__global__ void k_seg_repack(uint64_t *seg, uint64_t *plain, int64_t n, int32_t dim, int32_t shift, int64_t P,
                             int32_t to_seg) {
    const int64_t c = blockIdx.y;
    const int64_t mask = (int64_t(1) << shift) - 1;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = (e >> shift) * P * dim + c * P + (e & mask);
        if (to_seg) seg[j] = plain[c * n + e];
        else plain[c * n + e] = seg[j];
    }
}

// per-stream staging buffer of the segmented copies (grown on demand)
static void *stage_buffer(int32_t which, uint64_t bytes, int *rc) {
    static void *buf[3] = {nullptr, nullptr, nullptr};
    static uint64_t cap[3] = {0, 0, 0};
    const int k = which == ML_STREAM_H2D ? 1 : which == ML_STREAM_D2H ? 2 : 0;
    if (cap[k] < bytes) {
        if (buf[k]) cudaFree(buf[k]);              // synchronises: no copy still uses it
        buf[k] = nullptr;
        cap[k] = 0;
        if (cudaMalloc(&buf[k], bytes) != cudaSuccess) {
            *rc = ML_ENOMEM;
            return nullptr;
        }
        cap[k] = bytes;
    }
    *rc = ML_OK;
    return buf[k];
}

extern "C" int ml_seg_copy(void *dev, void *host, int64_t n, int32_t dim, int32_t itemsize, int32_t seg_shift,
                           int32_t to_device, int32_t stream) {
    int rc = ensure_init();
    if (rc) return rc;
    if (n < 0 || dim < 1 || dim > 65535 || itemsize != 8 || seg_shift < 1 || seg_shift > 30)
        ML_FAIL(ML_EINVAL, "ml_seg_copy: bad arguments");
    if (n == 0) return ML_OK;
    cudaStream_t s = stream_of(stream);
    const uint64_t bytes = uint64_t(n) * uint64_t(dim) * 8;
    const int64_t P = (int64_t(1) << seg_shift) + ML_SEG_PAD;
    const dim3 grid(unsigned(std::min<int64_t>((n + 255) / 256, 4 * g_dev.sm_count)), unsigned(dim));
    // download into pinned host memory: the repack kernel writes it directly
    // over PCIe (one pass)
    cudaPointerAttributes at{};
    if (!to_device && cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost &&
        at.devicePointer) {
        k_seg_repack<<<grid, 256, 0, s>>>(static_cast<uint64_t *>(dev), static_cast<uint64_t *>(at.devicePointer), n,
                                          dim, seg_shift, P, 0);
        ML_CUDA(cudaGetLastError());
        if (stream == ML_STREAM_COMPUTE) ML_CUDA(cudaStreamSynchronize(s));
        return ML_OK;
    }
    cudaGetLastError();                                // clear a pageable-pointer query error
    // upload on the H2D stream: alternate two staging buffers so the next PCIe
    // copy never waits for this one's repack (which runs on g_dev.repack)
    if (to_device && stream == ML_STREAM_H2D) {
        const int k = g_dev.stage_next;
        g_dev.stage_next ^= 1;
        if (g_dev.stage_cap[k] < bytes) {               // grow both: uploads alternate between them
            for (int j = 0; j < 2; ++j) {
                if (g_dev.stage[j]) cudaFree(g_dev.stage[j]);   // synchronises: no repack still reads it
                g_dev.stage[j] = nullptr;
                g_dev.stage_cap[j] = 0;
                if (cudaMalloc(&g_dev.stage[j], bytes) != cudaSuccess)
                    ML_FAIL(ML_ENOMEM, "ml_seg_copy: staging buffer of %llu bytes", (unsigned long long)bytes);
                g_dev.stage_cap[j] = bytes;
            }
        }
        ML_CUDA(cudaStreamWaitEvent(s, g_dev.stage_done[k], 0));
        ML_CUDA(cudaMemcpyAsync(g_dev.stage[k], host, bytes, cudaMemcpyHostToDevice, s));
        ML_CUDA(cudaEventRecord(g_dev.stage_copied[k], s));
        ML_CUDA(cudaStreamWaitEvent(g_dev.repack, g_dev.stage_copied[k], 0));
        k_seg_repack<<<grid, 256, 0, g_dev.repack>>>(static_cast<uint64_t *>(dev),
                                                     static_cast<uint64_t *>(g_dev.stage[k]), n, dim, seg_shift, P, 1);
        ML_CUDA(cudaGetLastError());
        ML_CUDA(cudaEventRecord(g_dev.stage_done[k], g_dev.repack));
        return ML_OK;
    }
    void *st = stage_buffer(stream, bytes, &rc);
    if (rc) ML_FAIL(ML_ENOMEM, "ml_seg_copy: staging buffer of %llu bytes", (unsigned long long)bytes);
    if (to_device) {
        ML_CUDA(cudaMemcpyAsync(st, host, bytes, cudaMemcpyHostToDevice, s));
        k_seg_repack<<<grid, 256, 0, s>>>(static_cast<uint64_t *>(dev), static_cast<uint64_t *>(st), n, dim,
                                          seg_shift, P, 1);
    } else {
        k_seg_repack<<<grid, 256, 0, s>>>(static_cast<uint64_t *>(dev), static_cast<uint64_t *>(st), n, dim,
                                          seg_shift, P, 0);
        ML_CUDA(cudaMemcpyAsync(host, st, bytes, cudaMemcpyDeviceToHost, s));
    }
    ML_CUDA(cudaGetLastError());
    if (!to_device && stream == ML_STREAM_COMPUTE) ML_CUDA(cudaStreamSynchronize(s));
    return ML_OK;
}
static cudaStream_t stream_of(int32_t which) {
    return which == ML_STREAM_H2D ? g_dev.copy[0] : which == ML_STREAM_D2H ? g_dev.copy[1] : g_dev.stream;
}
extern "C" int ml_copy_h2d(void *dst, const void *src, uint64_t bytes) {
    int rc = ensure_init();
    if (rc) return rc;
    if (bytes) ML_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g_dev.copy[0]));
    return ML_OK;
}
extern "C" int ml_copy_d2h(void *dst, const void *src, uint64_t bytes) {
    int rc = ensure_init();
    if (rc) return rc;
    if (bytes) ML_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g_dev.copy[1]));
    return ML_OK;
}
extern "C" int ml_order(int32_t from, int32_t to) {
    int rc = ensure_init();
    if (rc) return rc;
    if (from == to) return ML_OK;
    cudaEvent_t ev = g_dev.order_ev[g_dev.order_next];
    g_dev.order_next = (g_dev.order_next + 1) % 64;
    ML_CUDA(cudaEventRecord(ev, stream_of(from)));
    ML_CUDA(cudaStreamWaitEvent(stream_of(to), ev, 0));
    if (from == ML_STREAM_H2D) {                   // segmented uploads finish on the repack stream
        ML_CUDA(cudaEventRecord(g_dev.repack_ev, g_dev.repack));
        ML_CUDA(cudaStreamWaitEvent(stream_of(to), g_dev.repack_ev, 0));
    }
    return ML_OK;
}
extern "C" int ml_sync_all(void) {
    int rc = ensure_init();
    if (rc) return rc;
    ML_CUDA(cudaStreamSynchronize(g_dev.copy[0]));
    ML_CUDA(cudaStreamSynchronize(g_dev.repack));
    ML_CUDA(cudaStreamSynchronize(g_dev.stream));
    ML_CUDA(cudaStreamSynchronize(g_dev.copy[1]));
    return ML_OK;
}

extern "C" int ml_map_upload(int32_t *dst, const int64_t *table, int64_t rows, int32_t arity) {
    int rc = ensure_init();
    if (rc) return rc;
    const uint64_t n = uint64_t(rows) * arity;
    if (!n) return ML_OK;
    int64_t *tmp = nullptr;
    ML_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&tmp), n * 8, g_dev.stream));
    ML_CUDA(cudaMemcpyAsync(tmp, table, n * 8, cudaMemcpyHostToDevice, g_dev.stream));
    const int grid = int(std::min<uint64_t>((n + 255) / 256, 65535));
    k_map_to_i32<<<grid, 256, 0, g_dev.stream>>>(dst, tmp, rows, arity);
    ML_CUDA(cudaGetLastError());
    ML_CUDA(cudaFreeAsync(tmp, g_dev.stream));
    ML_CUDA(cudaStreamSynchronize(g_dev.stream));   // `table` is borrowed
    return ML_OK;
}

// ---- ABI: functors and loops --------------------------------------------------------------
extern "C" int ml_functor_lookup(const char *name, int32_t dtype, int32_t *functor_id) {
    auto &reg = registry();
    for (size_t i = 0; i < reg.size(); ++i)
        if (std::strcmp(reg[i].name, name) == 0 && reg[i].dtype == dtype) {
            *functor_id = int32_t(i);
            return ML_OK;
        }
    ML_FAIL(ML_ENOFUNCTOR, "no compiled functor '%s' for dtype %s", name, dtype == ML_F64 ? "float64" : "int64");
}

extern "C" int ml_chain_lookup(const char *first, const char *second, char *fused, int32_t buflen,
                               int32_t *na, int32_t *apos, int32_t *nb, int32_t *bpos) {
    for (const ChainEntry &c : chains())
        if (std::strcmp(c.first, first) == 0 && std::strcmp(c.second, second) == 0) {
            if (fused && buflen > 0) {
                std::strncpy(fused, c.fused, size_t(buflen) - 1);
                fused[buflen - 1] = 0;
            }
            if (na) *na = c.na;
            if (nb) *nb = c.nb;
            if (apos) std::memcpy(apos, c.apos, sizeof(int32_t) * size_t(c.na));
            if (bpos) std::memcpy(bpos, c.bpos, sizeof(int32_t) * size_t(c.nb));
            return ML_OK;
        }
    return ML_ENOFUNCTOR;      // no chain: not an error condition, no message set
}

extern "C" int ml_functor_signature(int32_t id, int32_t *nargs, int32_t *kinds, int32_t *modes,
                                    int32_t *dims, int32_t *dtypes) {
    auto &reg = registry();
    if (id < 0 || id >= int(reg.size())) ML_FAIL(ML_ENOFUNCTOR, "bad functor id %d", id);
    const FunctorEntry &f = reg[id];
    *nargs = f.nargs;
    for (int i = 0; i < f.nargs; ++i) {
        if (kinds) kinds[i] = f.kind[i];
        if (modes) modes[i] = f.mode[i];
        if (dims) dims[i] = f.dim[i];
        if (dtypes) dtypes[i] = f.atype[i];
    }
    return ML_OK;
}

extern "C" int ml_functor_count(int32_t *count) {
    *count = int32_t(registry().size());
    return ML_OK;
}

extern "C" int ml_functor_name(int32_t id, char *buf, int32_t buflen, int32_t *dtype) {
    auto &reg = registry();
    if (id < 0 || id >= int(reg.size())) ML_FAIL(ML_ENOFUNCTOR, "bad functor id %d", id);
    std::snprintf(buf, size_t(buflen), "%s", reg[id].name);
    if (dtype) *dtype = reg[id].dtype;
    return ML_OK;
}

extern "C" int ml_functor_rec_cols(int32_t id, int8_t *cols, int32_t *n) {
    auto &reg = registry();
    if (id < 0 || id >= int(reg.size()) || !n) ML_FAIL(ML_ENOFUNCTOR, "bad functor id %d", id);
    *n = reg[id].nrec_cols;
    if (cols)
        for (int i = 0; i < reg[id].nrec_cols; ++i) cols[i] = reg[id].rec_cols[i];
    return ML_OK;
}

extern "C" int ml_loop_scratch_bytes(const ml_loop_t *loop, uint64_t *bytes) {
    auto &reg = registry();
    if (loop->functor < 0 || loop->functor >= int(reg.size())) ML_FAIL(ML_ENOFUNCTOR, "bad functor id");
    *bytes = scratch_bytes(loop, reg[loop->functor]);
    return ML_OK;
}

extern "C" int ml_loop_pfold_slot_bytes(const ml_loop_t *L, uint64_t *bytes) {
    auto &reg = registry();
    if (!L || !bytes || L->functor < 0 || L->functor >= int(reg.size()))
        ML_FAIL(ML_EINVAL, "ml_loop_pfold_slot_bytes: bad arguments");
    const FunctorEntry &f = reg[L->functor];
    *bytes = f.pfold1[0] ? uint64_t(L->n) * uint64_t(f.pfold_nslot) * uint64_t(f.pfold_dgp) * 8 : 0;
    return ML_OK;
}

extern "C" int ml_loop_run(const ml_loop_t *loop) {
    int rc = ensure_init();
    if (rc) return rc;
    return enqueue_loop(loop, g_dev.stream);
}

// ---- ABI: programs -----------------------------------------------------------------------------
struct ml_program {
    std::vector<ml_loop_t> loops;
    std::vector<std::vector<ml_arg_t>> args;
    std::vector<std::vector<int64_t>> color_offsets;
    std::vector<std::string> names;
    void *ghost = nullptr, *gdev = nullptr;
    uint64_t gbytes = 0;
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t texec = nullptr;             // sequential graph with per-loop timing events
    cudaGraph_t tgraph = nullptr;
    std::vector<cudaEvent_t> events;
    std::vector<float> times;
    // concurrent loops (untimed runs and graphs): loop j waits only for the
    // earlier loops it conflicts with — sharing a dat or global buffer that
    // either of them writes — so independent loops overlap on side streams
    int32_t concurrent = 0;
    std::vector<std::vector<int>> deps;
    std::vector<int> lane;                       // stream of each loop (0: main)
    std::vector<cudaEvent_t> done;               // per loop, after its last kernel
    cudaStream_t side[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t fork = nullptr;
};

static constexpr int kLanes = 4;

// dependency DAG of a program: j depends on i < j when they share a buffer
// (dat payload or global slot) and at least one of them writes it
static void program_deps(ml_program *p) {
    const size_t n = p->loops.size();
    p->deps.assign(n, {});
    p->lane.assign(n, 0);
    for (size_t j = 0; j < n; ++j) {
        const ml_loop_t &B = p->loops[j];
        for (size_t i = 0; i < j; ++i) {
            const ml_loop_t &A = p->loops[i];
            bool conflict = false;
            for (int x = 0; x < A.nargs && !conflict; ++x)
                for (int y = 0; y < B.nargs && !conflict; ++y)
                    conflict = A.args[x].data && A.args[x].data == B.args[y].data &&
                               (A.args[x].mode != ML_READ || B.args[y].mode != ML_READ);
            if (conflict) p->deps[j].push_back(int(i));
        }
        // lane: the latest dependency's lane (fewest cross-stream waits), else a free one
        int lane = -1;
        if (!p->deps[j].empty()) lane = p->lane[p->deps[j].back()];
        if (lane < 0) {
            std::vector<int> last(kLanes, -1);
            for (size_t i = 0; i < j; ++i) last[p->lane[i]] = int(i);
            lane = 0;
            for (int k = 0; k < kLanes; ++k)
                if (last[k] < last[lane]) lane = k;
        }
        p->lane[j] = lane;
    }
}

// `external`: the timing events become event-record nodes of a graph being
// captured (cudaEventRecordExternal), so their elapsed times are readable
static int program_enqueue(ml_program *p, bool timed, bool external = false) {
    cudaStream_t s = g_dev.stream;
    const unsigned rec = external ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (p->gbytes) ML_CUDA(cudaMemcpyAsync(p->gdev, p->ghost, p->gbytes, cudaMemcpyHostToDevice, s));
    if (timed || !p->concurrent) {
        for (size_t i = 0; i < p->loops.size(); ++i) {
            if (timed) ML_CUDA(cudaEventRecordWithFlags(p->events[i], s, rec));
            int rc = enqueue_loop(&p->loops[i], s);
            if (rc) return rc;
        }
        if (timed) ML_CUDA(cudaEventRecordWithFlags(p->events[p->loops.size()], s, rec));
    } else {
        cudaStream_t lanes[kLanes] = {s, p->side[0], p->side[1], p->side[2]};
        ML_CUDA(cudaEventRecord(p->fork, s));                 // side lanes join (capture-safe)
        for (int k = 1; k < kLanes; ++k) ML_CUDA(cudaStreamWaitEvent(lanes[k], p->fork, 0));
        for (size_t i = 0; i < p->loops.size(); ++i) {
            cudaStream_t ls = lanes[p->lane[i]];
            for (int d : p->deps[i])
                if (p->lane[d] != p->lane[i]) ML_CUDA(cudaStreamWaitEvent(ls, p->done[d], 0));
            int rc = enqueue_loop(&p->loops[i], ls);
            if (rc) return rc;
            ML_CUDA(cudaEventRecord(p->done[i], ls));
        }
        for (size_t i = 0; i < p->loops.size(); ++i)          // join every lane's tail
            if (p->lane[i] != 0) ML_CUDA(cudaStreamWaitEvent(s, p->done[i], 0));
    }
    if (p->gbytes) ML_CUDA(cudaMemcpyAsync(p->ghost, p->gdev, p->gbytes, cudaMemcpyDeviceToHost, s));
    return ML_OK;
}

extern "C" int ml_program_create(const ml_loop_t *loops, int32_t nloops, void *globals_host,
                                 void *globals_dev, uint64_t globals_bytes, ml_program_t **out) {
    int rc = ensure_init();
    if (rc) return rc;
    ML_GUARD_BEGIN
    auto p = std::make_unique<ml_program>();
    p->loops.assign(loops, loops + nloops);
    p->args.resize(nloops);
    p->color_offsets.resize(nloops);
    p->names.resize(nloops);
    for (int i = 0; i < nloops; ++i) {
        ml_loop_t &L = p->loops[i];
        p->args[i].assign(L.args, L.args + L.nargs);
        L.args = p->args[i].data();
        p->names[i] = L.name ? L.name : "?";
        L.name = p->names[i].c_str();
        if (L.plan.color_offsets) {
            p->color_offsets[i].assign(L.plan.color_offsets, L.plan.color_offsets + L.plan.ncolors + 1);
            L.plan.color_offsets = p->color_offsets[i].data();
        }
        auto &reg = registry();
        if (L.functor < 0 || L.functor >= int(reg.size())) ML_FAIL(ML_ENOFUNCTOR, "bad functor id");
        rc = validate(&L, reg[L.functor]);
        if (rc) return rc;
    }
    p->ghost = globals_host;
    p->gdev = globals_dev;
    p->gbytes = globals_bytes;
    p->events.resize(size_t(nloops) + 1);
    for (auto &e : p->events) ML_CUDA(cudaEventCreate(&e));
    p->times.assign(nloops, 0.f);
    program_deps(p.get());
    p->done.resize(size_t(nloops));
    for (auto &e : p->done) ML_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ML_CUDA(cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming));
    for (auto &st : p->side) ML_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    *out = p.release();
    return ML_OK;
    ML_GUARD_END
}

static int program_capture(ml_program *p) {
    if (p->exec) return ML_OK;
    cudaStream_t s = g_dev.stream;
    ML_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int rc = program_enqueue(p, false);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) ML_FAIL(ML_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    p->graph = g;
    ML_CUDA(cudaGraphInstantiate(&p->exec, g, 0));
    return ML_OK;
}

// per-loop device times of the steady-state graph: a sequential capture with
// an event record node between loops (timing events work inside graphs)
static int program_capture_timed(ml_program *p) {
    if (p->texec) return ML_OK;
    cudaStream_t s = g_dev.stream;
    ML_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int rc = program_enqueue(p, true, true);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) ML_FAIL(ML_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    p->tgraph = g;
    ML_CUDA(cudaGraphInstantiate(&p->texec, g, 0));
    return ML_OK;
}

extern "C" int ml_program_replay_timed(ml_program_t *p, int32_t count, float *ms) {
    int rc = ensure_init();
    if (rc) return rc;
    if (!p || !ms || count < 1) ML_FAIL(ML_EINVAL, "ml_program_replay_timed: bad arguments");
    rc = program_capture_timed(p);
    if (rc) return rc;
    std::vector<double> acc(p->loops.size(), 0.0);
    for (int32_t i = 0; i < count; ++i) {
        ML_CUDA(cudaGraphLaunch(p->texec, g_dev.stream));
        ML_CUDA(cudaStreamSynchronize(g_dev.stream));
        for (size_t j = 0; j < p->loops.size(); ++j) {
            float t = 0.f;
            ML_CUDA(cudaEventElapsedTime(&t, p->events[j], p->events[j + 1]));
            acc[j] += t;
        }
    }
    for (size_t j = 0; j < p->loops.size(); ++j) ms[j] = float(acc[j] / count);
    return ML_OK;
}

extern "C" int ml_program_replay(ml_program_t *p, int32_t count) {
    int rc = ensure_init();
    if (rc) return rc;
    rc = program_capture(p);
    if (rc) return rc;
    for (int32_t i = 0; i < count; ++i) ML_CUDA(cudaGraphLaunch(p->exec, g_dev.stream));
    ML_CUDA(cudaStreamSynchronize(g_dev.stream));
    return ML_OK;
}

extern "C" int ml_program_run(ml_program_t *p, int32_t use_graph, int32_t time_loops) {
    int rc = ensure_init();
    if (rc) return rc;
    cudaStream_t s = g_dev.stream;
    if (use_graph) {
        rc = program_capture(p);
        if (rc) return rc;
        ML_CUDA(cudaGraphLaunch(p->exec, s));
        ML_CUDA(cudaStreamSynchronize(s));
        return ML_OK;
    }
    rc = program_enqueue(p, time_loops != 0);
    if (rc) return rc;
    ML_CUDA(cudaStreamSynchronize(s));
    if (time_loops)
        for (size_t i = 0; i < p->loops.size(); ++i)
            ML_CUDA(cudaEventElapsedTime(&p->times[i], p->events[i], p->events[i + 1]));
    return ML_OK;
}

extern "C" int ml_program_set_concurrent(ml_program_t *p, int32_t on) {
    if (!p) ML_FAIL(ML_EINVAL, "ml_program_set_concurrent: null");
    if (p->concurrent != (on != 0) && p->exec) {          // re-capture with the new structure
        cudaGraphExecDestroy(p->exec);
        cudaGraphDestroy(p->graph);
        p->exec = nullptr;
        p->graph = nullptr;
    }
    p->concurrent = on != 0;
    return ML_OK;
}

extern "C" int ml_program_deps(const ml_program_t *p, int32_t loop, int32_t *ndeps, int32_t *deps,
                               int32_t *lane) {
    if (!p || loop < 0 || loop >= int32_t(p->loops.size())) ML_FAIL(ML_EINVAL, "ml_program_deps: bad loop");
    if (ndeps) *ndeps = int32_t(p->deps[loop].size());
    if (deps) std::copy(p->deps[loop].begin(), p->deps[loop].end(), deps);
    if (lane) *lane = p->lane[loop];
    return ML_OK;
}

extern "C" int ml_program_loop_times(const ml_program_t *p, float *ms) {
    std::copy(p->times.begin(), p->times.end(), ms);
    return ML_OK;
}

extern "C" int ml_program_free(ml_program_t *p) {
    if (!p) return ML_OK;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    if (p->texec) cudaGraphExecDestroy(p->texec);
    if (p->tgraph) cudaGraphDestroy(p->tgraph);
    for (auto &e : p->events) cudaEventDestroy(e);
    for (auto &e : p->done) cudaEventDestroy(e);
    if (p->fork) cudaEventDestroy(p->fork);
    for (auto &st : p->side)
        if (st) cudaStreamDestroy(st);
    delete p;
    return ML_OK;
}

// ---- ABI: multi-GPU helpers --------------------------------------------------------------------
namespace ml {
// element (e, c) of a dat given the ABI's (elem_stride, comp_stride): a
// negative elem_stride -S means segmented SOA with segments of S elements
// and component stride comp_stride
__device__ __forceinline__ int64_t row_index(int64_t e, int c, int dim, int64_t se, int64_t sc) {
    if (se < 0) return (e / -se) * sc * dim + c * sc + (e % -se);
    return e * se + c * sc;
}
__global__ void k_pack_rows(double *dst, const double *dat, const int32_t *idx, int64_t nidx, int dim,
                            int64_t se, int64_t sc) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nidx * dim;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = k / dim, c = k % dim;
        dst[k] = dat[row_index(idx[r], int(c), dim, se, sc)];
    }
}
__global__ void k_unpack_rows(double *dat, const double *src, const int32_t *idx, int64_t nidx, int dim,
                              int64_t se, int64_t sc) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nidx * dim;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = k / dim, c = k % dim;
        dat[row_index(idx[r], int(c), dim, se, sc)] = src[k];
    }
}
// NVLink halo exchange: pack the export rows straight into the peer's import
// buffer (an IPC-mapped pointer), then — once every CTA's remote stores are
// fenced system-wide — bump the peer's arrival counter for this rank.
__global__ void k_put_rows(double *rdst, const double *dat, const int32_t *idx, int64_t nidx, int dim,
                           int64_t se, int64_t sc, unsigned long long *rflag, int *counter) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nidx * dim;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = k / dim, c = k % dim;
        rdst[k] = dat[row_index(idx[r], int(c), dim, se, sc)];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(counter, 1) == int(gridDim.x) - 1) {
        *counter = 0;                                   // ready for the next exchange
        __threadfence_system();
        atomicAdd_system(rflag, 1ull);
    }
}
// Wait (one thread) until the local arrival counter of a source reaches the
// next expected value; `expected` lives in device memory so graph replays
// keep counting.  Bounded by `timeout_ns` (globaltimer): on expiry the wait
// records `code` in `err` (first error wins) and lets the stream go on; the
// host raises ExchangeTimeout after the run (reference executor.py:343-359).
__global__ void k_wait_flag(const unsigned long long *flag, unsigned long long *expected,
                            unsigned long long timeout_ns, long long *err, long long code) {
    const unsigned long long want = *expected + 1;
    *expected = want;
    unsigned long long v, t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= want) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (timeout_ns && t - t0 > timeout_ns) {
            if (err) atomicCAS(reinterpret_cast<unsigned long long *>(err), 0ull,
                               static_cast<unsigned long long>(code));
            break;
        }
        __nanosleep(256);
    }
}

__global__ void k_signal(unsigned long long *rflag) {
    __threadfence_system();
    atomicAdd_system(rflag, 1ull);
}

__device__ __forceinline__ bool wait_counter(const unsigned long long *flag, unsigned long long want,
                                             unsigned long long timeout_ns, long long *err, long long code) {
    unsigned long long v, t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        if (v >= want) return true;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (timeout_ns && t - t0 > timeout_ns) {
            if (err) atomicCAS(reinterpret_cast<unsigned long long *>(err), 0ull,
                               static_cast<unsigned long long>(code));
            return false;
        }
        __nanosleep(64);
    }
}

// NVLink all-gather of a reduction partial: thread r waits until rank r has
// consumed this rank's previous row (credit), stores the partial into row `me`
// of rank r's gather buffer, fences system-wide and bumps r's delivery counter.
__global__ void k_reduce_put(const unsigned long long *partial, int nwords, unsigned long long *const *rrow,
                             unsigned long long *const *rdeliv, const unsigned long long *credit,
                             unsigned long long *credit_exp, int nranks, unsigned long long timeout_ns,
                             long long *err, long long code) {
    const int r = threadIdx.x;
    if (r >= nranks) return;
    const unsigned long long want = credit_exp[r] + 1;
    credit_exp[r] = want;
    wait_counter(credit + r, want, timeout_ns, err, -code);
    for (int w = 0; w < nwords; ++w) rrow[r][w] = partial[w];
    __threadfence_system();
    atomicAdd_system(rdeliv[r], 1ull);
}
// wait for every rank's row, fold the rows in rank order onto the value (the
// order of ml_combine_ranks), then return a credit to every source
template <class T, int M>
__global__ void k_reduce_fold(T *value, const T *rows, const unsigned long long *deliv,
                              unsigned long long *deliv_exp, unsigned long long *const *rcredit, int nranks,
                              int dim, unsigned long long timeout_ns, long long *err, long long code) {
    const int r = threadIdx.x;
    if (r < nranks) {
        const unsigned long long want = deliv_exp[r] + 1;
        deliv_exp[r] = want;
        wait_counter(deliv + r, want, timeout_ns, err, code);
    }
    __syncthreads();
    __threadfence_system();
    for (int c = threadIdx.x; c < dim; c += blockDim.x) {
        T v = value[c];
        for (int q = 0; q < nranks; ++q) v = combine<M>(v, __ldcv(rows + int64_t(q) * dim + c));
        value[c] = v;
    }
    __syncthreads();
    if (r < nranks) {
        __threadfence_system();
        atomicAdd_system(rcredit[r], 1ull);
    }
}

template <class T, int M>
__global__ void k_combine_ranks(T *value, const T *gathered, int nranks, int dim) {
    for (int c = threadIdx.x; c < dim; c += blockDim.x) {
        T v = value[c];
        for (int r = 0; r < nranks; ++r) v = combine<M>(v, gathered[r * dim + c]);
        value[c] = v;
    }
}
}  // namespace ml

extern "C" int ml_pack_rows(void *dst, const void *dat, const int32_t *idx, int64_t nidx, int32_t dim,
                            int64_t se, int64_t sc) {
    int rc = ensure_init();
    if (rc) return rc;
    if (nidx <= 0) return ML_OK;
    const int64_t work = nidx * dim;
    const int grid = int(std::min<int64_t>((work + 255) / 256, 4 * 148));
    k_pack_rows<<<grid, 256, 0, g_dev.stream>>>(static_cast<double *>(dst), static_cast<const double *>(dat),
                                               idx, nidx, dim, se, sc);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

extern "C" int ml_unpack_rows(void *dat, const void *src, const int32_t *idx, int64_t nidx, int32_t dim,
                              int64_t se, int64_t sc) {
    int rc = ensure_init();
    if (rc) return rc;
    if (nidx <= 0) return ML_OK;
    const int64_t work = nidx * dim;
    const int grid = int(std::min<int64_t>((work + 255) / 256, 4 * 148));
    k_unpack_rows<<<grid, 256, 0, g_dev.stream>>>(static_cast<double *>(dat), static_cast<const double *>(src),
                                                 idx, nidx, dim, se, sc);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

extern "C" int ml_ipc_handle(void *dptr, void *handle) {
    int rc = ensure_init();
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    ML_CUDA(cudaIpcGetMemHandle(&h, dptr));
    std::memcpy(handle, &h, sizeof h);
    return ML_OK;
}
extern "C" int ml_ipc_open(const void *handle, void **dptr) {
    int rc = ensure_init();
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    ML_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    return ML_OK;
}
extern "C" int ml_ipc_close(void *dptr) {
    if (dptr) ML_CUDA(cudaIpcCloseMemHandle(dptr));
    return ML_OK;
}
extern "C" int ml_put_rows(void *remote_dst, const void *dat, const int32_t *idx, int64_t nidx, int32_t dim,
                           int64_t se, int64_t sc, uint64_t *remote_flag, int32_t *counter) {
    int rc = ensure_init();
    if (rc) return rc;
    const int64_t work = std::max<int64_t>(nidx * dim, 1);
    const int grid = int(std::min<int64_t>((work + 255) / 256, 2 * 148));
    k_put_rows<<<grid, 256, 0, g_dev.stream>>>(static_cast<double *>(remote_dst), static_cast<const double *>(dat),
                                               idx, nidx, dim, se, sc,
                                               reinterpret_cast<unsigned long long *>(remote_flag), counter);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}
extern "C" int ml_signal_flag(uint64_t *remote_flag) {
    int rc = ensure_init();
    if (rc) return rc;
    k_signal<<<1, 1, 0, g_dev.stream>>>(reinterpret_cast<unsigned long long *>(remote_flag));
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}
extern "C" int ml_wait_flag(const uint64_t *flag, uint64_t *expected, uint64_t timeout_ns, int64_t *err,
                            int64_t code) {
    int rc = ensure_init();
    if (rc) return rc;
    k_wait_flag<<<1, 1, 0, g_dev.stream>>>(reinterpret_cast<const unsigned long long *>(flag),
                                            reinterpret_cast<unsigned long long *>(expected), timeout_ns,
                                            reinterpret_cast<long long *>(err), code);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

extern "C" int ml_reduce_put(const void *partial, int32_t nbytes, void *const *remote_rows,
                             uint64_t *const *remote_delivery, const uint64_t *credit, uint64_t *credit_expected,
                             int32_t nranks, uint64_t timeout_ns, int64_t *err, int64_t code) {
    int rc = ensure_init();
    if (rc) return rc;
    if (nranks < 1 || nranks > 1024 || nbytes % 8) ML_FAIL(ML_EINVAL, "ml_reduce_put: bad arguments");
    k_reduce_put<<<1, nranks, 0, g_dev.stream>>>(
        static_cast<const unsigned long long *>(partial), nbytes / 8,
        reinterpret_cast<unsigned long long *const *>(remote_rows),
        reinterpret_cast<unsigned long long *const *>(remote_delivery),
        reinterpret_cast<const unsigned long long *>(credit), reinterpret_cast<unsigned long long *>(credit_expected),
        nranks, timeout_ns, reinterpret_cast<long long *>(err), code);
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}
extern "C" int ml_reduce_fold(void *value, const void *rows, const uint64_t *delivery, uint64_t *delivery_expected,
                              uint64_t *const *remote_credit, int32_t nranks, int32_t dim, int32_t mode,
                              int32_t dtype, uint64_t timeout_ns, int64_t *err, int64_t code) {
    int rc = ensure_init();
    if (rc) return rc;
    if (nranks < 1 || nranks > 1024) ML_FAIL(ML_EINVAL, "ml_reduce_fold: bad arguments");
    cudaStream_t s = g_dev.stream;
    const int threads = std::max(32, (std::max<int>(nranks, dim) + 31) / 32 * 32);
    auto d = reinterpret_cast<const unsigned long long *>(delivery);
    auto de = reinterpret_cast<unsigned long long *>(delivery_expected);
    auto rcr = reinterpret_cast<unsigned long long *const *>(remote_credit);
    auto e = reinterpret_cast<long long *>(err);
#define ML_RF(T, M) k_reduce_fold<T, M><<<1, threads, 0, s>>>(static_cast<T *>(value), static_cast<const T *>(rows), \
                                                         d, de, rcr, nranks, dim, timeout_ns, e, code)
    if (dtype == ML_F64) {
        if (mode == ML_INC) ML_RF(double, MINC);
        else if (mode == ML_MIN) ML_RF(double, MMIN);
        else if (mode == ML_MAX) ML_RF(double, MMAX);
        else ML_FAIL(ML_EINVAL, "ml_reduce_fold: mode %d is not a reduction", mode);
    } else {
        if (mode == ML_INC) ML_RF(int64_t, MINC);
        else if (mode == ML_MIN) ML_RF(int64_t, MMIN);
        else if (mode == ML_MAX) ML_RF(int64_t, MMAX);
        else ML_FAIL(ML_EINVAL, "ml_reduce_fold: mode %d is not a reduction", mode);
    }
#undef ML_RF
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

extern "C" int ml_combine_ranks(void *value, const void *gathered, int32_t nranks, int32_t dim, int32_t mode,
                                int32_t dtype) {
    int rc = ensure_init();
    if (rc) return rc;
    cudaStream_t s = g_dev.stream;
#define ML_CR(T, M) k_combine_ranks<T, M><<<1, 32, 0, s>>>(static_cast<T *>(value), static_cast<const T *>(gathered), nranks, dim)
    if (dtype == ML_F64) {
        if (mode == ML_INC) ML_CR(double, MINC);
        else if (mode == ML_MIN) ML_CR(double, MMIN);
        else if (mode == ML_MAX) ML_CR(double, MMAX);
        else ML_FAIL(ML_EINVAL, "ml_combine_ranks: mode %d is not a reduction", mode);
    } else {
        if (mode == ML_INC) ML_CR(int64_t, MINC);
        else if (mode == ML_MIN) ML_CR(int64_t, MMIN);
        else if (mode == ML_MAX) ML_CR(int64_t, MMAX);
        else ML_FAIL(ML_EINVAL, "ml_combine_ranks: mode %d is not a reduction", mode);
    }
#undef ML_CR
    ML_CUDA(cudaGetLastError());
    return ML_OK;
}

extern "C" void *ml_stream(void) { return g_dev.stream; }

// ---- ABI: measurement helpers ----------------------------------------------------------------
extern "C" int ml_flush_l2(void) {
    int rc = ensure_init();
    if (rc) return rc;
    if (!g_dev.flush_buf) {
        g_dev.flush_bytes = size_t(std::max<int64_t>(g_dev.l2_bytes, 64 << 20)) * 2;
        ML_CUDA(cudaMalloc(&g_dev.flush_buf, g_dev.flush_bytes));
    }
    ML_CUDA(cudaMemsetAsync(g_dev.flush_buf, 0x5a, g_dev.flush_bytes, g_dev.stream));
    return ML_OK;
}

struct ml_timer {
    cudaEvent_t a, b;
};
extern "C" int ml_timer_create(ml_timer_t **t) {
    int rc = ensure_init();
    if (rc) return rc;
    auto *x = new ml_timer;
    ML_CUDA(cudaEventCreate(&x->a));
    ML_CUDA(cudaEventCreate(&x->b));
    *t = x;
    return ML_OK;
}
extern "C" int ml_timer_start(ml_timer_t *t) {
    ML_CUDA(cudaEventRecord(t->a, g_dev.stream));
    return ML_OK;
}
extern "C" int ml_timer_stop(ml_timer_t *t, float *ms) {
    ML_CUDA(cudaEventRecord(t->b, g_dev.stream));
    ML_CUDA(cudaEventSynchronize(t->b));
    ML_CUDA(cudaEventElapsedTime(ms, t->a, t->b));
    return ML_OK;
}
extern "C" int ml_timer_free(ml_timer_t *t) {
    if (!t) return ML_OK;
    cudaEventDestroy(t->a);
    cudaEventDestroy(t->b);
    delete t;
    return ML_OK;
}
