// Loop engine: one templated CUDA kernel family per loop *shape*, specialised
// at compile time for each hand-written functor (the B200 counterpart of the
// per-loop code OP2 generates; reference execution semantics executor.py:
// 149-275, plan consumption plan.py:30-45).
//
// A functor declares its argument signature (kind, access mode, dim, type)
// and a device `apply(consts, view0, view1, ...)`.  Views are
//   * Ref<T>/RefA<T>  — strided / contiguous references straight into HBM for
//     direct args, indirect READ args and (phased mode) indirect WRITE/RW
//     args; loads are issued at first use, so the compiler schedules them
//     and register pressure stays bounded for wide dats;
//   * T*              — a register array: increments of an indirect INC
//     argument, the running value of a gathered target, global INC/MIN/MAX
//     accumulators (block-reduced afterwards), and the two elements' rows a
//     thread of a vectorised direct loop owns.
//
// Layout policy (template parameter LP of every hot kernel).  LP = 0 reads
// each argument's strides at run time (element stride `se`, component stride
// `sc`: any AOS/SOA mix).  LP = 1 is the reference's default auto-SOA policy
// (core.py:403-404, threshold 4) fixed at compile time: a dat of dim <= 4 is
// AOS (base e * dim, component offsets are immediates), wider dats SOA in the
// device's segmented form (component offsets c * SEGP, immediates too).  The
// runtime picks LP = 1 when the loop's dats follow that policy — the common
// case — which removes the 64-bit stride arithmetic from every gathered load.
//
// Kernels (selected by runtime.cu enqueue_loop)
//   k_direct   — loops without indirect writes: persistent grid; with LP = 1
//                each thread owns two consecutive elements and moves their
//                direct rows with 16-byte loads/stores (north_star: coalesced
//                128-bit direct access).
//   k_gather   — target-centric INC-only or WRITE-only loops: one thread per
//                target re-evaluates the kernel for each incidence in serial
//                order (bitwise the serial result); hub targets split in rows
//                (k_gather_hubs folds them).
//   k_pfold1 + k_pfold_rest_w — primary fold for INC-only loops: each element
//                evaluated once by the owner of its first INC target; the other
//                increments through slots folded in element order (pass 2).
//   k_staged   — reference plan colours (one launch per block colour), INC
//                increments staged in registers and applied in element-colour
//                phases (run_threads, and loops the target-centric schedules
//                do not cover).
//   k_phased   — general colour schedule (indirect WRITE/RW): each element runs
//                entirely inside its colour phase.
// Global reductions: warp shuffle -> shared -> one partial per CTA;
// k_combine folds the partials in a fixed order onto the initial value.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda/std/limits>
#include <cuda/std/tuple>
#include <cuda/std/type_traits>
#include <cuda/std/utility>

#include "../../include/meshloop_b200.h"

namespace ml {

enum : int { KD = 0, KI = 1, KG = 2 };                        // direct / indirect / global
enum : int { MR = 0, MW = 1, MRW = 2, MINC = 3, MMIN = 4, MMAX = 5 };
constexpr int MAX_ARGS = 16;
constexpr int AUTO_SOA_DIM = 4;    // reference Mesh(auto_soa_threshold=4): dim > 4 is SOA
// Device SOA copies are *segmented*: the set is cut into segments of SEG
// elements and each segment stores its components one after another at a
// component stride of SEGP = SEG + 32 elements: element (e, c) at
// (e >> SEG_SHIFT) * SEGP * dim + c * SEGP + (e & (SEG - 1)).  Inside a
// segment a component is one contiguous run, so a warp's access is as
// coalesced as plain SOA; but the offset of component c from an element's
// base is the compile-time c * SEGP * 8 bytes — a load immediate — instead of
// c * set_size (a 64-bit multiply-add per load).  The 256-byte pad keeps the
// component stride off a power of two (a 32 KB stride maps all components
// of an element to one L1 set); SEG * 8 = 32 KB rows keep host<->device
// copies DMA-efficient (one 2-D copy per component).
constexpr int SEG_SHIFT = ML_SEG_SHIFT;          // include/meshloop_b200.h
constexpr int64_t SEG = int64_t(1) << SEG_SHIFT;
constexpr int64_t SEGP = SEG + ML_SEG_PAD;

// Programmatic dependent launch: the hot kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs can
// be resident while its predecessor on the stream drains; each such kernel
// waits (griddepcontrol.wait) for the predecessor's completion — and memory —
// before touching any data.  Without the attribute the wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();

template <class... KArgs, class... Args>
inline void launch_k(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args &&...args) {
    if (!pdl_enabled()) {
        k<<<g, b, smem, s>>>(static_cast<KArgs>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <int K, int M, int DIM, class T>
struct Arg {
    static constexpr int kind = K, mode = M, dim = DIM;
    using type = T;
};

template <class... As>
struct Sig {
    static constexpr int n = sizeof...(As);
};

template <class T>
constexpr int type_code() { return sizeof(T) == 8 && T(0.5) != T(0) ? 0 : 1; }   // 0 f64, 1 i64

struct ArgRt {
    void *data;
    const int32_t *map;   // map column (already offset by slot*from)
    int64_t se, sc;       // element stride, component stride (in elements)
    int32_t sh;           // segmented SOA: log2 of the segment length (0: linear)
    int64_t sb;           // segmented SOA: elements per segment (component stride * dim)
};

// offset (in elements) of element e's first component
__host__ __device__ __forceinline__ int64_t elem_base(const ArgRt &r, int64_t e) {
    if (r.sh) return (e >> r.sh) * r.sb + (e & ((int64_t(1) << r.sh) - 1));
    return e * r.se;
}

struct Consts {
    double f[4];
    int64_t i[4];
};

// Primary-fold schedule (INC-only loops): pass 1 gives each target the elements
// whose FIRST INC argument targets it; each element is evaluated once there,
// its first increment accumulated in the thread's registers and the others
// written to per-element slots; pass 2 folds each target's slots.
struct PFoldParams {
    int64_t n1;                          // targets with primary incidences
    const int32_t *off1, *elem1, *tl1;   // CSR (element ascending); tl1: target ids
    int64_t n2;                          // targets with secondary incidences
    const int32_t *off2, *elem2, *tl2;
    const uint8_t *pos2;                 // INC-argument position (>= 1) of each
    void *slots;                         // [secondary incidences][dgp], in off2 order
    const int32_t *slotpos;              // [n][nslot]: slot row of (element, INC position >= 1)
    int32_t nslot, dgp;
    // element records: per pass-1 incidence k, the map entries of its element
    // for each distinct (map, column) the loop uses — [n1 incidences][ncol];
    // rcol: record column of each indirect argument.  The rows' addresses then
    // depend on one load (the record) instead of two (element id, then map).
    const int32_t *rec;
    int32_t ncol;
    int8_t rcol[MAX_ARGS];
    // hub rows: a target with more than HUB_ROW incidences in a pass is split
    // into several rows; a split row accumulates from zero into partial slot
    // seg[row] of part (-1: ordinary row) and k_fold_parts adds each hub's
    // slots onto it in row (= element) order after the pass
    const int32_t *seg1, *seg2;
    void *part1, *part2;
};

struct LaunchParams {
    ArgRt a[MAX_ARGS];
    void *part[MAX_ARGS];       // reduction partials [nblocks][dim] per global reduce arg
    unsigned *ticket;           // single-launch schedules: CTA arrival counter, the last CTA
                                // folds the partials (nullptr: k_combine after the launches)
    int64_t n;
    int64_t rlim;               // elements >= rlim do not contribute to reductions
    int32_t bs;
    const int32_t *blocks;      // block ids of this launch (colour schedules)
    const uint16_t *ecol;       // element colours
    const int32_t *encol;       // per-block element colour count
    Consts k;
    // target-centric schedule: per target, its (element, INC-arg position)
    // incidences in serial order
    int64_t g_ntargets;
    const int32_t *g_off;
    const int32_t *g_elem;
    const uint8_t *g_pos;
    const int32_t *g_tlist;     // compacted target ids (nullptr: identity)
    // hub targets (INC only): a target with many incidences is split into
    // several rows; a split row accumulates from zero into partial slot
    // g_seg[row] (-1: ordinary row), k_gather_hubs folds the slots in order
    const int32_t *g_seg;
    void *g_part;
    int64_t g_nhub;
    const int32_t *g_hub_tl, *g_hub_off;
    PFoldParams pf;
};

// ---- views ----------------------------------------------------------------------------
// strided view of one element's components (runtime or SOA component stride)
template <class T>
struct Ref {
    T *p;
    int64_t sc;
    __device__ __forceinline__ T &operator[](int c) const { return p[c * sc]; }
};
// contiguous view (AOS with a compile-time layout): component offsets are immediates
template <class T>
struct RefA {
    T *p;
    __device__ __forceinline__ T &operator[](int c) const { return p[c]; }
};
// READ views of the target-centric schedules load through the read-only path
// (ld.global.nc): their eligibility rules (gather_eligible / fold_eligible)
// keep the written dat out of every other argument, so nothing a READ view
// reads is written during the launch.  The colour schedules keep coherent
// loads (a dat may be read there while other elements of the block update it).
template <class T>
struct RefNC {
    const T *p;
    int64_t sc;
    __device__ __forceinline__ T operator[](int c) const { return __ldg(p + c * sc); }
};
template <class T>
struct RefNCA {
    const T *p;
    __device__ __forceinline__ T operator[](int c) const { return __ldg(p + c); }
};

// layout class of argument A under policy LP: 0 runtime strides, 1 AOS (base
// e * dim, component stride 1), 2 segmented SOA (SEG_SHIFT, component stride
// SEGP), 3 plain SOA (component stride = the runtime pitch)
template <class A, int LP>
__host__ __device__ constexpr int lay_of() {
    return (LP == 0 || A::kind == KG) ? 0
           : A::dim <= AUTO_SOA_DIM                                 ? 1
           : (A::dim >= ML_SEG_MIN_DIM && A::dim <= ML_SEG_MAX_DIM) ? 2
                                                                    : 3;
}
// element base offset and component stride under layout class L
template <class A, int L>
__device__ __forceinline__ int64_t base_of(const ArgRt &r, int64_t e) {
    if constexpr (L == 1) return e * A::dim;
    else if constexpr (L == 2) return (e >> SEG_SHIFT) * (SEGP * A::dim) + (e & (SEG - 1));
    else if constexpr (L == 3) return e;
    else return elem_base(r, e);
}
template <class A, int L>
__device__ __forceinline__ int64_t sc_of(const ArgRt &r) {
    if constexpr (L == 1) return 1;
    else if constexpr (L == 2) return SEGP;
    else return r.sc;
}

template <class T, int M>
__device__ __forceinline__ T reduce_identity() {
    if (M == MMIN) return cuda::std::numeric_limits<T>::has_infinity
                              ? cuda::std::numeric_limits<T>::infinity()
                              : cuda::std::numeric_limits<T>::max();
    if (M == MMAX) return cuda::std::numeric_limits<T>::has_infinity
                              ? -cuda::std::numeric_limits<T>::infinity()
                              : cuda::std::numeric_limits<T>::lowest();
    return T(0);
}

template <int M, class T>
__device__ __forceinline__ T combine(T a, T b) {
    if (M == MMIN) return b < a ? b : a;
    if (M == MMAX) return b > a ? b : a;
    return a + b;
}

// 16-byte moves of two consecutive 8-byte values (16-byte aligned)
template <class T>
__device__ __forceinline__ void ld2(const T *p, T &a, T &b) {
    if constexpr (cuda::std::is_same_v<T, double>) {
        const double2 v = *reinterpret_cast<const double2 *>(p);
        a = v.x;
        b = v.y;
    } else {
        const longlong2 v = *reinterpret_cast<const longlong2 *>(p);
        a = T(v.x);
        b = T(v.y);
    }
}
template <class T>
__device__ __forceinline__ void st2(T *p, T a, T b) {
    if constexpr (cuda::std::is_same_v<T, double>) *reinterpret_cast<double2 *>(p) = make_double2(a, b);
    else *reinterpret_cast<longlong2 *>(p) = make_longlong2(static_cast<long long>(a), static_cast<long long>(b));
}

// ---- per-argument slot ------------------------------------------------------------
// MODE ST_NONE: views into HBM; ST_REG: indirect INC staged in registers and
// applied to HBM in colour phases; ST_GATHER: INC and WRITE indirect args
// staged in registers (zero-initialised); the target-centric kernels keep one.
enum : int { ST_NONE = 0, ST_REG = 1, ST_GATHER = 2 };

template <class A, int MODE, int L>
struct Slot {
    using T = typename A::type;
    static constexpr bool is_global = A::kind == KG;
    static constexpr bool is_reduce = is_global && A::mode != MR;
    static constexpr bool is_inc = A::kind == KI && A::mode == MINC;
    static constexpr bool is_ind_write = A::kind == KI && A::mode == MW;
    static constexpr bool staged = (is_inc && MODE != ST_NONE) || is_reduce ||
                                   (is_ind_write && MODE == ST_GATHER);

    T acc[staged ? A::dim : 1];
    T bak[is_reduce ? A::dim : 1];
    T *ptr;          // element base pointer
    int64_t sc;

    __device__ __forceinline__ void init_global(const LaunchParams &p, int i) {
        if constexpr (is_reduce) {
#pragma unroll
            for (int c = 0; c < A::dim; ++c) acc[c] = reduce_identity<T, A::mode>();
        } else if constexpr (is_global) {
            ptr = static_cast<T *>(p.a[i].data);
            sc = 1;
        }
    }
    __device__ __forceinline__ void bind(const ArgRt &r, int64_t t) {
        ptr = static_cast<T *>(r.data) + base_of<A, L>(r, t);
        sc = sc_of<A, L>(r);
        if constexpr (staged) {
#pragma unroll
            for (int c = 0; c < A::dim; ++c) acc[c] = T(0);
        }
    }
    __device__ __forceinline__ void init_elem(const LaunchParams &p, int i, int64_t e) {
        if constexpr (!is_global) {
            const ArgRt &r = p.a[i];
            bind(r, A::kind == KI ? int64_t(__ldg(r.map + e)) : e);
        }
    }
    // pass-1 element record (PFoldParams::rec): indirect targets from the record
    __device__ __forceinline__ void init_elem_rec(const LaunchParams &p, int i, int64_t e, const int32_t *rk) {
        if constexpr (!is_global) bind(p.a[i], A::kind == KI ? int64_t(__ldg(rk + p.pf.rcol[i])) : e);
    }
    // the same with the record column known at compile time (functor trait rec_cols)
    template <int COL>
    __device__ __forceinline__ void init_elem_rec_col(const LaunchParams &p, int i, int64_t e, const int32_t *rk) {
        if constexpr (!is_global) bind(p.a[i], A::kind == KI ? int64_t(__ldg(rk + COL)) : e);
    }
    __device__ __forceinline__ auto view() {
        if constexpr (staged) {
            return static_cast<T *>(acc);
        } else if constexpr (A::mode == MR && MODE == ST_GATHER && !is_global) {
            if constexpr (L == 1) return RefNCA<T>{ptr};
            else return RefNC<T>{ptr, sc};
        } else if constexpr (L == 1) {
            if constexpr (A::mode == MR) return RefA<const T>{ptr};
            else return RefA<T>{ptr};
        } else if constexpr (A::mode == MR) {
            return Ref<const T>{ptr, sc};
        } else {
            return Ref<T>{ptr, sc};
        }
    }
    __device__ __forceinline__ void apply_staged() {
        if constexpr (staged && !is_global) {
            // the components are distinct addresses: issue every load before
            // the first store so the read-modify-writes overlap
            T old[A::dim];
#pragma unroll
            for (int c = 0; c < A::dim; ++c) old[c] = ptr[c * sc];
#pragma unroll
            for (int c = 0; c < A::dim; ++c) ptr[c * sc] = old[c] + acc[c];
        }
    }
    __device__ __forceinline__ void backup() {
        if constexpr (is_reduce) {
#pragma unroll
            for (int c = 0; c < A::dim; ++c) bak[c] = acc[c];
        }
    }
    __device__ __forceinline__ void restore() {
        if constexpr (is_reduce) {
#pragma unroll
            for (int c = 0; c < A::dim; ++c) acc[c] = bak[c];
        }
    }
};

template <class T, int M>
__device__ __forceinline__ T block_reduce(T v, T *smem_t) {
    // warp shuffle, then warp leaders through shared memory
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = combine<M>(v, __shfl_down_sync(full, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) smem_t[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < nw ? smem_t[lane] : reduce_identity<T, M>();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = combine<M>(v, __shfl_down_sync(full, v, o));
    }
    return v;   // valid in thread 0
}

template <int MM, class... As>
struct ModeIndex {
    // position of argument I among the indirect arguments of mode MM (-1 if not one)
    template <size_t I>
    __host__ __device__ static constexpr int of() {
        constexpr bool in[] = {(As::kind == KI && As::mode == MM)...};
        if (!in[I]) return -1;
        int p = 0;
        for (size_t j = 0; j < I; ++j) p += in[j] ? 1 : 0;
        return p;
    }
    template <size_t I>
    __host__ __device__ static constexpr int first() {
        constexpr bool in[] = {(As::kind == KI && As::mode == MM)...};
        for (size_t j = 0; j < sizeof...(As); ++j)
            if (in[j]) return int(j);
        return -1;
    }
};
template <class... As>
using IncIndex = ModeIndex<MINC, As...>;

// Functor trait rec_cols: record column of every argument for the loops the
// functor is written for (-1: not indirect).  The host uses the LP = 2
// kernels (compile-time columns) only when a loop's records match it.
template <class F, class = void>
struct HasRecCols : cuda::std::false_type {};
template <class F>
struct HasRecCols<F, cuda::std::void_t<decltype(F::rec_cols)>> : cuda::std::true_type {};
template <class F>
__host__ __device__ constexpr int rec_ncol() {       // record width the trait implies
    if constexpr (HasRecCols<F>::value) {
        int m = 0;
        for (int i = 0; i < int(sizeof(F::rec_cols) / sizeof(F::rec_cols[0])); ++i)
            m = F::rec_cols[i] + 1 > m ? F::rec_cols[i] + 1 : m;
        return m;
    } else {
        return 0;
    }
}
// record width of a launch: compile-time with the trait's columns (LP 2)
template <class F, int LP>
__device__ __forceinline__ int64_t rec_width(const LaunchParams &p) {
    if constexpr (LP == 2) return rec_ncol<F>();
    else return p.pf.ncol;
}
template <class F, int I, class = void>
struct RecCol : cuda::std::integral_constant<int, 0> {};
template <class F, int I>
struct RecCol<F, I, cuda::std::enable_if_t<HasRecCols<F>::value>>
    : cuda::std::integral_constant<int, (F::rec_cols[I] < 0 ? 0 : F::rec_cols[I])> {};

template <class F, int MODE, int LP, class... As>
struct Engine {
    using Slots = cuda::std::tuple<Slot<As, MODE, lay_of<As, LP>()>...>;
    static constexpr int N = sizeof...(As);

    template <size_t... Is>
    __device__ __forceinline__ static void init_globals(Slots &s, const LaunchParams &p,
                                                        cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).init_global(p, int(Is)), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void init_elem(Slots &s, const LaunchParams &p, int64_t e,
                                                     cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).init_elem(p, int(Is), e), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void init_elem_rec(Slots &s, const LaunchParams &p, int64_t e,
                                                         const int32_t *rk, cuda::std::index_sequence<Is...>) {
        if constexpr (LP == 2)      // record columns from the functor (host-validated per loop)
            (cuda::std::get<Is>(s).template init_elem_rec_col<RecCol<F, int(Is)>::value>(p, int(Is), e, rk), ...);
        else
            (cuda::std::get<Is>(s).init_elem_rec(p, int(Is), e, rk), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void call_raw(Slots &s, const LaunchParams &p,
                                                    cuda::std::index_sequence<Is...>) {
        F::apply(p.k, cuda::std::get<Is>(s).view()...);
    }
    // apply the functor; contributions of elements past p.rlim (multi-GPU exec
    // halo) to global reductions are discarded (reference executor.py:519-524)
    template <size_t... Is>
    __device__ __forceinline__ static void call(Slots &s, const LaunchParams &p, int64_t e,
                                                cuda::std::index_sequence<Is...> idx) {
        if constexpr (has_reduce) {
            if (e >= p.rlim) {
                (cuda::std::get<Is>(s).backup(), ...);
                call_raw(s, p, idx);
                (cuda::std::get<Is>(s).restore(), ...);
                return;
            }
        }
        call_raw(s, p, idx);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void backup_all(Slots &s, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).backup(), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void restore_all(Slots &s, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).restore(), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void apply_staged(Slots &s, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).apply_staged(), ...);
    }
    // target-centric schedules, argument at position `a` among the mode-MM
    // indirect args: OP 0: run += its increments (INC); 1: its registers = run
    // (WRITE, before the call: the kernel sees the target's current value);
    // 2: run = its registers
    template <int MM, int OP, int DG, class TG, size_t... Is>
    __device__ __forceinline__ static void gather_op(Slots &s, int a, TG *run,
                                                     cuda::std::index_sequence<Is...>) {
        (gather_op_one<Is, MM, OP, DG>(s, a, run), ...);
    }
    template <size_t I, int MM, int OP, int DG, class TG>
    __device__ __forceinline__ static void gather_op_one(Slots &s, int a, TG *run) {
        using A = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>;
        if constexpr (A::kind == KI && A::mode == MM) {
            constexpr int pos = ModeIndex<MM, As...>::template of<I>();
            if (a == pos) {
                auto &acc = cuda::std::get<I>(s).acc;
#pragma unroll
                for (int c = 0; c < DG; ++c) {
                    if constexpr (OP == 0) run[c] += acc[c];
                    else if constexpr (OP == 1) acc[c] = run[c];
                    else run[c] = acc[c];
                }
            }
        }
    }
    // primary fold: INC arguments at positions >= 1 -> the element's slots;
    // the element's secondary increments go to the rows of the targets'
    // secondary CSR (slotpos[e][pos-1]), so pass 2 reads each target's rows
    // contiguously
    template <int DGP, size_t... Is>
    __device__ __forceinline__ static void stage_rest(Slots &s, void *slots, const int32_t *slotpos,
                                                      cuda::std::index_sequence<Is...>) {
        (stage_rest_one<Is, DGP>(s, slots, slotpos), ...);
    }
    template <size_t I, int DGP>
    __device__ __forceinline__ static void stage_rest_one(Slots &s, void *slots, const int32_t *slotpos) {
        using A = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>;
        if constexpr (A::kind == KI && A::mode == MINC) {
            constexpr int pos = IncIndex<As...>::template of<I>();
            if constexpr (pos >= 1) {
                using T = typename A::type;
                T *dst = static_cast<T *>(slots) + int64_t(__ldg(slotpos + pos - 1)) * DGP;
                if constexpr (A::dim % 2 == 0 && DGP % 2 == 0 && cuda::std::is_same_v<T, double>) {
#pragma unroll
                    for (int c = 0; c < A::dim; c += 2)
                        __stcg(reinterpret_cast<double2 *>(dst + c),
                               make_double2(cuda::std::get<I>(s).acc[c], cuda::std::get<I>(s).acc[c + 1]));
                } else {
#pragma unroll
                    for (int c = 0; c < A::dim; ++c) __stcg(dst + c, cuda::std::get<I>(s).acc[c]);
                }
            }
        }
    }
    template <size_t I>
    __device__ __forceinline__ static void reduce_one(Slots &s, const LaunchParams &p, int32_t b,
                                                      double *smem) {
        using S = cuda::std::tuple_element_t<I, Slots>;
        if constexpr (S::is_reduce) {
            using T = typename S::T;
            constexpr int M = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>::mode;
            constexpr int D = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>::dim;
#pragma unroll 1
            for (int c = 0; c < D; ++c) {
                T v = block_reduce<T, M>(cuda::std::get<I>(s).acc[c], reinterpret_cast<T *>(smem));
                if (threadIdx.x == 0) static_cast<T *>(p.part[I])[int64_t(b) * D + c] = v;
            }
        }
    }
    template <size_t... Is>
    __device__ __forceinline__ static void reduce_all(Slots &s, const LaunchParams &p, int32_t b,
                                                      double *smem, cuda::std::index_sequence<Is...>) {
        (reduce_one<Is>(s, p, b, smem), ...);
    }
    static constexpr bool has_reduce = ((As::kind == KG && As::mode != MR) || ...);

    // Last-CTA combine of a single-launch schedule: every CTA, after storing
    // its partials, takes a ticket; the CTA that arrives last folds all
    // gridDim.x partials onto the global exactly as k_combine would (same
    // strided accumulation and block tree over 256 threads, so the result is
    // bitwise k_combine's) and resets the ticket for the next launch or graph
    // replay.  Saves the combine kernel (and its graph node) per reduction loop.
    template <size_t I>
    __device__ __forceinline__ static void fold_one(const LaunchParams &p, double *smem) {
        using S = cuda::std::tuple_element_t<I, Slots>;
        if constexpr (S::is_reduce) {
            using T = typename S::T;
            constexpr int M = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>::mode;
            constexpr int D = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>::dim;
            T *g = static_cast<T *>(p.a[I].data);
            const T *part = static_cast<const T *>(p.part[I]);
#pragma unroll 1
            for (int c = 0; c < D; ++c) {
                T v = reduce_identity<T, M>();
                for (int64_t i = threadIdx.x; i < int64_t(gridDim.x); i += blockDim.x)
                    v = combine<M>(v, __ldcg(part + i * D + c));
                v = block_reduce<T, M>(v, reinterpret_cast<T *>(smem));
                if (threadIdx.x == 0) g[c] = combine<M>(g[c], v);
                __syncthreads();
            }
        }
    }
    template <size_t... Is>
    __device__ __forceinline__ static void finish_reduce(const LaunchParams &p, double *smem,
                                                         cuda::std::index_sequence<Is...>) {
        if (!p.ticket) return;
        __shared__ unsigned last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();                                   // this CTA's partials before its ticket
            last = atomicAdd(p.ticket, 1u) == gridDim.x - 1u;
        }
        __syncthreads();
        if (!last) return;
        __threadfence();
        (fold_one<Is>(p, smem), ...);
        if (threadIdx.x == 0) *p.ticket = 0u;
    }
};

// ---- direct loops -----------------------------------------------------------------
// Generic layouts: one element per thread, persistent grid striding over the
// elements; one reduction partial per CTA (folded in CTA order by k_combine).
template <class F, class... As>
__device__ __forceinline__ void run_direct(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_NONE, 0, As...>;
    __shared__ double smem[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    typename E::Slots s;
    E::init_globals(s, p, idx);
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < p.n;
         e += int64_t(gridDim.x) * blockDim.x) {
        E::init_elem(s, p, e, idx);
        E::call(s, p, e, idx);
    }
    if constexpr (E::has_reduce) {
        E::reduce_all(s, p, blockIdx.x, smem, idx);
        E::finish_reduce(p, smem, idx);
    }
}

// Direct rows of the two elements a vectorised thread owns: READ/RW/INC rows
// are loaded with 16-byte loads, WRITE/RW/INC rows stored with 16-byte stores
// (a WRITE row is loaded first unless the functor declares dense_writes —
// every component of a direct WRITE argument written, OP2's OP_WRITE).
template <class F, class = void>
struct DenseWrites : cuda::std::false_type {};
template <class F>
struct DenseWrites<F, cuda::std::void_t<decltype(F::dense_writes)>> : cuda::std::bool_constant<F::dense_writes> {};
template <class F>
__host__ __device__ constexpr bool dense_writes() { return DenseWrites<F>::value; }
// write_only: every component of every indirect WRITE argument is written and
// none is read (OP2's OP_WRITE taken literally): a target's final value is
// the one its last incidence in serial order writes
template <class F, class = void>
struct WriteOnly : cuda::std::false_type {};
template <class F>
struct WriteOnly<F, cuda::std::void_t<decltype(F::write_only)>> : cuda::std::bool_constant<F::write_only> {};

template <class A, class F, int LP>
struct DirRows {
    static constexpr bool on = A::kind == KD;
    static constexpr int L = lay_of<A, LP>();
    using T = typename A::type;
    T v[on ? 2 : 1][on ? A::dim : 1];
    // element e0 (even) and e0 + 1 (when two): 16-byte aligned pairs
    __device__ __forceinline__ void load(const ArgRt &r, int64_t e0, bool two) {
        if constexpr (on) {
            if constexpr (A::mode == MW && dense_writes<F>()) return;
            const T *b = static_cast<const T *>(r.data);
            if (!two) {
#pragma unroll
                for (int c = 0; c < A::dim; ++c) v[0][c] = b[base_of<A, L>(r, e0) + c * sc_of<A, L>(r)];
                return;
            }
            if constexpr (L == 1) {             // AOS: the pair's rows are 2*dim consecutive values
                T f[2 * A::dim];
#pragma unroll
                for (int k = 0; k < A::dim; ++k) ld2(b + e0 * A::dim + 2 * k, f[2 * k], f[2 * k + 1]);
#pragma unroll
                for (int c = 0; c < A::dim; ++c) {
                    v[0][c] = f[c];
                    v[1][c] = f[A::dim + c];
                }
            } else {                            // SOA: one pair per component
                const T *bb = b + base_of<A, L>(r, e0);
#pragma unroll
                for (int c = 0; c < A::dim; ++c) ld2(bb + c * sc_of<A, L>(r), v[0][c], v[1][c]);
            }
        }
    }
    __device__ __forceinline__ void store(const ArgRt &r, int64_t e0, bool two) {
        if constexpr (on && A::mode != MR) {
            T *b = static_cast<T *>(r.data);
            if (!two) {
#pragma unroll
                for (int c = 0; c < A::dim; ++c) b[base_of<A, L>(r, e0) + c * sc_of<A, L>(r)] = v[0][c];
                return;
            }
            if constexpr (L == 1) {
                T f[2 * A::dim];
#pragma unroll
                for (int c = 0; c < A::dim; ++c) {
                    f[c] = v[0][c];
                    f[A::dim + c] = v[1][c];
                }
#pragma unroll
                for (int k = 0; k < A::dim; ++k) st2(b + e0 * A::dim + 2 * k, f[2 * k], f[2 * k + 1]);
            } else {
                T *bb = b + base_of<A, L>(r, e0);
#pragma unroll
                for (int c = 0; c < A::dim; ++c) st2(bb + c * sc_of<A, L>(r), v[0][c], v[1][c]);
            }
        }
    }
};

template <class F, class... As>
struct DirectVec {
    using E = Engine<F, ST_NONE, 1, As...>;
    using Rows = cuda::std::tuple<DirRows<As, F, 1>...>;

    template <size_t I>
    __device__ __forceinline__ static auto view(typename E::Slots &s, Rows &rows, int k) {
        using A = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>;
        if constexpr (A::kind == KD) {
            using T = typename A::type;
            if constexpr (A::mode == MR) return static_cast<const T *>(cuda::std::get<I>(rows).v[k]);
            else return static_cast<T *>(cuda::std::get<I>(rows).v[k]);
        } else {
            return cuda::std::get<I>(s).view();
        }
    }
    template <size_t... Is>
    __device__ __forceinline__ static void call(typename E::Slots &s, Rows &rows, const LaunchParams &p,
                                                int64_t e, int k, cuda::std::index_sequence<Is...>) {
        if constexpr (E::has_reduce) {
            if (e >= p.rlim) {
                (cuda::std::get<Is>(s).backup(), ...);
                F::apply(p.k, view<Is>(s, rows, k)...);
                (cuda::std::get<Is>(s).restore(), ...);
                return;
            }
        }
        F::apply(p.k, view<Is>(s, rows, k)...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void load(Rows &rows, const LaunchParams &p, int64_t e0, bool two,
                                                cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(rows).load(p.a[Is], e0, two), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void store(Rows &rows, const LaunchParams &p, int64_t e0, bool two,
                                                 cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(rows).store(p.a[Is], e0, two), ...);
    }
};

// Reference auto-SOA layout (LP = 1, 16-byte aligned rows and even SOA
// pitch): each thread owns elements e0 = 2k and e0 + 1, moves their direct
// rows with 16-byte accesses and applies the functor to both in order.
template <class F, class... As>
__device__ __forceinline__ void run_direct_vec(const LaunchParams &p, Sig<As...>) {
    using DV = DirectVec<F, As...>;
    using E = typename DV::E;
    __shared__ double smem[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    typename E::Slots s;
    E::init_globals(s, p, idx);
    for (int64_t e0 = 2 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x); e0 < p.n;
         e0 += 2 * int64_t(gridDim.x) * blockDim.x) {
        const bool two = e0 + 1 < p.n;
        typename DV::Rows rows;
        DV::load(rows, p, e0, two, idx);
        E::init_elem(s, p, e0, idx);
        DV::call(s, rows, p, e0, 0, idx);
        if (two) {
            E::init_elem(s, p, e0 + 1, idx);
            DV::call(s, rows, p, e0 + 1, 1, idx);
        }
        DV::store(rows, p, e0, two, idx);
    }
    if constexpr (E::has_reduce) {
        E::reduce_all(s, p, blockIdx.x, smem, idx);
        E::finish_reduce(p, smem, idx);
    }
}

// ---- colour schedules (reference plan: run_threads, general indirect writes) --------
template <class F, class... As>
__device__ __forceinline__ void run_staged(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_REG, 0, As...>;
    __shared__ double smem[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    const int32_t b = p.blocks[blockIdx.x];
    const int64_t e = int64_t(b) * p.bs + threadIdx.x;
    const int64_t hi = int64_t(b) * p.bs + p.bs < p.n ? int64_t(b) * p.bs + p.bs : p.n;
    const bool active = threadIdx.x < p.bs && e < hi;
    const int ncol = p.encol[b];
    const int mine = active ? int(p.ecol[e]) : -1;
    typename E::Slots s;
    E::init_globals(s, p, idx);
    if (active) {
        E::init_elem(s, p, e, idx);
        E::call(s, p, e, idx);
    }
    if (ncol == 1) {
        if (active) E::apply_staged(s, idx);
    } else {
        for (int c = 0; c < ncol; ++c) {
            if (mine == c) E::apply_staged(s, idx);
            __syncthreads();
        }
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, b, smem, idx);
}

template <class F, class... As>
__device__ __forceinline__ void run_phased(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_NONE, 0, As...>;
    __shared__ double smem[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    const int32_t b = p.blocks[blockIdx.x];
    const int64_t lo = int64_t(b) * p.bs, hi = lo + p.bs < p.n ? lo + p.bs : p.n;
    const int ncol = p.encol[b];
    typename E::Slots s;
    E::init_globals(s, p, idx);
    for (int c = 0; c < ncol; ++c) {
        for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
            if (int(p.ecol[e]) != c) continue;
            E::init_elem(s, p, e, idx);
            E::call(s, p, e, idx);
        }
        __syncthreads();
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, b, smem, idx);
}

// ---- target-centric ("gather") schedule ----------------------------------------------
// For loops whose indirect writes all go to one dat with one mode — INC, or
// WRITE — and that write no direct argument: one thread per target element
// re-evaluates the kernel for every (element, argument) incidence of that
// target, in serial order, and keeps only that argument's effect on a running
// value that starts from the target's current value: INC adds the increment,
// WRITE replaces the value (the kernel is handed the running value in that
// argument, so it sees what the serial order would show it).  The target's
// final value is therefore exactly the serial one.  No colours, no shared
// memory, no atomics.  Global reductions count each element once (on its
// incidence through the first such argument).
template <class F, int LP, class... As>
__device__ __forceinline__ void run_gather(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_GATHER, LP, As...>;
    constexpr bool has_inc = ((As::kind == KI && As::mode == MINC) || ...);
    constexpr int MM = has_inc ? MINC : MW;
    constexpr int G = ModeIndex<MM, As...>::template first<0>();
    static_assert(G >= 0, "gather schedule needs an INC or WRITE indirect argument");
    using AG = cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>;
    using TG = typename AG::type;
    constexpr int DG = AG::dim;
    constexpr int LG = lay_of<AG, LP>();
    __shared__ double red[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    typename E::Slots s;
    E::init_globals(s, p, idx);
    const ArgRt &rg = p.a[G];
    const int64_t gsc = sc_of<AG, LG>(rg);
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
         t - threadIdx.x < p.g_ntargets; t += int64_t(gridDim.x) * blockDim.x) {
        if (t >= p.g_ntargets) continue;
        const int64_t tg = p.g_tlist ? int64_t(__ldg(p.g_tlist + t)) : t;
        TG *dst = static_cast<TG *>(rg.data) + base_of<AG, LG>(rg, tg);
        const int32_t seg = (MM == MINC && p.g_seg) ? __ldg(p.g_seg + t) : -1;
        TG run[DG];
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] = seg < 0 ? dst[c * gsc] : TG(0);
        // write-only WRITE loops without reductions: only the last incidence
        // in serial order decides the target's value
        constexpr bool last_only = MM == MW && !E::has_reduce && WriteOnly<F>::value;
        const int kb = __ldg(p.g_off + t), ke = __ldg(p.g_off + t + 1);
#ifndef ML_GATHER_UNROLL
#define ML_GATHER_UNROLL 4   // incidence loop unroll (1 / 2 / 3 / 4 / 6 / 8 measured; 4 best)
#endif
        constexpr int kUnroll = ML_GATHER_UNROLL;
#pragma unroll kUnroll
        for (int k = last_only && ke > kb ? ke - 1 : kb; k < ke; ++k) {
            const int64_t e = __ldg(p.g_elem + k);
            const int a = __ldg(p.g_pos + k);
#ifndef ML_GATHER_REC
#define ML_GATHER_REC 1      // per-incidence map records (grad_edge 0.1048 -> 0.1008 ms)
#endif
            if constexpr (ML_GATHER_REC)
                E::init_elem_rec(s, p, e, p.pf.rec + int64_t(k) * rec_width<F, LP>(p), idx);
            else
                E::init_elem(s, p, e, idx);
            if constexpr (MM == MW) E::template gather_op<MW, 1, DG>(s, a, run, idx);
            if constexpr (E::has_reduce) {
                if (a != 0 || e >= p.rlim) {
                    E::backup_all(s, idx);
                    E::call_raw(s, p, idx);
                    E::restore_all(s, idx);
                } else {
                    E::call_raw(s, p, idx);
                }
            } else {
                E::call_raw(s, p, idx);
            }
            E::template gather_op<MM, MM == MINC ? 0 : 2, DG>(s, a, run, idx);
        }
        if (seg >= 0) {
            TG *part = static_cast<TG *>(p.g_part) + int64_t(seg) * DG;
#pragma unroll
            for (int c = 0; c < DG; ++c) part[c] = run[c];
        } else {
#pragma unroll
            for (int c = 0; c < DG; ++c) dst[c * gsc] = run[c];
        }
    }
    if constexpr (E::has_reduce) {
        E::reduce_all(s, p, blockIdx.x, red, idx);
        E::finish_reduce(p, red, idx);
    }
}

// Hub targets of the gather schedule: value + the partial of each of its
// rows, in row (= element) order.
template <class T, int DG>
__global__ void __launch_bounds__(256) k_gather_hubs(const __grid_constant__ LaunchParams p, int ga) {
    pdl_wait();
    const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (h >= p.g_nhub) return;
    const ArgRt &rg = p.a[ga];
    T *dst = static_cast<T *>(rg.data) + elem_base(rg, int64_t(__ldg(p.g_hub_tl + h)));
    const T *part = static_cast<const T *>(p.g_part);
    T run[DG];
#pragma unroll
    for (int c = 0; c < DG; ++c) run[c] = dst[c * rg.sc];
    for (int q = __ldg(p.g_hub_off + h), qe = __ldg(p.g_hub_off + h + 1); q < qe; ++q)
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] += part[int64_t(q) * DG + c];
#pragma unroll
    for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
}

// ---- primary fold ---------------------------------------------------------------------
// Pass 1 (see PFoldParams): a persistent grid strides over the targets; thread
// t evaluates, in element order, every element whose first INC argument
// targets it — each element exactly once in the whole launch, its
// neighbours' rows read once per element instead of once per incidence —
// adds that argument's increments to a running value that starts from the
// target's current value, and stores the other INC arguments' increments in
// the element's slots.  Global reductions count every element here (once).
// Pass 2 (k_pfold_rest_w) adds each target's slots in element order.  Per
// target the result is value + primary increments + secondary increments:
// deterministic, within rounding of the serial order.
template <class TG, int DG>
struct PFoldShape {
    static constexpr int DGP = (DG + 1) / 2 * 2;   // slot rows of whole 16-byte pairs
};

template <class F, int LP, class... As>
__device__ __forceinline__ void run_pfold1(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_GATHER, LP, As...>;
    constexpr int G = IncIndex<As...>::template first<0>();
    static_assert(G >= 0, "primary fold needs an INC argument");
    using AG = cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>;
    using TG = typename AG::type;
    constexpr int DG = AG::dim;
    constexpr int LG = lay_of<AG, LP>();
    constexpr int NW = ((As::kind == KI && As::mode == MINC) + ...);
    constexpr int DGP = PFoldShape<TG, DG>::DGP;
    __shared__ double red[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    typename E::Slots s;
    E::init_globals(s, p, idx);
    const PFoldParams &pf = p.pf;
    const ArgRt &rg = p.a[G];
    const int64_t gsc = sc_of<AG, LG>(rg);
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t - threadIdx.x < pf.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        if (t >= pf.n1) continue;
        const int64_t tg = pf.tl1 ? int64_t(__ldg(pf.tl1 + t)) : t;
        TG *dst = static_cast<TG *>(rg.data) + base_of<AG, LG>(rg, tg);
        const int32_t seg = pf.seg1 ? __ldg(pf.seg1 + t) : -1;
        TG run[DG];
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] = seg < 0 ? dst[c * gsc] : TG(0);
        for (int k = __ldg(pf.off1 + t), ke = __ldg(pf.off1 + t + 1); k < ke; ++k) {
            const int64_t e = __ldg(pf.elem1 + k);
            // per-incidence records (no runtime switch: a branch here costs
            // more than the records save — fused flux loop 0.282 -> 0.272 ms)
            E::init_elem_rec(s, p, e, pf.rec + int64_t(k) * rec_width<F, LP>(p), idx);
            E::call(s, p, e, idx);
            E::template gather_op<MINC, 0, DG>(s, 0, run, idx);
            if constexpr (NW > 1)
                E::template stage_rest<DGP>(s, pf.slots, pf.slotpos + e * int64_t(NW - 1), idx);
        }
        if (seg >= 0) {
            TG *part = static_cast<TG *>(pf.part1) + int64_t(seg) * DG;
#pragma unroll
            for (int c = 0; c < DG; ++c) part[c] = run[c];
        } else {
#pragma unroll
            for (int c = 0; c < DG; ++c) dst[c * gsc] = run[c];
        }
    }
    if constexpr (E::has_reduce) {
        E::reduce_all(s, p, blockIdx.x, red, idx);
        E::finish_reduce(p, red, idx);
    }
}

// Pass 2, warp-cooperative: a warp owns 32 consecutive pass-2 rows, whose
// slots are one contiguous range; the lanes copy it through shared memory in
// coalesced 16-byte chunks, then each lane adds its own rows in order, with
// full-sector DRAM reads.
template <class T, int DG>
__global__ void __launch_bounds__(256) k_pfold_rest_w(const __grid_constant__ LaunchParams p, int ga) {
    pdl_wait();
    constexpr int DGP = PFoldShape<T, DG>::DGP;
    constexpr int CH = 5632 / int(DGP * sizeof(T));          // slot rows per chunk and warp (5.5 KB)
    __shared__ __align__(16) T buf[8][CH * DGP];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const PFoldParams &pf = p.pf;
    const ArgRt &rg = p.a[ga];
    const uint4 *slots = static_cast<const uint4 *>(pf.slots);
    for (int64_t t0 = (int64_t(blockIdx.x) * 8 + w) * 32; t0 < pf.n2; t0 += int64_t(gridDim.x) * 256) {
        const int64_t t = t0 + lane;
        const bool act = t < pf.n2;
        const int64_t te = t0 + 32 < pf.n2 ? t0 + 32 : pf.n2;
        const int wk0 = __ldg(pf.off2 + t0), wk1 = __ldg(pf.off2 + te);
        int k0 = 0, k1 = 0;
        T *dst = nullptr;
        int32_t seg = -1;
        T run[DG];
        if (act) {
            k0 = __ldg(pf.off2 + t);
            k1 = __ldg(pf.off2 + t + 1);
            const int64_t tg = pf.tl2 ? int64_t(__ldg(pf.tl2 + t)) : t;
            dst = static_cast<T *>(rg.data) + elem_base(rg, tg);
            seg = pf.seg2 ? __ldg(pf.seg2 + t) : -1;
#pragma unroll
            for (int c = 0; c < DG; ++c) run[c] = seg < 0 ? dst[c * rg.sc] : T(0);
        }
        for (int c0 = wk0; c0 < wk1; c0 += CH) {
            const int n = wk1 - c0 < CH ? wk1 - c0 : CH;
            const uint4 *src = slots + int64_t(c0) * (DGP * sizeof(T) / 16);
            uint4 *dstb = reinterpret_cast<uint4 *>(buf[w]);
            for (int i = lane; i < n * int(DGP * sizeof(T) / 16); i += 32) dstb[i] = __ldcs(src + i);
            __syncwarp();
            if (act) {
                const int a = k0 > c0 ? k0 : c0, b = k1 < c0 + n ? k1 : c0 + n;
                for (int k = a; k < b; ++k) {
#pragma unroll
                    for (int c = 0; c < DG; ++c) run[c] += buf[w][(k - c0) * DGP + c];
                }
            }
            __syncwarp();
        }
        if (act) {
            if (seg >= 0) {
                T *part = static_cast<T *>(pf.part2) + int64_t(seg) * DG;
#pragma unroll
                for (int c = 0; c < DG; ++c) part[c] = run[c];
            } else {
#pragma unroll
                for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
            }
        }
    }
}

// Pass 2 with Blackwell bulk copies: the same warp-per-32-rows split, but the
// warp's slot range moves global -> shared by the TMA engine
// (cp.async.bulk, completion on an mbarrier) in chunks of up to CH rows,
// double-buffered: lane 0 issues chunk i+1 before the lanes wait for and fold
// chunk i, so the copy overlaps the fold and the next group's target loads.
// Chunks follow the warp's groups in order, so one chunk never spans two
// groups; a group without slots issues nothing.
#ifndef ML_PF2_TMA
#define ML_PF2_TMA 1
#endif
#ifndef ML_PF2_CHUNK_BYTES
#define ML_PF2_CHUNK_BYTES 2816   // per buffer and warp; two buffers = the 5.5 KB of k_pfold_rest_w
#endif
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

template <class T, int DG>
__global__ void __launch_bounds__(256) k_pfold_rest_tma(const __grid_constant__ LaunchParams p, int ga) {
    constexpr int DGP = PFoldShape<T, DG>::DGP;
    constexpr int RB = int(DGP * sizeof(T));                  // bytes per slot row (multiple of 16)
    constexpr int CH = ML_PF2_CHUNK_BYTES / RB;               // slot rows per buffer
    static_assert(RB % 16 == 0 && CH > 0, "bulk copies move whole 16-byte units");
    __shared__ __align__(128) T buf[8][2][CH * DGP];
    __shared__ __align__(8) uint64_t bar[8][2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        mbar_init(&bar[w][0], 1);
        mbar_init(&bar[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    pdl_wait();
    const PFoldParams &pf = p.pf;
    const ArgRt &rg = p.a[ga];
    const char *slots = static_cast<const char *>(pf.slots);
    const int64_t n2 = pf.n2, stride = int64_t(gridDim.x) * 256;
    int64_t ct = (int64_t(blockIdx.x) * 8 + w) * 32;
    if (ct >= n2) return;
    auto group_end = [&](int64_t t0) { return __ldg(pf.off2 + (t0 + 32 < n2 ? t0 + 32 : n2)); };
    int cc = __ldg(pf.off2 + ct), ce = group_end(ct);        // consumer cursor: group, chunk, group end
    int64_t pt = ct;
    int pc = cc, pe = ce;                                     // producer cursor, one chunk ahead
    auto produce = [&](int b) {
        const int n = pe - pc < CH ? pe - pc : CH;
        if (n > 0 && lane == 0) bulk_g2s(buf[w][b], slots + int64_t(pc) * RB, uint32_t(n * RB), &bar[w][b]);
        pc += CH;
        if (pc >= pe) {
            pt += stride;
            if (pt < n2) {
                pc = __ldg(pf.off2 + pt);
                pe = group_end(pt);
            }
        }
    };
    produce(0);
    uint32_t phase = 0;
    int b = 0;
    bool start = true, act = false;
    int k0 = 0, k1 = 0;
    int32_t seg = -1;
    T *dst = nullptr;
    T run[DG];
    while (ct < n2) {
        if (pt < n2) {
            __syncwarp();
            produce(b ^ 1);
        }
        if (start) {
            const int64_t t = ct + lane;
            act = t < n2;
            if (act) {
                k0 = __ldg(pf.off2 + t);
                k1 = __ldg(pf.off2 + t + 1);
                const int64_t tg = pf.tl2 ? int64_t(__ldg(pf.tl2 + t)) : t;
                dst = static_cast<T *>(rg.data) + elem_base(rg, tg);
                seg = pf.seg2 ? __ldg(pf.seg2 + t) : -1;
#pragma unroll
                for (int c = 0; c < DG; ++c) run[c] = seg < 0 ? dst[c * rg.sc] : T(0);
            }
            start = false;
        }
        const int n = ce - cc < CH ? ce - cc : CH;
        if (n > 0) {
            mbar_wait(&bar[w][b], (phase >> b) & 1u);
            phase ^= 1u << b;
            if (act) {
                const int a = k0 > cc ? k0 : cc, e = k1 < cc + n ? k1 : cc + n;
                for (int k = a; k < e; ++k) {
#pragma unroll
                    for (int c = 0; c < DG; ++c) run[c] += buf[w][b][(k - cc) * DGP + c];
                }
            }
            // the next bulk copy into this buffer is an async-proxy write after
            // these generic-proxy reads
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        cc += CH;
        if (cc >= ce) {
            if (act) {
                if (seg >= 0) {
                    T *part = static_cast<T *>(pf.part2) + int64_t(seg) * DG;
#pragma unroll
                    for (int c = 0; c < DG; ++c) part[c] = run[c];
                } else {
#pragma unroll
                    for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
                }
            }
            ct += stride;
            start = true;
            if (ct < n2) {
                cc = __ldg(pf.off2 + ct);
                ce = group_end(ct);
            }
        }
        b ^= 1;
    }
}

// Hub targets of a split pass (pfold): value + each partial slot in order.
template <class T, int DG>
__global__ void __launch_bounds__(256) k_fold_parts(const __grid_constant__ LaunchParams p, int ga, int64_t nhub,
                                                    const int32_t *hub_tl, const int32_t *hub_off,
                                                    const void *parts) {
    pdl_wait();
    const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (h >= nhub) return;
    const ArgRt &rg = p.a[ga];
    T *dst = static_cast<T *>(rg.data) + elem_base(rg, int64_t(__ldg(hub_tl + h)));
    const T *part = static_cast<const T *>(parts);
    T run[DG];
#pragma unroll
    for (int c = 0; c < DG; ++c) run[c] = dst[c * rg.sc];
    for (int q = __ldg(hub_off + h), qe = __ldg(hub_off + h + 1); q < qe; ++q)
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] += part[int64_t(q) * DG + c];
#pragma unroll
    for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
}

// ---- kernels ------------------------------------------------------------------------
// resident CTAs per SM the direct kernels are compiled for: 1 lets a
// vectorised thread keep both elements' rows in registers (update: ~180);
// capping for 2 or 3 CTAs measured equal or slower (update 0.0549 ms at 1,
// 0.0575 at 3: spills)
#ifndef ML_DIRECT_MINB
#define ML_DIRECT_MINB 1
#endif
#if ML_DIRECT_MINB > 0
#define ML_DIRECT_BOUNDS __launch_bounds__(256, ML_DIRECT_MINB)
#else
#define ML_DIRECT_BOUNDS __launch_bounds__(256)   // no minimum: ptxas picks the register budget
#endif
template <class F, class T, int LP>
__global__ void ML_DIRECT_BOUNDS k_direct(const __grid_constant__ LaunchParams p) {
    pdl_wait();
    if constexpr (LP == 1) run_direct_vec<F>(p, typename F::template sig<T>{});
    else run_direct<F>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_staged(const __grid_constant__ LaunchParams p) {
    run_staged<F>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_phased(const __grid_constant__ LaunchParams p) {
    run_phased<F>(p, typename F::template sig<T>{});
}
template <class F, class T, int LP>
__global__ void __launch_bounds__(256) k_pfold1(const __grid_constant__ LaunchParams p) {
    pdl_wait();
    run_pfold1<F, LP>(p, typename F::template sig<T>{});
}
template <class F, class T, int LP>
__global__ void __launch_bounds__(256) k_gather(const __grid_constant__ LaunchParams p) {
    pdl_wait();
    run_gather<F, LP>(p, typename F::template sig<T>{});
}

// ---- compile-time signature introspection -------------------------------------
template <class S>
struct SigInfo;
template <class... As>
struct SigInfo<Sig<As...>> {
    static constexpr int n = sizeof...(As);
    static void fill(int32_t *kind, int32_t *mode, int32_t *dim, int32_t *dtype) {
        int i = 0;
        ((kind[i] = As::kind, mode[i] = As::mode, dim[i] = As::dim,
          dtype[i] = type_code<typename As::type>(), ++i), ...);
    }
    static constexpr bool ind_write = ((As::kind == KI && As::mode != MR) || ...);
    static constexpr bool ind_write_non_inc = ((As::kind == KI && (As::mode == MW || As::mode == MRW)) || ...);
    static constexpr bool direct_write = ((As::kind == KD && As::mode != MR) || ...);
    static constexpr bool ind_inc = ((As::kind == KI && As::mode == MINC) || ...);
    static constexpr int n_inc = ((As::kind == KI && As::mode == MINC) + ... + 0);
    static constexpr bool ind_w = ((As::kind == KI && As::mode == MW) || ...);
    static constexpr bool ind_rw = ((As::kind == KI && As::mode == MRW) || ...);
    // target-centric schedule: indirect writes of one mode (INC or WRITE), no direct writes
    static constexpr bool gather_ok = ind_write && !ind_rw && !(ind_inc && ind_w) && !direct_write;
    // primary fold: indirect writes all INC (direct writes allowed)
    static constexpr bool fold_ok = ind_inc && !ind_rw && !ind_w;
};

template <class S>
struct FirstInc;
template <class... As>
struct FirstInc<Sig<As...>> {
    static constexpr int value = IncIndex<As...>::template first<0>() < 0 ? 0 : IncIndex<As...>::template first<0>();
    using type = cuda::std::tuple_element_t<value, cuda::std::tuple<As...>>;
};

// ---- registry -------------------------------------------------------------------
using LaunchFn = void (*)(const LaunchParams &, dim3, dim3, size_t, cudaStream_t);

struct FunctorEntry {
    const char *name;
    int32_t dtype;
    int32_t nargs;
    int32_t kind[MAX_ARGS], mode[MAX_ARGS], dim[MAX_ARGS], atype[MAX_ARGS];
    bool ind_write, ind_write_non_inc;
    LaunchFn direct[2], staged, phased;              // [LP]
    LaunchFn gather[3], gather_hubs;                 // target-centric (INC-only or WRITE-only); [2]:
    LaunchFn pfold1[3], pfold2;                      // primary fold (INC-only)   fixed record columns
    int (*direct_occupancy[2])(int threads);
    int (*gather_occupancy[3])();
    int (*pfold_occupancy[3])();
    int32_t nrec_cols;                               // functor trait rec_cols (0: none)
    int8_t rec_cols[MAX_ARGS];
    void (*pfold_hubs)(const LaunchParams &, int64_t nhub, const int32_t *tl, const int32_t *off,
                       const void *parts, cudaStream_t);
    int32_t pfold_dgp, pfold_nslot;
};

void register_functor(const FunctorEntry &e);

template <class F, class T>
struct Registrar {
    template <int LP>
    static void direct(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        launch_k(k_direct<F, T, LP>, g, b, 0, s, p);
    }
    template <int LP>
    static int direct_occupancy(int threads) {
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_direct<F, T, LP>, threads, 0) != cudaSuccess) n = 0;
        return n;
    }
    static void staged(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        k_staged<F, T><<<g, b, 0, s>>>(p);
    }
    static void phased(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        k_phased<F, T><<<g, b, 0, s>>>(p);
    }
    // the target-centric kernels use no shared memory to speak of: the SM's
    // storage goes to L1, where consecutive targets share neighbour rows
    template <class K>
    static void carve_l1(K kernel) {
        static bool once = false;
        if (!once) {
            cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
            once = true;
        }
    }
    template <int LP>
    static void gather(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        carve_l1(k_gather<F, T, LP>);
        launch_k(k_gather<F, T, LP>, g, b, 0, s, p);
    }
    // resident CTAs of 256 threads per SM (sizes the persistent grids)
    template <int LP>
    static int gather_occupancy() {
        static int n = -1;
        if (n < 0) {
            carve_l1(k_gather<F, T, LP>);
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gather<F, T, LP>, 256, 0) != cudaSuccess) n = 0;
        }
        return n;
    }
    static void gather_hubs(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        using S = typename F::template sig<T>;
        using AG = typename FirstInc<S>::type;
        launch_k(k_gather_hubs<typename AG::type, AG::dim>, g, b, 0, s, p, int(FirstInc<S>::value));
    }
    template <int LP>
    static void pfold1(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        carve_l1(k_pfold1<F, T, LP>);
        launch_k(k_pfold1<F, T, LP>, g, b, 0, s, p);
    }
    template <int LP>
    static int pfold_occupancy() {
        static int n = -1;
        if (n < 0) {
            carve_l1(k_pfold1<F, T, LP>);
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_pfold1<F, T, LP>, 256, 0) != cudaSuccess) n = 0;
        }
        return n;
    }
    static void pfold_hubs(const LaunchParams &p, int64_t nhub, const int32_t *tl, const int32_t *off,
                           const void *parts, cudaStream_t s) {
        using S = typename F::template sig<T>;
        using AG = typename FirstInc<S>::type;
        launch_k(k_fold_parts<typename AG::type, AG::dim>, dim3(unsigned((nhub + 255) / 256)), dim3(256), 0, s, p,
                 int(FirstInc<S>::value), nhub, tl, off, parts);
    }
    static void pfold2(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        using S = typename F::template sig<T>;
        using AG = typename FirstInc<S>::type;
        #if ML_PF2_TMA
        launch_k(k_pfold_rest_tma<typename AG::type, AG::dim>, g, b, 0, s, p, int(FirstInc<S>::value));
#else
        launch_k(k_pfold_rest_w<typename AG::type, AG::dim>, g, b, 0, s, p, int(FirstInc<S>::value));
#endif
    }
    explicit Registrar(const char *name) {
        using S = typename F::template sig<T>;
        FunctorEntry e{};
        e.name = name;
        e.dtype = type_code<T>();
        e.nargs = SigInfo<S>::n;
        SigInfo<S>::fill(e.kind, e.mode, e.dim, e.atype);
        e.ind_write = SigInfo<S>::ind_write;
        e.ind_write_non_inc = SigInfo<S>::ind_write_non_inc;
        if constexpr (HasRecCols<F>::value) {
            e.nrec_cols = int32_t(sizeof(F::rec_cols) / sizeof(F::rec_cols[0]));
            for (int i = 0; i < e.nrec_cols && i < MAX_ARGS; ++i) e.rec_cols[i] = int8_t(F::rec_cols[i]);
        }
        if constexpr (!SigInfo<S>::ind_write) {
            e.direct[0] = &direct<0>;
            e.direct[1] = &direct<1>;
            e.direct_occupancy[0] = &direct_occupancy<0>;
            e.direct_occupancy[1] = &direct_occupancy<1>;
        } else {
            e.staged = !SigInfo<S>::ind_write_non_inc ? &staged : nullptr;
            e.phased = &phased;
        }
        if constexpr (SigInfo<S>::fold_ok) {
            e.pfold1[0] = &pfold1<0>;
            e.pfold1[1] = &pfold1<1>;
            e.pfold_occupancy[0] = &pfold_occupancy<0>;
            e.pfold_occupancy[1] = &pfold_occupancy<1>;
            if constexpr (HasRecCols<F>::value) {
                e.pfold1[2] = &pfold1<2>;
                e.pfold_occupancy[2] = &pfold_occupancy<2>;
            }
            e.pfold2 = &pfold2;
            e.pfold_hubs = &pfold_hubs;
            using AG = typename FirstInc<S>::type;
            e.pfold_dgp = PFoldShape<typename AG::type, AG::dim>::DGP;
            e.pfold_nslot = SigInfo<S>::n_inc - 1;
        }
        if constexpr (SigInfo<S>::gather_ok && SigInfo<S>::ind_inc) e.gather_hubs = &gather_hubs;
        if constexpr (SigInfo<S>::gather_ok) {
            e.gather[0] = &gather<0>;
            e.gather[1] = &gather<1>;
            e.gather_occupancy[0] = &gather_occupancy<0>;
            e.gather_occupancy[1] = &gather_occupancy<1>;
            if constexpr (HasRecCols<F>::value) {
                e.gather[2] = &gather<2>;
                e.gather_occupancy[2] = &gather_occupancy<2>;
            }
        }
        register_functor(e);
    }
};

// ---- loop chains -------------------------------------------------------------
// A chain declares that a loop running functor FIRST immediately followed by
// one running SECOND over the same set may execute as one loop of functor
// FUSED: FUSED::first_args[i] / second_args[j] give the fused argument that
// argument i of the first loop / j of the second binds to.  Arguments of the
// two loops that bind to one fused argument must be identical (same dat,
// map, slot and mode) and the loops may share no other written data — the
// executor checks both (chain.py) before fusing.
struct ChainEntry {
    const char *first, *second, *fused;
    int32_t na, nb;
    int32_t apos[MAX_ARGS], bpos[MAX_ARGS];
};
void register_chain(const ChainEntry &c);

template <class F>
struct ChainRegistrar {
    ChainRegistrar(const char *first, const char *second, const char *fused) {
        ChainEntry c{};
        c.first = first;
        c.second = second;
        c.fused = fused;
        c.na = int32_t(sizeof(F::first_args) / sizeof(F::first_args[0]));
        c.nb = int32_t(sizeof(F::second_args) / sizeof(F::second_args[0]));
        for (int i = 0; i < c.na; ++i) c.apos[i] = F::first_args[i];
        for (int i = 0; i < c.nb; ++i) c.bpos[i] = F::second_args[i];
        register_chain(c);
    }
};

#define ML_CAT2(a, b) a##b
#define ML_CAT(a, b) ML_CAT2(a, b)
#define ML_REGISTER(NAME, FUNCTOR, T) \
    static ::ml::Registrar<FUNCTOR, T> ML_CAT(ml_reg_, __COUNTER__)(NAME)
#define ML_REGISTER_CHAIN(FIRST, SECOND, FUSED, FUNCTOR) \
    static ::ml::ChainRegistrar<FUNCTOR> ML_CAT(ml_chain_, __COUNTER__)(FIRST, SECOND, FUSED)

// integer floor division with Python semantics (numpy int64 //)
__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    return (q * b != a && ((a < 0) != (b < 0))) ? q - 1 : q;
}

}  // namespace ml
